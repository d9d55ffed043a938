// runtime.cu -- the C ABI of libtnb200.so (include/tn_b200.h): plan build / load / info, the
// step-program executor and the kernel launches.  Every step of the contraction runs in the
// kernels of kernels.cuh; the host only sequences launches on the caller's stream.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/tn_b200.h"
#include "kernels.cuh"
#include "plan_format.h"
#include "planner.h"

using namespace tnb;

// ============================================================== errors
static thread_local std::string g_err;
static tn_status fail(tn_status s, const std::string& msg) {
  g_err = msg;
  return s;
}
#define CU(call)                                                                      \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess)                                                            \
      return fail(TN_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));      \
  } while (0)

// ============================================================== plan object
struct DevTables {
  StepRec* steps = nullptr;
  LeafRec* leaves = nullptr;
  ScalarRec* scalars = nullptr;
  ProgramRec* progs = nullptr;
};

struct ProfRec {
  cudaEvent_t a, b;
  double bytes;
  int32_t step_begin, step_end, kind, out_rank;
};

struct tn_plan {
  PlanHeader h{};
  std::vector<ProgramRec> progs;
  std::vector<LeafRec> leaves;
  std::vector<StepRec> steps;
  std::vector<OpRec> ops;
  std::vector<ScalarRec> scalars;
  std::vector<int32_t> prefix, sliced, residual, degrees;
  std::mutex mu;
  std::map<int, DevTables> dev;
  bool profiling = false;
  std::vector<ProfRec> prof;
  std::vector<cudaEvent_t> ev_pool;
  uint64_t all_launches = 0;
  bool batchable = false;   // every per-slice op is an interpreter run -> slices can run batched
  ~tn_plan() {
    for (auto& kv : dev) {
      cudaSetDevice(kv.first);
      cudaFree(kv.second.steps);
      cudaFree(kv.second.leaves);
      cudaFree(kv.second.scalars);
      cudaFree(kv.second.progs);
    }
    for (auto& p : prof) { cudaEventDestroy(p.a); cudaEventDestroy(p.b); }
    for (auto e : ev_pool) cudaEventDestroy(e);
  }
};

// ============================================================== serialization
namespace {

template <typename T>
void put(std::vector<uint8_t>& buf, const T* p, size_t n) {
  const uint8_t* b = reinterpret_cast<const uint8_t*>(p);
  buf.insert(buf.end(), b, b + n * sizeof(T));
}

template <typename T>
bool get(const uint8_t*& cur, const uint8_t* end, std::vector<T>& v, int64_t n) {
  if (n < 0) return false;
  const size_t bytes = (size_t)n * sizeof(T);
  if ((size_t)(end - cur) < bytes) return false;
  v.resize((size_t)n);
  if (bytes) std::memcpy(v.data(), cur, bytes);
  cur += bytes;
  return true;
}

size_t align256(size_t x) { return (x + 255) / 256 * 256; }

size_t ws_bytes_for(const PlanHeader& h, int dtype) {
  const size_t es = dtype == TN_C64 ? 8 : 16;
  const uint64_t nsl = 1ull << h.k;
  const uint64_t nres = std::max<uint64_t>(nsl, (uint64_t)h.n_programs);
  return align256(h.arena_elems * es) + align256(16 * nres) + 256;
}

}  // namespace

// ============================================================== C ABI: planning
extern "C" tn_status tn_plan_build(int32_t n_qubits, int32_t n_edges, const int32_t* edges,
                                   int32_t p, const tn_build_opts* opts, void** buf, size_t* len) {
  if (!opts || !buf || !len || (n_edges > 0 && !edges) || n_qubits <= 0 || n_edges < 0)
    return fail(TN_E_INVAL, "tn_plan_build: null or negative argument");
  if (p < 1 || p > kMaxP) return fail(TN_E_INVAL, "tn_plan_build: p out of range [1, 16]");
  if (opts->orderer < TN_ORDER_MIN_FILL || opts->orderer > TN_ORDER_RGREEDY_FILL)
    return fail(TN_E_INVAL, "tn_plan_build: unknown orderer");
  if (opts->rg_q < 0 || opts->rg_q > 4096 || opts->rg_tau_milli < 0)
    return fail(TN_E_INVAL, "tn_plan_build: bad rgreedy parameters");
  OrderSpec spec;
  spec.orderer = opts->orderer;
  spec.q = opts->rg_q == 0 ? 8 : opts->rg_q;
  spec.tau = opts->rg_tau_milli == 0 ? 0.5 : opts->rg_tau_milli / 1000.0;
  spec.seed = opts->rg_seed;
  if (opts->kind != TN_KIND_AMPLITUDE && opts->kind != TN_KIND_ENERGY)
    return fail(TN_E_INVAL, "tn_plan_build: unknown kind");
  if (opts->n_sliced < 0 || opts->n_sliced > 30 || opts->r < 0)
    return fail(TN_E_INVAL, "tn_plan_build: n_sliced must be in [0, 30], r >= 0");
  if (opts->kind == TN_KIND_ENERGY && opts->n_sliced != 0)
    return fail(TN_E_INVAL, "tn_plan_build: energy plans are unsliced");
  const int small_log2 = opts->small_log2 < 0 ? 12 : opts->small_log2;
  try {
    std::vector<int> ev(edges, edges + 2 * (size_t)n_edges);
    std::vector<Network> nets;
    if (opts->kind == TN_KIND_AMPLITUDE) {
      nets.push_back(build_amplitude_network(n_qubits, ev, p));
    } else {
      for (int e = 0; e < n_edges; ++e)
        nets.push_back(build_cone_network(n_qubits, ev, p, ev[2 * e], ev[2 * e + 1]));
    }
    PlanHeader h;
    std::memset(&h, 0, sizeof(h));
    h.magic = kPlanMagic;
    h.version = kPlanVersion;
    h.kind = opts->kind;
    h.n_qubits = n_qubits;
    h.p = p;
    h.n_edges = n_edges;
    h.orderer = opts->orderer;
    h.small_log2 = small_log2;
    h.n_labels = nets.empty() ? 0 : nets[0].n_labels;
    std::vector<ProgramRec> progs;
    std::vector<LeafRec> leaves;
    std::vector<StepRec> steps;
    std::vector<OpRec> ops;
    std::vector<ScalarRec> scal;
    Schedule sch0;
    std::vector<int> degrees0;
    uint64_t arena = 0;
    for (size_t ni = 0; ni < nets.size(); ++ni) {
      const Network& net = nets[ni];
      BitGraph g = BitGraph::from_network(net);
      Schedule sch = slice_search(g, opts->n_sliced, opts->r, spec);
      if (opts->max_width > 0 && sch.width > opts->max_width) {
        return fail(TN_E_TOO_WIDE, "contraction width " + std::to_string(sch.width) +
                                       " exceeds max_width " + std::to_string(opts->max_width));
      }
      std::string err;
      LoweredProgram lp = lower(net, sch, small_log2, &err);
      if (!err.empty()) return fail(TN_E_PLAN, "lowering: " + err);
      if (opts->max_width > 0 && lp.width > opts->max_width)
        return fail(TN_E_TOO_WIDE, "contraction width " + std::to_string(lp.width));
      const int32_t leaf0 = (int32_t)leaves.size(), step0 = (int32_t)steps.size();
      const int32_t op0 = (int32_t)ops.size(), sc0 = (int32_t)scal.size();
      for (auto l : lp.leaves) { l.off += arena; leaves.push_back(l); }
      for (auto s : lp.steps) {
        s.out_off += arena;
        for (int t = 0; t < s.n_in; ++t) s.in[t].off += arena;
        steps.push_back(s);
      }
      for (auto o : lp.ops) { o.begin += step0; o.end += step0; ops.push_back(o); }
      for (auto s : lp.scalars) { s.off += arena; s.program = (int32_t)ni; scal.push_back(s); }
      ProgramRec pr = lp.prog;
      pr.stepA_begin += step0; pr.stepA_end += step0;
      pr.stepB_begin += step0; pr.stepB_end += step0;
      pr.opA_begin += op0; pr.opA_end += op0;
      pr.opB_begin += op0; pr.opB_end += op0;
      pr.scal_begin += sc0; pr.scal_end += sc0;
      pr.arena_begin = arena;
      pr.arena_end = arena + lp.arena_elems;
      progs.push_back(pr);
      (void)leaf0;
      arena += lp.arena_elems;
      h.width = std::max(h.width, lp.width);
      h.unsliced_width = std::max(h.unsliced_width, sch.unsliced_width);
      if (ni == 0) {
        sch0 = sch;
        degrees0 = lp.degrees;
        h.k = (int32_t)sch.sliced.size();
        h.r = opts->r == 0 ? h.k : opts->r;
        h.slice_step = (int32_t)sch.prefix.size();
        h.persistent_elems = lp.persistent_elems;
      }
      h.pred_elems_slice += lp.elems_slice;
      h.pred_elems_prefix += lp.elems_prefix;
      h.pred_elems_big_slice += lp.elems_big_slice;
      h.big_launches_slice += lp.big_launches_slice;
      h.launches_prefix += lp.launches_prefix;
      h.launches_slice += lp.launches_slice;
    }
    h.arena_elems = arena;
    h.n_programs = (int32_t)progs.size();
    h.n_leaves = (int32_t)leaves.size();
    h.n_steps = (int32_t)steps.size();
    h.n_ops = (int32_t)ops.size();
    h.n_scalars = (int32_t)scal.size();
    h.n_prefix = (int32_t)sch0.prefix.size();
    h.n_residual = (int32_t)sch0.residual.size();
    h.n_degrees = (int32_t)degrees0.size();
    std::vector<uint8_t> out;
    put(out, &h, 1);
    put(out, progs.data(), progs.size());
    put(out, leaves.data(), leaves.size());
    put(out, steps.data(), steps.size());
    put(out, ops.data(), ops.size());
    put(out, scal.data(), scal.size());
    put(out, sch0.prefix.data(), sch0.prefix.size());
    put(out, sch0.sliced.data(), sch0.sliced.size());
    put(out, sch0.residual.data(), sch0.residual.size());
    put(out, degrees0.data(), degrees0.size());
    void* mem = std::malloc(out.size());
    if (!mem) return fail(TN_E_NOMEM, "tn_plan_build: out of host memory");
    std::memcpy(mem, out.data(), out.size());
    *buf = mem;
    *len = out.size();
    return TN_OK;
  } catch (const std::invalid_argument& e) {
    return fail(TN_E_PLAN, std::string("tn_plan_build: ") + e.what());
  } catch (const std::bad_alloc&) {
    return fail(TN_E_NOMEM, "tn_plan_build: out of host memory");
  } catch (const std::exception& e) {
    return fail(TN_E_PLAN, std::string("tn_plan_build: ") + e.what());
  }
}

extern "C" void tn_buffer_free(void* buf) { std::free(buf); }

// ============================================================== C ABI: load / info
extern "C" tn_status tn_plan_load(const void* buf, size_t len, tn_plan** out) {
  if (!buf || !out) return fail(TN_E_INVAL, "tn_plan_load: null argument");
  *out = nullptr;
  const uint8_t* cur = static_cast<const uint8_t*>(buf);
  const uint8_t* end = cur + len;
  if (len < sizeof(PlanHeader)) return fail(TN_E_PLAN, "tn_plan_load: buffer too short");
  std::unique_ptr<tn_plan> pl(new (std::nothrow) tn_plan());
  if (!pl) return fail(TN_E_NOMEM, "tn_plan_load: out of host memory");
  std::memcpy(&pl->h, cur, sizeof(PlanHeader));
  cur += sizeof(PlanHeader);
  const PlanHeader& h = pl->h;
  if (h.magic != kPlanMagic || h.version != kPlanVersion)
    return fail(TN_E_PLAN, "tn_plan_load: bad magic or version");
  if (h.k < 0 || h.k > 30 || h.p < 1 || h.p > kMaxP || h.n_programs < 1)
    return fail(TN_E_PLAN, "tn_plan_load: bad header");
  if (!get(cur, end, pl->progs, h.n_programs) || !get(cur, end, pl->leaves, h.n_leaves) ||
      !get(cur, end, pl->steps, h.n_steps) || !get(cur, end, pl->ops, h.n_ops) ||
      !get(cur, end, pl->scalars, h.n_scalars) || !get(cur, end, pl->prefix, h.n_prefix) ||
      !get(cur, end, pl->sliced, h.k) || !get(cur, end, pl->residual, h.n_residual) ||
      !get(cur, end, pl->degrees, h.n_degrees))
    return fail(TN_E_PLAN, "tn_plan_load: truncated buffer");
  if (cur != end) return fail(TN_E_PLAN, "tn_plan_load: trailing bytes");
  // validation: every access stays inside the arena
  const uint64_t A = h.arena_elems;
  for (const auto& l : pl->leaves)
    if (l.rank < 0 || l.rank > 2 || l.nfact < 1 || l.nfact > kMaxFactors || l.off + 4 > A + kAlign)
      return fail(TN_E_PLAN, "tn_plan_load: bad leaf record");
  for (const auto& s : pl->steps) {
    if (s.n_in < 1 || s.n_in > kMaxIn || s.out_rank < 0 || s.out_rank > 62)
      return fail(TN_E_PLAN, "tn_plan_load: bad step record");
    if (s.out_off + (1ull << s.out_rank) > A) return fail(TN_E_PLAN, "tn_plan_load: step output out of arena");
    for (int t = 0; t < s.n_in; ++t) {
      const InRec& in = s.in[t];
      const int full = (int)in.rank + __builtin_popcount(in.slice_mask);
      if (in.rank < 1 || full > 62 || in.pv >= in.rank ||
          __builtin_popcountll(in.out_mask) + 1 != (int)in.rank ||
          (s.out_rank < 64 && (in.out_mask >> s.out_rank) != 0) ||
          (in.slice_mask >> h.k) != 0 || in.off + (1ull << full) > A)
        return fail(TN_E_PLAN, "tn_plan_load: bad step input record");
    }
  }
  for (const auto& o : pl->ops)
    if (o.begin < 0 || o.end > h.n_steps || o.begin >= o.end ||
        (o.type != OP_BIG && o.type != OP_RUN && o.type != OP_CHAIN && o.type != OP_GROUP) ||
        (o.type == OP_GROUP && (o.end - o.begin > kMaxGroupPlan || o.end - o.begin < 2)) ||
        (o.type == OP_CHAIN && (o.end - o.begin > kMaxChain || pl->steps[o.end - 1].out_rank < 1)) ||
        (o.type == OP_BIG && pl->steps[o.begin].out_rank < 1))
      return fail(TN_E_PLAN, "tn_plan_load: bad op record");
  for (const auto& s : pl->scalars)
    if ((s.slice_mask >> h.k) != 0 || s.off + (1ull << __builtin_popcount(s.slice_mask)) > A)
      return fail(TN_E_PLAN, "tn_plan_load: bad scalar record");
  for (const auto& pr : pl->progs)
    if (pr.stepB_begin < 0 || pr.stepB_end > h.n_steps || pr.scal_begin < 0 || pr.scal_end > h.n_scalars ||
        pr.opA_begin < 0 || pr.opB_end > h.n_ops)
      return fail(TN_E_PLAN, "tn_plan_load: bad program record");
  pl->batchable = pl->h.kind == TN_KIND_AMPLITUDE && pl->h.n_programs == 1;
  for (int oi = pl->progs[0].opB_begin; oi < pl->progs[0].opB_end; ++oi)
    if (pl->ops[oi].type != OP_RUN) pl->batchable = false;
  *out = pl.release();
  return TN_OK;
}

extern "C" void tn_plan_free(tn_plan* plan) { delete plan; }

// workspace with `batch` windows: [base layout][windows 1..batch-1][batch results][batch angles]
static size_t ws_bytes_batched(const PlanHeader& h, int dtype, uint64_t batch) {
  const size_t es = dtype == TN_C64 ? 8 : 16;
  if (batch <= 1) return ws_bytes_for(h, dtype);
  return ws_bytes_for(h, dtype) + (batch - 1) * h.arena_elems * es +
         align256(16 * batch * (uint64_t)h.n_programs) + align256(sizeof(Angles) * batch);
}

extern "C" size_t tn_workspace_bytes(const tn_plan* plan, tn_dtype dtype, uint64_t batch) {
  if (!plan || (dtype != TN_C64 && dtype != TN_C128)) return 0;
  return ws_bytes_batched(plan->h, dtype, batch);
}

extern "C" tn_status tn_plan_info(const tn_plan* plan, tn_plan_info_t* o) {
  if (!plan || !o) return fail(TN_E_INVAL, "tn_plan_info: null argument");
  const PlanHeader& h = plan->h;
  std::memset(o, 0, sizeof(*o));
  o->kind = h.kind;
  o->n_qubits = h.n_qubits;
  o->p = h.p;
  o->n_edges = h.n_edges;
  o->width = h.width;
  o->unsliced_width = h.unsliced_width;
  o->k = h.k;
  o->slice_step = h.slice_step;
  o->n_programs = h.n_programs;
  o->n_labels = h.n_labels;
  o->n_slices = 1ull << h.k;
  uint64_t nA = 0, nB = 0;
  for (const auto& s : plan->steps) (s.phase == 0 ? nA : nB)++;
  o->prefix_steps = nA;
  o->steps_per_slice = nB;
  o->launches_prefix = h.launches_prefix;
  o->launches_per_slice = h.launches_slice;
  for (int d = 0; d < 2; ++d) {
    const double es = d == 0 ? 8.0 : 16.0;
    o->workspace_bytes[d] = ws_bytes_for(h, d);
    o->pred_bytes_per_slice[d] = h.pred_elems_slice * es;
    o->pred_bytes_prefix[d] = h.pred_elems_prefix * es;
    o->pred_bytes_big_per_slice[d] = h.pred_elems_big_slice * es;
  }
  o->big_launches_per_slice = h.big_launches_slice;
  o->slices_batchable = plan->batchable ? 1 : 0;
  return TN_OK;
}

extern "C" tn_status tn_plan_schedule(const tn_plan* plan, int32_t* prefix, int32_t* sliced,
                                      int32_t* residual, int32_t* degrees) {
  if (!plan) return fail(TN_E_INVAL, "tn_plan_schedule: null plan");
  if (prefix) std::copy(plan->prefix.begin(), plan->prefix.end(), prefix);
  if (sliced) std::copy(plan->sliced.begin(), plan->sliced.end(), sliced);
  if (residual) std::copy(plan->residual.begin(), plan->residual.end(), residual);
  if (degrees) std::copy(plan->degrees.begin(), plan->degrees.end(), degrees);
  return TN_OK;
}

extern "C" tn_status tn_plan_steps(const tn_plan* plan, tn_step_info_t* out, int64_t cap, int64_t* n) {
  if (!plan || !n) return fail(TN_E_INVAL, "tn_plan_steps: null argument");
  *n = (int64_t)plan->steps.size();
  std::vector<char> big(plan->steps.size(), 0);
  for (const auto& op : plan->ops)
    if (op.type == OP_BIG || op.type == OP_CHAIN || op.type == OP_GROUP)
      for (int i = op.begin; i < op.end; ++i) big[i] = op.type == OP_BIG ? 1 : (op.type == OP_CHAIN ? 2 : 3);
  for (int64_t i = 0; out && i < cap && i < *n; ++i) {
    const StepRec& s = plan->steps[i];
    tn_step_info_t& o = out[i];
    std::memset(&o, 0, sizeof(o));
    o.phase = s.phase;
    o.label = s.label;
    o.out_rank = s.out_rank;
    o.degree = s.degree;
    o.n_in = s.n_in;
    o.inplace = s.inplace;
    o.standalone = big[i];
    double el = std::ldexp(1.0, s.out_rank);
    for (int t = 0; t < s.n_in; ++t) {
      o.in_rank[t] = (int32_t)s.in[t].rank;
      o.in_out_mask[t] = s.in[t].out_mask;
      o.in_pv[t] = (int32_t)s.in[t].pv;
      el += std::ldexp(1.0, (int)s.in[t].rank);
    }
    o.bytes_c64 = 8.0 * el;
  }
  return TN_OK;
}

extern "C" tn_status tn_sum_partials(const tn_plan* plan, const double* partials, double out[2]) {
  if (!plan || !partials || !out) return fail(TN_E_INVAL, "tn_sum_partials: null argument");
  const uint64_t n = 1ull << plan->h.k;
  std::vector<double> buf(partials, partials + 2 * n);
  uint64_t m = n;
  while (m > 1) {
    uint64_t hh = 0;
    for (uint64_t i = 0; i + 1 < m; i += 2, ++hh) {
      buf[2 * hh] = buf[2 * i] + buf[2 * (i + 1)];
      buf[2 * hh + 1] = buf[2 * i + 1] + buf[2 * (i + 1) + 1];
    }
    if (m & 1) {
      buf[2 * hh] = buf[2 * (m - 1)];
      buf[2 * hh + 1] = buf[2 * (m - 1) + 1];
      ++hh;
    }
    m = hh;
  }
  out[0] = buf[0];
  out[1] = buf[1];
  return TN_OK;
}

// ============================================================== executor
namespace {

tn_status ensure_dev(tn_plan* pl, DevTables** out) {
  int dev = 0;
  CU(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(pl->mu);
  auto it = pl->dev.find(dev);
  if (it == pl->dev.end()) {
    DevTables t;
    auto up = [](void** dst, const void* src, size_t bytes) -> cudaError_t {
      cudaError_t e = cudaMalloc(dst, std::max<size_t>(bytes, 16));
      if (e != cudaSuccess) return e;
      return bytes ? cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice) : cudaSuccess;
    };
    CU(up((void**)&t.steps, pl->steps.data(), pl->steps.size() * sizeof(StepRec)));
    CU(up((void**)&t.leaves, pl->leaves.data(), pl->leaves.size() * sizeof(LeafRec)));
    CU(up((void**)&t.scalars, pl->scalars.data(), pl->scalars.size() * sizeof(ScalarRec)));
    CU(up((void**)&t.progs, pl->progs.data(), pl->progs.size() * sizeof(ProgramRec)));
    it = pl->dev.emplace(dev, t).first;
  }
  *out = &it->second;
  return TN_OK;
}

// opt in to more than 48 KB of (static + dynamic) shared memory, once per kernel instantiation
template <typename K>
void allow_smem(K kernel, size_t dyn) {
  static std::mutex mu;
  static std::map<const void*, size_t> granted;   // per kernel (per device is not needed: the
                                                   // attribute is a function property)
  if (dyn + 16 * 1024 <= 48 * 1024) return;
  std::lock_guard<std::mutex> lk(mu);
  size_t& g = granted[reinterpret_cast<const void*>(kernel)];
  if (dyn > g) {
    const size_t want = std::max<size_t>(dyn, 100 * 1024);
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)want);
    g = want;
  }
}

int g_num_sms = 0;
bool debug_checks() {
  static const int on = [] {
    const char* v = std::getenv("TNB_DEBUG");
    return (v && v[0] == '1') ? 1 : 0;
  }();
  return on != 0;
}
int num_sms() {
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

uint64_t host_pext(uint64_t x, uint64_t m) {
  uint64_t r = 0;
  int k = 0;
  while (m) {
    const uint64_t b = m & (~m + 1);
    if (x & b) r |= 1ull << k;
    ++k;
    m ^= b;
  }
  return r;
}

// host side of the staging decision (see kernels.cuh): an input is staged in shared memory when
// it holds some but not all of a tile's low output bits, those map to its lowest positions, and
// the chunks fit the budget
template <typename T>
void plan_staging(BigArgs& a) {
  constexpr int TB = TileBits<T>::v;
  const uint64_t inner = (1ull << TB) - 1;
  uint32_t off = 0;
  for (int t = 0; t < a.n_in; ++t) {
    a.flags[t] &= ~F_STAGED;
    const uint64_t lowm = a.out_mask[t] & inner;
    const int nlow = __builtin_popcountll(lowm);
    if (a.out_rank <= TB || nlow == 0 || nlow >= TB || nlow > 10) continue;
    // contiguity: the tile's low output bits must be the input's positions 0..nlow-1
    uint64_t f = 0;
    {
      uint64_t m = a.out_mask[t], r = 0;
      int k = 0;
      for (int b = 0; b < 64 && m; ++b) {
        if ((m >> b) & 1) {
          if ((lowm >> b) & 1) r |= 1ull << k;
          ++k;
          m &= ~(1ull << b);
        }
      }
      const uint64_t lo = r & ((1ull << a.pv[t]) - 1);
      f = lo | ((r >> a.pv[t]) << (a.pv[t] + 1));
    }
    if (f != (1ull << nlow) - 1) continue;
    const uint32_t need = 2u << nlow;  // both x
    if ((off + need) * sizeof(T) * 2 > 48 * 1024) continue;
    a.flags[t] |= F_STAGED;
    a.nlow[t] = (uint32_t)nlow;
    a.stage_off[t] = off;
    off += need;
  }
  a.stage_elems = off;
}

// traversal order of the tile-index bits: bits absent from the largest input first (its chunk
// is then reused by consecutive tiles), then bits absent from the second largest, then the rest
// in ascending order.  Streaming (evict-first) loads only for inputs without reuse.
template <typename T>
void plan_order(BigArgs& a) {
  constexpr int TB = TileBits<T>::v;
  int big[2] = {-1, -1};
  for (int t = 0; t < a.n_in; ++t) {
    const int r = __builtin_popcountll(a.out_mask[t]);
    if (big[0] < 0 || r > __builtin_popcountll(a.out_mask[big[0]])) { big[1] = big[0]; big[0] = t; }
    else if (big[1] < 0 || r > __builtin_popcountll(a.out_mask[big[1]])) big[1] = t;
  }
  std::vector<int> bits;
  for (int b = TB; b < 64; ++b) bits.push_back(b);
  auto has = [&](int t, int b) { return t >= 0 && ((a.out_mask[t] >> b) & 1); };
  std::stable_sort(bits.begin(), bits.end(), [&](int x, int y) {
    if (has(big[0], x) != has(big[0], y)) return !has(big[0], x);
    if (has(big[1], x) != has(big[1], y)) return !has(big[1], x);
    return x < y;
  });
  // bits at or above out_rank never change within the grid; keep them last
  std::stable_partition(bits.begin(), bits.end(), [&](int b) { return b < a.out_rank; });
  for (int i = 0; i < 64 - TB; ++i) a.perm[i] = (uint8_t)(bits[i] - TB);
  const uint64_t full = a.out_rank >= 64 ? ~0ull : ((1ull << a.out_rank) - 1);
  for (int t = 0; t < a.n_in; ++t) {
    if (a.out_mask[t] == full && a.out_rank >= 16) a.flags[t] |= F_STREAM;
    else a.flags[t] &= ~F_STREAM;
  }
}

template <typename T, int NIN>
void launch_bucket_n(BigArgs a, cudaStream_t st) {
  constexpr uint64_t TILE = 1ull << TileBits<T>::v;
  plan_order<T>(a);
  plan_staging<T>(a);
  const uint64_t n_out = 1ull << a.out_rank;
  const uint64_t tiles = (n_out + TILE - 1) / TILE;
  const uint64_t cap = (uint64_t)num_sms() * 4;
  const unsigned grid = (unsigned)std::min<uint64_t>(tiles, cap);
  const size_t smem = (size_t)a.stage_elems * sizeof(T) * 2;
  bool wide = false;   // any input with more than 32 bits -> 64-bit offsets
  for (int t = 0; t < a.n_in; ++t) wide |= (__builtin_popcountll(a.out_mask[t]) + 1 > 32);
  if (wide) {
    allow_smem(k_bucket<T, NIN, uint64_t>, smem);
    k_bucket<T, NIN, uint64_t><<<grid, kBucketThreads, smem, st>>>(a);
  } else {
    allow_smem(k_bucket<T, NIN, uint32_t>, smem);
    k_bucket<T, NIN, uint32_t><<<grid, kBucketThreads, smem, st>>>(a);
  }
}

// ---------------------------------------------------------------- k_group_t host side
struct GIn {
  const void* ptr;
  uint64_t out_mask;   // output bits present (relative to the group output)
  uint32_t pv;         // F_t(o) = ins0(pext(o, out_mask), pv)
  uint32_t rank;       // bits of the input (for 32/64-bit offsets)
  bool full;           // holds every output bit and every summed bit (read exactly once)
  uint64_t gx[1 << kMaxGroup];
};
struct GDesc {
  void* out;
  int out_rank;
  int M;
  int n;
  GIn in[kMaxIn];
};

uint64_t host_fmap(uint64_t o, uint64_t mask, uint32_t pv) {
  const uint64_t r = host_pext(o, mask);
  const uint64_t lo = r & ((1ull << pv) - 1);
  return lo | ((r >> pv) << (pv + 1));
}

template <typename T, typename OffT, int NDIR, int NSTG, int M, int NDV>
void launch_g(const GArgs& ga, unsigned grid, size_t smem, cudaStream_t st) {
  allow_smem(k_group_t<T, OffT, NDIR, NSTG, M, NDV>, smem);
  k_group_t<T, OffT, NDIR, NSTG, M, NDV><<<grid, kBucketThreads, smem, st>>>(ga);
}

template <typename T, typename OffT, int M>
bool dispatch_g(const GArgs& ga, int nd, int ns, int ndv, unsigned grid, size_t smem, cudaStream_t st) {
#define TN_G(D, S, V) \
  if (nd == D && ns == S && ndv == V) { launch_g<T, OffT, D, S, M, V>(ga, grid, smem, st); return true; }
  TN_G(1, 0, 1) TN_G(2, 0, 2) TN_G(0, 1, 0) TN_G(1, 1, 1) TN_G(0, 2, 0) TN_G(2, 1, 2) TN_G(1, 2, 1)
  TN_G(1, 0, 0) TN_G(2, 0, 1) TN_G(1, 1, 0) TN_G(2, 1, 1)
  if constexpr (M == 1) {
    TN_G(3, 0, 3) TN_G(2, 2, 2) TN_G(0, 3, 0) TN_G(1, 3, 1) TN_G(0, 4, 0) TN_G(3, 0, 2) TN_G(2, 0, 0)
  }
#undef TN_G
  return false;
}

// Classify the inputs (direct / staged / constant), build GArgs and launch k_group_t.  Returns
// false when the shape has no instantiation (the caller then runs the generic path).
template <typename T>
bool try_launch_group(const GDesc& g, cudaStream_t st) {
  constexpr int TB = TileBits<T>::v;
  constexpr uint64_t TILE = 1ull << TB;
  if (g.out_rank <= TB || g.M < 1 || g.M > kMaxGroup || g.n < 1 || g.n > kMaxIn) return false;
  const uint64_t inner = TILE - 1;
  const int NX = 1 << g.M;
  // traversal order of the tile bits: bits absent from the two largest varying inputs first
  int big[2] = {-1, -1};
  for (int t = 0; t < g.n; ++t) {
    const int r = __builtin_popcountll(g.in[t].out_mask);
    if (big[0] < 0 || r > __builtin_popcountll(g.in[big[0]].out_mask)) { big[1] = big[0]; big[0] = t; }
    else if (big[1] < 0 || r > __builtin_popcountll(g.in[big[1]].out_mask)) big[1] = t;
  }
  auto has = [&](int t, int b) { return t >= 0 && ((g.in[t].out_mask >> b) & 1); };
  std::vector<int> bits;
  for (int b = TB; b < 64; ++b) bits.push_back(b);
  std::stable_sort(bits.begin(), bits.end(), [&](int x, int y) {
    if (has(big[0], x) != has(big[0], y)) return !has(big[0], x);
    if (has(big[1], x) != has(big[1], y)) return !has(big[1], x);
    return x < y;
  });
  std::stable_partition(bits.begin(), bits.end(), [&](int b) { return b < g.out_rank; });

  int dir[kMaxIn], dirs[kMaxIn], stg[kMaxIn], cst[kMaxIn], nd = 0, nds = 0, ns = 0, nc = 0;
  int nlow_of[kMaxIn] = {0};
  uint32_t nparts_of[kMaxIn] = {0};
  uint32_t soff = 0;
  for (int t = 0; t < g.n; ++t) {
    const GIn& in = g.in[t];
    const uint64_t lowm = in.out_mask & inner;
    const int nlow = __builtin_popcountll(lowm);
    if (nlow == 0) { cst[nc++] = t; continue; }
    const bool vec_ok = (VecT<T>::n == 1) || ((in.out_mask & 1) && in.pv != 0);
    // staging needs the tile's low output bits at the input's lowest positions
    const bool contig = host_fmap(lowm, in.out_mask, in.pv) == (1ull << nlow) - 1;
    std::vector<uint64_t> parts;
    for (int x = 0; x < NX; ++x)
      if (std::find(parts.begin(), parts.end(), in.gx[x]) == parts.end()) parts.push_back(in.gx[x]);
    const uint32_t need = (uint32_t)parts.size() << nlow;
    const bool stageable = contig && nlow < TB && (nlow <= TB - 3 || !vec_ok) &&
                           (soff + need) * sizeof(T) * 2 <= 48 * 1024;
    if (stageable) {
      nlow_of[t] = nlow;
      nparts_of[t] = (uint32_t)parts.size();
      stg[ns++] = t;
      soff += need;
    } else if (vec_ok) {
      dir[nd++] = t;
    } else {
      dirs[nds++] = t;   // direct, 8-byte loads
    }
  }
  const int ndv = nd;
  for (int i = 0; i < nds; ++i) dir[nd++] = dirs[i];
  if (nd + ns == 0) return false;
  GArgs ga;   // host copy; passed by value as the launch parameters
  std::memset(&ga, 0, sizeof(ga));
  ga.out = g.out;
  ga.out_rank = g.out_rank;
  ga.nc = nc;
  for (int i = 0; i < 64 - TB; ++i) ga.perm[i] = (uint8_t)(bits[i] - TB);
  const uint64_t full = (1ull << g.out_rank) - 1;
  int k = 0;
  uint32_t off = 0;
  bool wide = false;
  auto put = [&](int t) {
    const GIn& in = g.in[t];
    ga.in[k] = in.ptr;
    ga.out_mask[k] = in.out_mask;
    ga.pv[k] = in.pv;
    ga.stream[k] = (in.full && in.out_mask == full && g.out_rank >= 16) ? 1u : 0u;
    for (int x = 0; x < NX; ++x) ga.gx[k][x] = in.gx[x];
    wide |= in.rank > 32;
    ++k;
  };
  for (int i = 0; i < nd; ++i) put(dir[i]);
  for (int i = 0; i < ns; ++i) {
    const int t = stg[i];
    std::vector<uint64_t> parts;
    for (int x = 0; x < NX; ++x) {
      auto it = std::find(parts.begin(), parts.end(), g.in[t].gx[x]);
      uint32_t pi;
      if (it == parts.end()) {
        pi = (uint32_t)parts.size();
        parts.push_back(g.in[t].gx[x]);
        ga.rep[k][pi] = (uint8_t)x;
      } else {
        pi = (uint32_t)(it - parts.begin());
      }
      ga.sx[k][x] = off + (pi << nlow_of[t]);
    }
    ga.nlow[k] = (uint32_t)nlow_of[t];
    ga.nparts[k] = nparts_of[t];
    off += nparts_of[t] << nlow_of[t];
    put(t);
  }
  for (int i = 0; i < nc; ++i) put(cst[i]);
  ga.stage_elems = off;
  const uint64_t tiles = ((1ull << g.out_rank) + TILE - 1) / TILE;
  const unsigned grid = (unsigned)std::min<uint64_t>(tiles, (uint64_t)num_sms() * 4);
  const size_t smem = (size_t)off * sizeof(T) * 2;
  if (wide) return g.M == 1 ? dispatch_g<T, uint64_t, 1>(ga, nd, ns, ndv, grid, smem, st) : false;
  switch (g.M) {
    case 1: return dispatch_g<T, uint32_t, 1>(ga, nd, ns, ndv, grid, smem, st);
    case 2: return dispatch_g<T, uint32_t, 2>(ga, nd, ns, ndv, grid, smem, st);
    case 3: return dispatch_g<T, uint32_t, 3>(ga, nd, ns, ndv, grid, smem, st);
    case 4: return dispatch_g<T, uint32_t, 4>(ga, nd, ns, ndv, grid, smem, st);
    case 5: return dispatch_g<T, uint32_t, 5>(ga, nd, ns, ndv, grid, smem, st);
    default: return false;
  }
}

// register-blocked pair kernel (k_pair) for groups with exactly two varying inputs
template <typename T, typename OffT, int M>
void launch_p(const PArgs& pa, unsigned grid, size_t smem, cudaStream_t st) {
  allow_smem(k_pair<T, OffT, M>, smem);
  k_pair<T, OffT, M><<<grid, kBucketThreads, smem, st>>>(pa);
}

template <typename T>
bool try_launch_pair(const GDesc& g, cudaStream_t st) {
  constexpr int TB = kPairTB;
  constexpr uint64_t TILE = 1ull << TB;
  if (g.out_rank < TB + 1 || g.M < 2 || g.M > kMaxGroup) return false;
  const uint64_t inner = TILE - 1;
  const int NX = 1 << g.M;
  int var[2], nv = 0, cst[kMaxIn], nc = 0;
  for (int t = 0; t < g.n; ++t) {
    if ((g.in[t].out_mask & inner) == 0) { cst[nc++] = t; continue; }
    if (nv == 2) return false;
    var[nv++] = t;
  }
  if (nv != 2) return false;
  PArgs pa;
  std::memset(&pa, 0, sizeof(pa));
  // staging layout: the tile bits of each input must be its lowest positions
  uint32_t off = 0;
  bool wide = false;
  for (int u = 0; u < 2; ++u) {
    const GIn& in = g.in[var[u]];
    const uint64_t lowm = in.out_mask & inner;
    const int nlow = __builtin_popcountll(lowm);
    if (host_fmap(lowm, in.out_mask, in.pv) != (1ull << nlow) - 1) return false;
    if ((1u << nlow) * sizeof(T) < 16) return false;
    std::vector<uint64_t> parts;
    for (int x = 0; x < NX; ++x) {
      auto it = std::find(parts.begin(), parts.end(), in.gx[x]);
      uint32_t pi;
      if (it == parts.end()) {
        pi = (uint32_t)parts.size();
        parts.push_back(in.gx[x]);
        pa.rep[u][pi] = (uint8_t)x;
      } else {
        pi = (uint32_t)(it - parts.begin());
      }
      pa.sx[u][x] = off + (pi << nlow);
    }
    pa.in[u] = in.ptr;
    pa.mask[u] = in.out_mask;
    pa.pv[u] = in.pv;
    for (int x = 0; x < NX; ++x) pa.gx[u][x] = in.gx[x];
    pa.nparts[u] = (uint32_t)parts.size();
    pa.nlow[u] = (uint32_t)nlow;
    off += (uint32_t)parts.size() << nlow;
    wide |= in.rank > 32;
  }
  const size_t smem = (size_t)off * sizeof(T) * 2;
  if (smem > 96 * 1024 || wide) return false;
  pa.stage_elems = off;
  // block bits: a tile bit in A only and one in B only, preferring bits >= 5 (lanes keep bits 0-4)
  const uint64_t mA = g.in[var[0]].out_mask & inner, mB = g.in[var[1]].out_mask & inner;
  int ra = -1, rb = -1;
  for (int b = TB - 1; b >= 0; --b) {
    if (ra < 0 && ((mA >> b) & 1) && !((mB >> b) & 1)) ra = b;
    if (rb < 0 && ((mB >> b) & 1) && !((mA >> b) & 1)) rb = b;
  }
  if (ra < 0 || rb < 0) return false;
  pa.ra = (uint32_t)ra;
  pa.rb = (uint32_t)rb;
  int k = 0;
  for (int b = 0; b < TB; ++b)
    if (b != ra && b != rb) pa.tbits[k++] = (uint32_t)b;
  for (int i = 0; i < nc; ++i) {
    const GIn& in = g.in[cst[i]];
    pa.cin[i] = in.ptr;
    pa.cmask[i] = in.out_mask;
    pa.cpv[i] = in.pv;
    for (int x = 0; x < NX; ++x) pa.cgx[i][x] = in.gx[x];
  }
  pa.nc = nc;
  pa.out = g.out;
  pa.out_rank = g.out_rank;
  // traversal: tile bits absent from the larger input first
  const int big = __builtin_popcountll(g.in[var[0]].out_mask) >= __builtin_popcountll(g.in[var[1]].out_mask) ? 0 : 1;
  auto has = [&](int u, int b) { return (g.in[var[u]].out_mask >> b) & 1; };
  std::vector<int> bits;
  for (int b = TB; b < 64; ++b) bits.push_back(b);
  std::stable_sort(bits.begin(), bits.end(), [&](int x, int y) {
    if (has(big, x) != has(big, y)) return !has(big, x);
    if (has(1 - big, x) != has(1 - big, y)) return !has(1 - big, x);
    return x < y;
  });
  std::stable_partition(bits.begin(), bits.end(), [&](int b) { return b < g.out_rank; });
  for (int i = 0; i < 64 - TB; ++i) pa.perm[i] = (uint8_t)(bits[i] - TB);
  const uint64_t tiles = ((1ull << g.out_rank) + TILE - 1) / TILE;
  const unsigned grid = (unsigned)std::min<uint64_t>(tiles, (uint64_t)num_sms() * 2);
  switch (g.M) {
    case 2: launch_p<T, uint32_t, 2>(pa, grid, smem, st); return true;
    case 3: launch_p<T, uint32_t, 3>(pa, grid, smem, st); return true;
    case 4: launch_p<T, uint32_t, 4>(pa, grid, smem, st); return true;
    case 5: launch_p<T, uint32_t, 5>(pa, grid, smem, st); return true;
    default: return false;
  }
}

// single bucket step as a group with M = 1 (G_t(x) = x << pv_t)
template <typename T>
bool try_launch_specialised(const BigArgs& a, cudaStream_t st) {
  GDesc g;
  std::memset(&g, 0, sizeof(g));
  g.out = a.out;
  g.out_rank = a.out_rank;
  g.M = 1;
  g.n = a.n_in;
  const uint64_t full = a.out_rank >= 64 ? ~0ull : ((1ull << a.out_rank) - 1);
  for (int t = 0; t < a.n_in; ++t) {
    g.in[t].ptr = a.in[t];
    g.in[t].out_mask = a.out_mask[t];
    g.in[t].pv = a.pv[t];
    g.in[t].rank = (uint32_t)__builtin_popcountll(a.out_mask[t]) + 1;
    g.in[t].full = a.out_mask[t] == full;
    g.in[t].gx[0] = 0;
    g.in[t].gx[1] = 1ull << a.pv[t];
  }
  return try_launch_group<T>(g, st);
}

template <typename T>
void launch_bucket(const BigArgs& a, cudaStream_t st) {
  if (try_launch_specialised<T>(a, st)) return;
  switch (a.n_in) {
    case 1: launch_bucket_n<T, 1>(a, st); break;
    case 2: launch_bucket_n<T, 2>(a, st); break;
    case 3: launch_bucket_n<T, 3>(a, st); break;
    case 4: launch_bucket_n<T, 4>(a, st); break;
    case 5: launch_bucket_n<T, 5>(a, st); break;
    case 6: launch_bucket_n<T, 6>(a, st); break;
    case 7: launch_bucket_n<T, 7>(a, st); break;
    default: launch_bucket_n<T, 8>(a, st); break;
  }
}

cudaEvent_t pool_event(tn_plan* pl) {
  if (!pl->ev_pool.empty()) {
    cudaEvent_t e = pl->ev_pool.back();
    pl->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

template <typename T>
uint64_t slice_off_of(const InRec& in, uint64_t j) {
  return in.slice_mask ? (host_pext(j, in.slice_mask) << in.rank) : 0ull;
}

struct ProfScope {
  tn_plan* pl;
  cudaStream_t st;
  ProfRec pr{};
  ProfScope(tn_plan* p, cudaStream_t s, double bytes, int b, int e, int kind, int out_rank) : pl(p), st(s) {
    if (!pl->profiling) return;
    pr.a = pool_event(pl);
    pr.b = pool_event(pl);
    pr.bytes = bytes;
    pr.step_begin = b;
    pr.step_end = e;
    pr.kind = kind;
    pr.out_rank = out_rank;
    cudaEventRecord(pr.a, st);
  }
  bool cancel = false;
  ~ProfScope() {
    if (!pl->profiling) return;
    if (cancel) {
      pl->ev_pool.push_back(pr.a);
      pl->ev_pool.push_back(pr.b);
      return;
    }
    cudaEventRecord(pr.b, st);
    pl->prof.push_back(pr);
  }
};

// one standalone bucket step (k_group_t with M = 1, else the generic k_bucket)
template <typename T>
void run_big(tn_plan* pl, int si, T* ws, uint64_t j, cudaStream_t st) {
  const StepRec& s = pl->steps[si];
  BigArgs a;
  std::memset(&a, 0, sizeof(a));
  a.out = ws + s.out_off;
  a.out_rank = s.out_rank;
  a.n_in = s.n_in;
  double bytes = std::ldexp((double)sizeof(T), s.out_rank);
  for (int t = 0; t < s.n_in; ++t) {
    const InRec& in = s.in[t];
    a.in[t] = ws + in.off + slice_off_of<T>(in, j);
    a.out_mask[t] = in.out_mask;
    a.pv[t] = in.pv;
    a.flags[t] = in.flags | ((t == 0 && s.inplace) ? 1u : 0u);
    bytes += std::ldexp((double)sizeof(T), (int)in.rank);
  }
  ProfScope ps(pl, st, bytes, si, si + 1, 1, s.out_rank);
  launch_bucket<T>(a, st);
}

template <typename T>
tn_status run_ops(tn_plan* pl, const DevTables& dt, int op_b, int op_e, T* ws, uint64_t j,
                  cudaStream_t st) {
  for (int oi = op_b; oi < op_e; ++oi) {
    const OpRec& op = pl->ops[oi];
    if (op.type == OP_BIG) {
      run_big<T>(pl, op.begin, ws, j, st);
    } else if (op.type == OP_CHAIN) {
      const StepRec& h = pl->steps[op.begin];
      const StepRec& last = pl->steps[op.end - 1];
      ChainArgs c;
      std::memset(&c, 0, sizeof(c));
      c.m = op.end - op.begin;
      c.out = ws + last.out_off;
      c.out_rank = last.out_rank;
      c.A = ws + h.in[0].off + slice_off_of<T>(h.in[0], j);
      for (int i = 0; i < c.m; ++i) {
        const StepRec& sk = pl->steps[op.begin + i];
        c.nw[i] = sk.n_in - 1;
        for (int k = 1; k < sk.n_in; ++k) c.w[i][k - 1] = ws + sk.in[k].off + slice_off_of<T>(sk.in[k], j);
      }
      const double bytes = (std::ldexp(1.0, (int)h.in[0].rank) + std::ldexp(1.0, c.out_rank)) * sizeof(T);
      ProfScope ps(pl, st, bytes, op.begin, op.end, 2, c.out_rank);
      constexpr int VEC = VecT<T>::n;
      const uint64_t work = ((1ull << c.out_rank) + VEC - 1) / VEC;
      const uint64_t blocks = (work + kBucketThreads - 1) / kBucketThreads;
      const unsigned grid = (unsigned)std::min<uint64_t>(blocks, (uint64_t)num_sms() * 8);
      k_chain<T><<<grid, kBucketThreads, 0, st>>>(c);
    } else if (op.type == OP_GROUP) {
      // head step + (M-1) in-place reduce followers with rank-1 weights, summed in one pass
      const StepRec& h = pl->steps[op.begin];
      const StepRec& last = pl->steps[op.end - 1];
      GDesc g;
      std::memset(&g, 0, sizeof(g));
      const int M = op.end - op.begin;
      const int Rf = last.out_rank;
      const uint64_t low = (1ull << Rf) - 1, xrest = (1ull << (M - 1)) - 1;
      const uint64_t hfull = (1ull << h.out_rank) - 1;
      g.out = ws + last.out_off;
      g.out_rank = Rf;
      g.M = M;
      double bytes = std::ldexp(1.0, Rf);
      bool ok = true;
      for (int t = 0; t < h.n_in && ok; ++t) {
        const InRec& in = h.in[t];
        GIn& gi = g.in[g.n++];
        gi.ptr = ws + in.off + slice_off_of<T>(in, j);
        gi.out_mask = in.out_mask & low;
        gi.pv = in.pv;
        gi.rank = in.rank;
        gi.full = in.out_mask == hfull;
        for (int x = 0; x < (1 << M); ++x)
          gi.gx[x] = host_fmap(((uint64_t)x & xrest) << Rf, in.out_mask, in.pv) +
                     ((uint64_t)((x >> (M - 1)) & 1) << in.pv);
        bytes += std::ldexp(1.0, (int)in.rank);
      }
      for (int i = 1; i < M && ok; ++i) {
        const StepRec& sk = pl->steps[op.begin + i];
        for (int k = 1; k < sk.n_in; ++k) {
          if (g.n >= kMaxIn) { ok = false; break; }
          GIn& gi = g.in[g.n++];
          gi.ptr = ws + sk.in[k].off + slice_off_of<T>(sk.in[k], j);
          gi.out_mask = 0;
          gi.pv = 0;
          gi.rank = 1;
          gi.full = false;
          for (int x = 0; x < (1 << M); ++x) gi.gx[x] = (uint64_t)((x >> (M - 1 - i)) & 1);
          bytes += 2.0;
        }
      }
      bool launched = false;
      if (ok) {
        ProfScope ps(pl, st, bytes * sizeof(T), op.begin, op.end, 3, Rf);
        launched = try_launch_pair<T>(g, st) || try_launch_group<T>(g, st);
        ps.cancel = !launched;
      }
      if (!launched)   // no instantiation for this shape: run the steps one by one
        for (int si = op.begin; si < op.end; ++si) run_big<T>(pl, si, ws, j, st);
    } else {
      k_program<T><<<1, kProgramThreads, 0, st>>>(dt.steps, op.begin, op.end, ws, j, dt.progs,
                                                  dt.scalars, nullptr, 0, 0, 0);
    }
    pl->all_launches++;
    if (debug_checks()) {
      const cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess)
        return fail(TN_E_CUDA, std::string("op ") + std::to_string(oi) + " (type " + std::to_string(op.type) +
                                   ", steps " + std::to_string(op.begin) + "-" + std::to_string(op.end) +
                                   "): " + cudaGetErrorString(e));
    }
  }
  CU(cudaGetLastError());
  return TN_OK;
}

template <typename T>
tn_status materialize(tn_plan* pl, const DevTables& dt, const double* gamma, const double* beta,
                      int p, T* ws, cudaStream_t st) {
  Angles ang;
  std::memset(&ang, 0, sizeof(ang));
  for (int l = 0; l < p; ++l) {
    ang.gamma[l] = gamma[l];
    ang.beta[l] = beta[l];
  }
  ang.p = p;
  const int n = (int)pl->leaves.size() * 4;
  if (n > 0)
    k_materialize<T><<<(n + 255) / 256, 256, 0, st>>>(dt.leaves, (int)pl->leaves.size(), ang, nullptr, ws, 0, 0);
  pl->all_launches++;
  CU(cudaGetLastError());
  return TN_OK;
}

tn_status check_call(const tn_plan* plan, int dtype, const double* gamma, const double* beta,
                     int p, void* ws, size_t ws_bytes) {
  if (!plan || !gamma || !beta || !ws) return fail(TN_E_INVAL, "null argument");
  if (dtype != TN_C64 && dtype != TN_C128) return fail(TN_E_DTYPE, "unsupported dtype");
  if (p != plan->h.p) return fail(TN_E_INVAL, "p does not match the plan");
  if (ws_bytes < ws_bytes_for(plan->h, dtype)) return fail(TN_E_INVAL, "workspace too small");
  if ((reinterpret_cast<uintptr_t>(ws) & 255) != 0) return fail(TN_E_INVAL, "workspace must be 256-byte aligned");
  return TN_OK;
}

template <typename T>
tn_status sliced_impl(tn_plan* pl, const double* gamma, const double* beta, int p, uint64_t begin,
                      uint64_t end, void* wsv, size_t ws_bytes, cudaStream_t st, double* partials_dev) {
  DevTables* dt = nullptr;
  tn_status s = ensure_dev(pl, &dt);
  if (s != TN_OK) return s;
  T* ws = static_cast<T*>(wsv);
  if ((s = materialize<T>(pl, *dt, gamma, beta, p, ws, st)) != TN_OK) return s;
  const ProgramRec& pr = pl->progs[0];
  if ((s = run_ops<T>(pl, *dt, pr.opA_begin, pr.opA_end, ws, 0, st)) != TN_OK) return s;
  // batched slices: every per-slice step runs in the interpreter -> one launch
  // runs up to nb slices, each CTA in its own window for the per-slice tensors
  const size_t es = sizeof(T);
  const size_t base_bytes = ws_bytes_for(pl->h, es == 8 ? TN_C64 : TN_C128);
  const uint64_t win_bytes = pl->h.arena_elems * es;
  uint64_t nb = 1;
  if (pl->batchable && win_bytes > 0 && ws_bytes > base_bytes)
    nb = 1 + (ws_bytes - base_bytes) / win_bytes;
  if (pl->batchable && nb >= 2) {
    const uint64_t win0 = base_bytes / es;
    for (uint64_t j = begin; j < end; j += nb) {
      const uint64_t cnt = std::min<uint64_t>(nb, end - j);
      k_program<T><<<(unsigned)cnt, kProgramThreads, 0, st>>>(dt->steps, 0, 0, ws, j, dt->progs, dt->scalars,
                                                               reinterpret_cast<double2*>(partials_dev), 2,
                                                               win0, pl->h.arena_elems);
      pl->all_launches++;
    }
    CU(cudaGetLastError());
    return TN_OK;
  }
  for (uint64_t j = begin; j < end; ++j) {
    if ((s = run_ops<T>(pl, *dt, pr.opB_begin, pr.opB_end, ws, j, st)) != TN_OK) return s;
    k_finalize<T><<<1, 32, 0, st>>>(dt->scalars, pr.scal_begin, pr.scal_end, ws, j, pr.log2_scale,
                                   partials_dev + 2 * j);
    pl->all_launches++;
  }
  CU(cudaGetLastError());
  return TN_OK;
}

double* scratch_ptr(const tn_plan* pl, int dtype, void* ws) {
  const size_t es = dtype == TN_C64 ? 8 : 16;
  return reinterpret_cast<double*>(static_cast<uint8_t*>(ws) + align256(pl->h.arena_elems * es));
}

}  // namespace

// ============================================================== C ABI: contraction
extern "C" tn_status tn_contract_sliced(const tn_plan* plan, tn_dtype dtype, const double* gamma,
                                        const double* beta, int32_t p, uint64_t begin, uint64_t end,
                                        void* ws, size_t ws_bytes, void* stream,
                                        double* partials_dev) {
  tn_status s = check_call(plan, dtype, gamma, beta, p, ws, ws_bytes);
  if (s != TN_OK) return s;
  if (plan->h.kind != TN_KIND_AMPLITUDE) return fail(TN_E_INVAL, "not an amplitude plan");
  if (!partials_dev) return fail(TN_E_INVAL, "null partials");
  if (begin > end || end > (1ull << plan->h.k)) return fail(TN_E_INVAL, "bad slice range");
  tn_plan* pl = const_cast<tn_plan*>(plan);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  return dtype == TN_C64 ? sliced_impl<float2>(pl, gamma, beta, p, begin, end, ws, ws_bytes, st, partials_dev)
                         : sliced_impl<double2>(pl, gamma, beta, p, begin, end, ws, ws_bytes, st, partials_dev);
}

extern "C" tn_status tn_contract(const tn_plan* plan, tn_dtype dtype, const double* gamma,
                                 const double* beta, int32_t p, void* ws, size_t ws_bytes,
                                 void* stream, double out[2]) {
  tn_status s = check_call(plan, dtype, gamma, beta, p, ws, ws_bytes);
  if (s != TN_OK) return s;
  if (!out) return fail(TN_E_INVAL, "null out");
  if (plan->h.kind != TN_KIND_AMPLITUDE) return fail(TN_E_INVAL, "not an amplitude plan");
  const uint64_t n = 1ull << plan->h.k;
  double* scratch = scratch_ptr(plan, dtype, ws);
  s = tn_contract_sliced(plan, dtype, gamma, beta, p, 0, n, ws, ws_bytes, stream, scratch);
  if (s != TN_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // scratch: 2*max(n, E) doubles of partials, then the pairwise result in the trailing pad
  double* res = reinterpret_cast<double*>(reinterpret_cast<uint8_t*>(scratch) + align256(16 * std::max<uint64_t>(n, plan->h.n_programs)));
  k_pairwise<<<1, 32, 0, st>>>(scratch, n, res);
  const_cast<tn_plan*>(plan)->all_launches++;
  CU(cudaGetLastError());
  CU(cudaMemcpyAsync(out, res, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  return TN_OK;
}

template <typename T>
tn_status energy_impl(tn_plan* pl, const double* gammas, const double* betas, int p, uint64_t B,
                      void* wsv, cudaStream_t st, double* zz, double* zz_imag_max, double* energy) {
  DevTables* dt = nullptr;
  tn_status s;
  if ((s = ensure_dev(pl, &dt)) != TN_OK) return s;
  T* ws = static_cast<T*>(wsv);
  const size_t es = sizeof(T);
  const int E = pl->h.n_programs;
  const size_t base_bytes = ws_bytes_for(pl->h, es == 8 ? TN_C64 : TN_C128);
  const uint64_t win0 = base_bytes / es;
  uint8_t* tail = static_cast<uint8_t*>(wsv) + base_bytes + (B > 1 ? (B - 1) * pl->h.arena_elems * es : 0);
  double2* results = B > 1 ? reinterpret_cast<double2*>(tail)
                           : reinterpret_cast<double2*>(scratch_ptr(pl, es == 8 ? TN_C64 : TN_C128, wsv));
  Angles* dang = B > 1 ? reinterpret_cast<Angles*>(tail + align256(16 * B * (uint64_t)E)) : nullptr;
  std::vector<Angles> hang(B);
  for (uint64_t b = 0; b < B; ++b) {
    std::memset(&hang[b], 0, sizeof(Angles));
    for (int l = 0; l < p; ++l) {
      hang[b].gamma[l] = gammas[b * p + l];
      hang[b].beta[l] = betas[b * p + l];
    }
    hang[b].p = p;
  }
  if (dang) CU(cudaMemcpyAsync(dang, hang.data(), sizeof(Angles) * B, cudaMemcpyHostToDevice, st));
  const int n = (int)pl->leaves.size() * 4;
  if (n > 0) {
    dim3 grid((n + 255) / 256, (unsigned)B);
    k_materialize<T><<<grid, 256, 0, st>>>(dt->leaves, (int)pl->leaves.size(), hang[0], dang, ws, win0,
                                           pl->h.arena_elems);
  }
  dim3 grid((unsigned)E, (unsigned)B);
  k_program<T><<<grid, kProgramThreads, 0, st>>>(dt->steps, 0, 0, ws, 0, dt->progs, dt->scalars, results, 1,
                                                 win0, pl->h.arena_elems);
  pl->all_launches += 2;
  CU(cudaGetLastError());
  std::vector<double> h(2 * (size_t)E * B);
  CU(cudaMemcpyAsync(h.data(), results, h.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  for (uint64_t b = 0; b < B; ++b) {
    double im = 0.0, en = 0.0;
    for (int e = 0; e < E; ++e) {
      const double re = h[2 * (b * E + e)], ie = h[2 * (b * E + e) + 1];
      zz[b * E + e] = re;
      im = std::max(im, std::fabs(ie));
      en += (1.0 - re) / 2.0;
    }
    if (zz_imag_max) zz_imag_max[b] = im;
    if (energy) energy[b] = en;
  }
  return TN_OK;
}

extern "C" tn_status tn_energy_batch(const tn_plan* plan, tn_dtype dtype, const double* gammas,
                                     const double* betas, int32_t p, uint64_t batch, void* ws,
                                     size_t ws_bytes, void* stream, double* zz, double* zz_imag_max,
                                     double* energy) {
  tn_status s = check_call(plan, dtype, gammas, betas, p, ws, ws_bytes);
  if (s != TN_OK) return s;
  if (plan->h.kind != TN_KIND_ENERGY) return fail(TN_E_INVAL, "not an energy plan");
  if (!zz || batch < 1 || batch > 65535) return fail(TN_E_INVAL, "bad zz / batch");
  if (ws_bytes < ws_bytes_batched(plan->h, dtype, batch)) return fail(TN_E_INVAL, "workspace too small for the batch");
  tn_plan* pl = const_cast<tn_plan*>(plan);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  return dtype == TN_C64 ? energy_impl<float2>(pl, gammas, betas, p, batch, ws, st, zz, zz_imag_max, energy)
                         : energy_impl<double2>(pl, gammas, betas, p, batch, ws, st, zz, zz_imag_max, energy);
}

extern "C" tn_status tn_energy(const tn_plan* plan, tn_dtype dtype, const double* gamma,
                               const double* beta, int32_t p, void* ws, size_t ws_bytes,
                               void* stream, double* zz, double* zz_imag_max, double* energy) {
  return tn_energy_batch(plan, dtype, gamma, beta, p, 1, ws, ws_bytes, stream, zz, zz_imag_max, energy);
}

extern "C" tn_status tn_eliminate(tn_dtype dtype, int32_t n_in, const void* const* in_dev,
                                  const uint64_t* out_mask, const int32_t* pv, void* out_dev,
                                  int32_t out_rank, void* stream) {
  if (n_in < 1 || n_in > kMaxIn || !in_dev || !out_mask || !pv || !out_dev)
    return fail(TN_E_INVAL, "tn_eliminate: bad argument");
  if (out_rank < 0 || out_rank > 40) return fail(TN_E_INVAL, "tn_eliminate: out_rank out of range");
  if (dtype != TN_C64 && dtype != TN_C128) return fail(TN_E_DTYPE, "unsupported dtype");
  BigArgs a;
  std::memset(&a, 0, sizeof(a));
  a.out = out_dev;
  a.out_rank = out_rank;
  a.n_in = n_in;
  for (int t = 0; t < n_in; ++t) {
    if (!in_dev[t] || pv[t] < 0 || pv[t] > 62) return fail(TN_E_INVAL, "tn_eliminate: bad input");
    if (out_rank < 64 && (out_mask[t] >> out_rank) != 0) return fail(TN_E_INVAL, "tn_eliminate: mask beyond out_rank");
    if (pv[t] > __builtin_popcountll(out_mask[t])) return fail(TN_E_INVAL, "tn_eliminate: pv beyond input rank");
    a.in[t] = in_dev[t];
    a.out_mask[t] = out_mask[t];
    a.pv[t] = (uint32_t)pv[t];
    const int r_in = __builtin_popcountll(out_mask[t]) + 1;
    a.flags[t] = (r_in + 2 >= out_rank && out_rank >= 16) ? 1u : 0u;  // as the lowering
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (out_rank == 0) {
    // a scalar output: route through the interpreter-style path of the standalone kernel is
    // not possible (VEC pairs); use a one-step program in a temporary device record
    StepRec rec;
    std::memset(&rec, 0, sizeof(rec));
    rec.out_rank = 0;
    rec.n_in = n_in;
    StepRec* d = nullptr;
    CU(cudaMallocAsync((void**)&d, sizeof(StepRec), st));
    // offsets relative to a null base: encode absolute element addresses
    const size_t es = dtype == TN_C64 ? 8 : 16;
    rec.out_off = reinterpret_cast<uintptr_t>(out_dev) / es;
    for (int t = 0; t < n_in; ++t) {
      rec.in[t].off = reinterpret_cast<uintptr_t>(in_dev[t]) / es;
      rec.in[t].out_mask = 0;
      rec.in[t].rank = 1;
      rec.in[t].pv = 0;
    }
    CU(cudaMemcpyAsync(d, &rec, sizeof(rec), cudaMemcpyHostToDevice, st));
    if (dtype == TN_C64)
      k_program<float2><<<1, 32, 0, st>>>(d, 0, 1, nullptr, 0, nullptr, nullptr, nullptr, 0, 0, 0);
    else
      k_program<double2><<<1, 32, 0, st>>>(d, 0, 1, nullptr, 0, nullptr, nullptr, nullptr, 0, 0, 0);
    CU(cudaFreeAsync(d, st));
    CU(cudaGetLastError());
    return TN_OK;
  }
  if (dtype == TN_C64) launch_bucket<float2>(a, st); else launch_bucket<double2>(a, st);
  CU(cudaGetLastError());
  return TN_OK;
}

extern "C" tn_status tn_profile_enable(tn_plan* plan, int32_t enable) {
  if (!plan) return fail(TN_E_INVAL, "null plan");
  plan->profiling = enable != 0;
  return TN_OK;
}

extern "C" tn_status tn_profile_read(tn_plan* plan, uint64_t* launches, double* total_ms,
                                     double* total_bytes, uint64_t* all_launches) {
  if (!plan) return fail(TN_E_INVAL, "null plan");
  double ms = 0.0, bytes = 0.0;
  for (auto& p : plan->prof) {
    CU(cudaEventSynchronize(p.b));
    float t = 0.f;
    CU(cudaEventElapsedTime(&t, p.a, p.b));
    ms += t;
    bytes += p.bytes;
    plan->ev_pool.push_back(p.a);
    plan->ev_pool.push_back(p.b);
  }
  if (launches) *launches = plan->prof.size();
  if (total_ms) *total_ms = ms;
  if (total_bytes) *total_bytes = bytes;
  if (all_launches) *all_launches = plan->all_launches;
  plan->prof.clear();
  plan->all_launches = 0;
  return TN_OK;
}

extern "C" tn_status tn_profile_records(tn_plan* plan, tn_prof_record_t* out, int64_t cap, int64_t* n) {
  if (!plan || !n) return fail(TN_E_INVAL, "null argument");
  *n = (int64_t)plan->prof.size();
  for (int64_t i = 0; out && i < cap && i < *n; ++i) {
    ProfRec& p = plan->prof[i];
    CU(cudaEventSynchronize(p.b));
    float t = 0.f;
    CU(cudaEventElapsedTime(&t, p.a, p.b));
    out[i].step_begin = p.step_begin;
    out[i].step_end = p.step_end;
    out[i].kind = p.kind;
    out[i].out_rank = p.out_rank;
    out[i].ms = t;
    out[i].bytes = p.bytes;
  }
  return TN_OK;
}

extern "C" const char* tn_last_error(void) { return g_err.c_str(); }
extern "C" int32_t tn_version(void) { return (int32_t)kPlanVersion; }
