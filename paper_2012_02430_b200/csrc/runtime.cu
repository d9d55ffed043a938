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
#include <tuple>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/tn_b200.h"
#include "kernels.cuh"
#include "launch.cuh"
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
// a captured tn_contract_sliced body (prefix + slices, all lanes) for one argument set: replayed by
// one cudaGraphLaunch (TNB_GRAPH=0 disables)
struct GraphKey {
  int dtype;
  uintptr_t ws, partials, stream;
  size_t ws_bytes;
  uint64_t begin, end;
  bool operator<(const GraphKey& o) const {
    return std::tie(dtype, ws, partials, stream, ws_bytes, begin, end) <
           std::tie(o.dtype, o.ws, o.partials, o.stream, o.ws_bytes, o.begin, o.end);
  }
};
struct GraphRec {
  cudaGraphExec_t exec = nullptr;
  uint64_t launches = 0;   // kernels in the graph
  bool direct = false;     // capture failed once: always run directly
};

struct DevTables {
  std::map<GraphKey, GraphRec> graphs;
  StepRec* steps = nullptr;
  LeafRec* leaves = nullptr;
  ScalarRec* scalars = nullptr;
  ProgramRec* progs = nullptr;
  uint32_t* fc_sem = nullptr;   // k_gemm_fc split-block counters: [lane][feed op][kFcSemPerOp], zeroed
  cudaStream_t side[kMaxLanes - 1] = {};   // slice lanes 1.. (tn_contract_sliced, one window each)
  cudaEvent_t ev_fork = nullptr, ev_join[kMaxLanes - 1] = {};
  // graphs are captured and replayed on a library stream ordered after / before the caller's (the
  // legacy default stream cannot be captured)
  cudaStream_t cap = nullptr;
  cudaEvent_t ev_cin = nullptr, ev_cout = nullptr;
};

struct ProfRec {
  cudaEvent_t a, b;
  double bytes;
  double flops;        // 8 x 2^(out_rank + M): one complex multiply-add per (output, summed value)
  int32_t step_begin, step_end, kind, out_rank, kernel;
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
  uint64_t graph_launches = 0;   // cudaGraphLaunch calls (each replays a captured slice range)
  bool batchable = false;   // every per-slice op is an interpreter run -> slices can run batched
  std::vector<int32_t> feed_slot;   // per op: index among the OP_GROUP_FEED ops (their fc_sem regions)
  int32_t n_feed = 0;
  std::vector<int32_t> waveA;   // per op: wave of independent prefix ops (-1: phase B), see prefix_waves
  ~tn_plan() {
    for (auto& kv : dev) {
      cudaSetDevice(kv.first);
      cudaFree(kv.second.steps);
      cudaFree(kv.second.leaves);
      cudaFree(kv.second.scalars);
      cudaFree(kv.second.progs);
      cudaFree(kv.second.fc_sem);
      for (int l = 0; l < kMaxLanes - 1; ++l) {
        if (kv.second.side[l]) cudaStreamDestroy(kv.second.side[l]);
        if (kv.second.ev_join[l]) cudaEventDestroy(kv.second.ev_join[l]);
      }
      if (kv.second.ev_fork) cudaEventDestroy(kv.second.ev_fork);
      if (kv.second.cap) cudaStreamDestroy(kv.second.cap);
      if (kv.second.ev_cin) cudaEventDestroy(kv.second.ev_cin);
      if (kv.second.ev_cout) cudaEventDestroy(kv.second.ev_cout);
      for (auto& g : kv.second.graphs)
        if (g.second.exec) cudaGraphExecDestroy(g.second.exec);
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
  const uint64_t nres = std::max<uint64_t>(nsl, (uint64_t)h.n_programs) << h.n_open;
  return align256(h.arena_elems * es) + align256(16 * nres) + align256(16ull << h.n_open);
}

}  // namespace

// ============================================================== C ABI: planning
// step-dependent slicing scan (Fig. slice_algo; Fig. hist_of_cost)
extern "C" tn_status tn_slice_scan(int32_t n_qubits, int32_t n_edges, const int32_t* edges, int32_t p,
                                   const tn_build_opts* opts, int32_t* s_out, int32_t* width_out,
                                   double* cost_out, int32_t cap, int32_t* n_out, int32_t* peak_out) {
  if (!opts || !n_out || (n_edges > 0 && !edges) || n_qubits <= 0 || n_edges < 0 || cap < 0)
    return fail(TN_E_INVAL, "tn_slice_scan: null or negative argument");
  if (p < 1 || p > kMaxP) return fail(TN_E_INVAL, "tn_slice_scan: p out of range [1, 16]");
  if (opts->kind != TN_KIND_AMPLITUDE) return fail(TN_E_INVAL, "tn_slice_scan: amplitude networks only");
  if (opts->orderer < TN_ORDER_MIN_FILL || opts->orderer > TN_ORDER_RGREEDY_FILL)
    return fail(TN_E_INVAL, "tn_slice_scan: unknown orderer");
  if (opts->n_sliced < 1 || opts->n_sliced > 30 || opts->r < 0)
    return fail(TN_E_INVAL, "tn_slice_scan: n_sliced must be in [1, 30], r >= 0");
  if (cap > 0 && (!s_out || !width_out || !cost_out)) return fail(TN_E_INVAL, "tn_slice_scan: null output");
  OrderSpec spec;
  spec.orderer = opts->orderer;
  spec.q = opts->rg_q == 0 ? 8 : opts->rg_q;
  spec.tau = opts->rg_tau_milli == 0 ? 0.5 : opts->rg_tau_milli / 1000.0;
  spec.seed = opts->rg_seed;
  try {
    std::vector<int> ev(edges, edges + 2 * (size_t)n_edges);
    std::vector<int> opened;
    for (int i = 0; i < opts->n_open; ++i) opened.push_back(opts->open_qubits[i]);
    const Network net = build_amplitude_network(n_qubits, ev, p, opened);
    std::vector<SliceCandidate> scan;
    int peak = -1;
    (void)slice_search(BitGraph::from_network(net), opts->n_sliced, opts->r, spec, &scan, &peak);
    *n_out = (int32_t)scan.size();
    if (peak_out) *peak_out = peak;
    for (int i = 0; i < (int)scan.size() && i < cap; ++i) {
      s_out[i] = scan[i].s;
      width_out[i] = scan[i].width;
      cost_out[i] = scan[i].cost;
    }
    return TN_OK;
  } catch (const std::invalid_argument& e) {
    return fail(TN_E_PLAN, std::string("tn_slice_scan: ") + e.what());
  } catch (const std::exception& e) {
    return fail(TN_E_NOMEM, std::string("tn_slice_scan: ") + e.what());
  }
}

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
    std::vector<int> opened;
    if (opts->n_open < 0 || opts->n_open > 20 || (opts->n_open > 0 && !opts->open_qubits))
      return fail(TN_E_INVAL, "tn_plan_build: n_open must be in [0, 20] with open_qubits given");
    if (opts->n_open > 0 && opts->kind != TN_KIND_AMPLITUDE)
      return fail(TN_E_INVAL, "tn_plan_build: open qubits need an amplitude plan");
    for (int i = 0; i < opts->n_open; ++i) opened.push_back(opts->open_qubits[i]);
    if (opts->kind == TN_KIND_AMPLITUDE) {
      nets.push_back(build_amplitude_network(n_qubits, ev, p, opened));
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
        h.n_open = (int32_t)net.open_labels.size();
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
  if (h.k < 0 || h.k > 30 || h.p < 1 || h.p > kMaxP || h.n_programs < 1 || h.n_open < 0 || h.n_open > 20)
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
  const int n_ops = (int)pl->ops.size();
  for (int oi = 0; oi < n_ops; ++oi) {
    const OpRec& o = pl->ops[oi];
    if (o.begin < 0 || o.end > h.n_steps || o.begin >= o.end ||
        (o.type != OP_BIG && o.type != OP_RUN && o.type != OP_CHAIN && o.type != OP_GROUP && o.type != OP_PRUN &&
         o.type != OP_GROUP_FEED) ||
        ((o.type == OP_GROUP || o.type == OP_GROUP_FEED) && (o.end - o.begin > kMaxGroupPlan || o.end - o.begin < 2)) ||
        (o.type == OP_GROUP_FEED && (oi + 1 >= n_ops || (pl->ops[oi + 1].type != OP_GROUP && pl->ops[oi + 1].type != OP_GROUP_FEED))) ||
        (o.type == OP_CHAIN && (o.end - o.begin > kMaxChain || pl->steps[o.end - 1].out_rank < 1)) ||
        (o.type == OP_BIG && pl->steps[o.begin].out_rank < 1))
      return fail(TN_E_PLAN, "tn_plan_load: bad op record");
  }
  for (const auto& s : pl->scalars)
    if ((s.slice_mask >> h.k) != 0 || (s.open_mask >> h.n_open) != 0 ||
        s.off + (1ull << (__builtin_popcount(s.slice_mask) + __builtin_popcount(s.open_mask))) > A)
      return fail(TN_E_PLAN, "tn_plan_load: bad scalar record");
  for (const auto& pr : pl->progs)
    if (pr.stepB_begin < 0 || pr.stepB_end > h.n_steps || pr.scal_begin < 0 || pr.scal_end > h.n_scalars ||
        pr.opA_begin < 0 || pr.opB_end > h.n_ops)
      return fail(TN_E_PLAN, "tn_plan_load: bad program record");
  pl->batchable = pl->h.kind == TN_KIND_AMPLITUDE && pl->h.n_programs == 1 && pl->h.n_open == 0;
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
  o->n_open = h.n_open;
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
    if (op.type == OP_BIG || op.type == OP_CHAIN || op.type == OP_GROUP || op.type == OP_GROUP_FEED)
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

extern "C" tn_status tn_sum_partials(const tn_plan* plan, const double* partials, double* out) {
  if (!plan || !partials || !out) return fail(TN_E_INVAL, "tn_sum_partials: null argument");
  const uint64_t n = 1ull << plan->h.k;
  const uint64_t A = 1ull << plan->h.n_open;
  std::vector<double> buf(2 * n);
  for (uint64_t o = 0; o < A; ++o) {        // batch entry o: fixed pairwise tree over j
    for (uint64_t j = 0; j < n; ++j) {
      buf[2 * j] = partials[2 * (j * A + o)];
      buf[2 * j + 1] = partials[2 * (j * A + o) + 1];
    }
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
    out[2 * o] = buf[0];
    out[2 * o + 1] = buf[1];
  }
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
    pl->feed_slot.assign(pl->ops.size(), 0);
    pl->n_feed = 0;
    for (size_t oi = 0; oi < pl->ops.size(); ++oi)
      if (pl->ops[oi].type == OP_GROUP_FEED) pl->feed_slot[oi] = pl->n_feed++;
    {
      const size_t sem_bytes = (size_t)kMaxLanes * std::max(pl->n_feed, 1) * kFcSemPerOp * sizeof(uint32_t);
      CU(cudaMalloc((void**)&t.fc_sem, sem_bytes));
      CU(cudaMemset(t.fc_sem, 0, sem_bytes));
    }
    for (int l = 0; l < kMaxLanes - 1; ++l) {
      CU(cudaStreamCreateWithFlags(&t.side[l], cudaStreamNonBlocking));
      CU(cudaEventCreateWithFlags(&t.ev_join[l], cudaEventDisableTiming));
    }
    CU(cudaEventCreateWithFlags(&t.ev_fork, cudaEventDisableTiming));
    CU(cudaStreamCreateWithFlags(&t.cap, cudaStreamNonBlocking));
    CU(cudaEventCreateWithFlags(&t.ev_cin, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&t.ev_cout, cudaEventDisableTiming));
    it = pl->dev.emplace(dev, t).first;
  }
  *out = &it->second;
  return TN_OK;
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
  return try_launch_gemm<T>(g, st) || try_launch_group<T>(g, st);
}

template <typename T>
void launch_bucket(const BigArgs& a, cudaStream_t st) {
  if (try_launch_specialised<T>(a, st)) return;
  launch_bucket_generic<T>(a, st);
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

// window b of the workspace (b >= 1): win0 + (b - 1) * arena elements (as k_program's window_rel)
inline uint64_t window_rel_host(uint64_t b, uint64_t win0, uint64_t win_elems) {
  return b == 0 ? 0ull : win0 + (b - 1) * win_elems;
}

// element offset of input `in` for slice j in the slice window at `rel` (per-slice tensors, F_REL,
// live in the window; leaves and prefix outputs are shared)
template <typename T>
uint64_t in_off(const InRec& in, uint64_t j, uint64_t rel) {
  return in.off + slice_off_of<T>(in, j) + ((in.flags & F_REL) ? rel : 0ull);
}
// output of a step: phase-B outputs are per-slice
inline uint64_t out_off(const StepRec& s, uint64_t rel) { return s.out_off + (s.phase == 1 ? rel : 0ull); }

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
    pr.flops = kind == 4 ? 0.0 : 8.0 * std::ldexp(1.0, out_rank + (e - b));
    last_kernel() = KID_NONE;
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
    pr.kernel = last_kernel();
    pl->prof.push_back(pr);
  }
};

// one standalone bucket step (k_group_t with M = 1, else the generic k_bucket)
template <typename T>
void run_big(tn_plan* pl, int si, T* ws, uint64_t j, cudaStream_t st, uint64_t rel) {
  const StepRec& s = pl->steps[si];
  BigArgs a;
  std::memset(&a, 0, sizeof(a));
  a.out = ws + out_off(s, rel);
  a.out_rank = s.out_rank;
  a.n_in = s.n_in;
  double bytes = std::ldexp((double)sizeof(T), s.out_rank);
  for (int t = 0; t < s.n_in; ++t) {
    const InRec& in = s.in[t];
    a.in[t] = ws + in_off<T>(in, j, rel);
    a.out_mask[t] = in.out_mask;
    a.pv[t] = in.pv;
    a.flags[t] = in.flags | ((t == 0 && s.inplace) ? 1u : 0u);
    bytes += std::ldexp((double)sizeof(T), (int)in.rank);
  }
  ProfScope ps(pl, st, bytes, si, si + 1, 1, s.out_rank);
  launch_bucket<T>(a, st);
}

// the GDesc of a fused merge group (OP_GROUP / OP_GROUP_FEED): head step + (M-1) in-place reduce
// followers whose other inputs are rank-1 weights on their summed index
template <typename T>
bool group_desc(const tn_plan* pl, const OpRec& op, T* ws, uint64_t j, uint64_t rel, GDesc& g, double& bytes) {
  const StepRec& h = pl->steps[op.begin];
  const StepRec& last = pl->steps[op.end - 1];
  std::memset(&g, 0, sizeof(g));
  const int M = op.end - op.begin;
  const int Rf = last.out_rank;
  const uint64_t low = (1ull << Rf) - 1, xrest = (1ull << (M - 1)) - 1;
  const uint64_t hfull = (1ull << h.out_rank) - 1;
  g.out = ws + out_off(last, rel);
  g.out_rank = Rf;
  g.M = M;
  bytes = std::ldexp(1.0, Rf);
  for (int t = 0; t < h.n_in; ++t) {
    const InRec& in = h.in[t];
    GIn& gi = g.in[g.n++];
    gi.ptr = ws + in_off<T>(in, j, rel);
    gi.out_mask = in.out_mask & low;
    gi.pv = in.pv;
    gi.rank = in.rank;
    gi.full = in.out_mask == hfull;
    for (int x = 0; x < (1 << M); ++x)
      gi.gx[x] = host_fmap(((uint64_t)x & xrest) << Rf, in.out_mask, in.pv) +
                 ((uint64_t)((x >> (M - 1)) & 1) << in.pv);
    bytes += std::ldexp(1.0, (int)in.rank);
  }
  for (int i = 1; i < M; ++i) {
    const StepRec& sk = pl->steps[op.begin + i];
    for (int k = 1; k < sk.n_in; ++k) {
      if (g.n >= kMaxIn) return false;
      GIn& gi = g.in[g.n++];
      gi.ptr = ws + in_off<T>(sk.in[k], j, rel);
      gi.out_mask = 0;
      gi.pv = 0;
      gi.rank = 1;
      gi.full = false;
      for (int x = 0; x < (1 << M); ++x) gi.gx[x] = (uint64_t)((x >> (M - 1 - i)) & 1);
      bytes += 2.0;
    }
  }
  return true;
}

template <typename T>
tn_status run_ops(tn_plan* pl, const DevTables& dt, int op_b, int op_e, T* ws, uint64_t j, uint64_t rel,
                  cudaStream_t st, int lane = 0) {
  for (int oi = op_b; oi < op_e; ++oi) {
    const OpRec& op = pl->ops[oi];
    if (op.type == OP_BIG) {
      run_big<T>(pl, op.begin, ws, j, st, rel);
    } else if (op.type == OP_CHAIN) {
      const StepRec& h = pl->steps[op.begin];
      const StepRec& last = pl->steps[op.end - 1];
      ChainArgs c;
      std::memset(&c, 0, sizeof(c));
      c.m = op.end - op.begin;
      c.out = ws + out_off(last, rel);
      c.out_rank = last.out_rank;
      c.A = ws + in_off<T>(h.in[0], j, rel);
      for (int i = 0; i < c.m; ++i) {
        const StepRec& sk = pl->steps[op.begin + i];
        c.nw[i] = sk.n_in - 1;
        for (int k = 1; k < sk.n_in; ++k) c.w[i][k - 1] = ws + in_off<T>(sk.in[k], j, rel);
      }
      const double bytes = (std::ldexp(1.0, (int)h.in[0].rank) + std::ldexp(1.0, c.out_rank)) * sizeof(T);
      ProfScope ps(pl, st, bytes, op.begin, op.end, 2, c.out_rank);
      constexpr int VEC = VecT<T>::n;
      const uint64_t work = ((1ull << c.out_rank) + VEC - 1) / VEC;
      const uint64_t blocks = (work + kBucketThreads - 1) / kBucketThreads;
      if (blocks < (uint64_t)num_sms() * 2 && c.m >= 3) {
        // few outputs, many rows: split the rows over the threads of a CTA (k_chain_split)
        // output vectors per CTA: enough CTAs for ~3 per SM (each thread then sums fewer rows,
        // more loads in flight per SM); at least 8 lanes (128 contiguous bytes) per row group
        const uint64_t n_vec = ((1ull << c.out_rank) + VEC - 1) / VEC;
        static const int nv_env = [] { const char* e = std::getenv("TNB_CHAIN_NV"); return e ? std::atoi(e) : 0; }();
        int nv = 32;
        while (nv > 8 && n_vec / (uint64_t)nv < 3ull * (uint64_t)num_sms()) nv >>= 1;
        if (nv_env >= 1 && nv_env <= 32) nv = nv_env;
        c.nv = nv;
        const uint64_t nblk = std::max<uint64_t>(1, n_vec / (uint64_t)nv);
        const unsigned g2 = (unsigned)std::min<uint64_t>(nblk, (uint64_t)num_sms() * 8);
        k_chain_split<T><<<g2, kBucketThreads, 0, st>>>(c);
        last_kernel() = KID_CHAIN_SPLIT;
      } else {
        const unsigned grid = (unsigned)std::min<uint64_t>(blocks, (uint64_t)num_sms() * 8);
        k_chain<T><<<grid, kBucketThreads, 0, st>>>(c);
        last_kernel() = KID_CHAIN;
      }
    } else if (op.type == OP_GROUP || op.type == OP_GROUP_FEED) {
      // head step + (M-1) in-place reduce followers with rank-1 weights, summed in one pass
      GDesc g;
      double bytes = 0.0;
      const bool ok = group_desc<T>(pl, op, ws, j, rel, g, bytes);
      if (ok && op.type == OP_GROUP_FEED && fc_enabled()) {
        // producer -> consumer: the next group reads this group's output as a full input; one
        // launch computes it tile by tile and consumes it in registers (k_gemm_fc)
        const OpRec& nx = pl->ops[oi + 1];
        GDesc g3;
        double bytes3 = 0.0;
        if (group_desc<T>(pl, nx, ws, j, rel, g3, bytes3)) {
          int tin = -1;
          for (int t = 0; t < g3.n; ++t)
            if (g3.in[t].ptr == g.out) tin = t;
          if (tin >= 0) {
            const double tb = std::ldexp(1.0, g.out_rank);   // the never-written intermediate
            ProfScope ps(pl, st, (bytes - tb + bytes3 - tb) * sizeof(T), op.begin, nx.end, 3, g3.out_rank);
            ps.pr.flops = 8.0 * (std::ldexp(1.0, g.out_rank + g.M) + std::ldexp(1.0, g3.out_rank + g3.M));
            const bool fused = (std::is_same<T, float2>::value && fc_tc_enabled() && try_launch_fc_tc(g, g3, tin, st)) ||
                               (std::is_same<T, float2>::value && fc_hm_enabled() && try_launch_fc_hm(g, g3, tin, st)) ||
                               try_launch_gemm_fc<T>(g, g3, tin, st,
                                                     dt.fc_sem + ((size_t)lane * std::max(pl->n_feed, 1) + pl->feed_slot[oi]) *
                                                                     kFcSemPerOp);
            ps.cancel = !fused;
            if (fused) {
              ++oi;
              pl->all_launches++;
              continue;
            }
          }
        }
      }
      bool launched = false;
      if (ok) {
        ProfScope ps(pl, st, bytes * sizeof(T), op.begin, op.end, 3, g.out_rank);
        launched = try_launch_gemm<T>(g, st) || try_launch_pair<T>(g, st) || try_launch_group<T>(g, st);
        ps.cancel = !launched;
      }
      if (!launched)   // no instantiation for this shape: run the steps one by one
        for (int si = op.begin; si < op.end; ++si) run_big<T>(pl, si, ws, j, st, rel);
    } else {
      double bytes = 0.0;
      for (int si = op.begin; si < op.end; ++si) {
        const StepRec& sk = pl->steps[si];
        bytes += std::ldexp((double)sizeof(T), sk.out_rank);
        for (int t = 0; t < sk.n_in; ++t) bytes += std::ldexp((double)sizeof(T), (int)sk.in[t].rank);
      }
      ProfScope ps(pl, st, bytes, op.begin, op.end, 4, pl->steps[op.end - 1].out_rank);
      if (op.type == OP_PRUN)   // independent steps of one prefix level: one CTA each
        k_program<T><<<(unsigned)(op.end - op.begin), kProgramThreads, 0, st>>>(
            dt.steps, op.begin, op.end, ws, j, dt.progs, dt.scalars, nullptr, 3, rel, 0);
      else
        k_program<T><<<1, kProgramThreads, 0, st>>>(dt.steps, op.begin, op.end, ws, j, dt.progs,
                                                    dt.scalars, nullptr, 0, rel, 0);
      last_kernel() = KID_PROGRAM;
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

// Prefix (phase A) ops in waves: consecutive ops that neither read nor write memory another op of
// the wave writes (the planner level-sorts phase A and releases a level's memory only when the level
// ends, so the ops of one dependency level form a wave).  A wave of >= 2 ops runs on forked streams:
// the prefix's critical path becomes its dependency depth instead of its op count.
inline void prefix_waves(tn_plan* pl) {
  std::lock_guard<std::mutex> lk(pl->mu);
  if (!pl->waveA.empty()) return;
  pl->waveA.assign(pl->ops.size(), -1);
  std::vector<std::pair<uint64_t, uint64_t>> rd, wr;
  int wave = 0;
  auto hit = [](const std::vector<std::pair<uint64_t, uint64_t>>& v, uint64_t lo, uint64_t hi) {
    for (const auto& x : v)
      if (lo < x.second && x.first < hi) return true;
    return false;
  };
  for (size_t oi = 0; oi < pl->ops.size(); ++oi) {
    const OpRec& op = pl->ops[oi];
    if (op.phase != 0) continue;
    std::vector<std::pair<uint64_t, uint64_t>> r2, w2;
    for (int si = op.begin; si < op.end; ++si) {
      const StepRec& st = pl->steps[si];
      w2.push_back({st.out_off, st.out_off + (1ull << st.out_rank)});
      for (int t = 0; t < st.n_in; ++t)
        r2.push_back({st.in[t].off, st.in[t].off + (1ull << (st.in[t].rank + __builtin_popcount(st.in[t].slice_mask)))});
    }
    bool conflict = false;
    for (const auto& x : w2) conflict = conflict || hit(rd, x.first, x.second) || hit(wr, x.first, x.second);
    for (const auto& x : r2) conflict = conflict || hit(wr, x.first, x.second);
    if (conflict) { ++wave; rd.clear(); wr.clear(); }
    rd.insert(rd.end(), r2.begin(), r2.end());
    wr.insert(wr.end(), w2.begin(), w2.end());
    pl->waveA[oi] = wave;
  }
}

template <typename T>
tn_status sliced_body(tn_plan* pl, DevTables* dt, uint64_t begin, uint64_t end, void* wsv, size_t ws_bytes,
                      cudaStream_t st, double* partials_dev);

// phase A: waves of independent ops on forked streams (TNB_PREFIX_WAVES=0: one stream)
template <typename T>
tn_status run_prefix(tn_plan* pl, DevTables* dt, int op_b, int op_e, T* ws, cudaStream_t st) {
  static const bool waves = !(std::getenv("TNB_PREFIX_WAVES") && std::getenv("TNB_PREFIX_WAVES")[0] == '0');
  if (!waves || pl->profiling) return run_ops<T>(pl, *dt, op_b, op_e, ws, 0, 0, st);
  prefix_waves(pl);
  tn_status s;
  int oi = op_b;
  while (oi < op_e) {
    int oe = oi + 1;
    while (oe < op_e && pl->waveA[oe] == pl->waveA[oi]) ++oe;
    const int n = std::min(oe - oi, kMaxLanes);
    if (n < 2) {
      if ((s = run_ops<T>(pl, *dt, oi, oe, ws, 0, 0, st)) != TN_OK) return s;
      oi = oe;
      continue;
    }
    CU(cudaEventRecord(dt->ev_fork, st));
    for (int k = 1; k < n; ++k) CU(cudaStreamWaitEvent(dt->side[k - 1], dt->ev_fork, 0));
    for (int k = 0; k < oe - oi; ++k) {
      cudaStream_t sk = (k % n) == 0 ? st : dt->side[(k % n) - 1];
      if ((s = run_ops<T>(pl, *dt, oi + k, oi + k + 1, ws, 0, 0, sk)) != TN_OK) return s;
    }
    for (int k = 1; k < n; ++k) {
      CU(cudaEventRecord(dt->ev_join[k - 1], dt->side[k - 1]));
      CU(cudaStreamWaitEvent(st, dt->ev_join[k - 1], 0));
    }
    oi = oe;
  }
  return TN_OK;
}

inline bool graphs_enabled() {
  const char* v = std::getenv("TNB_GRAPH");
  return !(v && v[0] == '0') && !env_flag("TNB_FT_TRACE") && !debug_checks();
}

// leaves from (gamma, beta) (a direct launch: the angles change every call), then the prefix and
// the slices -- captured once per argument set into a CUDA graph and replayed (host enqueue of one
// contraction: one graph launch instead of ~15 launches per slice)
template <typename T>
tn_status sliced_impl(tn_plan* pl, const double* gamma, const double* beta, int p, uint64_t begin,
                      uint64_t end, void* wsv, size_t ws_bytes, cudaStream_t st, double* partials_dev) {
  DevTables* dt = nullptr;
  tn_status s = ensure_dev(pl, &dt);
  if (s != TN_OK) return s;
  T* ws = static_cast<T*>(wsv);
  if ((s = materialize<T>(pl, *dt, gamma, beta, p, ws, st)) != TN_OK) return s;
  if (pl->profiling || !graphs_enabled())
    return sliced_body<T>(pl, dt, begin, end, wsv, ws_bytes, st, partials_dev);
  const GraphKey key{sizeof(T) == 8 ? 0 : 1, reinterpret_cast<uintptr_t>(wsv), reinterpret_cast<uintptr_t>(partials_dev),
                     reinterpret_cast<uintptr_t>(st), ws_bytes, begin, end};
  GraphRec rec;
  {
    // the first call with an argument set runs directly (single-shot calls never pay for a
    // capture); the second captures, later ones replay
    std::lock_guard<std::mutex> lk(pl->mu);
    auto it = dt->graphs.find(key);
    if (it == dt->graphs.end()) {
      if (dt->graphs.size() >= 256) {   // bounded cache
        for (auto& g : dt->graphs)
          if (g.second.exec) cudaGraphExecDestroy(g.second.exec);
        dt->graphs.clear();
      }
      dt->graphs[key] = GraphRec{};
      rec.launches = ~0ull;
    } else {
      rec = it->second;
    }
  }
  if (rec.launches == ~0ull || rec.direct) return sliced_body<T>(pl, dt, begin, end, wsv, ws_bytes, st, partials_dev);
  const cudaStream_t cs = dt->cap;
  CU(cudaEventRecord(dt->ev_cin, st));
  CU(cudaStreamWaitEvent(cs, dt->ev_cin, 0));
  if (!rec.exec) {
    const uint64_t l0 = pl->all_launches;
    bool ok = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
    cudaGraph_t graph = nullptr;
    if (ok) {
      s = sliced_body<T>(pl, dt, begin, end, wsv, ws_bytes, cs, partials_dev);
      ok = cudaStreamEndCapture(cs, &graph) == cudaSuccess && s == TN_OK;
      if (ok) ok = cudaGraphInstantiate(&rec.exec, graph, 0) == cudaSuccess;
      if (graph) cudaGraphDestroy(graph);
    }
    const uint64_t captured = pl->all_launches - l0;
    pl->all_launches = l0;   // counted when the graph runs
    if (!ok) {   // run this argument set directly from now on
      (void)cudaGetLastError();
      rec.exec = nullptr;
      rec.direct = true;
      {
        std::lock_guard<std::mutex> lk(pl->mu);
        dt->graphs[key] = rec;
      }
      CU(cudaEventRecord(dt->ev_cout, cs));
      CU(cudaStreamWaitEvent(st, dt->ev_cout, 0));
      return sliced_body<T>(pl, dt, begin, end, wsv, ws_bytes, st, partials_dev);
    }
    rec.launches = captured;
    std::lock_guard<std::mutex> lk(pl->mu);
    dt->graphs[key] = rec;
  }
  CU(cudaGraphLaunch(rec.exec, cs));
  CU(cudaEventRecord(dt->ev_cout, cs));
  CU(cudaStreamWaitEvent(st, dt->ev_cout, 0));
  pl->all_launches += rec.launches;
  pl->graph_launches++;
  return TN_OK;
}

template <typename T>
tn_status sliced_body(tn_plan* pl, DevTables* dt, uint64_t begin, uint64_t end, void* wsv, size_t ws_bytes,
                      cudaStream_t st, double* partials_dev) {
  tn_status s;
  T* ws = static_cast<T*>(wsv);
  const ProgramRec& pr = pl->progs[0];
  if ((s = run_prefix<T>(pl, dt, pr.opA_begin, pr.opA_end, ws, st)) != TN_OK) return s;
  // batched slices: every per-slice step runs in the interpreter -> one launch
  // runs up to nb slices, each CTA in its own window for the per-slice tensors
  const size_t es = sizeof(T);
  const size_t base_bytes = ws_bytes_for(pl->h, es == 8 ? TN_C64 : TN_C128);
  const uint64_t win_bytes = pl->h.arena_elems * es;
  uint64_t nb = 1;
  if (win_bytes > 0 && ws_bytes > base_bytes) nb = 1 + (ws_bytes - base_bytes) / win_bytes;
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
  // L slice lanes when the workspace holds L windows of per-slice tensors: slice j runs on lane
  // (j - begin) % L -- lane 0 on the caller's stream in the base arena, lane l >= 1 on a
  // library-owned stream in window l.  The latency-bound small steps, launch gaps and partial
  // waves of one slice overlap the kernels of the others (slices are independent, Eq. 1).
  const uint64_t L = std::min<uint64_t>({nb, (uint64_t)slice_lanes(), end - begin});
  if (L >= 2) {
    CU(cudaEventRecord(dt->ev_fork, st));
    for (uint64_t l = 1; l < L; ++l) CU(cudaStreamWaitEvent(dt->side[l - 1], dt->ev_fork, 0));
  }
  // every forked side lane joins back into the caller's stream on every exit path, so the caller
  // never reuses ws / partials while a side lane still runs (also after an error)
  struct JoinLanes {
    DevTables* dt;
    cudaStream_t st;
    uint64_t L;
    ~JoinLanes() {
      for (uint64_t l = 1; l < L; ++l) {
        cudaEventRecord(dt->ev_join[l - 1], dt->side[l - 1]);
        cudaStreamWaitEvent(st, dt->ev_join[l - 1], 0);
      }
    }
  } join{dt, st, L};
  for (uint64_t j = begin; j < end; ++j) {
    const uint64_t lane = L >= 2 ? (j - begin) % L : 0;
    cudaStream_t sj = lane ? dt->side[lane - 1] : st;
    const uint64_t rel = lane ? window_rel_host(lane, base_bytes / es, pl->h.arena_elems) : 0ull;
    if ((s = run_ops<T>(pl, *dt, pr.opB_begin, pr.opB_end, ws, j, rel, sj, (int)lane)) != TN_OK) return s;
    {
      const uint32_t A = 1u << pl->h.n_open;
      k_finalize<T><<<(A + 127) / 128, 128, 0, sj>>>(dt->scalars, pr.scal_begin, pr.scal_end, ws, j, pr.log2_scale,
                                                    partials_dev + 2 * (j << pl->h.n_open), rel, pl->h.n_open);
    }
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
                                 void* stream, double* out) {
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
  const uint64_t A = 1ull << plan->h.n_open;
  double* res = reinterpret_cast<double*>(reinterpret_cast<uint8_t*>(scratch) +
                                          align256(16 * (std::max<uint64_t>(n, plan->h.n_programs) * A)));
  k_pairwise<<<(unsigned)((A + 127) / 128), 128, 0, st>>>(scratch, n, A, res);
  const_cast<tn_plan*>(plan)->all_launches++;
  CU(cudaGetLastError());
  CU(cudaMemcpyAsync(out, res, 2 * A * sizeof(double), cudaMemcpyDeviceToHost, st));
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
  // shared-memory-resident cones for a single angle set when the largest cone arena fits (C3 c64:
  // 237 vs 296 us per call); batches keep the L2 path, whose CTAs share an SM (C3 c64 batch of 256:
  // 55 vs 111 us per energy with 187 KB cones); TNB_CONE_SMEM=0: always the L2 path
  uint64_t max_arena = 0;
  for (const auto& pr : pl->progs) max_arena = std::max<uint64_t>(max_arena, pr.arena_end - pr.arena_begin);
  const size_t cone_bytes = (size_t)max_arena * es;
  static const bool cone_smem = !(std::getenv("TNB_CONE_SMEM") && std::getenv("TNB_CONE_SMEM")[0] == '0');
  if (cone_smem && B == 1 && cone_bytes <= 200 * 1024) {
    if (cone_bytes > 48 * 1024) {
      static std::mutex mu;
      std::lock_guard<std::mutex> lk(mu);
      CU(cudaFuncSetAttribute(k_cone_smem<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    }
    k_cone_smem<T><<<grid, kProgramThreads, cone_bytes, st>>>(dt->steps, dt->progs, dt->scalars, ws, results, win0,
                                                              pl->h.arena_elems);
  } else {
    k_program<T><<<grid, kProgramThreads, 0, st>>>(dt->steps, 0, 0, ws, 0, dt->progs, dt->scalars, results, 1,
                                                   win0, pl->h.arena_elems);
  }
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

extern "C" tn_status tn_eliminate_group(tn_dtype dtype, int32_t M, int32_t n_in, const void* const* in_dev,
                                        const uint64_t* out_mask, const uint32_t* x_mask, void* out_dev,
                                        int32_t out_rank, int32_t kernel, void* stream) {
  if (M < 1 || M > kMaxGroup || n_in < 1 || n_in > kMaxIn || !in_dev || !out_mask || !x_mask || !out_dev)
    return fail(TN_E_INVAL, "tn_eliminate_group: bad argument");
  if (out_rank < 11 || out_rank > 40) return fail(TN_E_INVAL, "tn_eliminate_group: out_rank out of range");
  if (dtype != TN_C64 && dtype != TN_C128) return fail(TN_E_DTYPE, "unsupported dtype");
  if (kernel < 0 || kernel > 5) return fail(TN_E_INVAL, "tn_eliminate_group: unknown kernel");
  GDesc g;
  std::memset(&g, 0, sizeof(g));
  g.out = out_dev;
  g.out_rank = out_rank;
  g.M = M;
  g.n = n_in;
  const uint64_t full = (1ull << out_rank) - 1;
  for (int t = 0; t < n_in; ++t) {
    if (!in_dev[t] || (out_mask[t] & ~full) || (x_mask[t] >> M) || x_mask[t] == 0)
      return fail(TN_E_INVAL, "tn_eliminate_group: bad input " + std::to_string(t));
    GIn& gi = g.in[t];
    const int ro = __builtin_popcountll(out_mask[t]);
    const int rx = __builtin_popcount(x_mask[t]);
    gi.ptr = in_dev[t];
    gi.out_mask = out_mask[t];
    gi.pv = (uint32_t)ro;            // inserting a zero bit above every output bit: identity
    gi.rank = (uint32_t)(ro + rx);
    gi.full = out_mask[t] == full;
    for (int x = 0; x < (1 << M); ++x) {
      // held summed indices, x_0 most significant: x_i -> position ro + (number held above... )
      uint64_t off = 0;
      int pos = ro + rx - 1;
      for (int i = 0; i < M; ++i) {
        if (!((x_mask[t] >> i) & 1)) continue;
        if ((x >> (M - 1 - i)) & 1) off += 1ull << pos;   // x's bit (M-1-i) is x_i (x_0 = MSB)
        --pos;
      }
      gi.gx[x] = off;
    }
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  bool ok;
  if (dtype == TN_C64) {
    ok = kernel == 1 ? try_launch_gemm_simt<float2>(g, st)
       : kernel == 4 ? try_launch_gemm_tc(g, st)
       : kernel == 5 ? try_launch_gemm_hm(g, st)
       : kernel == 2 ? try_launch_pair<float2>(g, st)
       : kernel == 3 ? try_launch_group<float2>(g, st)
       : (try_launch_gemm<float2>(g, st) || try_launch_pair<float2>(g, st) || try_launch_group<float2>(g, st));
  } else {
    ok = kernel == 1 ? try_launch_gemm_simt<double2>(g, st)
       : kernel == 5 ? try_launch_gemm_hm64(g, st)
       : kernel == 2 ? try_launch_pair<double2>(g, st)
       : kernel == 3 ? try_launch_group<double2>(g, st)
       : (try_launch_gemm<double2>(g, st) || try_launch_pair<double2>(g, st) || try_launch_group<double2>(g, st));
  }
  if (!ok) return fail(TN_E_INVAL, "tn_eliminate_group: no kernel instantiation for this shape");
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
    out[i].kernel = p.kernel;
    out[i].pad = 0;
    out[i].flops = p.flops;
  }
  return TN_OK;
}

extern "C" const char* tn_last_error(void) { return g_err.c_str(); }
extern "C" int32_t tn_version(void) { return (int32_t)kPlanVersion; }
