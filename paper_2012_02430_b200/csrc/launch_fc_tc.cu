// launch_fc_tc.cu: k_fc_tc (producer -> consumer merge groups, OP_GROUP_FEED, with the producer's
// GEMM on tcgen05) -- part of libtnb200.so (see launch.cuh, kernels_fctc.cuh).  Host side: classify
// T's bits, pick the unit (7 row bits, NB column bits), order the traversal, size the rings.
#include "launch.cuh"
#include "kernels_fctc.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <array>
#include <cmath>
#include <cstdio>
#include <cstring>

namespace tnb {

// TNB_FC_TC=1 / 0 selects k_fc_tc / the FP32 SIMT k_gemm_fc for OP_GROUP_FEED pairs (read per call:
// the parity tests run both kernels in one process); default: kFcTcDefault
constexpr bool kFcTcDefault = false;
bool fc_tc_enabled() {
  const char* v = std::getenv("TNB_FC_TC");
  return v ? v[0] == '1' : kFcTcDefault;
}

// tensor maps of the launch (kernel parameters; unused in the cp.async mode)
struct FtMaps {
  CUtensorMap x, a;
};

template <int M, int NB, int NOB, int NL>
static void launch_ft(const FTArgs& fa, const FtMaps& mp, unsigned grid, size_t smem, cudaStream_t st) {
  allow_smem(k_fc_tc<M, NB, NOB, NL>, smem);
  last_kernel() = KID_FC_TC;
  k_fc_tc<M, NB, NOB, NL><<<grid, kFtThreads, smem, st>>>(fa, mp.x, mp.a);
}

// ---- TMA geometry: a tensor whose bits are "box" bits (the unit's) or traversal bits; dims = runs
// of box bits, each followed by the traversal bits above it (coordinates); the 5th dim takes every
// bit above its start; box bits of further runs become separate copies (at most 8)
struct TmaGeom {
  int ndim = 0;
  uint32_t s[5] = {0, 0, 0, 0, 0}, nt[5] = {0, 0, 0, 0, 0}, nb[5] = {0, 0, 0, 0, 0};
  int ncopy = 1;
  uint32_t cdelta[8][5] = {};
  uint32_t box_elems = 1;
  int smem_bit[64];
};

static bool tma_geom(int Rt, const std::vector<char>& isbox, TmaGeom& G) {
  if (Rt < 1 || Rt > 32 || !isbox[0]) return false;
  std::vector<std::array<int, 3>> runs;   // start, box bits, total bits
  for (int k = 0; k < Rt;) {
    const int st = k;
    int nb = 0;
    while (k < Rt && isbox[k]) { ++nb; ++k; }
    while (k < Rt && !isbox[k]) ++k;
    runs.push_back({st, nb, k - st});
  }
  G.ndim = std::min<int>(5, (int)runs.size());
  for (int& b : G.smem_bit) b = -1;
  int sb = 0;
  for (int d = 0; d < G.ndim; ++d) {
    G.s[d] = (uint32_t)runs[d][0];
    G.nb[d] = (uint32_t)runs[d][1];
    G.nt[d] = d + 1 < G.ndim ? (uint32_t)runs[d][2] : (uint32_t)(Rt - runs[d][0]);
    if (G.nb[d] > 8) return false;   // box dims <= 256
    for (uint32_t i = 0; i < G.nb[d]; ++i) G.smem_bit[G.s[d] + i] = sb++;
  }
  std::vector<int> extra;
  for (size_t r = G.ndim; r < runs.size(); ++r)
    for (int i = 0; i < runs[r][1]; ++i) extra.push_back(runs[r][0] + i);
  if (extra.size() > 3) return false;
  G.box_elems = 1u << sb;
  for (size_t j = 0; j < extra.size(); ++j) G.smem_bit[extra[j]] = sb + (int)j;
  G.ncopy = 1 << extra.size();
  const int last = G.ndim - 1;
  for (int i = 0; i < G.ncopy; ++i)
    for (size_t j = 0; j < extra.size(); ++j)
      if ((i >> j) & 1) G.cdelta[i][last] += 1u << (extra[j] - G.s[last]);
  return (G.box_elems * 8) % 128 == 0;   // every copy lands 128-byte aligned
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

static bool tma_encode(CUtensorMap* map, const void* base, int Rt, const TmaGeom& G) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dim[5], stride[4];
  cuuint32_t box[5], es[5] = {1, 1, 1, 1, 1};
  for (int d = 0; d < 5; ++d) {
    if (d < G.ndim) {
      dim[d] = 1ull << G.nt[d];
      box[d] = 1u << G.nb[d];
    } else {
      dim[d] = 1;
      box[d] = 1;
    }
    if (d >= 1) stride[d - 1] = (d < G.ndim ? (1ull << G.s[d]) : (1ull << Rt)) * 8ull;
  }
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, const_cast<void*>(base), dim, stride, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// instantiated shapes (column bits NB, output column bits NOB, line bits NL): 2^(NOB + NL) <= 32
// accumulators per epilogue thread
template <int M>
static bool dispatch_ft(const FTArgs& fa, const FtMaps& mp, int nb, int nob, int nl, unsigned grid, size_t smem,
                        cudaStream_t st) {
#define FT_CASE(B, O, L) \
  if (nb == B && nob == O && nl == L) { launch_ft<M, B, O, L>(fa, mp, grid, smem, st); return true; }
  FT_CASE(5, 4, 0) FT_CASE(5, 5, 0) FT_CASE(4, 4, 0) FT_CASE(4, 3, 0) FT_CASE(3, 3, 0)
  FT_CASE(5, 4, 1) FT_CASE(4, 4, 1) FT_CASE(4, 3, 1) FT_CASE(5, 3, 2) FT_CASE(4, 3, 2) FT_CASE(3, 3, 2)
#undef FT_CASE
  return false;
}

static bool ft_have(int nb, int nob, int nl) {
  static const int k[][3] = {{5, 4, 0}, {5, 5, 0}, {4, 4, 0}, {4, 3, 0}, {3, 3, 0}, {5, 4, 1}, {4, 4, 1},
                             {4, 3, 1}, {5, 3, 2}, {4, 3, 2}, {3, 3, 2}};
  for (const auto& e : k)
    if (e[0] == nb && e[1] == nob && e[2] == nl) return true;
  return false;
}

#define FT_DECLINE(why)                                                                   \
  do {                                                                                    \
    if (env_flag("TNB_GEMM_DEBUG")) std::fprintf(stderr, "k_fc_tc declined: %s\n", why);  \
    return false;                                                                         \
  } while (0)

// smem bytes of a configuration (must match k_fc_tc's layout): operand slots, S raw per-unit
// chunk slots, X group tiles (SX slots of NLS = 2^NL units), tables
static size_t ft_smem(int M, int NB, int NL, int SX, int S, int xp_bits, uint32_t* sm_b, uint32_t* sm_raw,
                      uint32_t* sm_x, uint32_t* sm_tab, uint32_t* sm_xp) {
  const size_t K = 1u << M, KP = 2 * K, NCOL = 1u << NB, N = 2 * NCOL, NLS = 1u << NL;
  const size_t a_part = 128 * KP * 4, b_part = N * KP * 4;
  const size_t raw_slot = (128 * K * 8 + NCOL * K * 8 + (size_t)kMaxIn * K * 8 + 127) / 128 * 128;
  const size_t x_tile = NLS * 128 * NCOL * 8;
  size_t o = 0;
  o += 2 * 2 * a_part;
  *sm_b = (uint32_t)o;
  o += 2 * 2 * b_part;
  *sm_raw = (uint32_t)o;
  o += (size_t)S * raw_slot;
  o = (o + 127) / 128 * 128;
  *sm_x = (uint32_t)o;
  o += (size_t)SX * x_tile;
  *sm_tab = (uint32_t)o;
  o += (512 + 2 * NCOL) * 4;
  *sm_xp = (uint32_t)o;
  if (xp_bits >= 5) o += (size_t)8 << (xp_bits - 5);
  return o;
}

bool try_launch_fc_tc(const GDesc& g, const GDesc& g3, int tin, cudaStream_t st) {
  if (g.M < 2 || g.M > 5 || g.n < 2) FT_DECLINE("producer M or inputs");
  const int R = g.out_rank, R3 = g3.out_rank, M3 = g3.M;
  if (R > 32 || R < 16 || R3 > 32 || R3 + M3 != R) FT_DECLINE("ranks");
  // producer operands: the two inputs with the most output bits
  int ia = -1, ib = -1;
  for (int t = 0; t < g.n; ++t) {
    const int r = __builtin_popcountll(g.in[t].out_mask);
    if (ia < 0 || r > __builtin_popcountll(g.in[ia].out_mask)) { ib = ia; ia = t; }
    else if (ib < 0 || r > __builtin_popcountll(g.in[ib].out_mask)) ib = t;
  }
  if (ib < 0 || g.in[ia].rank > 32 || g.in[ib].rank > 32) FT_DECLINE("operand ranks");
  // consumer: T (identity on the o bits, its summed values on bits >= R3), X, weights
  const GIn& Tin = g3.in[tin];
  for (int i = 0; i < R3; ++i)
    if (host_fmap(1ull << i, Tin.out_mask, Tin.pv) != (1ull << i)) FT_DECLINE("T layout");
  int ybit[kMaxGroup];
  for (int j = 0; j < M3; ++j) {
    const uint64_t v = Tin.gx[1u << j];
    if (v == 0 || (v & (v - 1)) || v < (1ull << R3) || v >= (1ull << R)) FT_DECLINE("T y offsets");
    ybit[j] = __builtin_ctzll(v);
  }
  int ix = -1, nw = 0;
  FTArgs fa;
  std::memset(&fa, 0, sizeof(fa));
  for (int t = 0; t < g3.n; ++t) {
    if (t == tin) continue;
    const GIn& in = g3.in[t];
    if (in.out_mask != 0) {
      if (ix >= 0) FT_DECLINE("two consumer factors");
      ix = t;
    } else {
      if (nw >= kMaxIn) FT_DECLINE("weights");
      fa.win[nw] = static_cast<const float2*>(in.ptr);
      for (int x = 0; x < (1 << M3); ++x) fa.wgx[nw][x] = (uint32_t)in.gx[x];
      ++nw;
    }
  }
  if (ix < 0 || g3.in[ix].rank > 32) FT_DECLINE("consumer factor X");
  const GIn& Xin = g3.in[ix];
  for (int x = 0; x < (1 << M3); ++x) {   // G_X additive over the y bits
    uint64_t s = 0;
    for (int j = 0; j < M3; ++j)
      if ((x >> j) & 1) s += Xin.gx[1u << j];
    if (s != Xin.gx[x]) FT_DECLINE("X y offsets");
  }
  // per T bit: offsets in A, B, X, out, y index
  auto xoff = [&](int b) -> uint64_t {
    if (b < R3) return host_fmap(1ull << b, Xin.out_mask, Xin.pv);
    for (int j = 0; j < M3; ++j)
      if (ybit[j] == b) return Xin.gx[1u << j];
    return 0;
  };
  auto yoff = [&](int b) -> uint32_t {
    for (int j = 0; j < M3; ++j)
      if (ybit[j] == b) return 1u << j;
    return 0;
  };
  for (int swap = 0; swap < 2; ++swap) {
    const GIn& A = g.in[swap ? ib : ia];
    const GIn& B = g.in[swap ? ia : ib];
    const uint64_t full = (1ull << R) - 1;
    const uint64_t ca = A.out_mask & ~B.out_mask & full, cb = B.out_mask & ~A.out_mask & full;
    // rows: 7 a-bits that are consumer output bits; row bit 0 = the one with X (and A) offset 1
    std::vector<int> rows, cand;
    for (int b = 0; b < R3; ++b)
      if ((ca >> b) & 1) cand.push_back(b);
    if ((int)cand.size() < kFtRows) continue;
    int r0 = -1;
    for (int b : cand)
      if (xoff(b) == 1) r0 = b;
    if (r0 < 0)
      for (int b : cand)
        if (host_fmap(1ull << b, A.out_mask, A.pv) == 1) r0 = b;
    if (r0 >= 0) rows.push_back(r0);
    for (int b : cand)
      if ((int)rows.size() < kFtRows && b != r0) rows.push_back(b);
    // line bits: output bits outside the rows whose offset in X and in A lies inside one 128-byte
    // line (16 c64 elements): units differing in them share DRAM lines, so they run back to back
    std::vector<int> ob, yb;
    for (int b = 0; b < R; ++b)
      if ((cb >> b) & 1) (b < R3 ? ob : yb).push_back(b);
    if ((int)ob.size() < 3) continue;
    std::vector<std::pair<int, int>> lc;   // (score, bit)
    {
      std::vector<char> isrow(R, 0);
      for (int b : rows) isrow[b] = 1;
      for (int b = 0; b < R3; ++b) {
        if (isrow[b] || ((cb >> b) & 1)) continue;
        const uint64_t xo = xoff(b);
        const uint64_t ao = ((A.out_mask >> b) & 1) ? host_fmap(1ull << b, A.out_mask, A.pv) : 0;
        const int sc = (xo > 0 && xo < 16 ? 1 : 0) + (ao > 0 && ao < 16 ? 1 : 0);
        if (sc > 0) lc.push_back({-sc, b});
      }
      std::sort(lc.begin(), lc.end());
    }
    // columns: output b-bits (low col bits) then y b-bits; NB <= 5, NOB >= 3, NCOL >= 8; the
    // cost model: units per CTA x (X tile + a fixed per-unit overhead)
    int best_nob = -1, best_nyb = 0, best_nl = 0;
    double best_cost = 1e300;
    const int n_o_free = R3 - kFtRows;   // o bits outside the rows
    for (int nl = 0; nl <= std::min<int>(2, (int)lc.size()); ++nl)
      for (int nob = 3; nob <= std::min<int>(5, (int)ob.size()); ++nob)
        for (int nyb = 0; nyb <= (int)yb.size() && nob + nyb <= 5; ++nyb) {
          const int nb = nob + nyb;
          if (!ft_have(nb, nob, nl)) continue;
          const double nblk = std::ldexp(1.0, n_o_free - nob - nl);
          const int nyt = M3 - nyb;
          const double per_cta = std::ceil(nblk / num_sms()) * std::ldexp(1.0, nyt + nl);
          // a line bit left in the block bits re-reads its lines from DRAM: x 2 per line bit
          const double waste = std::ldexp(1.0, std::min<int>(2, (int)lc.size()) - nl);
          const double cost = per_cta * (std::ldexp(1.0, nb) * waste + 16.0);
          if (cost < best_cost) { best_cost = cost; best_nob = nob; best_nyb = nyb; best_nl = nl; }
        }
    const int NOB = best_nob, NB = best_nob + best_nyb;
    std::vector<int> cols(ob.begin(), ob.begin() + NOB);
    for (int j = 0; j < best_nyb; ++j) cols.push_back(yb[j]);
    uint64_t unit = 0;
    for (int b : rows) unit |= 1ull << b;
    for (int b : cols) unit |= 1ull << b;
    // producer constants: no unit bit
    int nc = 0;
    bool ok = true;
    for (int t = 0; t < g.n && ok; ++t) {
      if (t == ia || t == ib) continue;
      if (g.in[t].out_mask & unit) ok = false;
      if (g.in[t].rank > 32) ok = false;
      ++nc;
    }
    if (!ok || nc > kMaxIn) continue;
    // traversal: the line bits, then the y bits (a block = one set of consumer outputs), then the
    // o bits X lacks (its tile is re-read from L2 soon after), then those A lacks, then the rest
    const int NL = best_nl;
    std::vector<int> trav;
    uint64_t lmask = 0;
    for (int i = 0; i < NL; ++i) { trav.push_back(lc[i].second); lmask |= 1ull << lc[i].second; }
    for (int b = R3; b < R; ++b)
      if (!((unit >> b) & 1)) trav.push_back(b);
    const int nyt = (int)trav.size() - NL;
    std::vector<int> rest;
    for (int b = 0; b < R3; ++b)
      if (!((unit >> b) & 1) && !((lmask >> b) & 1)) rest.push_back(b);
    std::stable_sort(rest.begin(), rest.end(), [&](int p, int q2) {
      auto key = [&](int b) {
        if (xoff(b) == 0) return 0;
        if (!((A.out_mask >> b) & 1)) return 1;
        return 2;
      };
      return key(p) < key(q2);
    });
    trav.insert(trav.end(), rest.begin(), rest.end());
    if ((int)trav.size() > kFtMaxTrav) continue;
    // ---- arguments
    auto amap = [&](int b) { return (uint32_t)(((A.out_mask >> b) & 1) ? host_fmap(1ull << b, A.out_mask, A.pv) : 0); };
    auto bmap = [&](int b) { return (uint32_t)(((B.out_mask >> b) & 1) ? host_fmap(1ull << b, B.out_mask, B.pv) : 0); };
    fa.A = static_cast<const float2*>(A.ptr);
    fa.B = static_cast<const float2*>(B.ptr);
    fa.X = static_cast<const float2*>(Xin.ptr);
    fa.out = static_cast<float2*>(g3.out);
    fa.ntrav = (int)trav.size();
    fa.nyt = nyt;
    fa.n_blocks = 1ull << (trav.size() - nyt - NL);
    for (int i = 0; i < kFtRows; ++i) {
      fa.arow[i] = amap(rows[i]);
      fa.xrow[i] = (uint32_t)xoff(rows[i]);
      fa.orow[i] = 1u << rows[i];
    }
    for (int j = 0; j < NB; ++j) {
      fa.bcol[j] = bmap(cols[j]);
      fa.xcol[j] = (uint32_t)xoff(cols[j]);
      fa.ocol[j] = cols[j] < R3 ? (1u << cols[j]) : 0u;
      fa.ycol[j] = yoff(cols[j]);
    }
    int q = 0;
    for (int t = 0; t < g.n; ++t) {
      if (t == ia || t == ib) continue;
      fa.cin[q] = static_cast<const float2*>(g.in[t].ptr);
      for (int x = 0; x < (1 << g.M); ++x) fa.cgx[q][x] = (uint32_t)g.in[t].gx[x];
      for (size_t j = 0; j < trav.size(); ++j) {
        const int b = trav[j];
        fa.tc[q][j] = ((g.in[t].out_mask >> b) & 1) ? (uint32_t)host_fmap(1ull << b, g.in[t].out_mask, g.in[t].pv) : 0u;
      }
      ++q;
    }
    fa.nc = nc;
    for (size_t j = 0; j < trav.size(); ++j) {
      const int b = trav[j];
      fa.ta[j] = amap(b);
      fa.tb[j] = bmap(b);
      fa.tx[j] = (uint32_t)xoff(b);
      fa.to[j] = b < R3 ? (1u << b) : 0u;
      fa.ty[j] = yoff(b);
    }
    for (int x = 0; x < (1 << g.M); ++x) {
      fa.gA[x] = (uint32_t)A.gx[x];
      fa.gB[x] = (uint32_t)B.gx[x];
    }
    fa.nw = nw;
    fa.M3 = M3;
    fa.apair = fa.arow[0] == 1 ? 1 : 0;
    fa.xpair = fa.xrow[0] == 1 ? 1 : 0;
    // shared-memory layouts of the X tile and the raw A chunk: TMA boxes when the unit bits allow
    // (TNB_FC_TMA=0 forces the cp.async path), else [c][r] / [x][r] by 8- or 16-byte cp.async
    FtMaps mp;
    std::memset(&mp, 0, sizeof(mp));
    fa.tma = 0;
    {
      // X tile loads: coalesced 16-byte cp.async pieces in the [line][column][row] layout when row
      // bit 0 pairs X elements (default: conflict-free epilogue reads; 2,016 cycles per unit with
      // two loader warps), or (TNB_FC_XLOAD=tma) TMA boxes in the tensor's own bit order (2,257)
      const char* e = std::getenv("TNB_FC_XLOAD");
      const bool want = e && std::strcmp(e, "tma") == 0;
      fa.xp_bits = 0;
      const int RX = (int)Xin.rank, RA = (int)A.rank;
      std::vector<char> bx(RX, 0), ba(RA, 0);
      auto lg = [](uint64_t v) { return v ? __builtin_ctzll(v) : -1; };
      for (int i = 0; i < kFtRows; ++i) {
        if (fa.xrow[i]) bx[lg(fa.xrow[i])] = 1;
        ba[lg(fa.arow[i])] = 1;
      }
      for (int j = 0; j < NB; ++j)
        if (fa.xcol[j]) bx[lg(fa.xcol[j])] = 1;
      for (int i = 0; i < NL; ++i)        // a line group's tile: the line bits are box bits too
        if (fa.tx[i]) bx[lg(fa.tx[i])] = 1;
      bool xok = true;
      for (int j = 0; j < g.M; ++j) {
        const uint64_t v = A.gx[1u << j];
        if (v == 0 || (v & (v - 1))) xok = false;
        else ba[lg(v)] = 1;
      }
      TmaGeom GX, GA;
      // raw A chunks: TMA boxes over the unit's rows and summed values (default; TNB_FC_ATMA=0 ->
      // cp.async), in the box layout the formatters index with as_row / as_x
      fa.atma = 0;
      {
        const char* ea = std::getenv("TNB_FC_ATMA");
        std::vector<char> ba2(RA, 0);
        for (int i = 0; i < kFtRows; ++i) ba2[lg(fa.arow[i])] = 1;
        bool aok = !(ea && ea[0] == '0') && xok;
        for (int j = 0; j < g.M && aok; ++j) ba2[lg(A.gx[1u << j])] = 1;
        if (aok && tma_geom(RA, ba2, GA) && GA.ncopy * GA.box_elems <= (128u << g.M) &&
            tma_encode(&mp.a, A.ptr, RA, GA)) {
          fa.atma = 1;
          for (int d = 0; d < 5; ++d) {
            fa.ts[1][d] = d < GA.ndim ? GA.s[d] : 0;
            fa.tmsk[1][d] = d < GA.ndim ? (uint32_t)((1ull << GA.nt[d]) - 1) : 0u;
            for (int i = 0; i < 8; ++i) fa.cdelta[1][i][d] = GA.cdelta[i][d];
          }
          fa.ncopy[1] = GA.ncopy;
          fa.copy_elems[1] = GA.box_elems;
          for (int i = 0; i < kFtRows; ++i) fa.as_row[i] = 1u << GA.smem_bit[lg(fa.arow[i])];
          for (int x = 0; x < (1 << g.M); ++x) {
            uint32_t o = 0;
            for (int j = 0; j < g.M; ++j)
              if ((x >> j) & 1) o += 1u << GA.smem_bit[lg(A.gx[1u << j])];
            fa.as_x[x] = o;
          }
        } else {
          for (int i = 0; i < kFtRows; ++i) fa.as_row[i] = 1u << i;
          for (int x = 0; x < (1 << g.M); ++x) fa.as_x[x] = 128u * (uint32_t)x;
        }
      }
      if (want && tma_geom(RX, bx, GX) && GX.ncopy * GX.box_elems <= (128u << NB) << NL &&
          tma_encode(&mp.x, Xin.ptr, RX, GX)) {
        fa.tma = 1;
        const TmaGeom* G[1] = {&GX};
        for (int t = 0; t < 1; ++t) {
          for (int d = 0; d < 5; ++d) {
            fa.ts[t][d] = d < G[t]->ndim ? G[t]->s[d] : 0;
            fa.tmsk[t][d] = d < G[t]->ndim ? (uint32_t)((1ull << G[t]->nt[d]) - 1) : 0u;
            for (int i = 0; i < 8; ++i) fa.cdelta[t][i][d] = G[t]->cdelta[i][d];
          }
          fa.ncopy[t] = G[t]->ncopy;
          fa.copy_elems[t] = G[t]->box_elems;
        }
        for (int i = 0; i < kFtRows; ++i) fa.xs_row[i] = fa.xrow[i] ? 1u << GX.smem_bit[lg(fa.xrow[i])] : 0u;
        for (int j = 0; j < NB; ++j) fa.xs_col[j] = fa.xcol[j] ? 1u << GX.smem_bit[lg(fa.xcol[j])] : 0u;
        for (int li = 0; li < (1 << NL); ++li) {
          uint32_t ox = 0;
          for (int i = 0; i < NL; ++i)
            if (((li >> i) & 1) && fa.tx[i]) ox += 1u << GX.smem_bit[lg(fa.tx[i])];
          fa.xs_line[li] = ox;
        }
      } else {
        if (fa.xpair) {
          std::vector<std::pair<uint32_t, uint32_t>> pb;   // (global, smem) per piece bit
          for (int i = 1; i < kFtRows; ++i) pb.push_back({fa.xrow[i], 1u << i});
          for (int j = 0; j < NB; ++j) pb.push_back({fa.xcol[j], 128u << j});
          for (int i = 0; i < NL; ++i) pb.push_back({fa.tx[i], (128u << NB) << i});
          std::stable_sort(pb.begin(), pb.end(), [](const auto& p1, const auto& p2) { return p1.first < p2.first; });
          if (pb.size() <= 24 && pb.size() >= 5) {
            fa.xp_bits = (int)pb.size();
            for (size_t k = 0; k < pb.size(); ++k) { fa.xp_g[k] = pb[k].first; fa.xp_s[k] = pb[k].second; }
          }
        }
        for (int i = 0; i < kFtRows; ++i) fa.xs_row[i] = 1u << i;
        for (int j = 0; j < NB; ++j) fa.xs_col[j] = 128u << j;
        for (int li = 0; li < (1 << NL); ++li) fa.xs_line[li] = (uint32_t)li * (128u << NB);
      }
    }
    const int N = 2 << NB;
    fa.tmem_cols = 32;
    while (fa.tmem_cols < (uint32_t)(2 * N)) fa.tmem_cols <<= 1;
    size_t smem = 0;
    int SX = 0, SU = 0;
    for (const auto& c : {std::make_pair(2, 4), std::make_pair(2, 3), std::make_pair(2, 2), std::make_pair(1, 3),
                          std::make_pair(1, 2)}) {
      smem = ft_smem(g.M, NB, NL, c.first, c.second, fa.xp_bits, &fa.sm_b, &fa.sm_raw, &fa.sm_x, &fa.sm_tab,
                     &fa.sm_xp);
      if (smem <= 218 * 1024) { SX = c.first; SU = c.second; break; }
    }
    if (SX == 0) continue;
    fa.S = SU;
    fa.SX = SX;
    const int S = SX * 10 + SU;   // (trace print)
    const unsigned grid = (unsigned)std::min<uint64_t>(fa.n_blocks, (uint64_t)num_sms());
    static unsigned long long* trace = nullptr;
    const bool want_trace = env_flag("TNB_FT_TRACE");
    if (want_trace && !trace && cudaMalloc(&trace, 256 * 8 * sizeof(unsigned long long)) != cudaSuccess) trace = nullptr;
    fa.trace = want_trace ? trace : nullptr;
    if (fa.trace) cudaMemsetAsync(fa.trace, 0, 256 * 8 * sizeof(unsigned long long), st);
    if (env_flag("TNB_GEMM_DEBUG")) {
      std::fprintf(stderr, "k_fc_tc R=%d M=%d R3=%d M3=%d swap=%d NB=%d NOB=%d NL=%d nyt=%d blocks=%llu S=%d smem=%zu "
                   "apair=%d xpair=%d tma=%d atma=%d xp_bits=%d (copies %d,%d) rows=", R, g.M, R3, M3, swap, NB, NOB, NL,
                   nyt, (unsigned long long)fa.n_blocks, S, smem, fa.apair, fa.xpair, fa.tma, fa.atma, fa.xp_bits,
                   fa.ncopy[0], fa.ncopy[1]);
      for (int b : rows) std::fprintf(stderr, "%d,", b);
      std::fprintf(stderr, " cols=");
      for (int b : cols) std::fprintf(stderr, "%d,", b);
      std::fprintf(stderr, " trav=");
      for (int b : trav) std::fprintf(stderr, "%d,", b);
      std::fprintf(stderr, "\n");
    }
    bool ok2 = false;
    switch (g.M) {
      case 2: ok2 = dispatch_ft<2>(fa, mp, NB, NOB, NL, grid, smem, st); break;
      case 3: ok2 = dispatch_ft<3>(fa, mp, NB, NOB, NL, grid, smem, st); break;
      case 4: ok2 = dispatch_ft<4>(fa, mp, NB, NOB, NL, grid, smem, st); break;
      case 5: ok2 = dispatch_ft<5>(fa, mp, NB, NOB, NL, grid, smem, st); break;
      default: return false;
    }
    if (ok2 && fa.trace) {   // debugging aid: CTA 0's pipeline timeline (clock64), averaged gaps
      unsigned long long h[256 * 8];
      cudaStreamSynchronize(st);
      cudaMemcpy(h, fa.trace, sizeof(h), cudaMemcpyDeviceToHost);
      const int n = (int)std::min<uint64_t>(256, (fa.n_blocks / grid) << (NL + nyt));
      const char* nm[8] = {"prod_start", "fmt_done", "mma_issue", "epi_start", "epi_end", "prod_done", "fmt_start", "epi_wait0"};
      std::fprintf(stderr, "k_fc_tc trace (CTA 0, %d units): per-unit mean of (event - ld_ready):", n);
      for (int e = 1; e < 8; ++e) {
        double sum = 0;
        int c = 0;
        for (int u = 8; u < n; ++u)
          if (h[u * 8 + e] && h[u * 8]) { sum += (double)(long long)(h[u * 8 + e] - h[u * 8]); ++c; }
        std::fprintf(stderr, " %s %.0f", nm[e], c ? sum / c : 0.0);
      }
      double per = n > 16 ? (double)(h[(n - 1) * 8 + 4] - h[8 * 8 + 4]) / (n - 9) : 0;
      std::fprintf(stderr, " | cycles per unit %.0f\n", per);
    }
    return ok2;
  }
  FT_DECLINE("no row / column assignment");
}

}  // namespace tnb
