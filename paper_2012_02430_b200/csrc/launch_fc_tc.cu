// launch_fc_tc.cu: k_fc_tc (producer -> consumer merge groups, OP_GROUP_FEED, with the producer's
// GEMM on tcgen05) -- part of libtnb200.so (see launch.cuh, kernels_fctc.cuh).  Host side: classify
// T's bits, pick the unit (7 row bits, NB column bits), order the traversal, size the rings.
#include "launch.cuh"
#include "kernels_fctc.cuh"

#include <cmath>
#include <cstdio>

namespace tnb {

// TNB_FC_TC=1 / 0 selects k_fc_tc / the FP32 SIMT k_gemm_fc for OP_GROUP_FEED pairs (read per call:
// the parity tests run both kernels in one process); default: kFcTcDefault
constexpr bool kFcTcDefault = false;
bool fc_tc_enabled() {
  const char* v = std::getenv("TNB_FC_TC");
  return v ? v[0] == '1' : kFcTcDefault;
}

template <int M, int NB, int NOB>
static void launch_ft(const FTArgs& fa, unsigned grid, size_t smem, cudaStream_t st) {
  allow_smem(k_fc_tc<M, NB, NOB>, smem);
  last_kernel() = KID_FC_TC;
  k_fc_tc<M, NB, NOB><<<grid, kFtThreads, smem, st>>>(fa);
}

template <int M>
static bool dispatch_ft(const FTArgs& fa, int nb, int nob, unsigned grid, size_t smem, cudaStream_t st) {
#define FT_CASE(B, O) \
  if (nb == B && nob == O) { launch_ft<M, B, O>(fa, grid, smem, st); return true; }
  FT_CASE(5, 4) FT_CASE(5, 5) FT_CASE(5, 3) FT_CASE(4, 4) FT_CASE(4, 3) FT_CASE(3, 3)
#undef FT_CASE
  return false;
}

#define FT_DECLINE(why)                                                                   \
  do {                                                                                    \
    if (env_flag("TNB_GEMM_DEBUG")) std::fprintf(stderr, "k_fc_tc declined: %s\n", why);  \
    return false;                                                                         \
  } while (0)

// smem bytes of a configuration (must match k_fc_tc's layout)
static size_t ft_smem(int M, int NB, int nc, int S, uint32_t* sm_b, uint32_t* sm_raw, uint32_t* sm_x,
                      uint32_t* sm_tab) {
  const size_t K = 1u << M, KP = 2 * K, NCOL = 1u << NB, N = 2 * NCOL;
  const size_t a_part = 128 * KP * 4, b_part = N * KP * 4;
  const size_t raw_slot = 128 * K * 8 + NCOL * K * 8 + (size_t)nc * K * 8;
  const size_t x_tile = 128 * NCOL * 8;
  size_t o = 0;
  o += 2 * 2 * a_part;
  *sm_b = (uint32_t)o;
  o += 2 * 2 * b_part;
  *sm_raw = (uint32_t)o;
  o += (size_t)S * raw_slot;
  o = (o + 127) / 128 * 128;
  *sm_x = (uint32_t)o;
  o += (size_t)S * x_tile;
  *sm_tab = (uint32_t)o;
  o += (256 + 2 * NCOL) * 4;
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
    // columns: output b-bits (low col bits) then y b-bits; NB <= 5, NOB >= 3, NCOL >= 8
    std::vector<int> ob, yb;
    for (int b = 0; b < R; ++b)
      if ((cb >> b) & 1) (b < R3 ? ob : yb).push_back(b);
    if ((int)ob.size() < 3) continue;
    int best_nob = -1, best_nyb = 0;
    double best_cost = 1e300;
    const int n_o_free = R3 - kFtRows;   // o bits outside the rows
    for (int nob = 3; nob <= std::min<int>(5, (int)ob.size()); ++nob)
      for (int nyb = 0; nyb <= (int)yb.size() && nob + nyb <= 5; ++nyb) {
        const int nb = nob + nyb;
        const double nblk = std::ldexp(1.0, n_o_free - nob);
        const int nyt = M3 - nyb;
        const double per_cta = std::ceil(nblk / num_sms()) * std::ldexp(1.0, nyt);
        const double cost = per_cta * (std::ldexp(1.0, nb) + 16.0);
        if (cost < best_cost) { best_cost = cost; best_nob = nob; best_nyb = nyb; }
      }
    if (best_nob < 0) continue;
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
    // traversal: y bits first (innermost: a block = one set of consumer outputs), then the o bits
    // X lacks (its tile is re-read from L2 right away), then those A lacks, then the rest
    std::vector<int> trav;
    for (int b = R3; b < R; ++b)
      if (!((unit >> b) & 1)) trav.push_back(b);
    const int nyt = (int)trav.size();
    std::vector<int> rest;
    for (int b = 0; b < R3; ++b)
      if (!((unit >> b) & 1)) rest.push_back(b);
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
    fa.n_blocks = 1ull << (trav.size() - nyt);
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
    const int N = 2 << NB;
    fa.tmem_cols = 32;
    while (fa.tmem_cols < (uint32_t)(2 * N)) fa.tmem_cols <<= 1;
    size_t smem = 0;
    int S = 3;
    for (; S >= 2; --S) {
      smem = ft_smem(g.M, NB, nc, S, &fa.sm_b, &fa.sm_raw, &fa.sm_x, &fa.sm_tab);
      if (smem <= 220 * 1024) break;
    }
    if (S < 2) continue;
    fa.S = S;
    const unsigned grid = (unsigned)std::min<uint64_t>(fa.n_blocks, (uint64_t)num_sms());
    if (env_flag("TNB_GEMM_DEBUG")) {
      std::fprintf(stderr, "k_fc_tc R=%d M=%d R3=%d M3=%d swap=%d NB=%d NOB=%d nyt=%d blocks=%llu S=%d smem=%zu "
                   "apair=%d xpair=%d rows=", R, g.M, R3, M3, swap, NB, NOB, nyt, (unsigned long long)fa.n_blocks,
                   S, smem, fa.apair, fa.xpair);
      for (int b : rows) std::fprintf(stderr, "%d,", b);
      std::fprintf(stderr, " cols=");
      for (int b : cols) std::fprintf(stderr, "%d,", b);
      std::fprintf(stderr, "\n");
    }
    switch (g.M) {
      case 2: return dispatch_ft<2>(fa, NB, NOB, grid, smem, st);
      case 3: return dispatch_ft<3>(fa, NB, NOB, grid, smem, st);
      case 4: return dispatch_ft<4>(fa, NB, NOB, grid, smem, st);
      case 5: return dispatch_ft<5>(fa, NB, NOB, grid, smem, st);
      default: return false;
    }
  }
  FT_DECLINE("no row / column assignment");
}

}  // namespace tnb
