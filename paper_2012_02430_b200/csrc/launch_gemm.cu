// launch_gemm.cu: k_gemm (register-blocked batched complex GEMM groups, FFMA2) -- part of libtnb200.so (see launch.cuh)
#include "launch.cuh"

#include <cstdio>

namespace tnb {

// dynamic shared memory per CTA so that two CTAs (plus ~5 KB static each) fit the 228 KB of an SM
constexpr size_t kGemmSmemBudget = 100 * 1024;

template <int M, int RAB, int RBB, int WB>
void launch_m(const MArgs& ma, unsigned grid, size_t smem, cudaStream_t st) {
  allow_smem(k_gemm<M, RAB, RBB, true, WB>, smem);
  last_kernel() = KID_GEMM;
  k_gemm<M, RAB, RBB, true, WB><<<grid, 32 << WB, smem, st>>>(ma);
}

template <int M, int WB>
bool dispatch_m(const MArgs& ma, int rab, int rbb, unsigned grid, size_t smem, cudaStream_t st) {
  if (rab == 2 && rbb == 2) { launch_m<M, 2, 2, WB>(ma, grid, smem, st); return true; }
  if (rab == 2 && rbb == 1) { launch_m<M, 2, 1, WB>(ma, grid, smem, st); return true; }
  if (rab == 1 && rbb == 2) { launch_m<M, 1, 2, WB>(ma, grid, smem, st); return true; }
  if (rab == 1 && rbb == 1) { launch_m<M, 1, 1, WB>(ma, grid, smem, st); return true; }
  return false;
}


// preferred CTA size: 2^WB warps (TNB_GEMM_WB = 2 or 3); 4-warp CTAs run 4 per SM (half the shared
// memory each), 8-warp CTAs 2 per SM.  Default 2 since the 8-lane / fused-pair state (C5a 88.7 vs
// 86.7 contractions/s); a shape whose chunks do not fit the 4-warp budget takes 8-warp CTAs
inline int gemm_wb() {
  static const int wb = [] {
    const char* v = std::getenv("TNB_GEMM_WB");
    const int x = v ? std::atoi(v) : 2;
    return x == 3 ? 3 : 2;
  }();
  return wb;
}

// A group whose varying inputs are two tensors holding a-only and b-only output bits runs as a
// register-blocked batched complex GEMM (k_gemm, c64).  Returns false when the shape does not
// qualify (the caller then tries k_pair / k_group_t).
template <typename T>
bool try_launch_gemm_impl(const GDesc& g, cudaStream_t st, int WB);

inline int gemm_min_m() {   // TNB_GEMM_MIN_M: groups summing fewer indices go to k_pair / k_group_t
  static const int v = [] {
    const char* e = std::getenv("TNB_GEMM_MIN_M");
    return e ? std::atoi(e) : 1;
  }();
  return v;
}

inline int hm64_min_r() {
  const char* e = std::getenv("TNB_HM64_MIN_R");
  return e ? std::atoi(e) : 20;
}

template <typename T>
bool try_launch_gemm(const GDesc& g, cudaStream_t st) {
  if (g.M < gemm_min_m()) return false;
  if (std::is_same<T, float2>::value && gemm_tc_enabled() && try_launch_gemm_tc(g, st)) return true;
  // k_gemm_hm where it measured faster on C5a's groups (M >= 3 and >= 2^22 outputs: 78 vs 95 us on
  // the top group; smaller or M = 2 groups are bound by its per-tile pipeline, profiles/r02/hm/)
  if (std::is_same<T, float2>::value && gemm_hm_enabled() && g.M >= 3 && g.out_rank >= 22 && try_launch_gemm_hm(g, st))
    return true;
  // c128: k_gemm_hm64 (DMMA) for groups of >= 2^TNB_HM64_MIN_R outputs (default 20; TNB_GEMM_HM64=0 off)
  if (std::is_same<T, double2>::value && gemm_hm_enabled() && !env_flag0("TNB_GEMM_HM64") && g.out_rank >= hm64_min_r() &&
      try_launch_gemm_hm64(g, st))
    return true;
  // the preferred CTA size (gemm_wb()) first, the other one when its shared-memory budget is too small
  const int wb0 = gemm_wb(), wb1 = 5 - wb0;
  return try_launch_gemm_impl<T>(g, st, wb0) || try_launch_gemm_impl<T>(g, st, wb1);
}

template <typename T>
bool try_launch_gemm_simt(const GDesc& g, cudaStream_t st) {
  const int wb0 = gemm_wb(), wb1 = 5 - wb0;
  return try_launch_gemm_impl<T>(g, st, wb0) || try_launch_gemm_impl<T>(g, st, wb1);
}

template <typename T>
bool try_launch_gemm_impl(const GDesc& g, cudaStream_t st, int WB) {
  if constexpr (!std::is_same<T, float2>::value) {
    (void)g; (void)st; (void)WB;
    return false;
  } else {
    if (gemm_disabled() || g.M < 1 || g.M > kMaxGroup || g.n < 2) return false;
    const int R = g.out_rank;
    if (R < 11 || R > 40) return false;
    // A, B: the two inputs with the most output bits
    int ia = -1, ib = -1;
    for (int t = 0; t < g.n; ++t) {
      const int r = __builtin_popcountll(g.in[t].out_mask);
      if (ia < 0 || r > __builtin_popcountll(g.in[ia].out_mask)) { ib = ia; ia = t; }
      else if (ib < 0 || r > __builtin_popcountll(g.in[ib].out_mask)) ib = t;
    }
    if (g.in[ia].rank > 32 || g.in[ib].rank > 32) return false;
    const uint64_t full = (1ull << R) - 1;
    uint64_t ca = g.in[ia].out_mask & ~g.in[ib].out_mask, cb = g.in[ib].out_mask & ~g.in[ia].out_mask;
    const uint64_t cc = g.in[ia].out_mask & g.in[ib].out_mask, cn = full & ~(g.in[ia].out_mask | g.in[ib].out_mask);
    if (cn & 31ull) return false;                       // lanes must be held by A or B
    int ra[3], rb[3], nra = 0, nrb = 0;
    for (int b = 5; b < R; ++b) {
      if (((ca >> b) & 1) && nra < 2) ra[nra++] = b;
      if (((cb >> b) & 1) && nrb < 2) rb[nrb++] = b;
    }
    if (nra == 0 || nrb == 0) return false;             // not GEMM-shaped: no reuse to exploit
    uint64_t used = 31ull;
    for (int i = 0; i < nra; ++i) used |= 1ull << ra[i];
    for (int i = 0; i < nrb; ++i) used |= 1ull << rb[i];
    int wb[3], nw = 0;
    // warp bits: the lowest free a/b bits (reuse), then c bits (round 1's TNB_GEMM_CONTIG -- the
    // lowest free bits of any class for a more contiguous tile -- measured slower and was removed)
    for (int pass = 0; pass < 2 && nw < WB; ++pass)
      for (int b = 5; b < R && nw < WB; ++b) {
        const uint64_t cls = pass == 0 ? (ca | cb) : cc;
        if (!((used >> b) & 1) && ((cls >> b) & 1)) { wb[nw++] = b; used |= 1ull << b; }
      }
    if (nw < WB) return false;
    // role of B (the operand formatted in shared memory, kept across consecutive tiles): the one
    // whose chunk changes least often.  The tile is symmetric in the roles; the traversal flips
    // A's exclusive non-tile bits first, so B stays for 2^(that count) tiles; ties -> B with fewer
    // tile bits (smaller formatted chunk)
    {
      const int exa = __builtin_popcountll(ca & ~used), exb = __builtin_popcountll(cb & ~used);
      const int ta = __builtin_popcountll(used & g.in[ia].out_mask), tb = __builtin_popcountll(used & g.in[ib].out_mask);
      if (exb > exa || (exb == exa && ta < tb)) {
        std::swap(ia, ib);
        std::swap(ca, cb);
        std::swap(ra, rb);
        std::swap(nra, nrb);
      }
    }
    const GIn& A = g.in[ia];
    const GIn& Bq = g.in[ib];
    const int TB = 5 + WB + nra + nrb;
    if (R < TB || TB > kGemmMaxTB) return false;
    MArgs ma;
    std::memset(&ma, 0, sizeof(ma));
    int u = 0;
    for (int b = 0; b < 5; ++b) ma.outbit[u++] = (uint8_t)b;
    for (int i = 0; i < WB; ++i) ma.outbit[u++] = (uint8_t)wb[i];
    for (int i = 0; i < nra; ++i) ma.outbit[u++] = (uint8_t)ra[i];
    for (int i = 0; i < nrb; ++i) ma.outbit[u++] = (uint8_t)rb[i];
    const uint64_t tmask = used;
    // constant inputs: no tile bit
    int nc = 0;
    for (int t = 0; t < g.n; ++t) {
      if (t == ia || t == ib) continue;
      if (g.in[t].out_mask & tmask) return false;
      if (g.in[t].rank > 32) return false;
      ma.cin[nc] = g.in[t].ptr;
      ma.cmask[nc] = g.in[t].out_mask;
      ma.cpv[nc] = g.in[t].pv;
      for (int x = 0; x < (1 << g.M); ++x) ma.cgx[nc][x] = (uint32_t)g.in[t].gx[x];
      ++nc;
    }
    ma.nc = nc;
    ma.c_tile_dep = 0;
    for (int t = 0; t < nc; ++t) ma.c_tile_dep |= ma.cmask[t] != 0 ? 1 : 0;
    // chunks: tile bits held by each input, by ascending output bit (= ascending input position)
    uint32_t smem_elems = 0;
    uint32_t sz[2];
    for (int s = 0; s < 2; ++s) {
      const GIn& in = s == 0 ? A : Bq;
      int k = 0;
      for (int b = 0; b < R; ++b) {
        if (!((tmask >> b) & 1) || !((in.out_mask >> b) & 1)) continue;
        for (int uu = 0; uu < TB; ++uu)
          if (ma.outbit[uu] == b) ma.chbit[s][uu] = (int8_t)k;
        ma.posoff[s][k] = (uint32_t)host_fmap(1ull << b, in.out_mask, in.pv);
        ++k;
      }
      for (int uu = 0; uu < TB; ++uu) {
        const int b = ma.outbit[uu];
        if (!((in.out_mask >> b) & 1)) ma.chbit[s][uu] = -1;
      }
      ma.nch[s] = (uint32_t)k;
      ma.lv[s] = (k >= 1 && ma.posoff[s][0] == 1) ? 1u : 0u;
      std::vector<uint64_t> parts;
      for (int x = 0; x < (1 << g.M); ++x) {
        auto it = std::find(parts.begin(), parts.end(), in.gx[x]);
        if (it == parts.end()) {
          ma.row[s][x] = (uint8_t)parts.size();
          parts.push_back(in.gx[x]);
        } else {
          ma.row[s][x] = (uint8_t)(it - parts.begin());
        }
      }
      for (size_t r = 0; r < parts.size(); ++r) ma.rowoff[s][r] = (uint32_t)parts[r];
      ma.nrows[s] = (uint32_t)parts.size();
      ma.in[s] = in.ptr;
      ma.mask[s] = in.out_mask;
      ma.pv[s] = in.pv;
      sz[s] = ma.nrows[s] << k;
    }
    // ring slots: as many as fit the per-CTA budget (2 CTAs per SM), at most gemm_stages()
    const uint32_t dep_u32 = (ma.nrows[0] << (ma.nch[0] - ma.lv[0])) + (ma.nrows[1] << (ma.nch[1] - ma.lv[1]));
    const size_t bf_bytes = ((size_t)16 << g.M) << ma.nch[1];
    int S = gemm_stages();
    const size_t budget = WB == 3 ? kGemmSmemBudget : kGemmSmemBudget / 2;   // 2 or 4 CTAs per SM
    while (S > 2 && ((size_t)S * (sz[0] + sz[1]) * 8 + dep_u32 * 4 + bf_bytes + 16) > budget) --S;
    ma.stages = S;
    for (int k = 0; k < S; ++k) {
      ma.sm_in[0][k] = k * sz[0];
      ma.sm_in[1][k] = S * sz[0] + k * sz[1];
    }
    smem_elems = S * (sz[0] + sz[1]);
    uint32_t u32 = 2 * smem_elems;                       // uint32 units
    for (int s = 0; s < 2; ++s) {
      ma.sm_dep[s] = u32;
      u32 += ma.nrows[s] << (ma.nch[s] - ma.lv[s]);
    }
    ma.sm_bf_bytes = (u32 * 4 + 15) / 16 * 16;
    const size_t smem = ma.sm_bf_bytes + bf_bytes;
    if (smem > budget) return false;
    // traversal of the tile index: a-only bits first (B chunk and B' unchanged), then b-only, then
    // the rest
    // (b-only bits first -- round 1's TNB_GEMM_BFIRST -- measured slower: B and B' change every tile)
    int np = 0;
    for (int pass = 0; pass < 3; ++pass)
      for (int b = 0; b < R; ++b) {
        if ((tmask >> b) & 1) continue;
        const uint64_t cls = pass == 0 ? ca : pass == 1 ? cb : (cc | cn);
        if ((cls >> b) & 1) ma.perm[np++] = (uint8_t)b;
      }
    if (np != R - TB) return false;
    ma.out = g.out;
    ma.out_rank = R;
    if (env_flag("TNB_GEMM_DEBUG")) {
      std::fprintf(stderr, "k_gemm R=%d M=%d TB=%d nra=%d nrb=%d nch=(%u,%u) lv=(%u,%u) rows=(%u,%u) S=%d smem=%zu nc=%d ctd=%d outbits=",
                   R, g.M, TB, nra, nrb, ma.nch[0], ma.nch[1], ma.lv[0], ma.lv[1], ma.nrows[0], ma.nrows[1],
                   ma.stages, smem, nc, ma.c_tile_dep);
      for (int uu = 0; uu < TB; ++uu) std::fprintf(stderr, "%d%s", ma.outbit[uu], uu + 1 < TB ? "," : "");
      std::fprintf(stderr, " perm=");
      for (int b = 0; b < np && b < 8; ++b) std::fprintf(stderr, "%d,", ma.perm[b]);
      std::fprintf(stderr, "\n");
      debug_group("k_gemm", g);
    }
    const uint64_t tiles = 1ull << (R - TB);
    const unsigned grid = (unsigned)std::min<uint64_t>(tiles, (uint64_t)num_sms() * (WB == 3 ? 2 : 4));
    if (WB == 2) {
      switch (g.M) {
        case 1: return dispatch_m<1, 2>(ma, nra, nrb, grid, smem, st);
        case 2: return dispatch_m<2, 2>(ma, nra, nrb, grid, smem, st);
        case 3: return dispatch_m<3, 2>(ma, nra, nrb, grid, smem, st);
        case 4: return dispatch_m<4, 2>(ma, nra, nrb, grid, smem, st);
        case 5: return dispatch_m<5, 2>(ma, nra, nrb, grid, smem, st);
        default: return false;
      }
    }
    switch (g.M) {
      case 1: return dispatch_m<1, 3>(ma, nra, nrb, grid, smem, st);
      case 2: return dispatch_m<2, 3>(ma, nra, nrb, grid, smem, st);
      case 3: return dispatch_m<3, 3>(ma, nra, nrb, grid, smem, st);
      case 4: return dispatch_m<4, 3>(ma, nra, nrb, grid, smem, st);
      case 5: return dispatch_m<5, 3>(ma, nra, nrb, grid, smem, st);
      default: return false;
    }
  }
}

template bool try_launch_gemm<float2>(const GDesc&, cudaStream_t);
template bool try_launch_gemm<double2>(const GDesc&, cudaStream_t);
template bool try_launch_gemm_simt<float2>(const GDesc&, cudaStream_t);
template bool try_launch_gemm_simt<double2>(const GDesc&, cudaStream_t);

}  // namespace tnb
