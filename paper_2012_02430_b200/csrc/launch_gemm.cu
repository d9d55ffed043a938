// launch_gemm.cu: k_gemm (register-blocked batched complex GEMM groups, FFMA2) -- part of libtnb200.so (see launch.cuh)
#include "launch.cuh"

namespace tnb {

template <int M, int RAB, int RBB>
void launch_m(const MArgs& ma, unsigned grid, size_t smem, cudaStream_t st) {
  allow_smem(k_gemm<M, RAB, RBB, true>, smem);
  k_gemm<M, RAB, RBB, true><<<grid, kGemmThreads, smem, st>>>(ma);
}

template <int M>
bool dispatch_m(const MArgs& ma, int rab, int rbb, unsigned grid, size_t smem, cudaStream_t st) {
  if (rab == 2 && rbb == 2) { launch_m<M, 2, 2>(ma, grid, smem, st); return true; }
  if (rab == 2 && rbb == 1) { launch_m<M, 2, 1>(ma, grid, smem, st); return true; }
  if (rab == 1 && rbb == 2) { launch_m<M, 1, 2>(ma, grid, smem, st); return true; }
  if (rab == 1 && rbb == 1) { launch_m<M, 1, 1>(ma, grid, smem, st); return true; }
  return false;
}

// A group whose varying inputs are two tensors holding a-only and b-only output bits runs as a
// register-blocked batched complex GEMM (k_gemm, c64).  Returns false when the shape does not
// qualify (the caller then tries k_pair / k_group_t).
template <typename T>
bool try_launch_gemm(const GDesc& g, cudaStream_t st) {
  if constexpr (!std::is_same<T, float2>::value) {
    (void)g; (void)st;
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
    const GIn& A = g.in[ia];
    const GIn& Bq = g.in[ib];
    if (A.rank > 32 || Bq.rank > 32) return false;
    const uint64_t full = (1ull << R) - 1;
    const uint64_t ca = A.out_mask & ~Bq.out_mask, cb = Bq.out_mask & ~A.out_mask;
    const uint64_t cc = A.out_mask & Bq.out_mask, cn = full & ~(A.out_mask | Bq.out_mask);
    if (cn & 31ull) return false;                       // lanes must be held by A or B
    int ra[2], rb[2], nra = 0, nrb = 0;
    for (int b = 5; b < R; ++b) {
      if (((ca >> b) & 1) && nra < 2) ra[nra++] = b;
      if (((cb >> b) & 1) && nrb < 2) rb[nrb++] = b;
    }
    if (nra == 0 || nrb == 0) return false;             // not GEMM-shaped: no reuse to exploit
    uint64_t used = 31ull;
    for (int i = 0; i < nra; ++i) used |= 1ull << ra[i];
    for (int i = 0; i < nrb; ++i) used |= 1ull << rb[i];
    int wb[3], nw = 0;
    for (int pass = 0; pass < 2 && nw < 3; ++pass)
      for (int b = 5; b < R && nw < 3; ++b) {
        const uint64_t cls = pass == 0 ? (ca | cb) : cc;
        if (!((used >> b) & 1) && ((cls >> b) & 1)) { wb[nw++] = b; used |= 1ull << b; }
      }
    if (nw < 3) return false;
    const int TB = 8 + nra + nrb;
    if (R < TB) return false;
    MArgs ma;
    std::memset(&ma, 0, sizeof(ma));
    int u = 0;
    for (int b = 0; b < 5; ++b) ma.outbit[u++] = (uint8_t)b;
    for (int i = 0; i < 3; ++i) ma.outbit[u++] = (uint8_t)wb[i];
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
    ma.sm_in[0][0] = 0;
    ma.sm_in[0][1] = sz[0];
    ma.sm_in[1][0] = 2 * sz[0];
    ma.sm_in[1][1] = 2 * sz[0] + sz[1];
    smem_elems = 2 * (sz[0] + sz[1]);
    uint32_t u32 = 2 * smem_elems;                       // uint32 units
    for (int s = 0; s < 2; ++s) {
      ma.sm_dep[s] = u32;
      u32 += 1u << (ma.nch[s] - ma.lv[s]);
    }
    const size_t smem = (size_t)u32 * 4;
    if (smem > 110 * 1024) return false;
    // traversal of the tile index: b-only bits first (A chunk unchanged), then a-only, then the rest
    int np = 0;
    for (int pass = 0; pass < 3; ++pass)
      for (int b = 0; b < R; ++b) {
        if ((tmask >> b) & 1) continue;
        const uint64_t cls = pass == 0 ? cb : pass == 1 ? ca : (cc | cn);
        if ((cls >> b) & 1) ma.perm[np++] = (uint8_t)b;
      }
    if (np != R - TB) return false;
    ma.out = g.out;
    ma.out_rank = R;
    const uint64_t tiles = 1ull << (R - TB);
    const unsigned grid = (unsigned)std::min<uint64_t>(tiles, (uint64_t)num_sms() * 2);
    switch (g.M) {
      case 1: return dispatch_m<1>(ma, nra, nrb, grid, smem, st);
      case 2: return dispatch_m<2>(ma, nra, nrb, grid, smem, st);
      case 3: return dispatch_m<3>(ma, nra, nrb, grid, smem, st);
      case 4: return dispatch_m<4>(ma, nra, nrb, grid, smem, st);
      case 5: return dispatch_m<5>(ma, nra, nrb, grid, smem, st);
      default: return false;
    }
  }
}

template bool try_launch_gemm<float2>(const GDesc&, cudaStream_t);
template bool try_launch_gemm<double2>(const GDesc&, cudaStream_t);

}  // namespace tnb
