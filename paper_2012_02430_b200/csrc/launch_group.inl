// launch_group.inl -- k_group_t host side (included by launch_group_c64.cu / _c128.cu)
#pragma once
#include "launch.cuh"

namespace tnb {

template <typename T, typename OffT, int NDIR, int NSTG, int M, int NDV>
void launch_g(const GArgs& ga, unsigned grid, size_t smem, cudaStream_t st) {
  allow_smem(k_group_t<T, OffT, NDIR, NSTG, M, NDV>, smem);
  last_kernel() = KID_GROUP;
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

}  // namespace tnb
