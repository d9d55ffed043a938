// launch_pair.cu: k_pair (2x2 register-blocked pair groups) -- part of libtnb200.so (see launch.cuh)
#include "launch.cuh"

namespace tnb {

// register-blocked pair kernel (k_pair) for groups with exactly two varying inputs
template <typename T, typename OffT, int M>
void launch_p(const PArgs& pa, unsigned grid, size_t smem, cudaStream_t st) {
  allow_smem(k_pair<T, OffT, M>, smem);
  last_kernel() = KID_PAIR;
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

template bool try_launch_pair<float2>(const GDesc&, cudaStream_t);
template bool try_launch_pair<double2>(const GDesc&, cudaStream_t);

}  // namespace tnb
