// launch_bucket.cu: standalone bucket step k_bucket<T, NIN> (generic gathers) -- part of libtnb200.so (see launch.cuh)
#include "launch.cuh"

namespace tnb {

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
  last_kernel() = KID_BUCKET;
  if (wide) {
    allow_smem(k_bucket<T, NIN, uint64_t>, smem);
    k_bucket<T, NIN, uint64_t><<<grid, kBucketThreads, smem, st>>>(a);
  } else {
    allow_smem(k_bucket<T, NIN, uint32_t>, smem);
    k_bucket<T, NIN, uint32_t><<<grid, kBucketThreads, smem, st>>>(a);
  }
}

template <typename T>
void launch_bucket_generic(const BigArgs& a, cudaStream_t st) {
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
template void launch_bucket_generic<float2>(const BigArgs&, cudaStream_t);
template void launch_bucket_generic<double2>(const BigArgs&, cudaStream_t);

}  // namespace tnb
