// launch_gemm_tc.cu: k_gemm_tc (tcgen05 kind::tf32, 3xTF32) for two-operand fused merge groups --
// part of libtnb200.so (see launch.cuh, kernels_tc.cuh)
#include "launch.cuh"
#include "kernels_tc.cuh"

#include <cstdio>
#include <tuple>

namespace tnb {

constexpr size_t kTcSmemLimit = 220 * 1024;   // + ~6 KB static <= 227 KB per block

// In a plan the tensor-core path is opt-in (TNB_GEMM_TC=1): measured slower than the FP32 k_gemm kernels on the
// C5a groups ("k_gemm_tc"); tn_eliminate_group(kernel = 4) always takes it.
bool gemm_tc_enabled() {
  static const bool on = env_flag("TNB_GEMM_TC");
  return on;
}

namespace {

struct TcTile {
  int nr = 0, nb = 0, nd = 0;
  int role[64];      // per output bit: -1 outside the tile, else 0 row / 1 col / 2 diag
  int run = 0;       // output bits 0 .. run-1 all in the tile
};

// greedy walk from the lowest output bit: row bits of class `rc` (7), col bits of class `cc` and
// diag bits (class c) within the caps
TcTile walk(int R, const char* cls, char rc, char cc, int nd_cap, int nbd_cap) {
  TcTile t;
  for (int b = 0; b < R; ++b) {
    t.role[b] = -1;
    if (cls[b] == rc && t.nr < 7) { t.role[b] = 0; ++t.nr; }
    else if (cls[b] == cc && t.nb + t.nd < nbd_cap) { t.role[b] = 1; ++t.nb; }
    else if (cls[b] == 'c' && t.nd < nd_cap && t.nd + 1 + std::max(t.nb, 3) <= nbd_cap) { t.role[b] = 2; ++t.nd; }
  }
  while (t.run < R && t.role[t.run] >= 0) ++t.run;
  return t;
}

}  // namespace

// dynamic shared memory of a k_gemm_tc tile (kernels_tc.cuh layout): A' buffers, two B' slots,
// two staging tiles, offset tables, raw A, S raw-B / C slots
size_t tc_smem(int nd, int nb, int K, int abufs, int S) {
  const int TB = 7 + nb + nd, ND = 1 << nd, NC = 1 << nb, kp = std::max(8, 2 * K);
  const size_t abytes = (size_t)128 * kp * 4, bbytes = (size_t)2 * NC * kp * 4;
  const size_t nA = (size_t)1 << (7 + nd), nBc = (size_t)1 << (nb + nd), nHi = (size_t)1 << (TB - 8);
  return (size_t)abufs * 2 * ND * abytes + 2 * 2 * ND * bbytes + 2 * ((size_t)8 << TB) +
         4 * (2 * nA + 3 * nBc + ((nHi + 1) & ~(size_t)1)) + 8 * (256 + nHi) +
         8 * ((size_t)K * nA + (size_t)S * ((size_t)K * nBc + (size_t)K * kMaxIn));
}

bool try_launch_gemm_tc(const GDesc& g, cudaStream_t st) {
  if (gemm_disabled() || g.M < 1 || g.M > kMaxGroup || g.n < 2) return false;
  const int R = g.out_rank;
  if (R < 11 || R > 40) return false;
  int ia = -1, ib = -1;
  for (int t = 0; t < g.n; ++t) {
    const int r = __builtin_popcountll(g.in[t].out_mask);
    if (ia < 0 || r > __builtin_popcountll(g.in[ia].out_mask)) { ib = ia; ia = t; }
    else if (ib < 0 || r > __builtin_popcountll(g.in[ib].out_mask)) ib = t;
  }
  if (g.in[ia].rank > 32 || g.in[ib].rank > 32) return false;
  char cls[64];
  for (int b = 0; b < R; ++b) {
    const bool ha = (g.in[ia].out_mask >> b) & 1, hb = (g.in[ib].out_mask >> b) & 1;
    cls[b] = ha && hb ? 'c' : ha ? 'a' : hb ? 'b' : 'n';
  }
  for (int t = 0; t < g.n; ++t) {
    if (t == ia || t == ib) continue;
    if (g.in[t].rank > 32) return false;
  }
  const int K = 1 << g.M, kp = std::max(8, 2 * K);
  // candidate tiles: every (diag cap, col+diag cap) and both operand roles.  Ranking: output
  // pieces of >= 8 elements (64 B: whole sectors), then the fewest diag blocks (each is its own
  // chain of 3 KC MMAs: a tf32 MMA at N <= 128 costs ~60-110 cycles whatever its N, so fewer and
  // wider MMAs), then the longer contiguous run, then the larger tile
  static const int caps[][2] = {{0, 6}, {1, 6}, {2, 6}, {0, 5}, {1, 5}, {2, 5}, {0, 4}, {1, 4}, {2, 4}};
  TcTile best;
  bool have = false, best_swap = false;
  int best_abufs = 1;
  auto key = [](const TcTile& t) {
    return std::make_tuple(t.run >= 3 ? 1 : 0, -t.nd, std::min(t.run, 5), t.nb + t.nd);
  };
  for (const auto& cp : caps) {
    for (int sw = 0; sw < 2; ++sw) {
      const char rc = sw ? 'b' : 'a', cc = sw ? 'a' : 'b';
      TcTile t = walk(R, cls, rc, cc, cp[0], cp[1]);
      if (t.nr != 7 || t.nb < 3 || t.nb + t.nd < 4) continue;
      const int ND = 1 << t.nd, NC = 1 << t.nb;
      // constant inputs may not hold tile bits
      bool ok = true;
      for (int q = 0; q < g.n && ok; ++q) {
        if (q == ia || q == ib) continue;
        for (int b = 0; b < R; ++b)
          if (t.role[b] >= 0 && ((g.in[q].out_mask >> b) & 1)) { ok = false; break; }
      }
      if (!ok) continue;
      if (2 * ND * NC > 128) continue;             // <= 128 accumulator columns per tile
      // two A' buffers when they fit (the next A chunk is formatted while MMAs read the current)
      for (int abufs = 2; abufs >= 1; --abufs) {
        const size_t smem = tc_smem(t.nd, t.nb, K, abufs, 2);
        if (smem > kTcSmemLimit) continue;
        if (!have || key(t) > key(best) || (key(t) == key(best) && abufs > best_abufs)) {
          best = t;
          best_swap = sw != 0;
          best_abufs = abufs;
          have = true;
        }
        break;
      }
    }
  }
  if (!have) return false;
  const GIn& A = g.in[best_swap ? ib : ia];
  const GIn& Bq = g.in[best_swap ? ia : ib];
  const char rcl = best_swap ? 'b' : 'a', ccl = best_swap ? 'a' : 'b';
  TArgs ta;
  std::memset(&ta, 0, sizeof(ta));
  ta.out = g.out;
  ta.A = static_cast<const float2*>(A.ptr);
  ta.B = static_cast<const float2*>(Bq.ptr);
  ta.maskA = A.out_mask;
  ta.maskB = Bq.out_mask;
  ta.pvA = A.pv;
  ta.pvB = Bq.pv;
  for (int x = 0; x < K; ++x) {
    ta.rowoffA[x] = (uint32_t)A.gx[x];
    ta.rowoffB[x] = (uint32_t)Bq.gx[x];
  }
  int nc = 0;
  for (int q = 0; q < g.n; ++q) {
    if (q == ia || q == ib) continue;
    ta.cin[nc] = g.in[q].ptr;
    ta.cmask[nc] = g.in[q].out_mask;
    ta.cpv[nc] = g.in[q].pv;
    for (int x = 0; x < K; ++x) ta.cgx[nc][x] = (uint32_t)g.in[q].gx[x];
    ++nc;
  }
  ta.nc = nc;
  ta.M = g.M;
  ta.nd = best.nd;
  ta.nb = best.nb;
  ta.TB = 7 + best.nb + best.nd;
  ta.kp = kp;
  int u = 0, cnt[3] = {0, 0, 0};
  uint64_t tmask = 0;
  for (int b = 0; b < R; ++b) {
    if (best.role[b] < 0) continue;
    ta.role[u] = (uint8_t)best.role[b];
    ta.rj[u] = (uint8_t)cnt[best.role[b]]++;
    ta.obit[u] = 1ull << b;
    ta.posA[u] = ((A.out_mask >> b) & 1) ? (uint32_t)host_fmap(1ull << b, A.out_mask, A.pv) : 0u;
    ta.posB[u] = ((Bq.out_mask >> b) & 1) ? (uint32_t)host_fmap(1ull << b, Bq.out_mask, Bq.pv) : 0u;
    tmask |= 1ull << b;
    ++u;
  }
  const int TB = ta.TB;
  // staging swizzle: the 5 lowest row bits are a warp's lanes; give each lane bit at compact
  // position >= 4 a 4-bit XOR so that the lanes' low nibbles span GF(2)^4 (2 wavefronts per store)
  {
    uint32_t span[16];
    int ns = 1;
    span[0] = 0;
    auto in_span = [&](uint32_t v) {
      for (int i = 0; i < ns; ++i) if (span[i] == v) return true;
      return false;
    };
    auto add = [&](uint32_t v) {
      const int n0 = ns;
      for (int i = 0; i < n0; ++i) span[ns++] = span[i] ^ v;
    };
    int lane_pos[5], nl = 0;
    for (int q = 0; q < TB && nl < 5; ++q)
      if (ta.role[q] == 0) lane_pos[nl++] = q;
    for (int i = 0; i < nl; ++i)
      if (lane_pos[i] < 4 && !in_span(1u << lane_pos[i])) add(1u << lane_pos[i]);
    for (int i = 0; i < nl; ++i) {
      if (lane_pos[i] < 4 || ns == 16) continue;
      for (uint32_t v = 1; v < 16; ++v)
        if (!in_span(v)) { ta.sw[lane_pos[i]] = (uint8_t)v; add(v); break; }
    }
  }
  // traversal: outer col bits first (A's chunk and A' stay), then row bits, then the rest
  int np = 0;
  for (int pass = 0; pass < 3; ++pass)
    for (int b = 0; b < R; ++b) {
      if ((tmask >> b) & 1) continue;
      const bool take = pass == 0 ? cls[b] == ccl : pass == 1 ? cls[b] == rcl : (cls[b] == 'c' || cls[b] == 'n');
      if (take) ta.perm[np++] = (uint8_t)b;
    }
  if (np != R - TB || np > kTcMaxPerm) return false;
  ta.nperm = np;
  ta.n_tiles = 1ull << (R - TB);
  ta.pair16 = best.role[0] >= 0 ? 1 : 0;
  const int ND = 1 << best.nd, NC = 1 << best.nb;
  ta.abytes_d = (uint32_t)(128 * kp * 4);
  ta.bbytes_d = (uint32_t)(2 * NC * kp * 4);
  ta.abufs = best_abufs;
  ta.sm_b = (uint32_t)best_abufs * 2u * ND * ta.abytes_d;
  ta.sm_stage = ta.sm_b + 2u * 2u * ND * ta.bbytes_d;
  ta.sm_tabs = ta.sm_stage + 2u * (8u << TB);
  size_t best_smem;
  {
    const uint32_t nA = 1u << (7 + best.nd), nBc = 1u << (best.nb + best.nd), nHi = 1u << (TB - 8);
    ta.sm_raw = ta.sm_tabs + 4u * (2u * nA + 3u * nBc + ((nHi + 1u) & ~1u)) + 8u * (256u + nHi);
    int S = 5;
    while (S > 2 && tc_smem(best.nd, best.nb, K, best_abufs, S) > kTcSmemLimit) --S;
    ta.bslots = S;
    best_smem = tc_smem(best.nd, best.nb, K, best_abufs, S);
  }
  const uint32_t tcol = (uint32_t)(2 * ND * 2 * NC);
  uint32_t cols = 32;
  while (cols < tcol) cols <<= 1;
  ta.tmem_cols = cols;
  if (env_flag("TNB_GEMM_DEBUG")) {
    std::fprintf(stderr, "k_gemm_tc R=%d M=%d TB=%d nb=%d nd=%d run=%d swap=%d smem=%zu S=%d abufs=%d tmem=%u roles=", R, g.M,
                 TB, best.nb, best.nd, best.run, (int)best_swap, best_smem, ta.bslots, best_abufs, cols);
    for (int b = 0; b < R; ++b) std::fprintf(stderr, "%c", best.role[b] < 0 ? '.' : "rcd"[best.role[b]]);
    std::fprintf(stderr, "\n");
  }
  static const bool granted = [] {
    cudaFuncSetAttribute(k_gemm_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTcSmemLimit);
    return true;
  }();
  (void)granted;
  {
    static const int dbg = [] { const char* v = std::getenv("TNB_TC_DBG"); return v ? std::atoi(v) : 0; }();
    ta.dbg = dbg;
  }
  const unsigned grid = (unsigned)std::min<uint64_t>(ta.n_tiles, (uint64_t)num_sms());
  last_kernel() = KID_GEMM_TC;
  if (ta.dbg & 8) {
    static unsigned long long* tr = nullptr;
    if (!tr) cudaMalloc(&tr, 64 * 8 * 8);
    cudaMemsetAsync(tr, 0, 64 * 8 * 8, st);
    ta.trace = tr;
    k_gemm_tc<<<grid, kTcThreads, best_smem, st>>>(ta);
    unsigned long long h[64 * 8];
    cudaMemcpyAsync(h, tr, sizeof(h), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    const unsigned long long b = h[0];
    for (int i = 0; i < 64 && h[i * 8 + 1]; ++i)
      std::fprintf(stderr, "tc trace tile %2d: ld_wait %7lld ld_b %7lld ld_done %7lld mma_start %7lld mma %7lld epi_ok %7lld staged %7lld stored %7lld\n", i,
                   (long long)(h[i * 8 + 6] - b), (long long)(h[i * 8 + 7] - b), (long long)(h[i * 8] - b), (long long)(h[i * 8 + 5] - b), (long long)(h[i * 8 + 1] - b), (long long)(h[i * 8 + 2] - b),
                   (long long)(h[i * 8 + 3] - b), (long long)(h[i * 8 + 4] - b));
    return true;
  }
  k_gemm_tc<<<grid, kTcThreads, best_smem, st>>>(ta);
  return true;
}

}  // namespace tnb
