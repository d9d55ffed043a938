// launch_gemm_hm64.cu: k_gemm_hm64 (c128 two-operand merge groups on mma.sync f64 / DMMA) -- part of
// libtnb200.so (see launch.cuh, kernels_hm.cuh); its own translation unit so nvcc builds it in parallel
#include "launch.cuh"
#include "kernels_hm.cuh"

#include <cstdio>

namespace tnb {
namespace {

constexpr int kHmWB = 2;                         // 4 consumer warps + the producer warp
constexpr size_t kHmSmemPerSm = 220 * 1024;

int hm_stages() {   // TNB_HM_STAGES=2..4 (default 3): ring slots of the R stream (Q: 2)
  static const int s = [] {
    const char* v = std::getenv("TNB_HM_STAGES");
    const int x = v ? std::atoi(v) : 3;
    return x < 2 ? 2 : (x > 4 ? 4 : x);
  }();
  return s;
}

int lowest_bits(uint64_t m, int n, int* out) {   // the n lowest set bits of m (fewer if m has fewer)
  int k = 0;
  for (int b = 0; b < 64 && k < n; ++b)
    if ((m >> b) & 1) out[k++] = b;
  return k;
}

}  // namespace
}  // namespace tnb

namespace tnb {
namespace {

template <int M, int NA, int NB, int NC>
void launch_hm64(const HArgs& ha, unsigned grid, size_t smem, cudaStream_t st) {
  allow_smem(k_gemm_hm64<M, NA, NB, NC, kHmWB>, smem);
  last_kernel() = KID_GEMM_HM;
  k_gemm_hm64<M, NA, NB, NC, kHmWB><<<grid, (32 << kHmWB) + 32, smem, st>>>(ha);
}

template <int M>
bool dispatch_hm64(const HArgs& ha, int na, int nb, int nc, unsigned grid, size_t smem, cudaStream_t st) {
#define HM64_CASE(A, B, C) \
  if (na == A && nb == B && nc == C) { launch_hm64<M, A, B, C>(ha, grid, smem, st); return true; }
  HM64_CASE(0, 3, 0) HM64_CASE(0, 2, 1) HM64_CASE(0, 1, 2) HM64_CASE(0, 0, 3) HM64_CASE(1, 2, 0)
  HM64_CASE(1, 1, 1) HM64_CASE(1, 0, 2) HM64_CASE(2, 1, 0) HM64_CASE(2, 0, 1) HM64_CASE(3, 0, 0)
#undef HM64_CASE
  return false;
}

}  // namespace

// c128 two-operand group on DMMA (k_gemm_hm64): R holds >= 3 output bits Q does not hold, Q >= 2,
// output bit 0 held by an operand (a register slot: whole 32-byte sectors per store)
bool try_launch_gemm_hm64(const GDesc& g, cudaStream_t st) {
  if (g.M < 1 || g.M > kMaxGroup || g.n < 2) return false;
  const int R = g.out_rank;
  const int TB = 5 + kHmWB + 3;
  if (R < TB + 1 || R > 40) return false;
  int ia = -1, ib = -1;
  for (int t = 0; t < g.n; ++t) {
    const int r = __builtin_popcountll(g.in[t].out_mask);
    if (ia < 0 || r > __builtin_popcountll(g.in[ia].out_mask)) { ib = ia; ia = t; }
    else if (ib < 0 || r > __builtin_popcountll(g.in[ib].out_mask)) ib = t;
  }
  if (g.in[ia].rank > 32 || g.in[ib].rank > 32) return false;
  uint64_t ca = g.in[ia].out_mask & ~g.in[ib].out_mask, cb = g.in[ib].out_mask & ~g.in[ia].out_mask;
  const uint64_t cc = g.in[ia].out_mask & g.in[ib].out_mask;
  if (__builtin_popcountll(cb) > __builtin_popcountll(ca)) { std::swap(ia, ib); std::swap(ca, cb); }
  if (__builtin_popcountll(ca) < 3 || __builtin_popcountll(cb) < 2) return false;
  for (int t = 0; t < g.n; ++t)
    if (t != ia && t != ib && (g.in[t].out_mask != 0 || g.in[t].rank > 32)) return false;
  auto cls = [&](int b) { return ((ca >> b) & 1) ? 0 : ((cb >> b) & 1) ? 1 : ((cc >> b) & 1) ? 2 : 3; };
  uint64_t used = 1ull;
  std::vector<int> fr[3];
  {
    const int c0 = cls(0);
    if (c0 == 3) return false;
    fr[c0].push_back(0);                           // output bit 0: a register slot
  }
  int tig[2], gb[3];
  if (lowest_bits(cb & ~used, 2, tig) < 2) return false;
  used |= (1ull << tig[0]) | (1ull << tig[1]);
  if (lowest_bits(ca & ~used, 3, gb) < 3) return false;
  for (int i = 0; i < 3; ++i) used |= 1ull << gb[i];
  auto nfrag = [&] { return (int)(fr[0].size() + fr[1].size() + fr[2].size()); };
  for (int pass = 0; pass < 3 && nfrag() < 3; ++pass) {
    const uint64_t m = (pass == 0 ? cb : pass == 1 ? cc : ca) & ~used;
    const int c = pass == 0 ? 1 : pass == 1 ? 2 : 0;
    for (int b = 0; b < R && nfrag() < 3; ++b)
      if ((m >> b) & 1) { fr[c].push_back(b); used |= 1ull << b; }
  }
  if (nfrag() != 3) return false;
  for (auto& v : fr) std::sort(v.begin(), v.end());
  int wb[kHmWB], nw = 0;
  for (int pass = 0; pass < 2 && nw < kHmWB; ++pass) {
    const uint64_t m = (pass == 0 ? cb : (ca | cb | cc)) & ~used;
    for (int b = 0; b < R && nw < kHmWB; ++b)
      if ((m >> b) & 1) { wb[nw++] = b; used |= 1ull << b; }
  }
  if (nw < kHmWB || (used >> 32)) return false;
  const int NA = (int)fr[0].size(), NB = (int)fr[1].size(), NC = (int)fr[2].size();
  HArgs ha;
  std::memset(&ha, 0, sizeof(ha));
  int u = 0;
  ha.outbit[u++] = (uint8_t)tig[0];
  ha.outbit[u++] = (uint8_t)tig[1];
  for (int i = 0; i < 3; ++i) ha.outbit[u++] = (uint8_t)gb[i];
  for (int i = 0; i < kHmWB; ++i) ha.outbit[u++] = (uint8_t)wb[i];
  for (int c = 0; c < 3; ++c)
    for (int b : fr[c]) ha.outbit[u++] = (uint8_t)b;
  ha.p0 = -1;
  for (int k = 0; k < 3; ++k)
    if (ha.outbit[5 + kHmWB + k] == 0) ha.p0 = k;
  if (ha.p0 < 0) return false;
  const uint64_t tmask = used;
  int nc = 0;
  for (int t = 0; t < g.n; ++t) {
    if (t == ia || t == ib) continue;
    ha.cin[nc] = g.in[t].ptr;
    for (int x = 0; x < (1 << g.M); ++x) ha.cgx[nc][x] = (uint32_t)g.in[t].gx[x];
    ++nc;
  }
  ha.nc = nc;
  const GIn* op[2] = {&g.in[ia], &g.in[ib]};
  uint32_t sz[2], nruns[2];
  for (int s = 0; s < 2; ++s) {
    const GIn& in = *op[s];
    int k = 0;
    for (int b = 0; b < R; ++b) {
      if (!((tmask >> b) & 1) || !((in.out_mask >> b) & 1)) continue;
      for (int uu = 0; uu < TB; ++uu)
        if (ha.outbit[uu] == b) ha.chbit[s][uu] = (int8_t)k;
      ha.posoff[s][k] = (uint32_t)host_fmap(1ull << b, in.out_mask, in.pv);
      ++k;
    }
    for (int uu = 0; uu < TB; ++uu)
      if (!((in.out_mask >> ha.outbit[uu]) & 1)) ha.chbit[s][uu] = -1;
    ha.nch[s] = (uint32_t)k;
    uint32_t L = 0;
    while ((int)L < k && ha.posoff[s][L] == (1u << L)) ++L;
    ha.runl[s] = L;                                // 16-byte elements: any run length copies
    std::vector<uint64_t> parts;
    for (int x = 0; x < (1 << g.M); ++x) {
      auto it = std::find(parts.begin(), parts.end(), in.gx[x]);
      if (it == parts.end()) {
        ha.row[s][x] = (uint8_t)parts.size();
        parts.push_back(in.gx[x]);
      } else {
        ha.row[s][x] = (uint8_t)(it - parts.begin());
      }
    }
    for (size_t r = 0; r < parts.size(); ++r) ha.rowoff[s][r] = (uint32_t)parts[r];
    ha.nrows[s] = (uint32_t)parts.size();
    ha.in[s] = in.ptr;
    ha.mask[s] = in.out_mask;
    ha.pv[s] = in.pv;
    sz[s] = ha.nrows[s] << k;
    nruns[s] = ha.nrows[s] << (k - L);
  }
  if (nruns[0] > 256 || nruns[1] > 1024) return false;   // bulk-copy counts per chunk
  const int KS = (1 << g.M) / 2;
  const size_t qf_bytes = (size_t)(1 << kHmWB) * (1 << NB) * (1 << NC) * KS * 32 * 8;
  int S[2] = {hm_stages(), 2};
  auto smem_for = [&]() {
    size_t b = qf_bytes;
    for (int s = 0; s < 2; ++s) b += (size_t)S[s] * sz[s] * 16 + (size_t)nruns[s] * 4;
    return b;
  };
  const size_t budget = kHmSmemPerSm / 2;
  while (smem_for() > budget && S[0] > 2) --S[0];
  const size_t smem = smem_for();
  if (smem > budget) return false;
  size_t off = 0;
  for (int s = 0; s < 2; ++s) {
    ha.stages[s] = S[s];
    for (int k = 0; k < S[s]; ++k) { ha.sm_in[s][k] = (uint32_t)off; off += (size_t)sz[s] * 16; }
  }
  ha.sm_q = (uint32_t)off;
  off += qf_bytes;
  for (int s = 0; s < 2; ++s) { ha.sm_run[s] = (uint32_t)off; off += (size_t)nruns[s] * 4; }
  int np = 0;
  for (int pass = 0; pass < 3; ++pass)
    for (int b = 0; b < R; ++b) {
      if ((tmask >> b) & 1) continue;
      const uint64_t m = pass == 0 ? ca : pass == 1 ? cb : ~(ca | cb);
      if ((m >> b) & 1) ha.perm[np++] = (uint8_t)b;
    }
  if (np != R - TB) return false;
  ha.out = g.out;
  ha.out_rank = R;
  const int cps = std::max(1, std::min(4, (int)(kHmSmemPerSm / smem)));
  if (env_flag("TNB_GEMM_DEBUG")) {
    std::fprintf(stderr, "k_gemm_hm64 R=%d M=%d frag(a,b,c)=(%d,%d,%d) p0=%d nch=(%u,%u) runl=(%u,%u) S=(%d,%d) smem=%zu cps=%d outbits=",
                 R, g.M, NA, NB, NC, ha.p0, ha.nch[0], ha.nch[1], ha.runl[0], ha.runl[1], S[0], S[1], smem, cps);
    for (int uu = 0; uu < TB; ++uu) std::fprintf(stderr, "%d%s", ha.outbit[uu], uu + 1 < TB ? "," : "\n");
  }
  const uint64_t tiles = 1ull << (R - TB);
  const unsigned grid = (unsigned)std::min<uint64_t>(tiles, (uint64_t)num_sms() * cps);
  switch (g.M) {
    case 1: return dispatch_hm64<1>(ha, NA, NB, NC, grid, smem, st);
    case 2: return dispatch_hm64<2>(ha, NA, NB, NC, grid, smem, st);
    case 3: return dispatch_hm64<3>(ha, NA, NB, NC, grid, smem, st);
    case 4: return dispatch_hm64<4>(ha, NA, NB, NC, grid, smem, st);
    case 5: return dispatch_hm64<5>(ha, NA, NB, NC, grid, smem, st);
    default: return false;
  }
}

}  // namespace tnb
