// launch_gemm_hm.cu: k_gemm_hm (two-operand merge groups on mma.sync tf32, 3xTF32) -- part of
// libtnb200.so (see launch.cuh, kernels_hm.cuh)
#include "launch.cuh"
#include "kernels_hm.cuh"

#include <cstdio>

namespace tnb {

bool gemm_hm_enabled() {   // TNB_GEMM_HM=0 keeps the FP32 k_gemm for every group (read per call: tests switch it)
  const char* v = std::getenv("TNB_GEMM_HM");
  return !(v && v[0] == '0');
}

bool fc_hm_enabled() {   // TNB_FC_HM=1: producer -> consumer pairs on k_fc_hm (opt-in: measured slower
                         // than k_gemm_fc on C5a's pair, 439 vs 222 us, profiles/r02/hm/)
  const char* v = std::getenv("TNB_FC_HM");
  return v && v[0] == '1' && gemm_hm_enabled();
}

namespace {

constexpr int kHmWB = 2;                         // 4-warp CTAs
constexpr size_t kHmSmemPerSm = 220 * 1024;      // dynamic shared memory over all CTAs of an SM

int hm_stages() {   // TNB_HM_STAGES=2..4 (default 3): bulk-copy ring slots per operand
  static const int s = [] {
    const char* v = std::getenv("TNB_HM_STAGES");
    const int x = v ? std::atoi(v) : 3;
    return x < 2 ? 2 : (x > 4 ? 4 : x);
  }();
  return s;
}

template <int M, int NA, int NB, int NC, bool FC>
void launch_hm(const HArgs& ha, const FHArgs& fa, unsigned grid, size_t smem, cudaStream_t st) {
  allow_smem(k_gemm_hm<M, NA, NB, NC, kHmWB, FC>, smem);
  last_kernel() = FC ? KID_FC_HM : KID_GEMM_HM;
  k_gemm_hm<M, NA, NB, NC, kHmWB, FC><<<grid, (32 << kHmWB) + 32, smem, st>>>(ha, fa);
}

template <int M, bool FC>
bool dispatch_hm(const HArgs& ha, const FHArgs& fa, int na, int nb, int nc, unsigned grid, size_t smem, cudaStream_t st) {
#define HM_CASE(A, B, C) \
  if (na == A && nb == B && nc == C) { launch_hm<M, A, B, C, FC>(ha, fa, grid, smem, st); return true; }
  HM_CASE(0, 3, 0) HM_CASE(0, 2, 1) HM_CASE(0, 1, 2) HM_CASE(0, 0, 3) HM_CASE(1, 2, 0)
  HM_CASE(1, 1, 1) HM_CASE(1, 0, 2) HM_CASE(2, 1, 0) HM_CASE(2, 0, 1) HM_CASE(3, 0, 0)
#undef HM_CASE
  return false;
}

template <bool FC>
bool dispatch_m(const HArgs& ha, const FHArgs& fa, int M, int na, int nb, int nc, unsigned grid, size_t smem, cudaStream_t st) {
  switch (M) {
    case 2: return dispatch_hm<2, FC>(ha, fa, na, nb, nc, grid, smem, st);
    case 3: return dispatch_hm<3, FC>(ha, fa, na, nb, nc, grid, smem, st);
    case 4: return dispatch_hm<4, FC>(ha, fa, na, nb, nc, grid, smem, st);
    case 5: return dispatch_hm<5, FC>(ha, fa, na, nb, nc, grid, smem, st);
    default: return false;
  }
}

int lowest_bits(uint64_t m, int n, int* out) {   // the n lowest set bits of m (fewer if m has fewer)
  int k = 0;
  for (int b = 0; b < 64 && k < n; ++b)
    if ((m >> b) & 1) out[k++] = b;
  return k;
}

}  // namespace

// A c64 group whose varying inputs are two tensors, one holding >= 4 output bits the other does
// not hold (MMA rows) and the other >= 2 (MMA columns), whose other inputs hold no output bit, and
// whose output bits 0 and 1 are held by at least one of the two.  false when the shape does not
// qualify (the caller then takes k_gemm).
struct HmPlan {
  HArgs ha;
  int na, nb, nc;
  size_t smem;
  int cps;
  uint64_t ca, cb;   // row-only / column-only output bits
};

// Tile, roles and shared-memory layout of a k_gemm_hm launch.  `allowed`: the output bits a tile
// may hold; `yfirst` (ny bits, outside `allowed`): traversal bits that flip first (FC: the consumer's
// summed bits), the rest of the traversal being R-only, Q-only, then other bits.
// contig: the tile is the lowest 11 eligible output bits (long contiguous runs for the bulk copies:
// FC, where the consumer factor X is the largest stream); else every Q-only bit goes into the tile
// first (the row operand is then read once)
bool plan_hm(const GDesc& g, uint64_t allowed, const int* yfirst, int ny, const GIn* xop, bool contig, HmPlan& pl) {
  if (g.M < 2 || g.M > kMaxGroup || g.n < 2) return false;
  const int R = g.out_rank;
  if (R < 14 || R > 40) return false;
  int ia = -1, ib = -1;
  for (int t = 0; t < g.n; ++t) {
    const int r = __builtin_popcountll(g.in[t].out_mask);
    if (ia < 0 || r > __builtin_popcountll(g.in[ia].out_mask)) { ib = ia; ia = t; }
    else if (ib < 0 || r > __builtin_popcountll(g.in[ib].out_mask)) ib = t;
  }
  if (g.in[ia].rank > 32 || g.in[ib].rank > 32) return false;
  uint64_t ca = g.in[ia].out_mask & ~g.in[ib].out_mask, cb = g.in[ib].out_mask & ~g.in[ia].out_mask;
  uint64_t cc = g.in[ia].out_mask & g.in[ib].out_mask;
  // roles: the column operand Q gets the side with fewer exclusive tile-eligible bits (all of them
  // fit the tile, so the row operand is read exactly once); rows need >= 4, columns >= 2
  if (__builtin_popcountll(cb & allowed) > __builtin_popcountll(ca & allowed)) { std::swap(ia, ib); std::swap(ca, cb); }
  const uint64_t ca_all = ca, cb_all = cb;
  ca &= allowed;
  cb &= allowed;
  cc &= allowed;
  if (contig) {
    uint64_t pool = 0;
    int k = 0;
    for (int b = 0; b < R && k < 6 + kHmWB + 3; ++b)
      if (((ca | cb | cc) >> b) & 1) { pool |= 1ull << b; ++k; }
    ca &= pool;
    cb &= pool;
    cc &= pool;
  }
  if (__builtin_popcountll(ca) < 4 || __builtin_popcountll(cb) < 2) return false;
  for (int t = 0; t < g.n; ++t)   // constant inputs: no output bit (C[x] folded into Q's fragments)
    if (t != ia && t != ib && (g.in[t].out_mask != 0 || g.in[t].rank > 32)) return false;
  auto cls = [&](int b) { return ((ca >> b) & 1) ? 0 : ((cb >> b) & 1) ? 1 : ((cc >> b) & 1) ? 2 : 3; };
  // register slots: output bits 0 and 1 (r8 if R-only, else a fragment bit), then the lanes, then
  // fragment bits up to 3 (Q-only first: the whole Q-only set in the tile reads R once), then warps
  uint64_t used = 0;
  int r8 = -1;
  std::vector<int> fr[3];   // fragment bits by class
  for (int b = 0; b < 2; ++b) {
    const int c = cls(b);
    if (c == 3) return false;
    if (c == 0 && r8 < 0) r8 = b; else fr[c].push_back(b);
    used |= 1ull << b;
  }
  int tig[2], gb[3];
  if (lowest_bits(cb & ~used, 2, tig) < 2) return false;
  used |= (1ull << tig[0]) | (1ull << tig[1]);
  if (lowest_bits(ca & ~used, 3, gb) < 3) return false;
  for (int i = 0; i < 3; ++i) used |= 1ull << gb[i];
  if (r8 < 0) {
    int x;
    if (lowest_bits(ca & ~used, 1, &x) < 1) return false;
    r8 = x;
    used |= 1ull << r8;
  }
  auto nfrag = [&] { return (int)(fr[0].size() + fr[1].size() + fr[2].size()); };
  for (int pass = 0; pass < 3 && nfrag() < 3; ++pass) {
    const uint64_t m = (pass == 0 ? cb : pass == 1 ? cc : ca) & ~used;
    const int c = pass == 0 ? 1 : pass == 1 ? 2 : 0;
    for (int b = 0; b < R && nfrag() < 3; ++b)
      if ((m >> b) & 1) { fr[c].push_back(b); used |= 1ull << b; }
  }
  if (nfrag() != 3) return false;
  int wb[kHmWB], nw = 0;
  for (int pass = 0; pass < 2 && nw < kHmWB; ++pass) {   // Q-only warp bits first: warps share R
    const uint64_t m = (pass == 0 ? cb : (ca | cb | cc)) & ~used;
    for (int b = 0; b < R && nw < kHmWB; ++b)
      if ((m >> b) & 1) { wb[nw++] = b; used |= 1ull << b; }
  }
  if (nw < kHmWB) return false;
  const int NA = (int)fr[0].size(), NB = (int)fr[1].size(), NC = (int)fr[2].size();
  const int TB = 6 + kHmWB + 3;
  if (R < TB || (used >> 32)) return false;        // 32-bit tile offsets
  HArgs& ha = pl.ha;
  std::memset(&ha, 0, sizeof(ha));
  int u = 0;
  ha.outbit[u++] = (uint8_t)tig[0];
  ha.outbit[u++] = (uint8_t)tig[1];
  for (int i = 0; i < 3; ++i) ha.outbit[u++] = (uint8_t)gb[i];
  ha.outbit[u++] = (uint8_t)r8;
  for (int i = 0; i < kHmWB; ++i) ha.outbit[u++] = (uint8_t)wb[i];
  for (int c = 0; c < 3; ++c)
    for (int b : fr[c]) ha.outbit[u++] = (uint8_t)b;
  auto slot_of = [&](int ob) {                     // register slot of output bit ob
    if (ob == r8) return 0;
    for (int k = 0; k < 3; ++k)
      if (ha.outbit[6 + kHmWB + k] == ob) return 1 + k;
    return -1;
  };
  ha.p0 = slot_of(0);
  ha.p1 = slot_of(1);
  if (ha.p0 < 0 || ha.p1 < 0) return false;
  const uint64_t tmask = used;
  int nc = 0;
  for (int t = 0; t < g.n; ++t) {
    if (t == ia || t == ib) continue;
    ha.cin[nc] = g.in[t].ptr;
    for (int x = 0; x < (1 << g.M); ++x) ha.cgx[nc][x] = (uint32_t)g.in[t].gx[x];
    ++nc;
  }
  ha.nc = nc;
  // streams: R, Q and (FC) the consumer factor X, one chunk row (its y offset is added per tile)
  const int nops = xop ? 3 : 2;
  GIn xin1;
  if (xop) {
    xin1 = *xop;
    for (int x = 0; x < (1 << g.M); ++x) xin1.gx[x] = 0;
  }
  const GIn* op[3] = {&g.in[ia], &g.in[ib], xop ? &xin1 : nullptr};
  uint32_t sz[3] = {0, 0, 0}, nruns[3] = {0, 0, 0};
  for (int s = 0; s < nops; ++s) {
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
    uint32_t L = 0;                                // run: leading chunk bits at positions 0, 1, 2, ...
    while ((int)L < k && ha.posoff[s][L] == (1u << L)) ++L;
    if (L < 1) return false;                       // 16-byte bulk copies need >= 2 contiguous elements
    ha.runl[s] = L;
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
    if (s == 0) {   // R rows 16 floats apart in the banks when the row stride is a multiple of 32 floats
      const char* e = std::getenv("TNB_HM_RPAD");
      ha.rpad = (e && e[0] == '0') ? 0u : (((2u << k) % 32u) == 0u ? 16u : 0u);
      sz[s] += ha.nrows[s] * ha.rpad / 2u;
    }
    nruns[s] = ha.nrows[s] << (k - L);
  }
  if (xop) {   // X quads: output bits 0, 1 at X chunk positions 0, 1
    const int s0 = ha.p0 == 0 ? 5 : 6 + kHmWB + ha.p0 - 1, s1 = ha.p1 == 0 ? 5 : 6 + kHmWB + ha.p1 - 1;
    if (ha.chbit[2][s0] != 0 || ha.chbit[2][s1] != 1) return false;
  }
  const size_t qf_bytes = (size_t)(1 << kHmWB) * (1 << NB) * (1 << NC) * ((1 << g.M) / 4) * 32 * 16;
  // ring slots: R and X TNB_HM_STAGES (default 3), Q (reloaded rarely) 2; fewer when the shared
  // memory of two CTAs per SM does not hold them
  int S[3] = {hm_stages(), 2, hm_stages()};
  auto smem_for = [&]() {
    size_t b = qf_bytes;
    for (int s = 0; s < nops; ++s) b += (size_t)S[s] * sz[s] * 8 + (size_t)nruns[s] * 4;
    return b;
  };
  const size_t budget = kHmSmemPerSm / 2;          // at least two CTAs per SM
  while (smem_for() > budget && (S[0] > 2 || S[2] > 2)) {
    if (S[2] >= S[0] && S[2] > 2) --S[2]; else --S[0];
  }
  const size_t smem = smem_for();
  if (smem > budget) return false;
  size_t off = 0;
  for (int s = 0; s < nops; ++s) {
    ha.stages[s] = S[s];
    for (int k = 0; k < S[s]; ++k) { ha.sm_in[s][k] = (uint32_t)off; off += (size_t)sz[s] * 8; }
  }
  ha.sm_q = (uint32_t)off;
  off += qf_bytes;
  for (int s = 0; s < nops; ++s) { ha.sm_run[s] = (uint32_t)off; off += (size_t)nruns[s] * 4; }
  // traversal: `yfirst`, then R-only bits (Q's chunk and fragments unchanged), Q-only, the rest
  int np = 0;
  uint64_t yset = 0;
  for (int k = 0; k < ny; ++k) { ha.perm[np++] = (uint8_t)yfirst[k]; yset |= 1ull << yfirst[k]; }
  for (int pass = 0; pass < 3; ++pass)
    for (int b = 0; b < R; ++b) {
      if (((tmask | yset) >> b) & 1) continue;
      const uint64_t m = pass == 0 ? ca_all : pass == 1 ? cb_all : ~(ca_all | cb_all);
      if ((m >> b) & 1) ha.perm[np++] = (uint8_t)b;
    }
  if (np != R - TB) return false;
  ha.out = g.out;
  ha.out_rank = R;
  {
    const char* e = std::getenv("TNB_HM_DBG");
    ha.dbg = e ? std::atoi(e) : 0;
  }
  const int cps = std::max(1, std::min(4, (int)(kHmSmemPerSm / smem)));
  if (env_flag("TNB_GEMM_DEBUG")) {
    std::fprintf(stderr, "k_gemm_hm R=%d M=%d frag(a,b,c)=(%d,%d,%d) p=(%d,%d) nch=(%u,%u,%u) runl=(%u,%u,%u) rows=(%u,%u) S=(%d,%d,%d) smem=%zu cps=%d nc=%d outbits=",
                 R, g.M, NA, NB, NC, ha.p0, ha.p1, ha.nch[0], ha.nch[1], ha.nch[2], ha.runl[0], ha.runl[1], ha.runl[2],
                 ha.nrows[0], ha.nrows[1], S[0], S[1], S[2], smem, cps, nc);
    for (int uu = 0; uu < TB; ++uu) std::fprintf(stderr, "%d%s", ha.outbit[uu], uu + 1 < TB ? "," : "\n");
  }
  pl.na = NA;
  pl.nb = NB;
  pl.nc = NC;
  pl.smem = smem;
  pl.cps = cps;
  pl.ca = ca_all;
  pl.cb = cb_all;
  return true;
}

bool try_launch_gemm_hm(const GDesc& g, cudaStream_t st) {
  HmPlan pl;
  if (!plan_hm(g, ~0ull, nullptr, 0, nullptr, false, pl)) return false;
  const int TB = 6 + kHmWB + 3;
  const uint64_t tiles = 1ull << (g.out_rank - TB);
  const unsigned grid = (unsigned)std::min<uint64_t>(tiles, (uint64_t)num_sms() * pl.cps);
  FHArgs fa;
  std::memset(&fa, 0, sizeof(fa));
  return dispatch_m<false>(pl.ha, fa, g.M, pl.na, pl.nb, pl.nc, grid, pl.smem, st);
}

// The producer group g (GEMM-shaped) computed tile by tile on the tensor cores and consumed by
// group g3 (its input tin = g's output T) in registers: T never written.  false when the shapes do
// not qualify (the caller then takes k_gemm_fc).
bool try_launch_fc_hm(const GDesc& g, const GDesc& g3, int tin, cudaStream_t st) {
  const int R = g.out_rank, R3 = g3.out_rank, M3 = g3.M;
  if (R3 < 11 || R3 > 32 || M3 < 1 || M3 > kMaxGroup || R != R3 + M3) return false;
  const GIn& tIn = g3.in[tin];
  if (tIn.out_mask != (1ull << R3) - 1 || tIn.gx[0] != 0) return false;
  int ybit[kMaxGroup];
  for (int k = 0; k < M3; ++k) {
    const uint64_t v = tIn.gx[1u << k];
    if (v == 0 || (v & (v - 1)) != 0) return false;
    ybit[k] = __builtin_ctzll(v);
    if (ybit[k] < R3 || ybit[k] >= R) return false;
  }
  for (int x = 0; x < (1 << M3); ++x) {            // G_T(y) is the bit map above
    uint64_t e = 0;
    for (int k = 0; k < M3; ++k)
      if ((x >> k) & 1) e |= 1ull << ybit[k];
    if (tIn.gx[x] != e) return false;
  }
  FHArgs fa;
  std::memset(&fa, 0, sizeof(fa));
  fa.out3 = g3.out;
  fa.M3 = M3;
  fa.omask = (1ull << R3) - 1;
  int xi = -1;
  for (int t = 0; t < g3.n; ++t) {
    if (t == tin) continue;
    const GIn& in = g3.in[t];
    if (in.rank > 32) return false;
    if (in.out_mask != 0) {
      if (xi >= 0) return false;                   // one consumer factor X at most
      xi = t;
    } else {
      fa.win[fa.nw++] = in.ptr;
    }
  }
  if (xi >= 0) {
    const GIn& X = g3.in[xi];
    // 256-bit loads of X quads: X holds output bits 0 and 1 at its positions 0 and 1
    if (host_fmap(1, X.out_mask, X.pv) != 1 || host_fmap(2, X.out_mask, X.pv) != 2) return false;
    fa.xin = X.ptr;
    fa.xmask = X.out_mask;
    fa.xpv = X.pv;
  }
  HmPlan pl;
  // y order: bits held by the row operand only first, then shared, then column-only (Q's chunk and
  // fragments then change only when a Q y bit flips); decide the roles first without y bits
  // roles as plan_hm will choose them: recompute the classes to order y
  int ia = -1, ib = -1;
  for (int t = 0; t < g.n; ++t) {
    const int r = __builtin_popcountll(g.in[t].out_mask);
    if (ia < 0 || r > __builtin_popcountll(g.in[ia].out_mask)) { ib = ia; ia = t; }
    else if (ib < 0 || r > __builtin_popcountll(g.in[ib].out_mask)) ib = t;
  }
  uint64_t ca = g.in[ia].out_mask & ~g.in[ib].out_mask, cb = g.in[ib].out_mask & ~g.in[ia].out_mask;
  const uint64_t om = (1ull << R3) - 1;
  if (__builtin_popcountll(cb & om) > __builtin_popcountll(ca & om)) std::swap(ca, cb);
  int yo[kMaxGroup], ny = 0;
  for (int pass = 0; pass < 3; ++pass)
    for (int k = 0; k < M3; ++k) {
      const int b = ybit[k];
      const int cls = ((ca >> b) & 1) ? 0 : ((cb >> b) & 1) ? 2 : 1;
      if (cls == pass) yo[ny++] = k;
    }
  int yfirst[kMaxGroup];
  for (int k = 0; k < M3; ++k) yfirst[k] = ybit[yo[k]];
  if (xi < 0) return false;
  if (!plan_hm(g, om, yfirst, M3, &g3.in[xi], true, pl) && !plan_hm(g, om, yfirst, M3, &g3.in[xi], false, pl)) return false;
  // consumer tables in traversal order: tile-index bit k is the consumer's summed bit yo[k]
  for (int yp = 0; yp < (1 << M3); ++yp) {
    int x = 0;
    for (int k = 0; k < M3; ++k)
      if ((yp >> k) & 1) x |= 1 << yo[k];
    if (xi >= 0) fa.xgx[yp] = (uint32_t)g3.in[xi].gx[x];
    int w = 0;
    for (int t = 0; t < g3.n; ++t)
      if (t != tin && t != xi) fa.wgx[w++][yp] = (uint32_t)g3.in[t].gx[x];
  }
  const int TB = 6 + kHmWB + 3;
  const uint64_t groups = 1ull << (R - TB - M3);
  const unsigned grid = (unsigned)std::min<uint64_t>(groups, (uint64_t)num_sms() * pl.cps);
  if (env_flag("TNB_GEMM_DEBUG")) std::fprintf(stderr, "k_fc_hm R=%d R3=%d M3=%d grid=%u x=%d nw=%d\n", R, R3, M3, grid, xi, fa.nw);
  return dispatch_m<true>(pl.ha, fa, g.M, pl.na, pl.nb, pl.nc, grid, pl.smem, st);
}

}  // namespace tnb

