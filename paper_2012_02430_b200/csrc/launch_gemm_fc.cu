// launch_gemm_fc.cu: k_gemm_fc (a GEMM-shaped merge group computed tile by tile and consumed by the
// next merge group without being written; OP_GROUP_FEED) -- part of libtnb200.so (see launch.cuh,
// kernels_fc.cuh).  The tile / chunk / ring set-up follows try_launch_gemm_impl (launch_gemm.cu);
// the differences: every tile bit is an output bit of the consumer, and the tile traversal runs
// over the consumer's summed indices first.
#include "launch.cuh"
#include "kernels_fc.cuh"

#include <cstdio>

namespace tnb {

constexpr size_t kFcSmemBudget = 100 * 1024;   // two CTAs per SM, as k_gemm

inline int fc_rbb() {   // TNB_FC_RBB = 1 (4 x 2 register blocks, 2 CTAs / SM) or 2 (4 x 4, 1 CTA / SM;
                        // default: C5a 75.2 vs 73.7 contractions/s)
  static const int v = [] {
    const char* e = std::getenv("TNB_FC_RBB");
    return e && e[0] == '1' ? 1 : 2;
  }();
  return v;
}

inline bool fc_shrink() {   // TNB_FC_SHRINK=1: smaller blocks for small consumers (measured slower with
                            // 8 slice lanes: C4b 52.3 vs 56.0 /s -- the lanes already fill the GPU)
  static const bool v = env_flag("TNB_FC_SHRINK");
  return v;
}

bool fc_enabled() {   // TNB_NO_FC=1: run producer and consumer as two launches
  static const bool off = env_flag("TNB_NO_FC");
  return !off;
}

template <int M, int RAB, int RBB, int WB>
void launch_fc(const MArgs& ma, const FArgs& fa, unsigned grid, size_t smem, cudaStream_t st) {
  allow_smem(k_gemm_fc<M, RAB, RBB, WB>, smem);
  last_kernel() = KID_GEMM_FC;
  k_gemm_fc<M, RAB, RBB, WB><<<grid, 32 << WB, smem, st>>>(ma, fa);
}

template <int M, int WB>
bool dispatch_fc(const MArgs& ma, const FArgs& fa, int rab, int rbb, unsigned grid, size_t smem, cudaStream_t st) {
  if (rab == 2 && rbb == 2) { launch_fc<M, 2, 2, WB>(ma, fa, grid, smem, st); return true; }
  if (rab == 2 && rbb == 1) { launch_fc<M, 2, 1, WB>(ma, fa, grid, smem, st); return true; }
  if (rab == 1 && rbb == 2) { launch_fc<M, 1, 2, WB>(ma, fa, grid, smem, st); return true; }
  if (rab == 1 && rbb == 1) { launch_fc<M, 1, 1, WB>(ma, fa, grid, smem, st); return true; }
  return false;
}

inline int fc_wb() {   // TNB_FC_WB = 2 (4-warp CTAs, 4 per SM) or 3 (8-warp CTAs, 2 per SM)
  static const int v = [] { const char* e = std::getenv("TNB_FC_WB"); return e && e[0] == '2' ? 2 : 3; }();
  return v;
}

#define FC_DECLINE(why)                                                                     \
  do {                                                                                      \
    if (env_flag("TNB_GEMM_DEBUG")) std::fprintf(stderr, "k_gemm_fc declined: %s\n", why);   \
    return false;                                                                           \
  } while (0)

template <typename T>
bool try_launch_gemm_fc_wb(const GDesc& g, const GDesc& g3, int tin, cudaStream_t st, int WB, uint32_t* sem);

inline bool fc_split() {   // TNB_FC_SPLIT=1: consumer blocks split between neighbouring CTAs (balanced
                           // per-SM load; C5a: the launch 209 vs 222 us alone, but the step with 16
                           // slice lanes 98.0 vs 100.5 /s -- the lanes fill the idle slots), off;
                           // read per launch (the parity test runs both in one process)
  const char* e = std::getenv("TNB_FC_SPLIT");
  return e && e[0] == '1';
}

inline unsigned fc_cps() {   // TNB_FC_CPS: k_gemm_fc CTAs per SM in the grid (default: as many as fit)
  static const unsigned v = [] { const char* e = std::getenv("TNB_FC_CPS"); return e ? (unsigned)std::atoi(e) : 0u; }();
  return v;
}

template <typename T>
bool try_launch_gemm_fc(const GDesc& g, const GDesc& g3, int tin, cudaStream_t st, uint32_t* sem) {
  const int wb0 = fc_wb();
  if (!fc_split()) sem = nullptr;
  return try_launch_gemm_fc_wb<T>(g, g3, tin, st, wb0, sem) || try_launch_gemm_fc_wb<T>(g, g3, tin, st, 5 - wb0, sem);
}

template <typename T>
bool try_launch_gemm_fc_wb(const GDesc& g, const GDesc& g3, int tin, cudaStream_t st, int WB, uint32_t* sem) {
  if constexpr (!std::is_same<T, float2>::value) {
    (void)g; (void)g3; (void)tin; (void)st; (void)WB; (void)sem;
    return false;
  } else {
    if (gemm_disabled() || g.M < 1 || g.M > kMaxGroup || g.n < 2) FC_DECLINE("producer M / inputs");
    const int R = g.out_rank, R3 = g3.out_rank, M3 = g3.M;
    if (R < 11 || R > 40 || R3 < 11 || R3 > 32 || M3 < 1 || M3 > kMaxGroup || R != R3 + M3) FC_DECLINE("ranks");
    // T = g.out is the consumer's input tin: full, its low R3 bits the consumer's output bits, y bit
    // k of the consumer's summed value at T bit ybit[k] >= R3
    const GIn& tIn = g3.in[tin];
    if (tIn.out_mask != (1ull << R3) - 1 || tIn.gx[0] != 0) FC_DECLINE("T not full");
    int ybit[kMaxGroup];
    for (int k = 0; k < M3; ++k) {
      const uint64_t v = tIn.gx[1u << k];
      if (v == 0 || (v & (v - 1)) != 0) FC_DECLINE("y map");
      ybit[k] = __builtin_ctzll(v);
      if (ybit[k] < R3 || ybit[k] >= R) FC_DECLINE("y bits");
    }
    for (int x = 0; x < (1 << M3); ++x) {   // G_T(y) is the bit map above
      uint64_t e = 0;
      for (int k = 0; k < M3; ++k)
        if ((x >> k) & 1) e |= 1ull << ybit[k];
      if (tIn.gx[x] != e) FC_DECLINE("y map linear");
    }
    FArgs fa;
    std::memset(&fa, 0, sizeof(fa));
    fa.out3 = g3.out;
    fa.M3 = M3;
    fa.omask = (1ull << R3) - 1;
    for (int t = 0; t < g3.n; ++t) {
      if (t == tin) continue;
      const GIn& in = g3.in[t];
      if (in.rank > 32) FC_DECLINE("consumer rank");
      if (in.out_mask != 0) {
        if (fa.nv >= kFcMaxV) FC_DECLINE("consumer inputs");
        fa.vin[fa.nv] = in.ptr;
        fa.vmask[fa.nv] = in.out_mask;
        fa.vpv[fa.nv] = in.pv;
        for (int x = 0; x < (1 << M3); ++x) fa.vgx[fa.nv][x] = (uint32_t)in.gx[x];
        ++fa.nv;
      } else {
        fa.win[fa.nw] = in.ptr;
        for (int x = 0; x < (1 << M3); ++x) fa.wgx[fa.nw][x] = (uint32_t)in.gx[x];
        ++fa.nw;
      }
    }
    {   // X prefetch (TNB_FC_XPF=0 off): X holds output bits 0..4 at its positions 0..4
      const char* e = std::getenv("TNB_FC_XPF");
      bool ok = fa.nv == 1 && !(e && e[0] == '0');
      for (int k = 0; k < 5 && ok; ++k) ok = host_fmap(1ull << k, fa.vmask[0], fa.vpv[0]) == (1ull << k);
      fa.xpf = ok ? 1 : 0;
    }
    // producer: A, B = the two inputs with the most output bits
    int ia = -1, ib = -1;
    for (int t = 0; t < g.n; ++t) {
      const int r = __builtin_popcountll(g.in[t].out_mask);
      if (ia < 0 || r > __builtin_popcountll(g.in[ia].out_mask)) { ib = ia; ia = t; }
      else if (ib < 0 || r > __builtin_popcountll(g.in[ib].out_mask)) ib = t;
    }
    if (g.in[ia].rank > 32 || g.in[ib].rank > 32) FC_DECLINE("producer rank");
    const uint64_t full = (1ull << R) - 1;
    uint64_t ca = g.in[ia].out_mask & ~g.in[ib].out_mask, cb = g.in[ib].out_mask & ~g.in[ia].out_mask;
    const uint64_t cc = g.in[ia].out_mask & g.in[ib].out_mask, cn = full & ~(g.in[ia].out_mask | g.in[ib].out_mask);
    if (cn & 31ull) FC_DECLINE("lanes");   // lanes must be held by A or B
    uint64_t ymask = 0;
    for (int k = 0; k < M3; ++k) ymask |= 1ull << ybit[k];
    // B (formatted in shared memory) = the operand holding fewer y bits: the y bits flip first
    if (__builtin_popcountll(cb & ymask) > __builtin_popcountll(ca & ymask)) {
      std::swap(ia, ib);
      std::swap(ca, cb);
    }
    // register-block and warp bits: output bits of the consumer (< R3) only
    // register blocks: 4 x 4 (TNB_FC_SHRINK=1: smaller when that leaves fewer consumer blocks than SMs)
    int rcap_a = 2, rcap_b = fc_rbb();
    while (rcap_a + rcap_b > 2 && R - (5 + WB + rcap_a + rcap_b) - M3 >= 0 &&
           (1ull << (R - (5 + WB + rcap_a + rcap_b) - M3)) < (uint64_t)num_sms() && fc_shrink()) {
      if (rcap_b >= rcap_a) --rcap_b; else --rcap_a;
    }
    int ra[2], rb[2], nra = 0, nrb = 0;
    for (int b = 5; b < R3; ++b) {
      if (((ca >> b) & 1) && nra < rcap_a) ra[nra++] = b;
      if (((cb >> b) & 1) && nrb < rcap_b) rb[nrb++] = b;
    }
    if (nra == 0 || nrb == 0) FC_DECLINE("no a / b register bits");
    uint64_t used = 31ull;
    for (int i = 0; i < nra; ++i) used |= 1ull << ra[i];
    for (int i = 0; i < nrb; ++i) used |= 1ull << rb[i];
    int wb[3], nw = 0;
    for (int pass = 0; pass < 2 && nw < WB; ++pass)
      for (int b = 5; b < R3 && nw < WB; ++b) {
        const uint64_t cls = pass == 0 ? (ca | cb) : cc;
        if (!((used >> b) & 1) && ((cls >> b) & 1)) { wb[nw++] = b; used |= 1ull << b; }
      }
    if (nw < WB) FC_DECLINE("warp bits");
    const GIn& A = g.in[ia];
    const GIn& Bq = g.in[ib];
    const int TB = 5 + WB + nra + nrb;
    if (R < TB + M3 || TB > kGemmMaxTB) FC_DECLINE("tile");
    MArgs ma;
    std::memset(&ma, 0, sizeof(ma));
    int u = 0;
    for (int b = 0; b < 5; ++b) ma.outbit[u++] = (uint8_t)b;
    for (int i = 0; i < WB; ++i) ma.outbit[u++] = (uint8_t)wb[i];
    for (int i = 0; i < nra; ++i) ma.outbit[u++] = (uint8_t)ra[i];
    for (int i = 0; i < nrb; ++i) ma.outbit[u++] = (uint8_t)rb[i];
    const uint64_t tmask = used;
    int nc = 0;
    for (int t = 0; t < g.n; ++t) {
      if (t == ia || t == ib) continue;
      if (g.in[t].out_mask & tmask) FC_DECLINE("constant holds a tile bit");
      if (g.in[t].rank > 32) FC_DECLINE("constant rank");
      ma.cin[nc] = g.in[t].ptr;
      ma.cmask[nc] = g.in[t].out_mask;
      ma.cpv[nc] = g.in[t].pv;
      for (int x = 0; x < (1 << g.M); ++x) ma.cgx[nc][x] = (uint32_t)g.in[t].gx[x];
      ++nc;
    }
    ma.nc = nc;
    ma.c_tile_dep = 0;
    for (int t = 0; t < nc; ++t) ma.c_tile_dep |= ma.cmask[t] != 0 ? 1 : 0;
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
    const uint32_t dep_u32 = (ma.nrows[0] << (ma.nch[0] - ma.lv[0])) + (ma.nrows[1] << (ma.nch[1] - ma.lv[1]));
    const size_t bf_bytes = ((size_t)16 << g.M) << ma.nch[1];
    int S = gemm_stages();
    const size_t budget = WB == 3 ? kFcSmemBudget : kFcSmemBudget / 2;   // 2 or 4 CTAs per SM
    while (S > 2 && ((size_t)S * (sz[0] + sz[1]) * 8 + dep_u32 * 4 + bf_bytes + 16) > budget) --S;
    ma.stages = S;
    for (int k = 0; k < S; ++k) {
      ma.sm_in[0][k] = k * sz[0];
      ma.sm_in[1][k] = S * sz[0] + k * sz[1];
    }
    uint32_t u32 = 2 * S * (sz[0] + sz[1]);
    for (int s = 0; s < 2; ++s) {
      ma.sm_dep[s] = u32;
      u32 += ma.nrows[s] << (ma.nch[s] - ma.lv[s]);
    }
    ma.sm_bf_bytes = (u32 * 4 + 15) / 16 * 16;
    const size_t smem = ma.sm_bf_bytes + bf_bytes;
    if (smem > budget) FC_DECLINE("smem");
    // traversal: the consumer's summed bits first (in the consumer's x order), then A-only bits
    // (B and B' unchanged), then B-only bits, then the rest
    // the y bits first, those held by A only before those B holds (B's chunk and B' then change
    // only when a B y bit flips); tile-index bit k is the consumer's summed bit yo[k], so the
    // consumer tables are re-indexed by the tile's low bits
    int yo[kMaxGroup], ny = 0;
    for (int pass = 0; pass < 3; ++pass)
      for (int k = 0; k < M3; ++k) {
        const int b = ybit[k];
        const int cls = ((cb >> b) & 1) ? 2 : ((cc >> b) & 1) ? 1 : 0;
        if (cls == pass) yo[ny++] = k;
      }
    if (ny != M3) FC_DECLINE("y order");
    {
      FArgs f2 = fa;
      for (int yp = 0; yp < (1 << M3); ++yp) {
        int x = 0;
        for (int k = 0; k < M3; ++k)
          if ((yp >> k) & 1) x |= 1 << yo[k];
        for (int v = 0; v < fa.nv; ++v) f2.vgx[v][yp] = fa.vgx[v][x];
        for (int w = 0; w < fa.nw; ++w) f2.wgx[w][yp] = fa.wgx[w][x];
      }
      fa = f2;
    }
    int np = 0;
    for (int k = 0; k < M3; ++k) ma.perm[np++] = (uint8_t)ybit[yo[k]];
    // TNB_FC_XFIRST=1: output bits the consumer factor X lacks right after the y bits, so the
    // consumer blocks reading the same X values run back to back -- measured worse on C5a (DRAM
    // 668 vs ~430 MB per launch: A's and B's chunks then change every block; 89.0 vs 90.4 /s), off
    static const bool xfirst = env_flag("TNB_FC_XFIRST");
    uint64_t xlack = 0;
    if (xfirst && fa.nv == 1)
      for (int b = 0; b < R3; ++b)
        if (!((fa.vmask[0] >> b) & 1) && !(((tmask | ymask) >> b) & 1)) xlack |= 1ull << b;
    for (int b = 0; b < R; ++b)
      if ((xlack >> b) & 1) ma.perm[np++] = (uint8_t)b;
    for (int pass = 0; pass < 3; ++pass)
      for (int b = 0; b < R; ++b) {
        if (((tmask | ymask | xlack) >> b) & 1) continue;
        const uint64_t cls = pass == 0 ? ca : pass == 1 ? cb : (cc | cn);
        if ((cls >> b) & 1) ma.perm[np++] = (uint8_t)b;
      }
    if (np != R - TB) FC_DECLINE("perm");
    ma.out = g.out;   // not written
    ma.out_rank = R;
    if (env_flag("TNB_GEMM_DEBUG"))
      std::fprintf(stderr, "k_gemm_fc R=%d M=%d R3=%d M3=%d TB=%d nra=%d nrb=%d nch=(%u,%u) S=%d smem=%zu nc=%d nv=%d nw=%d\n",
                   R, g.M, R3, M3, TB, nra, nrb, ma.nch[0], ma.nch[1], ma.stages, smem, nc, fa.nv, fa.nw);
    if (env_flag("TNB_GEMM_DEBUG")) { debug_group("producer", g); debug_group("consumer", g3); }
    const uint64_t groups = 1ull << (R - TB - M3);
    static const uint64_t min_groups = [] {   // TNB_FC_MIN_GROUPS: fewer consumer blocks -> two launches
      const char* e = std::getenv("TNB_FC_MIN_GROUPS");
      return e ? (uint64_t)std::atoll(e) : 0ull;
    }();
    if (groups < min_groups) FC_DECLINE("too few consumer blocks");
    const unsigned grid = (unsigned)std::min<uint64_t>(groups, (uint64_t)num_sms() * (fc_cps() ? fc_cps() : (WB == 3 ? 2 : 4)));
    // balanced tile ranges with consumer blocks split between neighbouring CTAs (C5a: 512 blocks on
    // 296 CTAs -- whole blocks left 40 CTAs idle and 108 SMs with 4 blocks against 3.46 on average)
    fa.sem = (sem && grid >= 2 && grid < (unsigned)kFcSemPerOp && (groups % grid) != 0) ? sem : nullptr;
    switch (g.M) {
      case 1: return WB == 3 ? dispatch_fc<1, 3>(ma, fa, nra, nrb, grid, smem, st) : dispatch_fc<1, 2>(ma, fa, nra, nrb, grid, smem, st);
      case 2: return WB == 3 ? dispatch_fc<2, 3>(ma, fa, nra, nrb, grid, smem, st) : dispatch_fc<2, 2>(ma, fa, nra, nrb, grid, smem, st);
      case 3: return WB == 3 ? dispatch_fc<3, 3>(ma, fa, nra, nrb, grid, smem, st) : dispatch_fc<3, 2>(ma, fa, nra, nrb, grid, smem, st);
      case 4: return WB == 3 ? dispatch_fc<4, 3>(ma, fa, nra, nrb, grid, smem, st) : dispatch_fc<4, 2>(ma, fa, nra, nrb, grid, smem, st);
      case 5: return WB == 3 ? dispatch_fc<5, 3>(ma, fa, nra, nrb, grid, smem, st) : dispatch_fc<5, 2>(ma, fa, nra, nrb, grid, smem, st);
      default: return false;
    }
  }
}

template bool try_launch_gemm_fc<float2>(const GDesc&, const GDesc&, int, cudaStream_t, uint32_t*);
template bool try_launch_gemm_fc_wb<float2>(const GDesc&, const GDesc&, int, cudaStream_t, int, uint32_t*);
template bool try_launch_gemm_fc_wb<double2>(const GDesc&, const GDesc&, int, cudaStream_t, int, uint32_t*);
template bool try_launch_gemm_fc<double2>(const GDesc&, const GDesc&, int, cudaStream_t, uint32_t*);

}  // namespace tnb
