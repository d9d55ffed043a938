// kernels_fctc.cuh -- k_fc_tc: a producer -> consumer pair of fused merge groups (OP_GROUP_FEED)
// with the producer's batched complex GEMM on the 5th-generation tensor cores (tcgen05.mma
// kind::tf32, 3xTF32 split, accumulators in TMEM) and the consumer's sum in the epilogue.
//
//   producer:  T[t] = sum_{x < 2^M} C1_x A[F_A(t) + G_A(x)] B[F_B(t) + G_B(x)]     (t = (o, y))
//   consumer:  out[o] = sum_{y < 2^M3} C3_y X[F_X(o, y)] T[o, y]
// Both are exact re-associations of consecutive bucket eliminations: the
// producer is a merge step plus the reduce steps after it, the consumer the bucket holding T.
// T is never written.
//
// Tiling (host: launch_fc_tc.cu).  T's bits are classified a (in A only), b (in B only), c (both).
// A UNIT is a 128 x 2^NB tile of T for fixed other bits:
//   rows  = 7 a-bits that are consumer output bits (the MMA's M = 128, one TMEM lane per row);
//   cols  = NB b-bits: the NOB low ones consumer output bits, the rest consumer summed bits (y);
//   real GEMM  D[r][2c + e] = sum_k' A'[r][k'] B'[2c + e][k'],  A' = (Re A, Im A) along k' = 2x + f,
//              B' = (Re C1B, -Im C1B ; Im C1B, Re C1B): D[r][2c] = Re T, D[r][2c + 1] = Im T.
// The remaining T bits are traversal bits: innermost NL "line" bits (output bits whose units share
// the 128-byte DRAM lines of X and A: run back to back, each with its own accumulator set), then
// the y bits not in cols (a BLOCK = the 2^(NL + nyt) units sharing one set of consumer outputs),
// then the block bits.  Each epilogue thread owns one row: it accumulates 2^(NL + NOB) consumer
// outputs in registers over the block's units (summing the y bits of its columns and of the
// traversal) and stores them once.
//
// Precision: every operand is split v = big + small (big = cvt.rna.tf32(v)); D = Ab Bb + Ab Bs +
// As Bb (3 MMAs per K step of 8), 7e-7 relative (scripts/probe/tc_probe.cu) vs 1e-4 parity.
//
// Warp roles (288 threads, one CTA per SM, persistent over a contiguous block range):
//   warps 0-3  epilogue: tcgen05.ld of its 32 TMEM lanes, X' = C3_y X from the X tile staged in
//              shared memory (column-major, conflict-free), out += X' T in registers;
//   warps 4-7  loaders: cp.async of the raw A / B / C1 chunks and of the X tile S - 1 units
//              ahead (the X copies arrive on x_full[slot] through cp.async.mbarrier.arrive),
//              then the TF32 split / B' block structure into the operand slot (unit & 1);
//   warp 8     MMA: one elected lane issues the 3 x KC tcgen05.mma of a unit into TMEM buffer
//              (unit & 1) and commits to mma_done[unit & 1].
#pragma once
#include <cuda.h>   // CUtensorMap (a 128-byte kernel parameter; no driver call in device code)
#define FT_TR(lu, ev)                                                                  \
  do {                                                                                 \
    if (a.trace && blockIdx.x == 0 && (lu) < 256u) a.trace[(lu) * 8u + (ev)] = clock64(); \
  } while (0)
#define TNB_TC_HELPERS_ONLY
#include "kernels_tc.cuh"
#undef TNB_TC_HELPERS_ONLY

namespace tnb {

constexpr int kFtRows = 7;                       // MMA M = 128
constexpr int kFtMaxTrav = 40;                   // traversal bits
constexpr int kFtEpi = 4, kFtLd = 4;
constexpr int kFtXw = 2;                         // X-tile loader warps
constexpr int kFtThreads = (kFtEpi + kFtLd + 2 + kFtXw) * 32;   // + the MMA warp, the producer warp, X loaders

struct FTArgs {
  const float2* A;
  const float2* B;
  const float2* X;
  float2* out;
  int32_t ntrav, nyt;                    // traversal bits: NL line bits, then nyt consumer y bits,
  uint64_t n_blocks;                     // then the block bits: 2^(ntrav - NL - nyt) blocks
  uint32_t arow[kFtRows], xrow[kFtRows], orow[kFtRows];   // offset of row bit i in A / X / out
  uint32_t bcol[8], xcol[8], ocol[8], ycol[8];            // col bit j: B / X / out / y-index
  uint32_t ta[kFtMaxTrav], tb[kFtMaxTrav], tx[kFtMaxTrav], to[kFtMaxTrav], ty[kFtMaxTrav];
  uint32_t tc[kMaxIn][kFtMaxTrav];       // producer constants (they hold no row / col bit)
  uint32_t gA[1 << kMaxGroup], gB[1 << kMaxGroup];        // G_A(x), G_B(x)
  const float2* cin[kMaxIn];
  uint32_t cgx[kMaxIn][1 << kMaxGroup];
  int32_t nc;
  const float2* win[kMaxIn];             // consumer weights: C3_y = prod_w win[w][wgx[w][y]]
  uint32_t wgx[kMaxIn][1 << kMaxGroup];
  int32_t nw, M3;
  int32_t apair, xpair;                  // row bit 0 has offset 1 in A / X: 16-byte copies
  // X tiles and raw A chunks by TMA (tensor maps tmX / tmA, 5-D boxes over the runs of unit bits in
  // each tensor's bit order): coordinate d of a unit = (base >> ts[t][d]) & tmsk[t][d] (+ the delta
  // of copy i when the unit bits form more than 5 runs); t = 0: X, 1: A
  int32_t tma;
  uint32_t ts[2][5], tmsk[2][5];
  int32_t ncopy[2];
  uint32_t cdelta[2][8][5];
  uint32_t copy_elems[2];
  // shared-memory element index of row bit i / col bit j in the X tile, of row bit i / summed value
  // x in the raw A chunk (the TMA box layout, or the cp.async layout [c][r] / [x][r])
  uint32_t xs_row[kFtRows], xs_col[8];
  uint32_t as_row[kFtRows], as_x[1 << kMaxGroup];
  unsigned long long* trace;
  // coalesced X pieces (16 bytes = a row pair): piece-index bit k adds xp_g[k] elements in X and
  // xp_s[k] in the tile; bits sorted by xp_g, the low 5 on the lanes, the high ones tabulated in
  // dynamic smem at sm_xp (2^(xp_bits - 5) pairs)
  int32_t xp_bits;
  uint32_t xp_g[24], xp_s[24];
  uint32_t sm_xp;             // TNB_FT_TRACE=1: clock64 of CTA 0's pipeline events [unit][8]
  int32_t SX, S;                         // ring slots of X group tiles / of per-unit raw chunks
  int32_t atma;                          // raw A chunks by TMA (tensor map tmA)
  uint32_t xs_line[4], as_line[4];       // smem index offset of line value li in the X tile / raw A chunk
  uint32_t tmem_cols;
  uint32_t sm_b, sm_raw, sm_x, sm_tab;   // dynamic smem byte offsets
};

__device__ __forceinline__ void ft_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc_smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void ft_tma5(void* dst, const CUtensorMap* map, const uint32_t* c, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::
          "r"(tc_smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]),
      "r"(c[4]), "r"(tc_smem_u32(bar))
      : "memory");
}

// traversal offsets of the streams (A, B, X, out, y, producer constants): offset(u) = sum over the
// set traversal bits j of u of tb[st][j]; consecutive units update incrementally (u -> u + 1 clears
// bits 0 .. r-1 and sets bit r, r = ctz(~u)): o += tb[r] - tc[r], tc[r] = sum_{j < r} tb[j]
enum : int { FT_A = 0, FT_B = 1, FT_X = 2, FT_O = 3, FT_Y = 4, FT_C = 5, FT_NS = 5 + kMaxIn };

template <int M, int NB, int NOB, int NL>
__global__ void __launch_bounds__(kFtThreads, 1) k_fc_tc(const FTArgs a, const __grid_constant__ CUtensorMap tmX,
                                                         const __grid_constant__ CUtensorMap tmA) {
  constexpr int K = 1 << M;                // complex summed values
  constexpr int KP = 2 * K;                // real K (floats per operand row)
  constexpr int KC = KP / 8;               // tf32 MMA K steps
  constexpr int NCOL = 1 << NB;            // complex columns
  constexpr int N = 2 * NCOL;              // real columns (MMA N)
  constexpr uint32_t SBO = (KP / 4) * 128; // bytes between 8-row groups (K-major, no swizzle)
  constexpr uint32_t A_PART = 128 * KP * 4, B_PART = N * KP * 4;   // one TF32 part (big or small)
  constexpr uint32_t A_RAW = 128 * K * 8, B_RAW = NCOL * K * 8, X_TILE = 128 * NCOL * 8;
  constexpr int NACC = 1 << NOB;
  constexpr int kL = kFtLd * 32;
  static_assert(M >= 2 && KP % 8 == 0, "K must fill a tf32 MMA step");
  static_assert(NOB >= 3 && NOB <= NB && NB <= 6, "column shape");
  extern __shared__ __align__(128) unsigned char dsm_ft[];
  __shared__ uint64_t op_full[2], mma_done[2], tmem_empty[2];
  __shared__ uint64_t x_full[4], x_empty[4], raw_full[4], raw_empty[4];
  __shared__ uint32_t tmem_base_sh;
  __shared__ float2 C3s[1 << kMaxGroup];
  __shared__ uint32_t tfb[FT_NS][kFtMaxTrav], tfc[FT_NS][kFtMaxTrav + 1];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int SX = a.SX, S = a.S;
  constexpr int NLS = 1 << NL;             // units of a line group (share their X tile and raw chunks)
  const int nst = FT_C + a.nc;
  // per-row / per-column tables
  uint32_t* t_arow = reinterpret_cast<uint32_t*>(dsm_ft + a.sm_tab);   // A offset of row r (cp.async path)
  uint32_t* t_xrow = t_arow + 128;                                       // X offset of row r (cp.async path)
  uint32_t* t_bcol = t_xrow + 128;                                       // B offset of column c
  uint32_t* t_xcol = t_bcol + NCOL;                                      // X offset of column c (cp.async path)
  uint32_t* t_xsrow = t_xcol + NCOL;                                     // smem index of row r in the X tile
  uint32_t* t_asrow = t_xsrow + 128;                                     // ... in the raw A chunk
  for (int r = tid; r < 128; r += kFtThreads) {
    uint32_t oa = 0, ox = 0, sx = 0, sa = 0;
    for (int i = 0; i < kFtRows; ++i)
      if ((r >> i) & 1) { oa += a.arow[i]; ox += a.xrow[i]; sx += a.xs_row[i]; sa += a.as_row[i]; }
    t_arow[r] = oa;
    t_xrow[r] = ox;
    t_xsrow[r] = sx;
    t_asrow[r] = sa;
  }
  for (int c = tid; c < NCOL; c += kFtThreads) {
    uint32_t ob = 0, ox = 0;
    for (int j = 0; j < NB; ++j)
      if ((c >> j) & 1) { ob += a.bcol[j]; ox += a.xcol[j]; }
    t_bcol[c] = ob;
    t_xcol[c] = ox;
  }
  if (a.xp_bits >= 5) {
    uint32_t* hi = reinterpret_cast<uint32_t*>(dsm_ft + a.sm_xp);
    for (int k = tid; k < (1 << (a.xp_bits - 5)); k += kFtThreads) {
      uint32_t go = 0, so = 0;
      for (int b = 5; b < a.xp_bits; ++b)
        if ((k >> (b - 5)) & 1) { go += a.xp_g[b]; so += a.xp_s[b]; }
      hi[2 * k] = go;
      hi[2 * k + 1] = so;
    }
  }
  for (int i = tid; i < nst * kFtMaxTrav; i += kFtThreads) {
    const int st = i / kFtMaxTrav, j = i % kFtMaxTrav;
    uint32_t v = 0;
    if (j < a.ntrav)
      v = st == FT_A ? a.ta[j] : st == FT_B ? a.tb[j] : st == FT_X ? a.tx[j] : st == FT_O ? a.to[j]
        : st == FT_Y ? a.ty[j] : a.tc[st - FT_C][j];
    tfb[st][j] = v;
  }
  if (tid < (1 << a.M3)) {
    float2 w = make_float2(1.f, 0.f);
    for (int q = 0; q < a.nw; ++q) w = cmul(w, __ldg(a.win[q] + a.wgx[q][tid]));
    C3s[tid] = w;
  }
  if (tid == 0) {
    for (int s = 0; s < 2; ++s) {
      tc_mbar_init(&op_full[s], kFtLd * 32);
      tc_mbar_init(&mma_done[s], 1);
      tc_mbar_init(&tmem_empty[s], kFtEpi);
    }
    for (int s = 0; s < 4; ++s) {
      // X tile: the producer's TMA expect_tx (1 arrival) or its 32 lanes' cp.async arrivals
      tc_mbar_init(&x_full[s], a.tma ? 1 : 32 * kFtXw);
      tc_mbar_init(&x_empty[s], kFtEpi);
      // raw A / B / C chunk: 32 cp.async arrivals of the producer lanes (+ 1 expect_tx for TMA A)
      tc_mbar_init(&raw_full[s], a.atma ? 33 : 32);
      tc_mbar_init(&raw_empty[s], kFtLd);
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc_smem_u32(&tmem_base_sh)),
                 "r"(a.tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid < nst) {
    uint32_t c = 0;
    for (int j = 0; j <= kFtMaxTrav; ++j) {
      tfc[tid][j] = c;
      if (j < kFtMaxTrav) c += tfb[tid][j];
    }
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base_sh;
  auto trav_at = [&](int st, uint64_t u) {
    uint32_t o = 0;
    for (int j = 0; j < a.ntrav && (u >> j); ++j)
      if ((u >> j) & 1) o += tfb[st][j];
    return o;
  };
  auto trav_step = [&](int st, uint32_t& o, uint64_t u) {   // offset at u -> offset at u + 1
    const int r = __ffsll((long long)~u) - 1;
    o += tfb[st][r] - tfc[st][r];
  };

  // this CTA's blocks [b0, b1) and units [b0 << (NL + nyt), b1 << (NL + nyt))
  const uint64_t b0 = (uint64_t)blockIdx.x * a.n_blocks / gridDim.x;
  const uint64_t b1 = ((uint64_t)blockIdx.x + 1) * a.n_blocks / gridDim.x;
  const uint64_t u0 = b0 << (NL + a.nyt);
  const uint32_t nU = (uint32_t)((b1 - b0) << (NL + a.nyt));

  if (warp == kFtEpi + kFtLd) {
    // ================================ MMA warp
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint64_t dhi = ((uint64_t)((SBO >> 4) & 0x3FFFu) << 32) | (1ull << 46) | ((uint64_t)(128u >> 4) << 16);
    const uint32_t sA0 = tc_smem_u32(dsm_ft), sB0 = tc_smem_u32(dsm_ft + a.sm_b);
    for (uint32_t lu = 0; lu < nU; ++lu) {
      const uint32_t s = lu & 1u;
      tc_mbar_wait(&op_full[s], (lu >> 1) & 1u);
      if (lu >= 2) tc_mbar_wait(&tmem_empty[s], ((lu - 2) >> 1) & 1u);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (lane == 0) FT_TR(lu, 2);
      if (lane == 0) {
        const uint32_t aS = sA0 + s * 2 * A_PART, bS = sB0 + s * 2 * B_PART;
        const uint32_t dcol = tmem + s * N;
#pragma unroll
        for (int kc = 0; kc < KC; ++kc)
#pragma unroll
          for (int pr = 0; pr < 3; ++pr) {
            const uint32_t ao = aS + (pr == 2 ? A_PART : 0u) + kc * 256u;
            const uint32_t bo = bS + (pr == 1 ? B_PART : 0u) + kc * 256u;
            umma_tf32(dcol, dhi | ((ao >> 4) & 0x3FFFu), dhi | ((bo >> 4) & 0x3FFFu), idesc, (kc | pr) ? 1u : 0u);
          }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         tc_smem_u32(&mma_done[s]))
                     : "memory");
      }
      __syncwarp();
    }
  } else if (warp >= kFtEpi + kFtLd + 2) {
    // ================================ X loader warps: the X tile of each line group (the 2^NL
    // units sharing X's and A's DRAM lines) into X slot g % SX once the epilogue released it --
    // coalesced 16-byte cp.async pieces in the [line][column][row] layout (the epilogue's reads are
    // then conflict-free) split over the loader warps, or TMA boxes issued by the first one
    const int xw = warp - (kFtEpi + kFtLd + 2);
    uint32_t ts0[5], tm0[5];
#pragma unroll
    for (int d = 0; d < 5; ++d) { ts0[d] = a.ts[0][d]; tm0[d] = a.tmsk[0][d]; }
    const int ncx = a.ncopy[0];
    const uint32_t cex = a.copy_elems[0];
    uint32_t lX[NLS];
#pragma unroll
    for (int li = 0; li < NLS; ++li) lX[li] = trav_at(FT_X, (uint64_t)li);
    uint32_t xp_g = 0, xp_s = 0;       // this lane's X piece: global / smem offsets of the low 5 piece bits
#pragma unroll
    for (int b = 0; b < 5; ++b)
      if ((lane >> b) & 1) { xp_g += a.xp_g[b]; xp_s += a.xp_s[b]; }
    const uint32_t nG = nU >> NL;
    for (uint32_t g = 0; g < nG; ++g) {
      const uint64_t u = u0 + ((uint64_t)g << NL);
      const uint32_t iX = trav_at(FT_X, u);
      const int xsl = (int)(g % (uint32_t)SX);
      float2* xs = reinterpret_cast<float2*>(dsm_ft + a.sm_x + (uint32_t)xsl * X_TILE * NLS);
      if (g >= (uint32_t)SX) tc_mbar_wait(&x_empty[xsl], ((g / SX) - 1) & 1u);
      if (a.tma) {
        if (xw == 0 && lane == 0) {
          uint32_t c[5];
          ft_expect_tx(&x_full[xsl], (uint32_t)ncx * cex * 8u);
          for (int i = 0; i < ncx; ++i) {
#pragma unroll
            for (int d = 0; d < 5; ++d) c[d] = ((iX >> ts0[d]) & tm0[d]) + a.cdelta[0][i][d];
            ft_tma5(xs + (size_t)i * cex, &tmX, c, &x_full[xsl]);
          }
        }
      } else {
        if (a.xp_bits >= 5) {
          const uint32_t* hi = reinterpret_cast<const uint32_t*>(dsm_ft + a.sm_xp);
          for (int k = xw; k < (1 << (a.xp_bits - 5)); k += kFtXw)
            cp_async16(xs + xp_s + hi[2 * k + 1], a.X + iX + xp_g + hi[2 * k]);
        } else {
#pragma unroll
          for (int li = 0; li < NLS; ++li) {
            float2* xl = xs + li * (X_TILE / 8);
            for (int p = lane + 32 * xw; p < 128 * NCOL; p += 32 * kFtXw) {
              const int r = p & 127, c = p >> 7;
              cp_async8(xl + c * 128 + r, a.X + iX + lX[li] + t_xrow[r] + t_xcol[c]);
            }
          }
        }
        mbar_cp_async_arrive(&x_full[xsl]);
      }
      if (lane == 0 && xw == 0) FT_TR(g, 5);
    }
    cp_async_wait<0>();
  } else if (warp == kFtEpi + kFtLd + 1) {
    // ================================ producer warp.  Per line group (the 2^NL units sharing X's
    // and A's DRAM lines): the X tile into X slot g % SX (coalesced 16-byte cp.async pieces in the
    // [line][column][row] layout, or TMA boxes).  Per unit v: the raw A chunk (TMA box or cp.async),
    // B chunk and producer constants into raw slot v % S.
    unsigned char* raw = dsm_ft + a.sm_raw;
    const uint32_t raw_slot = (A_RAW + B_RAW + (uint32_t)(kMaxIn * K * 8) + 127u) & ~127u;
    uint32_t ts0[5], tm0[5], ts1[5], tm1[5];
#pragma unroll
    for (int d = 0; d < 5; ++d) { ts0[d] = a.ts[0][d]; tm0[d] = a.tmsk[0][d]; ts1[d] = a.ts[1][d]; tm1[d] = a.tmsk[1][d]; }
    const int ncx = a.ncopy[0], nca = a.ncopy[1];
    const uint32_t cex = a.copy_elems[0], cea = a.copy_elems[1];
    uint32_t lX[NLS];
#pragma unroll
    for (int li = 0; li < NLS; ++li) lX[li] = trav_at(FT_X, (uint64_t)li);
    uint32_t xp_g = 0, xp_s = 0;       // this lane's X piece: global / smem offsets of the low 5 piece bits
#pragma unroll
    for (int b = 0; b < 5; ++b)
      if ((lane >> b) & 1) { xp_g += a.xp_g[b]; xp_s += a.xp_s[b]; }
    constexpr int NBP = (NCOL * K + 31) / 32;
    uint32_t boff[NBP];
#pragma unroll
    for (int k = 0; k < NBP; ++k) {
      const int p = lane + 32 * k;
      boff[k] = p < NCOL * K ? t_bcol[p & (NCOL - 1)] + a.gB[p >> NB] : 0u;
    }
    const bool has_c = lane < a.nc * K;
    const int cq = has_c ? (lane >> M) : 0;
    const float2* cptr = has_c ? a.cin[cq] + a.cgx[cq][lane & (K - 1)] : nullptr;
    uint32_t iA = 0, iB = 0, iX = 0, iC = 0;
    if (nU > 0) {
      iA = trav_at(FT_A, u0);
      iB = trav_at(FT_B, u0);
      iX = trav_at(FT_X, u0);
      iC = has_c ? trav_at(FT_C + cq, u0) : 0u;
    }
    for (uint32_t v = 0; v < nU; ++v) {
      const uint64_t u = u0 + v;
      const int sl = (int)(v % (uint32_t)S);
      float2* ra = reinterpret_cast<float2*>(raw + sl * raw_slot);
      float2* rb = reinterpret_cast<float2*>(raw + sl * raw_slot + A_RAW);
      float2* rc = reinterpret_cast<float2*>(raw + sl * raw_slot + A_RAW + B_RAW);
      if (v >= (uint32_t)S) tc_mbar_wait(&raw_empty[sl], ((v / S) - 1) & 1u);
      if (lane == 0) FT_TR(v, 0);
      if (a.atma) {
        if (lane == 0) {
          uint32_t c[5];
          ft_expect_tx(&raw_full[sl], (uint32_t)nca * cea * 8u);
          for (int i = 0; i < nca; ++i) {
#pragma unroll
            for (int d = 0; d < 5; ++d) c[d] = ((iA >> ts1[d]) & tm1[d]) + a.cdelta[1][i][d];
            ft_tma5(ra + (size_t)i * cea, &tmA, c, &raw_full[sl]);
          }
        }
      } else if (a.apair) {
        for (int p = lane; p < 64 * K; p += 32) {
          const int i = p & 63, x = p >> 6;
          cp_async16(ra + x * 128 + 2 * i, a.A + iA + t_arow[2 * i] + a.gA[x]);
        }
      } else {
        for (int p = lane; p < 128 * K; p += 32) {
          const int r = p & 127, x = p >> 7;
          cp_async8(ra + x * 128 + r, a.A + iA + t_arow[r] + a.gA[x]);
        }
      }
#pragma unroll
      for (int k = 0; k < NBP; ++k) {
        const int p = lane + 32 * k;
        if (p < NCOL * K) cp_async8(rb + p, a.B + iB + boff[k]);
      }
      if (has_c) cp_async8(rc + lane, cptr + iC);
      mbar_cp_async_arrive(&raw_full[sl]);
      if (v + 1 < nU) {
        trav_step(FT_A, iA, u);
        trav_step(FT_B, iB, u);
        trav_step(FT_X, iX, u);
        if (has_c) trav_step(FT_C + cq, iC, u);
      }
    }
    cp_async_wait<0>();
  } else if (warp >= kFtEpi) {
    // ================================ formatters (thread lt: row lt of the A chunk): TF32 split of
    // A and of C1-scaled B from the raw slot into the operand slot (unit & 1)
    const int lt = tid - kFtEpi * 32;
    unsigned char* raw = dsm_ft + a.sm_raw;
    const uint32_t raw_slot = (A_RAW + B_RAW + (uint32_t)(kMaxIn * K * 8) + 127u) & ~127u;
    const uint32_t my_asrow = t_asrow[lt];
    const uint32_t my_aoff = (uint32_t)(lt >> 3) * SBO + (uint32_t)(lt & 7) * 16u;
    constexpr int NBE = (NCOL * K + kL - 1) / kL;     // B elements per thread
    for (uint32_t lu = 0; lu < nU; ++lu) {
      const uint32_t s = lu & 1u;
      const int sl = (int)(lu % (uint32_t)S);
      tc_mbar_wait(&raw_full[sl], (lu / (uint32_t)S) & 1u);           // the raw chunks landed
      if (lt == 0) FT_TR(lu, 6);
      const float2* ra = reinterpret_cast<const float2*>(raw + sl * raw_slot);
      const float2* rb = reinterpret_cast<const float2*>(raw + sl * raw_slot + A_RAW);
      const float2* rc = reinterpret_cast<const float2*>(raw + sl * raw_slot + A_RAW + B_RAW);
      float2 ac[K], bc[NBE];
#pragma unroll
      for (int x = 0; x < K; ++x) ac[x] = ra[my_asrow + a.as_x[x]];
#pragma unroll
      for (int i = 0; i < NBE; ++i) {
        const int e = lt + kL * i;
        if (e < NCOL * K) {
          const int x = e >> NB;
          float2 v = rb[e];
          for (int q = 0; q < a.nc; ++q) v = cmul(v, rc[q * K + x]);
          bc[i] = v;
        }
      }
      __syncwarp();
      if (lane == 0) tc_mbar_arrive(&raw_empty[sl]);
      if (lu >= 2) tc_mbar_wait(&mma_done[s], ((lu - 2) >> 1) & 1u);   // operand slot s is free
      unsigned char* Ab = dsm_ft + s * 2 * A_PART;
      unsigned char* Bb = dsm_ft + a.sm_b + s * 2 * B_PART;
#pragma unroll
      for (int x = 0; x < K; x += 2) {     // 16-byte stores: summed values x, x + 1 of row lt
        float b0, s0, b1, s1, b2, s2, b3, s3;
        tf32_split(ac[x].x, b0, s0);
        tf32_split(ac[x].y, b1, s1);
        tf32_split(ac[x + 1].x, b2, s2);
        tf32_split(ac[x + 1].y, b3, s3);
        const uint32_t off = my_aoff + (uint32_t)(x >> 1) * 128u;
        *reinterpret_cast<float4*>(Ab + off) = make_float4(b0, b1, b2, b3);
        *reinterpret_cast<float4*>(Ab + A_PART + off) = make_float4(s0, s1, s2, s3);
      }
#pragma unroll
      for (int i = 0; i < NBE; ++i) {
        const int e = lt + kL * i;
        if (e < NCOL * K) {
          const int c = e & (NCOL - 1), x = e >> NB;
          float rbg, rsm, ibg, ism;
          tf32_split(bc[i].x, rbg, rsm);
          tf32_split(bc[i].y, ibg, ism);
          const uint32_t n = 2u * (uint32_t)c;
          const uint32_t off = (n >> 3) * SBO + (n & 7u) * 16u + (uint32_t)(x >> 1) * 128u + (uint32_t)(x & 1) * 8u;
          *reinterpret_cast<float2*>(Bb + off) = make_float2(rbg, -ibg);
          *reinterpret_cast<float2*>(Bb + off + 16) = make_float2(ibg, rbg);
          *reinterpret_cast<float2*>(Bb + B_PART + off) = make_float2(rsm, -ism);
          *reinterpret_cast<float2*>(Bb + B_PART + off + 16) = make_float2(ism, rsm);
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tc_mbar_arrive(&op_full[s]);
      if (lt == 0) FT_TR(lu, 1);
    }
  } else {
    // ================================ epilogue: thread = row r (TMEM lane)
    const int q = warp;
    const uint32_t r = (uint32_t)(32 * q + lane);
    uint32_t orow = 0;
#pragma unroll
    for (int i = 0; i < kFtRows; ++i)
      if ((r >> i) & 1u) orow += a.orow[i];
    uint32_t ocol[NACC];
#pragma unroll
    for (int c = 0; c < NACC; ++c) {
      uint32_t o = 0;
#pragma unroll
      for (int j = 0; j < NOB; ++j)
        if ((c >> j) & 1) o += a.ocol[j];
      ocol[c] = o;
    }
    // smem index of the 8 columns of chunk ch in the X tile: column part (compile-time unrolled)
    auto xcol_idx = [&](int c) {
      uint32_t ci = 0;
#pragma unroll
      for (int b = 0; b < NB; ++b)
        if ((c >> b) & 1) ci += a.xs_col[b];
      return ci;
    };
    const uint32_t my_xsrow = t_xsrow[r];
    // NL line bits are the lowest traversal bits (the 2^NL units sharing DRAM lines of X and A run
    // back to back): one accumulator set each, selected at compile time by unrolling over them
    float2 acc[NLS][NACC];
    const uint32_t bmask = (1u << (NL + a.nyt)) - 1u;   // units of a block (line bits + y bits)
    uint32_t oY = nU ? trav_at(FT_Y, u0) : 0u, oO = nU ? trav_at(FT_O, u0) : 0u;
    for (uint32_t lg = 0; lg < nU; lg += NLS) {
#pragma unroll
      for (int li = 0; li < NLS; ++li) {
        const uint32_t lu = lg + li;
        const uint32_t s = lu & 1u;
        const uint32_t g = lu >> NL;
        const int xsl = (int)(g % (uint32_t)SX);
        const uint64_t u = u0 + lu;
        const uint32_t yt = (uint32_t)u & bmask;
        if (yt < (uint32_t)NLS) {                      // first units of a block
#pragma unroll
          for (int c = 0; c < NACC; ++c) acc[li][c] = make_float2(0.f, 0.f);
        }
        if (r == 0) FT_TR(lu, 7);
        if (li == 0) tc_mbar_wait(&x_full[xsl], (g / (uint32_t)SX) & 1u);
        tc_mbar_wait(&mma_done[s], (lu >> 1) & 1u);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (r == 0) FT_TR(lu, 3);
        const float2* xs = reinterpret_cast<const float2*>(dsm_ft + a.sm_x + (uint32_t)xsl * X_TILE * NLS) + my_xsrow +
                           a.xs_line[li];
        const uint32_t tb = tmem + ((uint32_t)(32 * q) << 16) + s * N;
#pragma unroll
        for (int ch = 0; ch < NCOL / 8; ++ch) {             // 8 complex columns = 16 TMEM columns
          uint32_t v[16];
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
              : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
              : "r"(tb + 16u * ch));
          // the y index of these 8 columns (their low 3 bits are output bits: NOB >= 3)
          uint32_t yc = 0;
#pragma unroll
          for (int j = NOB; j < NB; ++j)
            if (((ch * 8) >> j) & 1) yc += a.ycol[j];
          const float2 w = C3s[oY + yc];
          float2 xv[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) xv[j] = xs[xcol_idx(ch * 8 + j)];
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int c = (ch * 8 + j) & (NACC - 1);
            const float2 t = make_float2(__uint_as_float(v[2 * j]), __uint_as_float(v[2 * j + 1]));
            const float2 wx = cmul(w, xv[j]);
            acc[li][c].x = fmaf(t.x, wx.x, fmaf(-t.y, wx.y, acc[li][c].x));
            acc[li][c].y = fmaf(t.x, wx.y, fmaf(t.y, wx.x, acc[li][c].y));
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          tc_mbar_arrive(&tmem_empty[s]);
          if (li == NLS - 1) tc_mbar_arrive(&x_empty[xsl]);
        }
        if (r == 0) FT_TR(lu, 4);
        if (yt + NLS > bmask) {                        // last units of a block: outputs final
          float2* o = a.out + oO + orow;
#pragma unroll
          for (int c = 0; c < NACC; ++c) __stcs(o + ocol[c], acc[li][c]);
        }
        if (lu + 1 < nU) {
          trav_step(FT_Y, oY, u);
          trav_step(FT_O, oO, u);
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(a.tmem_cols));
}

}  // namespace tnb
