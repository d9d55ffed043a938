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
// The remaining T bits are traversal bits: the y bits not in cols run innermost (a BLOCK = the
// 2^nyt units sharing one set of consumer outputs), then the block bits.  Each epilogue thread
// owns one row: it accumulates 2^NOB consumer outputs in registers over the block's units
// (summing the y bits of its columns and of the traversal) and stores them once.
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
#define TNB_TC_HELPERS_ONLY
#include "kernels_tc.cuh"
#undef TNB_TC_HELPERS_ONLY

namespace tnb {

constexpr int kFtRows = 7;                       // MMA M = 128
constexpr int kFtMaxTrav = 40;                   // traversal bits
constexpr int kFtEpi = 4, kFtLd = 4;
constexpr int kFtThreads = (kFtEpi + kFtLd + 1) * 32;

struct FTArgs {
  const float2* A;
  const float2* B;
  const float2* X;
  float2* out;
  int32_t ntrav, nyt;                    // traversal bits (the low nyt are consumer y bits)
  uint64_t n_blocks;                     // 2^(ntrav - nyt)
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
  int32_t S;                             // ring slots (raw chunks and X tiles), lookahead S - 1
  uint32_t tmem_cols;
  uint32_t sm_b, sm_raw, sm_x, sm_tab;   // dynamic smem byte offsets
};

__device__ __forceinline__ uint32_t ft_trav(const uint32_t* t, uint64_t u, int n) {
  uint32_t o = 0;
  for (int j = 0; j < n && (u >> j); ++j)
    if ((u >> j) & 1) o += t[j];
  return o;
}

template <int M, int NB, int NOB>
__global__ void __launch_bounds__(kFtThreads, 1) k_fc_tc(const FTArgs a) {
  constexpr int K = 1 << M;                // complex summed values
  constexpr int KP = 2 * K;                // real K (floats per operand row)
  constexpr int KC = KP / 8;               // tf32 MMA K steps
  constexpr int NCOL = 1 << NB;            // complex columns
  constexpr int N = 2 * NCOL;              // real columns (MMA N)
  constexpr uint32_t SBO = (KP / 4) * 128; // bytes between 8-row groups (K-major, no swizzle)
  constexpr uint32_t A_PART = 128 * KP * 4, B_PART = N * KP * 4;   // one TF32 part (big or small)
  constexpr uint32_t A_RAW = 128 * K * 8, B_RAW = NCOL * K * 8, X_TILE = 128 * NCOL * 8;
  constexpr int NACC = 1 << NOB;
  static_assert(M >= 2 && KP % 8 == 0, "K must fill a tf32 MMA step");
  static_assert(NOB >= 3 && NOB <= NB && NB <= 6, "column shape");
  extern __shared__ __align__(128) unsigned char dsm_ft[];
  __shared__ uint64_t op_full[2], mma_done[2], tmem_empty[2];
  __shared__ uint64_t x_full[4], x_empty[4];
  __shared__ uint32_t tmem_base_sh;
  __shared__ float2 C3s[1 << kMaxGroup];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int S = a.S, D = S - 1;
  // tables: A / X offset of row r, B / X / out offset of col c, y index of col chunk
  uint32_t* t_arow = reinterpret_cast<uint32_t*>(dsm_ft + a.sm_tab);
  uint32_t* t_xrow = t_arow + 128;
  uint32_t* t_bcol = t_xrow + 128;
  uint32_t* t_xcol = t_bcol + NCOL;
  for (int r = tid; r < 128; r += kFtThreads) {
    uint32_t oa = 0, ox = 0;
    for (int i = 0; i < kFtRows; ++i)
      if ((r >> i) & 1) { oa += a.arow[i]; ox += a.xrow[i]; }
    t_arow[r] = oa;
    t_xrow[r] = ox;
  }
  for (int c = tid; c < NCOL; c += kFtThreads) {
    uint32_t ob = 0, ox = 0;
    for (int j = 0; j < NB; ++j)
      if ((c >> j) & 1) { ob += a.bcol[j]; ox += a.xcol[j]; }
    t_bcol[c] = ob;
    t_xcol[c] = ox;
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
      tc_mbar_init(&x_full[s], kFtLd * 32);
      tc_mbar_init(&x_empty[s], kFtEpi);
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
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base_sh;

  // this CTA's blocks [b0, b1) and units [b0 << nyt, b1 << nyt)
  const uint64_t b0 = (uint64_t)blockIdx.x * a.n_blocks / gridDim.x;
  const uint64_t b1 = ((uint64_t)blockIdx.x + 1) * a.n_blocks / gridDim.x;
  const uint64_t u0 = b0 << a.nyt;
  const uint32_t nU = (uint32_t)((b1 - b0) << a.nyt);
  const uint32_t ymask = (1u << a.nyt) - 1u;

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
  } else if (warp >= kFtEpi) {
    // ================================ loaders
    const int lt = tid - kFtEpi * 32;
    constexpr int kL = kFtLd * 32;
    unsigned char* raw = dsm_ft + a.sm_raw;                  // S slots of [A raw | B raw | C raw]
    const uint32_t raw_slot = A_RAW + B_RAW + (uint32_t)(a.nc * K * 8);
    auto issue = [&](uint32_t v) {                            // unit v's chunks into ring slot v % S
      const uint64_t u = u0 + v;
      const int sl = (int)(v % (uint32_t)S);
      const uint32_t abase = ft_trav(a.ta, u, a.ntrav), bbase = ft_trav(a.tb, u, a.ntrav);
      const uint32_t xbase = ft_trav(a.tx, u, a.ntrav);
      float2* ra = reinterpret_cast<float2*>(raw + sl * raw_slot);
      float2* rb = reinterpret_cast<float2*>(raw + sl * raw_slot + A_RAW);
      float2* rc = reinterpret_cast<float2*>(raw + sl * raw_slot + A_RAW + B_RAW);
      if (v >= (uint32_t)S) tc_mbar_wait(&x_empty[sl], ((v / S) - 1) & 1u);   // the epilogue freed the X slot
      float2* xs = reinterpret_cast<float2*>(dsm_ft + a.sm_x + (uint32_t)sl * X_TILE);
      if (a.xpair) {
        for (int p = lt; p < 64 * NCOL; p += kL) {            // rows (2i, 2i + 1) of column c
          const int i = p & 63, c = p >> 6;
          cp_async16(xs + c * 128 + 2 * i, a.X + xbase + t_xrow[2 * i] + t_xcol[c]);
        }
      } else {
        for (int p = lt; p < 128 * NCOL; p += kL) {
          const int r = p & 127, c = p >> 7;
          cp_async8(xs + c * 128 + r, a.X + xbase + t_xrow[r] + t_xcol[c]);
        }
      }
      mbar_cp_async_arrive(&x_full[sl]);
      if (a.apair) {
        for (int p = lt; p < 64 * K; p += kL) {
          const int i = p & 63, x = p >> 6;
          cp_async16(ra + x * 128 + 2 * i, a.A + abase + t_arow[2 * i] + a.gA[x]);
        }
      } else {
        for (int p = lt; p < 128 * K; p += kL) {
          const int r = p & 127, x = p >> 7;
          cp_async8(ra + x * 128 + r, a.A + abase + t_arow[r] + a.gA[x]);
        }
      }
      for (int p = lt; p < NCOL * K; p += kL) {
        const int c = p & (NCOL - 1), x = p >> NB;
        cp_async8(rb + x * NCOL + c, a.B + bbase + t_bcol[c] + a.gB[x]);
      }
      for (int p = lt; p < a.nc * K; p += kL) {
        const int q = p >> M, x = p & (K - 1);
        cp_async8(rc + p, a.cin[q] + ft_trav(a.tc[q], u, a.ntrav) + a.cgx[q][x]);
      }
    };
    for (int v = 0; v < D; ++v) {
      if ((uint32_t)v < nU) issue((uint32_t)v);
      cp_async_commit();
    }
    for (uint32_t lu = 0; lu < nU; ++lu) {
      const uint32_t s = lu & 1u;
      const int sl = (int)(lu % (uint32_t)S);
      // groups committed: D + lu; unit lu's is complete when at most D - 1 are pending
      if (D <= 1) cp_async_wait<0>(); else if (D == 2) cp_async_wait<1>(); else cp_async_wait<2>();
      tc_named_bar(1, kL);
      if (lu >= 2) tc_mbar_wait(&mma_done[s], ((lu - 2) >> 1) & 1u);   // operand slot s is free
      const float2* ra = reinterpret_cast<const float2*>(raw + sl * raw_slot);
      const float2* rb = reinterpret_cast<const float2*>(raw + sl * raw_slot + A_RAW);
      const float2* rc = reinterpret_cast<const float2*>(raw + sl * raw_slot + A_RAW + B_RAW);
      unsigned char* Ab = dsm_ft + s * 2 * A_PART;
      unsigned char* Bb = dsm_ft + a.sm_b + s * 2 * B_PART;
      for (int e = lt; e < 128 * K; e += kL) {
        const int r = e & 127, x = e >> 7;
        const float2 v = ra[x * 128 + r];
        float rbg, rsm, ibg, ism;
        tf32_split(v.x, rbg, rsm);
        tf32_split(v.y, ibg, ism);
        const uint32_t off = (uint32_t)(r >> 3) * SBO + (uint32_t)(r & 7) * 16u + (uint32_t)(x >> 1) * 128u +
                             (uint32_t)(x & 1) * 8u;
        *reinterpret_cast<float2*>(Ab + off) = make_float2(rbg, ibg);
        *reinterpret_cast<float2*>(Ab + A_PART + off) = make_float2(rsm, ism);
      }
      for (int e = lt; e < NCOL * K; e += kL) {
        const int c = e & (NCOL - 1), x = e >> NB;
        float2 v = rb[x * NCOL + c];
        for (int q = 0; q < a.nc; ++q) v = cmul(v, rc[q * K + x]);
        float rbg, rsm, ibg, ism;
        tf32_split(v.x, rbg, rsm);
        tf32_split(v.y, ibg, ism);
        const uint32_t n = 2u * (uint32_t)c;
        const uint32_t off = (n >> 3) * SBO + (n & 7u) * 16u + (uint32_t)(x >> 1) * 128u + (uint32_t)(x & 1) * 8u;
        *reinterpret_cast<float2*>(Bb + off) = make_float2(rbg, -ibg);
        *reinterpret_cast<float2*>(Bb + off + 16) = make_float2(ibg, rbg);
        *reinterpret_cast<float2*>(Bb + B_PART + off) = make_float2(rsm, -ism);
        *reinterpret_cast<float2*>(Bb + B_PART + off + 16) = make_float2(ism, rsm);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tc_mbar_arrive(&op_full[s]);
      // raw slot (lu + D) % S = (lu - 1) % S: every loader finished formatting unit lu - 1 before
      // the barrier above
      if (lu + D < nU) issue(lu + D);
      cp_async_commit();
    }
    cp_async_wait<0>();
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
    float2 acc[NACC];
    for (uint32_t lu = 0; lu < nU; ++lu) {
      const uint32_t s = lu & 1u;
      const int sl = (int)(lu % (uint32_t)S);
      const uint64_t u = u0 + lu;
      const uint32_t yt = (uint32_t)u & ymask;
      if (yt == 0u) {
#pragma unroll
        for (int c = 0; c < NACC; ++c) acc[c] = make_float2(0.f, 0.f);
      }
      const uint32_t ybase = ft_trav(a.ty, u, a.ntrav);
      tc_mbar_wait(&x_full[sl], (lu / (uint32_t)S) & 1u);
      tc_mbar_wait(&mma_done[s], (lu >> 1) & 1u);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const float2* xs = reinterpret_cast<const float2*>(dsm_ft + a.sm_x + (uint32_t)sl * X_TILE) + r;
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
        const float2 w = C3s[ybase + yc];
        float2 xv[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) xv[j] = xs[(ch * 8 + j) * 128];
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int c = (ch * 8 + j) & (NACC - 1);
          const float2 t = make_float2(__uint_as_float(v[2 * j]), __uint_as_float(v[2 * j + 1]));
          const float2 wx = cmul(w, xv[j]);
          acc[c].x = fmaf(t.x, wx.x, fmaf(-t.y, wx.y, acc[c].x));
          acc[c].y = fmaf(t.x, wx.y, fmaf(t.y, wx.x, acc[c].y));
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        tc_mbar_arrive(&tmem_empty[s]);
        tc_mbar_arrive(&x_empty[sl]);
      }
      if (yt == ymask) {
        float2* o = a.out + ft_trav(a.to, u, a.ntrav) + orow;
#pragma unroll
        for (int c = 0; c < NACC; ++c) __stcs(o + ocol[c], acc[c]);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(a.tmem_cols));
}

}  // namespace tnb
