// kernels_tc.cuh -- k_gemm_tc: the two-operand fused merge group (batched complex GEMM,
// DESIGN.md section 5) on the 5th-generation tensor cores (tcgen05.mma kind::tf32, accumulators in
// TMEM), 3xTF32 split for FP32-level accuracy.
//
// The group computes  out[o] = sum_{x < 2^M} C_x(o) A[F_A(o) + G_A(x)] B[F_B(o) + G_B(x)]
// (an exact re-association of the merge step and the reduce steps after it, PAPER.md:361-368
// plus SURVEY F5).  Output bits are in A only ("row" class), in B only ("col" class) or in both
// ("diag" class = batch).  A CTA tile holds 7 row bits (the MMA's M = 128), nb col bits and nd
// diag bits.  For every diag value d of the tile one real GEMM
//     D_d[r][2n + e] = sum_{k'} A'_d[r][k'] B'_d[2n + e][k'],   k' = 2x + f
// with A'[r][2x] = Re A, A'[r][2x+1] = Im A and B' = (Re CB, -Im CB ; Im CB, Re CB) gives
// D[r][2n] = Re out, D[r][2n+1] = Im out.  Every operand is split v = big + small (big = v rounded
// to TF32, small = v - big exact in FP32) and D = Ab Bb + Ab Bs + As Bb (3 MMAs per K-chunk); the
// dropped As Bs term is <= 2^-22 |A||B|.
//
// Warp roles (416 threads, one CTA per SM, persistent over a contiguous tile range):
//   warps 8..11  loaders: raw B / C_x chunks by cp.async D tiles ahead, B' of every tile into one
//                of two slots, A' (two buffers) when A's chunk changes (the host orders the
//                traversal so that B-only bits flip first: A stays for 2^(#outer col bits) tiles);
//                arrive on ready[tile & 1];
//   warp 12      MMA: waits ready and tempty, issues the 3 KC ND MMAs of the tile (accumulators
//                interleaved) into TMEM buffer (tile & 1), commits to mdone[tile & 1];
//   warps 0..7   epilogue, two groups of four: group g takes the tiles with (tile & 1) == g, so
//                one group's staging overlaps the other group's store stream.  A thread reads its
//                TMEM lane (row) with tcgen05.ld, writes it into the group's shared staging tile in
//                output order (XOR-swizzled so a warp's 32 rows hit distinct bank pairs), releases
//                the TMEM buffer (tempty), then copies the tile out with coalesced 16-byte
//                streaming stores.
#pragma once
#include "kernels.cuh"

namespace tnb {

constexpr int kTcMaxTB = 14;          // 7 row + <= 6 col/diag bits (+1 spare)
constexpr int kTcMaxPerm = 32;        // tile-index bits (out_rank - TB)
constexpr int kTcEpiWarps = 8;
constexpr int kTcLdWarps = 4;
constexpr int kTcThreads = (kTcEpiWarps + kTcLdWarps + 1) * 32;   // + one MMA warp

struct TArgs {
  void* out;
  const float2* A;
  const float2* B;
  uint64_t maskA, maskB;               // F_t(o) = ins0(pext(o, mask_t), pv_t)
  uint32_t pvA, pvB;
  uint32_t rowoffA[1 << kMaxGroup];    // G_A(x), G_B(x): element offsets of summed value x
  uint32_t rowoffB[1 << kMaxGroup];
  const void* cin[kMaxIn];             // constant inputs (no tile bit; may depend on outer bits)
  uint64_t cmask[kMaxIn];
  uint32_t cpv[kMaxIn];
  uint32_t cgx[kMaxIn][1 << kMaxGroup];
  int32_t nc;
  int32_t M;                           // K = 2^M summed values
  int32_t TB, nd, nb;                  // tile bits = 7 row + nb col + nd diag
  int32_t kp;                          // floats per operand row (2K, at least 8)
  uint8_t role[kTcMaxTB];              // compact tile position u (ascending output bit): 0 row, 1 col, 2 diag
  uint8_t rj[kTcMaxTB];                // index of u within its role
  uint8_t sw[kTcMaxTB];                // staging swizzle: 4-bit XOR contributed by compact bit u >= 4
  uint8_t pad0[2];
  uint64_t obit[kTcMaxTB];             // output element offset of compact bit u (1 << output bit)
  uint32_t posA[kTcMaxTB];             // element offset within A / B of compact bit u (0: absent)
  uint32_t posB[kTcMaxTB];
  uint8_t perm[64];                    // tile index bit -> output bit (traversal order)
  int32_t nperm;
  uint64_t n_tiles;
  uint32_t sm_b, sm_stage, sm_tabs;    // dynamic smem byte offsets (A' buffers at 0, B' slots, two staging tiles, tables)
  uint32_t sm_raw;                     // raw A chunk, bslots raw B chunks, bslots C_x vectors (float2)
  int32_t bslots;                      // raw-B ring slots S (lookahead S - 1 tiles), 2..5
  int32_t pair16;                      // the lowest tile bit is output bit 0: 16-byte copy-out
  int32_t abufs;                       // A' buffers (2: the next A chunk is formatted while the MMAs read the current)
  int32_t dbg;                         // timing experiments only (TNB_TC_DBG): 1 skip B' after tile 0, 2 skip A' reloads, 4 skip stores, 8 trace CTA 0
  unsigned long long* trace;           // dbg & 8: [tile][event] clock64 of CTA 0 (events: 0 loader start, 1 MMA issued, 2 epi mdone ok, 3 epi staged, 4 epi stored)
  uint32_t abytes_d, bbytes_d;         // bytes of one d-block of A' / B' (big or small part)
  uint32_t tmem_cols;                  // allocated TMEM columns (2 accumulator buffers)
};

__device__ __forceinline__ uint32_t tc_smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void tc_mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(tc_smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void tc_mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tTC_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra TC_WAIT_%=;\n\t}" ::"r"(tc_smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tc_mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc_smem_u32(b)) : "memory");
}
__device__ __forceinline__ void tc_named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
// K-major, SWIZZLE_NONE shared-memory matrix descriptor (sm_100 "version 1"): core matrices of
// 8 rows x 16 bytes; lbo = byte distance between the two 16-byte K halves of an MMA (K = 8 TF32),
// sbo = byte distance between consecutive 8-row groups
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                          uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void tf32_split(float v, float& big, float& small) {
  uint32_t b;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(b) : "f"(v));
  big = __uint_as_float(b);
  small = v - big;
}

#ifndef TNB_TC_HELPERS_ONLY   // launch_fc_tc.cu includes only the helpers above
__global__ void __launch_bounds__(kTcThreads, 1) k_gemm_tc(const TArgs a) {
  extern __shared__ __align__(128) unsigned char dsm_tc[];
  __shared__ uint64_t bar_mdone[2], bar_tempty[2], bar_ready[2], bar_rawa;
  __shared__ uint32_t tmem_base_sh;
  __shared__ uint32_t tile_abuf[2];
  // incremental tile offsets (as in k_gemm): stream s = 0 output, 1 A, 2 B, 3 + q constant q;
  // tile index t -> t + 1 flips bits 0 .. r-1 to 0 and bit r to 1 (r = ctz(~t)), so an offset
  // advances by fbit[s][r] - fcum[s][r]
  __shared__ uint64_t fbit[3 + kMaxIn][kTcMaxPerm], fcum[3 + kMaxIn][kTcMaxPerm + 1];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int K = 1 << a.M, ND = 1 << a.nd, NC = 1 << a.nb, TB = a.TB;
  const int nA = 1 << (7 + a.nd), nBc = 1 << (a.nb + a.nd), nHi = 1 << (TB - 8);
  const uint32_t TCOL = (uint32_t)(ND * 2 * NC);                 // accumulator columns per tile
  const uint32_t SBO = (uint32_t)(a.kp / 4) * 128u;
  const uint32_t abuf_bytes = 2u * (uint32_t)ND * a.abytes_d;    // one A' buffer (big + small)
  uint32_t* a_goff = reinterpret_cast<uint32_t*>(dsm_tc + a.sm_tabs);
  uint32_t* a_soff = a_goff + nA;
  uint32_t* b_goff = a_soff + nA;
  uint32_t* b_soff = b_goff + nBc;
  uint32_t* pcol = b_soff + nBc;
  uint32_t* lsw_hi = pcol + nBc;
  uint64_t* dlo = reinterpret_cast<uint64_t*>(lsw_hi + ((nHi + 1) & ~1));
  uint64_t* dhi = dlo + 256;

  // ---- setup: zero the operand tiles (K padding), offset tables, barriers, TMEM
  {
    uint4* z = reinterpret_cast<uint4*>(dsm_tc);
    const uint32_t n16 = a.sm_stage / 16;
    for (uint32_t i = tid; i < n16; i += kTcThreads) z[i] = make_uint4(0, 0, 0, 0);
  }
  auto Lsw = [&](uint32_t c) {   // XOR swizzle of compact index c (bits >= 4)
    uint32_t s = 0;
    for (int u = 4; u < TB; ++u)
      if ((c >> u) & 1u) s ^= a.sw[u];
    return s;
  };
  for (int i = tid; i < nA; i += kTcThreads) {   // A chunk index: row / diag tile bits ascending
    uint32_t g = 0, r = 0, d = 0;
    int k = 0;
    for (int u = 0; u < TB; ++u) {
      if (a.role[u] == 1) continue;
      if ((i >> k) & 1) {
        g += a.posA[u];
        if (a.role[u] == 0) r |= 1u << a.rj[u]; else d |= 1u << a.rj[u];
      }
      ++k;
    }
    a_goff[i] = g;
    a_soff[i] = d * a.abytes_d + (r >> 3) * SBO + (r & 7u) * 16u;
  }
  for (int i = tid; i < nBc; i += kTcThreads) {  // B chunk index: col / diag tile bits ascending
    uint32_t g = 0, n = 0, d = 0;
    int k = 0;
    for (int u = 0; u < TB; ++u) {
      if (a.role[u] == 0) continue;
      if ((i >> k) & 1) {
        g += a.posB[u];
        if (a.role[u] == 1) n |= 1u << a.rj[u]; else d |= 1u << a.rj[u];
      }
      ++k;
    }
    b_goff[i] = g;
    b_soff[i] = d * a.bbytes_d + ((2u * n) >> 3) * SBO + ((2u * n) & 7u) * 16u;
  }
  for (int gc = tid; gc < nBc; gc += kTcThreads) {   // accumulator column gc = d NC + n
    const uint32_t n = gc & (NC - 1), d = gc >> a.nb;
    uint32_t c = 0;
    for (int u = 0; u < TB; ++u) {
      if (a.role[u] == 1 && ((n >> a.rj[u]) & 1u)) c |= 1u << u;
      if (a.role[u] == 2 && ((d >> a.rj[u]) & 1u)) c |= 1u << u;
    }
    pcol[gc] = c ^ Lsw(c);
  }
  for (int j = tid; j < nHi; j += kTcThreads) {
    uint32_t s = 0;
    uint64_t o = 0;
    for (int u = 8; u < TB; ++u)
      if ((j >> (u - 8)) & 1) { s ^= a.sw[u]; o += a.obit[u]; }
    lsw_hi[j] = s;
    dhi[j] = o;
  }
  for (int j = tid; j < 256; j += kTcThreads) {
    uint64_t o = 0;
    for (int u = 0; u < 8; ++u)
      if ((j >> u) & 1) o += a.obit[u];
    dlo[j] = o;
  }
  const int NS = 3 + a.nc;
  for (int i = tid; i < NS * kTcMaxPerm; i += kTcThreads) {
    const int st = i / kTcMaxPerm, b = i % kTcMaxPerm;
    uint64_t v = 0;
    if (b < a.nperm) {
      const uint64_t o = 1ull << a.perm[b];
      v = st == 0 ? o : st == 1 ? fmap(o, a.maskA, a.pvA) : st == 2 ? fmap(o, a.maskB, a.pvB)
                                 : fmap(o, a.cmask[st - 3], a.cpv[st - 3]);
    }
    fbit[st][b] = v;
  }
  __syncthreads();
  if (tid < NS) {
    uint64_t c = 0;
    for (int b = 0; b < kTcMaxPerm; ++b) { fcum[tid][b] = c; c += fbit[tid][b]; }
    fcum[tid][kTcMaxPerm] = c;
  }
  if (tid == 0) {
    tc_mbar_init(&bar_mdone[0], 1);
    tc_mbar_init(&bar_mdone[1], 1);
    tc_mbar_init(&bar_tempty[0], kTcEpiWarps / 2);
    tc_mbar_init(&bar_tempty[1], kTcEpiWarps / 2);
    tc_mbar_init(&bar_ready[0], kTcLdWarps * 32);
    tc_mbar_init(&bar_ready[1], kTcLdWarps * 32);
    tc_mbar_init(&bar_rawa, kTcLdWarps * 32);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc_smem_u32(&tmem_base_sh)),
                 "r"(a.tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base_sh;

  const uint64_t per = (a.n_tiles + gridDim.x - 1) / gridDim.x;
  const uint64_t t0 = (uint64_t)blockIdx.x * per;
  const uint64_t t1 = t0 + per < a.n_tiles ? t0 + per : a.n_tiles;
  auto off_at = [&](int st, uint64_t t) {     // offset of stream st at tile t (direct)
    uint64_t o = 0;
    for (int b = 0; b < a.nperm && (t >> b); ++b)
      if ((t >> b) & 1) o += fbit[st][b];
    return o;
  };
  auto step = [&](int st, uint64_t& o, uint64_t t) {   // o: offset at tile t -> offset at t + 1
    const int r = __ffsll((long long)~t) - 1;
    o = o + fbit[st][r] - fcum[st][r];
  };

  if (warp == kTcEpiWarps + kTcLdWarps) {
    // =========================== MMA warp: every lane walks the loop (descriptors stay
    // warp-uniform), one lane issues the tcgen05.mma of the tile and the commit
    const uint32_t sA = tc_smem_u32(dsm_tc);
    const uint32_t sB = tc_smem_u32(dsm_tc + a.sm_b);
    const uint32_t asmall = (uint32_t)ND * a.abytes_d;
    const uint32_t bslot = 2u * (uint32_t)ND * a.bbytes_d, bsmall = (uint32_t)ND * a.bbytes_d;
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)((2 * NC) >> 3) << 17) |
                           ((uint32_t)(128 >> 4) << 24);
    const uint64_t dhi_bits = ((uint64_t)((SBO >> 4) & 0x3FFFu) << 32) | (1ull << 46) | ((uint64_t)(128u >> 4) << 16);
    const int KC = a.kp / 8;
    uint32_t lt = 0;
    for (uint64_t t = t0; t < t1; ++t, ++lt) {
      const uint32_t slot = lt & 1u;
      tc_mbar_wait(&bar_ready[slot], (lt >> 1) & 1u);
      if (lt >= 2) tc_mbar_wait(&bar_tempty[slot], ((lt - 2) >> 1) & 1u);   // epilogue drained buffer
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if ((a.dbg & 8) && blockIdx.x == 0 && lane == 0 && lt < 64) a.trace[lt * 8 + 5] = clock64();
      if (lane == 0) {
        // one lane walks the MMAs of the tile (no per-MMA warp reconvergence); descriptors are
        // additive in their start-address field: base + (byte offset >> 4)
        const uint32_t aS = sA + tile_abuf[slot] * abuf_bytes;
        const uint32_t bS = sB + slot * bslot;
        const uint64_t dA0 = dhi_bits | ((aS >> 4) & 0x3FFFu), dB0 = dhi_bits | ((bS >> 4) & 0x3FFFu);
        const uint32_t tcol0 = tmem + slot * TCOL;
        const uint32_t ad16 = a.abytes_d >> 4, bd16 = a.bbytes_d >> 4, as16 = asmall >> 4, bs16 = bsmall >> 4;
        // the ND accumulators are independent: interleave them so consecutive MMAs never chain on
        // one accumulator (a dependent tf32 MMA at N <= 128 costs ~110 cycles, independent ones
        // ~60; scripts/probe/tc_rate.cu)
        for (int kc = 0; kc < KC; ++kc)
#pragma unroll
          for (int pr = 0; pr < 3; ++pr)
            for (int d = 0; d < ND; ++d) {
              const uint64_t da = dA0 + (uint32_t)(d * ad16 + kc * 16 + (pr == 0 ? as16 : 0u));
              const uint64_t db = dB0 + (uint32_t)(d * bd16 + kc * 16 + (pr == 1 ? bs16 : 0u));
              if (!((a.dbg & 32) && (kc | pr))) umma_tf32(tcol0 + (uint32_t)d * 2u * NC, da, db, idesc, (kc | pr) ? 1u : 0u);
            }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         tc_smem_u32(&bar_mdone[slot]))
                     : "memory");
      }
      __syncwarp();
      if ((a.dbg & 8) && blockIdx.x == 0 && lane == 0 && lt < 64) a.trace[lt * 8 + 1] = clock64();
    }
  } else if (warp >= kTcEpiWarps) {
    // =========================== loaders
    // Raw chunks come in by cp.async ahead of use: B's chunk and the constant factors C_x of tile
    // t + D during tile t (a ring of S = D + 1 raw-B / C slots), A's next chunk right after the
    // current one has been formatted (one raw-A slot).  Formatting (TF32 split, B' block
    // structure) reads shared memory only.  cp.async groups: one per iteration (plus D in the
    // prologue), so waiting until at most D groups are pending completes tile t's chunk.
    const int ltid = tid - kTcEpiWarps * 32;
    constexpr int kLd = kTcLdWarps * 32;
    const int S = a.bslots, D = S - 1;
    const uint32_t bslot = 2u * (uint32_t)ND * a.bbytes_d, bsmall = (uint32_t)ND * a.bbytes_d;
    const uint32_t asmall = (uint32_t)ND * a.abytes_d;
    float2* rawA = reinterpret_cast<float2*>(dsm_tc + a.sm_raw);
    float2* rawB = rawA + K * nA;                  // S slots of K * nBc
    float2* Cs = rawB + S * K * nBc;               // S slots of nc x K raw constant values
    auto issue_rawB = [&](uint64_t bb, int sl) {
      float2* dst = rawB + sl * K * nBc;
      for (int e = ltid; e < K * nBc; e += kLd) {
        const int x = e >> (a.nb + a.nd), j = e & (nBc - 1);
        cp_async8(dst + e, a.B + bb + b_goff[j] + a.rowoffB[x]);
      }
    };
    // raw A completes on its own mbarrier (bar_rawa: every loader thread arrives once its copies
    // -- and any older ones -- have landed), so waiting for it never waits for newer raw-B copies
    auto issue_rawA = [&](uint64_t ab) {
      for (int e = ltid; e < K * nA; e += kLd) {
        const int x = e >> (7 + a.nd), i = e & (nA - 1);
        cp_async8(rawA + e, a.A + ab + a_goff[i] + a.rowoffA[x]);
      }
      mbar_cp_async_arrive(&bar_rawa);
    };
    uint32_t a_ver = 0;                             // raw-A chunks consumed so far
    uint64_t cofs[kMaxIn];                          // constant offsets at the prefetch tile
    const int nCK = a.nc * K;
    auto issue_c = [&](int sl) {                    // element e < nc K: constant q = e / K, value x
      for (int e = ltid; e < nCK; e += kLd) {
        const int q = e >> a.M, x = e & (K - 1);
        uint64_t co = 0;
#pragma unroll
        for (int qq = 0; qq < kMaxIn; ++qq)
          if (qq == q) co = cofs[qq];
        cp_async8(Cs + sl * nCK + e, static_cast<const float2*>(a.cin[q]) + co + a.cgx[q][x]);
      }
    };
    // the next tile after t (within the range) whose A chunk differs (offset `ao` at t)
    auto next_a = [&](uint64_t t, uint64_t ao, uint64_t& nab) {
      uint64_t o = ao;
      for (uint64_t u = t; u + 1 < t1; ++u) {
        step(1, o, u);
        if (o != ao) { nab = o; return u + 1; }
      }
      return t1;
    };
    uint64_t a_tile = t0, a_next_base = 0, bpre = 0, pre_t = t0;   // pre_t: tile of bpre / cofs
    if (t0 < t1) {
      a_next_base = off_at(1, t0);
      bpre = off_at(2, t0);
#pragma unroll
      for (int q = 0; q < kMaxIn; ++q) cofs[q] = q < a.nc ? off_at(3 + q, t0) : 0;
      issue_rawA(a_next_base);
    }
    for (int i = 0; i < D; ++i) {                   // prologue: tiles t0 .. t0 + D - 1
      if (pre_t < t1) {
        if (i > 0) {
          step(2, bpre, pre_t - 1);
#pragma unroll
          for (int q = 0; q < kMaxIn; ++q)
            if (q < a.nc) step(3 + q, cofs[q], pre_t - 1);
        }
        issue_rawB(bpre, i);
        issue_c(i);
      }
      ++pre_t;
      cp_async_commit();
    }
    uint32_t lt = 0;
    int bs_cur = 0;                                 // ring slot of tile t (= lt mod S)
    uint32_t abuf = a.abufs - 1;                    // A' buffer of the current A chunk (first: 0)
    int a_last0 = -1, a_last1 = -1;                 // last local tile that read each A' buffer
    for (uint64_t t = t0; t < t1; ++t, ++lt) {
      const uint32_t slot = lt & 1u;
      // (1) prefetch tile t + D: raw B chunk and C_x (cp.async)
      const int bs_pre = bs_cur + D >= S ? bs_cur + D - S : bs_cur + D;
      if (pre_t < t1) {
        step(2, bpre, pre_t - 1);
#pragma unroll
        for (int q = 0; q < kMaxIn; ++q)
          if (q < a.nc) step(3 + q, cofs[q], pre_t - 1);
        issue_rawB(bpre, bs_pre);
        issue_c(bs_pre);
      }
      ++pre_t;
      cp_async_commit();
      // (2) the group of iteration lt - D (tile t's chunk) landed; visible to all loaders
      if (D <= 1) cp_async_wait<1>(); else if (D == 2) cp_async_wait<2>(); else if (D == 3) cp_async_wait<3>();
      else cp_async_wait<4>();
      tc_named_bar(1, kLd);
      if ((a.dbg & 8) && blockIdx.x == 0 && ltid == 0 && lt < 64) a.trace[lt * 8 + 6] = clock64();
      // (3) B'[slot] = (Re, -Im ; Im, Re) of C_x B, TF32 big / small; MMA(lt-2) read B'[slot]
      //     (and, completing in order, every MMA before it)
      if (lt >= 2) tc_mbar_wait(&bar_mdone[slot], ((lt - 2) >> 1) & 1u);
      if (!((a.dbg & 1) && lt >= 2)) {
        const float2* rb = rawB + bs_cur * K * nBc;
        const float2* cs = Cs + bs_cur * nCK;
        unsigned char* bs = dsm_tc + a.sm_b + slot * bslot;
        for (int e = ltid; e < K * nBc; e += kLd) {
          const int x = e >> (a.nb + a.nd), j = e & (nBc - 1);
          float2 v = rb[e];
          for (int q = 0; q < a.nc; ++q) v = cmul(v, cs[q * K + x]);
          float rbg, rsm, ibg, ism;
          tf32_split(v.x, rbg, rsm);
          tf32_split(v.y, ibg, ism);
          const uint32_t off = b_soff[j] + (uint32_t)(x >> 1) * 128u + (uint32_t)(x & 1) * 8u;
          *reinterpret_cast<float2*>(bs + off) = make_float2(rbg, -ibg);
          *reinterpret_cast<float2*>(bs + off + 16) = make_float2(ibg, rbg);
          *reinterpret_cast<float2*>(bs + bsmall + off) = make_float2(rsm, -ism);
          *reinterpret_cast<float2*>(bs + bsmall + off + 16) = make_float2(ism, rsm);
        }
      }
      if ((a.dbg & 8) && blockIdx.x == 0 && ltid == 0 && lt < 64) a.trace[lt * 8 + 7] = clock64();
      // (4) A' when A's chunk changes at this tile (its raw chunk was prefetched) into the other
      //     buffer; then prefetch the next chunk
      if (t == a_tile && !((a.dbg & 2) && lt > 0)) {
        tc_mbar_wait(&bar_rawa, a_ver & 1u);         // this chunk's raw copies landed (all loaders)
        ++a_ver;
        abuf = a.abufs == 2 ? abuf ^ 1u : 0u;
        // the MMAs that last read this buffer: all tiles <= lt - 2 are complete (step 3)
        if ((abuf ? a_last1 : a_last0) == (int)lt - 1) tc_mbar_wait(&bar_mdone[(lt - 1) & 1u], ((lt - 1) >> 1) & 1u);
        unsigned char* ab = dsm_tc + abuf * abuf_bytes;
        for (int e = ltid; e < K * nA; e += kLd) {
          const int x = e >> (7 + a.nd), i = e & (nA - 1);
          const float2 v = rawA[e];
          float rbg, rsm, ibg, ism;
          tf32_split(v.x, rbg, rsm);
          tf32_split(v.y, ibg, ism);
          const uint32_t off = a_soff[i] + (uint32_t)(x >> 1) * 128u + (uint32_t)(x & 1) * 8u;
          *reinterpret_cast<float2*>(ab + off) = make_float2(rbg, ibg);
          *reinterpret_cast<float2*>(ab + asmall + off) = make_float2(rsm, ism);
        }
        a_tile = next_a(t, a_next_base, a_next_base);
        tc_named_bar(1, kLd);                       // every loader is done reading raw A
        if (a_tile < t1) issue_rawA(a_next_base);
      }
      if (abuf) a_last1 = (int)lt; else a_last0 = (int)lt;
      if (ltid == 0) tile_abuf[slot] = abuf;
      bs_cur = bs_cur + 1 == S ? 0 : bs_cur + 1;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tc_mbar_arrive(&bar_ready[slot]);             // B'[slot], A' and tile_abuf of tile t ready
      if ((a.dbg & 8) && blockIdx.x == 0 && ltid == 0 && lt < 64) a.trace[lt * 8 + 0] = clock64();
      tc_named_bar(1, kLd);                         // raw-B / C slots of this tile free for reuse
    }
    cp_async_wait<0>();
  } else {
    // =========================== epilogue group g = warp >> 2: tiles with (local index & 1) == g
    const int g = warp >> 2, q = warp & 3;
    const uint32_t r = (uint32_t)(32 * q + lane);
    const uint32_t etid = (uint32_t)(tid & 127);
    float2* stage = reinterpret_cast<float2*>(dsm_tc + a.sm_stage) + ((size_t)g << TB);
    uint32_t prow = 0;
    for (int u = 0; u < TB; ++u)
      if (a.role[u] == 0 && ((r >> a.rj[u]) & 1u)) prow |= 1u << u;
    prow ^= Lsw(prow);
    // staging positions of accumulator column gc = 8 c + j: pcol is XOR-linear in gc, so
    // pcol[gc] = pcol[8 c] ^ pcol[j] (registers: no shared loads between the staging stores)
    uint32_t pj[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) pj[j] = pcol[j];
    auto lsw_lo_of = [&](uint32_t e) {             // swizzle of bits 4-7 of e
      uint32_t s2 = 0;
      for (int u = 4; u < 8 && u < TB; ++u)
        if ((e >> u) & 1u) s2 ^= a.sw[u];
      return s2;
    };
    // 16-byte path: pair (e, e + 1), e = 2 (etid + 128 i): bits 0-7 from 2 etid, bits >= 8 = i
    const uint64_t p_dlo = dlo[(2u * etid) & 255u];
    const uint32_t p_lsw = lsw_lo_of(2u * etid);
    // 8-byte path: e = etid + 128 i: bits 0-7 = etid + 128 (i & 1), bits >= 8 = i >> 1
    const uint64_t s_dlo0 = dlo[etid], s_dlo1 = dlo[etid + 128u];
    const uint32_t s_lsw0 = lsw_lo_of(etid), s_lsw1 = lsw_lo_of(etid + 128u);
    float2* out = static_cast<float2*>(a.out);
    const int ncb = (int)(TCOL >> 4);               // 16-column chunks of a tile (<= 8)
    uint32_t lt = 0;
    uint64_t ob = t0 < t1 ? off_at(0, t0) : 0;
    for (uint64_t t = t0; t < t1; ++t, ++lt) {
      if ((lt & 1u) != (uint32_t)g) {
        if (t + 1 < t1) step(0, ob, t);
        continue;
      }
      const uint32_t slot = lt & 1u;
      tc_mbar_wait(&bar_mdone[slot], (lt >> 1) & 1u);
      if ((a.dbg & 8) && blockIdx.x == 0 && etid == 0 && lt < 64) a.trace[lt * 8 + 2] = clock64();
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t tbase = tmem + ((uint32_t)(32 * q) << 16) + slot * TCOL;
      for (int c0 = 0; c0 < ((a.dbg & 16) ? 0 : ncb); c0 += 4) {         // up to 64 columns in flight, one wait
        uint32_t v[64];
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (c0 + c < ncb)
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                : "=r"(v[16 * c + 0]), "=r"(v[16 * c + 1]), "=r"(v[16 * c + 2]), "=r"(v[16 * c + 3]),
                  "=r"(v[16 * c + 4]), "=r"(v[16 * c + 5]), "=r"(v[16 * c + 6]), "=r"(v[16 * c + 7]),
                  "=r"(v[16 * c + 8]), "=r"(v[16 * c + 9]), "=r"(v[16 * c + 10]), "=r"(v[16 * c + 11]),
                  "=r"(v[16 * c + 12]), "=r"(v[16 * c + 13]), "=r"(v[16 * c + 14]), "=r"(v[16 * c + 15])
                : "r"(tbase + 16u * (c0 + c)));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        uint32_t pc[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) pc[c] = c0 + c < ncb ? pcol[8 * (c0 + c)] : 0u;
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (c0 + c < ncb) {
#pragma unroll
            for (int j = 0; j < 8; ++j)
              stage[prow ^ pc[c] ^ pj[j]] = make_float2(__uint_as_float(v[16 * c + 2 * j]), __uint_as_float(v[16 * c + 2 * j + 1]));
          }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) tc_mbar_arrive(&bar_tempty[slot]);
      tc_named_bar(2 + g, 128);
      if ((a.dbg & 8) && blockIdx.x == 0 && etid == 0 && lt < 64) a.trace[lt * 8 + 3] = clock64();
      if (a.dbg & 16) {
      } else if (a.pair16) {
        // 16-byte pieces: compact pair (e, e + 1) is adjacent in the output (the lowest tile bit
        // is output bit 0) and in staging (the swizzle moves bits 0-3 by a function of bits >= 4)
        float2* ot = out + ob + p_dlo;
#pragma unroll 4
        for (int i = 0; i < nHi; ++i) {
          const uint32_t e = 2u * etid + 256u * (uint32_t)i;
          const uint32_t L = p_lsw ^ lsw_hi[i];
          const float4 w = *reinterpret_cast<const float4*>(stage + ((e ^ L) & ~1u));
          const float4 val = (L & 1u) ? make_float4(w.z, w.w, w.x, w.y) : w;
          if (!(a.dbg & 4)) __stcs(reinterpret_cast<float4*>(ot + dhi[i]), val);
        }
      } else {
#pragma unroll 4
        for (int i = 0; i < 2 * nHi; ++i) {
          const uint32_t e = etid + 128u * (uint32_t)i;
          const uint32_t L = ((i & 1) ? s_lsw1 : s_lsw0) ^ lsw_hi[i >> 1];
          const float2 val = stage[e ^ L];
          if (!(a.dbg & 4)) __stcs(out + ob + ((i & 1) ? s_dlo1 : s_dlo0) + dhi[i >> 1], val);
        }
      }
      if (t + 1 < t1) step(0, ob, t);
      tc_named_bar(2 + g, 128);
      if ((a.dbg & 8) && blockIdx.x == 0 && etid == 0 && lt < 64) a.trace[lt * 8 + 4] = clock64();
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(a.tmem_cols));
}

#endif  // TNB_TC_HELPERS_ONLY

}  // namespace tnb
