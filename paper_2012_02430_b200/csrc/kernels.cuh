// kernels.cuh -- sm_100a kernels of the bucket-elimination hot path.
//
//   k_materialize  gate tensors from (gamma, beta) into the arena (the plan is
//                  reused across parameters, only the leaf values change)
//   k_bucket       one bucket step ("elimination of vertex i") as an
//                  HBM-streaming, output-tiled gather-multiply-sum:
//                      out[o] = sum_{x in {0,1}} prod_t in_t[F_t(o) + x * 2^{pv_t}],
//                      F_t(o) = ins0(pext(o, out_mask_t), pv_t)
//                  F_t is additive over disjoint bit sets, so it splits into a per-tile, a
//                  per-thread and a per-iteration part; the inner loop is adds + loads only.
//                  Inputs holding the output's lowest bit are read with 16-byte vector loads;
//                  broadcast inputs are read once per thread; large (read-once) inputs use
//                  evict-first streaming loads; outputs are written with 16-byte stores.
//   k_program      a batched interpreter: one CTA runs a list of (small) bucket steps with
//                  __syncthreads between steps -- runs of tiny steps of a big plan, or one whole
//                  light-cone network per CTA (all edges in one launch)
//   k_finalize     per slice: product of the rank-0 tensors in FP64, x 2^{log2_scale}
//   k_pairwise     fixed-order pairwise sum of the per-slice partials
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "plan_format.h"

#ifndef GEMM_U1
#define GEMM_U1 1    // k_gemm's chunk-load and B' rebuild loops kept rolled (as FC_U1): about half the SASS,
                     // C5a 101.8 vs 101.0 /s, C4b 105.4 vs 103.0 /s (`profiles/r02/session4/gemm_u1/`)
#endif
#if GEMM_U1
#define GEMM_LOOP_PRAGMA _Pragma("unroll 1")
#else
#define GEMM_LOOP_PRAGMA
#endif

namespace tnb {

// ------------------------------------------------------------------ complex helpers
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
template <typename T> __device__ __forceinline__ T cfrom(double re, double im);
template <> __device__ __forceinline__ float2 cfrom<float2>(double re, double im) {
  return make_float2((float)re, (float)im);
}
template <> __device__ __forceinline__ double2 cfrom<double2>(double re, double im) {
  return make_double2(re, im);
}
__device__ __forceinline__ double2 to_d2(float2 a) { return make_double2(a.x, a.y); }
__device__ __forceinline__ double2 to_d2(double2 a) { return a; }

// ------------------------------------------------------------------ bit helpers
// pext(x, m): gather the bits of x selected by m into the low bits (loop over set bits of x & m)
__device__ __forceinline__ uint64_t pext_bits(uint64_t x, uint64_t m) {
  uint64_t r = 0, y = x & m;
  while (y) {
    const uint64_t b = y & (~y + 1);
    r |= 1ull << __popcll(m & (b - 1));
    y ^= b;
  }
  return r;
}
// insert a zero bit at position pv
__device__ __forceinline__ uint64_t ins0(uint64_t x, uint32_t pv) {
  const uint64_t lo = x & ((1ull << pv) - 1);
  return lo | ((x >> pv) << (pv + 1));
}
__device__ __forceinline__ uint64_t fmap(uint64_t o, uint64_t mask, uint32_t pv) {
  return ins0(pext_bits(o, mask), pv);
}

// ------------------------------------------------------------------ materialize
struct Angles {
  double gamma[kMaxP];
  double beta[kMaxP];
  int p;
};

// blockIdx.y = parameter set y (batched energy): angles from dev_angles[y] (or `ang` when null),
// written into window y
template <typename T>
__global__ void k_materialize(const LeafRec* __restrict__ leaves, int n_leaves, Angles ang,
                              const Angles* __restrict__ dev_angles, T* __restrict__ ws,
                              uint64_t win0, uint64_t win_elems) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  const int li = idx >> 2, e = idx & 3;
  if (li >= n_leaves) return;
  const LeafRec lr = leaves[li];
  if (e >= (1 << lr.rank)) return;
  const Angles& A = dev_angles ? dev_angles[blockIdx.y] : ang;
  double re = 1.0, im = 0.0;
  for (int f = 0; f < lr.nfact; ++f) {
    double fr = 1.0, fi = 0.0;
    const int l = lr.layer[f];
    const int a = (lr.rank == 2) ? (e >> 1) : e, b = e & 1;
    switch (lr.code[f]) {
      case LC_PLUS: break;
      case LC_ZOBS: fr = e ? -1.0 : 1.0; break;
      case LC_RXROW0: {
        double s, c;
        sincos(A.beta[l], &s, &c);
        if (e == 0) { fr = c; } else { fr = 0.0; fi = -s; }
        break;
      }
      case LC_ZZ: {
        if (a != b) { double s, c; sincos(A.gamma[l], &s, &c); fr = c; fi = -s; }
        break;
      }
      case LC_RX: {
        double s, c;
        sincos(A.beta[l], &s, &c);
        if (a == b) { fr = c; } else { fr = 0.0; fi = -s; }
        break;
      }
      default: break;
    }
    if (lr.conj[f]) fi = -fi;
    const double nr = re * fr - im * fi, ni = re * fi + im * fr;
    re = nr;
    im = ni;
  }
  const uint64_t rel = blockIdx.y == 0 ? 0ull : win0 + (uint64_t)(blockIdx.y - 1) * win_elems;
  ws[rel + lr.off + e] = cfrom<T>(re, im);
}

// ------------------------------------------------------------------ standalone bucket step
struct BigArgs {
  void* out;
  const void* in[kMaxIn];
  uint64_t out_mask[kMaxIn];
  uint32_t pv[kMaxIn];
  uint32_t flags[kMaxIn];
  uint32_t stage_off[kMaxIn];  // staged inputs: element offset of buffer 0 in dynamic smem
  uint32_t nlow[kMaxIn];       // staged inputs: log2 of the per-tile chunk (per x)
  uint32_t stage_elems;        // elements of one smem buffer (all staged inputs, both x)
  int32_t out_rank;
  int32_t n_in;
  uint8_t perm[64];            // traversal order of the tile-index bits (logical bit b -> output
                               // bit TB + perm[b]); bits absent from the big inputs go first so
                               // tiles that share an input chunk run back to back (L2 / smem reuse)
};

template <typename T> struct VecT;
template <> struct VecT<float2> { using type = float4; static constexpr int n = 2; };
template <> struct VecT<double2> { using type = double2; static constexpr int n = 1; };

template <typename T>
__device__ __forceinline__ T ld_in(const T* p, bool stream) {  // stream: evict-first
  return stream ? __ldcs(p) : __ldg(p);
}
__device__ __forceinline__ float4 ld_in4(const float4* p, bool stream) {
  return stream ? __ldcs(p) : __ldg(p);
}

constexpr int kBucketThreads = 256;
constexpr int kBucketIters = 8;

template <typename T> struct TileBits;
template <> struct TileBits<float2> { static constexpr int v = 12; };   // 256 thr x 2 elem x 8 it
template <> struct TileBits<double2> { static constexpr int v = 11; };  // 256 thr x 1 elem x 8 it

// Input access modes (uniform per launch):
//   CONST: F_t has no bit inside a tile -> the two values (x = 0, 1) are loaded once per tile and
//          pre-multiplied into the tile constants C0, C1
//   VEC:   the input holds the output's bit 0 at its bit 0 -> 16-byte vector loads (c64)
//   BCAST: the input lacks output bit 0 -> one load serves both elements of a pair (c64)
//   PAIR:  output bit 0 sits elsewhere in the input -> two scalar loads (c64)
// Orthogonally an input is STAGED (flags bit1, set by the host) when it holds only part of a
// tile's low bits and those are its lowest positions: its per-tile chunk (two contiguous runs of
// 2^nlow elements, x = 0 and 1) is copied into shared memory with cp.async one tile ahead
// (double buffer) -- the reused merge operands -- instead of latency-bound direct loads.
enum : uint32_t { M_CONST = 0, M_VEC = 1, M_BCAST = 2, M_PAIR = 3 };
constexpr uint32_t F_STREAM = 1u, F_STAGED = 2u;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// OffT = uint32_t when every input has <= 32 bits (element offsets < 2^32), else uint64_t.
template <typename T, int NIN, typename OffT>
__global__ void __launch_bounds__(kBucketThreads, 4) k_bucket(const BigArgs a) {
  constexpr int VEC = VecT<T>::n;
  constexpr int TB = TileBits<T>::v;
  constexpr int STRIDE = kBucketThreads * VEC;
  constexpr uint64_t TILE = 1ull << TB;
  constexpr int NB = 64 - TB;
  const uint64_t n_out = 1ull << a.out_rank;
  const uint64_t n_tiles = (n_out + TILE - 1) >> TB;
  const uint32_t tid = threadIdx.x;
  extern __shared__ __align__(16) unsigned char dsm[];
  T* stage = reinterpret_cast<T*>(dsm);

  __shared__ OffT kofs[NIN][kBucketIters];
  __shared__ OffT fbit[NIN][NB];
  __shared__ OffT fcum[NIN][NB + 1];
  __shared__ uint64_t pbit[NB], pcum[NB + 1];
  if (tid < NIN * kBucketIters) {
    const int t = tid / kBucketIters, kk = tid % kBucketIters;
    kofs[t][kk] = (OffT)fmap((uint64_t)kk * STRIDE, a.out_mask[t], a.pv[t]);
  }
  for (int i = tid; i < NIN * NB; i += kBucketThreads) {
    const int t = i / NB, b = i % NB;
    fbit[t][b] = (OffT)fmap(1ull << (TB + a.perm[b]), a.out_mask[t], a.pv[t]);
  }
  for (int b = tid; b < NB; b += kBucketThreads) pbit[b] = 1ull << a.perm[b];
  __syncthreads();
  const int nbu = min(NB - 1, max(0, (int)a.out_rank - TB));   // tile-index bits in use
  if (tid < NIN) {
    OffT c = 0;
    fcum[tid][0] = 0;
    for (int b = 0; b < nbu; ++b) { c += fbit[tid][b]; fcum[tid][b + 1] = c; }
  }
  if (tid == NIN) {
    uint64_t c = 0;
    pcum[0] = 0;
    for (int b = 0; b < nbu; ++b) { c += pbit[b]; pcum[b + 1] = c; }
  }
  // this CTA's contiguous range of LOGICAL tiles; the physical tile is the perm-deposit of it
  const uint64_t per = (n_tiles + gridDim.x - 1) / gridDim.x;
  const uint64_t t0 = (uint64_t)blockIdx.x * per;
  const uint64_t t1 = t0 + per < n_tiles ? t0 + per : n_tiles;
  uint64_t ptile = 0;
  for (int b = 0; b < NB && (t0 >> b); ++b)
    if ((t0 >> b) & 1) ptile |= 1ull << a.perm[b];

  OffT thr[NIN], S[NIN], cur[NIN], pf[NIN], s1v[NIN];
  uint32_t mode[NIN];
  bool strm[NIN], stg[NIN];
  const T* in[NIN];
  const uint64_t inner = TILE - 1;
#pragma unroll
  for (int t = 0; t < NIN; ++t) {
    in[t] = static_cast<const T*>(a.in[t]);
    thr[t] = (OffT)fmap((uint64_t)tid * VEC, a.out_mask[t], a.pv[t]);
    S[t] = (OffT)1 << a.pv[t];
    s1v[t] = (OffT)fmap(1, a.out_mask[t], a.pv[t]);
    mode[t] = ((a.out_mask[t] & inner) == 0) ? M_CONST
              : (VEC == 1 || s1v[t] == 1)    ? M_VEC
              : (s1v[t] == 0)                ? M_BCAST
                                             : M_PAIR;
    strm[t] = (a.flags[t] & F_STREAM) != 0;
    stg[t] = (a.flags[t] & F_STAGED) != 0 && mode[t] != M_CONST;
    cur[t] = (OffT)fmap(ptile << TB, a.out_mask[t], a.pv[t]);
    pf[t] = cur[t];
  }
  T* out = static_cast<T*>(a.out);
  bool any_stage = false;
#pragma unroll
  for (int t = 0; t < NIN; ++t) any_stage |= stg[t];
  __syncthreads();

  // issue the cp.async copies of one tile's staged chunks into buffer `buf`
  auto prefetch = [&](int buf) {
#pragma unroll
    for (int t = 0; t < NIN; ++t) {
      if (!stg[t]) continue;
      const uint32_t n = 1u << a.nlow[t];                 // elements per x
      const uint32_t n16 = (n * sizeof(T)) >> 4;          // 16-byte pieces per x
      T* dst = stage + buf * a.stage_elems + a.stage_off[t];
      for (uint32_t c = tid; c < 2 * n16; c += kBucketThreads) {
        const uint32_t x = c >= n16, piece = c - x * n16;
        const char* src = reinterpret_cast<const char*>(in[t] + pf[t] + (x ? S[t] : (OffT)0)) + piece * 16;
        cp_async16(reinterpret_cast<char*>(dst + x * n) + piece * 16, src);
      }
    }
    cp_async_commit();
  };
  int buf = 0;
  if (any_stage && t0 < t1) prefetch(0);

  for (uint64_t tile = t0; tile < t1; ++tile) {
    const uint64_t base = ptile << TB;
    const int r = __ffsll((long long)~tile) - 1;     // tile -> tile + 1: clear r ones, set bit r
    const bool has_next = tile + 1 < t1;
    bool same = true;                                 // next tile's staged chunks == current ones
    if (any_stage) {
      if (has_next) {
#pragma unroll
        for (int t = 0; t < NIN; ++t)
          if (stg[t]) same &= (fbit[t][r] == fcum[t][r]);
        if (!same) {
#pragma unroll
          for (int t = 0; t < NIN; ++t) pf[t] = pf[t] + fbit[t][r] - fcum[t][r];
          prefetch(buf ^ 1);
          cp_async_wait<1>();
        } else {
          cp_async_wait<0>();
        }
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();
    }
    const T* sb = stage + buf * a.stage_elems;
    // tile constants: product of the CONST inputs for x = 0 and x = 1
    T C0 = cfrom<T>(1.0, 0.0), C1 = cfrom<T>(1.0, 0.0);
    bool has_c = false;
#pragma unroll
    for (int t = 0; t < NIN; ++t) {
      if (mode[t] == M_CONST) {
        const T c0 = __ldg(in[t] + cur[t]);
        const T c1 = __ldg(in[t] + cur[t] + S[t]);
        if (!has_c) { C0 = c0; C1 = c1; has_c = true; }
        else { C0 = cmul(C0, c0); C1 = cmul(C1, c1); }
      }
    }
#pragma unroll 2
    for (int kk = 0; kk < kBucketIters; ++kk) {
      const uint64_t o = base + (uint64_t)kk * STRIDE + (uint64_t)tid * VEC;
      if (o >= n_out) break;
      if constexpr (VEC == 2) {
        float2 p0[2], p1[2];
        bool first = !has_c;
        p0[0] = p0[1] = reinterpret_cast<const float2&>(C0);
        p1[0] = p1[1] = reinterpret_cast<const float2&>(C1);
#pragma unroll
        for (int t = 0; t < NIN; ++t) {
          if (mode[t] == M_CONST) continue;
          float2 x0[2], x1[2];
          if (stg[t]) {
            const uint32_t off = (uint32_t)(thr[t] + kofs[t][kk]);
            const float2* p = reinterpret_cast<const float2*>(sb + a.stage_off[t]);
            const uint32_t n = 1u << a.nlow[t];
            if (mode[t] == M_VEC) {
              const float4 u0 = *reinterpret_cast<const float4*>(p + off);
              const float4 u1 = *reinterpret_cast<const float4*>(p + n + off);
              x0[0] = make_float2(u0.x, u0.y); x0[1] = make_float2(u0.z, u0.w);
              x1[0] = make_float2(u1.x, u1.y); x1[1] = make_float2(u1.z, u1.w);
            } else if (mode[t] == M_BCAST) {
              x0[0] = x0[1] = p[off];
              x1[0] = x1[1] = p[n + off];
            } else {
              x0[0] = p[off]; x0[1] = p[off + s1v[t]];
              x1[0] = p[n + off]; x1[1] = p[n + off + s1v[t]];
            }
          } else {
            const OffT off = cur[t] + thr[t] + kofs[t][kk];
            const float2* pt = reinterpret_cast<const float2*>(in[t]);
            if (mode[t] == M_VEC) {
              const float4 u0 = ld_in4(reinterpret_cast<const float4*>(pt + off), strm[t]);
              const float4 u1 = ld_in4(reinterpret_cast<const float4*>(pt + off + S[t]), strm[t]);
              x0[0] = make_float2(u0.x, u0.y); x0[1] = make_float2(u0.z, u0.w);
              x1[0] = make_float2(u1.x, u1.y); x1[1] = make_float2(u1.z, u1.w);
            } else if (mode[t] == M_BCAST) {
              x0[0] = x0[1] = ld_in(pt + off, strm[t]);
              x1[0] = x1[1] = ld_in(pt + off + S[t], strm[t]);
            } else {
              x0[0] = ld_in(pt + off, strm[t]);
              x0[1] = ld_in(pt + off + s1v[t], strm[t]);
              x1[0] = ld_in(pt + off + S[t], strm[t]);
              x1[1] = ld_in(pt + off + s1v[t] + S[t], strm[t]);
            }
          }
          if (first) {
            p0[0] = x0[0]; p0[1] = x0[1]; p1[0] = x1[0]; p1[1] = x1[1];
            first = false;
          } else {
            p0[0] = cmul(p0[0], x0[0]); p0[1] = cmul(p0[1], x0[1]);
            p1[0] = cmul(p1[0], x1[0]); p1[1] = cmul(p1[1], x1[1]);
          }
        }
        const float2 r0 = cadd(p0[0], p1[0]), r1 = cadd(p0[1], p1[1]);
        __stcs(reinterpret_cast<float4*>(out + o), make_float4(r0.x, r0.y, r1.x, r1.y));
      } else {
        T p0 = C0, p1 = C1;
        bool first = !has_c;
#pragma unroll
        for (int t = 0; t < NIN; ++t) {
          if (mode[t] == M_CONST) continue;
          T x0, x1;
          if (stg[t]) {
            const uint32_t off = (uint32_t)(thr[t] + kofs[t][kk]);
            const T* p = sb + a.stage_off[t];
            x0 = p[off];
            x1 = p[(1u << a.nlow[t]) + off];
          } else {
            const OffT off = cur[t] + thr[t] + kofs[t][kk];
            x0 = ld_in(in[t] + off, strm[t]);
            x1 = ld_in(in[t] + off + S[t], strm[t]);
          }
          if (first) { p0 = x0; p1 = x1; first = false; }
          else { p0 = cmul(p0, x0); p1 = cmul(p1, x1); }
        }
        __stcs(out + o, cadd(p0, p1));
      }
    }
    if (any_stage) {
      __syncthreads();   // all reads of `buf` done before it is refilled
      if (has_next && !same) buf ^= 1;
    }
#pragma unroll
    for (int t = 0; t < NIN; ++t) cur[t] = cur[t] + fbit[t][r] - fcum[t][r];
    ptile = ptile + pbit[r] - pcum[r];
  }
}

// ------------------------------------------------------------------ specialised bucket group
// One launch eliminates a block of M consecutive indices x = (v_s .. v_{s+M-1}) (M = 1: a single
// bucket step; M > 1: a merge step fused with the in-place reduce steps that follow it -- exact
// re-association of the same sum):
//     out[o] = sum_{x < 2^M} prod_t in_t[F_t(o) + G_t(x)],   F_t(o) = ins0(pext(o, mask_t), pv_t)
// with G_t(x) host-computed tables (kernel parameters -> constant bank, compile-time indexed).
// Host-classified inputs (runtime.cu try_launch_group):
//   dir[0..NDIR)  hold output bit 0 at position 0 -> 16-byte global loads (evict-first if read once)
//   stg[0..NSTG)  hold SOME low tile bits at their lowest positions -> per-tile chunks (one per
//                 distinct x-part) staged in shared memory by cp.async one tile ahead
//   cst[0..nc)    hold NO low tile bit -> C[x] = prod_cst in_t[cur_t + G_t(x)] once per tile
// The inner loops have no per-input branches.
constexpr int kMaxGroup = 5;
struct GArgs {
  void* out;
  const void* in[kMaxIn];              // order: dir..., stg..., cst...
  uint64_t out_mask[kMaxIn];           // output bits present (relative to the group output)
  uint64_t gx[kMaxIn][1 << kMaxGroup]; // element offset of the x-part of input t for x
  uint32_t sx[kMaxIn][1 << kMaxGroup]; // staged: smem element offset of x's chunk (buffer 0)
  uint8_t rep[kMaxIn][1 << kMaxGroup]; // staged: an x for each distinct part (prefetch source)
  uint32_t nparts[kMaxIn];             // staged: distinct x-parts
  uint32_t nlow[kMaxIn];               // staged: log2 chunk
  uint32_t pv[kMaxIn];
  uint32_t stream[kMaxIn];
  uint32_t stage_elems;
  int32_t nc;
  int32_t out_rank;
  uint8_t perm[64];
};

// NDIR direct inputs: the first NDV use 16-byte vector loads (output bit 0 at their position
// 0), the remaining NDIR - NDV use two 8-byte loads (offsets p and p + F_t(1); F_t(1) = 0 when
// they lack output bit 0, i.e. one value serves both elements)
template <typename T, typename OffT, int NDIR, int NSTG, int M, int NDV>
__global__ void __launch_bounds__(kBucketThreads, (M >= 3 ? 2 : 4)) k_group_t(const GArgs a) {
  constexpr int VEC = VecT<T>::n;
  constexpr int TB = TileBits<T>::v;
  constexpr int STRIDE = kBucketThreads * VEC;
  constexpr uint64_t TILE = 1ull << TB;
  constexpr int NB = 64 - TB;
  constexpr int NV = NDIR + NSTG;
  constexpr int NX = 1 << M;
  const int nin = NV + a.nc;
  const uint64_t n_out = 1ull << a.out_rank;
  const uint64_t n_tiles = (n_out + TILE - 1) >> TB;
  const uint32_t tid = threadIdx.x;
  extern __shared__ __align__(16) unsigned char dsm[];
  T* stage = reinterpret_cast<T*>(dsm);

  __shared__ OffT kofs[NV][kBucketIters];
  __shared__ OffT fbit[kMaxIn][NB];
  __shared__ OffT fcum[kMaxIn][NB + 1];
  __shared__ uint64_t pbit[NB], pcum[NB + 1];
  __shared__ T Cs[2][NX];
  if (tid < NV * kBucketIters) {
    const int t = tid / kBucketIters, kk = tid % kBucketIters;
    kofs[t][kk] = (OffT)fmap((uint64_t)kk * STRIDE, a.out_mask[t], a.pv[t]);
  }
  for (int i = tid; i < nin * NB; i += kBucketThreads) {
    const int t = i / NB, b = i % NB;
    fbit[t][b] = (OffT)fmap(1ull << (TB + a.perm[b]), a.out_mask[t], a.pv[t]);
  }
  for (int b = tid; b < NB; b += kBucketThreads) pbit[b] = 1ull << a.perm[b];
  __syncthreads();
  const int nbu = min(NB - 1, max(0, (int)a.out_rank - TB));   // tile-index bits in use
  if (tid < (uint32_t)nin) {
    OffT c = 0;
    fcum[tid][0] = 0;
    for (int b = 0; b < nbu; ++b) { c += fbit[tid][b]; fcum[tid][b + 1] = c; }
  }
  if (tid == (uint32_t)nin) {
    uint64_t c = 0;
    pcum[0] = 0;
    for (int b = 0; b < nbu; ++b) { c += pbit[b]; pcum[b + 1] = c; }
  }
  const uint64_t per = (n_tiles + gridDim.x - 1) / gridDim.x;
  const uint64_t t0 = (uint64_t)blockIdx.x * per;
  const uint64_t t1 = t0 + per < n_tiles ? t0 + per : n_tiles;
  uint64_t ptile = 0;
  for (int b = 0; b < NB && (t0 >> b); ++b)
    if ((t0 >> b) & 1) ptile |= 1ull << a.perm[b];

  OffT thr[NV], cur[NV];
  OffT curc[kMaxIn];
  OffT s1v[NSTG > 0 ? NSTG : 1];
  OffT d1v[NDIR > 0 ? NDIR : 1];
#pragma unroll
  for (int t = 0; t < NDIR; ++t) d1v[t] = (OffT)fmap(1, a.out_mask[t], a.pv[t]);
#pragma unroll
  for (int t = 0; t < NV; ++t) {
    thr[t] = (OffT)fmap((uint64_t)tid * VEC, a.out_mask[t], a.pv[t]);
    cur[t] = (OffT)fmap(ptile << TB, a.out_mask[t], a.pv[t]);
  }
#pragma unroll
  for (int u = 0; u < NSTG; ++u) s1v[u] = (OffT)fmap(1, a.out_mask[NDIR + u], a.pv[NDIR + u]);
  for (int t = NV; t < nin; ++t) curc[t] = (OffT)fmap(ptile << TB, a.out_mask[t], a.pv[t]);
  OffT pf[NSTG > 0 ? NSTG : 1];
#pragma unroll
  for (int u = 0; u < NSTG; ++u) pf[u] = cur[NDIR + u];
  T* out = static_cast<T*>(a.out);
  __syncthreads();

  auto prefetch = [&](int buf) {
#pragma unroll
    for (int u = 0; u < NSTG; ++u) {
      const int t = NDIR + u;
      const uint32_t n = 1u << a.nlow[t];
      const uint32_t n16 = (n * sizeof(T)) >> 4;
      T* dst = stage + buf * a.stage_elems;
      const T* src = static_cast<const T*>(a.in[t]) + pf[u];
      const uint32_t total = a.nparts[t] * n16;
      for (uint32_t c = tid; c < total; c += kBucketThreads) {
        const uint32_t part = c / n16, piece = c - part * n16;
        const uint32_t xr = a.rep[t][part];
        cp_async16(reinterpret_cast<char*>(dst + a.sx[t][xr]) + piece * 16,
                   reinterpret_cast<const char*>(src + (OffT)a.gx[t][xr]) + piece * 16);
      }
    }
    cp_async_commit();
  };
  int buf = 0, cb = 0;
  if (NSTG > 0 && t0 < t1) prefetch(0);

  for (uint64_t tile = t0; tile < t1; ++tile) {
    const uint64_t base = ptile << TB;
    const int r = __ffsll((long long)~tile) - 1;
    const bool has_next = tile + 1 < t1;
    // per-tile constants C[x]
    if (tid < (uint32_t)NX) {
      T c = cfrom<T>(1.0, 0.0);
      for (int t = NV; t < nin; ++t)
        c = cmul(c, __ldg(static_cast<const T*>(a.in[t]) + curc[t] + (OffT)a.gx[t][tid]));
      Cs[cb][tid] = c;
    }
    bool same = true;
    if (NSTG > 0) {
      if (has_next) {
#pragma unroll
        for (int u = 0; u < NSTG; ++u) same &= (fbit[NDIR + u][r] == fcum[NDIR + u][r]);
        if (!same) {
#pragma unroll
          for (int u = 0; u < NSTG; ++u) pf[u] = pf[u] + fbit[NDIR + u][r] - fcum[NDIR + u][r];
          prefetch(buf ^ 1);
          cp_async_wait<1>();
        } else {
          cp_async_wait<0>();
        }
      } else {
        cp_async_wait<0>();
      }
    }
    __syncthreads();
    const T* sb = stage + buf * a.stage_elems;
    OffT db[NDIR > 0 ? NDIR : 1];
#pragma unroll
    for (int t = 0; t < NDIR; ++t) db[t] = cur[t] + thr[t];
    constexpr int KU = (M == 1) ? 2 : 1;
#pragma unroll KU
    for (int kk = 0; kk < kBucketIters; ++kk) {
      const uint64_t o = base + (uint64_t)kk * STRIDE + (uint64_t)tid * VEC;
      if (o >= n_out) break;
      if constexpr (VEC == 2) {
        float2 acc_a = make_float2(0.f, 0.f), acc_b = make_float2(0.f, 0.f);
        // x-rows in batches of XB: every direct (global) load of a batch is issued before the math
        // that consumes it, so up to NDIR x XB 16-byte loads per thread are in flight
        constexpr int XB = NX < 8 ? NX : 8;
#pragma unroll 1
        for (int x0 = 0; x0 < NX; x0 += XB) {
          float4 ld[NDIR > 0 ? NDIR : 1][XB];
#pragma unroll
          for (int xb = 0; xb < XB; ++xb)
#pragma unroll
            for (int t = 0; t < NDIR; ++t) {
              const float2* q = static_cast<const float2*>(a.in[t]) + (db[t] + kofs[t][kk] + (OffT)a.gx[t][x0 + xb]);
              if (t < NDV) {
                ld[t][xb] = a.stream[t] ? __ldcs(reinterpret_cast<const float4*>(q)) : __ldg(reinterpret_cast<const float4*>(q));
              } else {
                const float2 u0 = __ldg(q), u1 = __ldg(q + d1v[t]);
                ld[t][xb] = make_float4(u0.x, u0.y, u1.x, u1.y);
              }
            }
#pragma unroll
          for (int xb = 0; xb < XB; ++xb) {
          const int x = x0 + xb;
          float2 pa, pb;
#pragma unroll
          for (int t = 0; t < NDIR; ++t) {
            const float2 xa = make_float2(ld[t][xb].x, ld[t][xb].y), xb2 = make_float2(ld[t][xb].z, ld[t][xb].w);
            if (t == 0) { pa = xa; pb = xb2; } else { pa = cmul(pa, xa); pb = cmul(pb, xb2); }
          }
#pragma unroll
          for (int u = 0; u < NSTG; ++u) {
            const int t = NDIR + u;
            const float2* p = reinterpret_cast<const float2*>(sb + a.sx[t][x]) + (thr[t] + kofs[t][kk]);
            const float2 xa = p[0], xb2 = p[s1v[u]];
            if (NDIR == 0 && u == 0) { pa = xa; pb = xb2; } else { pa = cmul(pa, xa); pb = cmul(pb, xb2); }
          }
          const float2 c = reinterpret_cast<const float2&>(Cs[cb][x]);
          acc_a = cadd(acc_a, cmul(pa, c));
          acc_b = cadd(acc_b, cmul(pb, c));
          }
        }
        __stcs(reinterpret_cast<float4*>(out + o), make_float4(acc_a.x, acc_a.y, acc_b.x, acc_b.y));
      } else {
        T acc = cfrom<T>(0.0, 0.0);
#pragma unroll
        for (int x = 0; x < NX; ++x) {
          T pr;
#pragma unroll
          for (int t = 0; t < NDIR; ++t) {
            const T* pt = static_cast<const T*>(a.in[t]) + (db[t] + kofs[t][kk] + (OffT)a.gx[t][x]);
            const T v = __ldg(pt);
            if (t == 0) pr = v; else pr = cmul(pr, v);
          }
#pragma unroll
          for (int u = 0; u < NSTG; ++u) {
            const int t = NDIR + u;
            const T v = sb[a.sx[t][x] + thr[t] + kofs[t][kk]];
            if (NDIR == 0 && u == 0) pr = v; else pr = cmul(pr, v);
          }
          acc = cadd(acc, cmul(pr, Cs[cb][x]));
        }
        __stcs(out + o, acc);
      }
    }
    if (NSTG > 0) {
      __syncthreads();
      if (has_next && !same) buf ^= 1;
    }
    cb ^= 1;
#pragma unroll
    for (int t = 0; t < NV; ++t) cur[t] = cur[t] + fbit[t][r] - fcum[t][r];
    for (int t = NV; t < nin; ++t) curc[t] = curc[t] + fbit[t][r] - fcum[t][r];
    ptile = ptile + pbit[r] - pcum[r];
  }
}

// ------------------------------------------------------------------ register-blocked pair group
// A fused group whose varying inputs are exactly two tensors A and B is a batched complex GEMM
// with K = 2^M: out[o] = sum_x C[x] A[F_A(o) + G_A(x)] B[F_B(o) + G_B(x)], C[x] the
// per-tile product of the constant inputs.  Per tile (2^kPairTB outputs) the A and B chunks
// (one per distinct x-part) are staged in shared memory with cp.async (double buffer); every
// thread computes a 2x2 register block: outputs o, o + 2^rb, o + 2^ra, o + 2^ra + 2^rb where ra is
// a tile bit held by A only and rb one held by B only, so each loaded A value feeds two outputs
// and each B value two: per x, 4 shared loads + 2 cmul (A x C) + 4 complex FMA for 4 outputs.
constexpr int kPairTB = 10;
struct PArgs {
  void* out;
  const void* in[2];                   // A, B
  uint64_t mask[2];
  uint32_t pv[2];
  uint64_t gx[2][1 << kMaxGroup];      // global element offset of the x-part
  uint32_t sx[2][1 << kMaxGroup];      // staged chunk offset (buffer-relative)
  uint8_t rep[2][1 << kMaxGroup];
  uint32_t nparts[2], nlow[2];
  uint32_t stage_elems;
  const void* cin[kMaxIn];             // constant inputs
  uint64_t cmask[kMaxIn];
  uint32_t cpv[kMaxIn];
  uint64_t cgx[kMaxIn][1 << kMaxGroup];
  int32_t nc;
  int32_t out_rank;
  uint32_t ra, rb;                     // block bits (< kPairTB)
  uint32_t tbits[8];                   // tile bits taken from the thread index, ascending
  uint8_t perm[64];
};

template <typename T, typename OffT, int M>
__global__ void __launch_bounds__(kBucketThreads, 2) k_pair(const PArgs a) {
  constexpr int TB = kPairTB;
  constexpr uint64_t TILE = 1ull << TB;
  constexpr int NB = 64 - TB;
  constexpr int NX = 1 << M;
  const int nin = 2 + a.nc;
  const uint64_t n_out = 1ull << a.out_rank;
  const uint64_t n_tiles = (n_out + TILE - 1) >> TB;
  const uint32_t tid = threadIdx.x;
  extern __shared__ __align__(16) unsigned char dsm[];
  T* stage = reinterpret_cast<T*>(dsm);
  __shared__ OffT fbit[2 + kMaxIn][NB];
  __shared__ OffT fcum[2 + kMaxIn][NB + 1];
  __shared__ uint64_t pbit[NB], pcum[NB + 1];
  __shared__ T Cs[2][NX];
  auto mask_of = [&](int t) { return t < 2 ? a.mask[t] : a.cmask[t - 2]; };
  auto pv_of = [&](int t) { return t < 2 ? a.pv[t] : a.cpv[t - 2]; };
  for (int i = tid; i < nin * NB; i += kBucketThreads) {
    const int t = i / NB, b = i % NB;
    fbit[t][b] = (OffT)fmap(1ull << (TB + a.perm[b]), mask_of(t), pv_of(t));
  }
  for (int b = tid; b < NB; b += kBucketThreads) pbit[b] = 1ull << a.perm[b];
  __syncthreads();
  const int nbu = min(NB - 1, max(0, (int)a.out_rank - TB));   // tile-index bits in use
  if (tid < (uint32_t)nin) {
    OffT c = 0;
    fcum[tid][0] = 0;
    for (int b = 0; b < nbu; ++b) { c += fbit[tid][b]; fcum[tid][b + 1] = c; }
  }
  if (tid == (uint32_t)nin) {
    uint64_t c = 0;
    pcum[0] = 0;
    for (int b = 0; b < nbu; ++b) { c += pbit[b]; pcum[b + 1] = c; }
  }
  const uint64_t per = (n_tiles + gridDim.x - 1) / gridDim.x;
  const uint64_t t0 = (uint64_t)blockIdx.x * per;
  const uint64_t t1 = t0 + per < n_tiles ? t0 + per : n_tiles;
  uint64_t ptile = 0;
  for (int b = 0; b < NB && (t0 >> b); ++b)
    if ((t0 >> b) & 1) ptile |= 1ull << a.perm[b];
  // this thread's four outputs inside a tile and their chunk offsets
  uint32_t ol = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) ol |= ((tid >> i) & 1u) << a.tbits[i];
  const uint32_t oA = (uint32_t)fmap(ol, a.mask[0], a.pv[0]);
  const uint32_t oB = (uint32_t)fmap(ol, a.mask[1], a.pv[1]);
  const uint32_t dA = (uint32_t)fmap(1ull << a.ra, a.mask[0], a.pv[0]);
  const uint32_t dB = (uint32_t)fmap(1ull << a.rb, a.mask[1], a.pv[1]);
  const uint64_t sa = 1ull << a.ra, sbit = 1ull << a.rb;
  OffT cur[2], curc[kMaxIn];
  for (int t = 0; t < nin; ++t) {
    const OffT v = (OffT)fmap(ptile << TB, mask_of(t), pv_of(t));
    if (t < 2) cur[t] = v; else curc[t - 2] = v;
  }
  OffT pf[2] = {cur[0], cur[1]};
  T* out = static_cast<T*>(a.out);
  __syncthreads();

  auto prefetch = [&](int buf) {
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const uint32_t n = 1u << a.nlow[u];
      const uint32_t n16 = (n * sizeof(T)) >> 4;
      T* dst = stage + buf * a.stage_elems;
      const T* src = static_cast<const T*>(a.in[u]) + pf[u];
      const uint32_t total = a.nparts[u] * n16;
      for (uint32_t c = tid; c < total; c += kBucketThreads) {
        const uint32_t part = c / n16, piece = c - part * n16;
        const uint32_t xr = a.rep[u][part];
        cp_async16(reinterpret_cast<char*>(dst + a.sx[u][xr]) + piece * 16,
                   reinterpret_cast<const char*>(src + (OffT)a.gx[u][xr]) + piece * 16);
      }
    }
    cp_async_commit();
  };
  int buf = 0, cb = 0;
  if (t0 < t1) prefetch(0);
  for (uint64_t tile = t0; tile < t1; ++tile) {
    const uint64_t base = ptile << TB;
    const int r = __ffsll((long long)~tile) - 1;
    const bool has_next = tile + 1 < t1;
    if (tid < (uint32_t)NX) {
      T c = cfrom<T>(1.0, 0.0);
      for (int t = 0; t < a.nc; ++t)
        c = cmul(c, __ldg(static_cast<const T*>(a.cin[t]) + curc[t] + (OffT)a.cgx[t][tid]));
      Cs[cb][tid] = c;
    }
    bool same = true;
    if (has_next) {
      same = (fbit[0][r] == fcum[0][r]) && (fbit[1][r] == fcum[1][r]);
      if (!same) {
        pf[0] = pf[0] + fbit[0][r] - fcum[0][r];
        pf[1] = pf[1] + fbit[1][r] - fcum[1][r];
        prefetch(buf ^ 1);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const T* sb = stage + buf * a.stage_elems;
    T acc00 = cfrom<T>(0.0, 0.0), acc01 = acc00, acc10 = acc00, acc11 = acc00;
    constexpr int XU = NX < 8 ? NX : 8;
#pragma unroll XU
    for (int x = 0; x < NX; ++x) {
      const T c = Cs[cb][x];
      const T* pa = sb + a.sx[0][x] + oA;
      const T* pb = sb + a.sx[1][x] + oB;
      const T a0 = cmul(pa[0], c), a1 = cmul(pa[dA], c);
      const T b0 = pb[0], b1 = pb[dB];
      acc00 = cadd(acc00, cmul(a0, b0));
      acc01 = cadd(acc01, cmul(a0, b1));
      acc10 = cadd(acc10, cmul(a1, b0));
      acc11 = cadd(acc11, cmul(a1, b1));
    }
    const uint64_t o = base + ol;
    if (o < n_out) {
      __stcs(out + o, acc00);
      __stcs(out + o + sbit, acc01);
      __stcs(out + o + sa, acc10);
      __stcs(out + o + sa + sbit, acc11);
    }
    __syncthreads();
    if (has_next && !same) buf ^= 1;
    cb ^= 1;
    cur[0] = cur[0] + fbit[0][r] - fcum[0][r];
    cur[1] = cur[1] + fbit[1][r] - fcum[1][r];
    for (int t = 0; t < a.nc; ++t) curc[t] = curc[t] + fbit[2 + t][r] - fcum[2 + t][r];
    ptile = ptile + pbit[r] - pcum[r];
  }
}

// ------------------------------------------------------------------ register-blocked GEMM group
// k_gemm: a fused group (or single step) whose varying inputs are exactly two tensors A and B is a
// batched complex GEMM with K = 2^M:
//     out[o] = sum_{x < K} C[x] A[F_A(o) + G_A(x)] B[F_B(o) + G_B(x)]
// Output bits are of class a (in A only), b (in B only), c (in both: the batch).  A CTA tile is a
// set of TB = 5 + WB + RAB + RBB output bits chosen by the host (launch_gemm.cu try_launch_gemm):
//   tile-local bits 0..4  = output bits 0..4 (lanes: every warp store is 256 contiguous bytes),
//   tile-local bits 5..   = WB more output bits (the 2^WB warps), preferably of class a / b,
//   tile-local bits 8..   = RAB a-bits and RBB b-bits: each thread owns a 2^RAB x 2^RBB register
//                           block, so every A value feeds 2^RBB outputs and every B value 2^RAB.
// Per tile the A and B chunks (every x-row, every tile bit the input holds) are copied to shared
// memory with cp.async one tile ahead (double buffer per input; a chunk that does not change
// between consecutive tiles is not reloaded).  The tile-constant factor C[x] (inputs without tile
// bits) multiplies the B values.  Complex multiply-adds use packed FP32x2 FMAs (FFMA2: one complex
// MAC = 2 instructions).  Output written once with streaming stores.
constexpr int kGemmMaxTB = 16;
struct MArgs {
  void* out;
  const void* in[2];                   // A, B
  uint64_t mask[2];                    // F_t(o) = ins0(pext(o, mask_t), pv_t)
  uint32_t pv[2];
  uint32_t rowoff[2][1 << kMaxGroup];  // element offset G_t(x) of chunk row r (distinct x-part)
  uint8_t row[2][1 << kMaxGroup];      // x -> chunk row
  uint32_t nrows[2];
  uint32_t nch[2];                     // tile bits held by the input (chunk row = 2^nch elements)
  uint32_t lv[2];                      // 1: chunk bit 0 is the input's position 0 (16-byte copies)
  uint32_t posoff[2][kGemmMaxTB];      // element offset (within the input) of chunk bit k
  int8_t chbit[2][kGemmMaxTB];         // tile-local bit u -> chunk bit of A / B (-1: absent)
  uint8_t outbit[kGemmMaxTB];          // tile-local bit u -> output bit
  uint32_t sm_in[2][4];                // dynamic smem element offset of ring slot (input, slot)
  int32_t stages;                      // ring slots per input (2..4); lookahead = stages - 1 tiles
  uint32_t sm_dep[2];                  // dynamic smem uint32 offset of the piece offset table (nrows << (nch - lv) entries)
  uint32_t sm_bf_bytes;                // dynamic smem byte offset of the formatted B' chunk (2^M x 2^nch[1] float4)
  int32_t c_tile_dep;                  // a constant input holds an output bit: C changes between tiles
  const void* cin[kMaxIn];             // constant inputs (no tile bit)
  uint64_t cmask[kMaxIn];
  uint32_t cpv[kMaxIn];
  uint32_t cgx[kMaxIn][1 << kMaxGroup];
  int32_t nc;
  int32_t out_rank;
  uint8_t perm[64];                    // logical tile-index bit b -> output bit (traversal order)
};

__device__ __forceinline__ uint64_t f2_pack(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 f2_unpack(uint64_t v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
// acc += a * b (complex, packed FP32x2: ptxas folds the broadcasts / swaps into FFMA2 operand
// modifiers)
__device__ __forceinline__ void cmac2(uint64_t& acc, float2 a, float2 b) {
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(f2_pack(a.x, a.x)), "l"(f2_pack(b.x, b.y)));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(f2_pack(-a.y, a.y)), "l"(f2_pack(b.y, b.x)));
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}

template <int M, int RAB, int RBB, bool HASC, int WB>
__global__ void __launch_bounds__(32 << WB, (WB == 3 ? 2 : 4)) k_gemm(const MArgs a) {
  constexpr int kGemmThreads = 32 << WB;   // 2^WB warps; tile-local bits 5 .. 5+WB-1 on the warps
  constexpr int TL = 5 + WB;               // thread bits of the tile
  constexpr int K = 1 << M, RA = 1 << RAB, RB = 1 << RBB;
  constexpr int TB = TL + RAB + RBB;
  constexpr int NB = 64 - TB;
  const uint32_t tid = threadIdx.x;
  const uint64_t n_tiles = 1ull << (a.out_rank - TB);
  extern __shared__ __align__(16) unsigned char dsm[];
  float2* sm = reinterpret_cast<float2*>(dsm);
  uint32_t* smu = reinterpret_cast<uint32_t*>(dsm);
  __shared__ uint32_t fbit[2 + kMaxIn][NB];
  __shared__ uint32_t fcum[2 + kMaxIn][NB + 1];
  __shared__ uint64_t pbit[NB], pcum[NB + 1];
  __shared__ float2 Cs[K];
  const int nin = 2 + (HASC ? a.nc : 0);
  auto mask_of = [&](int t) { return t < 2 ? a.mask[t] : a.cmask[t - 2]; };
  auto pv_of = [&](int t) { return t < 2 ? a.pv[t] : a.cpv[t - 2]; };
  const int nperm = a.out_rank - TB;
  for (int i = tid; i < nin * NB; i += kGemmThreads) {
    const int t = i / NB, b = i % NB;
    fbit[t][b] = b < nperm ? (uint32_t)fmap(1ull << a.perm[b], mask_of(t), pv_of(t)) : 0u;
  }
  for (int b = tid; b < NB; b += kGemmThreads) pbit[b] = b < nperm ? 1ull << a.perm[b] : 0ull;
  // piece offset tables: piece c (2^lv elements) of input u's chunk -> element offset from the
  // tile's base offset (row part G_u(x) + in-row part), so a copy is one shared load + one add
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const uint32_t lp = a.nch[u] - a.lv[u];
    const uint32_t np = a.nrows[u] << lp;
    for (uint32_t c = tid; c < np; c += kGemmThreads) {
      const uint32_t ia = (c & ((1u << lp) - 1u)) << a.lv[u];
      uint32_t off = a.rowoff[u][c >> lp];
      for (uint32_t k = a.lv[u]; k < a.nch[u]; ++k)
        if ((ia >> k) & 1u) off += a.posoff[u][k];
      smu[a.sm_dep[u] + c] = off;
    }
  }
  __syncthreads();
  const int nbu = min(NB - 1, max(0, (int)a.out_rank - TB));   // tile-index bits in use
  if (tid < (uint32_t)nin) {
    uint32_t c = 0;
    fcum[tid][0] = 0;
    for (int b = 0; b < nbu; ++b) { c += fbit[tid][b]; fcum[tid][b + 1] = c; }
  }
  if (tid == (uint32_t)nin) {
    uint64_t c = 0;
    pcum[0] = 0;
    for (int b = 0; b < nbu; ++b) { c += pbit[b]; pcum[b + 1] = c; }
  }
  const uint64_t per = (n_tiles + gridDim.x - 1) / gridDim.x;
  const uint64_t t0 = (uint64_t)blockIdx.x * per;
  const uint64_t t1 = t0 + per < n_tiles ? t0 + per : n_tiles;
  uint64_t obase = 0;
  for (int b = 0; b < nperm && (t0 >> b); ++b)
    if ((t0 >> b) & 1) obase |= 1ull << a.perm[b];
  // this thread's tile-local output offset and chunk indices (lanes + warps), register blocks
  uint64_t othr = 0;
  uint32_t iathr = 0, ibthr = 0;
#pragma unroll
  for (int k = 0; k < TL; ++k) {
    if ((tid >> k) & 1u) {
      othr += 1ull << a.outbit[k];
      if (a.chbit[0][k] >= 0) iathr += 1u << a.chbit[0][k];
      if (a.chbit[1][k] >= 0) ibthr += 1u << a.chbit[1][k];
    }
  }
  uint64_t ora[RA], orb[RB];
  uint32_t iar[RA], ibr[RB];
#pragma unroll
  for (int i = 0; i < RA; ++i) {
    ora[i] = 0; iar[i] = 0;
#pragma unroll
    for (int k = 0; k < RAB; ++k)
      if ((i >> k) & 1) { ora[i] += 1ull << a.outbit[TL + k]; iar[i] += 1u << a.chbit[0][TL + k]; }
  }
#pragma unroll
  for (int j = 0; j < RB; ++j) {
    orb[j] = 0; ibr[j] = 0;
#pragma unroll
    for (int k = 0; k < RBB; ++k)
      if ((j >> k) & 1) { orb[j] += 1ull << a.outbit[TL + RAB + k]; ibr[j] += 1u << a.chbit[1][TL + RAB + k]; }
  }
  uint32_t cur[2], curc[kMaxIn - 2];
#pragma unroll
  for (int u = 0; u < 2; ++u) cur[u] = (uint32_t)fmap(obase, a.mask[u], a.pv[u]);
#pragma unroll
  for (int t = 0; t < kMaxIn - 2; ++t)
    curc[t] = (HASC && t < a.nc) ? (uint32_t)fmap(obase, a.cmask[t], a.cpv[t]) : 0u;
  float2* out = static_cast<float2*>(a.out);
  __syncthreads();

  // cp.async of input u's chunk (all rows) at base offset `base` into buffer `buf`
  auto prefetch = [&](int u, uint32_t base, int slot) {
    const float2* src = static_cast<const float2*>(a.in[u]) + base;
    float2* dst = sm + a.sm_in[u][slot];
    const uint32_t np = a.nrows[u] << (a.nch[u] - a.lv[u]);
    const uint32_t* tab = smu + a.sm_dep[u];
    if (a.lv[u]) {
GEMM_LOOP_PRAGMA
      for (uint32_t c = tid; c < np; c += kGemmThreads) cp_async16(dst + (c << 1), src + tab[c]);
    } else {
GEMM_LOOP_PRAGMA
      for (uint32_t c = tid; c < np; c += kGemmThreads) cp_async8(dst + c, src + tab[c]);
    }
  };
  // S-slot ring per input, lookahead D = S - 1 tiles.  An input's chunk version increments at
  // every tile where its offset changes; version v lives in slot v % S.  At tile t the chunk of
  // tile t + D is issued; the slot it overwrites held version <= ver(t) - 1 (finished).
  const int S = a.stages, D = S - 1;
  int ver[2] = {0, 0}, lver[2] = {0, 0};
  int cslot[2] = {0, 0}, lslot[2] = {0, 0};   // ver % S and lver % S, kept incrementally
  uint32_t lcur[2] = {cur[0], cur[1]};
  uint64_t lt = t0;                     // the lookahead tile (last tile issued)
  if (t0 < t1) { prefetch(0, lcur[0], 0); prefetch(1, lcur[1], 0); }
  cp_async_commit();
  auto advance_lookahead = [&]() {      // issue the chunks of tile lt + 1 (if inside the range)
    if (lt + 1 < t1) {
      const int rr = __ffsll((long long)~lt) - 1;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        if (fbit[u][rr] != fcum[u][rr]) {
          lcur[u] = lcur[u] + fbit[u][rr] - fcum[u][rr];
          ++lver[u];
          lslot[u] = lslot[u] + 1 == S ? 0 : lslot[u] + 1;
          prefetch(u, lcur[u], lslot[u]);
        }
      }
    }
    ++lt;
    cp_async_commit();
  };
  for (int d = 1; d < D; ++d) advance_lookahead();
  float4* bf = reinterpret_cast<float4*>(dsm + a.sm_bf_bytes);   // C-scaled, pre-formatted B chunk
  const uint32_t nB = 1u << a.nch[1];

  int fixed_ver = -1;                   // version of B held (formatted) in bf
  for (uint64_t tile = t0; tile < t1; ++tile) {
    const int r = __ffsll((long long)~tile) - 1;
    // B' is rebuilt only when B's chunk (or a tile-dependent constant factor) changes; the host
    // orders the tile traversal so that consecutive tiles mostly share B
    const bool refix = ver[1] != fixed_ver || a.c_tile_dep;
    if (HASC && refix && tid < (uint32_t)K) {
      float2 c = make_float2(1.f, 0.f);
#pragma unroll
      for (int t = 0; t < kMaxIn - 2; ++t)
        if (t < a.nc) c = cmul(c, __ldg(static_cast<const float2*>(a.cin[t]) + curc[t] + a.cgx[t][tid]));
      Cs[tid] = c;
    }
    if (D <= 1) cp_async_wait<0>(); else if (D == 2) cp_async_wait<1>(); else cp_async_wait<2>();
    __syncthreads();                    // chunks of this tile landed; every thread is past tile - 1
    advance_lookahead();                // tile + D (its slot held a version <= this tile's - 1)
    // B' [x][idx] = C[x] B[row(x)][idx], stored as (re, im, -im, re): a complex multiply-add is
    // then two FFMA2 on operands read straight from shared memory (no register shuffles)
    if (refix) {
      const float2* sBraw = sm + a.sm_in[1][cslot[1]];
GEMM_LOOP_PRAGMA
      for (uint32_t e = tid; e < (uint32_t)K * nB; e += kGemmThreads) {
        const uint32_t x = e >> a.nch[1], idx = e & (nB - 1u);
        float2 b = sBraw[((uint32_t)a.row[1][x] << a.nch[1]) + idx];
        if (HASC) b = cmul(b, Cs[x]);
        bf[e] = make_float4(b.x, b.y, -b.y, b.x);
      }
      fixed_ver = ver[1];
      __syncthreads();
    }
    const float2* sA = sm + a.sm_in[0][cslot[0]] + iathr;
    const float4* sB = bf + ibthr;
    uint64_t acc[RA][RB];
#pragma unroll
    for (int i = 0; i < RA; ++i)
#pragma unroll
      for (int j = 0; j < RB; ++j) acc[i][j] = 0ull;
#pragma unroll
    for (int x = 0; x < K; ++x) {
      const float2* pa = sA + ((uint32_t)a.row[0][x] << a.nch[0]);
      const float4* pb = sB + ((uint32_t)x << a.nch[1]);
      float2 av[RA];
      float4 bv[RB];
#pragma unroll
      for (int i = 0; i < RA; ++i) av[i] = pa[iar[i]];
#pragma unroll
      for (int j = 0; j < RB; ++j) bv[j] = pb[ibr[j]];
#pragma unroll
      for (int i = 0; i < RA; ++i)
#pragma unroll
        for (int j = 0; j < RB; ++j) {
          asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc[i][j]) : "l"(f2_pack(av[i].x, av[i].x)), "l"(f2_pack(bv[j].x, bv[j].y)));
          asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc[i][j]) : "l"(f2_pack(av[i].y, av[i].y)), "l"(f2_pack(bv[j].z, bv[j].w)));
        }
    }
    float2* ot = out + obase + othr;
#pragma unroll
    for (int i = 0; i < RA; ++i)
#pragma unroll
      for (int j = 0; j < RB; ++j) __stcs(ot + ora[i] + orb[j], f2_unpack(acc[i][j]));
#pragma unroll
    for (int u = 0; u < 2; ++u)
      if (fbit[u][r] != fcum[u][r]) {
        ++ver[u];
        cslot[u] = cslot[u] + 1 == S ? 0 : cslot[u] + 1;
      }
    if (HASC && a.c_tile_dep) {            // constants holding output bits (else their offsets stay 0)
#pragma unroll
      for (int t = 0; t < kMaxIn - 2; ++t)
        if (t < a.nc) curc[t] = curc[t] + fbit[2 + t][r] - fcum[2 + t][r];
    }
    obase = obase + pbit[r] - pcum[r];
  }
  cp_async_wait<0>();
}

// ------------------------------------------------------------------ mbarrier helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_cp_async_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred P;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      " @!P bra WAIT_%=;\n}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// ------------------------------------------------------------------ fused reduce chain
// m consecutive reduce steps eliminate the top m bits of A; the weights of step i are rank-1 on
// its summed index.  Re-associated (exact): out[o] = sum_x W[x] A[o + x n_out], W[x] =
// prod_i w_i[bit_{m-1-i}(x)].  A is read once (streaming), out written once; may alias A.
struct ChainArgs {
  void* out;
  const void* A;
  const void* w[kMaxChain][kMaxChainW];
  int32_t nw[kMaxChain];
  int32_t m;
  int32_t out_rank;
  int32_t nv;       // k_chain_split: output vectors per CTA (lanes per row group), 1..32; 0 = min(32, all)
};

template <typename T>
__device__ __forceinline__ void chain_weights(const ChainArgs& a, T* W) {
  const int nx = 1 << a.m;
  for (int x = threadIdx.x; x < nx; x += blockDim.x) {
    T acc = cfrom<T>(1.0, 0.0);
    for (int i = 0; i < a.m; ++i) {
      const int b = (x >> (a.m - 1 - i)) & 1;
      for (int k = 0; k < a.nw[i]; ++k) acc = cmul(acc, static_cast<const T*>(a.w[i][k])[b]);
    }
    W[x] = acc;
  }
}

// small outputs: a CTA takes nv = min(32, n_out / VEC) output vectors and splits the 2^m rows into
// 256 / nv groups (thread t: vector t % nv, group t / nv); the groups' partial sums are combined in
// a fixed order in shared memory.  Every thread of the CTA works even for a 2-element output.
template <typename T>
__global__ void __launch_bounds__(kBucketThreads) k_chain_split(const ChainArgs a) {
  constexpr int VEC = VecT<T>::n;
  __shared__ T W[1 << kMaxChain];
  __shared__ T part[kBucketThreads * VEC];
  chain_weights<T>(a, W);
  __syncthreads();
  const uint64_t n_out = 1ull << a.out_rank;
  const T* A = static_cast<const T*>(a.A);
  T* out = static_cast<T*>(a.out);
  const uint64_t n_vec = (n_out + VEC - 1) / VEC;
  const int nvmax = a.nv > 0 ? a.nv : 32;
  const int nv = (int)(n_vec < (uint64_t)nvmax ? n_vec : (uint64_t)nvmax);
  const int ng = kBucketThreads / nv;
  const int v = threadIdx.x % nv, grp = threadIdx.x / nv;
  const int nx = 1 << a.m;
  const int per = (nx + ng - 1) / ng;
  const int x0 = grp < ng ? grp * per : nx, x1 = min(nx, x0 + per);
  for (uint64_t blk = blockIdx.x; blk * nv < n_vec; blk += gridDim.x) {
    const uint64_t o = (blk * nv + v) * VEC;
    if constexpr (VEC == 2) {
      float2 acc0 = make_float2(0.f, 0.f), acc1 = make_float2(0.f, 0.f);
      if (o + 1 < n_out) {
#pragma unroll 8
        for (int x = x0; x < x1; ++x) {
          const float4 u = __ldcs(reinterpret_cast<const float4*>(A + o + (uint64_t)x * n_out));
          const float2 wv = reinterpret_cast<const float2&>(W[x]);
          acc0.x = fmaf(wv.x, u.x, fmaf(-wv.y, u.y, acc0.x));
          acc0.y = fmaf(wv.x, u.y, fmaf(wv.y, u.x, acc0.y));
          acc1.x = fmaf(wv.x, u.z, fmaf(-wv.y, u.w, acc1.x));
          acc1.y = fmaf(wv.x, u.w, fmaf(wv.y, u.z, acc1.y));
        }
      } else if (o < n_out) {   // a 1-element output (out_rank 0 never reaches a chain; kept safe)
        for (int x = x0; x < x1; ++x) {
          const float2 u = __ldcs(A + o + (uint64_t)x * n_out);
          acc0 = cadd(acc0, cmul(reinterpret_cast<const float2&>(W[x]), u));
        }
      }
      if (grp < ng) {
        part[(grp * nv + v) * 2] = reinterpret_cast<const T&>(acc0);
        part[(grp * nv + v) * 2 + 1] = reinterpret_cast<const T&>(acc1);
      }
    } else {
      T acc = cfrom<T>(0.0, 0.0);
      if (o < n_out) {
#pragma unroll 4
        for (int x = x0; x < x1; ++x) acc = cadd(acc, cmul(W[x], __ldcs(A + o + (uint64_t)x * n_out)));
      }
      if (grp < ng) part[grp * nv + v] = acc;
    }
    __syncthreads();
    if (threadIdx.x < nv * VEC) {
      const uint64_t oo = blk * nv * VEC + threadIdx.x;
      T s = part[threadIdx.x];
      for (int k = 1; k < ng; ++k) s = cadd(s, part[k * nv * VEC + threadIdx.x]);   // fixed order
      if (oo < n_out) out[oo] = s;
    }
    __syncthreads();
  }
}

template <typename T>
__global__ void __launch_bounds__(kBucketThreads) k_chain(const ChainArgs a) {
  constexpr int VEC = VecT<T>::n;
  __shared__ T W[1 << kMaxChain];
  chain_weights<T>(a, W);
  const int nx = 1 << a.m;
  __syncthreads();
  const uint64_t n_out = 1ull << a.out_rank;
  const T* A = static_cast<const T*>(a.A);
  T* out = static_cast<T*>(a.out);
  const uint64_t step = (uint64_t)gridDim.x * blockDim.x * VEC;
  for (uint64_t o = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * VEC; o < n_out; o += step) {
    if constexpr (VEC == 2) {
      float2 acc0 = make_float2(0.f, 0.f), acc1 = make_float2(0.f, 0.f);
#pragma unroll 4
      for (int x = 0; x < nx; ++x) {
        const float4 u = __ldcs(reinterpret_cast<const float4*>(A + o + (uint64_t)x * n_out));
        const float2 w = reinterpret_cast<const float2&>(W[x]);
        acc0.x = fmaf(w.x, u.x, fmaf(-w.y, u.y, acc0.x));
        acc0.y = fmaf(w.x, u.y, fmaf(w.y, u.x, acc0.y));
        acc1.x = fmaf(w.x, u.z, fmaf(-w.y, u.w, acc1.x));
        acc1.y = fmaf(w.x, u.w, fmaf(w.y, u.z, acc1.y));
      }
      __stcs(reinterpret_cast<float4*>(out + o), make_float4(acc0.x, acc0.y, acc1.x, acc1.y));
    } else {
      T acc = cfrom<T>(0.0, 0.0);
#pragma unroll 4
      for (int x = 0; x < nx; ++x) acc = cadd(acc, cmul(W[x], __ldcs(A + o + (uint64_t)x * n_out)));
      __stcs(out + o, acc);
    }
  }
}

// ------------------------------------------------------------------ interpreter (small steps)
constexpr int kProgramThreads = 512;

__device__ __forceinline__ uint64_t slice_offset(uint64_t j, uint32_t slice_mask, uint32_t rank) {
  return slice_mask ? (pext_bits(j, slice_mask) << rank) : 0ull;
}

// rel: element offset added to per-slice tensors (F_REL inputs, every output) -- the window of a
// batched slice; 0 otherwise
template <typename T>
__device__ void run_step(const StepRec& st, T* ws, uint64_t j, uint64_t rel, bool rel_all) {
  const uint64_t n_out = 1ull << st.out_rank;
  T* out = ws + st.out_off + rel;
  const int nin = st.n_in;
  for (uint64_t o = threadIdx.x; o < n_out; o += blockDim.x) {
    T p0 = cfrom<T>(1.0, 0.0), p1 = cfrom<T>(1.0, 0.0);
    for (int t = 0; t < nin; ++t) {
      const InRec& ir = st.in[t];
      const T* base = ws + ir.off + ((rel_all || (ir.flags & F_REL)) ? rel : 0ull) +
                      slice_offset(j, ir.slice_mask, ir.rank);
      const uint64_t off = fmap(o, ir.out_mask, ir.pv);
      const T x0 = base[off];
      const T x1 = base[off + (1ull << ir.pv)];
      if (t == 0) { p0 = x0; p1 = x1; }
      else { p0 = cmul(p0, x0); p1 = cmul(p1, x1); }
    }
    out[o] = cadd(p0, p1);
  }
}

template <typename T>
__device__ double2 final_product(const ScalarRec* scal, int b, int e, const T* ws, uint64_t j,
                                 double log2_scale, uint64_t rel, bool rel_all = false) {
  double re = 1.0, im = 0.0;
  for (int i = b; i < e; ++i) {
    const uint64_t off = scal[i].off + ((rel_all || (scal[i].flags & F_REL)) ? rel : 0ull) +
                         (scal[i].slice_mask ? pext_bits(j, scal[i].slice_mask) : 0);
    const double2 v = to_d2(ws[off]);
    const double nr = re * v.x - im * v.y, ni = re * v.y + im * v.x;
    re = nr;
    im = ni;
  }
  const double s = exp2(log2_scale);
  return make_double2(re * s, im * s);
}

// window of batch member b: b = 0 -> the base arena; b >= 1 -> win0 + (b - 1) * win_elems
__device__ __forceinline__ uint64_t window_rel(uint32_t b, uint64_t win0, uint64_t win_elems) {
  return b == 0 ? 0ull : win0 + (uint64_t)(b - 1) * win_elems;
}

// mode 0: CTA 0 runs steps [begin, end) of the plan (slice j).
// mode 3: CTA i runs step begin + i (the independent steps of one prefix level).
// mode 1: CTA (b, y) runs program b's phase-B steps in window y (parameter set y of a batched
//         energy), then writes its final value to results[y * gridDim.x + b].
// mode 2: CTA b runs program 0's phase-B steps for slice j + b in window b (batched slices) and
//         writes the slice's complex128 result to results[j + b].
template <typename T>
__global__ void __launch_bounds__(kProgramThreads) k_program(const StepRec* __restrict__ steps,
                                                             int begin, int end, T* ws, uint64_t j,
                                                             const ProgramRec* __restrict__ progs,
                                                             const ScalarRec* __restrict__ scal,
                                                             double2* results, int mode,
                                                             uint64_t win0, uint64_t win_elems) {
  int b = begin, e = end;
  uint64_t rel = (mode == 0 || mode == 3) ? win0 : 0ull, jj = j;   // modes 0, 3: win0 = window offset
  if (mode == 3) {   // CTA i runs step begin + i (independent steps of one level)
    b = begin + (int)blockIdx.x;
    e = b + 1;
  }
  const ProgramRec* pr = nullptr;
  if (mode == 1) {
    pr = &progs[blockIdx.x];
    rel = window_rel(blockIdx.y, win0, win_elems);
  } else if (mode == 2) {
    pr = &progs[0];
    rel = window_rel(blockIdx.x, win0, win_elems);
    jj = j + blockIdx.x;
  }
  if (pr) {
    b = pr->stepB_begin;
    e = pr->stepB_end;
  }
  // mode 1 (energy batch): the whole network, leaves included, lives in window y
  for (int s = b; s < e; ++s) {
    run_step<T>(steps[s], ws, jj, rel, mode == 1);
    __syncthreads();
  }
  if (pr && threadIdx.x == 0) {
    const double2 v = final_product<T>(scal, pr->scal_begin, pr->scal_end, ws, jj, pr->log2_scale, rel, mode == 1);
    if (mode == 1) results[(uint64_t)blockIdx.y * gridDim.x + blockIdx.x] = v;
    else results[jj] = v;
  }
}

// energy (§8 a12): one CTA per light cone (x) and angle set (y), as k_program mode 1, with the cone's
// whole arena -- leaves included -- copied into shared memory first, so the ~150-200 small steps of
// a cone read and write shared memory instead of L2 (the host launches it when the largest
// cone arena fits)
template <typename T>
__global__ void __launch_bounds__(kProgramThreads) k_cone_smem(const StepRec* __restrict__ steps,
                                                               const ProgramRec* __restrict__ progs,
                                                               const ScalarRec* __restrict__ scal, const T* ws,
                                                               double2* results, uint64_t win0, uint64_t win_elems) {
  extern __shared__ __align__(16) unsigned char dsm_cone[];
  T* sm = reinterpret_cast<T*>(dsm_cone);
  const ProgramRec& pr = progs[blockIdx.x];
  const uint64_t rel = window_rel(blockIdx.y, win0, win_elems);
  const uint64_t a0 = pr.arena_begin, n = pr.arena_end - pr.arena_begin;
  for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) sm[i] = ws[rel + a0 + i];
  __syncthreads();
  T* base = sm - a0;   // every tensor of the cone at its arena offset
  for (int s = pr.stepB_begin; s < pr.stepB_end; ++s) {
    run_step<T>(steps[s], base, 0, 0ull, true);
    __syncthreads();
  }
  if (threadIdx.x == 0)
    results[(uint64_t)blockIdx.y * gridDim.x + blockIdx.x] =
        final_product<T>(scal, pr.scal_begin, pr.scal_end, base, 0, pr.log2_scale, 0ull, true);
}

// per slice: the product of the final factors in FP64 x 2^{log2_scale}; with open indices (§6)
// thread o computes batch entry o (element pext(o, open_mask) of every factor)
template <typename T>
__global__ void k_finalize(const ScalarRec* __restrict__ scal, int b, int e, const T* ws,
                           uint64_t j, double log2_scale, double* __restrict__ dst, uint64_t rel,
                           int n_open) {
  const uint32_t o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= (1u << n_open)) return;
  double re = 1.0, im = 0.0;
  for (int i = b; i < e; ++i) {
    const ScalarRec& r = scal[i];
    const uint64_t off = r.off + ((r.flags & F_REL) ? rel : 0ull) +
                         (r.slice_mask ? (pext_bits(j, r.slice_mask) << __popc(r.open_mask)) : 0ull) +
                         pext_bits(o, r.open_mask);
    const double2 v = to_d2(ws[off]);
    const double nr = re * v.x - im * v.y, ni = re * v.y + im * v.x;
    re = nr;
    im = ni;
  }
  const double sc = exp2(log2_scale);
  dst[2 * o] = re * sc;
  dst[2 * o + 1] = im * sc;
}

// fixed pairwise tree over j (identical to the host tn_sum_partials); buf[2 (j A + o)], one
// thread per batch entry o
static __global__ void k_pairwise(double* __restrict__ buf, uint64_t n, uint64_t A, double* __restrict__ out) {
  const uint64_t o = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= A) return;
  if (n == 0) { out[2 * o] = out[2 * o + 1] = 0.0; return; }
  uint64_t m = n;
  while (m > 1) {
    uint64_t h = 0;
    for (uint64_t i = 0; i + 1 < m; i += 2, ++h) {
      buf[2 * (h * A + o)] = buf[2 * (i * A + o)] + buf[2 * ((i + 1) * A + o)];
      buf[2 * (h * A + o) + 1] = buf[2 * (i * A + o) + 1] + buf[2 * ((i + 1) * A + o) + 1];
    }
    if (m & 1) {
      buf[2 * (h * A + o)] = buf[2 * ((m - 1) * A + o)];
      buf[2 * (h * A + o) + 1] = buf[2 * ((m - 1) * A + o) + 1];
      ++h;
    }
    m = h;
  }
  out[2 * o] = buf[2 * o];
  out[2 * o + 1] = buf[2 * o + 1];
}

}  // namespace tnb
