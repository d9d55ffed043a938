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

template <typename T>
__global__ void k_materialize(const LeafRec* __restrict__ leaves, int n_leaves, Angles ang,
                              T* __restrict__ ws) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  const int li = idx >> 2, e = idx & 3;
  if (li >= n_leaves) return;
  const LeafRec lr = leaves[li];
  if (e >= (1 << lr.rank)) return;
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
        sincos(ang.beta[l], &s, &c);
        if (e == 0) { fr = c; } else { fr = 0.0; fi = -s; }
        break;
      }
      case LC_ZZ: {
        if (a != b) { double s, c; sincos(ang.gamma[l], &s, &c); fr = c; fi = -s; }
        break;
      }
      case LC_RX: {
        double s, c;
        sincos(ang.beta[l], &s, &c);
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
  ws[lr.off + e] = cfrom<T>(re, im);
}

// ------------------------------------------------------------------ standalone bucket step
struct BigArgs {
  void* out;
  const void* in[kMaxIn];
  uint64_t out_mask[kMaxIn];
  uint32_t pv[kMaxIn];
  uint32_t flags[kMaxIn];
  int32_t out_rank;
  int32_t n_in;
};

template <typename T> struct VecT;
template <> struct VecT<float2> { using type = float4; static constexpr int n = 2; };
template <> struct VecT<double2> { using type = double2; static constexpr int n = 1; };

template <typename T>
__device__ __forceinline__ T ld_in(const T* p, bool stream) {
  return stream ? __ldcs(p) : __ldg(p);
}
__device__ __forceinline__ float4 ld_in4(const float4* p, bool stream) {
  return stream ? __ldcs(p) : __ldg(p);
}

constexpr int kBucketThreads = 256;
constexpr int kBucketIters = 8;

template <typename T, int NIN>
__global__ void __launch_bounds__(kBucketThreads, 4) k_bucket(const BigArgs a) {
  constexpr int VEC = VecT<T>::n;
  constexpr int STRIDE = kBucketThreads * VEC;           // elements per iteration of a CTA
  constexpr int TILE = STRIDE * kBucketIters;            // elements per tile
  const uint64_t n_out = 1ull << a.out_rank;
  const uint64_t n_tiles = (n_out + TILE - 1) / TILE;
  const uint32_t tid = threadIdx.x;

  __shared__ uint64_t kofs[NIN][kBucketIters];
  if (tid < NIN * kBucketIters) {
    const int t = tid / kBucketIters, kk = tid % kBucketIters;
    kofs[t][kk] = fmap((uint64_t)kk * STRIDE, a.out_mask[t], a.pv[t]);
  }
  uint64_t thr[NIN], S[NIN], step1[NIN];
  const T* in[NIN];
  bool strm[NIN];
#pragma unroll
  for (int t = 0; t < NIN; ++t) {
    in[t] = static_cast<const T*>(a.in[t]);
    thr[t] = fmap((uint64_t)tid * VEC, a.out_mask[t], a.pv[t]);
    S[t] = 1ull << a.pv[t];
    step1[t] = fmap(1, a.out_mask[t], a.pv[t]);   // offset of the next output element (VEC = 2)
    strm[t] = (a.flags[t] & 1u) != 0;
  }
  T* out = static_cast<T*>(a.out);
  __syncthreads();

  for (uint64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const uint64_t base = tile * TILE;
    uint64_t tb[NIN];
#pragma unroll
    for (int t = 0; t < NIN; ++t) tb[t] = fmap(base, a.out_mask[t], a.pv[t]) + thr[t];
#pragma unroll 2
    for (int kk = 0; kk < kBucketIters; ++kk) {
      const uint64_t o = base + (uint64_t)kk * STRIDE + (uint64_t)tid * VEC;
      if (o >= n_out) break;
      if constexpr (VEC == 2) {
        float2 p0[2], p1[2];
#pragma unroll
        for (int t = 0; t < NIN; ++t) {
          const uint64_t off = tb[t] + kofs[t][kk];
          const float2* pt = reinterpret_cast<const float2*>(in[t]);
          float2 x0[2], x1[2];
          if (step1[t] == 1) {
            const float4 u0 = ld_in4(reinterpret_cast<const float4*>(pt + off), strm[t]);
            const float4 u1 = ld_in4(reinterpret_cast<const float4*>(pt + off + S[t]), strm[t]);
            x0[0] = make_float2(u0.x, u0.y); x0[1] = make_float2(u0.z, u0.w);
            x1[0] = make_float2(u1.x, u1.y); x1[1] = make_float2(u1.z, u1.w);
          } else if (step1[t] == 0) {
            x0[0] = x0[1] = ld_in(pt + off, strm[t]);
            x1[0] = x1[1] = ld_in(pt + off + S[t], strm[t]);
          } else {
            x0[0] = ld_in(pt + off, strm[t]);
            x0[1] = ld_in(pt + off + step1[t], strm[t]);
            x1[0] = ld_in(pt + off + S[t], strm[t]);
            x1[1] = ld_in(pt + off + step1[t] + S[t], strm[t]);
          }
          if (t == 0) {
            p0[0] = x0[0]; p0[1] = x0[1]; p1[0] = x1[0]; p1[1] = x1[1];
          } else {
            p0[0] = cmul(p0[0], x0[0]); p0[1] = cmul(p0[1], x0[1]);
            p1[0] = cmul(p1[0], x1[0]); p1[1] = cmul(p1[1], x1[1]);
          }
        }
        const float2 r0 = cadd(p0[0], p1[0]), r1 = cadd(p0[1], p1[1]);
        __stcs(reinterpret_cast<float4*>(out + o), make_float4(r0.x, r0.y, r1.x, r1.y));
      } else {
        T p0, p1;
#pragma unroll
        for (int t = 0; t < NIN; ++t) {
          const uint64_t off = tb[t] + kofs[t][kk];
          const T x0 = ld_in(in[t] + off, strm[t]);
          const T x1 = ld_in(in[t] + off + S[t], strm[t]);
          if (t == 0) { p0 = x0; p1 = x1; }
          else { p0 = cmul(p0, x0); p1 = cmul(p1, x1); }
        }
        __stcs(out + o, cadd(p0, p1));
      }
    }
  }
}

// ------------------------------------------------------------------ interpreter (small steps)
constexpr int kProgramThreads = 512;

__device__ __forceinline__ uint64_t slice_offset(uint64_t j, uint32_t slice_mask, uint32_t rank) {
  return slice_mask ? (pext_bits(j, slice_mask) << rank) : 0ull;
}

template <typename T>
__device__ void run_step(const StepRec& st, T* ws, uint64_t j) {
  const uint64_t n_out = 1ull << st.out_rank;
  T* out = ws + st.out_off;
  const int nin = st.n_in;
  for (uint64_t o = threadIdx.x; o < n_out; o += blockDim.x) {
    T p0 = cfrom<T>(1.0, 0.0), p1 = cfrom<T>(1.0, 0.0);
    for (int t = 0; t < nin; ++t) {
      const InRec& ir = st.in[t];
      const T* base = ws + ir.off + slice_offset(j, ir.slice_mask, ir.rank);
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
                                 double log2_scale) {
  double re = ldexp(1.0, 0), im = 0.0;
  for (int i = b; i < e; ++i) {
    const double2 v = to_d2(ws[scal[i].off + (scal[i].slice_mask ? pext_bits(j, scal[i].slice_mask) : 0)]);
    const double nr = re * v.x - im * v.y, ni = re * v.y + im * v.x;
    re = nr;
    im = ni;
  }
  const double s = exp2(log2_scale);
  return make_double2(re * s, im * s);
}

// mode 0: CTA 0 runs steps [begin, end) of the plan.
// mode 1: CTA b runs program b's phase-B steps, then writes its final value to results[b].
template <typename T>
__global__ void __launch_bounds__(kProgramThreads) k_program(const StepRec* __restrict__ steps,
                                                             int begin, int end, T* ws, uint64_t j,
                                                             const ProgramRec* __restrict__ progs,
                                                             const ScalarRec* __restrict__ scal,
                                                             double2* results, int mode) {
  int b = begin, e = end;
  if (mode == 1) {
    const ProgramRec& pr = progs[blockIdx.x];
    b = pr.stepB_begin;
    e = pr.stepB_end;
  }
  for (int s = b; s < e; ++s) {
    run_step<T>(steps[s], ws, j);
    __syncthreads();
  }
  if (mode == 1 && threadIdx.x == 0) {
    const ProgramRec& pr = progs[blockIdx.x];
    results[blockIdx.x] = final_product<T>(scal, pr.scal_begin, pr.scal_end, ws, j, pr.log2_scale);
  }
}

template <typename T>
__global__ void k_finalize(const ScalarRec* __restrict__ scal, int b, int e, const T* ws,
                           uint64_t j, double log2_scale, double* __restrict__ dst) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    const double2 v = final_product<T>(scal, b, e, ws, j, log2_scale);
    dst[0] = v.x;
    dst[1] = v.y;
  }
}

// fixed pairwise tree over j (identical to the host tn_sum_partials)
__global__ void k_pairwise(double* __restrict__ buf, uint64_t n, double* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (n == 0) { out[0] = out[1] = 0.0; return; }
  uint64_t m = n;
  while (m > 1) {
    uint64_t h = 0;
    for (uint64_t i = 0; i + 1 < m; i += 2, ++h) {
      buf[2 * h] = buf[2 * i] + buf[2 * (i + 1)];
      buf[2 * h + 1] = buf[2 * i + 1] + buf[2 * (i + 1) + 1];
    }
    if (m & 1) {
      buf[2 * h] = buf[2 * (m - 1)];
      buf[2 * h + 1] = buf[2 * (m - 1) + 1];
      ++h;
    }
    m = h;
  }
  out[0] = buf[0];
  out[1] = buf[1];
}

}  // namespace tnb
