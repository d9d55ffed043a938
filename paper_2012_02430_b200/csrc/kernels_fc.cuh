// kernels_fc.cuh -- k_gemm_fc: a producer merge group (batched complex GEMM, as k_gemm) whose
// output T is consumed by the next merge group without ever being written (OP_GROUP_FEED).
//
// Producer (steps [b, m)):  T[o, y] = sum_x C1_x A[F_A(o,y) + G_A(x)] B[F_B(o,y) + G_B(x)]
// Consumer (steps [m, e)):  out[o]  = sum_y C3_y X(o, y) T[o, y],   X = product of the consumer's
//                           other inputs that hold output bits (at most 2)
// T is a full input of the consumer: its low R3 bits are the consumer's output bits o, its top M3
// bits the consumer's summed indices y (T[o + G_T(y)]).  Exact re-association of the same sums
// (bucket elimination; the consumer's bucket contains T).
//
// Same tiles as k_gemm over T's bits, with every tile bit an o bit; the tile index runs over the
// M3 y bits first, so 2^M3 consecutive tiles of a CTA share their o part: each thread accumulates
// its register block of out (RA x RB complex) over them and stores it once.  Chunk loading, the
// pre-formatted (Re, Im, -Im, Re) C1-scaled B' and the FFMA2 inner loop are k_gemm's.
#pragma once
#include "kernels.cuh"

#ifndef FC_OCC
#define FC_OCC 2
#endif
#ifndef FC_PREFETCH
#define FC_PREFETCH 0   // prefetch.global.L1 of the consumer factors: no gain in round 1 (0.228 ms either way),
                        // slower in the final state (224.4 vs 209.7 us, C5a 99.0 vs 102.8 /s; session4/fc_prefetch)
#endif
#ifndef FC_XV_AT
#define FC_XV_AT 2   // consumer loads at x = FC_XV_AT * K / 2 (0: before the GEMM, 2: after it; 0 and 1 spill at 4x4)
#endif

#ifndef FC_U1
#define FC_U1 1      // keep the chunk-load and B' rebuild loops rolled: 4,144 vs 6,480 SASS instructions, fewer
                     // instruction-fetch stalls (launch 212 vs 221 us, C5a 101.8 vs 101.1 /s; `profiles/r02/session4/`)
#endif
#if FC_U1
#define FC_LOOP_PRAGMA _Pragma("unroll 1")
#else
#define FC_LOOP_PRAGMA
#endif

namespace tnb {

constexpr int kFcMaxV = 1;   // consumer inputs (besides T) that hold output bits

struct FArgs {
  void* out3;                                  // consumer output (2^R3 elements)
  int32_t M3;                                  // consumer summed indices (y bits of T)
  int32_t nv;                                  // varying consumer inputs (besides T)
  const void* vin[kFcMaxV];
  uint64_t vmask[kFcMaxV];                     // F_v(o) = ins0(pext(o, vmask), vpv)
  uint32_t vpv[kFcMaxV];
  uint32_t vgx[kFcMaxV][1 << kMaxGroup];       // G_v(y)
  int32_t nw;                                  // consumer inputs holding no output bit (weights)
  const void* win[kMaxIn];
  uint32_t wgx[kMaxIn][1 << kMaxGroup];
  uint64_t omask;                              // (1 << R3) - 1: the o part of a T offset
  int32_t xpf;                                 // 1: prefetch the next tile's X lines into L2 (X holds
                                               // output bits 0..4 at its positions 0..4)
  uint32_t* sem;                               // split consumer blocks: one zeroed counter per CTA
                                               // boundary (nullptr: whole blocks per CTA)
};

template <int M, int RAB, int RBB, int WB>
__global__ void __launch_bounds__(32 << WB, (WB == 3 ? FC_OCC : 2 * FC_OCC)) k_gemm_fc(const MArgs a, const FArgs f) {
  constexpr int kThreads = 32 << WB;       // 2^WB warps: tile bits 5 .. 5 + WB - 1 on the warps
  constexpr int TL = 5 + WB;               // 5 lane bits + WB warp bits
  constexpr int K = 1 << M, RA = 1 << RAB, RB = 1 << RBB;
  constexpr int TB = TL + RAB + RBB;
  // consumer loads X at x = XV * K / 2: after the GEMM (2) with 4 x 4 blocks (earlier spills), at
  // the start of the tile (0) with 4 x 2 blocks (the loads then overlap the tile's GEMM)
  constexpr int XV = RBB <= 1 ? 0 : FC_XV_AT;
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
  __shared__ float2 C3s[1 << kMaxGroup];   // product of the consumer's weights per summed value y
  const int nin = 2 + a.nc;
  auto mask_of = [&](int t) { return t < 2 ? a.mask[t] : a.cmask[t - 2]; };
  auto pv_of = [&](int t) { return t < 2 ? a.pv[t] : a.cpv[t - 2]; };
  const int nperm = a.out_rank - TB;
  for (int i = tid; i < nin * NB; i += kThreads) {
    const int t = i / NB, b = i % NB;
    fbit[t][b] = b < nperm ? (uint32_t)fmap(1ull << a.perm[b], mask_of(t), pv_of(t)) : 0u;
  }
  for (int b = tid; b < NB; b += kThreads) pbit[b] = b < nperm ? 1ull << a.perm[b] : 0ull;
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const uint32_t lp = a.nch[u] - a.lv[u];
    const uint32_t np = a.nrows[u] << lp;
    for (uint32_t c = tid; c < np; c += kThreads) {
      const uint32_t ia = (c & ((1u << lp) - 1u)) << a.lv[u];
      uint32_t off = a.rowoff[u][c >> lp];
      for (uint32_t k = a.lv[u]; k < a.nch[u]; ++k)
        if ((ia >> k) & 1u) off += a.posoff[u][k];
      smu[a.sm_dep[u] + c] = off;
    }
  }
  __syncthreads();
  const int nbu = min(NB - 1, max(0, (int)a.out_rank - TB));
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
  uint64_t t0, t1;
  if (f.sem) {
    // balanced contiguous tile ranges (floor partition; >= 2^M3 tiles each, the host keeps grid <=
    // the number of blocks): a consumer output block (2^M3 consecutive tiles) spans at most two
    // CTAs, whose two partial sums meet through sem[boundary] (see the flush below)
    t0 = (uint64_t)blockIdx.x * n_tiles / gridDim.x;
    t1 = ((uint64_t)blockIdx.x + 1) * n_tiles / gridDim.x;
  } else {
    // whole groups of 2^M3 tiles per CTA (a consumer output block is finished inside one CTA)
    const uint64_t n_groups = n_tiles >> f.M3;
    const uint64_t gper = (n_groups + gridDim.x - 1) / gridDim.x;
    t0 = ((uint64_t)blockIdx.x * gper) << f.M3;
    const uint64_t t1e = (((uint64_t)blockIdx.x + 1) * gper) << f.M3;
    t1 = t1e < n_tiles ? t1e : n_tiles;
  }
  __shared__ uint32_t s_arrive;
  uint64_t obase = 0;
  for (int b = 0; b < nperm && (t0 >> b); ++b)
    if ((t0 >> b) & 1) obase |= 1ull << a.perm[b];
  uint32_t othr = 0;                       // tile bits are consumer output bits (< 2^32 elements)
  uint32_t iathr = 0, ibthr = 0;
#pragma unroll
  for (int k = 0; k < TL; ++k) {
    if ((tid >> k) & 1u) {
      othr += 1u << a.outbit[k];
      if (a.chbit[0][k] >= 0) iathr += 1u << a.chbit[0][k];
      if (a.chbit[1][k] >= 0) ibthr += 1u << a.chbit[1][k];
    }
  }
  uint32_t ora[RA], orb[RB];
  uint32_t iar[RA], ibr[RB];
#pragma unroll
  for (int i = 0; i < RA; ++i) {
    ora[i] = 0; iar[i] = 0;
#pragma unroll
    for (int k = 0; k < RAB; ++k)
      if ((i >> k) & 1) { ora[i] += 1u << a.outbit[TL + k]; iar[i] += 1u << a.chbit[0][TL + k]; }
  }
#pragma unroll
  for (int j = 0; j < RB; ++j) {
    orb[j] = 0; ibr[j] = 0;
#pragma unroll
    for (int k = 0; k < RBB; ++k)
      if ((j >> k) & 1) { orb[j] += 1u << a.outbit[TL + RAB + k]; ibr[j] += 1u << a.chbit[1][TL + RAB + k]; }
  }
  // consumer offsets of this thread's outputs (F_v additive over disjoint bits)
  uint32_t vthr[kFcMaxV], va[kFcMaxV][RA], vb[kFcMaxV][RB];
#pragma unroll
  for (int v = 0; v < kFcMaxV; ++v) {
    const bool on = v < f.nv;
    vthr[v] = on ? (uint32_t)fmap(othr, f.vmask[v], f.vpv[v]) : 0u;
#pragma unroll
    for (int i = 0; i < RA; ++i) va[v][i] = on ? (uint32_t)fmap(ora[i], f.vmask[v], f.vpv[v]) : 0u;
#pragma unroll
    for (int j = 0; j < RB; ++j) vb[v][j] = on ? (uint32_t)fmap(orb[j], f.vmask[v], f.vpv[v]) : 0u;
  }
  uint32_t cur[2], curc[kMaxIn - 2];
#pragma unroll
  for (int u = 0; u < 2; ++u) cur[u] = (uint32_t)fmap(obase, a.mask[u], a.pv[u]);
#pragma unroll
  for (int t = 0; t < kMaxIn - 2; ++t) curc[t] = t < a.nc ? (uint32_t)fmap(obase, a.cmask[t], a.cpv[t]) : 0u;
  // X prefetch: a warp's RA x RB consumer loads cover 2 RA RB 128-byte lines of X (lanes = output
  // bits 0..4 = X positions 0..4); lane l < 2 RA RB fetches line l & 1 of load l >> 1 for the next tile
  uint32_t pfo = 0;
  const bool pf_lane = f.xpf && f.nv > 0 && (tid & 31u) < 2u * RA * RB;
  if (pf_lane) {
    const uint32_t q = (tid & 31u) >> 1, i = q / RB, j = q % RB;
    uint32_t o = (othr & ~31u) + ((tid & 1u) << 4);
#pragma unroll
    for (int k = 0; k < RAB; ++k)
      if ((i >> k) & 1) o += 1u << a.outbit[TL + k];
#pragma unroll
    for (int k = 0; k < RBB; ++k)
      if ((j >> k) & 1) o += 1u << a.outbit[TL + RAB + k];
    pfo = (uint32_t)fmap(o, f.vmask[0], f.vpv[0]);
  }
  float2* out3 = static_cast<float2*>(f.out3);
  if (tid < (1u << f.M3)) {
    float2 c3 = make_float2(1.f, 0.f);
    for (int w = 0; w < f.nw; ++w) c3 = cmul(c3, __ldg(static_cast<const float2*>(f.win[w]) + f.wgx[w][tid]));
    C3s[tid] = c3;
  }
  __syncthreads();

  auto prefetch = [&](int u, uint32_t base, int slot) {
    const float2* src = static_cast<const float2*>(a.in[u]) + base;
    float2* dst = sm + a.sm_in[u][slot];
    const uint32_t np = a.nrows[u] << (a.nch[u] - a.lv[u]);
    const uint32_t* tab = smu + a.sm_dep[u];
    if (a.lv[u]) {
FC_LOOP_PRAGMA
      for (uint32_t c = tid; c < np; c += kThreads) cp_async16(dst + (c << 1), src + tab[c]);
    } else {
FC_LOOP_PRAGMA
      for (uint32_t c = tid; c < np; c += kThreads) cp_async8(dst + c, src + tab[c]);
    }
  };
  const int S = a.stages, D = S - 1;
  int ver[2] = {0, 0}, lver[2] = {0, 0};
  int cslot[2] = {0, 0}, lslot[2] = {0, 0};
  uint32_t lcur[2] = {cur[0], cur[1]};
  uint64_t lt = t0;
  if (t0 < t1) { prefetch(0, lcur[0], 0); prefetch(1, lcur[1], 0); }
  cp_async_commit();
  auto advance_lookahead = [&]() {
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
  float4* bf = reinterpret_cast<float4*>(dsm + a.sm_bf_bytes);
  const uint32_t nB = 1u << a.nch[1];
  const uint32_t ymask = (1u << f.M3) - 1u;

  uint64_t oacc[RA][RB];                   // consumer accumulators (packed complex)
  uint64_t acc[RA][RB];                    // the tile's T block
  float2 xv[kFcMaxV][RA][RB];              // consumer factors of the tile (T's partner values)
  float2 c3 = make_float2(0.f, 0.f);
  uint32_t vcur[kFcMaxV];
#pragma unroll
  for (int v = 0; v < kFcMaxV; ++v) vcur[v] = 0u;
  int fixed_ver = -1;
  // consumer: oacc += C3_y X(o, y) T[o, y]
  auto consume = [&]() {
#pragma unroll
    for (int i = 0; i < RA; ++i)
#pragma unroll
      for (int j = 0; j < RB; ++j) {
        float2 xx = c3;
#pragma unroll
        for (int v = 0; v < kFcMaxV; ++v)
          if (v < f.nv) xx = cmul(xx, xv[v][i][j]);
        const float2 tv = f2_unpack(acc[i][j]);
        asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(oacc[i][j]) : "l"(f2_pack(tv.x, tv.x)), "l"(f2_pack(xx.x, xx.y)));
        asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(oacc[i][j]) : "l"(f2_pack(-tv.y, tv.y)), "l"(f2_pack(xx.y, xx.x)));
      }
  };
  // store the consumer block that tile tl (summed value yy, o part ob) ends
  auto flush = [&](uint64_t tl, uint32_t yy, uint32_t ob) {
    float2* ot = out3 + ob + othr;
    if (tl - yy >= t0 && yy == ymask) {    // the whole block ran here: the consumer output is final
#pragma unroll
      for (int i = 0; i < RA; ++i)
#pragma unroll
        for (int j = 0; j < RB; ++j) __stcs(ot + ora[i] + orb[j], f2_unpack(oacc[i][j]));
    } else {
      // a block split between this CTA and its neighbour: out = P_first + P_second, the first
      // arriving CTA stores its partial and publishes it, the second adds its own (float
      // addition commutes, so the bits do not depend on the arrival order)
      uint32_t* sem = f.sem + (tl - yy < t0 ? blockIdx.x : blockIdx.x + 1);
      __syncthreads();
      if (tid == 0) s_arrive = atomicAdd(sem, 1u);
      __syncthreads();
      if (s_arrive == 0u) {
#pragma unroll
        for (int i = 0; i < RA; ++i)
#pragma unroll
          for (int j = 0; j < RB; ++j) __stcg(ot + ora[i] + orb[j], f2_unpack(oacc[i][j]));
        __threadfence();
        __syncthreads();
        if (tid == 0) atomicAdd(sem, 1u);   // published (2 arrivals + 1 publish = 3)
      } else {
        if (tid == 0) {
          while (atomicAdd(sem, 0u) != 3u) __nanosleep(64);
          *sem = 0u;                        // zero again for the next launch (stream-ordered)
        }
        __syncthreads();
        __threadfence();
#pragma unroll
        for (int i = 0; i < RA; ++i)
#pragma unroll
          for (int j = 0; j < RB; ++j) {
            const float2 p = __ldcg(ot + ora[i] + orb[j]);
            const float2 q = f2_unpack(oacc[i][j]);
            __stcs(ot + ora[i] + orb[j], make_float2(p.x + q.x, p.y + q.y));
          }
      }
    }
  };
  // (Software-pipelining the consumer step -- tile t's X loads consumed after the barrier and chunk
  // issue of tile t + 1 -- was measured slower: 128 registers with spills, 225-227 vs 209.5 us.)
  for (uint64_t tile = t0; tile < t1; ++tile) {
    const bool refix = ver[1] != fixed_ver || a.c_tile_dep;
    if (refix && tid < (uint32_t)K) {
      float2 c = make_float2(1.f, 0.f);
#pragma unroll
      for (int t = 0; t < kMaxIn - 2; ++t)
        if (t < a.nc) c = cmul(c, __ldg(static_cast<const float2*>(a.cin[t]) + curc[t] + a.cgx[t][tid]));
      Cs[tid] = c;
    }
    if (D <= 1) cp_async_wait<0>(); else if (D == 2) cp_async_wait<1>(); else cp_async_wait<2>();
    __syncthreads();
    advance_lookahead();
    const int r = __ffsll((long long)~tile) - 1;
    const uint32_t y = (uint32_t)tile & ymask;
    if (y == 0u || tile == t0) {           // a new consumer output block (or this CTA's part of one)
#pragma unroll
      for (int i = 0; i < RA; ++i)
#pragma unroll
        for (int j = 0; j < RB; ++j) oacc[i][j] = 0ull;
      const uint64_t obo = obase & f.omask;
#pragma unroll
      for (int v = 0; v < kFcMaxV; ++v) vcur[v] = v < f.nv ? (uint32_t)fmap(obo, f.vmask[v], f.vpv[v]) : 0u;
    }
    c3 = C3s[y];
    if (pf_lane && y < ymask)              // the next tile (same block, y + 1): its X lines into L2
      asm volatile("prefetch.global.L2 [%0];" ::"l"(static_cast<const float2*>(f.vin[0]) + vcur[0] + pfo + f.vgx[0][y + 1]));
#if FC_PREFETCH
    // the consumer factors of this tile are loaded after its GEMM: pull their lines into L1 now
    // (no registers held; the GEMM covers the latency)
#pragma unroll
    for (int v = 0; v < kFcMaxV; ++v)
      if (v < f.nv) {
        const float2* src = static_cast<const float2*>(f.vin[v]) + vcur[v] + vthr[v] + f.vgx[v][y];
#pragma unroll
        for (int i = 0; i < RA; ++i)
#pragma unroll
          for (int j = 0; j < RB; ++j)
            asm volatile("prefetch.global.L1 [%0];" ::"l"(src + va[v][i] + vb[v][j]));
      }
#endif
    if (refix) {
      const float2* sBraw = sm + a.sm_in[1][cslot[1]];
FC_LOOP_PRAGMA
      for (uint32_t e = tid; e < (uint32_t)K * nB; e += kThreads) {
        const uint32_t x = e >> a.nch[1], idx = e & (nB - 1u);
        float2 b = sBraw[((uint32_t)a.row[1][x] << a.nch[1]) + idx];
        b = cmul(b, Cs[x]);
        bf[e] = make_float4(b.x, b.y, -b.y, b.x);
      }
      fixed_ver = ver[1];
      __syncthreads();
    }
    const float2* sA = sm + a.sm_in[0][cslot[0]] + iathr;
    const float4* sB = bf + ibthr;
#pragma unroll
    for (int i = 0; i < RA; ++i)
#pragma unroll
      for (int j = 0; j < RB; ++j) acc[i][j] = 0ull;
    // the X loads are issued inside the GEMM (4 x 2 blocks: at its start) or after it (4 x 4:
    // earlier spills)
#pragma unroll
    for (int x = 0; x < K; ++x) {
      if (x == (XV * K) / 2) {
#pragma unroll
        for (int v = 0; v < kFcMaxV; ++v)
          if (v < f.nv) {
            const float2* src = static_cast<const float2*>(f.vin[v]) + vcur[v] + vthr[v] + f.vgx[v][y];
#pragma unroll
            for (int i = 0; i < RA; ++i)
#pragma unroll
              for (int j = 0; j < RB; ++j) xv[v][i][j] = __ldg(src + va[v][i] + vb[v][j]);
          }
      }
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
    if (XV == 2) {   // after the GEMM
#pragma unroll
      for (int v = 0; v < kFcMaxV; ++v)
        if (v < f.nv) {
          const float2* src = static_cast<const float2*>(f.vin[v]) + vcur[v] + vthr[v] + f.vgx[v][y];
#pragma unroll
          for (int i = 0; i < RA; ++i)
#pragma unroll
            for (int j = 0; j < RB; ++j) xv[v][i][j] = __ldg(src + va[v][i] + vb[v][j]);
        }
    }
    consume();
    if (y == ymask || tile + 1 == t1)      // last y of the block (or of this CTA's part of it)
      flush(tile, y, (uint32_t)(obase & f.omask));
#pragma unroll
    for (int u = 0; u < 2; ++u)
      if (fbit[u][r] != fcum[u][r]) {
        ++ver[u];
        cslot[u] = cslot[u] + 1 == S ? 0 : cslot[u] + 1;
      }
    if (a.c_tile_dep) {                    // constants holding output bits (else their offsets stay 0)
#pragma unroll
      for (int t = 0; t < kMaxIn - 2; ++t)
        if (t < a.nc) curc[t] = curc[t] + fbit[2 + t][r] - fcum[2 + t][r];
    }
    obase = obase + pbit[r] - pcum[r];
  }
  cp_async_wait<0>();
}

}  // namespace tnb
