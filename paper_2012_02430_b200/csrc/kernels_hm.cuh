// kernels_hm.cuh -- k_gemm_hm: the two-operand merge group of k_gemm (a batched complex GEMM with
// K = 2^M summed values; the re-associated bucket elimination of PAPER.md:361-368)
// on the warp-level tensor cores: mma.sync.m16n8k8 kind tf32 with a 3xTF32 split.
//
//   out[o] = sum_{x < K} C[x] R[F_R(o) + G_R(x)] Q[F_Q(o) + G_Q(x)]
//
// R (the "row" operand) holds >= 4 output bits Q does not hold; Q (the "column" operand) >= 2 bits
// R does not hold.  As a real GEMM per batch (bits held by both):
//   [Re T, Im T][m][2j+f] = sum_{x,e} R'[m][2x+e] Q'[2x+e][2j+f],
//   R'[m][2x+e] = (Re, Im)_e of R[m][x],
//   Q'[2x][2j] = Re q, Q'[2x][2j+1] = Im q, Q'[2x+1][2j] = -Im q, Q'[2x+1][2j+1] = Re q  (q = C[x] Q[x][j]),
// so the MMA's (c0, c1) are (Re, Im) of one complex output.  Every operand value v is split as
// big = v truncated to TF32, small = v - big; D += Rs Qb + Rb Qs + Rb Qb (the dropped Rs Qs term is
// ~2^-20 relative; 3xTF32 measured 7e-7 against 7e-4 for one TF32 product, profiles/r01/tc/NOTES.md).
//
// Why mma.sync and not tcgen05 here: an MMA row of R is a set of R-only output bits whose elements
// are scattered over R's bit order (SURVEY F5 layouts), so each thread gathers its fragment values
// from the shared-memory chunk itself -- the register-fed warp MMA takes any row -> address map,
// while tcgen05 needs canonical shared-memory tiles (the formatting pass that made k_fc_tc / k_gemm_tc
// latency-bound).  What it buys over k_gemm's FFMA2: one HMMA does the work of
// 16 FFMA2 at 3.8x the FP32 FMA rate (scripts/probe/mma_rate.cu), and k_gemm was bound by its
// instruction stream (711 warp instructions per tile, issue 50 %, profiles/r02/hm/).
//
// Tile-local bits (HArgs.outbit order, chosen by launch_gemm_hm.cu):
//   0, 1      tig bits (lane & 3): two Q-only bits = the MMA's complex column within an n8 block
//   2, 3, 4   g bits (lane >> 2): three R-only bits = MMA rows 0..7
//   5         r8: an R-only bit = MMA rows 8..15 (register slot 0)
//   6 ..      WB warp bits
//   then the fragment bits (register slots 1 ..): NFA R-only bits (row blocks), NFB Q-only bits
//   (column blocks), NFC shared bits (batches): 2^(NFA+NFB+NFC) accumulator fragments of 16 x 8.
// Output bits 0 and 1 are register slots (P0, P1), so each thread writes whole 32-byte sectors with
// one 256-bit store: the MMA's lane -> output map alone would write half sectors (the low output
// bits are often of the shared class), which HBM3e turns into read-modify-writes.
// Warp roles: one producer warp (lane 0 arms a slot, the 32 lanes issue its copies) streams the R chunk of every tile and, when it changes,
// the Q chunk -- every x-row, every tile bit the operand holds -- as cp.async.bulk copies of whole
// contiguous runs into an S-slot ring per operand (full / empty mbarriers, no block-wide barrier);
// 2^WB consumer warps each own a part of the tile.  A consumer keeps its Q fragments (split, in
// fragment order, one float4 per lane per (column block, batch, k-step)) in shared memory, rebuilt
// only when Q's chunk changes; R fragments are gathered from the raw chunk and split in registers.
#pragma once
#include "kernels.cuh"

namespace tnb {

struct HArgs {
  void* out;
  // streams: 0 = R (MMA rows), 1 = Q (MMA columns), 2 = X (FC mode: the consumer factor, one row)
  const void* in[3];
  uint64_t mask[3];                    // F_t(o) = ins0(pext(o, mask_t), pv_t)
  uint32_t pv[3];
  uint8_t row[3][1 << kMaxGroup];      // x -> chunk row
  uint32_t rowoff[3][1 << kMaxGroup];  // element offset G_t(x) of chunk row r (distinct x-part)
  uint32_t posoff[3][kGemmMaxTB];      // element offset (within the operand) of chunk bit k
  uint32_t nrows[3];                   // chunk rows (distinct x parts)
  uint32_t nch[3];                     // tile bits held by the operand (chunk row = 2^nch elements)
  uint32_t runl[3];                    // log2 elements of one contiguous run (one bulk copy), >= 1
  int8_t chbit[3][kGemmMaxTB];         // tile-local bit u -> chunk bit (-1: absent)
  uint8_t outbit[kGemmMaxTB];          // tile-local bit u -> output bit (all < 32)
  uint8_t sbit[kGemmMaxTB];            // tile-local bit u -> staging bit (rank among the tile's output bits)
  uint32_t sm_in[3][4];                // dynamic smem byte offset of ring slot (stream, slot)
  uint32_t sm_run[3];                  // dynamic smem byte offset of the run table (element offset of run q)
  uint32_t sm_q;                       // dynamic smem byte offset of the Q fragments
  int32_t p0, p1;                      // register slots holding output bits 0 and 1
  uint32_t rpad;                       // floats of padding after every R chunk row (shared-memory banks)
  int32_t dbg;                         // TNB_HM_DBG (diagnostics only, wrong results): 1 skip the MMAs, 2 skip the consumer math
  int32_t stages[3];                   // ring slots per stream (2..4)
  const void* cin[kMaxIn];             // constant inputs: no output bit (C[x] = prod_t cin[t][cgx[t][x]])
  uint32_t cgx[kMaxIn][1 << kMaxGroup];
  int32_t nc;
  int32_t out_rank;
  uint8_t perm[64];                    // logical tile-index bit b -> output bit (traversal order)
};

// v = big + small with big = v truncated to TF32 (the low 13 mantissa bits cleared: one LOP3; the
// cvt.rna.tf32 rounding form is a ~5-instruction sequence on sm_100a) and small = v - big exactly;
// the MMA then truncates small to TF32 as well, so big + small carries ~21 bits of v
__device__ __forceinline__ void tf32_split(float v, uint32_t& big, uint32_t& small) {
  const uint32_t b = __float_as_uint(v) & 0xFFFFE000u;
  big = b;
  small = __float_as_uint(v - __uint_as_float(b));
}

__device__ __forceinline__ void mma_tf32(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void hm_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void hm_bulk(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void hm_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred P;\n HM_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      " @!P bra HM_WAIT_%=;\n}" ::"r"(bar), "r"(parity) : "memory");
}
__device__ __forceinline__ void hm_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void st_v8_cs(float* p, const float (&v)[8]) {
  asm volatile("st.global.cs.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(v[0]), "f"(v[1]), "f"(v[2]),
               "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
               : "memory");
}

// The thread's 2^NR complex outputs (register slot 0 = r8: acc[f][0..1] / acc[f][2..3]; slots 1.. =
// fragment index f) as 256-bit stores of the 4 values whose output bits 0 / 1 are slots P0 / P1.
template <int P0, int P1, int NR, int NF>
__device__ __forceinline__ void hm_store(float* ob, const float (&acc)[NF][4], const uint32_t (&so)[NR]) {
#pragma unroll
  for (int q = 0; q < (1 << NR); ++q) {
    if (q & ((1 << P0) | (1 << P1))) continue;
    uint32_t o = 0;
#pragma unroll
    for (int k = 0; k < NR; ++k)
      if ((q >> k) & 1) o += so[k];
    float v[8];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int reg = q | ((e & 1) << P0) | ((e >> 1) << P1);
      v[2 * e] = acc[reg >> 1][2 * (reg & 1)];
      v[2 * e + 1] = acc[reg >> 1][2 * (reg & 1) + 1];
    }
    st_v8_cs(ob + 2 * (size_t)o, v);
  }
}

// k_fc_hm mode (FC = true): the group's output T is never written -- it is the full input of the
// next group (OP_GROUP_FEED, kernels_fc.cuh), out3[o] = sum_y C3_y X(o, y) T[o, y].  Tile bits are
// consumer output bits o; the traversal runs over the consumer's summed bits y first (HArgs.perm),
// so 2^M3 consecutive tiles of a CTA share o and every thread accumulates its outputs in registers.
// X (the consumer's other input holding output bits) arrives by 256-bit loads issued at the start of
// the tile (the tile's MMAs cover their latency).
struct FHArgs {
  void* out3;                                  // consumer output (2^R3 elements)
  int32_t M3;                                  // consumer summed indices (y bits of T)
  const void* xin;                             // X, or nullptr (the consumer has only weights)
  uint64_t xmask;                              // F_X(o) = ins0(pext(o, xmask), xpv)
  uint32_t xpv;
  uint32_t xgx[1 << kMaxGroup];                // G_X(y), y in traversal order
  int32_t nw;                                  // consumer inputs holding no output bit (weights)
  const void* win[kMaxIn];
  uint32_t wgx[kMaxIn][1 << kMaxGroup];        // y in traversal order
  uint64_t omask;                              // (1 << R3) - 1
};

__device__ __forceinline__ void ld_v8_stream(float (&v)[8], const float* p) {
  asm volatile("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
               : "l"(p));
}

// FC: the thread's 2^NR consumer factors X (register-slot order, as hm_store's values) from the X
// chunk in shared memory: the quads whose output bits 0 / 1 are slots P0 / P1 (X chunk positions 0, 1)
// as two 16-byte loads each
template <int P0, int P1, int NR>
__device__ __forceinline__ void hm_load_x(float (&xr)[1 << NR][2], const float2* xb, const uint32_t (&xs)[NR]) {
#pragma unroll
  for (int q = 0; q < (1 << NR); ++q) {
    if (q & ((1 << P0) | (1 << P1))) continue;
    uint32_t o = 0;
#pragma unroll
    for (int k = 0; k < NR; ++k)
      if ((q >> k) & 1) o += xs[k];
    const float4 v0 = *reinterpret_cast<const float4*>(xb + o), v1 = *reinterpret_cast<const float4*>(xb + o + 2);
    const float v[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int reg = q | ((e & 1) << P0) | ((e >> 1) << P1);
      xr[reg][0] = v[2 * e];
      xr[reg][1] = v[2 * e + 1];
    }
  }
}

template <int M, int NFA, int NFB, int NFC, int WB, bool FC = false>
__global__ void __launch_bounds__((32 << WB) + 32, FC ? 2 : 3) k_gemm_hm(const HArgs a, const FHArgs f) {
  constexpr int NW = 1 << WB;              // consumer warps; warp NW is the producer
  constexpr int kThreads = 32 * NW + 32;
  constexpr int K = 1 << M;
  constexpr int KS = K / 4;                // k-steps of 8 real values (4 complex x)
  constexpr int RA = 1 << NFA, RB = 1 << NFB, RC = 1 << NFC;
  constexpr int NFR = NFA + NFB + NFC;     // fragment bits
  constexpr int NF = 1 << NFR;
  constexpr int NR = 1 + NFR;              // register slots (r8 + fragment bits)
  constexpr int TB = 6 + WB + NFR;
  constexpr int NB = 64 - TB;
  static_assert(M >= 2 && M <= kMaxGroup, "k_gemm_hm: 2 <= M <= 5");
  static_assert(NFR >= 1 && NFR <= 3, "k_gemm_hm: 1..3 fragment bits");
  const uint32_t tid = threadIdx.x, lane = tid & 31u, wid = tid >> 5;
  const uint32_t g = lane >> 2, tig = lane & 3u;
  const uint64_t n_tiles = 1ull << (a.out_rank - TB);
  extern __shared__ __align__(16) unsigned char dsm[];
  constexpr int NOPS = FC ? 3 : 2;         // streams
  __shared__ uint32_t fbit[NOPS][NB];
  __shared__ uint32_t fcum[NOPS][NB + 1];
  __shared__ uint64_t pbit[NB], pcum[NB + 1];
  __shared__ float2 Cs[K];
  __shared__ uint32_t rowf[K];             // R chunk row of x, in floats (row << nch, x 2)
  __shared__ __align__(8) uint64_t bars[2][3][4];   // [full / empty][stream][slot]
  __shared__ float2 C3s[FC ? (1 << kMaxGroup) : 1];   // product of the consumer's weights per y
  const int nperm = a.out_rank - TB;
  for (int i = tid; i < NOPS * NB; i += kThreads) {
    const int t = i / NB, b = i % NB;
    fbit[t][b] = b < nperm ? (uint32_t)fmap(1ull << a.perm[b], a.mask[t], a.pv[t]) : 0u;
  }
  for (int b = tid; b < NB; b += kThreads) pbit[b] = b < nperm ? 1ull << a.perm[b] : 0ull;
  if (tid < (uint32_t)K) {
    rowf[tid] = ((uint32_t)a.row[0][tid] << a.nch[0]) * 2u + (uint32_t)a.row[0][tid] * a.rpad;
    float2 c = make_float2(1.f, 0.f);
    for (int t = 0; t < a.nc; ++t) c = cmul(c, __ldg(static_cast<const float2*>(a.cin[t]) + a.cgx[t][tid]));
    Cs[tid] = c;
  }
  // run tables: run q of stream u's chunk (2^runl contiguous elements) -> element offset from the base
#pragma unroll
  for (int u = 0; u < NOPS; ++u) {
    const uint32_t lp = a.nch[u] - a.runl[u];
    const uint32_t nr = a.nrows[u] << lp;
    uint32_t* tab = reinterpret_cast<uint32_t*>(dsm + a.sm_run[u]);
    for (uint32_t q = tid; q < nr; q += kThreads) {
      const uint32_t w = (q & ((1u << lp) - 1u)) << a.runl[u];
      uint32_t off = a.rowoff[u][q >> lp];
      for (uint32_t k = a.runl[u]; k < a.nch[u]; ++k)
        if ((w >> k) & 1u) off += a.posoff[u][k];
      tab[q] = off;
    }
  }
  if (FC && tid < (1u << f.M3)) {
    float2 c3 = make_float2(1.f, 0.f);
    for (int w = 0; w < f.nw; ++w) c3 = cmul(c3, __ldg(static_cast<const float2*>(f.win[w]) + f.wgx[w][tid]));
    C3s[tid] = c3;
  }
  if (tid == 0) {
    for (int u = 0; u < NOPS; ++u)
      for (int s = 0; s < a.stages[u]; ++s) {
        mbar_init(&bars[0][u][s], 1);
        mbar_init(&bars[1][u][s], NW);
      }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int nbu = min(NB - 1, max(0, nperm));
  if (tid < (uint32_t)NOPS) {
    uint32_t c = 0;
    fcum[tid][0] = 0;
    for (int b = 0; b < nbu; ++b) { c += fbit[tid][b]; fcum[tid][b + 1] = c; }
  }
  if (tid == 3u) {
    uint64_t c = 0;
    pcum[0] = 0;
    for (int b = 0; b < nbu; ++b) { c += pbit[b]; pcum[b + 1] = c; }
  }
  __syncthreads();
  uint64_t t0, t1;
  if (FC) {   // whole groups of 2^M3 tiles per CTA (a consumer output block is finished inside one CTA)
    const uint64_t n_groups = n_tiles >> f.M3;
    const uint64_t gper = (n_groups + gridDim.x - 1) / gridDim.x;
    t0 = ((uint64_t)blockIdx.x * gper) << f.M3;
    const uint64_t t1e = (((uint64_t)blockIdx.x + 1) * gper) << f.M3;
    t1 = t1e < n_tiles ? t1e : n_tiles;
  } else {
    const uint64_t per = (n_tiles + gridDim.x - 1) / gridDim.x;
    t0 = (uint64_t)blockIdx.x * per;
    t1 = t0 + per < n_tiles ? t0 + per : n_tiles;
  }
  uint64_t obase = 0;
  for (int b = 0; b < nperm && (t0 >> b); ++b)
    if ((t0 >> b) & 1) obase |= 1ull << a.perm[b];
  const uint32_t bar_full = smem_u32(&bars[0][0][0]);   // + (u * 4 + slot) * 8
  const uint32_t bar_empty = smem_u32(&bars[1][0][0]);

  if (wid == (uint32_t)NW) {
    // ---------------------------------------------------------------- producer warp: lane 0 arms
    // the slot's full barrier, the 32 lanes issue the chunk's bulk copies
    if (t0 < t1) {
      uint32_t cur[3];
      int ver[3] = {0, 0, 0};
      for (int u = 0; u < NOPS; ++u) cur[u] = (uint32_t)fmap(obase, a.mask[u], a.pv[u]);
      auto issue = [&](int u, uint32_t base) {
        const int S = a.stages[u];
        const int v = ver[u], slot = v % S;
        if (v >= S) hm_wait(bar_empty + (uint32_t)(u * 4 + slot) * 8u, (uint32_t)((v / S) - 1) & 1u);
        const uint32_t nr = a.nrows[u] << (a.nch[u] - a.runl[u]);
        const uint32_t bytes = 8u << a.runl[u];
        const uint32_t bar = bar_full + (uint32_t)(u * 4 + slot) * 8u;
        if (lane == 0) hm_expect_tx(bar, nr * bytes);
        __syncwarp();
        const float2* src = static_cast<const float2*>(a.in[u]) + base;
        const uint32_t dst = smem_u32(dsm + a.sm_in[u][slot]);
        const uint32_t* tab = reinterpret_cast<const uint32_t*>(dsm + a.sm_run[u]);
        // R rows are padded by rpad floats (run q of row q >> (nch - runl))
        const uint32_t pad_b = u == 0 ? a.rpad * 4u : 0u, lpr = a.nch[u] - a.runl[u];
        for (uint32_t q = lane; q < nr; q += 32) hm_bulk(dst + q * bytes + (q >> lpr) * pad_b, src + tab[q], bytes, bar);
      };
      issue(0, cur[0]);
      issue(1, cur[1]);
      if (FC) issue(2, cur[2] + f.xgx[0]);
      for (uint64_t tile = t0; tile + 1 < t1; ++tile) {
        const int r = __ffsll((long long)~tile) - 1;
#pragma unroll
        for (int u = 0; u < NOPS; ++u) {
          const bool changed = fbit[u][r] != fcum[u][r];
          if (changed) cur[u] = cur[u] + fbit[u][r] - fcum[u][r];
          if (u == 2) {                  // X: a new chunk every tile (the tile's y)
            ++ver[2];
            issue(2, cur[2] + f.xgx[(uint32_t)(tile + 1) & ((1u << f.M3) - 1u)]);
          } else if (changed) {
            ++ver[u];
            issue(u, cur[u]);
          }
        }
      }
    }
    return;
  }

  // ------------------------------------------------------------------ consumers
  auto chunk_off = [&](int u, int k) -> uint32_t { return a.chbit[u][k] >= 0 ? 1u << a.chbit[u][k] : 0u; };
  auto obit = [&](int k) -> uint32_t { return 1u << a.outbit[k]; };
  constexpr int FB0 = 6 + WB;              // tile-local index of the first fragment bit
  uint32_t othr = 0, ia_thr = 0, ib_w = 0;
#pragma unroll
  for (int k = 0; k < 2; ++k)
    if ((tig >> k) & 1u) othr += obit(k);
#pragma unroll
  for (int k = 0; k < 3; ++k)
    if ((g >> k) & 1u) { othr += obit(2 + k); ia_thr += chunk_off(0, 2 + k); }
#pragma unroll
  for (int k = 0; k < WB; ++k)
    if ((wid >> k) & 1u) { othr += obit(6 + k); ia_thr += chunk_off(0, 6 + k); ib_w += chunk_off(1, 6 + k); }
  const uint32_t ia_r8 = chunk_off(0, 5) * 2u;
  // output offset of each register slot (0 = r8, 1 + k = fragment bit k)
  uint32_t so[NR];
  so[0] = obit(5);
#pragma unroll
  for (int k = 0; k < NFR; ++k) so[1 + k] = obit(FB0 + k);
  // Q fragment entry of this lane: column j = g >> 1 (tile bits 0, 1), f = g & 1, e = tig & 1
  const uint32_t ib_lane = ib_w + (((g >> 1) & 1u) ? chunk_off(1, 0) : 0u) + (((g >> 2) & 1u) ? chunk_off(1, 1) : 0u);
  const uint32_t qf = g & 1u, qe = tig & 1u;
  // this warp's Q fragments: [batch][column block][k-step][lane] float4 (b0 big, b1 big, b0 small, b1 small)
  float4* qfrag = reinterpret_cast<float4*>(dsm + a.sm_q) + (size_t)wid * RB * RC * KS * 32 + lane;
  float* out = static_cast<float*>(a.out);
  // FC: X chunk index of this thread's outputs: lanes / warps, register slots
  uint32_t xthr = 0, xs[NR];
  float oacc[FC ? NF : 1][4];
  const uint32_t ymask = FC ? (1u << f.M3) - 1u : 0u;
  if (FC) {
#pragma unroll
    for (int k = 0; k < 2; ++k)
      if ((tig >> k) & 1u) xthr += chunk_off(2, k);
#pragma unroll
    for (int k = 0; k < 3; ++k)
      if ((g >> k) & 1u) xthr += chunk_off(2, 2 + k);
#pragma unroll
    for (int k = 0; k < WB; ++k)
      if ((wid >> k) & 1u) xthr += chunk_off(2, 6 + k);
    xs[0] = chunk_off(2, 5);
#pragma unroll
    for (int k = 0; k < NFR; ++k) xs[1 + k] = chunk_off(2, FB0 + k);
  }

  // R chunk row offsets (in floats) of this lane's x values per k-step (x = 4s + tig/2 and + 2)
  uint32_t rfr[KS][2];
#pragma unroll
  for (int s = 0; s < KS; ++s) {
    const uint32_t r0 = a.row[0][4 * s + (tig >> 1)], r1 = a.row[0][4 * s + 2 + (tig >> 1)];
    rfr[s][0] = (r0 << a.nch[0]) * 2u + r0 * a.rpad;
    rfr[s][1] = (r1 << a.nch[0]) * 2u + r1 * a.rpad;
  }
  // R chunk index (in floats) of each (batch, row block) fragment set, hoisted out of the tile loop
  uint32_t iaf[RC][RA];
#pragma unroll
  for (int fc = 0; fc < RC; ++fc)
#pragma unroll
    for (int fa = 0; fa < RA; ++fa) {
      uint32_t ia = ia_thr;
#pragma unroll
      for (int k = 0; k < NFA; ++k)
        if ((fa >> k) & 1) ia += chunk_off(0, FB0 + k);
#pragma unroll
      for (int k = 0; k < NFC; ++k)
        if ((fc >> k) & 1) ia += chunk_off(0, FB0 + NFA + NFB + k);
      iaf[fc][fa] = ia * 2u;
    }

  int cslot[3] = {0, 0, 0};
  uint32_t cpar[3] = {0u, 0u, 0u};
  bool qready = false;
  for (uint64_t tile = t0; tile < t1; ++tile) {
    const int r = __ffsll((long long)~tile) - 1;
    const uint32_t y = (uint32_t)tile & ymask;
    if constexpr (FC) {
      if (y == 0u) {                     // a new consumer output block
#pragma unroll
        for (int i = 0; i < NF; ++i)
#pragma unroll
          for (int k = 0; k < 4; ++k) oacc[i][k] = 0.f;
      }
    }
    if (!qready) {                       // Q's chunk changed: rebuild this warp's Q fragments
      hm_wait(bar_full + (uint32_t)(4 + cslot[1]) * 8u, cpar[1]);
      const float2* Qraw = reinterpret_cast<const float2*>(dsm + a.sm_in[1][cslot[1]]);
#pragma unroll
      for (int fc = 0; fc < RC; ++fc)
#pragma unroll
        for (int fb = 0; fb < RB; ++fb) {
          uint32_t ib = ib_lane;
#pragma unroll
          for (int k = 0; k < NFB; ++k)
            if ((fb >> k) & 1) ib += chunk_off(1, FB0 + NFA + k);
#pragma unroll
          for (int k = 0; k < NFC; ++k)
            if ((fc >> k) & 1) ib += chunk_off(1, FB0 + NFA + NFB + k);
#pragma unroll
          for (int s = 0; s < KS; ++s) {
            float v[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int x = 4 * s + 2 * h + (int)(tig >> 1);
              const float2 q = cmul(Qraw[((uint32_t)a.row[1][x] << a.nch[1]) + ib], Cs[x]);
              // Q'[2x+e][2j+f]: (e, f) = (0, 0) Re, (0, 1) Im, (1, 0) -Im, (1, 1) Re
              v[h] = qe == qf ? q.x : (qe ? -q.y : q.y);
            }
            uint32_t b0, b1, s0, s1;
            tf32_split(v[0], b0, s0);
            tf32_split(v[1], b1, s1);
            qfrag[((fc * RB + fb) * KS + s) * 32] =
                make_float4(__uint_as_float(b0), __uint_as_float(b1), __uint_as_float(s0), __uint_as_float(s1));
          }
        }
      __syncwarp();
      if (lane == 0) hm_arrive(bar_empty + (uint32_t)(4 + cslot[1]) * 8u);   // raw Q no longer read
      qready = true;
    }
    hm_wait(bar_full + (uint32_t)cslot[0] * 8u, cpar[0]);
    const float* Rraw = reinterpret_cast<const float*>(dsm + a.sm_in[0][cslot[0]]) + qe;
    float acc[NF][4];
#pragma unroll
    for (int fi = 0; fi < NF; ++fi)
#pragma unroll
      for (int k = 0; k < 4; ++k) acc[fi][k] = 0.f;
#pragma unroll
    for (int s = 0; s < KS; ++s) {
      if (a.dbg & 1) break;
      const uint32_t rf0 = rfr[s][0], rf1 = rfr[s][1];
      uint32_t ab[RC][RA][4], as[RC][RA][4];
#pragma unroll
      for (int fc = 0; fc < RC; ++fc)
#pragma unroll
        for (int fa = 0; fa < RA; ++fa) {
          const uint32_t ia = iaf[fc][fa];
          tf32_split(Rraw[rf0 + ia], ab[fc][fa][0], as[fc][fa][0]);
          tf32_split(Rraw[rf0 + ia + ia_r8], ab[fc][fa][1], as[fc][fa][1]);
          tf32_split(Rraw[rf1 + ia], ab[fc][fa][2], as[fc][fa][2]);
          tf32_split(Rraw[rf1 + ia + ia_r8], ab[fc][fa][3], as[fc][fa][3]);
        }
      float4 qv[RC][RB];
#pragma unroll
      for (int fc = 0; fc < RC; ++fc)
#pragma unroll
        for (int fb = 0; fb < RB; ++fb) qv[fc][fb] = qfrag[((fc * RB + fb) * KS + s) * 32];
#pragma unroll
      for (int pass = 0; pass < 3; ++pass)
#pragma unroll
        for (int fc = 0; fc < RC; ++fc)
#pragma unroll
          for (int fb = 0; fb < RB; ++fb)
#pragma unroll
            for (int fa = 0; fa < RA; ++fa) {
              const int fi = fa + RA * (fb + RB * fc);
              const float4 q = qv[fc][fb];
              if (pass == 0) mma_tf32(acc[fi], as[fc][fa], __float_as_uint(q.x), __float_as_uint(q.y));
              else if (pass == 1) mma_tf32(acc[fi], ab[fc][fa], __float_as_uint(q.z), __float_as_uint(q.w));
              else mma_tf32(acc[fi], ab[fc][fa], __float_as_uint(q.x), __float_as_uint(q.y));
            }
    }
    // chunk versions for the next tile; release the slots this warp is done with
#pragma unroll
    for (int u = 0; u < 2; ++u)
      if (fbit[u][r] != fcum[u][r]) {
        if (u == 0) {
          __syncwarp();
          if (lane == 0) hm_arrive(bar_empty + (uint32_t)cslot[0] * 8u);
        } else {
          qready = false;
        }
        if (++cslot[u] == a.stages[u]) { cslot[u] = 0; cpar[u] ^= 1u; }
      }
    if constexpr (FC) {
      // consumer: oacc += C3_y X(o, y) T[o, y], X from this tile's X chunk (4 complex per quad)
      hm_wait(bar_full + (uint32_t)(8 + cslot[2]) * 8u, cpar[2]);
      float xr[2 * NF][2];
      {
        const float2* xb = reinterpret_cast<const float2*>(dsm + a.sm_in[2][cslot[2]]) + xthr;
        switch (a.p0 * 4 + a.p1) {
#define HM_LD(P0, P1) \
          case P0 * 4 + P1: if constexpr (P0 < NR && P1 < NR) hm_load_x<P0, P1, NR>(xr, xb, xs); break;
          HM_LD(0, 1) HM_LD(0, 2) HM_LD(0, 3) HM_LD(1, 0) HM_LD(1, 2) HM_LD(1, 3)
          HM_LD(2, 0) HM_LD(2, 1) HM_LD(2, 3) HM_LD(3, 0) HM_LD(3, 1) HM_LD(3, 2)
#undef HM_LD
          default: break;
        }
      }
      __syncwarp();
      if (lane == 0) hm_arrive(bar_empty + (uint32_t)(8 + cslot[2]) * 8u);
      if (++cslot[2] == a.stages[2]) { cslot[2] = 0; cpar[2] ^= 1u; }
      const float2 c3 = C3s[y];
#pragma unroll
      for (int reg = 0; reg < 2 * NF && !(a.dbg & 2); ++reg) {
        const float xx0 = c3.x * xr[reg][0] - c3.y * xr[reg][1], xx1 = c3.x * xr[reg][1] + c3.y * xr[reg][0];
        const float t0r = acc[reg >> 1][2 * (reg & 1)], t0i = acc[reg >> 1][2 * (reg & 1) + 1];
        oacc[reg >> 1][2 * (reg & 1)] += xx0 * t0r - xx1 * t0i;
        oacc[reg >> 1][2 * (reg & 1) + 1] += xx0 * t0i + xx1 * t0r;
      }
      if (y == ymask) {                  // last y of the block: the consumer output is final
        float* ob = static_cast<float*>(f.out3) + 2 * ((obase & f.omask) + othr);
        switch (a.p0 * 4 + a.p1) {
#define HM_ST(P0, P1) \
          case P0 * 4 + P1: if constexpr (P0 < NR && P1 < NR) hm_store<P0, P1, NR, NF>(ob, oacc, so); break;
          HM_ST(0, 1) HM_ST(0, 2) HM_ST(0, 3) HM_ST(1, 0) HM_ST(1, 2) HM_ST(1, 3)
          HM_ST(2, 0) HM_ST(2, 1) HM_ST(2, 3) HM_ST(3, 0) HM_ST(3, 1) HM_ST(3, 2)
#undef HM_ST
          default: break;
        }
      }
    } else {
      float* ob = out + 2 * (obase + othr);
      switch (a.p0 * 4 + a.p1) {
#define HM_ST(P0, P1) \
        case P0 * 4 + P1: if constexpr (P0 < NR && P1 < NR) hm_store<P0, P1, NR, NF>(ob, acc, so); break;
        HM_ST(0, 1) HM_ST(0, 2) HM_ST(0, 3) HM_ST(1, 0) HM_ST(1, 2) HM_ST(1, 3)
        HM_ST(2, 0) HM_ST(2, 1) HM_ST(2, 3) HM_ST(3, 0) HM_ST(3, 1) HM_ST(3, 2)
#undef HM_ST
        default: break;
      }
    }
    obase = obase + pbit[r] - pcum[r];
  }
}

}  // namespace tnb

namespace tnb {

// ---------------------------------------------------------------- complex128: k_gemm_hm64
// The same two-operand merge group for c128 on the FP64 tensor path: mma.sync.m8n8k4.f64 (DMMA),
// one product, no split (DMMA and DFMA both measured ~18 TMAC/s on B200, profiles/r02/hm/mma_rate.txt;
// what DMMA buys is 256 MACs per warp instruction instead of 32, for a kernel family bound by its
// instruction stream).  Fragments (lane = 4 g + tig): A'[g][tig] with x = 2s + tig/2, e = tig & 1;
// B'[k = tig][n = g] (complex column g / 2, f = g & 1); C[g][2 tig], C[g][2 tig + 1] = (Re, Im) of
// complex column tig.  Tile-local bits: 0, 1 tig (Q-only), 2, 3, 4 g (R-only), then WB warp bits,
// then the fragment bits (register slots 0 .. 2: NFA R-only, NFB Q-only, NFC shared); output bit 0
// is register slot P0, so two complex values = one 32-byte sector leave in one 256-bit store.
// Ring, producer warp and traversal as k_gemm_hm (HArgs; element = double2, run bytes 16 << runl).
__device__ __forceinline__ void mma_f64(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}
__device__ __forceinline__ void st_v4d_cs(double* p, double a, double b, double c, double d) {
  asm volatile("st.global.cs.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}
template <int P0, int NF>
__device__ __forceinline__ void hm64_store(double* ob, const double (&acc)[NF][2], const uint32_t (&so)[3]) {
  constexpr int NR = NF == 8 ? 3 : (NF == 4 ? 2 : 1);
#pragma unroll
  for (int q = 0; q < NF; ++q) {
    if (q & (1 << P0)) continue;
    uint32_t o = 0;
#pragma unroll
    for (int k = 0; k < NR; ++k)
      if ((q >> k) & 1) o += so[k];
    const int q1 = q | (1 << P0);
    st_v4d_cs(ob + 2 * (size_t)o, acc[q][0], acc[q][1], acc[q1][0], acc[q1][1]);
  }
}

template <int M, int NFA, int NFB, int NFC, int WB>
__global__ void __launch_bounds__((32 << WB) + 32, 2) k_gemm_hm64(const HArgs a) {
  constexpr int NW = 1 << WB;
  constexpr int kThreads = 32 * NW + 32;
  constexpr int K = 1 << M;
  constexpr int KS = K / 2;                // k-steps of 4 real values (2 complex x)
  constexpr int RA = 1 << NFA, RB = 1 << NFB, RC = 1 << NFC;
  constexpr int NFR = NFA + NFB + NFC;
  constexpr int NF = 1 << NFR;
  constexpr int TB = 5 + WB + NFR;
  constexpr int NB = 64 - TB;
  static_assert(M >= 1 && M <= kMaxGroup && NFR == 3, "k_gemm_hm64: 1 <= M <= 5, 3 fragment bits");
  const uint32_t tid = threadIdx.x, lane = tid & 31u, wid = tid >> 5;
  const uint32_t g = lane >> 2, tig = lane & 3u;
  const uint64_t n_tiles = 1ull << (a.out_rank - TB);
  extern __shared__ __align__(16) unsigned char dsm[];
  __shared__ uint32_t fbit[2][NB];
  __shared__ uint32_t fcum[2][NB + 1];
  __shared__ uint64_t pbit[NB], pcum[NB + 1];
  __shared__ double2 Cs[K];
  __shared__ __align__(8) uint64_t bars[2][2][4];
  const int nperm = a.out_rank - TB;
  for (int i = tid; i < 2 * NB; i += kThreads) {
    const int t = i / NB, b = i % NB;
    fbit[t][b] = b < nperm ? (uint32_t)fmap(1ull << a.perm[b], a.mask[t], a.pv[t]) : 0u;
  }
  for (int b = tid; b < NB; b += kThreads) pbit[b] = b < nperm ? 1ull << a.perm[b] : 0ull;
  if (tid < (uint32_t)K) {
    double2 c = make_double2(1.0, 0.0);
    for (int t = 0; t < a.nc; ++t) c = cmul(c, __ldg(static_cast<const double2*>(a.cin[t]) + a.cgx[t][tid]));
    Cs[tid] = c;
  }
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const uint32_t lp = a.nch[u] - a.runl[u];
    const uint32_t nr = a.nrows[u] << lp;
    uint32_t* tab = reinterpret_cast<uint32_t*>(dsm + a.sm_run[u]);
    for (uint32_t q = tid; q < nr; q += kThreads) {
      const uint32_t w = (q & ((1u << lp) - 1u)) << a.runl[u];
      uint32_t off = a.rowoff[u][q >> lp];
      for (uint32_t k = a.runl[u]; k < a.nch[u]; ++k)
        if ((w >> k) & 1u) off += a.posoff[u][k];
      tab[q] = off;
    }
  }
  if (tid == 0) {
    for (int u = 0; u < 2; ++u)
      for (int s = 0; s < a.stages[u]; ++s) {
        mbar_init(&bars[0][u][s], 1);
        mbar_init(&bars[1][u][s], NW);
      }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int nbu = min(NB - 1, max(0, nperm));
  if (tid < 2u) {
    uint32_t c = 0;
    fcum[tid][0] = 0;
    for (int b = 0; b < nbu; ++b) { c += fbit[tid][b]; fcum[tid][b + 1] = c; }
  }
  if (tid == 3u) {
    uint64_t c = 0;
    pcum[0] = 0;
    for (int b = 0; b < nbu; ++b) { c += pbit[b]; pcum[b + 1] = c; }
  }
  __syncthreads();
  const uint64_t per = (n_tiles + gridDim.x - 1) / gridDim.x;
  const uint64_t t0 = (uint64_t)blockIdx.x * per;
  const uint64_t t1 = t0 + per < n_tiles ? t0 + per : n_tiles;
  uint64_t obase = 0;
  for (int b = 0; b < nperm && (t0 >> b); ++b)
    if ((t0 >> b) & 1) obase |= 1ull << a.perm[b];
  const uint32_t bar_full = smem_u32(&bars[0][0][0]);
  const uint32_t bar_empty = smem_u32(&bars[1][0][0]);

  if (wid == (uint32_t)NW) {                // producer warp (as k_gemm_hm)
    if (t0 < t1) {
      uint32_t cur[2];
      int ver[2] = {0, 0};
      for (int u = 0; u < 2; ++u) cur[u] = (uint32_t)fmap(obase, a.mask[u], a.pv[u]);
      auto issue = [&](int u) {
        const int S = a.stages[u];
        const int v = ver[u], slot = v % S;
        if (v >= S) hm_wait(bar_empty + (uint32_t)(u * 4 + slot) * 8u, (uint32_t)((v / S) - 1) & 1u);
        const uint32_t nr = a.nrows[u] << (a.nch[u] - a.runl[u]);
        const uint32_t bytes = 16u << a.runl[u];
        const uint32_t bar = bar_full + (uint32_t)(u * 4 + slot) * 8u;
        if (lane == 0) hm_expect_tx(bar, nr * bytes);
        __syncwarp();
        const double2* src = static_cast<const double2*>(a.in[u]) + cur[u];
        const uint32_t dst = smem_u32(dsm + a.sm_in[u][slot]);
        const uint32_t* tab = reinterpret_cast<const uint32_t*>(dsm + a.sm_run[u]);
        for (uint32_t q = lane; q < nr; q += 32) hm_bulk(dst + q * bytes, src + tab[q], bytes, bar);
      };
      issue(0);
      issue(1);
      for (uint64_t tile = t0; tile + 1 < t1; ++tile) {
        const int r = __ffsll((long long)~tile) - 1;
#pragma unroll
        for (int u = 0; u < 2; ++u)
          if (fbit[u][r] != fcum[u][r]) {
            cur[u] = cur[u] + fbit[u][r] - fcum[u][r];
            ++ver[u];
            issue(u);
          }
      }
    }
    return;
  }

  auto chunk_off = [&](int u, int k) -> uint32_t { return a.chbit[u][k] >= 0 ? 1u << a.chbit[u][k] : 0u; };
  auto obit = [&](int k) -> uint32_t { return 1u << a.outbit[k]; };
  constexpr int FB0 = 5 + WB;
  uint32_t othr = 0, ia_thr = 0, ib_w = 0;
#pragma unroll
  for (int k = 0; k < 2; ++k)
    if ((tig >> k) & 1u) othr += obit(k);
#pragma unroll
  for (int k = 0; k < 3; ++k)
    if ((g >> k) & 1u) { othr += obit(2 + k); ia_thr += chunk_off(0, 2 + k); }
#pragma unroll
  for (int k = 0; k < WB; ++k)
    if ((wid >> k) & 1u) { othr += obit(5 + k); ia_thr += chunk_off(0, 5 + k); ib_w += chunk_off(1, 5 + k); }
  uint32_t so[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) so[k] = obit(FB0 + k);
  const uint32_t ib_lane = ib_w + (((g >> 1) & 1u) ? chunk_off(1, 0) : 0u) + (((g >> 2) & 1u) ? chunk_off(1, 1) : 0u);
  const uint32_t qf = g & 1u, qe = tig & 1u;
  double* qfrag = reinterpret_cast<double*>(dsm + a.sm_q) + (size_t)wid * RB * RC * KS * 32 + lane;
  uint32_t rfr[KS];                        // R chunk row offset (in doubles) of x = 2s + tig / 2
#pragma unroll
  for (int s = 0; s < KS; ++s) rfr[s] = ((uint32_t)a.row[0][2 * s + (tig >> 1)] << a.nch[0]) * 2u;
  uint32_t iaf[RC][RA];
#pragma unroll
  for (int fc = 0; fc < RC; ++fc)
#pragma unroll
    for (int fa = 0; fa < RA; ++fa) {
      uint32_t ia = ia_thr;
#pragma unroll
      for (int k = 0; k < NFA; ++k)
        if ((fa >> k) & 1) ia += chunk_off(0, FB0 + k);
#pragma unroll
      for (int k = 0; k < NFC; ++k)
        if ((fc >> k) & 1) ia += chunk_off(0, FB0 + NFA + NFB + k);
      iaf[fc][fa] = ia * 2u + qe;
    }
  double* out = static_cast<double*>(a.out);
  int cslot[2] = {0, 0};
  uint32_t cpar[2] = {0u, 0u};
  bool qready = false;
  for (uint64_t tile = t0; tile < t1; ++tile) {
    const int r = __ffsll((long long)~tile) - 1;
    if (!qready) {
      hm_wait(bar_full + (uint32_t)(4 + cslot[1]) * 8u, cpar[1]);
      const double2* Qraw = reinterpret_cast<const double2*>(dsm + a.sm_in[1][cslot[1]]);
#pragma unroll
      for (int fc = 0; fc < RC; ++fc)
#pragma unroll
        for (int fb = 0; fb < RB; ++fb) {
          uint32_t ib = ib_lane;
#pragma unroll
          for (int k = 0; k < NFB; ++k)
            if ((fb >> k) & 1) ib += chunk_off(1, FB0 + NFA + k);
#pragma unroll
          for (int k = 0; k < NFC; ++k)
            if ((fc >> k) & 1) ib += chunk_off(1, FB0 + NFA + NFB + k);
#pragma unroll
          for (int s = 0; s < KS; ++s) {
            const int x = 2 * s + (int)(tig >> 1);
            const double2 q = cmul(Qraw[((uint32_t)a.row[1][x] << a.nch[1]) + ib], Cs[x]);
            qfrag[((fc * RB + fb) * KS + s) * 32] = qe == qf ? q.x : (qe ? -q.y : q.y);
          }
        }
      __syncwarp();
      if (lane == 0) hm_arrive(bar_empty + (uint32_t)(4 + cslot[1]) * 8u);
      qready = true;
    }
    hm_wait(bar_full + (uint32_t)cslot[0] * 8u, cpar[0]);
    const double* Rraw = reinterpret_cast<const double*>(dsm + a.sm_in[0][cslot[0]]);
    double acc[NF][2];
#pragma unroll
    for (int fi = 0; fi < NF; ++fi) { acc[fi][0] = 0.0; acc[fi][1] = 0.0; }
#pragma unroll
    for (int s = 0; s < KS; ++s) {
      double av[RC][RA], qv[RC][RB];
#pragma unroll
      for (int fc = 0; fc < RC; ++fc) {
#pragma unroll
        for (int fa = 0; fa < RA; ++fa) av[fc][fa] = Rraw[rfr[s] + iaf[fc][fa]];
#pragma unroll
        for (int fb = 0; fb < RB; ++fb) qv[fc][fb] = qfrag[((fc * RB + fb) * KS + s) * 32];
      }
#pragma unroll
      for (int fc = 0; fc < RC; ++fc)
#pragma unroll
        for (int fb = 0; fb < RB; ++fb)
#pragma unroll
          for (int fa = 0; fa < RA; ++fa) mma_f64(acc[fa + RA * (fb + RB * fc)], av[fc][fa], qv[fc][fb]);
    }
#pragma unroll
    for (int u = 0; u < 2; ++u)
      if (fbit[u][r] != fcum[u][r]) {
        if (u == 0) {
          __syncwarp();
          if (lane == 0) hm_arrive(bar_empty + (uint32_t)cslot[0] * 8u);
        } else {
          qready = false;
        }
        if (++cslot[u] == a.stages[u]) { cslot[u] = 0; cpar[u] ^= 1u; }
      }
    double* ob = out + 2 * (obase + othr);
    switch (a.p0) {
      case 0: hm64_store<0, NF>(ob, acc, so); break;
      case 1: hm64_store<1, NF>(ob, acc, so); break;
      case 2: hm64_store<2, NF>(ob, acc, so); break;
      default: break;
    }
    obase = obase + pbit[r] - pcum[r];
  }
}

}  // namespace tnb
