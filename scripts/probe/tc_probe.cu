// tc_probe.cu: standalone check of the tcgen05 kind::tf32 descriptors used by k_gemm_tc
// (K-major SWIZZLE_NONE canonical layouts, M=128, N=Np, 3xTF32 split).  Not part of the library.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>

constexpr int MR = 128, KP = 16, NP = 64;

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
// element (row, k) of a K-major no-swizzle tile with K floats per row: core matrix = 8 rows x 16 B
__device__ __forceinline__ uint32_t canon(int row, int k, int kf) {
  return (row >> 3) * (kf / 4) * 128 + (k >> 2) * 128 + (row & 7) * 16 + (k & 3) * 4;
}

__global__ void probe(const float* A, const float* B, float* D, int split) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  float* sAb = (float*)sm;              // 128 x 16
  float* sAs = sAb + MR * KP;
  float* sBb = sAs + MR * KP;           // 64 x 16
  float* sBs = sBb + NP * KP;
  const int tid = threadIdx.x;
  for (int i = tid; i < MR * KP; i += blockDim.x) {
    int r = i / KP, k = i % KP;
    float v = A[i];
    float big = split ? __uint_as_float(__float_as_uint(v) & 0xFFFFE000u) : v;
    *(float*)((char*)sAb + canon(r, k, KP)) = big;
    *(float*)((char*)sAs + canon(r, k, KP)) = v - big;
  }
  for (int i = tid; i < NP * KP; i += blockDim.x) {
    int n = i / KP, k = i % KP;
    float v = B[i];
    float big = split ? __uint_as_float(__float_as_uint(v) & 0xFFFFE000u) : v;
    *(float*)((char*)sBb + canon(n, k, KP)) = big;
    *(float*)((char*)sBs + canon(n, k, KP)) = v - big;
  }
  if (tid == 0) {
    uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (tid < 32) {
    uint32_t dst = (uint32_t)__cvta_generic_to_shared(&tbase);
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(dst));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  if (tid == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(NP >> 3) << 17) | ((uint32_t)(MR >> 4) << 24);
    const uint32_t aB = (uint32_t)__cvta_generic_to_shared(sAb), aS = (uint32_t)__cvta_generic_to_shared(sAs);
    const uint32_t bB = (uint32_t)__cvta_generic_to_shared(sBb), bS = (uint32_t)__cvta_generic_to_shared(sBs);
    const uint32_t sbo = (KP / 4) * 128, lbo = 128;
    int first = 1;
    const int nprod = split ? 3 : 1;
    for (int pr = 0; pr < nprod; ++pr) {
      const uint32_t a0 = pr == 2 ? aS : aB, b0 = pr == 1 ? bS : bB;
      for (int kc = 0; kc < KP / 8; ++kc) {
        uint64_t da = sdesc(a0 + kc * 256, lbo, sbo), db = sdesc(b0 + kc * 256, lbo, sbo);
        uint32_t acc = first ? 0u : 1u;
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
                     ::"r"(tm), "l"(da), "l"(db), "r"(idesc), "r"(acc));
        first = 0;
      }
    }
    uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(b));
  }
  __syncwarp();
  {
    uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
    asm volatile("{\n\t.reg .pred P1;\n\tLAB_WAIT:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t"
                 "@P1 bra DONE;\n\tbra LAB_WAIT;\n\tDONE:\n\t}" ::"r"(b));
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int w = tid >> 5, lane = tid & 31;
  const int row = w * 32 + lane;
  for (int c0 = 0; c0 < NP; c0 += 16) {
    uint32_t v[16];
    const uint32_t addr = tm + ((uint32_t)(w * 32) << 16) + c0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                 : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 16; ++j) D[row * NP + c0 + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tm));
}

int main() {
  std::vector<float> A(MR * KP), B(NP * KP), D(MR * NP);
  srand(1);
  for (auto& x : A) x = (float)rand() / RAND_MAX * 2 - 1;
  for (auto& x : B) x = (float)rand() / RAND_MAX * 2 - 1;
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  const int smem = (MR * KP * 2 + NP * KP * 2) * 4;
  for (int split = 0; split < 2; ++split) {
    cudaMemset(dD, 0, D.size() * 4);
    probe<<<1, 128, smem>>>(dA, dB, dD, split);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0, maxref = 0;
    for (int m = 0; m < MR; ++m)
      for (int n = 0; n < NP; ++n) {
        double r = 0;
        for (int k = 0; k < KP; ++k) r += (double)A[m * KP + k] * B[n * KP + k];
        maxerr = fmax(maxerr, fabs(r - D[m * NP + n]));
        maxref = fmax(maxref, fabs(r));
      }
    printf("split=%d max|err|=%.3e max|ref|=%.3e rel=%.3e  D[0]=%f D[1]=%f D[64]=%f\n", split, maxerr, maxref,
           maxerr / maxref, D[0], D[1], D[NP]);
  }
  return 0;
}
