// tc_rate.cu: throughput probe for tcgen05.mma (M=128) kind::tf32 / kind::f16 at several N and
// shared-memory layouts (SWIZZLE_NONE vs SWIZZLE_128B, K-major), one CTA per SM.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | ((uint64_t)layout << 61);
}
template <int N, int SW, int F16, int NACC, int RND>
__global__ void rate(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x;
  for (int i = tid; i < (128 * 64 + 256 * 64); i += blockDim.x) ((float*)sm)[i] = RND ? __sinf(i * 0.37f + 0.1f) : 0.f;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"((uint32_t)__cvta_generic_to_shared(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  if (tid < 32) {
    const uint32_t fmt = F16 ? 1u : 2u;   // bf16 : tf32
    const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint32_t a0 = (uint32_t)__cvta_generic_to_shared(sm), b0 = a0 + 128 * 64 * 4;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kc = 0; kc < 8; ++kc) {
        // SWIZZLE_NONE: 256 B per kc (two 16-B K halves, LBO 128), 8-row groups SBO = 8 * 256... (rows of 64 floats)
        // SWIZZLE_128B: rows of 128 B, 8-row atoms SBO = 1024; K step = +32 B inside the atom
        uint64_t da, db;
        if (SW) {
          da = sdesc(a0 + (kc & 3) * 32 + (kc >> 2) * 128 * 128, 16, 1024, 2);
          db = sdesc(b0 + (kc & 3) * 32 + (kc >> 2) * 256 * 128, 16, 1024, 2);
        } else {
          da = sdesc(a0 + kc * 256, 128, 2048, 0);
          db = sdesc(b0 + kc * 256, 128, 2048, 0);
        }
        if (tid == 0) {
          uint32_t acc = (it | (kc / NACC)) ? 1u : 0u;
          const uint32_t tmd = tm + (uint32_t)((kc % NACC) * N);
          if (F16)
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmd), "l"(da), "l"(db), "r"(idesc), "r"(acc));
          else
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmd), "l"(da), "l"(db), "r"(idesc), "r"(acc));
        }
        __syncwarp();
      }
    }
    if (tid == 0) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
    long long t1 = clock64();
    asm volatile("{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
    long long t2 = clock64();
    if (tid == 0 && blockIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tm));
}
template <int N, int SW, int F16, int NACC, int RND> void run() {
  unsigned long long* d; cudaMalloc(&d, 16);
  const int smem = (128 * 64 + 256 * 64) * 4;
  cudaFuncSetAttribute(rate<N, SW, F16, NACC, RND>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 200;
  rate<N, SW, F16, NACC, RND><<<148, 128, smem>>>(iters, d);
  cudaDeviceSynchronize();
  rate<N, SW, F16, NACC, RND><<<148, 128, smem>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  const double n = iters * 8.0, k = F16 ? 16 : 8;
  printf("rnd=%d nacc=%d %s N=%3d %s %s: issue %.1f clk/mma, complete %.1f clk/mma, %.0f MAC/clk/SM\n", RND, NACC, F16 ? "bf16" : "tf32", N,
         SW ? "SW128" : "NONE ", cudaGetErrorString(e), h[0] / n, h[1] / n, 128.0 * N * k * n / h[1]);
}
int main() {
  run<32, 0, 0, 2, 0>(); run<32, 0, 0, 2, 1>(); run<128, 0, 0, 2, 0>(); run<128, 0, 0, 2, 1>(); run<256, 0, 0, 1, 1>();
  run<32, 0, 1, 2, 1>();
  return 0;
}
