// mma_rate.cu: throughput of the warp-level (legacy) tensor-core path on sm_100a --
// mma.sync m16n8k8 tf32, m16n8k16 bf16 (f32 accumulate), m8n8k4 f64 -- against packed FP32 FFMA2.
// One CTA of W warps per SM x (148 x CPS) CTAs, NACC independent accumulators per warp.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mma_rate scripts/probe/mma_rate.cu
#include <cstdio>
#include <cstdint>

template <int NACC>
__global__ void k_tf32(int iters, float* sink) {
  float c[NACC][4] = {};
  uint32_t a0 = __float_as_uint(1.0f + threadIdx.x * 1e-3f), a1 = a0 ^ 1, a2 = a0 ^ 2, a3 = a0 ^ 3;
  uint32_t b0 = __float_as_uint(0.5f), b1 = b0 ^ 5;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int n = 0; n < NACC; ++n)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(c[n][0]), "+f"(c[n][1]), "+f"(c[n][2]), "+f"(c[n][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0;
#pragma unroll
  for (int n = 0; n < NACC; ++n) s += c[n][0] + c[n][1] + c[n][2] + c[n][3];
  if (s == 12345.f) sink[threadIdx.x] = s;
}

template <int NACC>
__global__ void k_bf16(int iters, float* sink) {
  float c[NACC][4] = {};
  uint32_t a0 = 0x3f803f80u + threadIdx.x, a1 = a0 ^ 1, a2 = a0 ^ 2, a3 = a0 ^ 3;
  uint32_t b0 = 0x3f003f00u, b1 = b0 ^ 5;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int n = 0; n < NACC; ++n)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(c[n][0]), "+f"(c[n][1]), "+f"(c[n][2]), "+f"(c[n][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0;
#pragma unroll
  for (int n = 0; n < NACC; ++n) s += c[n][0] + c[n][1] + c[n][2] + c[n][3];
  if (s == 12345.f) sink[threadIdx.x] = s;
}

template <int NACC>
__global__ void k_f64(int iters, float* sink) {
  double c[NACC][2] = {};
  double a = 1.0 + threadIdx.x * 1e-3, b = 0.5;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int n = 0; n < NACC; ++n)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[n][0]), "+d"(c[n][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int n = 0; n < NACC; ++n) s += c[n][0] + c[n][1];
  if (s == 12345.0) sink[threadIdx.x] = (float)s;
}

template <int NACC>
__global__ void k_ffma2(int iters, float* sink) {
  uint64_t c[NACC];
#pragma unroll
  for (int n = 0; n < NACC; ++n) c[n] = 0;
  float av = 1.0f + threadIdx.x * 1e-3f;
  uint64_t a, b;
  asm("mov.b64 %0, {%1, %1};" : "=l"(a) : "f"(av));
  asm("mov.b64 %0, {%1, %2};" : "=l"(b) : "f"(0.5f), "f"(0.25f));
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int n = 0; n < NACC; ++n) asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(c[n]) : "l"(a), "l"(b));
  }
  float s = 0;
#pragma unroll
  for (int n = 0; n < NACC; ++n) { float x, y; asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(c[n])); s += x + y; }
  if (s == 12345.f) sink[threadIdx.x] = s;
}

template <int NACC>
__global__ void k_dfma(int iters, float* sink) {
  double c[NACC];
#pragma unroll
  for (int n = 0; n < NACC; ++n) c[n] = 0.0;
  const double a = 1.0 + threadIdx.x * 1e-3, b = 0.5;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int n = 0; n < NACC; ++n) asm volatile("fma.rn.f64 %0, %1, %2, %0;" : "+d"(c[n]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int n = 0; n < NACC; ++n) s += c[n];
  if (s == 12345.0) sink[threadIdx.x] = (float)s;
}

template <typename K>
void run(const char* name, K kern, int warps, int cps, int iters, double macs_per_inst_per_warp, int nacc) {
  float* sink;
  cudaMalloc(&sink, 4096 * sizeof(float));
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  kern<<<sms * cps, 32 * warps>>>(iters / 10, sink);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<<<sms * cps, 32 * warps>>>(iters, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double insts = (double)sms * cps * warps * iters * nacc;
  const double macs = insts * macs_per_inst_per_warp;
  const double cyc = ms * 1e-3 * clk * 1e3;   // at the nominal max clock
  std::printf("%-28s warps/CTA %2d CTAs/SM %d: %8.3f ms  %7.1f TMAC/s  %7.1f MAC/clk/SM  %.3f warp-inst/clk/SM  err=%s\n", name,
              warps, cps, ms, macs / ms / 1e9, macs / cyc / sms, insts / cyc / sms, cudaGetErrorString(cudaGetLastError()));
  cudaFree(sink);
}

int main() {
  const int it = 20000;
  for (int w : {4, 8, 16}) {
    run("mma.sync tf32 m16n8k8 x4", k_tf32<4>, w, 1, it, 16 * 8 * 8, 4);
    run("mma.sync tf32 m16n8k8 x8", k_tf32<8>, w, 1, it, 16 * 8 * 8, 8);
    run("mma.sync bf16 m16n8k16 x8", k_bf16<8>, w, 1, it, 16 * 8 * 16, 8);
    run("mma.sync f64 m8n8k4 x8", k_f64<8>, w, 1, it / 4, 8 * 8 * 4, 8);
    run("ffma2 x8", k_ffma2<8>, w, 1, it * 4, 64, 8);
    run("dfma x8", k_dfma<8>, w, 1, it, 32, 8);
  }
  run("mma.sync tf32 m16n8k8 x8", k_tf32<8>, 8, 2, it, 16 * 8 * 8, 8);
  run("mma.sync tf32 m16n8k8 x8", k_tf32<8>, 16, 2, it, 16 * 8 * 8, 8);
  return 0;
}
