// launch.cuh -- host-side launch helpers shared by the translation units of libtnb200.so:
// shape classification of a bucket step / fused group and the per-kernel launch entry points
// (launch_bucket.cu: k_bucket; launch_group_c64.cu / launch_group_c128.cu: k_group_t;
// launch_pair.cu: k_pair; launch_gemm.cu: k_gemm).  Split so nvcc compiles them in parallel.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <type_traits>
#include <utility>
#include <vector>

#include "kernels.cuh"

namespace tnb {

// opt in to more than 48 KB of (static + dynamic) shared memory, once per (device, kernel
// instantiation): cudaFuncSetAttribute applies to the current device
template <typename K>
inline void allow_smem(K kernel, size_t dyn) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> granted;
  if (dyn + 16 * 1024 <= 48 * 1024) return;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  size_t& g = granted[{dev, reinterpret_cast<const void*>(kernel)}];
  if (dyn > g) {
    const size_t want = std::max<size_t>(dyn, 100 * 1024);
    if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)want) == cudaSuccess)
      g = want;
    else
      (void)cudaGetLastError();   // the launch then fails and reports the error
  }
}

inline bool debug_checks() {
  static const int on = [] {
    const char* v = std::getenv("TNB_DEBUG");
    return (v && v[0] == '1') ? 1 : 0;
  }();
  return on != 0;
}
inline int num_sms() {
  static int g_num_sms = 0;
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

inline uint64_t host_pext(uint64_t x, uint64_t m) {
  uint64_t r = 0;
  int k = 0;
  while (m) {
    const uint64_t b = m & (~m + 1);
    if (x & b) r |= 1ull << k;
    ++k;
    m ^= b;
  }
  return r;
}

// ---------------------------------------------------------------- k_group_t host side
struct GIn {
  const void* ptr;
  uint64_t out_mask;   // output bits present (relative to the group output)
  uint32_t pv;         // F_t(o) = ins0(pext(o, out_mask), pv)
  uint32_t rank;       // bits of the input (for 32/64-bit offsets)
  bool full;           // holds every output bit and every summed bit (read exactly once)
  uint64_t gx[1 << kMaxGroup];
};
struct GDesc {
  void* out;
  int out_rank;
  int M;
  int n;
  GIn in[kMaxIn];
};

inline uint64_t host_fmap(uint64_t o, uint64_t mask, uint32_t pv) {
  const uint64_t r = host_pext(o, mask);
  const uint64_t lo = r & ((1ull << pv) - 1);
  return lo | ((r >> pv) << (pv + 1));
}

inline bool env_flag(const char* name) {
  const char* v = std::getenv(name);
  return v && v[0] == '1';
}
inline bool env_flag0(const char* name) {   // set to "0"
  const char* v = std::getenv(name);
  return v && v[0] == '0';
}
inline int gemm_stages() {   // TNB_GEMM_STAGES=2..4 (default 3)
  static const int s = [] {
    const char* v = std::getenv("TNB_GEMM_STAGES");
    const int x = v ? std::atoi(v) : 3;
    return x < 2 ? 2 : (x > 4 ? 4 : x);
  }();
  return s;
}
constexpr int kMaxLanes = 32;
inline int slice_lanes() {   // TNB_LANES=1..32 (default 16); TNB_ONE_LANE=1 == 1
  static const int n = [] {
    if (env_flag("TNB_ONE_LANE")) return 1;
    const char* v = std::getenv("TNB_LANES");
    const int x = v ? std::atoi(v) : 16;
    return x < 1 ? 1 : (x > kMaxLanes ? kMaxLanes : x);
  }();
  return n;
}
inline bool gemm_disabled() {
  static const bool off = env_flag("TNB_NO_GEMM");
  return off;
}

// TNB_GEMM_DEBUG: one line per input of a group: rank, output bits held (bit 0 first), and which
// summed values x it varies over (distinct gx rows)
inline void debug_group(const char* tag, const GDesc& g) {
  std::fprintf(stderr, "  %s R=%d M=%d n=%d\n", tag, g.out_rank, g.M, g.n);
  for (int t = 0; t < g.n; ++t) {
    char bits[65];
    for (int b = 0; b < g.out_rank && b < 64; ++b) bits[b] = ((g.in[t].out_mask >> b) & 1) ? '1' : '.';
    bits[g.out_rank < 64 ? g.out_rank : 64] = 0;
    int nrow = 0;
    uint64_t seen[1 << kMaxGroup];
    for (int x = 0; x < (1 << g.M); ++x) {
      bool f = false;
      for (int r = 0; r < nrow; ++r) f = f || seen[r] == g.in[t].gx[x];
      if (!f) seen[nrow++] = g.in[t].gx[x];
    }
    std::fprintf(stderr, "    in%d rank=%u rows=%d pv=%u %s\n", t, g.in[t].rank, nrow, g.in[t].pv, bits);
  }
}


// which kernel the last launcher on this thread used (per-launch profile records)
enum KernelId : int { KID_NONE = 0, KID_BUCKET = 1, KID_CHAIN = 2, KID_GROUP = 3, KID_PAIR = 4,
                      KID_GEMM = 5, KID_CHAIN_SPLIT = 6, KID_PROGRAM = 7,
                      KID_GEMM_TC = 8, KID_GEMM_FC = 9, KID_FC_TC = 10, KID_GEMM_HM = 11, KID_FC_HM = 12 };
inline int& last_kernel() {
  static thread_local int k = KID_NONE;
  return k;
}

// entry points (explicitly instantiated for float2 and double2 in their translation units);
// each returns false when the shape has no instantiation / does not qualify
template <typename T> bool try_launch_gemm(const GDesc& g, cudaStream_t st);   // k_gemm_tc first (c64), else k_gemm
bool try_launch_gemm_tc(const GDesc& g, cudaStream_t st);
// the same GEMM groups on mma.sync tf32 (k_gemm_hm, c64, 3xTF32); false when the shape does not qualify
bool try_launch_gemm_hm(const GDesc& g, cudaStream_t st);
bool gemm_hm_enabled();                                                          // TNB_GEMM_HM=0 off
// c128 groups on mma.sync f64 (k_gemm_hm64); false when the shape does not qualify
bool try_launch_gemm_hm64(const GDesc& g, cudaStream_t st);
// producer group g on mma.sync tf32 consumed by g3 in registers (k_fc_hm); false when it does not qualify
bool try_launch_fc_hm(const GDesc& g, const GDesc& g3, int tin, cudaStream_t st);
bool fc_hm_enabled();                                                            // TNB_FC_HM=0 off
bool gemm_tc_enabled();                                                          // TNB_GEMM_TC=1
// producer group g (GEMM-shaped) computed tile by tile and consumed by group g3 (its input tin)
// sem: kFcSemPerOp zeroed counters owned by this launch site (k_gemm_fc's split consumer blocks;
// nullptr: whole blocks per CTA)
constexpr int kFcSemPerOp = 1024;
template <typename T> bool try_launch_gemm_fc(const GDesc& g, const GDesc& g3, int tin, cudaStream_t st,
                                              uint32_t* sem = nullptr);
// the same pair with the producer GEMM on tcgen05 (k_fc_tc, c64); false when the shape does not qualify
bool try_launch_fc_tc(const GDesc& g, const GDesc& g3, int tin, cudaStream_t st);
bool fc_tc_enabled();                                                            // TNB_FC_TC=0/1
bool fc_enabled();                                                               // TNB_NO_FC=1 off
template <typename T> bool try_launch_gemm_simt(const GDesc& g, cudaStream_t st);   // k_gemm only                        // tcgen05 kind::tf32, c64
template <typename T> bool try_launch_pair(const GDesc& g, cudaStream_t st);
template <typename T> bool try_launch_group(const GDesc& g, cudaStream_t st);
template <typename T> void launch_bucket_generic(const BigArgs& a, cudaStream_t st);   // k_bucket<T, n_in>

}  // namespace tnb
