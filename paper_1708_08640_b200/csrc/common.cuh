// common.cuh -- shared device helpers for the S^3CMTF B200 kernels.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace cmtfb {

constexpr int kMaxOrder = 16;    // as the reference (src/gradients.cpp:14, src/tucker.cpp:13)
constexpr int kMaxRank = 64;     // per-mode rank bound of the device path
constexpr int kEvalBlock = 1024; // src/eval.cpp:10 (kBlock)

__host__ __device__ constexpr int round_up4(int j) { return (j + 3) & ~3; }

// Hogwild parameter access (the reference's relaxed.hpp:13-20 contract):
// rows are shared mutably between concurrent workers.  Loads bypass L1
// (L1 is not coherent across SMs, so an L1 hit could return a row this SM
// read long ago); stores are plain global stores, which land in L2.
// Lost updates and stale reads are allowed by design.
#ifndef CMTF_ROW_LOAD
#define CMTF_ROW_LOAD 0
#endif
__device__ __forceinline__ float4 ld_row4(const float* p) {
#if CMTF_ROW_LOAD == 0
  return __ldcg(reinterpret_cast<const float4*>(p));
#else
  return *reinterpret_cast<const float4*>(p);
#endif
}
__device__ __forceinline__ float ld_row1(const float* p) {
#if CMTF_ROW_LOAD == 0
  return __ldcg(p);
#else
  return *p;
#endif
}
__device__ __forceinline__ void st_row4(float* p, float4 v) {
#if CMTF_ROW_LOAD == 2
  *reinterpret_cast<float4*>(p) = v;
#else
  __stcg(reinterpret_cast<float4*>(p), v);
#endif
}
__device__ __forceinline__ void st_row1(float* p, float v) {
#if CMTF_ROW_LOAD == 2
  *p = v;
#else
  __stcg(p, v);
#endif
}

// Per-mode/per-matrix device tables passed by value to kernels.
struct ModeTables {
  float* U[kMaxOrder];          // factor rows, I_n x JP_n (JP_n = round_up4)
  const float* reg[kMaxOrder];  // lambda / count_n(i), 0 where count is 0
  const uint32_t* count[kMaxOrder];
  uint32_t J[kMaxOrder];
  uint32_t JP[kMaxOrder];
  uint32_t dims[kMaxOrder];
};

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace cmtfb
