// Micro benchmark: scattered 48-byte row updates (the epoch's cold-row step
// pattern: J = 10 floats padded to 12) into a large factor array, issued as
//   (0) three red.global.add.v4.f32 per row (the current hog3tm step),
//   (1) one cp.reduce.async.bulk.global.shared::cta.add.f32 of 48 bytes per
//       row from a shared-memory staging row (registers free at issue),
//   (2) a plain gather (3 x cp.async 16 B) + wait, for reference.
// Every thread owns a stream of random rows; `rows_per_thread` updates each.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o red_bench red_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#ifndef WORK
#define WORK 64
#endif
__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16;
  return x;
}
__device__ __forceinline__ void red_v4(float* p, float4 v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w) : "memory");
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

template <int MODE, int DEPTH>
__global__ void __launch_bounds__(256) k(float* U, uint32_t rows, int per_thread, float* sink) {
  __shared__ __align__(128) float st[DEPTH + 1][256][12];
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  float acc = 0.f;
  for (int i = 0; i < per_thread; ++i) {
    const uint32_t r = hash32(t * 7919u + i * 104729u) % rows;
    float* row = U + (uint64_t)r * 12;
    const int s = i % (DEPTH + 1);
    float d[12];
#pragma unroll
    for (int q = 0; q < 12; ++q) d[q] = q < 10 ? 1e-6f * (float)(q + i) : 0.f;
    if (MODE == 0) {
      red_v4(row, make_float4(d[0], d[1], d[2], d[3]));
      red_v4(row + 4, make_float4(d[4], d[5], d[6], d[7]));
      red_v4(row + 8, make_float4(d[8], d[9], d[10], d[11]));
    } else if (MODE == 1) {
      // the staging row of two iterations ago must have been read
      asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(DEPTH) : "memory");
#pragma unroll
      for (int q = 0; q < 12; q += 4)
        *reinterpret_cast<float4*>(&st[s][threadIdx.x][q]) = make_float4(d[q], d[q + 1], d[q + 2], d[q + 3]);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], 48;"
                   ::"l"(row), "r"(smem_u32(&st[s][threadIdx.x][0])) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    } else {
      const uint32_t sa = smem_u32(&st[s][threadIdx.x][0]);
#pragma unroll
      for (int q = 0; q < 12; q += 4)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa + q * 4), "l"(row + q));
      asm volatile("cp.async.commit_group;");
      asm volatile("cp.async.wait_group %0;" ::"n"(DEPTH) : "memory");
      acc += st[(i + 1) % (DEPTH + 1)][threadIdx.x][0];
    }
    // a little independent work between updates (the epoch does ~1.5k instr/entry)
#pragma unroll 4
    for (int w = 0; w < WORK; ++w) acc = fmaf(acc, 0.999f, d[w % 10]);
  }
  if (MODE == 1) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  if (MODE == 2) asm volatile("cp.async.wait_all;" ::: "memory");
  if (acc == 12345.f) sink[0] = acc;
}

int main() {
  const uint32_t rows = 10000000;  // 1e7 rows x 48 B = 480 MB (L2 misses)
  float* U;
  float* sink;
  cudaMalloc(&U, (size_t)rows * 48);
  cudaMalloc(&sink, 4);
  cudaMemset(U, 0, (size_t)rows * 48);
  const int threads = 256;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](const char* name, auto kern, int bps, int depth) {
    const int blocks = 148 * bps, per = 2048 / bps;
    const double n = (double)blocks * threads * per;
    float ms = 0;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      kern<<<blocks, threads>>>(U, rows, per, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
    }
    printf("%-26s blocks/SM %d depth %d: %8.3f ms  %.3g rows/s  %s\n", name, bps, depth, ms,
           n / (ms * 1e-3), cudaGetErrorString(cudaGetLastError()));
  };
  for (int bps : {1, 2, 4}) {
    run("red.v4 x3", k<0, 1>, bps, 0);
    run("cp.reduce.async.bulk 48B", k<1, 1>, bps, 1);
    run("cp.reduce.async.bulk 48B", k<1, 3>, bps, 3);
    run("cp.async gather 3x16B", k<2, 1>, bps, 1);
    run("cp.async gather 3x16B", k<2, 3>, bps, 3);
    run("cp.async gather 3x16B", k<2, 2>, bps, 2);
  }
  return 0;
}
