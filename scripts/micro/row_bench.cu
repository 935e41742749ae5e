// Micro benchmark: does the factor-row stride matter for scattered row traffic
// beyond L2?  J = 10 rows are 40 bytes of payload; stored at a 48-byte stride
// (JP = 12 floats) two rows in three straddle a 64-byte boundary, at a 64-byte
// stride (16 floats, 64-byte aligned) none does.  The epoch's pattern per
// entry: three random rows (one per mode table of 1e7 rows) are gathered
// (cp.async 16 B x 3) one entry ahead, then each gets a 3 x red.v4 step.
//   MODE 0: gathers only   MODE 1: REDs only   MODE 2: gather + RED (the epoch)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o row_bench row_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

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

template <int RS, int MODE, int WORK>
__global__ void __launch_bounds__(256) k(float* U0, float* U1, float* U2, uint32_t rows,
                                         int per_thread, float* sink) {
  extern __shared__ __align__(128) float stb[];
  float (*st)[3][256][12] = reinterpret_cast<float (*)[3][256][12]>(stb);
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  float* U[3] = {U0, U1, U2};
  float acc = 0.f;
  auto rowid = [&](int i, int n) { return hash32(t * 7919u + i * 104729u + n * 15485863u) % rows; };
  auto issue = [&](int i) {
    if (MODE != 1) {
#pragma unroll
      for (int n = 0; n < 3; ++n) {
        const float* row = U[n] + (uint64_t)rowid(i, n) * RS;
        const uint32_t sa = smem_u32(&st[i & 1][n][threadIdx.x][0]);
#pragma unroll
        for (int q = 0; q < 12; q += 4)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa + q * 4), "l"(row + q));
      }
    }
    asm volatile("cp.async.commit_group;");
  };
  issue(0);
  for (int i = 0; i < per_thread; ++i) {
    issue(i + 1);
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    float d[12];
#pragma unroll
    for (int q = 0; q < 12; ++q) d[q] = q < 10 ? 1e-6f * (float)(q + i) : 0.f;
    if (MODE != 1) acc += st[i & 1][0][threadIdx.x][0] + st[i & 1][1][threadIdx.x][1] + st[i & 1][2][threadIdx.x][2];
#pragma unroll 4
    for (int w = 0; w < WORK; ++w) acc = fmaf(acc, 0.999f, d[w % 10]);
    if (MODE != 0) {
#pragma unroll
      for (int n = 0; n < 3; ++n) {
        float* row = U[n] + (uint64_t)rowid(i, n) * RS;
        red_v4(row, make_float4(d[0], d[1], d[2], d[3]));
        red_v4(row + 4, make_float4(d[4], d[5], d[6], d[7]));
        red_v4(row + 8, make_float4(d[8], d[9], d[10], d[11]));
      }
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  if (acc == 12345.f) sink[0] = acc;
}

int main() {
  const uint32_t rows = 10000000;
  float* U[2][3];
  float* sink;
  for (int s = 0; s < 2; ++s)
    for (int n = 0; n < 3; ++n) {
      const size_t b = (size_t)rows * (s ? 64 : 48);
      cudaMalloc(&U[s][n], b);
      cudaMemset(U[s][n], 0, b);
    }
  cudaMalloc(&sink, 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](const char* name, auto kern, int s, int bps) {
    const int blocks = 148 * bps, per = 1024 / bps;
    const double n = (double)blocks * 256 * per;
    float ms = 0;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 3 * 256 * 12 * 4);
      kern<<<blocks, 256, 2 * 3 * 256 * 12 * 4>>>(U[s][0], U[s][1], U[s][2], rows, per, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
    }
    printf("%-34s blocks/SM %d: %8.3f ms  %.3g entries/s (%.3g rows/s)  %s\n", name, bps, ms,
           n / (ms * 1e-3), 3 * n / (ms * 1e-3), cudaGetErrorString(cudaGetLastError()));
  };
  for (int bps : {1, 2, 3}) {
    run("stride 48  gather", k<12, 0, 64>, 0, bps);
    run("stride 64  gather", k<16, 0, 64>, 1, bps);
    run("stride 48  red", k<12, 1, 64>, 0, bps);
    run("stride 64  red", k<16, 1, 64>, 1, bps);
    run("stride 48  gather+red", k<12, 2, 64>, 0, bps);
    run("stride 64  gather+red", k<16, 2, 64>, 1, bps);
    run("stride 48  gather+red work 512", k<12, 2, 512>, 0, bps);
    run("stride 64  gather+red work 512", k<16, 2, 512>, 1, bps);
  }
  return 0;
}
