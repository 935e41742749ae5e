// Microbenchmark: sustained rate of mma.sync m16n8k8 TF32 (HMMA.1688) and of
// 3-register FFMA on one B200, 148 blocks x NW warps, independent chains.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void mma_tf32(float* d, const uint32_t* a, const uint32_t* b) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 "
      "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

template <int CH>
__global__ void mma_kernel(float* out, int iters) {
  uint32_t a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = __float_as_uint(1.0f + threadIdx.x * 1e-3f + i);
  for (int i = 0; i < 2; ++i) b[i] = __float_as_uint(0.5f + i);
  float d[CH][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) mma_tf32(d[c], a, b);
  }
  float s = 0.f;
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  if (s == 12345.f) out[0] = s;
}

template <int CH>
__global__ void ffma_kernel(float* out, int iters, float x, float y) {
  float acc[CH];
  float m[CH];
  float yy[CH];
  for (int c = 0; c < CH; ++c) { acc[c] = threadIdx.x * 1e-3f + c; m[c] = x + c * 1e-4f; yy[c] = y * (threadIdx.x + c); }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = fmaf(acc[c], m[c], yy[c]);
  }
  float s = 0.f;
  for (int c = 0; c < CH; ++c) s += acc[c];
  if (s == 12345.f) out[0] = s;
}

int main() {
  float* out;
  cudaMalloc(&out, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int nw : {4, 8, 16}) {
    const int iters = 20000;
    mma_kernel<8><<<sms, nw * 32>>>(out, 100);
    cudaEventRecord(e0);
    mma_kernel<8><<<sms, nw * 32>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double mmas = (double)sms * nw * iters * 8;
    printf("mma.sync m16n8k8 tf32: warps/SM %2d  %.3e warp-mma/s  %.1f TFLOP/s  %.2f mma/clk/SM @1.9GHz\n",
           nw, mmas / (ms * 1e-3), mmas * 2048 / (ms * 1e-3) / 1e12, mmas / (ms * 1e-3) / sms / 1.9e9);
  }
  for (int nw : {4, 8, 16, 32}) {
    const int iters = 20000;
    ffma_kernel<8><<<sms, nw * 32>>>(out, 100, 1.0001f, 1e-7f);
    cudaEventRecord(e0);
    ffma_kernel<8><<<sms, nw * 32>>>(out, iters, 1.0001f, 1e-7f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double f = (double)sms * nw * 32 * iters * 8;
    printf("ffma (reg,reg,reg):    warps/SM %2d  %.1f TFLOP/s  %.1f lane-FMA/clk/SM @1.9GHz\n", nw,
           2 * f / (ms * 1e-3) / 1e12, f / (ms * 1e-3) / sms / 1.9e9);
  }
  return 0;
}
