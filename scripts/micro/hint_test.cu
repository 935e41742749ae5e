// Which L2 cache-hint forms run on sm_100a: createpolicy kinds, cp.async /
// red.v4 / ld / st with .L2::cache_hint.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int KIND>
__device__ uint64_t pol() {
  uint64_t p;
  if (KIND == 0) asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  if (KIND == 1) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  if (KIND == 2) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  if (KIND == 3) asm volatile("createpolicy.fractional.L2::evict_last.L2::evict_unchanged.b64 %0, 1.0;" : "=l"(p));
  return p;
}
template <int KIND, int OP>
__global__ void k(float* U, float* out) {
  __shared__ __align__(16) float st[32 * 4];
  const uint64_t p = pol<KIND>();
  float* row = U + threadIdx.x * 4;
  if (OP == 0) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(st + threadIdx.x * 4);
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(d), "l"(row), "l"(p) : "memory");
    asm volatile("cp.async.wait_all;" ::: "memory");
    out[threadIdx.x] = st[threadIdx.x * 4];
  } else if (OP == 1) {
    asm volatile("red.relaxed.gpu.global.add.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(row),
                 "f"(1.f), "f"(1.f), "f"(1.f), "f"(1.f), "l"(p) : "memory");
  } else if (OP == 2) {
    float4 v;
    asm volatile("ld.global.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(row), "l"(p) : "memory");
    out[threadIdx.x] = v.x;
  } else if (OP == 3) {
    asm volatile("red.relaxed.gpu.global.add.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(row), "f"(1.f), "l"(p) : "memory");
  } else if (OP == 4) {
    asm volatile("red.global.add.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(row),
                 "f"(1.f), "f"(1.f), "f"(1.f), "f"(1.f), "l"(p) : "memory");
  }
}
template <int KIND, int OP>
void run(float* U, float* out) {
  k<KIND, OP><<<1, 32>>>(U, out);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kind %d op %d: %s\n", KIND, OP, cudaGetErrorString(e));
  if (e != cudaSuccess) exit(1);
}
int main(int argc, char** argv) {
  float *U, *out;
  cudaMalloc(&U, 4096);
  cudaMalloc(&out, 4096);
  cudaMemset(U, 0, 4096);
  const int which = argc > 1 ? atoi(argv[1]) : 0;
  switch (which) {
    case 0: run<0, 0>(U, out); break;
    case 1: run<1, 0>(U, out); break;
    case 2: run<2, 0>(U, out); break;
    case 3: run<3, 0>(U, out); break;
    case 4: run<1, 1>(U, out); break;
    case 5: run<1, 2>(U, out); break;
    case 6: run<1, 3>(U, out); break;
    case 7: run<1, 4>(U, out); break;
    case 8: run<0, 1>(U, out); break;
    case 9: run<2, 1>(U, out); break;
  }
  return 0;
}
