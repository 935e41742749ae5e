// Micro test: TMA tile::gather4 of factor rows into shared memory and
// tile::scatter4 add-reduction of row deltas back (sm_100a), on a 2-D
// tensor map over a row-major factor table (rows x JP floats, box JP x 1).
// Checks values and times both against LDGSTS / per-row bulk reductions.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tma_gs4 tma_gs4.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

constexpr int JP = 12;

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16;
  return x;
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// one warp per group of 32 rows; lane l owns row r(l); lanes 4g..4g+3 share
// one gather4 / scatter4 op issued by lane 4g
__global__ void __launch_bounds__(256) gs4_kernel(const __grid_constant__ CUtensorMap tmap,
                                                  uint32_t rows, int per_thread, float* check,
                                                  int mode) {
  __shared__ __align__(128) float buf[8][8][64];  // [warp][group][4 rows x 12 floats + pad]
  __shared__ __align__(8) uint64_t mbar[8][8];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, g = l >> 2, q = l & 3;
  if (q == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar[w][g])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  float acc = 0.f;
  for (int i = 0; i < per_thread; ++i) {
    const uint32_t r = hash32(t * 7919u + i * 104729u) % rows;
    const int r0 = __shfl_sync(0xffffffffu, (int)r, l & ~3);
    const int r1 = __shfl_sync(0xffffffffu, (int)r, (l & ~3) + 1);
    const int r2 = __shfl_sync(0xffffffffu, (int)r, (l & ~3) + 2);
    const int r3 = __shfl_sync(0xffffffffu, (int)r, (l & ~3) + 3);
    float* grp = &buf[w][g][0];
    if (mode == 0) {  // gather4 + check + scatter4 reduce (+1 on cols < 10)
      if (q == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                         smem_u32(&mbar[w][g])), "r"(4 * JP * 4) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(grp)),
            "l"(&tmap), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(&mbar[w][g]))
            : "memory");
      }
      // wait for phase i of this group's barrier
      asm volatile(
          "{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }"
          ::"r"(smem_u32(&mbar[w][g])), "r"((uint32_t)(i & 1)) : "memory");
      const float* myrow = grp + q * JP;
      acc += myrow[0] + myrow[9];
      if (check && i == 0) {
        for (int k = 0; k < JP; ++k) check[(uint64_t)t * JP + k] = myrow[k];
      }
      __syncwarp();
      float* dst = grp + q * JP;
      for (int k = 0; k < JP; ++k) dst[k] = k < 10 ? 1.f : 0.f;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (q == 0) {
        asm volatile(
            "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile::scatter4.bulk_group"
            " [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(&tmap), "r"(0), "r"(r0), "r"(r1),
            "r"(r2), "r"(r3), "r"(smem_u32(grp)) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      }
      __syncwarp();
    }
  }
  if (l % 4 == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  if (acc == 12345.f) check[0] = acc;
}

int main() {
  const uint32_t rows = 10000000;
  std::vector<float> h((size_t)rows * JP, 0.f);
  for (uint32_t i = 0; i < rows; ++i)
    for (int k = 0; k < 10; ++k) h[(size_t)i * JP + k] = (float)(i % 100000) + 0.01f * k;
  float* U;
  cudaMalloc(&U, h.size() * 4);
  cudaMemcpy(U, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &qr);
  if (!encode) {
    printf("no cuTensorMapEncodeTiled\n");
    return 1;
  }
  CUtensorMap tmap;
  cuuint64_t gdim[2] = {JP, rows};
  cuuint64_t gstride[1] = {JP * 4};
  cuuint32_t box[2] = {JP, 1};
  cuuint32_t estr[2] = {1, 1};
  CUresult cr = encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, U, gdim, gstride, box, estr,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                       CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode: %d\n", (int)cr);
  const int blocks = 148, threads = 256;
  float* check;
  cudaMalloc(&check, (size_t)blocks * threads * JP * 4);
  // correctness: one iteration per thread
  gs4_kernel<<<blocks, threads>>>(tmap, rows, 1, check, 0);
  cudaError_t e = cudaDeviceSynchronize();
  printf("gather/scatter: %s\n", cudaGetErrorString(e));
  std::vector<float> hc((size_t)blocks * threads * JP);
  cudaMemcpy(hc.data(), check, hc.size() * 4, cudaMemcpyDeviceToHost);
  std::vector<float> h2(h.size());
  cudaMemcpy(h2.data(), U, h.size() * 4, cudaMemcpyDeviceToHost);
  auto hash32h = [](uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16;
    return x;
  };
  int bad_g = 0;
  std::vector<int> hits(rows, 0);
  for (uint32_t t = 0; t < (uint32_t)blocks * threads; ++t) {
    const uint32_t r = hash32h(t * 7919u) % rows;
    hits[r]++;
    for (int k = 0; k < JP; ++k)
      if (hc[(size_t)t * JP + k] != h[(size_t)r * JP + k]) { ++bad_g; break; }
  }
  int bad_s = 0, changed = 0, shown = 0;
  for (uint32_t r = 0; r < rows; ++r) {
    bool ch = false;
    for (int k = 0; k < JP; ++k) if (h2[(size_t)r * JP + k] != h[(size_t)r * JP + k]) ch = true;
    changed += ch;
    for (int k = 0; k < JP; ++k) {
      const float want = h[(size_t)r * JP + k] + (k < 10 ? (float)hits[r] : 0.f);
      if (h2[(size_t)r * JP + k] != want) {
        ++bad_s;
        if (shown < 4) {
          ++shown;
          printf("row %u hits %d: got", r, hits[r]);
          for (int kk = 0; kk < JP; ++kk) printf(" %g", h2[(size_t)r * JP + kk] - h[(size_t)r * JP + kk]);
          printf("\n");
        }
        break;
      }
    }
  }
  printf("gather4 mismatches %d, scatter4-reduce mismatched rows %d, changed rows %d\n", bad_g, bad_s, changed);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int per = 1024;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a);
    gs4_kernel<<<blocks, threads>>>(tmap, rows, per, nullptr, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (rep == 2)
      printf("gather4+scatter4 round trips: %.3f ms  %.3g rows/s  %s\n", ms,
             (double)blocks * threads * per / (ms * 1e-3), cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
