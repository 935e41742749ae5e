// umma_test.cu -- validates the tcgen05 TF32 MMA patterns used by the
// order-3 tensor-memory epoch kernel (hog3tm) against a host fp64 GEMM:
//   1. T[e][ab]  = U3[e][c] * G[c][ab]       A K-major (rows e),  B K-major (rows ab)
//   2. g3[e][c]  = P[e][ab] * G[ab][c]       A K-major (rows e),  B MN-major (G buffer)
//   3. Dc[ab][c] = P^T[ab][e] * S[e][c]      A MN-major (P buffer), B MN-major (S buffer)
// Variant 0 (LBO = K-direction stride, SBO = row-direction stride, every
// operand K-major) is the layout the kernels use; exit status 1 if it is off.
// Variant 2 reads two operands as MN-major: tf32 MN-major operands come back
// as zeros on B200, which is why the kernels never use them.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I ../../paper_1708_08640_b200/csrc umma_test.cu -o umma_test
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "umma.cuh"

using namespace cmtfb;

constexpr int E = 128;   // entries (M of MMA 1/2, K of MMA 3)
constexpr int C = 16;    // padded c
constexpr int AB = 104;  // padded ab (K of MMA 2)
constexpr int ABM = 128; // M of MMA 3

// byte offset of element (r, k) in a buffer tiled in core matrices of
// 8 rows x 4 cols; `rs` = stride between row groups of 8, `ks` = between col
// groups of 4.
__host__ __device__ inline uint32_t off(int r, int k, uint32_t rs, uint32_t ks) {
  return (r / 8) * rs + (k / 4) * ks + (r % 8) * 16 + (k % 4) * 4;
}

// smem: U3 [E rows][C cols]  (rows e): rs=128, ks=E/8*128=2048
//       G  [AB rows (ab)][C cols (c)]: rs=128, ks=AB/8*128=1664 (+ pad to 128 rows)
//       P  [E rows][ABM cols]        : rs=128, ks=2048
//       S  [E rows][C cols]          : rs=128, ks=2048
struct Res { float T[E][112]; float g3[E][16]; float Dc[ABM][16]; };

__global__ void kern(const float* U3, const float* G, const float* P, const float* S, Res* out,
                     int variant) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sU3 = sm;                    // 8 KB
  uint8_t* sG = sU3 + E * C * 4;        // 128 rows x 16 -> 8 KB
  uint8_t* sP = sG + 128 * C * 4;       // 64 KB
  uint8_t* sS = sP + E * ABM * 4;       // 8 KB
  uint8_t* sGt = sS + E * C * 4;        // [16 c][128 ab] 8 KB (rs 128, ks 256)
  uint8_t* sPt = sGt + 16 * 128 * 4;    // [128 ab][128 e] 64 KB (rs 128, ks 2048)
  uint8_t* sSt = sPt + 128 * 128 * 4;   // [16 c][128 e] 8 KB (rs 128, ks 256)
  __shared__ uint64_t mbar;
  __shared__ uint32_t tbase;
  const int t = threadIdx.x;
  for (int i = t; i < E * C; i += blockDim.x) {
    int r = i / C, k = i % C;
    *(float*)(sU3 + off(r, k, 128, 2048)) = U3[i];
    *(float*)(sS + off(r, k, 128, 2048)) = S[i];
  }
  for (int i = t; i < 128 * C; i += blockDim.x) {
    int r = i / C, k = i % C;
    *(float*)(sG + off(r, k, 128, 2048)) = r < AB ? G[r * C + k] : 0.f;
  }
  for (int i = t; i < E * ABM; i += blockDim.x) {
    int r = i / ABM, k = i % ABM;
    *(float*)(sP + off(r, k, 128, 2048)) = P[i];
  }
  for (int i = t; i < 16 * 128; i += blockDim.x) {
    int c = i / 128, x = i % 128;
    *(float*)(sGt + off(c, x, 128, 256)) = x < AB ? G[x * C + c] : 0.f;
    *(float*)(sSt + off(c, x, 128, 256)) = S[x * C + c];
  }
  for (int i = t; i < 128 * 128; i += blockDim.x) {
    int ab = i / 128, e = i % 128;
    *(float*)(sPt + off(ab, e, 128, 2048)) = P[e * ABM + ab];
  }
  if (t == 0) { umma::mbar_init(&mbar, 1); umma::fence_mbar_init(); }
  if (t < 32) umma::tmem_alloc<256>(&tbase);
  umma::fence_async_smem();
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tb = tbase;
  const bool sw = variant & 1;
  auto D = [&](const void* p, uint32_t kstride, uint32_t rstride) {
    // variant 0: LBO = K-direction stride, SBO = row-direction stride
    return sw ? umma::desc(umma::smem_u32(p), rstride, kstride)
              : umma::desc(umma::smem_u32(p), kstride, rstride);
  };
  const bool sw2 = variant & 2;  // MN-major operands
  auto Dmn = [&](const void* p, uint32_t mnstride, uint32_t kstride) {
    return sw2 ? umma::desc(umma::smem_u32(p), kstride, mnstride)
               : umma::desc(umma::smem_u32(p), mnstride, kstride);
  };
  if (t == 0) {
    // 1: T[128 x 112] = U3[128 x 16] * G^T ; B K-major rows = ab (N), cols = c (K)
    const uint32_t id1 = umma::idesc_tf32(128, 112, false, false);
    for (int k = 0; k < C / 8; ++k)
      umma::mma_tf32(tb + 0, D(sU3 + k * 2 * 2048, 2048, 128), D(sG + k * 2 * 2048, 2048, 128),
                     id1, k > 0);
    // 2: g3[128 x 16] = P[128 x 104] * G[104 x 16]; B MN-major: rows = ab (K), 16B along c (N)
    if (variant == 0) {
    const uint32_t id2 = umma::idesc_tf32(128, 16, false, false);
    for (int k = 0; k < AB / 8; ++k)
      umma::mma_tf32(tb + 112, D(sP + k * 2 * 2048, 2048, 128), D(sGt + k * 2 * 256, 256, 128), id2,
                     k > 0);
    } else {
    const uint32_t id2 = umma::idesc_tf32(128, 16, false, true);
    for (int k = 0; k < AB / 8; ++k)
      umma::mma_tf32(tb + 112, D(sP + k * 2 * 2048, 2048, 128), Dmn(sG + k * 128, 2048, 128), id2,
                     k > 0);
    }
    // 3: Dc[128 x 16] = P^T[128(ab) x 128(e)] * S[128(e) x 16]; A MN-major (16B along ab),
    //    B MN-major (16B along c)
    if (variant == 0) {
    const uint32_t id3 = umma::idesc_tf32(128, 16, false, false);
    for (int k = 0; k < E / 8; ++k)
      umma::mma_tf32(tb + 128, D(sPt + k * 2 * 2048, 2048, 128), D(sSt + k * 2 * 256, 256, 128), id3,
                     k > 0);
    } else {
    const uint32_t id3 = umma::idesc_tf32(128, 16, true, true);
    for (int k = 0; k < E / 8; ++k)
      umma::mma_tf32(tb + 128, Dmn(sP + k * 128, 2048, 128), Dmn(sS + k * 128, 2048, 128), id3,
                     k > 0);
    }
    umma::commit(&mbar);
  }
  umma::mbar_wait(&mbar, 0);
  umma::fence_after();
  const int w = t >> 5;
  const uint32_t lane_base = (uint32_t)(32 * (w & 3)) << 16;
  const int row = 32 * (w & 3) + (t & 31);
  float v[16];
  for (int c0 = 0; c0 < 144; c0 += 16) {
    umma::ld16(tb + lane_base + c0, v);
    umma::ld_wait();
    umma::ld_fence_regs<16>(v);
    for (int i = 0; i < 16; ++i) {
      int col = c0 + i;
      if (col < 112) out->T[row][col] = v[i];
      else if (col < 128) out->g3[row][col - 112] = v[i];
      else out->Dc[row][col - 128] = v[i];
    }
  }
  umma::fence_before();
  __syncthreads();
  if (t < 32) umma::tmem_free<256>(tb);
}

int main() {
  srand(1);
  auto rnd = [] { return (float)rand() / RAND_MAX - 0.5f; };
  std::vector<float> U3(E * C), G(AB * C), P(E * ABM), S(E * C);
  for (auto& x : U3) x = rnd();
  for (auto& x : G) x = rnd();
  for (auto& x : P) x = rnd();
  for (auto& x : S) x = rnd();
  float *dU3, *dG, *dP, *dS; Res* dR;
  cudaMalloc(&dU3, U3.size() * 4); cudaMalloc(&dG, G.size() * 4);
  cudaMalloc(&dP, P.size() * 4); cudaMalloc(&dS, S.size() * 4); cudaMalloc(&dR, sizeof(Res));
  cudaMemcpy(dU3, U3.data(), U3.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dG, G.data(), G.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dP, P.data(), P.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dS, S.data(), S.size() * 4, cudaMemcpyHostToDevice);
  const int smem = E * C * 4 + 128 * C * 4 + E * ABM * 4 + E * C * 4 + 16*128*4*2 + 128*128*4;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  Res* h = new Res;
  int bad = 0;
  for (int variant = 0; variant < 4; variant += 2) {
    cudaMemset(dR, 0, sizeof(Res));
    kern<<<1, 128, smem>>>(dU3, dG, dP, dS, dR, variant);
    cudaError_t err = cudaDeviceSynchronize();
    if (err != cudaSuccess) { printf("variant %d: CUDA error %s\n", variant, cudaGetErrorString(err)); return 1; }
    cudaMemcpy(h, dR, sizeof(Res), cudaMemcpyDeviceToHost);
    double e1 = 0, e2 = 0, e3 = 0, m1 = 0, m2 = 0, m3 = 0;
    for (int e = 0; e < E; ++e)
      for (int ab = 0; ab < 112; ++ab) {
        double s = 0;
        if (ab < AB) for (int c = 0; c < C; ++c) s += (double)U3[e * C + c] * G[ab * C + c];
        e1 = fmax(e1, fabs(s - h->T[e][ab])); m1 = fmax(m1, fabs(s));
      }
    for (int e = 0; e < E; ++e)
      for (int c = 0; c < C; ++c) {
        double s = 0;
        for (int ab = 0; ab < AB; ++ab) s += (double)P[e * ABM + ab] * G[ab * C + c];
        e2 = fmax(e2, fabs(s - h->g3[e][c])); m2 = fmax(m2, fabs(s));
      }
    for (int ab = 0; ab < ABM; ++ab)
      for (int c = 0; c < C; ++c) {
        double s = 0;
        for (int e = 0; e < E; ++e) s += (double)P[e * ABM + ab] * S[e * C + c];
        e3 = fmax(e3, fabs(s - h->Dc[ab][c])); m3 = fmax(m3, fabs(s));
      }
    printf("  g3[0][0..3] got %g %g %g %g   Dc[0][0..3] got %g %g %g %g\n", h->g3[0][0], h->g3[0][1], h->g3[0][2], h->g3[0][3], h->Dc[0][0], h->Dc[0][1], h->Dc[0][2], h->Dc[0][3]);
    printf("variant %d (K-major swap %d, MN-major swap %d): T err %.3g/%.3g  g3 err %.3g/%.3g  "
           "Dc err %.3g/%.3g\n", variant, variant & 1, (variant >> 1) & 1, e1, m1, e2, m2, e3, m3);
    // TF32 operands: ~2^-11 relative per product
    if (variant == 0 && (e1 > 2e-3 * m1 || e2 > 2e-3 * m2 || e3 > 2e-3 * m3)) bad = 1;
  }
  printf(bad ? "UMMA descriptors: FAIL\n" : "UMMA descriptors: ok\n");
  return bad;
}
