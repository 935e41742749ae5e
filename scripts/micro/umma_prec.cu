// umma_prec.cu -- checks the tcgen05 kind::f16 operand layouts and the split
// (hi + lo) fp16 arithmetic that the order-3 epoch kernel (hog3tm) uses,
// against a host fp64 GEMM:
//   A. T[e][n] = sum_c U[e][c] G[n][c]    A K-major (rows e), B K-major (rows n),
//      three MMAs: Uhi*Ghi + Uhi*Glo + Ulo*Ghi
//   B. D[ab][c] = sum_e P[e][ab] S[e][c]  A MN-major (P rows written per entry),
//      B MN-major (S rows written per entry), entries in four 32-entry warp
//      slices sharing two slots (warps w and w+2 take turns), one accumulator
//      per slot, three MMAs per K step
// The MN-major descriptor convention is selected by `variant` (0: LBO = K
// stride, SBO = MN stride -- CUTLASS's SWIZZLE_NONE; 1: swapped).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I ../../paper_1708_08640_b200/csrc umma_prec.cu -o umma_prec
#include <cuda_fp16.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "umma.cuh"

using namespace cmtfb;

constexpr int E = 128, C = 16, NT = 112, JJ = 10, AB = 100;
constexpr float SU = 64.f, SG = 64.f, SP = 256.f, SS = 256.f;

__host__ __device__ constexpr uint32_t idesc_f16mn(int M, int N, bool amn, bool bmn) {
  return (1u << 4) | ((amn ? 1u : 0u) << 15) | ((bmn ? 1u : 0u) << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

struct Res {
  float T[E][NT];
  float T1[E][NT];  // hi only
  float D[128][16];
  float D1[128][16];
};

__device__ inline void split(float x, __half& h, __half& l) {
  h = __float2half_rn(x);
  l = __float2half_rn(x - __half2float(h));
}

__global__ void kern(const float* U, const float* G, const float* P, const float* S, Res* out,
                     int variant) {
  extern __shared__ __align__(1024) uint8_t sm[];
  // A: U hi/lo tiles [128 e][16 c] K-major: SBO 128 (8-row groups), LBO 2048 (K groups)
  uint8_t* Uh = sm;
  uint8_t* Ul = Uh + 4096;
  // G hi/lo [112 n][16 c] K-major: SBO 128, LBO 1792
  uint8_t* Gh = Ul + 4096;
  uint8_t* Gl = Gh + 3584;
  // B: per slot P hi/lo [128 ab][32 e] MN-major (8 KB each), S hi/lo [16 c][32 e] (1 KB each)
  uint8_t* slots = Gl + 3584;  // 2 slots x (Ph, Pl, Sh, Sl) = 2 x 18 KB
  constexpr int SLOT = 2 * 8192 + 2 * 1024;
  __shared__ uint64_t mbar[3];
  __shared__ uint32_t tbase;
  const int t = threadIdx.x, w = t >> 5, lane = t & 31;
  for (int i = t; i < (int)(8192 + 7168 + 2 * SLOT) / 4; i += blockDim.x)
    reinterpret_cast<float*>(sm)[i] = 0.f;
  __syncthreads();
  // thread t owns entry t: its U row and its P / S rows
  {
    for (int c = 0; c < C; ++c) {
      __half h, l;
      split(U[t * C + c] * SU, h, l);
      const int off = (t / 8) * 128 + (c / 8) * 2048 + (t % 8) * 16 + (c % 8) * 2;
      *reinterpret_cast<__half*>(Uh + off) = h;
      *reinterpret_cast<__half*>(Ul + off) = l;
    }
  }
  for (int i = t; i < NT * C; i += blockDim.x) {
    const int n = i / C, c = i % C;
    __half h, l;
    split(n < AB && c < JJ ? G[n * C + c] * SG : 0.f, h, l);
    const int off = (n / 8) * 128 + (c / 8) * 1792 + (n % 8) * 16 + (c % 8) * 2;
    *reinterpret_cast<__half*>(Gh + off) = h;
    *reinterpret_cast<__half*>(Gl + off) = l;
  }
  if (t == 0) {
    umma::mbar_init(&mbar[0], 1);
    umma::mbar_init(&mbar[1], 1);
    umma::mbar_init(&mbar[2], 1);
    umma::fence_mbar_init();
  }
  if (w == 0) umma::tmem_alloc<512>(&tbase);
  umma::fence_async_smem();
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tb = tbase;
  // ---- A: sweep, 3 terms into cols [0,112), hi only into [112, 224) ----
  if (t == 0) {
    const uint32_t id = idesc_f16mn(128, NT, false, false);
    const uint32_t uh = umma::smem_u32(Uh), ul = umma::smem_u32(Ul);
    const uint32_t gh = umma::smem_u32(Gh), gl = umma::smem_u32(Gl);
    umma::mma_f16(tb, umma::desc(uh, 2048, 128), umma::desc(gh, 1792, 128), id, 0);
    umma::mma_f16(tb, umma::desc(uh, 2048, 128), umma::desc(gl, 1792, 128), id, 1);
    umma::mma_f16(tb, umma::desc(ul, 2048, 128), umma::desc(gh, 1792, 128), id, 1);
    umma::mma_f16(tb + NT, umma::desc(uh, 2048, 128), umma::desc(gh, 1792, 128), id, 0);
    umma::commit(&mbar[2]);
  }
  // ---- B: warps take turns on two slots ----
  {
    const int slot = w & 1, turn = w >> 1;
    uint8_t* sb = slots + slot * SLOT;
    uint8_t *Ph = sb, *Pl = sb + 8192, *Sh = sb + 16384, *Sl = sb + 17408;
    if (turn == 1) umma::mbar_wait(&mbar[slot], 0);
    const int el = lane;  // K index within the slot
    for (int j = 0; j < 16; ++j) {  // 8-wide ab chunks
      __align__(16) __half h[8], l[8];
      for (int q = 0; q < 8; ++q) {
        const int ab = 8 * j + q;
        split(P[t * 128 + ab] * SP, h[q], l[q]);
      }
      const int off = variant == 0 ? j * 512 + (el / 8) * 128 + (el % 8) * 16
                                   : j * 128 + (el / 8) * 2048 + (el % 8) * 16;
      *reinterpret_cast<uint4*>(Ph + (variant == 0 ? off : off % 8192)) = *reinterpret_cast<uint4*>(h);
      *reinterpret_cast<uint4*>(Pl + (variant == 0 ? off : off % 8192)) = *reinterpret_cast<uint4*>(l);
    }
    for (int j = 0; j < 2; ++j) {
      __align__(16) __half h[8], l[8];
      for (int q = 0; q < 8; ++q) split(S[t * 16 + 8 * j + q] * SS, h[q], l[q]);
      const int off = j * 512 + (el / 8) * 128 + (el % 8) * 16;
      *reinterpret_cast<uint4*>(Sh + off) = *reinterpret_cast<uint4*>(h);
      *reinterpret_cast<uint4*>(Sl + off) = *reinterpret_cast<uint4*>(l);
    }
    umma::fence_async_smem();
    __syncwarp();
    if (lane == 0) {
      umma::fence_after();
      const uint32_t id = idesc_f16mn(128, 16, true, true);
      const uint32_t d = tb + 256 + slot * 16, d1 = tb + 288 + slot * 16;
      const uint32_t ph = umma::smem_u32(Ph), pl = umma::smem_u32(Pl);
      const uint32_t sh = umma::smem_u32(Sh), sl = umma::smem_u32(Sl);
      for (int ks = 0; ks < 2; ++ks) {
        const uint32_t ko = ks * 256;
        const uint32_t acc = (turn == 0 && ks == 0) ? 0u : 1u;
        umma::mma_f16(d, umma::desc(ph + ko, 128, 512), umma::desc(sh + ko, 128, 512), id, acc);
        umma::mma_f16(d, umma::desc(ph + ko, 128, 512), umma::desc(sl + ko, 128, 512), id, 1);
        umma::mma_f16(d, umma::desc(pl + ko, 128, 512), umma::desc(sh + ko, 128, 512), id, 1);
        umma::mma_f16(d1, umma::desc(ph + ko, 128, 512), umma::desc(sh + ko, 128, 512), id, acc);
      }
      umma::commit(&mbar[slot]);
    }
  }
  umma::mbar_wait(&mbar[2], 0);
  umma::mbar_wait(&mbar[0], 1);
  umma::mbar_wait(&mbar[1], 1);
  umma::fence_after();
  const uint32_t lb = (uint32_t)(32 * (w & 3)) << 16;
  const int row = 32 * (w & 3) + lane;
  float v[16];
  for (int c0 = 0; c0 < 2 * NT; c0 += 16) {
    umma::ld16(tb + lb + c0, v);
    umma::ld_wait();
    umma::ld_fence_regs<16>(v);
    for (int i = 0; i < 16; ++i) {
      const int col = c0 + i;
      if (col < NT) out->T[row][col] = v[i] / (SU * SG);
      else out->T1[row][col - NT] = v[i] / (SU * SG);
    }
  }
  float a0[16], a1[16], b0[16], b1[16];
  umma::ld16(tb + lb + 256, a0);
  umma::ld16(tb + lb + 272, a1);
  umma::ld16(tb + lb + 288, b0);
  umma::ld16(tb + lb + 304, b1);
  umma::ld_wait();
  umma::ld_fence_regs<16>(a0);
  umma::ld_fence_regs<16>(a1);
  umma::ld_fence_regs<16>(b0);
  umma::ld_fence_regs<16>(b1);
  for (int i = 0; i < 16; ++i) {
    out->D[row][i] = (a0[i] + a1[i]) / (SP * SS);
    out->D1[row][i] = (b0[i] + b1[i]) / (SP * SS);
  }
  umma::fence_before();
  __syncthreads();
  if (w == 0) umma::tmem_free<512>(tb);
}

int main() {
  srand(7);
  auto rnd = [] { return (float)rand() / RAND_MAX; };
  std::vector<float> U(E * C, 0.f), G(AB * C, 0.f), P(E * 128, 0.f), S(E * 16, 0.f);
  // realistic magnitudes: rows ~U(0, 1/sqrt(J)), core ~U(0,1), residual-scaled S
  for (int e = 0; e < E; ++e)
    for (int c = 0; c < JJ; ++c) U[e * C + c] = rnd() / sqrtf(10.f);
  for (int n = 0; n < AB; ++n)
    for (int c = 0; c < JJ; ++c) G[n * C + c] = rnd();
  for (int e = 0; e < E; ++e) {
    std::vector<float> u1(JJ), u2(JJ);
    for (auto& x : u1) x = rnd() / sqrtf(10.f);
    for (auto& x : u2) x = rnd() / sqrtf(10.f);
    for (int a = 0; a < JJ; ++a)
      for (int b = 0; b < JJ; ++b) P[e * 128 + a * JJ + b] = u1[a] * u2[b];
    const float r = (rnd() - 0.5f) * 2.f;
    for (int c = 0; c < JJ; ++c) S[e * 16 + c] = -r * rnd() / sqrtf(10.f);
  }
  float *dU, *dG, *dP, *dS;
  Res* dR;
  cudaMalloc(&dU, U.size() * 4);
  cudaMalloc(&dG, G.size() * 4);
  cudaMalloc(&dP, P.size() * 4);
  cudaMalloc(&dS, S.size() * 4);
  cudaMalloc(&dR, sizeof(Res));
  cudaMemcpy(dU, U.data(), U.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dG, G.data(), G.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dP, P.data(), P.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dS, S.data(), S.size() * 4, cudaMemcpyHostToDevice);
  const int smem = 8192 + 7168 + 2 * (2 * 8192 + 2 * 1024) + 1024;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  Res* h = new Res;
  int bad = 0;
  for (int variant = 0; variant < 1; ++variant) {
    cudaMemset(dR, 0, sizeof(Res));
    kern<<<1, 128, smem>>>(dU, dG, dP, dS, dR, variant);
    cudaError_t err = cudaDeviceSynchronize();
    if (err != cudaSuccess) {
      printf("variant %d: CUDA error %s\n", variant, cudaGetErrorString(err));
      return 2;
    }
    cudaMemcpy(h, dR, sizeof(Res), cudaMemcpyDeviceToHost);
    double eT = 0, eT1 = 0, sT = 0, eD = 0, eD1 = 0, sD = 0;
    for (int e = 0; e < E; ++e)
      for (int n = 0; n < AB; ++n) {
        double s = 0, sa = 0;
        for (int c = 0; c < JJ; ++c) {
          s += (double)U[e * C + c] * G[n * C + c];
          sa += fabs((double)U[e * C + c] * G[n * C + c]);
        }
        eT = fmax(eT, fabs(s - h->T[e][n]) / sa);
        eT1 = fmax(eT1, fabs(s - h->T1[e][n]) / sa);
        sT = fmax(sT, sa);
      }
    for (int ab = 0; ab < AB; ++ab)
      for (int c = 0; c < JJ; ++c) {
        double s = 0, sa = 0;
        for (int e = 0; e < E; ++e) {
          s += (double)P[e * 128 + ab] * S[e * 16 + c];
          sa += fabs((double)P[e * 128 + ab] * S[e * 16 + c]);
        }
        eD = fmax(eD, fabs(s - h->D[ab][c]) / sa);
        eD1 = fmax(eD1, fabs(s - h->D1[ab][c]) / sa);
        sD = fmax(sD, sa);
      }
    printf("variant %d: sweep split rel err %.3g (hi only %.3g) | core split rel err %.3g (hi only %.3g)\n",
           variant, eT, eT1, eD, eD1);
    printf("  T[0][0..2] %g %g %g  D[0][0..2] %g %g %g\n", h->T[0][0], h->T[0][1], h->T[0][2],
           h->D[0][0], h->D[0][1], h->D[0][2]);
    if (eT > 2e-6 || eD > 2e-6) bad = 1;
  }
  printf(bad ? "split-fp16 UMMA: FAIL\n" : "split-fp16 UMMA: ok\n");
  return bad;
}
