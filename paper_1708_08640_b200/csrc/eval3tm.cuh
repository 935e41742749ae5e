// eval3tm.cuh -- order-3 evaluation pass (predict_entry + squared residuals,
// src/tucker.cpp:96-127, src/eval.cpp:14-65) with the core contraction on
// tcgen05: per tile of 128 entries (thread e = entry e = TMEM lane e)
//
//   T[e][(a,b)] = sum_c u3_e[c] G[a,b,c]      MMA  A = U3 tile (K-major), B = G ((a,b) x c)
//   x_hat_e     = sum_a u1[a] sum_b T[ab] u2[b]     FP32, J^2 + J FMAs per entry
//
// instead of eval3_kernel's J^3 + J^2 + J CUDA-core FMAs.  Operands are the
// same split-fp16 pairs as hog3tm's sweep (hi*hi + hi*lo + lo*hi, fp32
// accumulate: ~5e-7 relative per product), so the sums hold the 1e-5 bound of
// the stats tests.  Residuals are squared and summed in double; a block of
// 128 threads owns one 1024-entry eval block at a time (8 tiles) and writes
// its partial sum -- the same partial layout as eval3_kernel, combined
// pairwise on the host (the reference's blocked_sum, src/eval.cpp:14-40).
// Four blocks per SM (128 TMEM columns each) hide the row-gather latency;
// records run two tiles ahead and rows one tile ahead in registers.
#pragma once

#include <cuda_fp16.h>

#include "common.cuh"
#include "hog3tm.cuh"
#include "umma.cuh"

namespace cmtfb {

template <int J>
struct EvalTMLayout {
  using L = TMLayout<J>;
  static constexpr int NT = L::NT;
  static constexpr int TM_COLS = NT <= 32 ? 32 : NT <= 64 ? 64 : 128;
  static_assert(NT <= 128, "eval3tm: J^2 <= 128");
};

#ifndef CMTF_EVAL_TM_OCC
#define CMTF_EVAL_TM_OCC 3  // blocks per SM the register budget is set for
#endif

template <int J>
__global__ void __launch_bounds__(128, CMTF_EVAL_TM_OCC)
eval3tm_kernel(const uint4* __restrict__ rec, uint64_t nnz, const float* __restrict__ U1,
               const float* __restrict__ U2, const float* __restrict__ U3,
               const float* __restrict__ G, double* __restrict__ partial, uint64_t nblk) {
  using L = TMLayout<J>;
  constexpr int JP = L::JP, AB = L::AB, NT = L::NT;
  constexpr int TMC = EvalTMLayout<J>::TM_COLS;
  __shared__ __align__(1024) uint8_t Gh[L::G_TILE];
  __shared__ __align__(16) uint8_t Gl[L::G_TILE];
  __shared__ __align__(1024) uint8_t tUh[L::U_TILE];
  __shared__ __align__(16) uint8_t tUl[L::U_TILE];
  __shared__ uint64_t mbar;
  __shared__ uint32_t tmem_base;
  __shared__ double acc_s[4];
  const int e = threadIdx.x, w = e >> 5, lane = e & 31;

  // ---- prologue: core copy (fp16 hi/lo, (a,b) rows x c), zeroed tiles ----
  for (int q = e; q < L::G_TILE / 4; q += 128) {
    reinterpret_cast<uint32_t*>(Gh)[q] = 0u;
    reinterpret_cast<uint32_t*>(Gl)[q] = 0u;
  }
  for (int q = e; q < L::U_TILE / 4; q += 128) {
    reinterpret_cast<uint32_t*>(tUh)[q] = 0u;
    reinterpret_cast<uint32_t*>(tUl)[q] = 0u;
  }
  __syncthreads();
  for (int q = e; q < AB * J; q += 128) {
    const int ab = q / J, c = q - ab * J;
    __half h, l;
    split_h(__ldg(G + q) * kSG, h, l);
    const int o = (ab >> 3) * 128 + (ab & 7) * 16 + (c >> 3) * L::G_LBO + (c & 7) * 2;
    *reinterpret_cast<__half*>(Gh + o) = h;
    *reinterpret_cast<__half*>(Gl + o) = l;
  }
  if (e == 0) {
    umma::mbar_init(&mbar, 1);
    umma::fence_mbar_init();
  }
  if (w == 0) umma::tmem_alloc<TMC>(&tmem_base);
  umma::fence_async_smem();
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tm = tmem_base;
  const uint32_t tm_lane = (uint32_t)(32 * w) << 16;
  const uint32_t sUh = umma::smem_u32(tUh), sUl = umma::smem_u32(tUl);
  const uint32_t sGh = umma::smem_u32(Gh), sGl = umma::smem_u32(Gl);
  constexpr uint32_t ID = umma::idesc_f16(128, NT);
  constexpr float kInvT = 1.f / (kSU * kSG);
  uint8_t* myUh = tUh + e * 16;
  uint8_t* myUl = tUl + e * 16;

  auto load_row = [&](const float* U, uint32_t i, float* r) {
#pragma unroll
    for (int k = 0; k < JP; k += 4) {
      const float4 q = __ldg(reinterpret_cast<const float4*>(U + (uint64_t)i * JP + k));
      r[k] = q.x; r[k + 1] = q.y; r[k + 2] = q.z; r[k + 3] = q.w;
    }
  };

  // the block's tiles form one sequence over its eval blocks: tile s of the
  // block is tile (s & 7) of eval block blockIdx.x + (s >> 3) * gridDim.x
  const uint64_t nmine = blockIdx.x < nblk ? (nblk - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const uint64_t ntile = nmine * 8;
  auto entry_of = [&](uint64_t s) -> uint64_t {
    const uint64_t blk = blockIdx.x + (s >> 3) * (uint64_t)gridDim.x;
    return blk * kEvalBlock + (s & 7) * 128 + e;
  };
  auto block_hi = [&](uint64_t s) -> uint64_t {
    const uint64_t blk = blockIdx.x + (s >> 3) * (uint64_t)gridDim.x;
    const uint64_t h = (blk + 1) * kEvalBlock;
    return h < nnz ? h : nnz;
  };
  const uint4 zero4 = make_uint4(0u, 0u, 0u, 0u);
  uint4 rc = ntile > 0 && entry_of(0) < block_hi(0) ? __ldg(rec + entry_of(0)) : zero4;
  uint4 rc1 = ntile > 1 && entry_of(1) < block_hi(1) ? __ldg(rec + entry_of(1)) : zero4;
  float u1[JP], u2[JP], u3[JP];
  load_row(U1, rc.x, u1);
  load_row(U2, rc.y, u2);
  load_row(U3, rc.z, u3);

  uint32_t par = 0;
  double acc = 0.0;
  for (uint64_t s = 0; s < ntile; ++s) {
    const bool act = entry_of(s) < block_hi(s);
    const uint4 rc2 = s + 2 < ntile && entry_of(s + 2) < block_hi(s + 2) ? __ldg(rec + entry_of(s + 2))
                                                                          : zero4;
    // this entry's u3 as fp16 hi/lo rows of the A tile (K = 16, zero padded)
    {
      float v[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) v[k] = k < J ? u3[k] * kSU : 0.f;
      uint4 h0, l0, h1, l1;
      split8(v, h0, l0);
      split8(v + 8, h1, l1);
      *reinterpret_cast<uint4*>(myUh) = h0;
      *reinterpret_cast<uint4*>(myUh + L::U_LBO) = h1;
      *reinterpret_cast<uint4*>(myUl) = l0;
      *reinterpret_cast<uint4*>(myUl + L::U_LBO) = l1;
    }
    umma::fence_async_smem();
    umma::fence_before();  // orders the previous tile's TMEM reads before the barrier
    __syncthreads();
    if (e == 0) {
      umma::fence_after();
      const uint64_t dUh = umma::desc(sUh, L::U_LBO, 128), dUl = umma::desc(sUl, L::U_LBO, 128);
      const uint64_t dGh = umma::desc(sGh, L::G_LBO, 128), dGl = umma::desc(sGl, L::G_LBO, 128);
      umma::mma_f16(tm, dUh, dGh, ID, 0u);
      umma::mma_f16(tm, dUh, dGl, ID, 1u);
      umma::mma_f16(tm, dUl, dGh, ID, 1u);
      umma::commit(&mbar);
    }
    // next tile's rows while the MMAs run (this tile's u3 is in the A tile)
    float n1[JP], n2[JP];
    load_row(U3, rc1.z, u3);
    load_row(U1, rc1.x, n1);
    load_row(U2, rc1.y, n2);
    float w1[J];
#pragma unroll
    for (int k = 0; k < J; ++k) w1[k] = 0.f;
    umma::mbar_wait(&mbar, par);
    par ^= 1u;
    umma::fence_after();
#pragma unroll
    for (int c0 = 0; c0 < NT; c0 += 16) {
      float v[16];
      umma::ld16(tm + tm_lane + c0, v);
      umma::ld_wait();
      umma::ld_fence_regs<16>(v);
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int col = c0 + q;
        if (col < AB) {
          const int ia = col / J, ib = col % J;
          w1[ia] = fmaf(v[q], u2[ib], w1[ia]);
        }
      }
    }
    float xh = 0.f;
#pragma unroll
    for (int k = 0; k < J; ++k) xh = fmaf(w1[k], u1[k], xh);
    xh *= kInvT;  // undoes the operand scales (powers of two)
    if (act) {
      const double r = (double)__uint_as_float(rc.w) - (double)xh;
      acc += r * r;
    }
    if ((s & 7) == 7) {  // the eval block is complete: its partial sum
      const double ws = warp_sum_d(acc);
      if (lane == 0) acc_s[w] = ws;
      __syncthreads();
      if (e == 0)
        partial[blockIdx.x + (s >> 3) * (uint64_t)gridDim.x] =
            (acc_s[0] + acc_s[1]) + (acc_s[2] + acc_s[3]);
      acc = 0.0;
      // acc_s is rewritten only after the next tile's barrier
    }
    rc = rc1;
    rc1 = rc2;
#pragma unroll
    for (int k = 0; k < JP; ++k) {
      u1[k] = n1[k];
      u2[k] = n2[k];
    }
  }
  umma::fence_before();
  __syncthreads();
  if (w == 0) umma::tmem_free<TMC>(tmem_base);
}

}  // namespace cmtfb
