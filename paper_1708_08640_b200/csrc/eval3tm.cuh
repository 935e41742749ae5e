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
#include "hog4tm.cuh"
#include "umma.cuh"

namespace cmtfb {

template <int J>
struct EvalTMLayout {
  using L = TMLayout<J>;
  static constexpr int NT = L::NT;
  static constexpr int TM_COLS = NT <= 32 ? 32 : NT <= 64 ? 64 : 128;
  static_assert(NT <= 128, "eval3tm: J^2 <= 128");
};

#ifndef CMTF_EVAL_TM_POLICY
#define CMTF_EVAL_TM_POLICY 1  // streamed rows: explicit L2 evict-first policy (0: ld.global.cs)
#endif
#ifndef CMTF_EVAL_TM_OCC
#define CMTF_EVAL_TM_OCC 3  // blocks per SM the register budget is set for
#endif

template <int J>
__global__ void __launch_bounds__(128, CMTF_EVAL_TM_OCC)
eval3tm_kernel(const uint4* __restrict__ rec, uint64_t nnz, const float* __restrict__ U1,
               const float* __restrict__ U2, const float* __restrict__ U3,
               const float* __restrict__ G, double* __restrict__ partial, uint64_t nblk,
               int stream3) {
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

  // stream: evict-first loads.  Under the L2-blocked record layout (modes 1
  // and 2 in row blocks) the mode-3 rows are the random ones: read
  // evict-first, their lines do not push the active row blocks out of L2
  uint64_t pol_first;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_first));
  auto load_row = [&](const float* U, uint32_t i, float* r, bool stream = false) {
#pragma unroll
    for (int k = 0; k < JP; k += 4) {
      const float4* p = reinterpret_cast<const float4*>(U + (uint64_t)i * JP + k);
      float4 q;
      if (stream) {
#if CMTF_EVAL_TM_POLICY
        asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
                     : "=f"(q.x), "=f"(q.y), "=f"(q.z), "=f"(q.w)
                     : "l"(p), "l"(pol_first));
#else
        q = __ldcs(p);
#endif
      } else {
        q = __ldg(p);
      }
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
  uint4 rc = ntile > 0 && entry_of(0) < block_hi(0) ? __ldcs(rec + entry_of(0)) : zero4;
  uint4 rc1 = ntile > 1 && entry_of(1) < block_hi(1) ? __ldcs(rec + entry_of(1)) : zero4;
  float u1[JP], u2[JP], u3[JP];
  load_row(U1, rc.x, u1);
  load_row(U2, rc.y, u2);
  load_row(U3, rc.z, u3, stream3 != 0);

  uint32_t par = 0;
  double acc = 0.0;
  for (uint64_t s = 0; s < ntile; ++s) {
    const bool act = entry_of(s) < block_hi(s);
    const uint4 rc2 = s + 2 < ntile && entry_of(s + 2) < block_hi(s + 2) ? __ldcs(rec + entry_of(s + 2))
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
    load_row(U3, rc1.z, u3, stream3 != 0);
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

// Order 4, J = 8 (BASELINE configs[3]): hog4tm's first sweep contraction per
// tile of 128 entries,
//   M1[e][(a,b)] = sum_cd q_e[cd] G[ab][cd],  q[(c,d)] = u3[c] u4[d]
// (A = Q tile, 8 planes of [128 entries][8 fp16], K-major; B = G, K-major;
// K = 64 in four steps, split-fp16 x3), then x_hat = sum_ab M1[ab] u1[a] u2[b]
// in FP32: J^2 + J FMAs and J^2 packed-fp16 operand products per entry instead
// of eval4_kernel's J^4 + ... CUDA-core FMAs.  Same block / partial scheme as
// eval3tm_kernel; dynamic shared memory: G hi, G lo, Q hi, Q lo.
constexpr int kEval4tmSmem = 2 * TM4Layout::G_TILE + 2 * TM4Layout::TILE;

__global__ void __launch_bounds__(128, CMTF_EVAL_TM_OCC)
eval4tm_kernel(const uint32_t* __restrict__ rec, uint64_t nnz, const float* __restrict__ U1,
               const float* __restrict__ U2, const float* __restrict__ U3,
               const float* __restrict__ U4, const float* __restrict__ G,
               double* __restrict__ partial, uint64_t nblk) {
  using L = TM4Layout;
  constexpr int J = 8;
  extern __shared__ __align__(1024) uint8_t smb4[];
  uint8_t* Gh = smb4;
  uint8_t* Gl = Gh + L::G_TILE;
  uint8_t* Qh = Gl + L::G_TILE;
  uint8_t* Ql = Qh + L::TILE;
  __shared__ uint64_t mbar;
  __shared__ uint32_t tmem_base;
  __shared__ double acc_s[4];
  const int e = threadIdx.x, w = e >> 5, lane = e & 31;

  for (int q = e; q < 4096; q += 128) {  // G[(a,b)][(c,d)]: plane c, row (a,b)
    const int ab = q >> 6, cd = q & 63;
    __half h, l;
    split_h(__ldg(G + q) * kS4g, h, l);
    const int o = (cd >> 3) * L::G_PLANE + ab * 16 + (cd & 7) * 2;
    *reinterpret_cast<__half*>(Gh + o) = h;
    *reinterpret_cast<__half*>(Gl + o) = l;
  }
  if (e == 0) {
    umma::mbar_init(&mbar, 1);
    umma::fence_mbar_init();
  }
  if (w == 0) umma::tmem_alloc<64>(&tmem_base);
  umma::fence_async_smem();
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tm = tmem_base;
  const uint32_t tm_lane = (uint32_t)(32 * w) << 16;
  const uint32_t sQh = umma::smem_u32(Qh), sQl = umma::smem_u32(Ql);
  const uint32_t sGh = umma::smem_u32(Gh), sGl = umma::smem_u32(Gl);
  constexpr uint32_t ID = umma::idesc_f16(128, 64, false, false);
  constexpr float kInv = 1.f / (kS4a * kS4b * kS4g);

  auto load_row = [&](const float* U, uint32_t i, float* r) {
    const float4 q0 = __ldg(reinterpret_cast<const float4*>(U + (uint64_t)i * 8));
    const float4 q1 = __ldg(reinterpret_cast<const float4*>(U + (uint64_t)i * 8 + 4));
    r[0] = q0.x; r[1] = q0.y; r[2] = q0.z; r[3] = q0.w;
    r[4] = q1.x; r[5] = q1.y; r[6] = q1.z; r[7] = q1.w;
  };
  struct Rec5 { uint32_t i[4]; float x; };
  auto load_rec = [&](uint64_t p) -> Rec5 {  // records are 5 words: i1..i4, bits(x)
    Rec5 r;
    const uint32_t* q = rec + 5 * p;
    r.i[0] = __ldg(q); r.i[1] = __ldg(q + 1); r.i[2] = __ldg(q + 2); r.i[3] = __ldg(q + 3);
    r.x = __uint_as_float(__ldg(q + 4));
    return r;
  };
  const uint64_t nmine = blockIdx.x < nblk ? (nblk - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const uint64_t ntile = nmine * 8;
  auto entry_of = [&](uint64_t s) -> uint64_t {
    const uint64_t blk = blockIdx.x + (s >> 3) * (uint64_t)gridDim.x;
    return blk * kEvalBlock + (s & 7) * 128 + e;
  };
  const Rec5 zero{{0u, 0u, 0u, 0u}, 0.f};
  Rec5 rc = ntile > 0 && entry_of(0) < nnz ? load_rec(entry_of(0)) : zero;
  Rec5 rc1 = ntile > 1 && entry_of(1) < nnz ? load_rec(entry_of(1)) : zero;
  float u1[8], u2[8], u3[8], u4[8];
  load_row(U1, rc.i[0], u1);
  load_row(U2, rc.i[1], u2);
  load_row(U3, rc.i[2], u3);
  load_row(U4, rc.i[3], u4);

  uint32_t par = 0;
  double acc = 0.0;
  for (uint64_t s = 0; s < ntile; ++s) {
    const bool act = entry_of(s) < nnz;
    const Rec5 rc2 = s + 2 < ntile && entry_of(s + 2) < nnz ? load_rec(entry_of(s + 2)) : zero;
    {  // this entry's Q planes (fp16 hi / lo) by packed fp16 arithmetic
      __half2 yh[4], yl[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float x0 = u4[2 * k] * kS4b, x1 = u4[2 * k + 1] * kS4b;
        const float h0 = __uint_as_float(__float_as_uint(x0) & 0xffffe000u);
        const float h1 = __uint_as_float(__float_as_uint(x1) & 0xffffe000u);
        yh[k] = __floats2half2_rn(h0, h1);
        yl[k] = __floats2half2_rn(x0 - h0, x1 - h1);
      }
#pragma unroll
      for (int ic = 0; ic < J; ++ic) {
        __half h, l;
        split_h(u3[ic] * kS4a, h, l);
        uint4 qh, ql;
        split_outer8(__half2half2(h), __half2half2(l), yh, yl, qh, ql);
        *reinterpret_cast<uint4*>(Qh + ic * L::PLANE + e * 16) = qh;
        *reinterpret_cast<uint4*>(Ql + ic * L::PLANE + e * 16) = ql;
      }
    }
    umma::fence_async_smem();
    umma::fence_before();
    __syncthreads();
    if (e == 0) {
      umma::fence_after();
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const uint64_t dAh = umma::desc(sQh + ks * 2 * L::PLANE, L::PLANE, 128);
        const uint64_t dAl = umma::desc(sQl + ks * 2 * L::PLANE, L::PLANE, 128);
        const uint64_t dBh = umma::desc(sGh + ks * 2 * L::G_PLANE, L::G_PLANE, 128);
        const uint64_t dBl = umma::desc(sGl + ks * 2 * L::G_PLANE, L::G_PLANE, 128);
        umma::mma_f16(tm, dAh, dBh, ID, ks > 0 ? 1u : 0u);
        umma::mma_f16(tm, dAh, dBl, ID, 1u);
        umma::mma_f16(tm, dAl, dBh, ID, 1u);
      }
      umma::commit(&mbar);
    }
    // next tile's rows while the MMAs run (this tile's u3, u4 are in the Q tile)
    float n1[8], n2[8];
    load_row(U3, rc1.i[2], u3);
    load_row(U4, rc1.i[3], u4);
    load_row(U1, rc1.i[0], n1);
    load_row(U2, rc1.i[1], n2);
    float w1[J];
#pragma unroll
    for (int k = 0; k < J; ++k) w1[k] = 0.f;
    umma::mbar_wait(&mbar, par);
    par ^= 1u;
    umma::fence_after();
#pragma unroll
    for (int c0 = 0; c0 < 64; c0 += 16) {
      float v[16];
      umma::ld16(tm + tm_lane + c0, v);
      umma::ld_wait();
      umma::ld_fence_regs<16>(v);
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int ia = (c0 + q) >> 3, ib = (c0 + q) & 7;
        w1[ia] = fmaf(v[q], u2[ib], w1[ia]);
      }
    }
    float xh = 0.f;
#pragma unroll
    for (int k = 0; k < J; ++k) xh = fmaf(w1[k], u1[k], xh);
    xh *= kInv;
    if (act) {
      const double r = (double)rc.x - (double)xh;
      acc += r * r;
    }
    if ((s & 7) == 7) {
      const double ws = warp_sum_d(acc);
      if (lane == 0) acc_s[w] = ws;
      __syncthreads();
      if (e == 0)
        partial[blockIdx.x + (s >> 3) * (uint64_t)gridDim.x] =
            (acc_s[0] + acc_s[1]) + (acc_s[2] + acc_s[3]);
      acc = 0.0;
    }
    rc = rc1;
    rc1 = rc2;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      u1[k] = n1[k];
      u2[k] = n2[k];
    }
  }
  umma::fence_before();
  __syncthreads();
  if (w == 0) umma::tmem_free<64>(tmem_base);
}

}  // namespace cmtfb
