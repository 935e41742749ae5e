// hog4tm.cuh -- order-4 S^3CMTF epoch kernel (J = 8, BASELINE configs[3]) with
// the per-entry core contractions and the core gradient on the 5th-generation
// tensor cores (tcgen05.mma, accumulators in tensor memory), at fp32-level
// accuracy.  Same epoch contract as hog4 (one launch = one epoch over the
// tensor and the coupled matrices, hot-row replicas with damped merges,
// interleaved matrix entries, damped block-level core push).
//
// Algorithm 3's quantities (src/gradients.cpp:130-223) for an order-4 entry
// with rows u1..u4, written over the two Kronecker vectors
//   p[(a,b)] = u1[a] u2[b],   q[(c,d)] = u3[c] u4[d]      (64 values each)
// and the core as the 64 x 64 matrix G[(a,b)][(c,d)]:
//   M1[e][(a,b)] = sum_cd q_e[cd] G[ab][cd]     MMA  A = Q tile,  B = G  (K = cd)
//   M2[e][(c,d)] = sum_ab p_e[ab] G[ab][cd]     MMA  A = P tile,  B = G  (K = ab)
//   g1[a] = sum_b u2[b] M1[ab],  g2[b] = sum_a u1[a] M1[ab],  x_hat = g1 . u1,
//   g3[c] = sum_d u4[d] M2[cd],  g4[d] = sum_c u3[c] M2[cd]     FP32, ~5 J^2 FMAs
//   dG[(a,b)][(c,d)] += sum_e (-r_e p_e[ab]) q_e[cd]   MMA  A = P' tile, B = Q tile
// so an entry costs ~5 J^2 FP32 FMAs and ~6 J^2 packed-fp16 operations instead
// of hog4's 2 J^4 FMAs.
//
// A block is 2 warpgroups; each sweeps a tile of 128 entries per iteration,
// thread e owning entry e (TMEM lane e).  Operand tiles (umma.cuh's
// no-swizzle canonical layout): a tile is 8 planes of [128 entries][8 fp16];
// plane j of the Q tile holds q[(c = j, d = 0..7)].  The SAME bytes are a
// K-major A operand of the sweep (rows = entries, K = cd) and an MN-major B
// operand of the core gradient (N = cd, K = entries) -- only the descriptor
// strides change.  Likewise one fp16 copy of G serves M1 (K-major B: rows ab,
// K = cd) and M2 (MN-major B: N = cd, K = ab).
//
// Accuracy: every operand is x = hi + lo in fp16 (after a power-of-two scale)
// and every product hi*hi + hi*lo + lo*hi in three kind::f16 MMAs with fp32
// accumulation (~22 mantissa bits), as hog3tm.  p and q are formed directly as
// fp16 hi/lo pairs by packed fp16 arithmetic (see split_outer8).
#pragma once

#include <cuda_fp16.h>

#include "common.cuh"
#include "hog3tm.cuh"
#include "hog4.cuh"
#include "umma.cuh"

namespace cmtfb {

struct TM4Layout {
  static constexpr int J = 8, JP = 8;
  static constexpr int PLANE = 128 * 16;        // [128 entries][8 fp16]
  static constexpr int TILE = 8 * PLANE;        // 16 KB: one hi or lo tile
  static constexpr int G_PLANE = 64 * 16;       // [64 (a,b)][8 fp16] of one c
  static constexpr int G_TILE = 8 * G_PLANE;    // 8 KB: G hi or lo
  static constexpr int G_BYTES = 2 * G_TILE;
  static constexpr int WG_BYTES = 4 * TILE;     // Q hi, Q lo, P hi, P lo
  static constexpr int STAGE_WG = 128 * 4 * JP * 4;  // gathered rows, 128 B per entry
  // G | WG0 tiles | WG1 tiles | WG0 staging | WG1 staging.  The M = 128 core
  // gradient MMA reads 16 (a,b) planes of P': those past the tile's 8 lie in
  // the buffer that follows (valid shared memory) and only feed the ignored
  // accumulator rows (a,b) >= 64.
  static constexpr int FIXED_BYTES = G_BYTES + 2 * WG_BYTES + 2 * STAGE_WG;
  static constexpr int FIXED_FLOATS = FIXED_BYTES / 4;
  // tensor memory per warpgroup: M1 [0, 64), M2 [64, 128), dG [128, 192)
  static constexpr int TM_COLS = 256;
};

// operand scales (powers of two): p = (64 u1)(8 u2), q = (64 u3)(8 u4); an
// |u1 u2| or |u3 u4| beyond 127, or |r u1 u2| beyond 1023, overflows fp16 and
// surfaces as a non-finite parameter (DivergenceError), like a diverged model
constexpr float kS4a = 64.f, kS4b = 8.f, kS4g = 64.f, kS4r = 64.f;

// One plane of an outer-product tile: out[k] = x * y[k], k = 0..7, as fp16
// hi / lo pairs without forming the fp32 products: x = (xh, xl) and the y
// pairs (yh, yl) are fp16 splits (11 significant bits each); hi = rn16(xh yh),
// its rounding residual xh yh - hi has at most 11 significant bits so one
// packed FMA returns it exactly, lo = residual + xl yh + xh yl.
__device__ __forceinline__ void split_outer8(__half2 xh, __half2 xl, const __half2* yh,
                                             const __half2* yl, uint4& hi, uint4& lo) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const __half2 ph = __hmul2(xh, yh[q]);
    __half2 rl = __hfma2(xh, yh[q], __hneg2(ph));
    rl = __hfma2(xl, yh[q], rl);
    rl = __hfma2(xh, yl[q], rl);
    h[q] = *reinterpret_cast<const uint32_t*>(&ph);
    l[q] = *reinterpret_cast<const uint32_t*>(&rl);
  }
  hi = make_uint4(h[0], h[1], h[2], h[3]);
  lo = make_uint4(l[0], l[1], l[2], l[3]);
}

__global__ void __launch_bounds__(256, 1) hog4tm_kernel(Hog4Args a) {
  using L = TM4Layout;
  constexpr int J = 8, JP = 8, NW = 8;
  extern __shared__ __align__(1024) float sm[];
  uint8_t* smb = reinterpret_cast<uint8_t*>(sm);
  uint8_t* Gh = smb;
  uint8_t* Gl = Gh + L::G_TILE;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = threadIdx.x >> 7;   // warpgroup
  const int e = threadIdx.x & 127;  // tile row = TMEM lane
  const int wk = w & 3;
  uint8_t* Qh = smb + L::G_BYTES + g * L::WG_BYTES;
  uint8_t* Ql = Qh + L::TILE;
  uint8_t* Ph = Ql + L::TILE;
  uint8_t* Pl = Ph + L::TILE;
  float* myst = reinterpret_cast<float*>(smb + L::G_BYTES + 2 * L::WG_BYTES + g * L::STAGE_WG) +
                e * 4 * JP;
  __shared__ uint64_t mbar[2][2];  // [warpgroup][sweep MMAs, core-gradient MMAs]
  __shared__ uint32_t tmem_base;
  __shared__ float red_kw[NW], red_lam[NW];

  // core element G[(a,b)][(c,d)] into the fp16 copies: plane c, row (a,b)
  auto put_g = [&](int ab, int cd, float v) {
    __half h, l;
    split_h(v * kS4g, h, l);
    const int o = (cd >> 3) * L::G_PLANE + ab * 16 + (cd & 7) * 2;
    *reinterpret_cast<__half*>(Gh + o) = h;
    *reinterpret_cast<__half*>(Gl + o) = l;
  };

  for (int q = threadIdx.x; q < L::FIXED_FLOATS; q += blockDim.x) sm[q] = 0.f;
  __syncthreads();
  for (int q = threadIdx.x; q < 4096; q += blockDim.x) put_g(q >> 6, q & 63, __ldcg(a.G + q));
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < 4; ++k) umma::mbar_init(&mbar[k >> 1][k & 1], 1);
    umma::fence_mbar_init();
  }
  if (w == 0) umma::tmem_alloc<512>(&tmem_base);
#pragma unroll
  for (int n = 0; n < 4; ++n)
    if (a.hot[n].H) load_hot<JP>(a.hot[n], a.U[n], sm + a.hot[n].off, sm + a.hot[n].stat_off);
  for (int m = 0; m < a.n_mat; ++m)
    if (a.mats[m].hotV.H)
      load_hot<JP>(a.mats[m].hotV, a.mats[m].V, sm + a.mats[m].hotV.off,
                   sm + a.mats[m].hotV.stat_off);
  umma::fence_async_smem();
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tm = tmem_base + (uint32_t)(g * L::TM_COLS);
  const uint32_t tm_lane = (uint32_t)(32 * wk) << 16;
  const uint32_t sQh = umma::smem_u32(Qh), sQl = umma::smem_u32(Ql);
  const uint32_t sPh = umma::smem_u32(Ph), sPl = umma::smem_u32(Pl);
  const uint32_t sGh = umma::smem_u32(Gh), sGl = umma::smem_u32(Gl);
  constexpr uint32_t ID_M1 = umma::idesc_f16(128, 64, false, false);  // A K-major, B K-major
  constexpr uint32_t ID_M2 = umma::idesc_f16(128, 64, false, true);   // B = G MN-major
  constexpr uint32_t ID_DG = umma::idesc_f16(128, 64, true, true);    // P', Q MN-major
  constexpr float kInvM = 1.f / (kS4a * kS4b * kS4g);
  constexpr float kInvD = 1.f / (kS4r * kS4a * kS4b);

  const uint64_t Wt = (uint64_t)gridDim.x * NW * 32;
  const uint64_t gl = ((uint64_t)blockIdx.x * NW + w) * 32 + lane;
  const uint64_t lo = a.nnz * gl / Wt, hi = a.nnz * (gl + 1) / Wt;
  const uint64_t iters = (a.nnz + Wt - 1) / Wt;
  const uint64_t mlo = a.mnnz * gl / Wt, mhi = a.mnnz * (gl + 1) / Wt;
  uint64_t mpos = mlo;
  uint4 mrn = mlo < mhi ? __ldg(a.mrec + mphys(a, mlo)) : make_uint4(0, 0, 0, 0);
  MatSched msched;
  msched.init(mlo, mhi, iters);
  float kw = 0.f, lamG = 0.f;

  float* rep[4];
  float* stat[4];
#pragma unroll
  for (int n = 0; n < 4; ++n) {
    rep[n] = sm + a.hot[n].off;
    stat[n] = sm + a.hot[n].stat_off;
  }

  // records two ahead, hot slots and regulariser coefficients one ahead; the
  // next entry's cold rows are copied (cp.async) into this thread's staging
  // rows as soon as this entry's rows are in registers
  auto issue_rows = [&](const uint32_t* ix, const int* slx, bool act) {
    if (act) {
#pragma unroll
      for (int n = 0; n < 4; ++n)
        if (slx[n] < 0) {
          const float* src = a.U[n] + (uint64_t)ix[n] * JP;
          cp_async16(myst + n * JP, src);
          cp_async16(myst + n * JP + 4, src + 4);
        }
    }
    cp_async_commit();
  };
  uint32_t ix[4] = {0, 0, 0, 0}, nx[4] = {0, 0, 0, 0}, n2x[4] = {0, 0, 0, 0};
  uint32_t xv = 0, nxv = 0, n2xv = 0;
  int sl[4] = {-1, -1, -1, -1}, nsl[4] = {-1, -1, -1, -1};
  float reg[4] = {0.f, 0.f, 0.f, 0.f}, nreg[4] = {0.f, 0.f, 0.f, 0.f};
  if (lo < hi) {
#pragma unroll
    for (int n = 0; n < 4; ++n) ix[n] = __ldg(a.rec + lo * 5 + n);
    xv = __ldg(a.rec + lo * 5 + 4);
#pragma unroll
    for (int n = 0; n < 4; ++n) {
      sl[n] = a.hot[n].slot ? __ldg(a.hot[n].slot + ix[n]) : -1;
      reg[n] = __ldg(a.reg[n] + ix[n]);
    }
  }
  issue_rows(ix, sl, lo < hi);
  if (lo + 1 < hi) {
#pragma unroll
    for (int n = 0; n < 4; ++n) nx[n] = __ldg(a.rec + (lo + 1) * 5 + n);
    nxv = __ldg(a.rec + (lo + 1) * 5 + 4);
#pragma unroll
    for (int n = 0; n < 4; ++n) {
      nsl[n] = a.hot[n].slot ? __ldg(a.hot[n].slot + nx[n]) : -1;
      nreg[n] = __ldg(a.reg[n] + nx[n]);
    }
  }
  bool dg_fresh = true;  // the next core-gradient MMA overwrites the accumulator

  for (uint64_t it = 0; it < iters; ++it) {
    const uint64_t ee = lo + it;
    const bool active = ee < hi;
    const uint32_t par = (uint32_t)(it & 1);
    if (active && a.visits) atomicAdd(a.visits + ee, 1u);
    const float x = __uint_as_float(xv);
    if (ee + 2 < hi) {
#pragma unroll
      for (int n = 0; n < 4; ++n) n2x[n] = __ldg(a.rec + (ee + 2) * 5 + n);
      n2xv = __ldg(a.rec + (ee + 2) * 5 + 4);
    }

    // ---- this entry's rows (cold ones landed in the staging rows) ----
    cp_async_wait_group<0>();
    float u[4][JP];
    if (active) {
#pragma unroll
      for (int n = 0; n < 4; ++n) {
        const float* s = sl[n] >= 0 ? rep[n] + sl[n] * JP : myst + n * JP;
        const float4 q0 = *reinterpret_cast<const float4*>(s);
        const float4 q1 = *reinterpret_cast<const float4*>(s + 4);
        u[n][0] = q0.x; u[n][1] = q0.y; u[n][2] = q0.z; u[n][3] = q0.w;
        u[n][4] = q1.x; u[n][5] = q1.y; u[n][6] = q1.z; u[n][7] = q1.w;
      }
    } else {
#pragma unroll
      for (int n = 0; n < 4; ++n)
#pragma unroll
        for (int k = 0; k < JP; ++k) u[n][k] = 0.f;
    }
    // the next entry's gathers have the whole iteration to land
    issue_rows(nx, nsl, ee + 1 < hi);
    int n2sl[4] = {-1, -1, -1, -1};
    float n2reg[4] = {0.f, 0.f, 0.f, 0.f};
    if (ee + 2 < hi) {
#pragma unroll
      for (int n = 0; n < 4; ++n) {
        n2sl[n] = a.hot[n].slot ? __ldg(a.hot[n].slot + n2x[n]) : -1;
        n2reg[n] = __ldg(a.reg[n] + n2x[n]);
      }
    }

    // ---- P and Q rows of this entry as fp16 hi/lo (the previous iteration's
    // core-gradient MMAs, the tiles' last readers, must be done) ----
    if (it > 0) umma::mbar_wait(&mbar[g][1], par ^ 1u);
    {
      __half2 yh[4], yl[4];
      auto split_pairs = [&](const float* v, float scale) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float x0 = v[2 * k] * scale, x1 = v[2 * k + 1] * scale;
          const float h0 = __uint_as_float(__float_as_uint(x0) & 0xffffe000u);
          const float h1 = __uint_as_float(__float_as_uint(x1) & 0xffffe000u);
          yh[k] = __floats2half2_rn(h0, h1);
          yl[k] = __floats2half2_rn(x0 - h0, x1 - h1);
        }
      };
      split_pairs(u[1], kS4b);  // p: plane a, pairs over b
#pragma unroll
      for (int ia = 0; ia < J; ++ia) {
        __half h, l;
        split_h(u[0][ia] * kS4a, h, l);
        uint4 ph, pl;
        split_outer8(__half2half2(h), __half2half2(l), yh, yl, ph, pl);
        *reinterpret_cast<uint4*>(Ph + ia * L::PLANE + e * 16) = ph;
        *reinterpret_cast<uint4*>(Pl + ia * L::PLANE + e * 16) = pl;
      }
      split_pairs(u[3], kS4b);  // q: plane c, pairs over d
#pragma unroll
      for (int ic = 0; ic < J; ++ic) {
        __half h, l;
        split_h(u[2][ic] * kS4a, h, l);
        uint4 qh, ql;
        split_outer8(__half2half2(h), __half2half2(l), yh, yl, qh, ql);
        *reinterpret_cast<uint4*>(Qh + ic * L::PLANE + e * 16) = qh;
        *reinterpret_cast<uint4*>(Ql + ic * L::PLANE + e * 16) = ql;
      }
    }
    umma::fence_async_smem();
    umma::fence_before();
    umma::bar_sync(1 + g, 128);
    if (e == 0) {
      umma::fence_after();
      // K = 64 in four steps of 16 = two 8-wide planes each.  A (K-major):
      // LBO = plane stride (K direction), SBO = 128 (8-row groups).  B = G
      // K-major for M1 (LBO = G plane stride, SBO = 128); MN-major for M2
      // (K = (a,b): 8-row groups 128 B apart = LBO, N planes = SBO).
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const uint64_t dAh = umma::desc(sQh + ks * 2 * L::PLANE, L::PLANE, 128);
        const uint64_t dAl = umma::desc(sQl + ks * 2 * L::PLANE, L::PLANE, 128);
        const uint64_t dBh = umma::desc(sGh + ks * 2 * L::G_PLANE, L::G_PLANE, 128);
        const uint64_t dBl = umma::desc(sGl + ks * 2 * L::G_PLANE, L::G_PLANE, 128);
        umma::mma_f16(tm, dAh, dBh, ID_M1, ks > 0 ? 1u : 0u);
        umma::mma_f16(tm, dAh, dBl, ID_M1, 1u);
        umma::mma_f16(tm, dAl, dBh, ID_M1, 1u);
      }
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const uint64_t dAh = umma::desc(sPh + ks * 2 * L::PLANE, L::PLANE, 128);
        const uint64_t dAl = umma::desc(sPl + ks * 2 * L::PLANE, L::PLANE, 128);
        const uint64_t dBh = umma::desc(sGh + ks * 2 * 128, 128, L::G_PLANE);
        const uint64_t dBl = umma::desc(sGl + ks * 2 * 128, 128, L::G_PLANE);
        umma::mma_f16(tm + 64, dAh, dBh, ID_M2, ks > 0 ? 1u : 0u);
        umma::mma_f16(tm + 64, dAh, dBl, ID_M2, 1u);
        umma::mma_f16(tm + 64, dAl, dBh, ID_M2, 1u);
      }
      umma::commit(&mbar[g][0]);
    }

    // ---- contractions out of tensor memory (FP32) ----
    float g1[J], g2[J], g3[J], g4[J];
#pragma unroll
    for (int k = 0; k < J; ++k) g1[k] = g2[k] = g3[k] = g4[k] = 0.f;
    umma::mbar_wait(&mbar[g][0], par);
    umma::fence_after();
#pragma unroll
    for (int c0 = 0; c0 < 64; c0 += 32) {
      float v[32];
      umma::ld16(tm + tm_lane + c0, v);
      umma::ld16(tm + tm_lane + c0 + 16, v + 16);
      umma::ld_wait();
      umma::ld_fence_regs<32>(v);
#pragma unroll
      for (int q = 0; q < 32; ++q) {
        const int ia = (c0 + q) >> 3, ib = (c0 + q) & 7;
        g1[ia] = fmaf(v[q], u[1][ib], g1[ia]);
        g2[ib] = fmaf(v[q], u[0][ia], g2[ib]);
      }
    }
#pragma unroll
    for (int c0 = 0; c0 < 64; c0 += 32) {
      float v[32];
      umma::ld16(tm + tm_lane + 64 + c0, v);
      umma::ld16(tm + tm_lane + 64 + c0 + 16, v + 16);
      umma::ld_wait();
      umma::ld_fence_regs<32>(v);
#pragma unroll
      for (int q = 0; q < 32; ++q) {
        const int ic = (c0 + q) >> 3, id = (c0 + q) & 7;
        g3[ic] = fmaf(v[q], u[3][id], g3[ic]);
        g4[id] = fmaf(v[q], u[2][ic], g4[id]);
      }
    }
    float xh = 0.f;
#pragma unroll
    for (int k = 0; k < J; ++k) {
      g1[k] *= kInvM; g2[k] *= kInvM; g3[k] *= kInvM; g4[k] *= kInvM;
      xh = fmaf(g1[k], u[0][k], xh);
    }

    // ---- residual, row steps ----
    const float r = active ? x - xh : 0.f;
    {
      float nrm[4] = {0.f, 0.f, 0.f, 0.f}, cur[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int k = 0; k < J; ++k) {
        nrm[0] = fmaf(u[0][k], u[0][k], nrm[0]); nrm[1] = fmaf(u[1][k], u[1][k], nrm[1]);
        nrm[2] = fmaf(u[2][k], u[2][k], nrm[2]); nrm[3] = fmaf(u[3][k], u[3][k], nrm[3]);
        cur[0] = fmaf(g1[k], g1[k], cur[0]); cur[1] = fmaf(g2[k], g2[k], cur[1]);
        cur[2] = fmaf(g3[k], g3[k], cur[2]); cur[3] = fmaf(g4[k], g4[k], cur[3]);
      }
      if (active) {
        lamG += (nrm[0] * nrm[1]) * (nrm[2] * nrm[3]);
        kw += 1.f;
      }
      const float* gn[4] = {g1, g2, g3, g4};
#pragma unroll
      for (int n = 0; n < 4; ++n) {
        float gr[J];
#pragma unroll
        for (int k = 0; k < J; ++k) gr[k] = fmaf(-r, gn[n][k], reg[n] * u[n][k]);
        if (active)
          step_row<J, JP>(a.U[n], ix[n], sl[n], rep[n], stat[n], u[n], gr, a.eta, a.nonneg, cur[n]);
      }
    }

    // ---- P' = -r p over the P tile (its sweep MMAs are done), then the
    // warpgroup's core-gradient MMAs: K = its 128 entries ----
    {
      const float rs = -r * kS4r;
#pragma unroll
      for (int ia = 0; ia < J; ++ia) {
        float v[8];
        const float s = rs * u[0][ia];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = s * u[1][k];
        uint4 ph, pl;
        split8(v, ph, pl);
        *reinterpret_cast<uint4*>(Ph + ia * L::PLANE + e * 16) = ph;
        *reinterpret_cast<uint4*>(Pl + ia * L::PLANE + e * 16) = pl;
      }
    }
    const bool push = (it + 1) % (uint64_t)a.core_every == 0 || it + 1 == iters;
    if (push) {
      const float kws = warp_sum(kw);
      const float lgs = warp_sum(lamG);
      if (lane == 0) {
        red_kw[w] = kws;
        red_lam[w] = lgs;
      }
      kw = 0.f;
      lamG = 0.f;
    }
    umma::fence_async_smem();
    umma::fence_before();
    umma::bar_sync(1 + g, 128);
    if (e == 0) {
      umma::fence_after();
      // MN-major operands: K = entries in 16 steps of 8 (LBO = 128), M / N
      // planes 2048 B apart (SBO); an instruction takes K = 16 = 256 B
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        const uint64_t dAh = umma::desc(sPh + ks * 256, 128, L::PLANE);
        const uint64_t dAl = umma::desc(sPl + ks * 256, 128, L::PLANE);
        const uint64_t dBh = umma::desc(sQh + ks * 256, 128, L::PLANE);
        const uint64_t dBl = umma::desc(sQl + ks * 256, 128, L::PLANE);
        umma::mma_f16(tm + 128, dAh, dBh, ID_DG, (ks > 0 || !dg_fresh) ? 1u : 0u);
        umma::mma_f16(tm + 128, dAh, dBl, ID_DG, 1u);
        umma::mma_f16(tm + 128, dAl, dBh, ID_DG, 1u);
      }
      umma::commit(&mbar[g][1]);
    }
    dg_fresh = false;

    // ---- matrix entries due by this iteration (interleaved) ----
    matrix_entries_until<J, JP>(a, sm, mpos, mrn, mlo + msched.step(), mhi, lane);

    // ---- damped block-level core push, refresh of the fp16 core copies ----
    if (push) {
      umma::mbar_wait(&mbar[g][1], par);  // this iteration's core-gradient MMAs
      umma::fence_after();
      __syncthreads();  // red_kw / red_lam of both warpgroups; all sweep MMAs done
      float kb = 0.f, lb = 0.f;
#pragma unroll
      for (int q = 0; q < NW; ++q) {
        kb += red_kw[q];
        lb += red_lam[q];
      }
      if (kb > 0.f && e < 64) {
        const float qd = a.eta * (lb / kb) * a.nhat_core;
        const float alpha = qd > a.kappa_core ? a.kappa_core / qd : 1.f;
        const float s = -a.eta * alpha;
        const float kr = g == 0 ? kb * a.core_reg : 0.f;  // the regulariser once per block
        float* Grow = a.G + e * 64;
        // the regulariser reads the block's own copy of the core (hi + lo of
        // the fp16 operand copies: 22 bits) -- a global read here would queue
        // behind every block's REDs to the same 128 lines
        auto g_of = [&](int cd) {
          const int o = (cd >> 3) * L::G_PLANE + e * 16 + (cd & 7) * 2;
          return (__half2float(*reinterpret_cast<const __half*>(Gh + o)) +
                  __half2float(*reinterpret_cast<const __half*>(Gl + o))) * (1.f / kS4g);
        };
#pragma unroll
        for (int c0 = 0; c0 < 64; c0 += 16) {
          float v[16];
          umma::ld16(tm + tm_lane + 128 + c0, v);
          umma::ld_wait();
          umma::ld_fence_regs<16>(v);
#pragma unroll
          for (int q = 0; q < 16; q += 4) {
            float4 d;
            d.x = s * fmaf(kr, g_of(c0 + q + 0), v[q + 0] * kInvD);
            d.y = s * fmaf(kr, g_of(c0 + q + 1), v[q + 1] * kInvD);
            d.z = s * fmaf(kr, g_of(c0 + q + 2), v[q + 2] * kInvD);
            d.w = s * fmaf(kr, g_of(c0 + q + 3), v[q + 3] * kInvD);
            if (a.probe_core) {
              atomicAdd(a.probe_core + e * 64 + c0 + q + 0, v[q + 0] * kInvD);
              atomicAdd(a.probe_core + e * 64 + c0 + q + 1, v[q + 1] * kInvD);
              atomicAdd(a.probe_core + e * 64 + c0 + q + 2, v[q + 2] * kInvD);
              atomicAdd(a.probe_core + e * 64 + c0 + q + 3, v[q + 3] * kInvD);
            }
            if (a.nonneg) {
              atomic_add_clamp0(Grow + c0 + q + 0, d.x);
              atomic_add_clamp0(Grow + c0 + q + 1, d.y);
              atomic_add_clamp0(Grow + c0 + q + 2, d.z);
              atomic_add_clamp0(Grow + c0 + q + 3, d.w);
            } else {
              red_add_v4(Grow + c0 + q, d);
            }
          }
        }
      }
      dg_fresh = true;
      umma::fence_before();
      __syncthreads();  // both warpgroups' steps issued
      // refresh: every thread re-reads 16 core elements (after the block's
      // REDs; other blocks' pushes arrive as they come) into the fp16 copies
#pragma unroll
      for (int q = 0; q < 16; q += 4) {
        const int o = threadIdx.x * 16 + q;
        const float4 gv = ld_strong4(a.G + o);
        put_g(o >> 6, (o & 63) + 0, gv.x);
        put_g(o >> 6, (o & 63) + 1, gv.y);
        put_g(o >> 6, (o & 63) + 2, gv.z);
        put_g(o >> 6, (o & 63) + 3, gv.w);
      }
      umma::fence_async_smem();
      __syncthreads();
    }
    if ((it + 1) % (uint64_t)a.flush_every == 0 || it + 1 == iters)
      flush_all_hot<J, JP, NW, 4>(a, sm, w, lane);
#pragma unroll
    for (int n = 0; n < 4; ++n) {
      ix[n] = nx[n];
      nx[n] = n2x[n];
      sl[n] = nsl[n];
      nsl[n] = n2sl[n];
      reg[n] = nreg[n];
      nreg[n] = n2reg[n];
    }
    xv = nxv;
    nxv = n2xv;
  }
  matrix_entries_until<J, JP>(a, sm, mpos, mrn, mhi, mhi, lane);
  cp_async_wait_all();
  umma::fence_before();
  __syncthreads();
  flush_all_hot<J, JP, NW, 4>(a, sm, w, lane);
  if (w == 0) umma::tmem_free<512>(tmem_base);
}

}  // namespace cmtfb
