// hog4.cuh -- order-4 S^3CMTF epoch kernel for J = 8 (BASELINE configs[3]:
// 4-way tensor, 8^4 core, two coupled matrices).
//
// Same execution model as hog3v2 (one launch per epoch, a contiguous chunk
// of the randomly permuted COO per lane, interleaved matrix entries, hot-row
// shared-memory replicas with damped merges, relaxed Hogwild on cold rows),
// with the order-4 specifics:
//
// * sweep (Algorithm 3 reuse, src/gradients.cpp:150-206 restated): for every
//   core row (a,b,c) one pair of broadcast LDS.128 of G[a,b,c,0:8] feeds
//   t = G.u4 (8 FMA) and g4 += G * (u1[a]u2[b]u3[c]) (8 FMA); then
//   s_ab += t u3[c], g3[c] += t u1[a]u2[b]; per (a,b): W1[a] += s_ab u2[b],
//   g2[b] += s_ab u1[a].  The a-loop is rolled (u1 and W1 live in the lane's
//   staging row) so the unrolled b,c,d body fits the instruction cache.
// * core gradient dG[a,b,c,d] = sum_e -r_e u1[a]u2[b]u3[c]u4[d] on the
//   tensor cores, block-wide: each lane stages (-r u1, u2, u3, u4), and after
//   a block barrier warp w (NW = J = 8) computes the slab a = w over all 256
//   staged entries: D[d][(b,c)] = sum_e u4_e[d] * Q_e[(b,c)] with
//   Q_e[(b,c)] = (-r u1_e[w]) u2_e[b] u3_e[c], mma.sync m16n8k8 TF32 with
//   the n-tile = b and the 8 columns = c.  The 16 live accumulators per lane
//   stay in registers until the (damped, block-level) core push, which also
//   refreshes the shared core slab a = w from the global core.
#pragma once

#include "hog3v2.cuh"

namespace cmtfb {

struct Hog4Args {
  const uint32_t* rec;  // tensor records (i1, i2, i3, i4, bits(x)), random order
  uint64_t nnz;
  const uint4* mrec;    // matrix records {row, col, bits(y), matrix id}
  uint64_t mnnz;
  int n_mr;
  uint64_t mr_lo[kV2MaxMats];
  uint64_t mr_n[kV2MaxMats];
  int n_mat;
  MatDesc3 mats[kV2MaxMats];
  float* U[4];
  const float* reg[4];
  HotDesc hot[4];
  float* G;
  float eta;
  float core_reg;
  float kappa;
  float kappa_core;
  float nhat_core;
  int flush_every;
  int core_every;
  int nonneg;
  float* probe;       // unused (hog3tm only)
  float* probe_core;
  uint32_t* visits;   // debug_count_visits: +1 per tensor / matrix record visit
  uint32_t* mvisits;
};

// D += A B on the tensor cores at fp32-level accuracy: every operand is
// split x = hi + lo (split_tf32) and the product formed as
// hi*hi + hi*lo + lo*hi (3xTF32, ~21 mantissa bits; the lo*lo term is below
// fp32 rounding) -- the per-entry contractions keep the north_star's 1e-5
// per-entry tolerance instead of TF32's ~1e-3
__device__ __forceinline__ void mma_3xtf32(float* d, const uint32_t* ah, const uint32_t* al,
                                           const uint32_t* b) {
  uint32_t bh[2], bl[2];
  split_tf32(__uint_as_float(b[0]), bh[0], bl[0]);
  split_tf32(__uint_as_float(b[1]), bh[1], bl[1]);
  mma_tf32(d, ah, bl);
  mma_tf32(d, al, bh);
  mma_tf32(d, ah, bh);
}
__device__ __forceinline__ void split4(const uint32_t* a, uint32_t* ah, uint32_t* al) {
#pragma unroll
  for (int k = 0; k < 4; ++k) split_tf32(__uint_as_float(a[k]), ah[k], al[k]);
}

template <int J, int NW, bool TC = false>
struct V4Layout {
  static_assert(J == 8 && NW == 8, "hog4 is specialised for J = 8 (one core slab per warp)");
  static constexpr int JP = J;
  static constexpr int ABC = J * J * J;           // core rows (a,b,c), d fastest
  static constexpr int SW = 40;                   // >= 4*JP, == 8 (mod 32)
  static constexpr int G_FLOATS = ABC * JP;       // 16 KB, [abc][d]
  static constexpr int S1 = 12;                   // TC: [abc][12] copy, conflict-free B rows
  static constexpr int G1_FLOATS = TC ? ABC * S1 : 0;
  static constexpr int STAGE_FLOATS = NW * 32 * SW;  // one of two (double-buffered)
  static constexpr int META_WORDS = TC ? NW * 32 * 16 : 0;
  static constexpr int FIXED_FLOATS = G_FLOATS + G1_FLOATS + 2 * STAGE_FLOATS + META_WORDS;
};

// MODE 0: Algorithm 2 (CUDA cores); 1: Algorithm 3 (CUDA cores); 2: Algorithm 3
// with the two core contractions on the tensor cores (see the TC block).
template <int J, int MODE, int NW>
__global__ void __launch_bounds__(NW * 32, 1)
hog4_kernel(Hog4Args a) {
  constexpr bool OPT = MODE >= 1;
  constexpr bool TC = MODE == 2;
  using L = V4Layout<J, NW, TC>;
  constexpr int JP = L::JP;
  constexpr int ABC = L::ABC;
  constexpr int SW = L::SW;
  extern __shared__ __align__(16) float sm[];
  __shared__ float red_kw[NW], red_lam[NW];
  float* Gs = sm;
  float* G1 = sm + L::G_FLOATS;  // TC only
  float* stg0 = G1 + L::G1_FLOATS;  // [2][NW*32][SW]: iteration t uses buffer t % 2
  uint32_t* meta = reinterpret_cast<uint32_t*>(stg0 + 2 * L::STAGE_FLOATS);  // TC only
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g8 = lane >> 2, t4 = lane & 3;

  for (int q = threadIdx.x; q < ABC * JP; q += blockDim.x) {
    const float v = __ldcg(a.G + q);
    Gs[q] = v;
    if (TC) G1[(q / JP) * L::S1 + q % JP] = v;
  }
#pragma unroll
  for (int n = 0; n < 4; ++n)
    if (a.hot[n].H) load_hot<JP>(a.hot[n], a.U[n], sm + a.hot[n].off, sm + a.hot[n].stat_off);
  for (int m = 0; m < a.n_mat; ++m)
    if (a.mats[m].hotV.H)
      load_hot<JP>(a.mats[m].hotV, a.mats[m].V, sm + a.mats[m].hotV.off,
                   sm + a.mats[m].hotV.stat_off);
  __syncthreads();

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
  float acc[J][2];  // dG[a=w][b][c=2t4 (+1)][d=g8] since the last push
#pragma unroll
  for (int i = 0; i < J; ++i) acc[i][0] = acc[i][1] = 0.f;

  const float* rep[4];
  float* stat[4];
#pragma unroll
  for (int n = 0; n < 4; ++n) {
    rep[n] = sm + a.hot[n].off;
    stat[n] = sm + a.hot[n].stat_off;
  }

  // Software pipeline: while entry t is computed, the cold rows of entry t+1
  // are copied (cp.async, L1 bypass) into the other staging buffer, the
  // record of t+2 and (after the sweep) its hot slots are loaded.
  auto issue_rows = [&](float* row, const uint32_t* ix, const int* slx) {
#pragma unroll
    for (int n = 0; n < 4; ++n)
      if (slx[n] < 0) {
        const float* src = a.U[n] + (uint64_t)ix[n] * JP;
        cp_async16(row + n * JP, src);
        cp_async16(row + n * JP + 4, src + 4);
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
    issue_rows(stg0 + (w * 32 + lane) * SW, ix, sl);
  }
  cp_async_commit();  // (empty) core-refresh group: see the push
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

  for (uint64_t it = 0; it < iters; ++it) {
    const uint64_t e = lo + it;
    const bool active = e < hi;
    if (active && a.visits) atomicAdd(a.visits + e, 1u);
    float* stg = stg0 + (it & 1) * L::STAGE_FLOATS;
    float* myst = stg + (w * 32 + lane) * SW;
    const float x = __uint_as_float(xv);
    if (e + 2 < hi) {
#pragma unroll
      for (int n = 0; n < 4; ++n) n2x[n] = __ldg(a.rec + (e + 2) * 5 + n);
      n2xv = __ldg(a.rec + (e + 2) * 5 + 4);
    }
    // this entry's rows; the newest group (the last core refresh) may fly on
    cp_async_wait_group<1>();
    int n2sl[4] = {-1, -1, -1, -1};
    float n2reg[4] = {0.f, 0.f, 0.f, 0.f};
    if constexpr (!TC) {
      float u2[JP], u3[JP], u4[JP];
      if (active) {
        if (sl[0] >= 0) {
  #pragma unroll
          for (int k = 0; k < JP; k += 4)
            *reinterpret_cast<float4*>(myst + k) =
                *reinterpret_cast<const float4*>(rep[0] + sl[0] * JP + k);
        }
        const float* s2 = sl[1] >= 0 ? rep[1] + sl[1] * JP : myst + JP;
        const float* s3 = sl[2] >= 0 ? rep[2] + sl[2] * JP : myst + 2 * JP;
        const float* s4 = sl[3] >= 0 ? rep[3] + sl[3] * JP : myst + 3 * JP;
  #pragma unroll
        for (int k = 0; k < JP; k += 4) {
          const float4 q2 = *reinterpret_cast<const float4*>(s2 + k);
          const float4 q3 = *reinterpret_cast<const float4*>(s3 + k);
          const float4 q4 = *reinterpret_cast<const float4*>(s4 + k);
          u2[k] = q2.x; u2[k + 1] = q2.y; u2[k + 2] = q2.z; u2[k + 3] = q2.w;
          u3[k] = q3.x; u3[k + 1] = q3.y; u3[k + 2] = q3.z; u3[k + 3] = q3.w;
          u4[k] = q4.x; u4[k + 1] = q4.y; u4[k + 2] = q4.z; u4[k + 3] = q4.w;
        }
      } else {
  #pragma unroll
        for (int k = 0; k < JP; ++k) u2[k] = u3[k] = u4[k] = 0.f;
  #pragma unroll
        for (int k = 0; k < JP; k += 4)
          *reinterpret_cast<float4*>(myst + k) = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      // the other buffer was last read by the previous iteration's block MMA
      // (before its closing barrier): start entry t+1's gathers into it
      if (e + 1 < hi)
        issue_rows(stg0 + ((it + 1) & 1) * L::STAGE_FLOATS + (w * 32 + lane) * SW, nx, nsl);

      float g2[J], g3[J], g4[J];
  #pragma unroll
      for (int k = 0; k < J; ++k) g2[k] = g3[k] = g4[k] = 0.f;
      float xh = 0.f;
      if (OPT) {
  #pragma unroll 1
        for (int ia = 0; ia < J; ++ia) {
          const float ua = myst[ia];
          const float* ga = Gs + ia * J * J * JP;
          float wsum = 0.f;
  #pragma unroll
          for (int ib = 0; ib < J; ++ib) {
            const float pab = ua * u2[ib];
            float sab = 0.f;
  #pragma unroll
            for (int ic = 0; ic < J; ++ic) {
              const float* gr = ga + (ib * J + ic) * JP;
              const float4 q0 = *reinterpret_cast<const float4*>(gr);
              const float4 q1 = *reinterpret_cast<const float4*>(gr + 4);
              const float gv[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
              float t = 0.f;
  #pragma unroll
              for (int d = 0; d < J; ++d) t = fmaf(gv[d], u4[d], t);
              const float pabc = pab * u3[ic];
  #pragma unroll
              for (int d = 0; d < J; ++d) g4[d] = fmaf(gv[d], pabc, g4[d]);
              sab = fmaf(t, u3[ic], sab);
              g3[ic] = fmaf(t, pab, g3[ic]);
            }
            wsum = fmaf(sab, u2[ib], wsum);
            g2[ib] = fmaf(sab, ua, g2[ib]);
          }
          myst[JP + ia] = wsum;
          xh = fmaf(wsum, ua, xh);
        }
      } else {
        // Algorithm 2: one walk for the prediction, then one per mode
  #pragma unroll 1
        for (int ia = 0; ia < J; ++ia) {
          const float ua = myst[ia];
          const float* ga = Gs + ia * J * J * JP;
          float wsum = 0.f;
  #pragma unroll
          for (int ib = 0; ib < J; ++ib)
  #pragma unroll
            for (int ic = 0; ic < J; ++ic) {
              const float* gr = ga + (ib * J + ic) * JP;
              float t = 0.f;
  #pragma unroll
              for (int d = 0; d < J; ++d) t = fmaf(gr[d], u4[d], t);
              wsum = fmaf(t, u2[ib] * u3[ic], wsum);
            }
          xh = fmaf(wsum, ua, xh);
        }
        asm volatile("" ::: "memory");
  #pragma unroll 1
        for (int ia = 0; ia < J; ++ia) {  // mode 1
          const float* ga = Gs + ia * J * J * JP;
          float wsum = 0.f;
  #pragma unroll
          for (int ib = 0; ib < J; ++ib)
  #pragma unroll
            for (int ic = 0; ic < J; ++ic) {
              const float* gr = ga + (ib * J + ic) * JP;
              float t = 0.f;
  #pragma unroll
              for (int d = 0; d < J; ++d) t = fmaf(gr[d], u4[d], t);
              wsum = fmaf(t, u2[ib] * u3[ic], wsum);
            }
          myst[JP + ia] = wsum;
        }
        asm volatile("" ::: "memory");
  #pragma unroll 1
        for (int ia = 0; ia < J; ++ia) {  // mode 2
          const float ua = myst[ia];
          const float* ga = Gs + ia * J * J * JP;
  #pragma unroll
          for (int ib = 0; ib < J; ++ib)
  #pragma unroll
            for (int ic = 0; ic < J; ++ic) {
              const float* gr = ga + (ib * J + ic) * JP;
              float t = 0.f;
  #pragma unroll
              for (int d = 0; d < J; ++d) t = fmaf(gr[d], u4[d], t);
              g2[ib] = fmaf(t, ua * u3[ic], g2[ib]);
            }
        }
        asm volatile("" ::: "memory");
  #pragma unroll 1
        for (int ia = 0; ia < J; ++ia) {  // mode 3
          const float ua = myst[ia];
          const float* ga = Gs + ia * J * J * JP;
  #pragma unroll
          for (int ib = 0; ib < J; ++ib)
  #pragma unroll
            for (int ic = 0; ic < J; ++ic) {
              const float* gr = ga + (ib * J + ic) * JP;
              float t = 0.f;
  #pragma unroll
              for (int d = 0; d < J; ++d) t = fmaf(gr[d], u4[d], t);
              g3[ic] = fmaf(t, ua * u2[ib], g3[ic]);
            }
        }
        asm volatile("" ::: "memory");
  #pragma unroll 1
        for (int ia = 0; ia < J; ++ia) {  // mode 4
          const float ua = myst[ia];
          const float* ga = Gs + ia * J * J * JP;
  #pragma unroll
          for (int ib = 0; ib < J; ++ib)
  #pragma unroll
            for (int ic = 0; ic < J; ++ic) {
              const float* gr = ga + (ib * J + ic) * JP;
              const float p = ua * u2[ib] * u3[ic];
  #pragma unroll
              for (int d = 0; d < J; ++d) g4[d] = fmaf(gr[d], p, g4[d]);
            }
        }
      }

      if (e + 2 < hi) {
  #pragma unroll
        for (int n = 0; n < 4; ++n) {
          n2sl[n] = a.hot[n].slot ? __ldg(a.hot[n].slot + n2x[n]) : -1;
          n2reg[n] = __ldg(a.reg[n] + n2x[n]);
        }
      }

      // ---- residual, row steps, staging (-r u1, u2, u3, u4) ----
      {
        float u1[JP], w1[J];
  #pragma unroll
        for (int k = 0; k < JP; ++k) u1[k] = myst[k];
  #pragma unroll
        for (int k = 0; k < J; ++k) w1[k] = myst[JP + k];
        const float r = active ? x - xh : 0.f;
        float n1 = 0.f, n2 = 0.f, n3 = 0.f, n4 = 0.f;
        float c1 = 0.f, c2 = 0.f, c3 = 0.f, c4 = 0.f;
  #pragma unroll
        for (int k = 0; k < J; ++k) {
          n1 = fmaf(u1[k], u1[k], n1); n2 = fmaf(u2[k], u2[k], n2);
          n3 = fmaf(u3[k], u3[k], n3); n4 = fmaf(u4[k], u4[k], n4);
          c1 = fmaf(w1[k], w1[k], c1); c2 = fmaf(g2[k], g2[k], c2);
          c3 = fmaf(g3[k], g3[k], c3); c4 = fmaf(g4[k], g4[k], c4);
        }
        if (active) {
          lamG += (n1 * n2) * (n3 * n4);
          kw += 1.f;
        }
        // row steps: every lane of the warp takes part (hot-row aggregation)
        float gr[J];
  #pragma unroll
        for (int k = 0; k < J; ++k) gr[k] = fmaf(-r, w1[k], reg[0] * u1[k]);
        step_row_warp<J, JP>(a.U[0], ix[0], sl[0], const_cast<float*>(rep[0]), stat[0],
                             (int)a.hot[0].off, active, u1, gr, a.eta, a.nonneg, c1, lane);
  #pragma unroll
        for (int k = 0; k < J; ++k) gr[k] = fmaf(-r, g2[k], reg[1] * u2[k]);
        step_row_warp<J, JP>(a.U[1], ix[1], sl[1], const_cast<float*>(rep[1]), stat[1],
                             (int)a.hot[1].off, active, u2, gr, a.eta, a.nonneg, c2, lane);
  #pragma unroll
        for (int k = 0; k < J; ++k) gr[k] = fmaf(-r, g3[k], reg[2] * u3[k]);
        step_row_warp<J, JP>(a.U[2], ix[2], sl[2], const_cast<float*>(rep[2]), stat[2],
                             (int)a.hot[2].off, active, u3, gr, a.eta, a.nonneg, c3, lane);
  #pragma unroll
        for (int k = 0; k < J; ++k) gr[k] = fmaf(-r, g4[k], reg[3] * u4[k]);
        step_row_warp<J, JP>(a.U[3], ix[3], sl[3], const_cast<float*>(rep[3]), stat[3],
                             (int)a.hot[3].off, active, u4, gr, a.eta, a.nonneg, c4, lane);
  #pragma unroll
        for (int k = 0; k < JP; k += 4) {
          *reinterpret_cast<float4*>(myst + k) =
              make_float4(-r * u1[k], -r * u1[k + 1], -r * u1[k + 2], -r * u1[k + 3]);
          *reinterpret_cast<float4*>(myst + JP + k) = make_float4(u2[k], u2[k + 1], u2[k + 2], u2[k + 3]);
          *reinterpret_cast<float4*>(myst + 2 * JP + k) =
              make_float4(u3[k], u3[k + 1], u3[k + 2], u3[k + 3]);
          *reinterpret_cast<float4*>(myst + 3 * JP + k) =
              make_float4(u4[k], u4[k + 1], u4[k + 2], u4[k + 3]);
        }
      }
    } else {
      // ================= tensor-core sweep (MODE 2) =================
      // A warp's 32 entries form two m-tiles of 16; lane (g8, t4) serves the
      // entries R0 = g8, R1 = g8 + 8 of a tile together with its quad.
      //  GEMM1  T[e][(a,b,c)] = sum_d u4_e[d] G[a,b,c,d]   (M=e, K=d, N=c per (a,b))
      //  GEMM2  g4[e][d] = sum_{abc} (u1[a]u2[b]u3[c])_e G[a,b,c,d]  (K=c per (a,b))
      // From T (lane holds c = 2t4, 2t4+1): s_ab = T.u3 (quad partial),
      // W1[a] = sum_b s_ab u2[b], g2[b] = sum_a s_ab u1[a] (quad-reduced),
      // g3[c] = sum_ab u1[a]u2[b] T[abc] (complete per lane), x = W1.u1.
      // Row steps are split over the quad: each lane owns two components of
      // every row (mode 2: 4(t4&1) + 2(t4>>1) + {0,1}; others 2t4 + {0,1}).
      // (1) this entry's rows into its staging row (hot rows from replicas)
      if (active) {
#pragma unroll
        for (int n = 0; n < 4; ++n)
          if (sl[n] >= 0) {
            *reinterpret_cast<float4*>(myst + n * JP) =
                *reinterpret_cast<const float4*>(rep[n] + sl[n] * JP);
            *reinterpret_cast<float4*>(myst + n * JP + 4) =
                *reinterpret_cast<const float4*>(rep[n] + sl[n] * JP + 4);
          }
      } else {
#pragma unroll
        for (int k = 0; k < 4 * JP; k += 4)
          *reinterpret_cast<float4*>(myst + k) = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      {
        uint32_t* mm = meta + (w * 32 + lane) * 16;
        *reinterpret_cast<uint4*>(mm) = make_uint4(ix[0], ix[1], ix[2], ix[3]);
        *reinterpret_cast<uint4*>(mm + 4) =
            make_uint4((uint32_t)(active ? sl[0] : -1), (uint32_t)(active ? sl[1] : -1),
                       (uint32_t)(active ? sl[2] : -1), (uint32_t)(active ? sl[3] : -1));
        *reinterpret_cast<uint4*>(mm + 8) =
            make_uint4(__float_as_uint(reg[0]), __float_as_uint(reg[1]), __float_as_uint(reg[2]),
                       __float_as_uint(reg[3]));
        *reinterpret_cast<uint2*>(mm + 12) = make_uint2(xv, active ? 1u : 0u);
      }
      if (e + 1 < hi)
        issue_rows(stg0 + ((it + 1) & 1) * L::STAGE_FLOATS + (w * 32 + lane) * SW, nx, nsl);
      if (e + 2 < hi) {
#pragma unroll
        for (int n = 0; n < 4; ++n) {
          n2sl[n] = a.hot[n].slot ? __ldg(a.hot[n].slot + n2x[n]) : -1;
          n2reg[n] = __ldg(a.reg[n] + n2x[n]);
        }
      }
      __syncwarp();
      const int own2 = 4 * (t4 & 1) + 2 * (t4 >> 1);  // mode-2 components of this lane
#pragma unroll 1
      for (int mt = 0; mt < 2; ++mt) {
        const int R0 = w * 32 + mt * 16 + g8, R1 = R0 + 8;
        float* s0 = stg + R0 * SW;
        float* s1 = stg + R1 * SW;
        uint32_t av1[4];
        av1[0] = __float_as_uint(s0[3 * JP + t4]);
        av1[1] = __float_as_uint(s1[3 * JP + t4]);
        av1[2] = __float_as_uint(s0[3 * JP + t4 + 4]);
        av1[3] = __float_as_uint(s1[3 * JP + t4 + 4]);
        uint32_t av1h[4], av1l[4];
        split4(av1, av1h, av1l);
        const float2 c0 = *reinterpret_cast<const float2*>(s0 + 2 * JP + 2 * t4);
        const float2 c1 = *reinterpret_cast<const float2*>(s1 + 2 * JP + 2 * t4);
        const float u3c[4] = {c0.x, c0.y, c1.x, c1.y};
        const float u3k[4] = {s0[2 * JP + t4], s1[2 * JP + t4], s0[2 * JP + t4 + 4],
                              s1[2 * JP + t4 + 4]};
        float u2r0[J], u2r1[J];
#pragma unroll
        for (int k = 0; k < J; k += 4) {
          const float4 p0 = *reinterpret_cast<const float4*>(s0 + JP + k);
          const float4 p1 = *reinterpret_cast<const float4*>(s1 + JP + k);
          u2r0[k] = p0.x; u2r0[k + 1] = p0.y; u2r0[k + 2] = p0.z; u2r0[k + 3] = p0.w;
          u2r1[k] = p1.x; u2r1[k + 1] = p1.y; u2r1[k + 2] = p1.z; u2r1[k + 3] = p1.w;
        }
        // four independent g4 accumulators (ib & 3): the MMA chain stays short
        float d4x[4][4] = {}, g3v[4] = {0.f, 0.f, 0.f, 0.f};
        float g2p0[J], g2p1[J];
#pragma unroll
        for (int k = 0; k < J; ++k) g2p0[k] = g2p1[k] = 0.f;
        float W1o[4] = {0.f, 0.f, 0.f, 0.f};
        float xh0 = 0.f, xh1 = 0.f;
#pragma unroll 1
        for (int ia = 0; ia < J; ++ia) {
          const float ua0 = s0[ia], ua1 = s1[ia];
          const float* g1a = G1 + ia * J * J * L::S1;
          const float* g2a = Gs + ia * J * J * JP;
          float w1p0 = 0.f, w1p1 = 0.f;
#pragma unroll
          for (int ib = 0; ib < J; ++ib) {
            uint32_t bb[2];
            bb[0] = __float_as_uint(g1a[(ib * J + g8) * L::S1 + t4]);
            bb[1] = __float_as_uint(g1a[(ib * J + g8) * L::S1 + t4 + 4]);
            float d[4] = {0.f, 0.f, 0.f, 0.f};
            mma_3xtf32(d, av1h, av1l, bb);  // T[R0][2t4], T[R0][2t4+1], T[R1][2t4], T[R1][2t4+1]
            const float pab0 = ua0 * u2r0[ib], pab1 = ua1 * u2r1[ib];
            const float sp0 = fmaf(d[1], u3c[1], d[0] * u3c[0]);
            const float sp1 = fmaf(d[3], u3c[3], d[2] * u3c[2]);
            w1p0 = fmaf(sp0, u2r0[ib], w1p0);
            w1p1 = fmaf(sp1, u2r1[ib], w1p1);
            g2p0[ib] = fmaf(sp0, ua0, g2p0[ib]);
            g2p1[ib] = fmaf(sp1, ua1, g2p1[ib]);
            g3v[0] = fmaf(d[0], pab0, g3v[0]);
            g3v[1] = fmaf(d[1], pab0, g3v[1]);
            g3v[2] = fmaf(d[2], pab1, g3v[2]);
            g3v[3] = fmaf(d[3], pab1, g3v[3]);
            uint32_t ap[4], b2[2];
            ap[0] = __float_as_uint(pab0 * u3k[0]);
            ap[1] = __float_as_uint(pab1 * u3k[1]);
            ap[2] = __float_as_uint(pab0 * u3k[2]);
            ap[3] = __float_as_uint(pab1 * u3k[3]);
            b2[0] = __float_as_uint(g2a[(ib * J + t4) * JP + g8]);
            b2[1] = __float_as_uint(g2a[(ib * J + t4 + 4) * JP + g8]);
            uint32_t aph[4], apl[4];
            split4(ap, aph, apl);
            mma_3xtf32(d4x[ib & 3], aph, apl, b2);  // g4[R0][2t4], [R0][2t4+1], [R1][2t4], [R1][2t4+1]
          }
          w1p0 += __shfl_xor_sync(0xffffffffu, w1p0, 1);
          w1p1 += __shfl_xor_sync(0xffffffffu, w1p1, 1);
          w1p0 += __shfl_xor_sync(0xffffffffu, w1p0, 2);
          w1p1 += __shfl_xor_sync(0xffffffffu, w1p1, 2);
          xh0 = fmaf(w1p0, ua0, xh0);
          xh1 = fmaf(w1p1, ua1, xh1);
          if ((ia >> 1) == t4) {
            if (ia & 1) { W1o[1] = w1p0; W1o[3] = w1p1; }
            else { W1o[0] = w1p0; W1o[2] = w1p1; }
          }
        }
        float d4[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) d4[k] = (d4x[0][k] + d4x[1][k]) + (d4x[2][k] + d4x[3][k]);
        // g2: reduce-scatter over the quad -> components own2, own2 + 1
        float g2o[4];
        {
          const bool b0 = t4 & 1, b1 = t4 >> 1;
          float k0[4], k1[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float s0v = b0 ? g2p0[i] : g2p0[i + 4], s1v = b0 ? g2p1[i] : g2p1[i + 4];
            k0[i] = (b0 ? g2p0[i + 4] : g2p0[i]) + __shfl_xor_sync(0xffffffffu, s0v, 1);
            k1[i] = (b0 ? g2p1[i + 4] : g2p1[i]) + __shfl_xor_sync(0xffffffffu, s1v, 1);
          }
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const float s0v = b1 ? k0[i] : k0[i + 2], s1v = b1 ? k1[i] : k1[i + 2];
            g2o[i] = (b1 ? k0[i + 2] : k0[i]) + __shfl_xor_sync(0xffffffffu, s0v, 2);
            g2o[2 + i] = (b1 ? k1[i + 2] : k1[i]) + __shfl_xor_sync(0xffffffffu, s1v, 2);
          }
        }
        // residuals and the owned components of every row step
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          float* sq = q ? s1 : s0;
          const uint32_t* mq = meta + (q ? R1 : R0) * 16;
          const bool act = mq[13] != 0u;
          const float r = act ? __uint_as_float(mq[12]) - (q ? xh1 : xh0) : 0.f;
          const float2 v1 = *reinterpret_cast<const float2*>(sq + 2 * t4);
          const float2 v2 = *reinterpret_cast<const float2*>(sq + JP + own2);
          const float2 v4 = *reinterpret_cast<const float2*>(sq + 3 * JP + 2 * t4);
          const float uu[4][2] = {{v1.x, v1.y}, {v2.x, v2.y}, {u3c[2 * q], u3c[2 * q + 1]},
                                  {v4.x, v4.y}};
          const float gg[4][2] = {{W1o[2 * q], W1o[2 * q + 1]}, {g2o[2 * q], g2o[2 * q + 1]},
                                  {g3v[2 * q], g3v[2 * q + 1]}, {d4[2 * q], d4[2 * q + 1]}};
          const int comp[4] = {2 * t4, own2, 2 * t4, 2 * t4};
          // full-row norms (quad sums of the owned parts): |u_n|^2 and |c_n|^2
          float nrm[8];
#pragma unroll
          for (int n = 0; n < 4; ++n) {
            nrm[n] = fmaf(uu[n][0], uu[n][0], uu[n][1] * uu[n][1]);
            nrm[4 + n] = fmaf(gg[n][0], gg[n][0], gg[n][1] * gg[n][1]);
          }
#pragma unroll
          for (int n = 0; n < 8; ++n) {
            nrm[n] += __shfl_xor_sync(0xffffffffu, nrm[n], 1);
            nrm[n] += __shfl_xor_sync(0xffffffffu, nrm[n], 2);
          }
          if (act && t4 == 0) {
            lamG += (nrm[0] * nrm[1]) * (nrm[2] * nrm[3]);
            kw += 1.f;
          }
          if (act) {
#pragma unroll
            for (int n = 0; n < 4; ++n) {
              const float rg = __uint_as_float(mq[8 + n]);
              float nv0 = uu[n][0] - a.eta * fmaf(-r, gg[n][0], rg * uu[n][0]);
              float nv1 = uu[n][1] - a.eta * fmaf(-r, gg[n][1], rg * uu[n][1]);
              const int slot = (int)mq[4 + n];
              if (slot >= 0) {
                float2* rp = reinterpret_cast<float2*>(const_cast<float*>(rep[n]) + slot * JP + comp[n]);
                float2 cur = *rp;
                cur.x += nv0 - uu[n][0];
                cur.y += nv1 - uu[n][1];
                if (a.nonneg) { cur.x = fmaxf(cur.x, 0.f); cur.y = fmaxf(cur.y, 0.f); }
                *rp = cur;
                if (t4 == 0) {
                  stat[n][3 * slot] += nrm[4 + n];
                  atomicAdd(reinterpret_cast<int*>(stat[n]) + 3 * slot + 1, 1);
                }
              } else if (!a.nonneg && CMTF_COLD_RED) {
                float* gp = a.U[n] + (uint64_t)mq[n] * JP + comp[n];
                asm volatile("red.relaxed.gpu.global.add.v2.f32 [%0], {%1,%2};" ::"l"(gp),
                             "f"(nv0 - uu[n][0]), "f"(nv1 - uu[n][1])
                             : "memory");
              } else {
                if (a.nonneg) { nv0 = fmaxf(nv0, 0.f); nv1 = fmaxf(nv1, 0.f); }
                *reinterpret_cast<float2*>(a.U[n] + (uint64_t)mq[n] * JP + comp[n]) =
                    make_float2(nv0, nv1);
              }
            }
          }
          // stage -r u1 (pre-update) for the block's core gradient
          *reinterpret_cast<float2*>(sq + 2 * t4) = make_float2(-r * v1.x, -r * v1.y);
        }
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
    __syncthreads();  // (A) all NW*32 entries staged

    // ---- core gradient slab a = w on the tensor cores (K = the block's entries) ----
#pragma unroll 2
    for (int ks = 0; ks < NW * 4; ++ks) {
      const float* s0 = stg + (ks * 8 + t4) * SW;
      const float* s1 = s0 + 4 * SW;
      const float p0 = s0[w] * s0[2 * JP + g8];  // -r u1[a=w] u3[c=g8]
      const float p1 = s1[w] * s1[2 * JP + g8];
      uint32_t av[4];
      av[0] = __float_as_uint(s0[3 * JP + g8]);  // A[d=g8][e0] = u4_e0[g8]
      av[1] = 0u;
      av[2] = __float_as_uint(s1[3 * JP + g8]);
      av[3] = 0u;
      uint32_t avh[4], avl[4];
      split4(av, avh, avl);
      const float4 b00 = *reinterpret_cast<const float4*>(s0 + JP);
      const float4 b01 = *reinterpret_cast<const float4*>(s0 + JP + 4);
      const float4 b10 = *reinterpret_cast<const float4*>(s1 + JP);
      const float4 b11 = *reinterpret_cast<const float4*>(s1 + JP + 4);
      const float v0[8] = {b00.x, b00.y, b00.z, b00.w, b01.x, b01.y, b01.z, b01.w};
      const float v1[8] = {b10.x, b10.y, b10.z, b10.w, b11.x, b11.y, b11.z, b11.w};
#pragma unroll
      for (int ib = 0; ib < J; ++ib) {
        uint32_t bv[2];
        bv[0] = __float_as_uint(p0 * v0[ib]);  // B[e0][c=g8] = Q_e0[(ib, g8)]
        bv[1] = __float_as_uint(p1 * v1[ib]);
        float d[4] = {acc[ib][0], acc[ib][1], 0.f, 0.f};
        mma_3xtf32(d, avh, avl, bv);
        acc[ib][0] = d[0];  // D[d=g8][c=2t4], D[g8][2t4+1]
        acc[ib][1] = d[1];
      }
    }

    // ---- interleaved matrix entries ----
    matrix_entries_until<J, JP>(a, sm, mpos, mrn, mlo + msched.step(), mhi, lane);

    // ---- damped block-level core push of slab a = w, refresh from global ----
    if (push) {
      float kb = 0.f, lb = 0.f;
#pragma unroll
      for (int q = 0; q < NW; ++q) {
        kb += red_kw[q];
        lb += red_lam[q];
      }
      if (kb > 0.f) {
        const float q = a.eta * (lb / kb) * a.nhat_core;
        const float alpha = q > a.kappa_core ? a.kappa_core / q : 1.f;
        const float s = -a.eta * alpha;
        const float kr = kb * a.core_reg;
#pragma unroll
        for (int ib = 0; ib < J; ++ib)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int o = ((w * J + ib) * J + 2 * t4 + h) * JP + g8;
            const float delta = s * fmaf(kr, Gs[o], acc[ib][h]);
            if (a.nonneg) {
              const float v = atomic_add_clamp0(a.G + o, delta);
              Gs[o] = v;
              if (TC) G1[((w * J + ib) * J + 2 * t4 + h) * L::S1 + g8] = v;
            } else {
              // fire-and-forget RED, then refresh the shared copies from the
              // global core asynchronously (the read follows our RED to the
              // same address; other warps see the old or the new value)
              red_add_f32(a.G + o, delta);
              cp_async4(Gs + o, a.G + o);
              if (TC) cp_async4(G1 + ((w * J + ib) * J + 2 * t4 + h) * L::S1 + g8, a.G + o);
            }
            acc[ib][h] = 0.f;
          }
      }
    }
    cp_async_commit();  // core refresh group (possibly empty)
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
    __syncthreads();  // (B) core slabs refreshed, staging consumed
  }
  matrix_entries_until<J, JP>(a, sm, mpos, mrn, mhi, mhi, lane);
  cp_async_wait_all();
  __syncthreads();
  flush_all_hot<J, JP, NW, 4>(a, sm, w, lane);
}

// Eval pass for order 4, J = 8: thread per entry, fixed kEvalBlock-entry
// blocks (src/eval.cpp:10-65), double accumulation, deterministic order.
__global__ void __launch_bounds__(256)
eval4_kernel(const uint32_t* rec, uint64_t nnz, const float* U1, const float* U2,
             const float* U3, const float* U4, const float* G, double* partial) {
  constexpr int J = 8, BT = 256;
  extern __shared__ __align__(16) float sm[];
  float* Gs = sm;  // [abc][d]
  __shared__ double acc_s[BT / 32];
  const int t = threadIdx.x;
  for (int q = t; q < J * J * J * J; q += BT) Gs[q] = G[q];
  __syncthreads();
  const uint64_t lo = (uint64_t)blockIdx.x * kEvalBlock;
  const uint64_t hi = lo + kEvalBlock < nnz ? lo + kEvalBlock : nnz;
  double acc = 0.0;
  for (uint64_t e = lo + t; e < hi; e += BT) {
    const uint32_t* rp = rec + e * 5;
    float u1[J], u2[J], u3[J], u4[J];
    load_row<J>(U1, __ldg(rp), -1, nullptr, u1);
    load_row<J>(U2, __ldg(rp + 1), -1, nullptr, u2);
    load_row<J>(U3, __ldg(rp + 2), -1, nullptr, u3);
    load_row<J>(U4, __ldg(rp + 3), -1, nullptr, u4);
    float xh = 0.f;
#pragma unroll 1
    for (int ia = 0; ia < J; ++ia) {
      float ua = 0.f;  // select u1[ia] without local-memory indexing
#pragma unroll
      for (int k = 0; k < J; ++k) ua = k == ia ? u1[k] : ua;
      const float* ga = Gs + ia * J * J * J;
      float w = 0.f;
#pragma unroll
      for (int ib = 0; ib < J; ++ib) {
        float sab = 0.f;
#pragma unroll
        for (int ic = 0; ic < J; ++ic) {
          const float4 q0 = *reinterpret_cast<const float4*>(ga + (ib * J + ic) * J);
          const float4 q1 = *reinterpret_cast<const float4*>(ga + (ib * J + ic) * J + 4);
          float t0 = q0.x * u4[0], t1 = q0.y * u4[1];
          t0 = fmaf(q0.z, u4[2], t0); t1 = fmaf(q0.w, u4[3], t1);
          t0 = fmaf(q1.x, u4[4], t0); t1 = fmaf(q1.y, u4[5], t1);
          t0 = fmaf(q1.z, u4[6], t0); t1 = fmaf(q1.w, u4[7], t1);
          sab = fmaf(t0 + t1, u3[ic], sab);
        }
        w = fmaf(sab, u2[ib], w);
      }
      xh = fmaf(w, ua, xh);
    }
    const double r = (double)__uint_as_float(__ldg(rp + 4)) - (double)xh;
    acc += r * r;
  }
  acc = warp_sum_d(acc);
  if ((t & 31) == 0) acc_s[t >> 5] = acc;
  __syncthreads();
  if (t == 0) {
    double s2 = 0.0;
    for (int i = 0; i < BT / 32; ++i) s2 += acc_s[i];
    partial[blockIdx.x] = s2;
  }
}

}  // namespace cmtfb
