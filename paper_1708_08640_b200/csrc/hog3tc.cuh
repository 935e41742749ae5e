// hog3tc.cuh -- order-3 S^3CMTF epoch kernel with the sweep's core
// contractions on the tensor cores (opt kernel, J in {4,5,8,10}).
//
// Same execution model as hog3v2 (one launch per epoch, grid 148 x 8 warps,
// a contiguous chunk of the per-epoch reshuffled COO per lane, interleaved
// matrix entries, hot-row replicas with damped merges, cold-row steps as
// vector REDs, cp.async row gathers overlapped with the iteration tail, the
// core gradient on the tensor cores, block-level damped core push).  What
// changes is the per-entry contraction (Algorithm 3, src/gradients.cpp:
// 130-223 restated): a warp's 32 entries form two m-tiles of 16 and
//   GEMM1  T[e][(a,b)] = sum_c u3_e[c] G[a,b,c]     (M = e, K = c, N = b per a)
//   GEMM2  g3[e][c]    = sum_(a,b) u1_e[a]u2_e[b] G[a,b,c]  (K = b per a)
// run as mma.sync m16n8k8 TF32 (b and c zero-padded to KB = 8 or 16); from T
// the quad of lanes that holds an entry forms W1[a] = sum_b T u2[b] (quad
// sum), g2[b] = sum_a T u1[a] (complete per lane: the lane owns its b
// columns) and x = W1.u1.  Each lane then steps its owned components of the
// entry's three rows.  FP32 work per entry drops from 2*Pi to O(J*KB).
#pragma once

#include "hog3v2.cuh"

#ifndef CMTF_TC3_UNROLL
#define CMTF_TC3_UNROLL 2
#endif

namespace cmtfb {

template <int J, int NW>
struct V3TCLayout {
  static constexpr int JP = round_up4(J);
  static constexpr int KB = J <= 8 ? 8 : 16;   // padded b / c extent
  static constexpr int H = KB / 8;             // 8-wide b halves = c k-steps = c n-tiles
  static constexpr int S1 = KB == 8 ? 12 : 20; // G1 [a][b][c]: rows g8 x cols t4 conflict-free
  static constexpr int S2 = KB == 8 ? 8 : 24;  // G2 [a][b][c]: rows t4 x cols g8 conflict-free
  static constexpr int G1_FLOATS = J * KB * S1;
  static constexpr int G2_FLOATS = J * KB * S2;
  static constexpr int AB = J * J;
  static constexpr int sw_pick(int x) {
    return ((x % 32) == 8 || (x % 32) == 24) ? x : sw_pick(x + 4);
  }
  static constexpr int SW = sw_pick(3 * KB);   // stage row: u1 | u2 | u3, stride KB
  static constexpr int NT = (AB + 7) / 8;      // core-gradient n-tiles (ab)
  static constexpr int MT = (J + 15) / 16;     // core-gradient m-tiles (c)
  static constexpr int DG_FLOATS = AB * KB;    // per-warp core-gradient accumulator
  static constexpr int STAGE_FLOATS = 32 * SW;
  static constexpr int META_WORDS = 32 * 12;   // ix[3], slot[3], reg[3], x, active
  static constexpr int WARP_FLOATS = DG_FLOATS + STAGE_FLOATS + META_WORDS;
  static constexpr int FIXED_FLOATS = G1_FLOATS + G2_FLOATS + NW * WARP_FLOATS;
};

template <int J, int NW>
__global__ void __launch_bounds__(NW * 32, 1)
hog3tc_kernel(Hog3v2Args a) {
  using L = V3TCLayout<J, NW>;
  constexpr int JP = L::JP, KB = L::KB, H = L::H, S1 = L::S1, S2 = L::S2, SW = L::SW;
  constexpr int AB = L::AB;
  constexpr int kUnrollA = CMTF_TC3_UNROLL;
  extern __shared__ __align__(16) float sm[];
  float* G1 = sm;
  float* G2 = G1 + L::G1_FLOATS;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g8 = lane >> 2, t4 = lane & 3;
  float* dGw = G2 + L::G2_FLOATS + w * L::WARP_FLOATS;
  float* stg = dGw + L::DG_FLOATS;  // [32][SW]
  uint32_t* meta = reinterpret_cast<uint32_t*>(stg + L::STAGE_FLOATS);  // [32][12]
  float* myst = stg + lane * SW;

  // ---- prologue: padded core copies, zeroed staging, hot replicas ----
  for (int q = threadIdx.x; q < J * KB * KB; q += blockDim.x) {
    const int c = q % KB, b = (q / KB) % KB, ia = q / (KB * KB);
    const float v = (b < J && c < J) ? __ldcg(a.G + (ia * J + b) * J + c) : 0.f;
    G1[(ia * KB + b) * S1 + c] = v;
    G2[(ia * KB + b) * S2 + c] = v;
  }
  for (int q = lane; q < L::DG_FLOATS + L::STAGE_FLOATS; q += 32) dGw[q] = 0.f;
#pragma unroll
  for (int n = 0; n < 3; ++n)
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
  float kw = 0.f, lamG = 0.f;
#define REP(n) (sm + a.hot[n].off)
#define STAT(n) (sm + a.hot[n].stat_off)

  // ---- software pipeline (records two ahead, slots / reg one ahead, the
  // next entry's cold rows cp.async'ed into the staging row) ----
  auto issue_rows = [&](const uint4 r, const int* slx) {
    const uint32_t ix[3] = {r.x, r.y, r.z};
#pragma unroll
    for (int n = 0; n < 3; ++n)
      if (slx[n] < 0) {
        const float* src = a.U[n] + (uint64_t)ix[n] * JP;
#pragma unroll
        for (int k = 0; k < JP; k += 4) cp_async16(myst + n * KB + k, src + k);
      }
    cp_async_commit();
  };
  uint4 rc = lo < hi ? __ldg(a.rec + lo) : make_uint4(0, 0, 0, 0);
  uint4 rc1 = lo + 1 < hi ? __ldg(a.rec + lo + 1) : make_uint4(0, 0, 0, 0);
  int sl[3];
  float rg[3];
  {
    const uint32_t ix[3] = {rc.x, rc.y, rc.z};
#pragma unroll
    for (int n = 0; n < 3; ++n) {
      sl[n] = (lo < hi && a.hot[n].slot) ? __ldg(a.hot[n].slot + ix[n]) : -1;
      rg[n] = lo < hi ? __ldg(a.reg[n] + ix[n]) : 0.f;
    }
  }
  if (lo < hi) issue_rows(rc, sl);
  cp_async_commit();  // (empty) core-refresh group: see the push

  for (uint64_t it = 0; it < iters; ++it) {
    const uint64_t e = lo + it;
    const bool active = e < hi;
    const uint4 rc2 = e + 2 < hi ? __ldg(a.rec + e + 2) : make_uint4(0, 0, 0, 0);
    int nsl[3];
    float nrg[3];
    {
      const bool nxt = e + 1 < hi;
      const uint32_t nx[3] = {rc1.x, rc1.y, rc1.z};
#pragma unroll
      for (int n = 0; n < 3; ++n) {
        nsl[n] = a.hot[n].slot ? __ldg(a.hot[n].slot + (nxt ? nx[n] : 0u)) : -1;
        nrg[n] = __ldg(a.reg[n] + (nxt ? nx[n] : 0u));
      }
    }
    cp_async_wait_group<1>();

    // ---- the lane's entry: rows into its staging row, metadata ----
    if (active) {
#pragma unroll
      for (int n = 0; n < 3; ++n)
        if (sl[n] >= 0) {
#pragma unroll
          for (int k = 0; k < JP; k += 4)
            *reinterpret_cast<float4*>(myst + n * KB + k) =
                *reinterpret_cast<const float4*>(REP(n) + sl[n] * JP + k);
        }
    } else {
#pragma unroll
      for (int n = 0; n < 3; ++n)
#pragma unroll
        for (int k = 0; k < JP; k += 4)
          *reinterpret_cast<float4*>(myst + n * KB + k) = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    {
      uint32_t* mm = meta + lane * 12;
      *reinterpret_cast<uint4*>(mm) =
          make_uint4(rc.x, rc.y, rc.z, (uint32_t)(active ? sl[0] : -1));
      *reinterpret_cast<uint4*>(mm + 4) =
          make_uint4((uint32_t)(active ? sl[1] : -1), (uint32_t)(active ? sl[2] : -1),
                     __float_as_uint(rg[0]), __float_as_uint(rg[1]));
      *reinterpret_cast<uint4*>(mm + 8) =
          make_uint4(__float_as_uint(rg[2]), rc.w, active ? 1u : 0u, 0u);
    }
    __syncwarp();

    // ---- tensor-core contractions, two m-tiles of 16 entries ----
#pragma unroll 1
    for (int mt = 0; mt < 2; ++mt) {
      const int R0 = mt * 16 + g8, R1 = R0 + 8;
      float* s0 = stg + R0 * SW;
      float* s1 = stg + R1 * SW;
      uint32_t av[H][4];  // GEMM1 A: u3[e][c], k-step ks = c / 8
#pragma unroll
      for (int ks = 0; ks < H; ++ks) {
        av[ks][0] = __float_as_uint(s0[2 * KB + ks * 8 + t4]);
        av[ks][1] = __float_as_uint(s1[2 * KB + ks * 8 + t4]);
        av[ks][2] = __float_as_uint(s0[2 * KB + ks * 8 + t4 + 4]);
        av[ks][3] = __float_as_uint(s1[2 * KB + ks * 8 + t4 + 4]);
      }
      float u2o[2][H][2], u2k[2][H][2];  // owned b columns; GEMM2 A columns
#pragma unroll
      for (int h = 0; h < H; ++h) {
        const float2 p0 = *reinterpret_cast<const float2*>(s0 + KB + h * 8 + 2 * t4);
        const float2 p1 = *reinterpret_cast<const float2*>(s1 + KB + h * 8 + 2 * t4);
        u2o[0][h][0] = p0.x; u2o[0][h][1] = p0.y;
        u2o[1][h][0] = p1.x; u2o[1][h][1] = p1.y;
        u2k[0][h][0] = s0[KB + h * 8 + t4];
        u2k[0][h][1] = s0[KB + h * 8 + t4 + 4];
        u2k[1][h][0] = s1[KB + h * 8 + t4];
        u2k[1][h][1] = s1[KB + h * 8 + t4 + 4];
      }
      float g2o[2][H][2] = {};
      float g3a[H][4] = {};  // g3[R0][c], g3[R0][c+1], g3[R1][c], g3[R1][c+1], c = nt*8+2t4
      float W1o[2][2 * H] = {};
      float xh0 = 0.f, xh1 = 0.f;
#pragma unroll kUnrollA
      for (int ia = 0; ia < J; ++ia) {
        const float ua0 = s0[ia], ua1 = s1[ia];
        const float* g1a = G1 + ia * KB * S1;
        const float* g2a = G2 + ia * KB * S2;
        float w1p0 = 0.f, w1p1 = 0.f;
#pragma unroll
        for (int h = 0; h < H; ++h) {
          float d[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int ks = 0; ks < H; ++ks) {
            uint32_t bb[2];
            bb[0] = __float_as_uint(g1a[(h * 8 + g8) * S1 + ks * 8 + t4]);
            bb[1] = __float_as_uint(g1a[(h * 8 + g8) * S1 + ks * 8 + t4 + 4]);
            mma_tf32(d, av[ks], bb);  // T[R0][b], T[R0][b+1], T[R1][b], T[R1][b+1], b = h*8+2t4
          }
          w1p0 = fmaf(d[1], u2o[0][h][1], fmaf(d[0], u2o[0][h][0], w1p0));
          w1p1 = fmaf(d[3], u2o[1][h][1], fmaf(d[2], u2o[1][h][0], w1p1));
          g2o[0][h][0] = fmaf(d[0], ua0, g2o[0][h][0]);
          g2o[0][h][1] = fmaf(d[1], ua0, g2o[0][h][1]);
          g2o[1][h][0] = fmaf(d[2], ua1, g2o[1][h][0]);
          g2o[1][h][1] = fmaf(d[3], ua1, g2o[1][h][1]);
          uint32_t ap[4];
          ap[0] = __float_as_uint(ua0 * u2k[0][h][0]);
          ap[1] = __float_as_uint(ua1 * u2k[1][h][0]);
          ap[2] = __float_as_uint(ua0 * u2k[0][h][1]);
          ap[3] = __float_as_uint(ua1 * u2k[1][h][1]);
#pragma unroll
          for (int nt = 0; nt < H; ++nt) {
            uint32_t b2[2];
            b2[0] = __float_as_uint(g2a[(h * 8 + t4) * S2 + nt * 8 + g8]);
            b2[1] = __float_as_uint(g2a[(h * 8 + t4 + 4) * S2 + nt * 8 + g8]);
            mma_tf32(g3a[nt], ap, b2);
          }
        }
        w1p0 += __shfl_xor_sync(0xffffffffu, w1p0, 1);
        w1p1 += __shfl_xor_sync(0xffffffffu, w1p1, 1);
        w1p0 += __shfl_xor_sync(0xffffffffu, w1p0, 2);
        w1p1 += __shfl_xor_sync(0xffffffffu, w1p1, 2);
        xh0 = fmaf(w1p0, ua0, xh0);
        xh1 = fmaf(w1p1, ua1, xh1);
        // owned mode-1 components: a = h*8 + 2t4 + {0,1}
#pragma unroll
        for (int h = 0; h < H; ++h) {
          if (ia == h * 8 + 2 * t4) { W1o[0][2 * h] = w1p0; W1o[1][2 * h] = w1p1; }
          if (ia == h * 8 + 2 * t4 + 1) { W1o[0][2 * h + 1] = w1p0; W1o[1][2 * h + 1] = w1p1; }
        }
      }

      // ---- residuals; each lane steps its owned components ----
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        float* sq = q ? s1 : s0;
        const uint32_t* mq = meta + (q ? R1 : R0) * 12;
        const bool act = mq[10] != 0u;
        const float r = act ? __uint_as_float(mq[9]) - (q ? xh1 : xh0) : 0.f;
        // owned pairs: mode 1 a = h*8+2t4, mode 2 b = h*8+2t4, mode 3 c = h*8+2t4
        float uv[3][H][2], gv[3][H][2];
#pragma unroll
        for (int h = 0; h < H; ++h) {
          const int k = h * 8 + 2 * t4;
          const float2 x1 = *reinterpret_cast<const float2*>(sq + k);
          const float2 x3 = *reinterpret_cast<const float2*>(sq + 2 * KB + k);
          uv[0][h][0] = x1.x; uv[0][h][1] = x1.y;
          uv[1][h][0] = u2o[q][h][0]; uv[1][h][1] = u2o[q][h][1];
          uv[2][h][0] = x3.x; uv[2][h][1] = x3.y;
          gv[0][h][0] = W1o[q][2 * h]; gv[0][h][1] = W1o[q][2 * h + 1];
          gv[1][h][0] = g2o[q][h][0]; gv[1][h][1] = g2o[q][h][1];
          gv[2][h][0] = g3a[h][2 * q]; gv[2][h][1] = g3a[h][2 * q + 1];
        }
        float nrm[6];
#pragma unroll
        for (int n = 0; n < 3; ++n) {
          float su = 0.f, sg = 0.f;
#pragma unroll
          for (int h = 0; h < H; ++h) {
            su = fmaf(uv[n][h][0], uv[n][h][0], fmaf(uv[n][h][1], uv[n][h][1], su));
            sg = fmaf(gv[n][h][0], gv[n][h][0], fmaf(gv[n][h][1], gv[n][h][1], sg));
          }
          nrm[n] = su;
          nrm[3 + n] = sg;
        }
#pragma unroll
        for (int n = 0; n < 6; ++n) {
          nrm[n] += __shfl_xor_sync(0xffffffffu, nrm[n], 1);
          nrm[n] += __shfl_xor_sync(0xffffffffu, nrm[n], 2);
        }
        if (act && t4 == 0) {
          lamG += nrm[0] * nrm[1] * nrm[2];
          kw += 1.f;
        }
        if (act) {
#pragma unroll
          for (int n = 0; n < 3; ++n) {
            const float rgn = __uint_as_float(mq[6 + n]);
            const int slot = (int)mq[3 + n];
            const uint32_t row = mq[n];
#pragma unroll
            for (int h = 0; h < H; ++h) {
              const int k = h * 8 + 2 * t4;
              if (k >= J) continue;
              float d0 = -a.eta * fmaf(-r, gv[n][h][0], rgn * uv[n][h][0]);
              float d1 = k + 1 < J ? -a.eta * fmaf(-r, gv[n][h][1], rgn * uv[n][h][1]) : 0.f;
              if (slot >= 0) {
                float2* rp = reinterpret_cast<float2*>(REP(n) + slot * JP + k);
                float2 cur = *rp;
                cur.x += d0;
                cur.y += d1;
                if (a.nonneg) { cur.x = fmaxf(cur.x, 0.f); cur.y = fmaxf(cur.y, 0.f); }
                *rp = cur;
              } else if (!a.nonneg) {
                float* gp = a.U[n] + (uint64_t)row * JP + k;
                asm volatile("red.relaxed.gpu.global.add.v2.f32 [%0], {%1,%2};" ::"l"(gp),
                             "f"(d0), "f"(d1)
                             : "memory");
              } else {
                *reinterpret_cast<float2*>(a.U[n] + (uint64_t)row * JP + k) =
                    make_float2(fmaxf(uv[n][h][0] + d0, 0.f), fmaxf(uv[n][h][1] + d1, 0.f));
              }
            }
            if (slot >= 0 && t4 == 0) {
              STAT(n)[3 * slot] += nrm[3 + n];
              atomicAdd(reinterpret_cast<int*>(STAT(n)) + 3 * slot + 1, 1);
            }
          }
        }
        // stage -r u1 (pre-update) for the core gradient
#pragma unroll
        for (int h = 0; h < H; ++h)
          *reinterpret_cast<float2*>(sq + h * 8 + 2 * t4) =
              make_float2(-r * uv[0][h][0], -r * uv[0][h][1]);
      }
    }
    __syncwarp();

    // ---- core gradient of the warp's 32 entries (tensor cores) ----
    core_grad_mma<J, KB, SW, AB, L::NT, L::MT>(stg, dGw, g8, t4);
    __syncwarp();  // staging row free: start the next entry's gathers
    if (e + 1 < hi) issue_rows(rc1, nsl);

    // ---- matrix entries due by this iteration (interleaved) ----
    matrix_entries_until<J, JP>(a, sm, mpos, mrn, mlo + (mhi - mlo) * (it + 1) / iters, mhi,
                                lane);
    rc = rc1;
    rc1 = rc2;
#pragma unroll
    for (int n = 0; n < 3; ++n) {
      sl[n] = nsl[n];
      rg[n] = nrg[n];
    }

    // ---- block-level damped core push (every core_every iterations) ----
    if ((it + 1) % (uint64_t)a.core_every == 0 || it + 1 == iters) {
      __shared__ float red_kw[NW], red_lam[NW];
      const float kws = warp_sum(kw);
      const float lgs = warp_sum(lamG);
      if (lane == 0) {
        red_kw[w] = kws;
        red_lam[w] = lgs;
      }
      kw = 0.f;
      lamG = 0.f;
      __syncthreads();
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
        float* dG0 = G2 + L::G2_FLOATS;
        for (int el = threadIdx.x; el < AB * J; el += NW * 32) {
          const int ab = el / J, c = el - (el / J) * J;
          const int ia = ab / J, ib = ab - (ab / J) * J;
          const int o = ab * KB + c;
          float sum = 0.f;
#pragma unroll
          for (int q2 = 0; q2 < NW; ++q2) {
            float* dq = dG0 + q2 * L::WARP_FLOATS + o;
            sum += *dq;
            *dq = 0.f;
          }
          float* p1 = G1 + (ia * KB + ib) * S1 + c;
          float* p2 = G2 + (ia * KB + ib) * S2 + c;
          const float delta = s * fmaf(kb * a.core_reg, *p1, sum);
          if (a.nonneg) {
            const float v = atomic_add_clamp0(a.G + el, delta);
            *p1 = v;
            *p2 = v;
          } else {
            red_add_f32(a.G + el, delta);
            cp_async4(p1, a.G + el);
            cp_async4(p2, a.G + el);
          }
        }
      }
      __syncthreads();
    }
    cp_async_commit();  // core refresh group (possibly empty)
    if ((it + 1) % (uint64_t)a.flush_every == 0 || it + 1 == iters)
      flush_all_hot<J, JP, NW>(a, sm, w, lane);
  }
  matrix_entries_until<J, JP>(a, sm, mpos, mrn, mhi, mhi, lane);
  cp_async_wait_all();
  __syncthreads();
  flush_all_hot<J, JP, NW>(a, sm, w, lane);
#undef REP
#undef STAT
}

}  // namespace cmtfb
