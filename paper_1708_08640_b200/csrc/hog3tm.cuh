// hog3tm.cuh -- order-3 S^3CMTF epoch kernel with the per-entry core
// contractions AND the core gradient on the 5th-generation tensor cores
// (tcgen05.mma, accumulators in tensor memory).
//
// Same epoch contract as hog3v2 (one launch = one epoch over the tensor and
// the coupled matrices, hot-row replicas with damped merges, interleaved
// matrix entries, block-level damped core push); only the arithmetic of a
// tensor entry moves.  A block is 2 warpgroups; each warpgroup sweeps a tile
// of 128 entries per iteration, thread e of the warpgroup owning entry e of
// the tile (TMEM lane e).  Per tile (Algorithm 3's quantities,
// src/gradients.cpp:130-223):
//
//   T[e][(a,b)] = sum_c u3_e[c] G[a,b,c]      MMA  A = U3 tile, B = G (ab x c)
//   V[e][(a,c)] = sum_b u2_e[b] G[a,b,c]      MMA  A = U2 tile, B = G (ac x b)
//   W1[a] = sum_b T[ab] u2[b],  g2[b] = sum_a T[ab] u1[a],  g3[c] = sum_a V[ac] u1[a],
//   x_hat = sum_a W1[a] u1[a]                 FP32, 3 J^2 FMAs per entry
//   dG[(a,b)][c] += sum_e P^T[ab][e] S[e][c]  MMA  A = P^T (u1[a] u2[b] per entry),
//                                                  B = S^T (-r u3 per entry), fp16
//
// so an entry costs ~3J^2 FP32 FMAs instead of hog3v2's 2J^3 + 3J^2, and the
// core gradient accumulates in tensor memory across the tile's 128 entries.
// All operands are K-major, no-swizzle canonical layouts (umma.cuh): the
// factor rows gathered with cp.async land directly in the U2/U3 operand tiles
// (row e = 16-byte chunks at stride 2048 B), P^T and S^T are written as
// transposed columns (one 4-byte store per element, bank-conflict-free).
// The sweep MMAs take TF32 operands (the gathered fp32 rows as they are); the
// core-gradient operands are fp16 (the same 10-bit mantissa as TF32, half the
// shared memory: it goes to hot-row replicas), S^T pre-scaled by 2^8 so small
// residuals stay normal; fp32 accumulation everywhere.
#pragma once

#include <cuda_fp16.h>

#include "common.cuh"
#include "hog3v2.cuh"
#include "umma.cuh"

#ifndef CMTF_TM_REFRESH
#define CMTF_TM_REFRESH 4  // pushes between refreshes of the shared core copies
#endif
#ifndef CMTF_TM_MPF
#define CMTF_TM_MPF 0  // matrix entries fetched one entry ahead: config 2 -0.9%, config 5 (rank 5) +13% -- off
#endif
#ifndef CMTF_TM_FSTAGE
#define CMTF_TM_FSTAGE 1  // hot-row merges with cp.async-staged global reads
#endif
#ifndef CMTF_TM_PROF
#define CMTF_TM_PROF 0
#endif
#ifndef CMTF_TM_EXACT
#define CMTF_TM_EXACT 0
#endif

namespace cmtfb {

__host__ __device__ constexpr int round_up8(int x) { return (x + 7) & ~7; }
__host__ __device__ constexpr int round_up16(int x) { return (x + 15) & ~15; }

template <int J>
struct TMLayout {
  static constexpr int JP = round_up4(J);
  static constexpr int KT = round_up8(J);      // K of the sweep MMAs (c or b, zero padded)
  static constexpr int AB = J * J;
  static constexpr int NT = round_up16(AB);    // N of the sweep MMAs ((a,b) or (a,c))
  static constexpr int MR = round_up8(AB);     // stored rows of P^T (the MMA reads 128)
  static constexpr int KC = 16;                // N of the core-gradient MMA (c, zero padded)
  // byte strides between 4-column groups (K direction); rows are 16 B apart
  static constexpr int G_KS = NT * 16;
  static constexpr int U_KS = 128 * 16;
  // fp16 core-gradient operands: 8 entries per 16-byte row chunk
  static constexpr int PT_KS = MR * 16 + 16;   // +16: column writes hit distinct banks
  // S^T column-group stride: holds the 16 c rows, makes a warp's 4 column
  // groups (its own slab) big enough for its push transpose (32 x J floats),
  // and keeps the column writes conflict-free ((ST_KS / 4) mod 8 == 4)
  static constexpr int st_ks(int v) { return (v % 16 == 0 && (v / 4) % 8 == 4) ? v : st_ks(v + 16); }
  static constexpr int ST_KS = st_ks(KC * 16 > 32 * J ? KC * 16 : 32 * J);
  static constexpr int G_BYTES = (KT / 4) * G_KS;
  static constexpr int U_BYTES = (KT / 4) * U_KS;
  static constexpr int U1_BYTES = 128 * JP * 4;
  static constexpr int PT_BYTES = 16 * PT_KS;  // 128 entries = 16 groups of 8
  // S^T also serves as the core push's transpose scratch (4 warps x 32 rows x J)
  static constexpr int ST_BYTES = 16 * ST_KS;
  // per warpgroup: P^T first (the M = 128 MMA reads rows MR..127 of the last
  // column group past its end: they land in S^T / U tiles, and only feed the
  // ignored core-gradient rows ab >= J^2)
  static constexpr int WG_BYTES = PT_BYTES + ST_BYTES + 2 * U_BYTES + U1_BYTES;
  static constexpr int FIXED_BYTES = 2 * G_BYTES + 2 * WG_BYTES;
  static constexpr int FIXED_FLOATS = FIXED_BYTES / 4;
  // tensor memory per warpgroup: T [0, NT), V [NT, 2 NT), dG [2 NT, 2 NT + KC)
  static constexpr int TM_COLS = 2 * NT + KC;
  static_assert(TM_COLS <= 256, "two warpgroups must fit in 512 TMEM columns");
  static_assert(AB <= 128, "core-gradient MMA has M = 128 rows (a,b)");
  // the staged hot-row merge fits a warp's P^T slice (J >= 8)
  static constexpr bool FSTAGE = 2 * 32 * 2 * JP * 4 <= 4 * PT_KS;
};

// Hot-row merge (flush_hot's arithmetic, hog3v2.cuh) with the two global reads
// of each row -- its current value and this block's base -- staged through
// shared memory with cp.async two rows per lane ahead, so a lane's rows cost
// one L2 round trip in all instead of one each.  `stage`: the warp's slice of
// its P^T buffer (free after the core MMA), 2 slots x 32 lanes x 2 JP floats.
template <int J, int JP>
__device__ void flush_hot_staged(const HotDesc& h, float* U, float* rep, float* stat, float eta,
                                 float kappa, int r0, int r1, int lane, float* stage) {
  float* base_b = h.base + (uint64_t)blockIdx.x * h.H * JP;
  auto issue = [&](int s, int slot) {
    if (s < r1) {
      float* st = stage + (slot * 32 + lane) * 2 * JP;
      const float* g = U + (uint64_t)__ldg(h.row_of + s) * JP;
#pragma unroll
      for (int k = 0; k < JP; k += 4) {
        cp_async16(st + k, g + k);
        cp_async16(st + JP + k, base_b + s * JP + k);
      }
    }
    cp_async_commit();
  };
  issue(r0 + lane, 0);
  int slot = 0;
  for (int s = r0 + lane; s < r1; s += 32, slot ^= 1) {
    issue(s + 32, slot ^ 1);
    cp_async_wait_group<1>();
    const float* st = stage + (slot * 32 + lane) * 2 * JP;
    float4 gv[JP / 4], bv[JP / 4], sv[JP / 4];
#pragma unroll
    for (int k = 0; k < JP / 4; ++k) {
      gv[k] = *reinterpret_cast<const float4*>(st + 4 * k);
      bv[k] = *reinterpret_cast<const float4*>(st + JP + 4 * k);
      sv[k] = *reinterpret_cast<const float4*>(rep + s * JP + 4 * k);
    }
    const float cnt = (float)atomicExch(reinterpret_cast<int*>(stat) + 3 * s + 1, 0);
    const float lam = stat[3 * s];
    stat[3 * s] = 0.f;
    float alpha = 0.f;
    if (cnt > 0.f) {
      const float n_other = stat[3 * s + 2] * (1.f - 1.f / (float)gridDim.x);
      const float gain = CMTF_SAT_GAIN ? -expm1f(-eta * lam) : eta * lam;
      alpha = kappa / (kappa + (n_other / cnt) * gain);
    }
    float* g = U + (uint64_t)__ldg(h.row_of + s) * JP;
#pragma unroll
    for (int k = 0; k < JP / 4; ++k) {
      float4 dl = make_float4(alpha * (sv[k].x - bv[k].x), alpha * (sv[k].y - bv[k].y),
                              alpha * (sv[k].z - bv[k].z), alpha * (sv[k].w - bv[k].w));
      if (cnt > 0.f) red_add_v4(g + 4 * k, dl);
      const float4 nb = make_float4(gv[k].x + dl.x, gv[k].y + dl.y, gv[k].z + dl.z, gv[k].w + dl.w);
      st_weak4(base_b + s * JP + 4 * k, nb);
      float4 cur = *reinterpret_cast<float4*>(rep + s * JP + 4 * k);
      cur.x += nb.x - sv[k].x; cur.y += nb.y - sv[k].y;
      cur.z += nb.z - sv[k].z; cur.w += nb.w - sv[k].w;
      *reinterpret_cast<float4*>(rep + s * JP + 4 * k) = cur;
    }
  }
  cp_async_wait_all();
}

template <int J, int JP, int NW, class Args>
__device__ __forceinline__ void flush_all_hot_staged(const Args& a, float* sm, int w, int lane,
                                                     float* stage) {
#pragma unroll
  for (int n = 0; n < 3; ++n) {
    const HotDesc& h = a.hot[n];
    if (h.H) {
      const int r0 = (int)((uint64_t)h.H * w / NW), r1 = (int)((uint64_t)h.H * (w + 1) / NW);
      flush_hot_staged<J, JP>(h, a.U[n], sm + h.off, sm + h.stat_off, a.eta, a.kappa, r0, r1,
                              lane, stage);
    }
  }
  for (int m = 0; m < a.n_mat; ++m) {
    const HotDesc& h = a.mats[m].hotV;
    if (h.H) {
      const int r0 = (int)((uint64_t)h.H * w / NW), r1 = (int)((uint64_t)h.H * (w + 1) / NW);
      flush_hot_staged<J, JP>(h, a.mats[m].V, sm + h.off, sm + h.stat_off, a.eta, a.kappa, r0,
                              r1, lane, stage);
    }
  }
}

template <int J>
__global__ void __launch_bounds__(256, 1) hog3tm_kernel(Hog3v2Args a) {
  using L = TMLayout<J>;
  constexpr int JP = L::JP, KT = L::KT, AB = L::AB, NT = L::NT;
  constexpr int NW = 8;
  extern __shared__ __align__(1024) float sm[];
  uint8_t* smb = reinterpret_cast<uint8_t*>(sm);
  uint8_t* Gc = smb;                 // B of T:  rows (a,b), K = c
  uint8_t* Gb = smb + L::G_BYTES;    // B of V:  rows (a,c), K = b
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = threadIdx.x >> 7;    // warpgroup
  const int e = threadIdx.x & 127;   // tile row = TMEM lane
  uint8_t* wgb = smb + 2 * L::G_BYTES + g * L::WG_BYTES;
  uint8_t* PT = wgb;
  uint8_t* ST = PT + L::PT_BYTES;
  uint8_t* tU2 = ST + L::ST_BYTES;
  uint8_t* tU3 = tU2 + L::U_BYTES;
  float* sU1 = reinterpret_cast<float*>(tU3 + L::U_BYTES);
  __shared__ uint64_t mbar[2][2];    // [warpgroup][sweep MMAs done, core MMA done]
  __shared__ uint32_t st_arrive[2];  // warps done with their S^T columns (monotonic)
  __shared__ uint32_t tmem_base;

  auto gc_off = [](int ab, int c) { return (c >> 2) * L::G_KS + ab * 16 + (c & 3) * 4; };

  // ---- prologue: zero the operand tiles, core copies, TMEM, hot replicas ----
  for (int q = threadIdx.x; q < L::FIXED_FLOATS; q += blockDim.x) sm[q] = 0.f;
  __syncthreads();
  for (int q = threadIdx.x; q < AB * J; q += blockDim.x) {
    const int ab = q / J, c = q - (q / J) * J, ia = ab / J, ib = ab - (ab / J) * J;
    const float v = __ldcg(a.G + q);
    *reinterpret_cast<float*>(Gc + gc_off(ab, c)) = v;
    *reinterpret_cast<float*>(Gb + gc_off(ia * J + c, ib)) = v;
  }
  if (threadIdx.x == 0) {
    umma::mbar_init(&mbar[0][0], 1);
    umma::mbar_init(&mbar[0][1], 1);
    umma::mbar_init(&mbar[1][0], 1);
    umma::mbar_init(&mbar[1][1], 1);
    st_arrive[0] = st_arrive[1] = 0u;
    umma::fence_mbar_init();
  }
  if (w == 0) umma::tmem_alloc<512>(&tmem_base);
#pragma unroll
  for (int n = 0; n < 3; ++n)
    if (a.hot[n].H) load_hot<JP>(a.hot[n], a.U[n], sm + a.hot[n].off, sm + a.hot[n].stat_off);
  for (int m = 0; m < a.n_mat; ++m)
    if (a.mats[m].hotV.H)
      load_hot<JP>(a.mats[m].hotV, a.mats[m].V, sm + a.mats[m].hotV.off,
                   sm + a.mats[m].hotV.stat_off);
  umma::fence_async_smem();
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tm = tmem_base + (uint32_t)(g * 256);
  const uint32_t tm_lane = (uint32_t)(32 * (w & 3)) << 16;
  const uint32_t sPT = umma::smem_u32(PT), sST = umma::smem_u32(ST);
  const uint32_t sU2 = umma::smem_u32(tU2), sU3 = umma::smem_u32(tU3);
  const uint32_t sGc = umma::smem_u32(Gc), sGb = umma::smem_u32(Gb);
  constexpr uint32_t ID_SWEEP = umma::idesc_tf32(128, NT, false, false);
  constexpr uint32_t ID_CORE = umma::idesc_f16(128, L::KC);
  constexpr float kSScale = 256.f;  // S^T = -r u3 * 2^8 in fp16
  constexpr uint32_t kRefresh = CMTF_TM_REFRESH;

  const uint64_t Wt = (uint64_t)gridDim.x * NW * 32;
  const uint64_t gl = ((uint64_t)blockIdx.x * NW + w) * 32 + lane;
  const uint64_t lo = a.nnz * gl / Wt, hi = a.nnz * (gl + 1) / Wt;
  const uint64_t iters = (a.nnz + Wt - 1) / Wt;
  const uint64_t mlo = a.mnnz * gl / Wt, mhi = a.mnnz * (gl + 1) / Wt;
  uint64_t mpos = mlo;
#if CMTF_TM_MPF
  MatPrefetch mpf;
  mat_prefetch_init<JP>(a, mpf, mlo, mhi);
#else
  uint4 mrn = mlo < mhi ? __ldg(a.mrec + mphys(a, mlo)) : make_uint4(0, 0, 0, 0);
#endif
  float kw = 0.f, lamG = 0.f;

  const float* rep[3];
  float* stat[3];
#pragma unroll
  for (int n = 0; n < 3; ++n) {
    rep[n] = sm + a.hot[n].off;
    stat[n] = sm + a.hot[n].stat_off;
  }
  // core row (a,b) = e of this thread in the two shared core copies
  const int ia_e = e / J, ib_e = e - (e / J) * J;
  const int gb_row = (ib_e >> 2) * L::G_KS + (ib_e & 3) * 4;
  uint32_t npush = 0;
  float* myU1 = sU1 + e * JP;
  uint8_t* myU2 = tU2 + e * 16;  // chunk k4 at + k4 * U_KS
  uint8_t* myU3 = tU3 + e * 16;

  // records two ahead, slots and coefficients one ahead; the next entry's
  // cold rows are copied (cp.async) straight into the operand tiles once the
  // sweep MMAs of the current tile are done
  auto issue_rows = [&](const uint4& r, const int* slx, bool act) {
    if (act) {
      if (slx[0] < 0) {
        const float* src = a.U[0] + (uint64_t)r.x * JP;
#pragma unroll
        for (int k = 0; k < JP; k += 4) cp_async16(myU1 + k, src + k);
      }
      if (slx[1] < 0) {
        const float* src = a.U[1] + (uint64_t)r.y * JP;
#pragma unroll
        for (int k = 0; k < JP; k += 4)
          cp_async16(reinterpret_cast<float*>(myU2 + (k >> 2) * L::U_KS), src + k);
      }
      if (slx[2] < 0) {
        const float* src = a.U[2] + (uint64_t)r.z * JP;
#pragma unroll
        for (int k = 0; k < JP; k += 4)
          cp_async16(reinterpret_cast<float*>(myU3 + (k >> 2) * L::U_KS), src + k);
      }
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
  issue_rows(rc, sl, lo < hi);
  cp_async_commit();  // (empty) core-refresh group

#if CMTF_TM_PROF
  long long tprof[14] = {0};
  long long tlast = clock64();
#define TMP(k) do { const long long tn = clock64(); tprof[k] += tn - tlast; tlast = tn; } while (0)
#else
#define TMP(k) do {} while (0)
#endif
  for (uint64_t it = 0; it < iters; ++it) {
    const uint64_t e0 = lo + it;
    const bool active = e0 < hi;
    const uint32_t par = (uint32_t)(it & 1);
    const uint4 rc2 = e0 + 2 < hi ? __ldg(a.rec + e0 + 2) : make_uint4(0, 0, 0, 0);
    int nsl[3];
    float nrg[3];
    {
      const bool nxt = e0 + 1 < hi;
      const uint32_t nx[3] = {rc1.x, rc1.y, rc1.z};
#pragma unroll
      for (int n = 0; n < 3; ++n) {
        nsl[n] = a.hot[n].slot ? __ldg(a.hot[n].slot + (nxt ? nx[n] : 0u)) : -1;
        nrg[n] = __ldg(a.reg[n] + (nxt ? nx[n] : 0u));
      }
    }

    // ---- this entry's rows (cold ones landed in the tiles) ----
    cp_async_wait_group<1>();
    float u1[JP], u2[JP], u3[JP];
    if (active) {
      const float* s1 = sl[0] >= 0 ? rep[0] + sl[0] * JP : myU1;
#pragma unroll
      for (int k = 0; k < JP; k += 4) {
        const float4 q = *reinterpret_cast<const float4*>(s1 + k);
        u1[k] = q.x; u1[k + 1] = q.y; u1[k + 2] = q.z; u1[k + 3] = q.w;
      }
#pragma unroll
      for (int k = 0; k < JP; k += 4) {
        float4* d2 = reinterpret_cast<float4*>(myU2 + (k >> 2) * L::U_KS);
        float4* d3 = reinterpret_cast<float4*>(myU3 + (k >> 2) * L::U_KS);
        float4 q2, q3;
        if (sl[1] >= 0) {
          q2 = *reinterpret_cast<const float4*>(rep[1] + sl[1] * JP + k);
          *d2 = q2;
        } else {
          q2 = *d2;
        }
        if (sl[2] >= 0) {
          q3 = *reinterpret_cast<const float4*>(rep[2] + sl[2] * JP + k);
          *d3 = q3;
        } else {
          q3 = *d3;
        }
        u2[k] = q2.x; u2[k + 1] = q2.y; u2[k + 2] = q2.z; u2[k + 3] = q2.w;
        u3[k] = q3.x; u3[k + 1] = q3.y; u3[k + 2] = q3.z; u3[k + 3] = q3.w;
      }
    } else {
#pragma unroll
      for (int k = 0; k < JP; ++k) u1[k] = u2[k] = u3[k] = 0.f;
    }

    // ---- P^T column (the previous tile's core MMA must be done with it) ----
    if (it > 0) umma::mbar_wait(&mbar[g][1], par ^ 1u);
    {
      uint8_t* pcol = PT + (e >> 3) * L::PT_KS + (e & 7) * 2;
#pragma unroll
      for (int ia = 0; ia < J; ++ia)
#pragma unroll
        for (int ib = 0; ib < J; ++ib)
          *reinterpret_cast<__half*>(pcol + (ia * J + ib) * 16) = __float2half_rn(u1[ia] * u2[ib]);
    }
    umma::fence_async_smem();
    TMP(0);
    // a hardware barrier here (the last-warp-issues scheme used for the core
    // MMA measured 2% slower: the early warps then spin on the mbarrier)
    umma::bar_sync(1 + g, 128);
    if (e == 0) {
      umma::fence_after();
#pragma unroll
      for (int ks = 0; ks < KT / 8; ++ks) {
        umma::mma_tf32(tm, umma::desc(sU3 + ks * 2 * L::U_KS, L::U_KS, 128),
                       umma::desc(sGc + ks * 2 * L::G_KS, L::G_KS, 128), ID_SWEEP, ks > 0);
        umma::mma_tf32(tm + NT, umma::desc(sU2 + ks * 2 * L::U_KS, L::U_KS, 128),
                       umma::desc(sGb + ks * 2 * L::G_KS, L::G_KS, 128), ID_SWEEP, ks > 0);
      }
      umma::commit(&mbar[g][0]);
    }

    TMP(1);
    // ---- contractions out of tensor memory (FP32) ----
    float w1[J], g2[J], g3[J];
#pragma unroll
    for (int k = 0; k < J; ++k) w1[k] = g2[k] = g3[k] = 0.f;
    umma::mbar_wait(&mbar[g][0], par);
    TMP(2);
    umma::fence_after();
#pragma unroll
    for (int c0 = 0; c0 < NT; c0 += 32) {
      float v[32];
      umma::ld16(tm + tm_lane + c0, v);
      if (c0 + 16 < NT) umma::ld16(tm + tm_lane + c0 + 16, v + 16);
      umma::ld_wait();
      umma::ld_fence_regs<32>(v);
#pragma unroll
      for (int q = 0; q < 32; ++q) {
        const int col = c0 + q;
        if (col < AB) {
          const int ia = col / J, ib = col % J;
          w1[ia] = fmaf(v[q], u2[ib], w1[ia]);
          g2[ib] = fmaf(v[q], u1[ia], g2[ib]);
        }
      }
    }
#pragma unroll
    for (int c0 = 0; c0 < NT; c0 += 32) {
      float v[32];
      umma::ld16(tm + tm_lane + NT + c0, v);
      if (c0 + 16 < NT) umma::ld16(tm + tm_lane + NT + c0 + 16, v + 16);
      umma::ld_wait();
      umma::ld_fence_regs<32>(v);
#pragma unroll
      for (int q = 0; q < 32; ++q) {
        const int col = c0 + q;
        if (col < AB) {
          const int ia = col / J, ic = col % J;
          g3[ic] = fmaf(v[q], u1[ia], g3[ic]);
        }
      }
    }
#if CMTF_TM_EXACT  // diagnostics: the contractions in FP32 from the shared core copy
#pragma unroll
    for (int k = 0; k < J; ++k) w1[k] = g2[k] = g3[k] = 0.f;
#pragma unroll 1
    for (int ia = 0; ia < J; ++ia)
#pragma unroll
      for (int ib = 0; ib < J; ++ib) {
        float tab = 0.f;
        const float p = u1[ia] * u2[ib];
#pragma unroll
        for (int c = 0; c < J; ++c) {
          const float gv = *reinterpret_cast<const float*>(Gc + gc_off(ia * J + ib, c));
          tab = fmaf(gv, u3[c], tab);
          g3[c] = fmaf(gv, p, g3[c]);
        }
        w1[ia] = fmaf(tab, u2[ib], w1[ia]);
        g2[ib] = fmaf(tab, u1[ia], g2[ib]);
      }
#endif
    float xh = 0.f;
#pragma unroll
    for (int k = 0; k < J; ++k) xh = fmaf(w1[k], u1[k], xh);

    TMP(3);
    // ---- residual, row steps ----
    const float r = active ? __uint_as_float(rc.w) - xh : 0.f;
    {
      float n1 = 0.f, n2 = 0.f, n3 = 0.f, c1 = 0.f, c2 = 0.f, c3 = 0.f;
#pragma unroll
      for (int k = 0; k < J; ++k) {
        n1 = fmaf(u1[k], u1[k], n1); n2 = fmaf(u2[k], u2[k], n2); n3 = fmaf(u3[k], u3[k], n3);
        c1 = fmaf(w1[k], w1[k], c1); c2 = fmaf(g2[k], g2[k], c2); c3 = fmaf(g3[k], g3[k], c3);
      }
      if (active) {
        lamG += n1 * n2 * n3;
        kw += 1.f;
      }
      float gr[J];
#pragma unroll
      for (int k = 0; k < J; ++k) gr[k] = fmaf(-r, w1[k], rg[0] * u1[k]);
      step_row_warp<J, JP>(a.U[0], rc.x, sl[0], const_cast<float*>(rep[0]), stat[0],
                           (int)a.hot[0].off, active, u1, gr, a.eta, a.nonneg, c1, lane);
#pragma unroll
      for (int k = 0; k < J; ++k) gr[k] = fmaf(-r, g2[k], rg[1] * u2[k]);
      step_row_warp<J, JP>(a.U[1], rc.y, sl[1], const_cast<float*>(rep[1]), stat[1],
                           (int)a.hot[1].off, active, u2, gr, a.eta, a.nonneg, c2, lane);
#pragma unroll
      for (int k = 0; k < J; ++k) gr[k] = fmaf(-r, g3[k], rg[2] * u3[k]);
      step_row_warp<J, JP>(a.U[2], rc.z, sl[2], const_cast<float*>(rep[2]), stat[2],
                           (int)a.hot[2].off, active, u3, gr, a.eta, a.nonneg, c3, lane);
    }

    TMP(4);
    // push statistics of this warpgroup; they cross the barrier below
    // (per warp: the warpgroup's count and curvature sum are taken as 4x the
    // warp's -- the damping only needs their ratio, the regulariser the count)
    const bool push = (it + 1) % (uint64_t)a.core_every == 0 || it + 1 == iters;
    float kb = 0.f, lb = 0.f;
    if (push) {
      kb = 4.f * warp_sum(kw);
      lb = 4.f * warp_sum(lamG);
      kw = 0.f;
      lamG = 0.f;
    }

    // ---- S^T column (-r u3 at pre-update values), core-gradient MMA ----
    {
      uint8_t* scol = ST + (e >> 3) * L::ST_KS + (e & 7) * 2;
#pragma unroll
      for (int c = 0; c < J; ++c)
        *reinterpret_cast<__half*>(scol + c * 16) =
            __float2half_rn(fminf(fmaxf(-r * kSScale * u3[c], -65504.f), 65504.f));
    }
    umma::fence_async_smem();
    umma::fence_before();
    // no barrier: the last of the warpgroup's 4 warps to finish its S^T
    // columns issues the core MMA; nobody waits
    __syncwarp();
    bool issue_core = false;
    if (lane == 0) {
      __threadfence_block();
      issue_core = (atomicAdd(&st_arrive[g], 1u) & 3u) == 3u;
      __threadfence_block();
    }
    if (issue_core) {
      umma::fence_after();
      const uint32_t acc0 = (it % (uint64_t)a.core_every) != 0 ? 1u : 0u;
#pragma unroll
      for (int ks = 0; ks < 8; ++ks)
        umma::mma_f16(tm + 2 * NT, umma::desc(sPT + ks * 2 * L::PT_KS, L::PT_KS, 128),
                      umma::desc(sST + ks * 2 * L::ST_KS, L::ST_KS, 128), ID_CORE,
                      ks > 0 ? 1u : acc0);
      umma::commit(&mbar[g][1]);
    }

    TMP(5);
    // ---- next entry's rows into the tiles (the sweep MMAs are done) ----
    issue_rows(rc1, nsl, e0 + 1 < hi);

    TMP(6);
    // ---- matrix entries due by this iteration (interleaved) ----
#if CMTF_TM_MPF
    matrix_entries_until_pf<J, JP>(a, sm, mpos, mpf, mlo + (mhi - mlo) * (it + 1) / iters, mhi,
                                   lane);
#else
    matrix_entries_until<J, JP>(a, sm, mpos, mrn, mlo + (mhi - mlo) * (it + 1) / iters, mhi,
                                lane);
#endif

    TMP(7);
    rc = rc1;
    rc1 = rc2;
#pragma unroll
    for (int n = 0; n < 3; ++n) {
      sl[n] = nsl[n];
      rg[n] = nrg[n];
    }

    TMP(8);
    // ---- periodic core push / refresh (per warpgroup, no block barrier).
    // TMEM lane e holds core row (a,b) = e; each warp transposes its 32 rows
    // through its slice of the S^T buffer (free until the next barrier) so the
    // REDs to the global core are coalesced ----
    if (push) {
      umma::mbar_wait(&mbar[g][1], par);
      TMP(11);
      umma::fence_after();
      float v[16];
      umma::ld16(tm + tm_lane + 2 * NT, v);
      umma::ld_wait();
      umma::ld_fence_regs<16>(v);
      TMP(12);
      float* scr = reinterpret_cast<float*>(ST + (w & 3) * 4 * L::ST_KS);  // own slab
      const int row0 = 32 * (w & 3);
      if (kb > 0.f && row0 < AB) {
        const float q = a.eta * (lb / kb) * a.nhat_core;
        const float alpha = q > a.kappa_core ? a.kappa_core / q : 1.f;
        const float s = -a.eta * alpha;
        const float creg = kb * a.core_reg;
        float* Grow = a.G + e * J;
        // the shared copies follow the global core every kRefresh pushes
        // (and right away in nonnegative mode)
        const bool refresh = ++npush % kRefresh == 0;
        if (e < AB) {
          // row owner: the gradient of its row plus the regulariser, and the
          // refresh of its row in both shared copies
#pragma unroll
          for (int c = 0; c < J; ++c) {
            float* gc = reinterpret_cast<float*>(Gc + gc_off(e, c));
            float* gb = reinterpret_cast<float*>(Gb + gb_row + (ia_e * J + c) * 16);
            const float gr = fmaf(creg, *gc, v[c] * (1.f / kSScale));
            if (a.nonneg) {
              const float nv = atomic_add_clamp0(Grow + c, s * gr);
              *gc = nv;
              *gb = nv;
            } else {
              scr[lane * J + c] = gr;
              if (refresh) {
                cp_async4(gc, Grow + c);
                cp_async4(gb, Grow + c);
              }
            }
          }
        }
        __syncwarp();
        if (!a.nonneg) {  // coalesced REDs of the warp's 32 rows
          const int nval = (AB - row0 < 32 ? AB - row0 : 32) * J;
          float* Gw = a.G + row0 * J;
          // vector REDs: 4 consecutive core elements per request
          for (int m4 = lane; m4 < nval / 4; m4 += 32) {
            const float4 d = *reinterpret_cast<const float4*>(scr + 4 * m4);
            red_add_v4(Gw + 4 * m4, make_float4(s * d.x, s * d.y, s * d.z, s * d.w));
          }
          for (int m = (nval & ~3) + lane; m < nval; m += 32) red_add_f32(Gw + m, s * scr[m]);
        }
      }
      umma::fence_before();
    }
    TMP(9);
    cp_async_commit();  // core refresh group (possibly empty)
    if ((it + 1) % (uint64_t)a.flush_every == 0 || it + 1 == iters) {
      if (CMTF_TM_FSTAGE && L::FSTAGE) {
        // staging: this warp's 4 column groups of its P^T buffer (only its
        // own threads write them; the core MMA that read them is complete)
        umma::mbar_wait(&mbar[g][1], par);
        flush_all_hot_staged<J, JP, NW>(
            a, sm, w, lane, reinterpret_cast<float*>(PT + (w & 3) * 4 * L::PT_KS));
      } else {
        flush_all_hot<J, JP, NW>(a, sm, w, lane);
      }
    }
    TMP(10);
  }
#if CMTF_TM_MPF
  matrix_entries_until_pf<J, JP>(a, sm, mpos, mpf, mhi, mhi, lane);
#else
  matrix_entries_until<J, JP>(a, sm, mpos, mrn, mhi, mhi, lane);
#endif
  cp_async_wait_all();
  umma::fence_before();
  __syncthreads();
  flush_all_hot<J, JP, NW>(a, sm, w, lane);
  if (w == 0) umma::tmem_free<512>(tmem_base);
#if CMTF_TM_PROF
  if (blockIdx.x == 0 && (threadIdx.x & 127) == 0)
    printf("prof wg%d iters %llu: wait+tiles+PT %lld | bar1+issue %lld | mma wait %lld | contract %lld | "
           "rowsteps %lld | ST+bar2+issue %lld | issue_rows %lld | matrix %lld | misc %lld | push %lld | flush %lld | push.mbar %lld | push.tmem %lld\n",
           g, (unsigned long long)iters, tprof[0], tprof[1], tprof[2], tprof[3], tprof[4], tprof[5],
           tprof[6], tprof[7], tprof[8], tprof[9], tprof[10], tprof[11], tprof[12]);
#endif
}

}  // namespace cmtfb
