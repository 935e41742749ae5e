// hog3tm.cuh -- order-3 S^3CMTF epoch kernel with the per-entry core
// contractions AND the core gradient on the 5th-generation tensor cores
// (tcgen05.mma, accumulators in tensor memory), at fp32-level accuracy.
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
//   dG[(a,b)][c] += sum_e P[e][ab] S[e][c]    MMA  A = P (u1[a] u2[b] per entry),
//                                                  B = S (-r u3 per entry)
//
// so an entry costs ~3J^2 FP32 FMAs instead of hog3v2's 2J^3 + 3J^2.
//
// Accuracy: every operand is split x = hi + lo into two fp16 values (after a
// power-of-two scale that keeps both in range) and each product is formed as
// hi*hi + hi*lo + lo*hi in three kind::f16 MMAs accumulating in fp32 -- about
// 22 mantissa bits per product (5e-7 relative on the B200,
// scripts/micro/umma_prec.cu), i.e. the north_star's 1e-5 per-entry bound
// holds for the kernel's own arithmetic (tests/test_gpu_parity.py,
// test_hog3tm_kernel_probe_*).
//
// Operand layouts (umma.cuh): the sweep operands are K-major (entry rows of
// 16 bytes, so the cp.async row gathers land in the tile and the owning
// thread rewrites its row as fp16 hi/lo with 16-byte stores); the core
// gradient's P and S are MN-major, so thread e writes its own P row (J^2
// values) and S row with 16-byte stores.  The core gradient runs per warp: a
// warp's 32 entries are K = 32 of the MMA, the warpgroup's 4 warps share two
// operand slots (warps 0/2 and 1/3 take turns: the second waits for the
// first's MMA to finish reading) with one TMEM accumulator per slot, summed
// at the push.
#pragma once

#include <cuda_fp16.h>

#include "common.cuh"
#include "hog3v2.cuh"
#include "umma.cuh"

#ifndef CMTF_TM_REFRESH
#define CMTF_TM_REFRESH 1  // pushes between refreshes of the shared core copies (4: config 5
                           // converges measurably slower -- epoch-1 RMSE 0.870 vs 0.763)
#endif
#ifndef CMTF_TM_MPF
#define CMTF_TM_MPF 0  // matrix entries fetched one entry ahead: config 2 -0.9%, config 5 (rank 5) +13% -- off
#endif
#ifndef CMTF_TM_MPFL2
#define CMTF_TM_MPFL2 0  // > 0: the rows (slot, coefficient) of a lane's next matrix entry are
                         // prefetched into L2 this many iterations before the warp's matrix step
                         // is due (the step itself fetches them synchronously).  Measured same-box
                         // with 2: config 5 @1e9 +0.7%, config 3 +0.4%, config 2 +0.8% -- off: the
                         // matrix phase's 13% of the warp's cycles is not its DRAM round trips
#endif
#ifndef CMTF_TM_FSTAGE
#define CMTF_TM_FSTAGE 1  // hot-row merges with cp.async-staged global reads
#endif
#ifndef CMTF_TM_PROF
#define CMTF_TM_PROF 0
#endif
#ifndef CMTF_TM_EARLY_GATHER
#define CMTF_TM_EARLY_GATHER 0  // 1: next entry's row gathers issued as soon as the sweep MMAs are
                                // done (measured same-box: config 5 @1e9 +1.1%, config 3 -0.7%: off)
#endif
#ifndef CMTF_TM_PH2
#define CMTF_TM_PH2 1  // even J: the P rows' hi/lo halves by packed fp16 arithmetic (see core_phase)
#endif
#ifndef CMTF_TM_EXACT
#define CMTF_TM_EXACT 0
#endif

namespace cmtfb {

__host__ __device__ constexpr int round_up8(int x) { return (x + 7) & ~7; }
__host__ __device__ constexpr int round_up16(int x) { return (x + 15) & ~15; }

// Operand scales (powers of two, exact) that keep the fp16 hi/lo parts of
// ordinary values in the normal range; a value beyond 1023 overflows to inf
// in fp16, which -- like a diverged model -- surfaces as a non-finite
// parameter (DivergenceError) rather than as a silently clamped result.
constexpr float kSU = 64.f, kSG = 64.f, kSP = 64.f, kSS = 64.f;
// packed-fp16 P rows (CMTF_TM_PH2): u1 is scaled by kSP, u2 by kSP2 before
// their fp16 splits, so P carries kSP * kSP2 (a product beyond 127 overflows)
constexpr float kSP2 = 8.f;
template <int J>
constexpr bool tm_ph2() { return CMTF_TM_PH2 && J % 2 == 0; }

template <int J>
struct TMLayout {
  static constexpr int JP = round_up4(J);
  static constexpr int AB = J * J;
  static constexpr int NT = round_up16(AB);  // N of the sweep MMAs ((a,b) or (a,c))
  static constexpr int NCH = (AB + 7) / 8;   // 8-wide (a,b) chunks of a P row
  // sweep operands, fp16 K-major, K = 16 (c or b, zero padded): rows 16 B
  // apart in 8-row groups of 128 B (SBO), the two K groups LBO apart
  static constexpr int U_LBO = 128 * 16;
  static constexpr int U_TILE = 2 * U_LBO;  // one hi or lo tile of 128 entries
  static constexpr int G_LBO = NT * 16;
  static constexpr int G_TILE = 2 * G_LBO;
  // core-gradient slot: 32 entries (K) of P (M = (a,b)) and S (N = c),
  // MN-major: 16-byte chunks of 8 (a,b) / c values, the 4 K groups of 8
  // entries 128 B apart (LBO), chunks 512 B apart (SBO)
  static constexpr int P_LBO = 128, P_SBO = 512;
  static constexpr int P_BYTES = NCH * P_SBO;
  static constexpr int S_BYTES = 2 * P_SBO;
  static constexpr int SLOT = 2 * P_BYTES + 2 * S_BYTES;  // P hi, P lo, S hi, S lo
  static constexpr int U1_BYTES = 128 * JP * 4;            // fp32 staging of u1
  // the warpgroup's fp32 view of the core, row (a,b) = thread (a,b) (odd
  // stride: conflict-free); the push's regulariser reads it and the refresh
  // lands in it with cp.async before it is converted into the fp16 copies
  static constexpr int JG = J | 1;
  static constexpr int G32_BYTES = (AB * JG * 4 + 15) / 16 * 16;
  // per warpgroup: the two slots first (the M = 128 core MMA reads 16 (a,b)
  // chunks of P; those past NCH land in the following buffers and only feed
  // the ignored accumulator rows ab >= J^2)
  static constexpr int WG_BYTES = 2 * SLOT + 4 * U_TILE + U1_BYTES + G32_BYTES;
  static constexpr int G_BYTES = 4 * G_TILE;  // G (ab x c) hi, lo; G (ac x b) hi, lo
  static constexpr int FIXED_BYTES = G_BYTES + 2 * WG_BYTES;
  static constexpr int FIXED_FLOATS = FIXED_BYTES / 4;
  // tensor memory per warpgroup: T [0, NT), V [NT, 2 NT), dG of slot 0 / 1
  static constexpr int TM_COLS = 2 * NT + 32;
  static_assert(TM_COLS <= 256, "two warpgroups must fit in 512 TMEM columns");
  static_assert(AB <= 128, "core-gradient MMA has M = 128 rows (a,b)");
  // while the slots are free (after the iteration's core MMAs), each of the
  // two warps sharing a slot owns one half of it: its push transpose scratch
  // (32 rows x J floats) and its staged hot-row merge buffer (2 stages x 32
  // lanes x 2 JP floats) both live there
  static constexpr int HALF = SLOT / 2;
  static_assert(32 * J * 4 <= HALF, "push transpose scratch fits half a slot");
  static constexpr int STAGE_WARP = 2 * 32 * 2 * JP * 4;
  static constexpr bool FSTAGE = STAGE_WARP <= HALF;
};

// The record streams are read once per epoch: evict-first loads keep L2 for
// the factor rows (with the blocked order, the active row blocks).
#ifndef CMTF_TM_STREAM_LD
#define CMTF_TM_STREAM_LD 1
#endif
template <class T>
__device__ __forceinline__ T tm_ld_stream(const T* p) {
#if CMTF_TM_STREAM_LD
  return __ldcs(p);
#else
  return __ldg(p);
#endif
}

// Virtual visiting order: virtual record v of the epoch lies in segment k
// (a stratum of the physical layout, in this epoch's stratum sequence); its
// physical place is the segment's group-affine image: group g = rel / 8 ->
// (a g + b) mod ng (Barrett reduction with m = floor((2^64 - 1) / ng)), the
// offset inside the 8-record group kept, the records past the last whole
// group in place.  k is the lane's cursor: a lane's v only grow.  Eight
// consecutive lanes read one 128-byte group, so the gathers stay full-line.
__device__ __forceinline__ uint32_t vphys(const uint4* vt, uint32_t& k, uint32_t v) {
  if (!vt) return v;
  while (v >= __ldg(&vt[2 * (k + 1)].x)) ++k;
  const uint4 s0 = __ldg(vt + 2 * k), s1 = __ldg(vt + 2 * k + 1);
  const uint32_t rel = v - s0.x;
  if (rel >= s0.z) return s0.y + rel;
  const uint64_t x = (uint64_t)s1.x * (rel >> 3) + s1.y;
  const uint64_t m = ((uint64_t)s1.w << 32) | s1.z;
  uint64_t r = x - __umul64hi(x, m) * s0.w;
  if (r >= s0.w) r -= s0.w;
  return s0.y + (uint32_t)r * 8u + (rel & 7u);
}

// x -> hi + lo, two fp16 values (x already scaled): hi keeps x's top 11
// significant bits (exactly an fp16 for |x| >= 2^-14), lo = x - hi is exact
// in fp32 and rounded to fp16; hi + lo carries ~21 bits
__device__ __forceinline__ void split_h(float x, __half& h, __half& l) {
  const float hx = __uint_as_float(__float_as_uint(x) & 0xffffe000u);
  h = __float2half_rn(hx);
  l = __float2half_rn(x - hx);
}
// 8 scaled values -> one 16-byte chunk of hi halves and one of lo halves
__device__ __forceinline__ void split8(const float* v, uint4& hi, uint4& lo) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float h0 = __uint_as_float(__float_as_uint(v[2 * q]) & 0xffffe000u);
    const float h1 = __uint_as_float(__float_as_uint(v[2 * q + 1]) & 0xffffe000u);
    const __half2 hh = __floats2half2_rn(h0, h1);
    const __half2 ll = __floats2half2_rn(v[2 * q] - h0, v[2 * q + 1] - h1);
    h[q] = *reinterpret_cast<const uint32_t*>(&hh);
    l[q] = *reinterpret_cast<const uint32_t*>(&ll);
  }
  hi = make_uint4(h[0], h[1], h[2], h[3]);
  lo = make_uint4(l[0], l[1], l[2], l[3]);
}

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

// Cold-row step as one asynchronous bulk reduction (cp.reduce.async.bulk
// .add.f32) of the row's delta, staged in this thread's shared-memory row:
// the step leaves the thread at issue (a vector RED keeps its four source
// registers until the memory pipe takes them, which under scattered L2-missing
// traffic stalls the next writer of those registers).  Per element the add
// is atomic, as the RED it replaces (no lost updates on cold rows).  Hot rows
// and nonnegative mode keep step_row.  The caller waits for the previous
// entry's reductions to have read the staging (bulk_wait_read) before.
template <int J, int JP>
__device__ __forceinline__ void tm_step_row(float* U, uint32_t i, int slot, float* rep, float* stat,
                                            bool act, const float* u, const float* grad, float eta,
                                            int nonneg, float curv, float* stage) {
  if (!act) return;
  if (slot >= 0 || !stage) {
    step_row<J, JP>(U, i, slot, rep, stat, u, grad, eta, nonneg, curv);
    return;
  }
#pragma unroll
  for (int k = 0; k < JP; k += 4)
    *reinterpret_cast<float4*>(stage + k) =
        make_float4(k + 0 < J ? -eta * grad[k] : 0.f, k + 1 < J ? -eta * grad[k + 1] : 0.f,
                    k + 2 < J ? -eta * grad[k + 2] : 0.f, k + 3 < J ? -eta * grad[k + 3] : 0.f);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;"
               ::"l"(U + (uint64_t)i * JP), "r"(umma::smem_u32(stage)), "n"(JP * 4)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int J>
__global__ void __launch_bounds__(256, 1) hog3tm_kernel(Hog3v2Args a) {
  using L = TMLayout<J>;
  constexpr int JP = L::JP, AB = L::AB, NT = L::NT, NCH = L::NCH;
  constexpr int NW = 8;
  extern __shared__ __align__(1024) float sm[];
  uint8_t* smb = reinterpret_cast<uint8_t*>(sm);
  uint8_t* Gch = smb;                  // B of T: rows (a,b), K = c
  uint8_t* Gcl = Gch + L::G_TILE;
  uint8_t* Gbh = Gcl + L::G_TILE;      // B of V: rows (a,c), K = b
  uint8_t* Gbl = Gbh + L::G_TILE;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = threadIdx.x >> 7;      // warpgroup
  const int e = threadIdx.x & 127;     // tile row = TMEM lane
  const int wk = w & 3;                // warp within the warpgroup
  const int slot = wk & 1, turn = wk >> 1;
  uint8_t* wgb = smb + L::G_BYTES + g * L::WG_BYTES;
  uint8_t* myslot = wgb + slot * L::SLOT;
  uint8_t* tU2h = wgb + 2 * L::SLOT;
  uint8_t* tU2l = tU2h + L::U_TILE;
  uint8_t* tU3h = tU2l + L::U_TILE;
  uint8_t* tU3l = tU3h + L::U_TILE;
  float* sU1 = reinterpret_cast<float*>(tU3l + L::U_TILE);
  float* myG32 = reinterpret_cast<float*>(tU3l + L::U_TILE + L::U1_BYTES) + e * L::JG;
  // [warpgroup][sweep MMAs, slot 0 turn 0, slot 1 turn 0, slot 0 turn 1,
  // slot 1 turn 1]: one completion per iteration each, so a parity names the
  // iteration unambiguously (no warp is more than one iteration ahead)
  __shared__ uint64_t mbar[2][5];
  __shared__ uint32_t tmem_base;

  // core element (a,b,c) into the four fp16 copies
  auto put_g = [&](int ab, int c, float v) {
    __half h, l;
    split_h(v * kSG, h, l);
    const int ia = ab / J, ib = ab - (ab / J) * J;
    const int oc = (ab >> 3) * 128 + (ab & 7) * 16 + (c >> 3) * L::G_LBO + (c & 7) * 2;
    const int rb = ia * J + c;
    const int ob = (rb >> 3) * 128 + (rb & 7) * 16 + (ib >> 3) * L::G_LBO + (ib & 7) * 2;
    *reinterpret_cast<__half*>(Gch + oc) = h;
    *reinterpret_cast<__half*>(Gcl + oc) = l;
    *reinterpret_cast<__half*>(Gbh + ob) = h;
    *reinterpret_cast<__half*>(Gbl + ob) = l;
  };

  // ---- prologue: zero the operand tiles, core copies, TMEM, hot replicas ----
  for (int q = threadIdx.x; q < L::FIXED_FLOATS; q += blockDim.x) sm[q] = 0.f;
  __syncthreads();
  for (int q = threadIdx.x; q < AB * J; q += blockDim.x) put_g(q / J, q % J, __ldcg(a.G + q));
  if (e < AB)
#pragma unroll
    for (int c = 0; c < J; ++c) myG32[c] = __ldcg(a.G + e * J + c);
  bool g32_fresh = false;  // a refresh landed in myG32: convert it
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < 10; ++k) umma::mbar_init(&mbar[k / 5][k % 5], 1);
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
  const uint32_t tm_lane = (uint32_t)(32 * wk) << 16;
  const uint32_t sU2h = umma::smem_u32(tU2h), sU2l = umma::smem_u32(tU2l);
  const uint32_t sU3h = umma::smem_u32(tU3h), sU3l = umma::smem_u32(tU3l);
  const uint32_t sGch = umma::smem_u32(Gch), sGcl = umma::smem_u32(Gcl);
  const uint32_t sGbh = umma::smem_u32(Gbh), sGbl = umma::smem_u32(Gbl);
  const uint32_t sPh = umma::smem_u32(myslot), sPl = sPh + L::P_BYTES;
  const uint32_t sSh = sPl + L::P_BYTES, sSl = sSh + L::S_BYTES;
  constexpr uint32_t ID_SWEEP = umma::idesc_f16(128, NT);
  constexpr uint32_t ID_CORE = umma::idesc_f16(128, 16, true, true);
  constexpr float kInvT = 1.f / (kSU * kSG);
  constexpr float kInvD = 1.f / (kSP * (tm_ph2<J>() ? kSP2 : 1.f) * kSS);
  constexpr uint32_t kRefresh = CMTF_TM_REFRESH;

  const uint64_t Wt = (uint64_t)gridDim.x * NW * 32;
  const uint64_t gl = ((uint64_t)blockIdx.x * NW + w) * 32 + lane;
  // a lane's entries: a contiguous chunk (st = 1), or -- strided -- every
  // Wt-th record from its lane id, so that the whole grid sweeps the record
  // array front to back (an L2-blocked record order then keeps the active
  // row blocks L2-resident)
  const uint64_t st = a.strided ? Wt : 1;
  const uint64_t lo = a.strided ? gl : a.nnz * gl / Wt;
  const uint64_t hi = a.strided ? a.nnz : a.nnz * (gl + 1) / Wt;
  const uint64_t iters = (a.nnz + Wt - 1) / Wt;
  const uint64_t mlo = a.mnnz * gl / Wt, mhi = a.mnnz * (gl + 1) / Wt;
  uint64_t mpos = mlo;
  MatSched msched;  // warp-uniform interleaving of the matrix entries (hog3v2.cuh)
  msched.init(mlo, mhi, (a.nnz + Wt - 1) / Wt);
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
  uint32_t npush = 0;
  float* myU1 = sU1 + e * JP;
  // bulk row-step staging: 3 rows of this thread (null: REDs)
  float* mystage = a.stage_off ? sm + a.stage_off + threadIdx.x * 3 * JP : nullptr;
  // this thread's row in the sweep tiles: K group k at + k * U_LBO
  uint8_t* myU2h = tU2h + e * 16;
  uint8_t* myU2l = tU2l + e * 16;
  uint8_t* myU3h = tU3h + e * 16;
  uint8_t* myU3l = tU3l + e * 16;
  // fp32 landing place of gathered row chunk q (4 floats): hi K group 0,
  // hi K group 1, lo K group 0 -- rewritten as fp16 hi/lo before the MMA
  auto land = [&](uint8_t* th, uint8_t* tl, int q) -> float* {
    return reinterpret_cast<float*>(q == 0 ? th : q == 1 ? th + L::U_LBO : tl);
  };

  // records two ahead, slots and coefficients one ahead; the next entry's
  // cold rows are copied (cp.async) straight into the operand tiles once the
  // sweep MMAs of the current tile are done
  const bool gca = a.gather_ca != 0;
  auto issue_rows = [&](const uint4& r, const int* slx, bool act) {
    if (act) {
      if (slx[0] < 0) {
        const float* src = a.U[0] + (uint64_t)r.x * JP;
#pragma unroll
        for (int k = 0; k < JP; k += 4) cp_async16_sel(myU1 + k, src + k, gca);
      }
      if (slx[1] < 0) {
        const float* src = a.U[1] + (uint64_t)r.y * JP;
#pragma unroll
        for (int k = 0; k < JP; k += 4) cp_async16_sel(land(myU2h, myU2l, k >> 2), src + k, gca);
      }
      if (slx[2] < 0) {
        const float* src = a.U[2] + (uint64_t)r.z * JP;
#pragma unroll
        for (int k = 0; k < JP; k += 4) cp_async16_sel(land(myU3h, myU3l, k >> 2), src + k, gca);
      }
    }
    cp_async_commit();
  };
  // a row (JP floats, zero padded to K = 16) as fp16 hi/lo into this thread's tile rows
  auto put_row = [&](uint8_t* th, uint8_t* tl, const float* u) {
    float v[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = k < J ? u[k] * kSU : 0.f;
    uint4 h0, l0, h1, l1;
    split8(v, h0, l0);
    split8(v + 8, h1, l1);
    *reinterpret_cast<uint4*>(th) = h0;
    *reinterpret_cast<uint4*>(th + L::U_LBO) = h1;
    *reinterpret_cast<uint4*>(tl) = l0;
    *reinterpret_cast<uint4*>(tl + L::U_LBO) = l1;
  };
  // physical places of the records one (p1) and zero (p0) iterations ahead
  uint32_t vk = 0;
  uint32_t p0 = lo < hi ? vphys(a.vtab, vk, (uint32_t)lo) : 0u;
  uint32_t p1 = lo + st < hi ? vphys(a.vtab, vk, (uint32_t)(lo + st)) : 0u;
  uint4 rc = lo < hi ? __ldg(a.rec + p0) : make_uint4(0, 0, 0, 0);
  uint4 rc1 = lo + st < hi ? __ldg(a.rec + p1) : make_uint4(0, 0, 0, 0);
  int sl[3];
  float rg[3];
  {
    const uint32_t ix[3] = {rc.x, rc.y, rc.z};
#pragma unroll
    for (int n = 0; n < 3; ++n) {
      sl[n] = (lo < hi && a.hot[n].slot) ? __ldg(a.hot[n].slot + ix[n]) : -1;
    }
    const float4 r0 = lo < hi ? __ldg(a.rrec + p0) : make_float4(0.f, 0.f, 0.f, 0.f);
    rg[0] = r0.x;
    rg[1] = r0.y;
    rg[2] = r0.z;
  }
  issue_rows(rc, sl, lo < hi);

#if CMTF_TM_PROF
  long long tprof[14] = {0};
  long long tlast = clock64();
#define TMP(k) do { const long long tn = clock64(); tprof[k] += tn - tlast; tlast = tn; } while (0)
#else
#define TMP(k) do {} while (0)
#endif
  // the previous iteration's core push and hot-row merges, run at the top of
  // the next iteration (or after the last): every core MMA of that iteration
  // is done first, so the slots are free (until this iteration's barrier) for
  // the push transpose and the merge staging.  Runs every iteration (the
  // barrier and the slot waits; the push and merges when due), so that each
  // iteration starts with both slots' MMAs complete.
  bool pend_push = false, pend_flush = false;
  int cnt_push = 0, cnt_flush = 0;  // iterations since the last push / merge
  float pkb = 0.f, plb = 0.f;
  auto push_flush = [&](uint32_t ph) {
    // both slots' last MMAs (turn 1) of the previous iteration, parity ph
    umma::mbar_wait(&mbar[g][3], ph);
    umma::mbar_wait(&mbar[g][4], ph);
    TMP(10);
    if (pend_push) {
      // TMEM lane e holds core row (a,b) = e of both slot accumulators; each
      // warp transposes its 32 rows through its half of a slot so the REDs to
      // the global core are coalesced
      umma::fence_after();
      float v0[16], v1[16];
      umma::ld16(tm + tm_lane + 2 * NT, v0);
      umma::ld16(tm + tm_lane + 2 * NT + 16, v1);
      umma::ld_wait();
      umma::ld_fence_regs<16>(v0);
      umma::ld_fence_regs<16>(v1);
      TMP(11);
      float* scr = reinterpret_cast<float*>(myslot + turn * L::HALF);
      const int row0 = 32 * wk;
      // every warp pushes its 32 accumulator rows -- they hold all four
      // warps' entries -- even when it had no entries of its own
      if (row0 < AB) {
        const float q = pkb > 0.f ? a.eta * (plb / pkb) * a.nhat_core : 0.f;
        const float alpha = q > a.kappa_core ? a.kappa_core / q : 1.f;
        const float s = -a.eta * alpha;
        const float creg = pkb * a.core_reg;
        float* Grow = a.G + e * J;
        // the shared copies follow the global core every kRefresh pushes
        // (and right away in nonnegative mode); the refresh read is issued
        // before this push's REDs and gets this push's own delta added
        // (g_alt: the shared fp16 copies are common to both warpgroups, so
        // they take turns -- each refresh is converted once, and the copies
        // still follow the global core every push of either warpgroup)
        ++npush;
        const bool refresh =
            a.g_alt ? (npush + (uint32_t)g) % (2 * kRefresh) == 0 : npush % kRefresh == 0;
        if (e < AB) {
#pragma unroll
          for (int c = 0; c < J; ++c) {
            const float dat = (v0[c] + v1[c]) * kInvD;
            if (a.probe_core) atomicAdd(a.probe_core + e * J + c, dat);
            const float gr = fmaf(creg, myG32[c], dat);
            if (a.nonneg) {
              const float nv = atomic_add_clamp0(Grow + c, s * gr);
              myG32[c] = nv;
              put_g(e, c, nv);
            } else {
              scr[lane * J + c] = gr;
            }
          }
        }
        __syncwarp();
        if (!a.nonneg) {  // coalesced REDs of the warp's 32 rows
          const int nval = (AB - row0 < 32 ? AB - row0 : 32) * J;
          float* Gw = a.G + row0 * J;
          for (int m4 = lane; m4 < nval / 4; m4 += 32) {
            const float4 d = *reinterpret_cast<const float4*>(scr + 4 * m4);
            red_add_v4(Gw + 4 * m4, make_float4(s * d.x, s * d.y, s * d.z, s * d.w));
          }
          for (int m = (nval & ~3) + lane; m < nval; m += 32) red_add_f32(Gw + m, s * scr[m]);
          if (refresh && e < AB) {
            // the global row (with this push) lands in the fp32 view; it is
            // converted into the fp16 copies at the top of the next iteration
#pragma unroll
            for (int c = 0; c < J; ++c) cp_async4(myG32 + c, Grow + c);
            g32_fresh = true;
          }
        }
      }
      __syncwarp();
      TMP(12);
    }
    if (pend_flush) {
      if (CMTF_TM_FSTAGE && L::FSTAGE) {
        flush_all_hot_staged<J, JP, NW>(
            a, sm, w, lane, reinterpret_cast<float*>(myslot + turn * L::HALF));
      } else {
        flush_all_hot<J, JP, NW>(a, sm, w, lane);
      }
    }
    pend_push = pend_flush = false;
    TMP(13);
  };

  for (uint64_t it = 0; it < iters; ++it) {
    const uint64_t e0 = lo + it * st;
    const bool active = e0 < hi;
    const uint32_t par = (uint32_t)(it & 1);
    const uint32_t p2 = e0 + 2 * st < hi ? vphys(a.vtab, vk, (uint32_t)(e0 + 2 * st)) : 0u;
    const uint4 rc2 = e0 + 2 * st < hi ? tm_ld_stream(a.rec + p2) : make_uint4(0, 0, 0, 0);
    int nsl[3];
    float nrg[3];
    {
      const bool nxt = e0 + st < hi;
      const uint32_t nx[3] = {rc1.x, rc1.y, rc1.z};
#pragma unroll
      for (int n = 0; n < 3; ++n)
        nsl[n] = a.hot[n].slot ? __ldg(a.hot[n].slot + (nxt ? nx[n] : 0u)) : -1;
      if (a.pf_l2 && nxt) {
#pragma unroll
        for (int n = 0; n < 3; ++n)
          if (nsl[n] < 0) prefetch_row_l2<JP>(a.U[n] + (uint64_t)nx[n] * JP);
      }
      // the regulariser coefficients stream beside the records (rrec)
      const float4 rr = nxt ? tm_ld_stream(a.rrec + p1) : make_float4(0.f, 0.f, 0.f, 0.f);
      nrg[0] = rr.x;
      nrg[1] = rr.y;
      nrg[2] = rr.z;
    }

    // ---- this entry's rows (cold ones landed in the tiles) -> fp16 hi/lo ----
    cp_async_wait_group<0>();
    if (g32_fresh) {
#pragma unroll
      for (int c = 0; c < J; ++c) put_g(e, c, myG32[c]);
      g32_fresh = false;
    }
    float u1[JP], u2[JP], u3[JP];
    if (active) {
      const float* s1 = sl[0] >= 0 ? rep[0] + sl[0] * JP : myU1;
#pragma unroll
      for (int k = 0; k < JP; k += 4) {
        const float4 q1 = *reinterpret_cast<const float4*>(s1 + k);
        const float4 q2 = sl[1] >= 0 ? *reinterpret_cast<const float4*>(rep[1] + sl[1] * JP + k)
                                     : *reinterpret_cast<const float4*>(land(myU2h, myU2l, k >> 2));
        const float4 q3 = sl[2] >= 0 ? *reinterpret_cast<const float4*>(rep[2] + sl[2] * JP + k)
                                     : *reinterpret_cast<const float4*>(land(myU3h, myU3l, k >> 2));
        u1[k] = q1.x; u1[k + 1] = q1.y; u1[k + 2] = q1.z; u1[k + 3] = q1.w;
        u2[k] = q2.x; u2[k + 1] = q2.y; u2[k + 2] = q2.z; u2[k + 3] = q2.w;
        u3[k] = q3.x; u3[k + 1] = q3.y; u3[k + 2] = q3.z; u3[k + 3] = q3.w;
      }
    } else {
#pragma unroll
      for (int k = 0; k < JP; ++k) u1[k] = u2[k] = u3[k] = 0.f;
    }
    put_row(myU2h, myU2l, u2);
    put_row(myU3h, myU3l, u3);
    TMP(0);
    if (it > 0) push_flush(par ^ 1u);
    umma::fence_async_smem();
    umma::fence_before();
    TMP(9);
    umma::bar_sync(1 + g, 128);
    if (e == 0) {
      umma::fence_after();
      const uint64_t dU3h = umma::desc(sU3h, L::U_LBO, 128), dU3l = umma::desc(sU3l, L::U_LBO, 128);
      const uint64_t dU2h = umma::desc(sU2h, L::U_LBO, 128), dU2l = umma::desc(sU2l, L::U_LBO, 128);
      const uint64_t dGch = umma::desc(sGch, L::G_LBO, 128), dGcl = umma::desc(sGcl, L::G_LBO, 128);
      const uint64_t dGbh = umma::desc(sGbh, L::G_LBO, 128), dGbl = umma::desc(sGbl, L::G_LBO, 128);
      umma::mma_f16(tm, dU3h, dGch, ID_SWEEP, 0u);
      umma::mma_f16(tm, dU3h, dGcl, ID_SWEEP, 1u);
      umma::mma_f16(tm, dU3l, dGch, ID_SWEEP, 1u);
      umma::mma_f16(tm + NT, dU2h, dGbh, ID_SWEEP, 0u);
      umma::mma_f16(tm + NT, dU2h, dGbl, ID_SWEEP, 1u);
      umma::mma_f16(tm + NT, dU2l, dGbh, ID_SWEEP, 1u);
      umma::commit(&mbar[g][0]);
    }

    TMP(1);
    // ---- contractions out of tensor memory (FP32) ----
    float w1[J], g2[J], g3[J], u1t[J], u2t[J];  // u * 2^-12 undoes the operand scales
#pragma unroll
    for (int k = 0; k < J; ++k) {
      w1[k] = g2[k] = g3[k] = 0.f;
      u1t[k] = u1[k] * kInvT;
      u2t[k] = u2[k] * kInvT;
    }
    umma::mbar_wait(&mbar[g][0], par);
    TMP(2);
    umma::fence_after();
#if CMTF_TM_EARLY_GATHER
    // ---- next entry's rows into the tiles: the sweep MMAs (the tiles' only
    // readers) are done, so the gathers would get the rest of the iteration
    // to land instead of the matrix phase (turn-0 warps) ----
    issue_rows(rc1, nsl, e0 + st < hi);
#endif
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
          w1[ia] = fmaf(v[q], u2t[ib], w1[ia]);
          g2[ib] = fmaf(v[q], u1t[ia], g2[ib]);
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
          g3[ic] = fmaf(v[q], u1t[ia], g3[ic]);
        }
      }
    }
    float xh = 0.f;
#pragma unroll
    for (int k = 0; k < J; ++k) xh = fmaf(w1[k], u1[k], xh);

    TMP(3);
    // ---- residual, row steps ----
    const float r = active ? __uint_as_float(rc.w) - xh : 0.f;
    float* pr = a.probe && active ? a.probe + p0 * (uint64_t)(2 + 3 * J) : nullptr;
    if (pr) {
      pr[0] = xh;
      pr[1] = r;
    }
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
        if (a.visits) atomicAdd(a.visits + p0, 1u);
      }
      float gr[J];
#pragma unroll
      for (int k = 0; k < J; ++k) gr[k] = fmaf(-r, w1[k], rg[0] * u1[k]);
      if (pr)
#pragma unroll
        for (int k = 0; k < J; ++k) pr[2 + k] = gr[k];
      if (mystage) bulk_wait_read();  // the previous entry's reductions read their staging
      tm_step_row<J, JP>(a.U[0], rc.x, sl[0], const_cast<float*>(rep[0]), stat[0], active, u1, gr,
                         a.eta, a.nonneg, c1, (a.bulk_mask & 1) ? mystage : nullptr);
#pragma unroll
      for (int k = 0; k < J; ++k) gr[k] = fmaf(-r, g2[k], rg[1] * u2[k]);
      if (pr)
#pragma unroll
        for (int k = 0; k < J; ++k) pr[2 + J + k] = gr[k];
      tm_step_row<J, JP>(a.U[1], rc.y, sl[1], const_cast<float*>(rep[1]), stat[1], active, u2, gr,
                         a.eta, a.nonneg, c2, mystage && (a.bulk_mask & 2) ? mystage + JP : nullptr);
#pragma unroll
      for (int k = 0; k < J; ++k) gr[k] = fmaf(-r, g3[k], rg[2] * u3[k]);
      if (pr)
#pragma unroll
        for (int k = 0; k < J; ++k) pr[2 + 2 * J + k] = gr[k];
      tm_step_row<J, JP>(a.U[2], rc.z, sl[2], const_cast<float*>(rep[2]), stat[2], active, u3, gr,
                         a.eta, a.nonneg, c3, mystage && (a.bulk_mask & 4) ? mystage + 2 * JP : nullptr);
      if (mystage) bulk_commit();
    }

    TMP(4);
    // push statistics of this warpgroup (per warp: the warpgroup's count and
    // curvature sum are taken as 4x the warp's -- the damping only needs
    // their ratio, the regulariser the count); the push itself runs at the
    // top of the next iteration
    // iteration counters instead of 64-bit remainders (a software routine)
    const bool first_of_push = cnt_push == 0;
    if (++cnt_push == a.core_every) cnt_push = 0;
    if (++cnt_flush == a.flush_every) cnt_flush = 0;
    pend_push = cnt_push == 0 || it + 1 == iters;
    pend_flush = cnt_flush == 0 || it + 1 == iters;
    if (pend_push) {
      pkb = 4.f * warp_sum(kw);
      plb = 4.f * warp_sum(lamG);
      kw = 0.f;
      lamG = 0.f;
    }

    // ---- core gradient: this warp's P and S rows (pre-update values) into
    // its slot, then one warp-issued MMA (K = 32 entries) into the slot's
    // accumulator (turn 0 overwrites it at the first iteration after a push,
    // turn 1 accumulates).  Turn-0 warps do it right away; turn-1 warps first
    // issue their row gathers and matrix entries, so the turn-0 MMA is long
    // done ----
    auto core_phase = [&]() {
      if (turn == 0) {  // the slot's turn-1 MMA of the previous iteration
        if (it > 0) umma::mbar_wait(&mbar[g][3 + slot], (uint32_t)((it - 1) & 1));
      } else {          // the slot's turn-0 MMA of this iteration
        umma::mbar_wait(&mbar[g][1 + slot], par);
      }
      uint8_t* Ph = myslot + lane * 16;
      if constexpr (tm_ph2<J>()) {
        // P[ab] = u1[a] u2[b] as fp16 hi + lo without forming the fp32
        // product: with u1 = h1 + l1 and u2 = h2 + l2 split into fp16 halves
        // (11 significant bits each), hi = rn16(h1 h2), and the rounding
        // residual h1 h2 - hi has at most 11 significant bits, so one packed
        // fp16 FMA returns it exactly; lo = residual + l1 h2 + h1 l2 (the
        // l1 l2 term is below 2^-22).  Four packed instructions per two
        // elements instead of two multiplies and six split operations.
        __half2 H1[J], L1[J], h2p[J / 2], l2p[J / 2];
#pragma unroll
        for (int k = 0; k < J; ++k) {
          __half h, l;
          split_h(u1[k] * kSP, h, l);
          H1[k] = __half2half2(h);
          L1[k] = __half2half2(l);
        }
#pragma unroll
        for (int k = 0; k < J / 2; ++k) {
          const float x0 = u2[2 * k] * kSP2, x1 = u2[2 * k + 1] * kSP2;
          const float h0 = __uint_as_float(__float_as_uint(x0) & 0xffffe000u);
          const float h1 = __uint_as_float(__float_as_uint(x1) & 0xffffe000u);
          h2p[k] = __floats2half2_rn(h0, h1);
          l2p[k] = __floats2half2_rn(x0 - h0, x1 - h1);
        }
#pragma unroll
        for (int j = 0; j < NCH; ++j) {
          uint32_t hw[4], lw[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int ab = 8 * j + 2 * q;  // even, and J is even: (ab, ab + 1) share a
            if (ab < AB) {
              const int ia = ab / J, pb = (ab % J) / 2;
              const __half2 ph = __hmul2(H1[ia], h2p[pb]);
              __half2 rl = __hfma2(H1[ia], h2p[pb], __hneg2(ph));
              rl = __hfma2(L1[ia], h2p[pb], rl);
              rl = __hfma2(H1[ia], l2p[pb], rl);
              hw[q] = *reinterpret_cast<const uint32_t*>(&ph);
              lw[q] = *reinterpret_cast<const uint32_t*>(&rl);
            } else {
              hw[q] = lw[q] = 0u;
            }
          }
          *reinterpret_cast<uint4*>(Ph + j * L::P_SBO) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
          *reinterpret_cast<uint4*>(Ph + L::P_BYTES + j * L::P_SBO) =
              make_uint4(lw[0], lw[1], lw[2], lw[3]);
        }
      } else {
        float u1s[J];
#pragma unroll
        for (int k = 0; k < J; ++k) u1s[k] = u1[k] * kSP;
#pragma unroll
        for (int j = 0; j < NCH; ++j) {
          float v[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int ab = 8 * j + q;
            v[q] = ab < AB ? u1s[ab / J] * u2[ab % J] : 0.f;
          }
          uint4 h, l;
          split8(v, h, l);
          *reinterpret_cast<uint4*>(Ph + j * L::P_SBO) = h;
          *reinterpret_cast<uint4*>(Ph + L::P_BYTES + j * L::P_SBO) = l;
        }
      }
      uint8_t* Sh = myslot + 2 * L::P_BYTES + lane * 16;
      const float rs = -r * kSS;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        float v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int c = 8 * j + q;
          v[q] = c < J ? rs * u3[c] : 0.f;
        }
        uint4 h, l;
        split8(v, h, l);
        *reinterpret_cast<uint4*>(Sh + j * L::P_SBO) = h;
        *reinterpret_cast<uint4*>(Sh + L::S_BYTES + j * L::P_SBO) = l;
      }
      umma::fence_async_smem();
      __syncwarp();
      if (lane == 0) {
        umma::fence_after();
        const uint32_t d = tm + 2 * NT + 16 * slot;
        const uint32_t acc0 = (turn == 1 || !first_of_push) ? 1u : 0u;
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          const uint32_t ko = ks * 2 * L::P_LBO;
          const uint64_t dPh = umma::desc(sPh + ko, L::P_LBO, L::P_SBO);
          const uint64_t dPl = umma::desc(sPl + ko, L::P_LBO, L::P_SBO);
          const uint64_t dSh = umma::desc(sSh + ko, L::P_LBO, L::P_SBO);
          const uint64_t dSl = umma::desc(sSl + ko, L::P_LBO, L::P_SBO);
          umma::mma_f16(d, dPh, dSh, ID_CORE, ks > 0 ? 1u : acc0);
          umma::mma_f16(d, dPh, dSl, ID_CORE, 1u);
          umma::mma_f16(d, dPl, dSh, ID_CORE, 1u);
        }
        umma::commit(&mbar[g][1 + 2 * turn + slot]);
      }
    };
    if (turn == 0) core_phase();

    TMP(5);
#if !CMTF_TM_EARLY_GATHER
    // ---- next entry's rows into the tiles (the sweep MMAs are done) ----
    issue_rows(rc1, nsl, e0 + st < hi);
#endif

    TMP(6);
    // ---- matrix entries due by this iteration (interleaved) ----
    const uint64_t mdue = mlo + msched.step();
#if CMTF_TM_MPFL2 > 0 && !CMTF_TM_MPF
    // the warp's next matrix step comes exactly CMTF_TM_MPFL2 iterations from
    // now: pull the lines it will read (record mrn is in registers) into L2
    if (msched.due_in(CMTF_TM_MPFL2) && mpos >= mdue && mpos < mhi) {
      const MatDesc3& M = a.mats[mrn.w];
      if (a.hot[M.mode].slot) prefetch_l2(a.hot[M.mode].slot + mrn.x);
      if (M.hotV.slot) prefetch_l2(M.hotV.slot + mrn.y);
      prefetch_l2(M.vreg + mrn.y);
      prefetch_row_l2<JP>(a.U[M.mode] + (uint64_t)mrn.x * JP);
      prefetch_row_l2<JP>(M.V + (uint64_t)mrn.y * JP);
    }
#endif
#if CMTF_TM_MPF
    matrix_entries_until_pf<J, JP>(a, sm, mpos, mpf, mdue, mhi, lane);
#else
    matrix_entries_until<J, JP>(a, sm, mpos, mrn, mdue, mhi, lane);
#endif
    TMP(7);
    if (turn == 1) core_phase();

    TMP(8);
    rc = rc1;
    rc1 = rc2;
    p0 = p1;
    p1 = p2;
#pragma unroll
    for (int n = 0; n < 3; ++n) {
      sl[n] = nsl[n];
      rg[n] = nrg[n];
    }
  }
#if CMTF_TM_MPF
  matrix_entries_until_pf<J, JP>(a, sm, mpos, mpf, mhi, mhi, lane);
#else
  matrix_entries_until<J, JP>(a, sm, mpos, mrn, mhi, mhi, lane);
#endif
  if (iters > 0) push_flush((uint32_t)((iters - 1) & 1));
  cp_async_wait_all();
  if (mystage) bulk_wait_all();
  umma::fence_before();
  __syncthreads();
  flush_all_hot<J, JP, NW>(a, sm, w, lane);
  if (w == 0) umma::tmem_free<512>(tmem_base);
#if CMTF_TM_PROF
  if (blockIdx.x == 0 && (threadIdx.x & 31) == 0)
    printf("prof wg%d w%d iters %llu: wait+tiles %lld | push+flush %lld | bar+issue %lld | mma wait %lld | "
           "contract %lld | rowsteps %lld | core(turn0) %lld | issue_rows %lld | matrix %lld | core(turn1) %lld\n",
           g, w, (unsigned long long)iters, tprof[0], tprof[9], tprof[1], tprof[2], tprof[3], tprof[4],
           tprof[5], tprof[6], tprof[7], tprof[8]);
  if (blockIdx.x == 0 && (threadIdx.x & 31) == 0)
    printf("prof wg%d w%d push/flush: slot wait %lld | tmem ld %lld | push %lld | flush %lld\n", g, w,
           tprof[10], tprof[11], tprof[12], tprof[13]);
#endif
}

}  // namespace cmtfb
