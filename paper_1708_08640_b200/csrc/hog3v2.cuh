// hog3v2.cuh -- order-3 S^3CMTF epoch kernel, B200 design (v2).
//
// One launch = one epoch over the tensor AND the coupled matrices.
//
// Work split: every lane of every warp owns a contiguous chunk of the
// (randomly permuted) tensor COO and a contiguous chunk of the merged
// matrix COO.  Warps run free (no block barrier inside the sweep); each
// iteration a lane updates one tensor entry and the matrix entries that are
// due so that matrix updates stay interleaved with tensor updates over the
// whole epoch (as in the reference's merged shuffled schedule,
// src/trainer.cpp:114-128).
//
// Per tensor entry (OPT = Algorithm 3 reuse; NAIVE =
// Algorithm 2): the core G sits in shared memory and every
// G[a,b,c] read (a broadcast LDS) feeds two FP32 FMAs -- t_ab += G u3[c] and
// g3[c] += G u1[a]u2[b] -- then the J^2 terms W1, g2, x_hat.
//
// Core gradient dG = sum_e -r_e u1 (x) u2 (x) u3: per warp a 32-entry GEMM
// on the tensor cores, D[c][ab] += U3^T[c][e] * Q[e][ab] with
// Q[e][ab] = (-r u1)_e[a] u2_e[b], mma.sync m16n8k8 TF32 with the 3xTF32
// split (hi*hi + hi*lo + lo*hi, ~fp32 accurate), accumulated into a
// warp-private shared-memory copy and pushed to the global core with vector
// REDs every `flush_every` iterations (the reference's designated-worker
// core step, src/trainer.cpp:211-219, becomes a damped batched step).
//
// Parameter rows:
//  * cold rows: relaxed Hogwild directly on global memory (the reference's
//    relaxed.hpp contract; lost updates and stale reads allowed);
//  * hot rows (small modes, Zipf heads, small coupled factors): a per-block
//    shared-memory replica updated with shared atomics; the block pushes
//    alpha * (replica - base) to global and re-bases every flush window,
//    alpha = min(1, kappa / (eta * lambda_hat * n_hat)) with lambda_hat the
//    mean curvature |c|^2 of the row's recent updates and n_hat the expected
//    number of concurrent updates of that row GPU-wide in one window.  With
//    no contention alpha = 1 (plain SGD); with heavy contention the merged
//    step is the largest stable step of the batched least-squares problem.
#pragma once

#include "common.cuh"

#ifndef CMTF_COLD_RED
#define CMTF_COLD_RED 1  // cold-row steps as vector REDs (no lost updates)
#endif

namespace cmtfb {

constexpr int kV2MaxMats = 8;

struct HotDesc {
  const int32_t* slot;     // row -> slot, -1 cold; nullptr = no hot rows
  const uint32_t* row_of;  // slot -> row
  const uint32_t* count;   // per row observation count (for n_hat)
  uint32_t H;              // number of hot rows
  uint32_t off;            // float offset of the replica in shared memory
  uint32_t stat_off;       // float offset of the (lam, cnt, n_hat) stats
  float* base;             // [gridDim.x][H][JP] global per-block base copies
  float nhat_scale;        // n_hat = count * nhat_scale
};

struct MatDesc3 {
  int mode;
  float* V;
  const float* vreg;  // lambda_m * lambda / col count
  float weight;
  HotDesc hotV;
};

struct Hog3v2Args {
  const uint4* rec;     // tensor records {i1, i2, i3, bits(x)}, random order
  const float4* rrec;   // hog3tm: per record {lambda/count_n(i_n)}, n = 1..3, aligned with rec
  uint64_t nnz;
  const uint4* mrec;    // matrix records {row, col, bits(y), matrix id}
  uint64_t mnnz;        // total over the ranges below
  int n_mr;             // matrix record ranges swept (virtual concatenation)
  uint64_t mr_lo[kV2MaxMats];
  uint64_t mr_n[kV2MaxMats];
  int n_mat;
  MatDesc3 mats[kV2MaxMats];
  float* U[3];
  const float* reg[3];
  HotDesc hot[3];
  float* G;
  float eta;
  float core_reg;   // lambda / nnz
  float kappa;      // damping constant (hot rows)
  float kappa_core; // damping constant (core)
  float nhat_core;  // expected GPU-wide entries between two core pushes of a warp
  int flush_every;  // iterations between hot-row flushes
  int core_every;   // iterations between core pushes
  int nonneg;
  // kernel probe (hog3tm, eta = 0): per record {x_hat, r, grad u1[J], grad u2[J],
  // grad u3[J]} and the summed data term of the core gradient (null: off)
  float* probe;
  float* probe_core;
  uint32_t stage_off;  // hog3tm: shared-memory staging of the bulk row steps (floats; 0 = REDs)
  // debug_count_visits (include/cmtf/trainer.hpp:31-32): +1 per visit of a
  // tensor record (indexed like rec) / matrix record (indexed like mrec)
  uint32_t* visits;
  uint32_t* mvisits;
  int g_alt;      // hog3tm: the two warpgroups take turns converting core refreshes
  int bulk_mask;  // hog3tm: modes (bit n) whose cold-row steps use the bulk staging
  int strided;  // hog3tm: lanes take every W-th record (grid-wide front-to-back sweep)
  // hog3tm: this epoch's virtual visiting order (null = physical order):
  // segments of 2 uint4 {vbeg, src, body, ng} {a, b, m_lo, m_hi}, then a
  // sentinel with vbeg = UINT32_MAX (see vphys in hog3tm.cuh)
  const uint4* vtab;
  // hog3tm: factor tables beyond L2 -- the next entry's cold rows are
  // requested into L2 (prefetch.global.L2) at the top of the iteration, most
  // of an iteration before their cp.async gathers are issued (the gathers
  // land in the operand tiles, so they must wait for the sweep MMAs)
  int pf_l2;
  int gather_ca;        // row gathers through L1 (cp_async16_sel)
};

// ---------------------------------------------------------------------
// small PTX helpers
// ---------------------------------------------------------------------
__device__ __forceinline__ uint32_t to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}
// 3xTF32 split by truncation: hi keeps the top 10 mantissa bits (exactly a
// tf32), lo = x - hi is exact in fp32 and is passed as raw bits (the tensor
// core reads the tf32 field, truncating lo's last bits): x - (hi + lo_tf32)
// is below 2^-21 |x|.  Two instructions instead of two cvt.rna sequences.
__device__ __forceinline__ void split_tf32(float x, uint32_t& hi, uint32_t& lo) {
  hi = __float_as_uint(x) & 0xffffe000u;
  lo = __float_as_uint(x - __uint_as_float(hi));
}
__device__ __forceinline__ void mma_tf32(float* d, const uint32_t* a, const uint32_t* b) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 "
      "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
__device__ __forceinline__ void red_add_v4(float* p, float4 v) {
  asm volatile("red.relaxed.gpu.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p),
               "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ void red_add_f32(float* p, float v) {
  asm volatile("red.relaxed.gpu.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
// p <- max(p + d, 0) atomically (nonnegative mode); returns the new value
__device__ __forceinline__ float atomic_add_clamp0(float* p, float d) {
  int* ip = reinterpret_cast<int*>(p);
  int old = *ip, assumed;
  float nv;
  do {
    assumed = old;
    nv = fmaxf(__int_as_float(assumed) + d, 0.f);
    old = atomicCAS(ip, assumed, __float_as_int(nv));
  } while (old != assumed);
  return nv;
}
__device__ __forceinline__ float ld_strong(const float* p) {
  float v;
  asm volatile("ld.relaxed.gpu.global.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
  return v;
}
// 16-byte global -> shared copies that bypass L1 (the rows of the next
// iteration's entries land in the staging rows while this one finishes)
__device__ __forceinline__ void cp_async16(float* smem_dst, const float* gsrc) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gsrc) : "memory");
}
// through L1 (.ca) when `ca`: the 16-byte chunks of one gathered row then
// reach L2 as one request instead of three.  Worth -3.6% of the epoch where
// the rows miss L2 (config 5 @1e9: 185.4 -> 178.7 ms) and +8% where they hit
// (config 3), so the host sets it when the factor tables exceed L2 (naive
// kernel on config 5 @1e9: 433.2 -> 403.4 ms).
// An L1 line outlives one iteration at most here (the block gathers ~100 KB
// per iteration into an L1 of a few tens of KB beside its shared memory), the
// staleness the one-entry-ahead gathers already have.
__device__ __forceinline__ void cp_async16_sel(float* smem_dst, const float* gsrc, bool ca) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  if (ca) asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gsrc) : "memory");
  else asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async4(float* smem_dst, const float* gsrc) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
// the 128-byte line(s) of a factor row of JP floats
template <int JP>
__device__ __forceinline__ void prefetch_row_l2(const float* row) {
  prefetch_l2(row);
  if (JP * 4 > 16 && (reinterpret_cast<uintptr_t>(row) & 127u) > 128u - JP * 4u)
    prefetch_l2(row + JP - 1);
}
template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}
__device__ __forceinline__ float4 ld_strong4(const float* p) {
  float4 v;
  asm volatile("ld.relaxed.gpu.global.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ float4 ld_weak4(const float* p) {
  return *reinterpret_cast<const float4*>(p);
}
__device__ __forceinline__ void st_weak4(float* p, float4 v) {
  *reinterpret_cast<float4*>(p) = v;
}

// Row access: hot rows live in the shared replica, cold rows in global.
template <int JP>
__device__ __forceinline__ void load_row(const float* U, uint32_t i, int slot,
                                         const float* rep, float* u) {
  if (slot >= 0) {
#pragma unroll
    for (int k = 0; k < JP; k += 4) {
      const float4 q = *reinterpret_cast<const float4*>(rep + slot * JP + k);
      u[k] = q.x; u[k + 1] = q.y; u[k + 2] = q.z; u[k + 3] = q.w;
    }
  } else {
#pragma unroll
    for (int k = 0; k < JP; k += 4) {
      const float4 q = ld_weak4(U + (uint64_t)i * JP + k);
      u[k] = q.x; u[k + 1] = q.y; u[k + 2] = q.z; u[k + 3] = q.w;
    }
  }
}

// Apply a row step u <- u - eta * grad (clamped if nonneg).  Hot rows: the
// delta is added to the shared replica atomically and the curvature stat is
// accumulated; cold rows: plain store of the new value.
template <int J, int JP>
__device__ __forceinline__ void step_row(float* U, uint32_t i, int slot, float* rep,
                                         float* stat, const float* u, const float* grad,
                                         float eta, int nonneg, float curv) {
  if (slot >= 0) {
    // Hogwild on the block's replica: plain RMW of the delta (shared float
    // atomics are CAS loops on this part; lost updates are allowed, as in
    // the reference's relaxed.hpp contract).  The curvature stat is a plain
    // RMW too; the observation count is a native integer atomic.
    float* rp = rep + slot * JP;
#pragma unroll
    for (int k = 0; k < JP; k += 4) {
      float4 cur = *reinterpret_cast<float4*>(rp + k);
      float d0 = k + 0 < J ? -eta * grad[k + 0] : 0.f;
      float d1 = k + 1 < J ? -eta * grad[k + 1] : 0.f;
      float d2 = k + 2 < J ? -eta * grad[k + 2] : 0.f;
      float d3 = k + 3 < J ? -eta * grad[k + 3] : 0.f;
      cur.x += d0; cur.y += d1; cur.z += d2; cur.w += d3;
      if (nonneg) {
        cur.x = fmaxf(cur.x, 0.f); cur.y = fmaxf(cur.y, 0.f);
        cur.z = fmaxf(cur.z, 0.f); cur.w = fmaxf(cur.w, 0.f);
      }
      *reinterpret_cast<float4*>(rp + k) = cur;
    }
    stat[3 * slot] += curv;
    atomicAdd(reinterpret_cast<int*>(stat) + 3 * slot + 1, 1);
  } else if (!nonneg && CMTF_COLD_RED) {
    // cold row: add the step with vector REDs instead of storing the whole
    // row, so a concurrent update of the same row made between our read and
    // our write is not overwritten (no lost updates on cold rows)
#pragma unroll
    for (int k = 0; k < JP; k += 4)
      red_add_v4(U + (uint64_t)i * JP + k,
                 make_float4(k + 0 < J ? -eta * grad[k] : 0.f, k + 1 < J ? -eta * grad[k + 1] : 0.f,
                             k + 2 < J ? -eta * grad[k + 2] : 0.f,
                             k + 3 < J ? -eta * grad[k + 3] : 0.f));
  } else {
    float v[JP];
#pragma unroll
    for (int k = 0; k < JP; ++k) {
      float x = k < J ? u[k] - eta * grad[k] : 0.f;
      if (nonneg) x = fmaxf(x, 0.f);
      v[k] = x;
    }
#pragma unroll
    for (int k = 0; k < JP; k += 4)
      st_weak4(U + (uint64_t)i * JP + k, make_float4(v[k], v[k + 1], v[k + 2], v[k + 3]));
  }
}

#ifndef CMTF_WARP_AGG
#define CMTF_WARP_AGG 0  // measured: +5% epoch time, DSGD unstable
#endif
// Tree sum of x[0..N) over the lanes of `peers` (the lanes sharing a key);
// the lowest lane of every group ends with its group's sum.  All 32 lanes
// call it; log2(largest group) rounds of N shuffles.
template <int N>
__device__ __forceinline__ void reduce_peers(unsigned peers, float* x, int lane) {
  unsigned rel = __popc(peers & ((1u << lane) - 1u));  // my rank in the group
  unsigned above = peers & (0xfffffffeu << lane);
  while (__any_sync(0xffffffffu, above != 0u)) {
    const int next = __ffs(above);  // next remaining group member above me
    const int src = next ? next - 1 : lane;
#pragma unroll
    for (int k = 0; k < N; ++k) {
      const float t = __shfl_sync(0xffffffffu, x[k], src);
      if (next) x[k] += t;
    }
    above &= __ballot_sync(0xffffffffu, !(rel & 1u));  // odd ranks are consumed
    rel >>= 1;
  }
}

// Warp-cooperative row step (all 32 lanes call; `act`: this lane steps a
// row).  Cold rows: plain store (as step_row).  Hot rows: the lanes stepping
// the same replica row in this instruction first sum their deltas and
// curvature stats, and the group's lowest lane applies the sum, so no update
// is lost to an intra-warp write collision on the replica.  `key` is the
// replica row's shared-memory offset (unique across modes and matrices).
template <int J, int JP>
__device__ __forceinline__ void step_row_warp(float* U, uint32_t i, int slot, float* rep,
                                              float* stat, int key_base, bool act,
                                              const float* u, const float* grad, float eta,
                                              int nonneg, float curv, int lane) {
#if CMTF_WARP_AGG
  if (act && slot < 0) step_row<J, JP>(U, i, -1, rep, stat, u, grad, eta, nonneg, curv);
  const bool hot = act && slot >= 0;
  if (!__any_sync(0xffffffffu, hot)) return;
  const int key = hot ? key_base + slot * JP : -1 - lane;
  const unsigned peers = __match_any_sync(0xffffffffu, key);
  float v[J + 1];
#pragma unroll
  for (int k = 0; k < J; ++k) v[k] = grad[k];
  v[J] = curv;
  reduce_peers<J + 1>(peers, v, lane);
  if (hot && __ffs(peers) - 1 == lane) {
    // n steps taken from one point: the summed step overshoots the n
    // sequential steps it stands for once eta * sum|c|^2 is not small; scale
    // it to the sequential gain along the curvature, 1 - (1 - x/n)^n over x
    // (x = eta * sum|c|^2; exactly 1 for n = 1)
    const int n = __popc(peers);
    float sc = 1.f;
    if (n > 1) {
      const float x = eta * v[J];
      const float b = fmaxf(0.f, 1.f - x / (float)n);
      if (x > 1e-6f) sc = (1.f - __powf(b, (float)n)) / x;
    }
    const float es = -eta * sc;
    float* rp = rep + slot * JP;
#pragma unroll
    for (int k = 0; k < JP; k += 4) {
      float4 cur = *reinterpret_cast<float4*>(rp + k);
      cur.x += k + 0 < J ? es * v[k + 0] : 0.f;
      cur.y += k + 1 < J ? es * v[k + 1] : 0.f;
      cur.z += k + 2 < J ? es * v[k + 2] : 0.f;
      cur.w += k + 3 < J ? es * v[k + 3] : 0.f;
      if (nonneg) {
        cur.x = fmaxf(cur.x, 0.f); cur.y = fmaxf(cur.y, 0.f);
        cur.z = fmaxf(cur.z, 0.f); cur.w = fmaxf(cur.w, 0.f);
      }
      *reinterpret_cast<float4*>(rp + k) = cur;
    }
    stat[3 * slot] += v[J];
    atomicAdd(reinterpret_cast<int*>(stat) + 3 * slot + 1, n);
  }
#else
  (void)key_base;
  (void)lane;
  if (act) step_row<J, JP>(U, i, slot, rep, stat, u, grad, eta, nonneg, curv);
#endif
}

#ifndef CMTF_SAT_GAIN
#define CMTF_SAT_GAIN 1
#endif
// Push the block's progress on hot rows [r0, r1) to global and re-base.
// stat row layout: {sum |c|^2, observation count (int), n_hat}.  All loads
// of a row are independent and issued together; the new base is the global
// value read plus our own pushed delta (no load-after-RED round trip).
template <int J, int JP>
__device__ void flush_hot(const HotDesc& h, float* U, float* rep, float* stat, float eta,
                          float kappa, int r0, int r1, int lane) {
  float* base_b = h.base + (uint64_t)blockIdx.x * h.H * JP;
  for (int s = r0 + lane; s < r1; s += 32) {
    const uint32_t row = __ldg(h.row_of + s);
    float* g = U + (uint64_t)row * JP;
    float4 gv[JP / 4], bv[JP / 4], sv[JP / 4];
#pragma unroll
    for (int k = 0; k < JP / 4; ++k) {
      gv[k] = ld_strong4(g + 4 * k);
      bv[k] = ld_weak4(base_b + s * JP + 4 * k);
      sv[k] = *reinterpret_cast<const float4*>(rep + s * JP + 4 * k);
    }
    const float cnt = (float)atomicExch(reinterpret_cast<int*>(stat) + 3 * s + 1, 0);
    const float lam = stat[3 * s];
    stat[3 * s] = 0.f;
    float alpha = 0.f;
    if (cnt > 0.f) {
      // This block's delta is cnt sequential steps of size ~eta * lam_hat:
      // its gain along the row's curvature saturates at 1 (the block's local
      // optimum).  The merge adds the deltas of the other blocks taken from
      // the same base, n_other / cnt of them (n_other: expected updates of the
      // row GPU-wide in one window minus this block's share), so the merged
      // step is damped by 1 / (1 + q / kappa), q = (n_other / cnt) * gain:
      // alpha = 1 without concurrency, ~kappa / q under heavy contention.
      const float n_other = stat[3 * s + 2] * (1.f - 1.f / (float)gridDim.x);
      const float gain = CMTF_SAT_GAIN ? -expm1f(-eta * lam) : eta * lam;
      const float q = (n_other / cnt) * gain;
      alpha = kappa / (kappa + q);
    }
#pragma unroll
    for (int k = 0; k < JP / 4; ++k) {
      float4 dl = make_float4(alpha * (sv[k].x - bv[k].x), alpha * (sv[k].y - bv[k].y),
                              alpha * (sv[k].z - bv[k].z), alpha * (sv[k].w - bv[k].w));
      if (cnt > 0.f) red_add_v4(g + 4 * k, dl);
      const float4 nb = make_float4(gv[k].x + dl.x, gv[k].y + dl.y, gv[k].z + dl.z, gv[k].w + dl.w);
      st_weak4(base_b + s * JP + 4 * k, nb);
      // re-base, keeping local progress made since the snapshot
      float4 cur = *reinterpret_cast<float4*>(rep + s * JP + 4 * k);
      cur.x += nb.x - sv[k].x; cur.y += nb.y - sv[k].y;
      cur.z += nb.z - sv[k].z; cur.w += nb.w - sv[k].w;
      *reinterpret_cast<float4*>(rep + s * JP + 4 * k) = cur;
    }
  }
}

// Initial replica load (also sets the per-block base).
template <int JP>
__device__ void load_hot(const HotDesc& h, const float* U, float* rep, float* stat) {
  float* base_b = h.base + (uint64_t)blockIdx.x * h.H * JP;
  for (uint32_t q = threadIdx.x; q < h.H * (JP / 4); q += blockDim.x) {
    const uint32_t s = q / (JP / 4), k = (q % (JP / 4)) * 4;
    const float4 v = ld_strong4(U + (uint64_t)__ldg(h.row_of + s) * JP + k);
    *reinterpret_cast<float4*>(rep + s * JP + k) = v;
    st_weak4(base_b + s * JP + k, v);
  }
  for (uint32_t s = threadIdx.x; s < h.H; s += blockDim.x) {
    stat[3 * s] = 0.f;
    stat[3 * s + 1] = 0.f;
    stat[3 * s + 2] = (float)__ldg(h.count + __ldg(h.row_of + s)) * h.nhat_scale;
  }
}

template <int J, bool OPT, int NW, int E>
struct V2Layout {
  static constexpr int JP = round_up4(J);
  static constexpr int AB = J * J;            // core rows (a,b)
  // stage row width: >= 3*JP, multiple of 4, and == 8 or 24 mod 32 so the
  // 4 entry rows a quad touches fall in distinct bank groups
  static constexpr int sw_pick(int x) {
    return ((x % 32) == 8 || (x % 32) == 24) ? x : sw_pick(x + 4);
  }
  static constexpr int SW = sw_pick(3 * JP);
  static constexpr int NT = (AB + 7) / 8;     // ab tiles of 8 (mma N)
  static constexpr int MT = (J + 15) / 16;    // c tiles of 16 (mma M)
  static constexpr int G_FLOATS = AB * JP;    // shared core [ab][JP]
  static constexpr int DG_FLOATS = AB * JP;   // per-warp core-grad accum
  static constexpr int STAGE_FLOATS = 32 * E * SW;
  static constexpr int FIXED_FLOATS = G_FLOATS + NW * (DG_FLOATS + STAGE_FLOATS);
};

// Tensor-core core gradient of 32 staged entries (rows stg[0..32) of width
// SW holding (-r u1, u2, u3)): dGw[ab][c] += sum_e u3_e[c] (-r u1)_e[a] u2_e[b].
// SPLIT3 = 3xTF32 (hi*hi + hi*lo + lo*hi, ~fp32); otherwise the fp32 operand
// registers are passed as tf32 (the tensor core reads the top 19 bits:
// ~1e-3 relative per product on a block-summed gradient).
#ifndef CMTF_CORE_SPLIT3
#define CMTF_CORE_SPLIT3 0
#endif
template <int J, int JP, int SW, int AB, int NT, int MT>
__device__ __forceinline__ void core_grad_mma(const float* stg, float* dGw, int g8, int t4) {
  constexpr int NP = CMTF_CORE_SPLIT3 ? 3 : 1;
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    uint32_t ah[4][4], al[4][4];
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      const int e0 = ks * 8 + t4, e1 = e0 + 4;
      const int c0 = mt * 16 + g8, c1 = c0 + 8;
      const float x0 = c0 < J ? stg[e0 * SW + 2 * JP + c0] : 0.f;
      const float x1 = c1 < J ? stg[e0 * SW + 2 * JP + c1] : 0.f;
      const float x2 = c0 < J ? stg[e1 * SW + 2 * JP + c0] : 0.f;
      const float x3 = c1 < J ? stg[e1 * SW + 2 * JP + c1] : 0.f;
      if (NP == 3) {
        split_tf32(x0, ah[ks][0], al[ks][0]);
        split_tf32(x1, ah[ks][1], al[ks][1]);
        split_tf32(x2, ah[ks][2], al[ks][2]);
        split_tf32(x3, ah[ks][3], al[ks][3]);
      } else {
        ah[ks][0] = __float_as_uint(x0);
        ah[ks][1] = __float_as_uint(x1);
        ah[ks][2] = __float_as_uint(x2);
        ah[ks][3] = __float_as_uint(x3);
      }
    }
#pragma unroll 1
    for (int nt0 = 0; nt0 < NT; nt0 += 2) {
      // two n-tiles per step; with the 3xTF32 split three independent
      // accumulators each (hi*hi, hi*lo, lo*hi) so HMMA chains stay 4 deep
      float d[2][NP][4];
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int p = 0; p < NP; ++p)
#pragma unroll
          for (int q = 0; q < 4; ++q) d[j][p][q] = 0.f;
      int iaj[2], ibj[2];
      bool okj[2];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int ab = (nt0 + j) * 8 + g8;
        okj[j] = (nt0 + j) < NT && ab < AB;
        iaj[j] = ab / J;
        ibj[j] = ab - iaj[j] * J;
      }
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const float* s0 = stg + (ks * 8 + t4) * SW;
        const float* s1 = s0 + 4 * SW;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const float q0 = okj[j] ? s0[iaj[j]] * s0[JP + ibj[j]] : 0.f;
          const float q1 = okj[j] ? s1[iaj[j]] * s1[JP + ibj[j]] : 0.f;
          uint32_t bh[2], bl[2];
          if (NP == 3) {
            split_tf32(q0, bh[0], bl[0]);
            split_tf32(q1, bh[1], bl[1]);
            mma_tf32(d[j][0], ah[ks], bh);
            mma_tf32(d[j][NP > 1 ? 1 : 0], ah[ks], bl);
            mma_tf32(d[j][NP > 2 ? 2 : 0], al[ks], bh);
          } else {
            bh[0] = __float_as_uint(q0);
            bh[1] = __float_as_uint(q1);
            mma_tf32(d[j][0], ah[ks], bh);
          }
        }
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        if (nt0 + j >= NT) break;
        float dd[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          dd[q] = d[j][0][q];
#pragma unroll
          for (int p = 1; p < NP; ++p) dd[q] += d[j][p][q];
        }
        // dd: (c = mt*16+g8, ab' = nt*8+2t4 (+1)), (c+8, ...)
        const int abo = (nt0 + j) * 8 + 2 * t4;
        const int cr0 = mt * 16 + g8, cr1 = cr0 + 8;
        if (abo < AB) {
          if (cr0 < J) dGw[abo * JP + cr0] += dd[0];
          if (cr1 < J) dGw[abo * JP + cr1] += dd[2];
        }
        if (abo + 1 < AB) {
          if (cr0 < J) dGw[(abo + 1) * JP + cr0] += dd[1];
          if (cr1 < J) dGw[(abo + 1) * JP + cr1] += dd[3];
        }
      }
    }
  }
}

// virtual index over the swept matrix ranges -> physical record index
template <class Args>
__device__ __forceinline__ uint64_t mphys(const Args& a, uint64_t k) {
  for (int r = 0; r < a.n_mr; ++r) {
    if (k < a.mr_n[r]) return a.mr_lo[r] + k;
    k -= a.mr_n[r];
  }
  return 0;
}

// One coupled-matrix entry per lane (src/gradients.cpp:225-248;
// trainer.cpp:220-235); all 32 lanes call, `has` = this lane has an entry.
template <int J, int JP, class Args>
__device__ __forceinline__ void matrix_entry(const Args& a, float* sm, const uint4 mr, bool has,
                                             int lane) {
  const MatDesc3& M = a.mats[has ? mr.w : 0];
  const int mode = M.mode;
  const int su = has && a.hot[mode].slot ? __ldg(a.hot[mode].slot + mr.x) : -1;
  const int sv = has && M.hotV.slot ? __ldg(M.hotV.slot + mr.y) : -1;
  float uu[JP], vv[JP];
  float* repU = sm + a.hot[mode].off;
  float* repV = sm + M.hotV.off;
  if (has) {
    load_row<JP>(a.U[mode], mr.x, su, repU, uu);
    load_row<JP>(M.V, mr.y, sv, repV, vv);
  } else {
#pragma unroll
    for (int k = 0; k < JP; ++k) uu[k] = vv[k] = 0.f;
  }
  float yh = 0.f, nu = 0.f, nv = 0.f;
#pragma unroll
  for (int k = 0; k < J; ++k) {
    yh = fmaf(uu[k], vv[k], yh);
    nu = fmaf(uu[k], uu[k], nu);
    nv = fmaf(vv[k], vv[k], nv);
  }
  const float rr = has ? __uint_as_float(mr.z) - yh : 0.f;
  const float vr = has ? __ldg(M.vreg + mr.y) : 0.f;
  float du[J], dv[J];
#pragma unroll
  for (int k = 0; k < J; ++k) {
    du[k] = -M.weight * rr * vv[k];
    dv[k] = fmaf(-M.weight * rr, uu[k], vr * vv[k]);
  }
  step_row_warp<J, JP>(a.U[mode], mr.x, su, repU, sm + a.hot[mode].stat_off,
                       (int)a.hot[mode].off, has, uu, du, a.eta, a.nonneg, M.weight * nv, lane);
  step_row_warp<J, JP>(M.V, mr.y, sv, repV, sm + M.hotV.stat_off, (int)M.hotV.off, has, vv, dv,
                       a.eta, a.nonneg, M.weight * nu, lane);
}

// Prefetching variant (hog3tm): the next entry's record, row slots and global
// rows are in registers before it is due, so an entry costs no L2 round trip
// (matrix entries come every few iterations; a cold row read is up to that
// stale, hot rows are read from the replica at use time).
struct MatPrefetch {
  uint4 mr;       // next entry's record
  uint4 mr2;      // the one after
  int su, sv;     // hot slots of its rows
  float vr;       // its V row's regularisation coefficient
  float4 u[3], v[3];
};

// Record flags set by prepare (hog3tm): the row of the record's U / V is a
// hot (replicated) row.  Low byte of .w = matrix id.
constexpr uint32_t kMrecHotU = 1u << 30, kMrecHotV = 1u << 31, kMrecMat = 0xffu;

// Hot rows come from the replica at use time (only their slot is fetched
// ahead); cold rows are loaded from global ahead of use.  A hot row's global
// line is the most contended one in the system, so it is never read here.
template <int JP, class Args>
__device__ __forceinline__ void mat_prefetch_rows(const Args& a, MatPrefetch& p, bool valid) {
  const MatDesc3& M = a.mats[valid ? (p.mr.w & kMrecMat) : 0];
  const int mode = M.mode;
  const uint32_t i = valid ? p.mr.x : 0u, j = valid ? p.mr.y : 0u;
  const bool hu = valid && (p.mr.w & kMrecHotU), hv = valid && (p.mr.w & kMrecHotV);
  p.su = hu ? __ldg(a.hot[mode].slot + i) : -1;
  p.sv = hv ? __ldg(M.hotV.slot + j) : -1;
  p.vr = valid ? __ldg(M.vreg + j) : 0.f;
  if (valid && !hu) {
#pragma unroll
    for (int k = 0; k < JP / 4; ++k) p.u[k] = ld_weak4(a.U[mode] + (uint64_t)i * JP + 4 * k);
  }
  if (valid && !hv) {
#pragma unroll
    for (int k = 0; k < JP / 4; ++k) p.v[k] = ld_weak4(M.V + (uint64_t)j * JP + 4 * k);
  }
}

template <int JP, class Args>
__device__ __forceinline__ void mat_prefetch_init(const Args& a, MatPrefetch& p, uint64_t mlo,
                                                  uint64_t mhi) {
  p.mr = mlo < mhi ? __ldg(a.mrec + mphys(a, mlo)) : make_uint4(0, 0, 0, 0);
  p.mr2 = mlo + 1 < mhi ? __ldg(a.mrec + mphys(a, mlo + 1)) : make_uint4(0, 0, 0, 0);
  mat_prefetch_rows<JP>(a, p, mlo < mhi);
}

template <int J, int JP, class Args>
__device__ __forceinline__ void matrix_entries_until_pf(const Args& a, float* sm, uint64_t& mpos,
                                                        MatPrefetch& p, uint64_t due,
                                                        uint64_t mhi, int lane) {
  static_assert(JP <= 12, "prefetch holds rows of up to 12 floats");
  while (__any_sync(0xffffffffu, mpos < due)) {
    const bool has = mpos < due;
    const uint4 mr = p.mr;
    const MatDesc3& M = a.mats[has ? (mr.w & kMrecMat) : 0];
    const int mode = M.mode;
    const int su = has ? p.su : -1, sv = has ? p.sv : -1;
    const float vr = has ? p.vr : 0.f;
    float uu[JP], vv[JP];
    float* repU = sm + a.hot[mode].off;
    float* repV = sm + M.hotV.off;
#pragma unroll
    for (int k = 0; k < JP / 4; ++k) {
      float4 qu = p.u[k], qv = p.v[k];
      if (su >= 0) qu = *reinterpret_cast<const float4*>(repU + su * JP + 4 * k);
      if (sv >= 0) qv = *reinterpret_cast<const float4*>(repV + sv * JP + 4 * k);
      if (!has) qu = qv = make_float4(0.f, 0.f, 0.f, 0.f);
      uu[4 * k] = qu.x; uu[4 * k + 1] = qu.y; uu[4 * k + 2] = qu.z; uu[4 * k + 3] = qu.w;
      vv[4 * k] = qv.x; vv[4 * k + 1] = qv.y; vv[4 * k + 2] = qv.z; vv[4 * k + 3] = qv.w;
    }
    if (has) {  // advance: the record after next, and the next entry's rows
      if (a.mvisits) atomicAdd(a.mvisits + mphys(a, mpos), 1u);
      ++mpos;
      p.mr = p.mr2;
      if (mpos + 1 < mhi) p.mr2 = __ldg(a.mrec + mphys(a, mpos + 1));
      mat_prefetch_rows<JP>(a, p, mpos < mhi);
    }
    float yh = 0.f, nu = 0.f, nv = 0.f;
#pragma unroll
    for (int k = 0; k < J; ++k) {
      yh = fmaf(uu[k], vv[k], yh);
      nu = fmaf(uu[k], uu[k], nu);
      nv = fmaf(vv[k], vv[k], nv);
    }
    const float rr = has ? __uint_as_float(mr.z) - yh : 0.f;
    float du[J], dv[J];
#pragma unroll
    for (int k = 0; k < J; ++k) {
      du[k] = -M.weight * rr * vv[k];
      dv[k] = fmaf(-M.weight * rr, uu[k], vr * vv[k]);
    }
    step_row_warp<J, JP>(a.U[mode], mr.x, su, repU, sm + a.hot[mode].stat_off,
                         (int)a.hot[mode].off, has, uu, du, a.eta, a.nonneg, M.weight * nv, lane);
    step_row_warp<J, JP>(M.V, mr.y, sv, repV, sm + M.hotV.stat_off, (int)M.hotV.off, has, vv, dv,
                         a.eta, a.nonneg, M.weight * nu, lane);
  }
}

// Even interleaving of a lane's matrix entries with its tensor iterations on
// a WARP-uniform schedule.  The lanes' matrix counts differ by at most one;
// with per-lane schedules (count * (it + 1) / iters) the due iterations drift
// apart over the epoch and nearly every iteration runs the matrix path for a
// few lanes only (config 5: 3.5 of 32, a synchronous row fetch each time).
// All lanes follow the warp's largest count instead and step together; the
// quotient is kept incrementally (no 64-bit division per iteration).
// 32-bit counters: iters <= nnz / 256 < 2^24; a lane's matrix entries beyond
// 2^31 - 1 -- none in practice -- are swept after the loop.
struct MatSched {
  uint32_t cnt_l, cnt_w, iters, acc, rel;
  __device__ __forceinline__ void init(uint64_t mlo, uint64_t mhi, uint64_t n_iters) {
    cnt_l = (uint32_t)(mhi - mlo < 0x7fffffffull ? mhi - mlo : 0x7fffffffull);
    cnt_w = __reduce_max_sync(0xffffffffu, cnt_l);
    iters = (uint32_t)(n_iters < 0x7fffffffull ? n_iters : 0x7fffffffull);
    acc = rel = 0;
  }
  // entries of this lane due by the end of the next iteration (relative)
  __device__ __forceinline__ uint32_t step() {
    acc += cnt_w;
    while (acc >= iters) {
      acc -= iters;
      ++rel;
    }
    return rel < cnt_l ? rel : cnt_l;
  }
  // after step(): the next step that advances `rel` is exactly d iterations
  // away (fewer than one matrix entry per iteration)
  __device__ __forceinline__ bool due_in(uint32_t d) const {
    return cnt_w < iters && acc + d * cnt_w >= iters && acc + (d - 1) * cnt_w < iters;
  }
};

// Matrix entries of this lane up to `due`, in lockstep across the warp.
template <int J, int JP, class Args>
__device__ __forceinline__ void matrix_entries_until(const Args& a, float* sm, uint64_t& mpos,
                                                     uint4& mrn, uint64_t due, uint64_t mhi,
                                                     int lane) {
  while (__any_sync(0xffffffffu, mpos < due)) {
    const bool has = mpos < due;
    const uint4 mr = mrn;  // record prefetched one entry ahead
    if (has) {
      if (a.mvisits) atomicAdd(a.mvisits + mphys(a, mpos), 1u);
      ++mpos;
      if (mpos < mhi) mrn = __ldg(a.mrec + mphys(a, mpos));
    }
    matrix_entry<J, JP>(a, sm, mr, has, lane);
  }
}

template <int J, int JP, int NW, int NM = 3, class Args>
__device__ __forceinline__ void flush_all_hot(const Args& a, float* sm, int w, int lane) {
#pragma unroll
  for (int n = 0; n < NM; ++n) {
    const HotDesc& h = a.hot[n];
    if (h.H) {
      const int r0 = (int)((uint64_t)h.H * w / NW), r1 = (int)((uint64_t)h.H * (w + 1) / NW);
      flush_hot<J, JP>(h, a.U[n], sm + h.off, sm + h.stat_off, a.eta, a.kappa, r0, r1, lane);
    }
  }
  for (int m = 0; m < a.n_mat; ++m) {
    const HotDesc& h = a.mats[m].hotV;
    if (h.H) {
      const int r0 = (int)((uint64_t)h.H * w / NW), r1 = (int)((uint64_t)h.H * (w + 1) / NW);
      flush_hot<J, JP>(h, a.mats[m].V, sm + h.off, sm + h.stat_off, a.eta, a.kappa, r0, r1,
                       lane);
    }
  }
}

// E = entries per lane per iteration: every broadcast LDS of a core row feeds
// 2E FMAs and each lane carries E independent FMA chains.
template <int J, bool OPT, int NW, int E>
__global__ void __launch_bounds__(NW * 32, 1)
hog3v2_kernel(Hog3v2Args a) {
  using L = V2Layout<J, OPT, NW, E>;
  constexpr int JP = L::JP;
  constexpr int AB = L::AB;
  constexpr int SW = L::SW;
  extern __shared__ __align__(16) float sm[];
  float* Gs = sm;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* dGw = sm + L::G_FLOATS + w * (L::DG_FLOATS + L::STAGE_FLOATS);
  float* stg = dGw + L::DG_FLOATS;  // [E*32][SW]; entry j of this lane -> row j*32+lane
  const int g8 = lane >> 2, t4 = lane & 3;

  // ---- prologue: core copy, hot replicas ----
  for (int q = threadIdx.x; q < AB * JP; q += blockDim.x) {
    const int c = q % JP, ab = q / JP;
    Gs[q] = c < J ? __ldcg(a.G + ab * J + c) : 0.f;
  }
  for (int q = lane; q < L::DG_FLOATS; q += 32) dGw[q] = 0.f;
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
  const uint64_t maxchunk = (a.nnz + Wt - 1) / Wt;
  const uint64_t iters = (maxchunk + E - 1) / E;
  const uint64_t mlo = a.mnnz * gl / Wt, mhi = a.mnnz * (gl + 1) / Wt;
  uint64_t mpos = mlo;
  uint4 mrn = mlo < mhi ? __ldg(a.mrec + mphys(a, mlo)) : make_uint4(0, 0, 0, 0);
  MatSched msched;
  msched.init(mlo, mhi, iters);
  float kw = 0.f;      // entries since the warp's last core flush (lane-local)
  float lamG = 0.f;    // sum |phi|^2 since the last flush (lane-local)

  const float* rep[3];
  float* stat[3];
#pragma unroll
  for (int n = 0; n < 3; ++n) {
    rep[n] = sm + a.hot[n].off;
    stat[n] = sm + a.hot[n].stat_off;
  }

  // software pipeline: records two groups ahead; slots and regularisation
  // coefficients one group ahead; the next group's cold rows are copied
  // (cp.async) into the staging rows at the end of each iteration, so the
  // L2 gathers overlap the matrix entries, the core push and the barrier.
  uint4 rc[E], rc1[E];
  int sl[E][3];
  float rg[E][3];
  auto issue_rows = [&](const uint4* r, const int (*slx)[3], uint64_t ebase) {
#pragma unroll
    for (int j = 0; j < E; ++j) {
      if (ebase + j >= hi) continue;
      float* myst = stg + (j * 32 + lane) * SW;
      const uint32_t ix[3] = {r[j].x, r[j].y, r[j].z};
#pragma unroll
      for (int n = 0; n < 3; ++n)
        if (slx[j][n] < 0) {
          const float* src = a.U[n] + (uint64_t)ix[n] * JP;
#pragma unroll
          for (int k = 0; k < JP; k += 4) cp_async16_sel(myst + n * JP + k, src + k, a.gather_ca != 0);
        }
    }
    cp_async_commit();
  };
#pragma unroll
  for (int j = 0; j < E; ++j) {
    const uint64_t e = lo + j, e1 = lo + E + j;
    rc[j] = e < hi ? __ldg(a.rec + e) : make_uint4(0, 0, 0, 0);
    rc1[j] = e1 < hi ? __ldg(a.rec + e1) : make_uint4(0, 0, 0, 0);
  }
#pragma unroll
  for (int j = 0; j < E; ++j) {
    const uint32_t ix[3] = {rc[j].x, rc[j].y, rc[j].z};
#pragma unroll
    for (int n = 0; n < 3; ++n) {
      sl[j][n] = (lo + j < hi && a.hot[n].slot) ? __ldg(a.hot[n].slot + ix[n]) : -1;
      rg[j][n] = lo + j < hi ? __ldg(a.reg[n] + ix[n]) : 0.f;
    }
  }
  issue_rows(rc, sl, lo);
  cp_async_commit();  // (empty) core-refresh group: see the push

  for (uint64_t it = 0; it < iters; ++it) {
    const uint64_t e0 = lo + it * E;
    bool active[E];
    uint4 rc2[E];
    int nsl[E][3];
    float nrg[E][3];
#pragma unroll
    for (int j = 0; j < E; ++j) {
      active[j] = e0 + j < hi;
      const uint64_t e2 = e0 + 2 * E + j;
      rc2[j] = e2 < hi ? __ldg(a.rec + e2) : make_uint4(0, 0, 0, 0);
      const bool nxt = e0 + E + j < hi;
      const uint32_t nx[3] = {rc1[j].x, rc1[j].y, rc1[j].z};
#pragma unroll
      for (int n = 0; n < 3; ++n) {
        // no select on the loaded value (that would wait here); an invalid
        // next entry is never used (`active` gates every use)
        nsl[j][n] = a.hot[n].slot ? __ldg(a.hot[n].slot + (nxt ? nx[n] : 0u)) : -1;
        nrg[j][n] = __ldg(a.reg[n] + (nxt ? nx[n] : 0u));
      }
    }

    // ---- this group's rows: cold ones already in the staging rows (the
    // newest cp.async group, the last core refresh, may still fly) ----
    cp_async_wait_group<1>();
    float u2[E][JP], u3[E][JP], g2[E][J], g3[E][J], xh[E];
#pragma unroll
    for (int j = 0; j < E; ++j) {
      float* myst = stg + (j * 32 + lane) * SW;
      if (active[j]) {
        if (sl[j][0] >= 0) {
#pragma unroll
          for (int k = 0; k < JP; k += 4)
            *reinterpret_cast<float4*>(myst + k) =
                *reinterpret_cast<const float4*>(rep[0] + sl[j][0] * JP + k);
        }
        const float* s2 = sl[j][1] >= 0 ? rep[1] + sl[j][1] * JP : myst + JP;
        const float* s3 = sl[j][2] >= 0 ? rep[2] + sl[j][2] * JP : myst + 2 * JP;
#pragma unroll
        for (int k = 0; k < JP; k += 4) {
          const float4 q2 = *reinterpret_cast<const float4*>(s2 + k);
          const float4 q3 = *reinterpret_cast<const float4*>(s3 + k);
          u2[j][k] = q2.x; u2[j][k + 1] = q2.y; u2[j][k + 2] = q2.z; u2[j][k + 3] = q2.w;
          u3[j][k] = q3.x; u3[j][k + 1] = q3.y; u3[j][k + 2] = q3.z; u3[j][k + 3] = q3.w;
        }
      } else {
#pragma unroll
        for (int k = 0; k < JP; ++k) { u2[j][k] = 0.f; u3[j][k] = 0.f; }
#pragma unroll
        for (int k = 0; k < JP; k += 4)
          *reinterpret_cast<float4*>(myst + k) = make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int k = 0; k < J; ++k) { g2[j][k] = 0.f; g3[j][k] = 0.f; }
      xh[j] = 0.f;
    }

    // ---- contractions (FP32 CUDA cores, core rows broadcast from smem) ----
    if (OPT) {
#pragma unroll 1
      for (int ia = 0; ia < J; ++ia) {
        const float* grow = Gs + ia * J * JP;
        float ua[E], wsum[E];
#pragma unroll
        for (int j = 0; j < E; ++j) {
          ua[j] = stg[(j * 32 + lane) * SW + ia];
          wsum[j] = 0.f;
        }
#pragma unroll
        for (int ib = 0; ib < J; ++ib) {
          float gv[JP];
#pragma unroll
          for (int c = 0; c < JP; c += 4) {
            const float4 q = *reinterpret_cast<const float4*>(grow + ib * JP + c);
            gv[c] = q.x; gv[c + 1] = q.y; gv[c + 2] = q.z; gv[c + 3] = q.w;
          }
#pragma unroll
          for (int j = 0; j < E; ++j) {
            float tab = 0.f;
#pragma unroll
            for (int c = 0; c < J; ++c) tab = fmaf(gv[c], u3[j][c], tab);
            const float p = ua[j] * u2[j][ib];
#pragma unroll
            for (int c = 0; c < J; ++c) g3[j][c] = fmaf(gv[c], p, g3[j][c]);
            wsum[j] = fmaf(tab, u2[j][ib], wsum[j]);
            g2[j][ib] = fmaf(tab, ua[j], g2[j][ib]);
          }
        }
#pragma unroll
        for (int j = 0; j < E; ++j) {
          stg[(j * 32 + lane) * SW + JP + ia] = wsum[j];
          xh[j] = fmaf(wsum[j], ua[j], xh[j]);
        }
      }
    } else {
      // Algorithm 2: separate walks (predict, then each contract_all_but)
#pragma unroll 1
      for (int ia = 0; ia < J; ++ia) {
        const float* grow = Gs + ia * J * JP;
#pragma unroll
        for (int j = 0; j < E; ++j) {
          const float ua = stg[(j * 32 + lane) * SW + ia];
#pragma unroll
          for (int ib = 0; ib < J; ++ib) {
            float tab = 0.f;
#pragma unroll
            for (int c = 0; c < J; ++c) tab = fmaf(grow[ib * JP + c], u3[j][c], tab);
            xh[j] = fmaf(tab * u2[j][ib], ua, xh[j]);
          }
        }
      }
      asm volatile("" ::: "memory");
#pragma unroll 1
      for (int ia = 0; ia < J; ++ia) {
        const float* grow = Gs + ia * J * JP;
#pragma unroll
        for (int j = 0; j < E; ++j) {
          float wsum = 0.f;
#pragma unroll
          for (int ib = 0; ib < J; ++ib) {
            float tab = 0.f;
#pragma unroll
            for (int c = 0; c < J; ++c) tab = fmaf(grow[ib * JP + c], u3[j][c], tab);
            wsum = fmaf(tab, u2[j][ib], wsum);
          }
          stg[(j * 32 + lane) * SW + JP + ia] = wsum;
        }
      }
      asm volatile("" ::: "memory");
#pragma unroll 1
      for (int ia = 0; ia < J; ++ia) {
        const float* grow = Gs + ia * J * JP;
#pragma unroll
        for (int j = 0; j < E; ++j) {
          const float ua = stg[(j * 32 + lane) * SW + ia];
#pragma unroll
          for (int ib = 0; ib < J; ++ib) {
            float tab = 0.f;
#pragma unroll
            for (int c = 0; c < J; ++c) tab = fmaf(grow[ib * JP + c], u3[j][c], tab);
            g2[j][ib] = fmaf(tab, ua, g2[j][ib]);
          }
        }
      }
      asm volatile("" ::: "memory");
#pragma unroll 1
      for (int ia = 0; ia < J; ++ia) {
        const float* grow = Gs + ia * J * JP;
#pragma unroll
        for (int j = 0; j < E; ++j) {
          const float ua = stg[(j * 32 + lane) * SW + ia];
#pragma unroll
          for (int ib = 0; ib < J; ++ib) {
            const float p = ua * u2[j][ib];
#pragma unroll
            for (int c = 0; c < J; ++c) g3[j][c] = fmaf(grow[ib * JP + c], p, g3[j][c]);
          }
        }
      }
    }

    // ---- residuals, row steps, staging for the core gradient ----
#pragma unroll
    for (int j = 0; j < E; ++j) {
      float* myst = stg + (j * 32 + lane) * SW;
      float u1[JP], w1[J];
#pragma unroll
      for (int k = 0; k < JP; ++k) u1[k] = myst[k];
#pragma unroll
      for (int k = 0; k < J; ++k) w1[k] = myst[JP + k];
      const float r = active[j] ? __uint_as_float(rc[j].w) - xh[j] : 0.f;
      float n1 = 0.f, n2 = 0.f, n3 = 0.f, c1 = 0.f, c2 = 0.f, c3 = 0.f;
#pragma unroll
      for (int k = 0; k < J; ++k) {
        n1 = fmaf(u1[k], u1[k], n1); n2 = fmaf(u2[j][k], u2[j][k], n2);
        n3 = fmaf(u3[j][k], u3[j][k], n3);
        c1 = fmaf(w1[k], w1[k], c1); c2 = fmaf(g2[j][k], g2[j][k], c2);
        c3 = fmaf(g3[j][k], g3[j][k], c3);
      }
      if (active[j]) {
        lamG += n1 * n2 * n3;
        kw += 1.f;
        if (a.visits) atomicAdd(a.visits + e0 + j, 1u);
      }
      // row steps: every lane of the warp takes part (hot-row aggregation)
      float gr[J];
#pragma unroll
      for (int k = 0; k < J; ++k) gr[k] = fmaf(-r, w1[k], rg[j][0] * u1[k]);
      step_row_warp<J, JP>(a.U[0], rc[j].x, sl[j][0], const_cast<float*>(rep[0]), stat[0],
                           (int)a.hot[0].off, active[j], u1, gr, a.eta, a.nonneg, c1, lane);
#pragma unroll
      for (int k = 0; k < J; ++k) gr[k] = fmaf(-r, g2[j][k], rg[j][1] * u2[j][k]);
      step_row_warp<J, JP>(a.U[1], rc[j].y, sl[j][1], const_cast<float*>(rep[1]), stat[1],
                           (int)a.hot[1].off, active[j], u2[j], gr, a.eta, a.nonneg, c2, lane);
#pragma unroll
      for (int k = 0; k < J; ++k) gr[k] = fmaf(-r, g3[j][k], rg[j][2] * u3[j][k]);
      step_row_warp<J, JP>(a.U[2], rc[j].z, sl[j][2], const_cast<float*>(rep[2]), stat[2],
                           (int)a.hot[2].off, active[j], u3[j], gr, a.eta, a.nonneg, c3, lane);
      // stage (-r u1, u2, u3) at pre-update values (zeros for idle lanes)
#pragma unroll
      for (int k = 0; k < JP; k += 4) {
        *reinterpret_cast<float4*>(myst + k) =
            make_float4(-r * u1[k], -r * u1[k + 1], -r * u1[k + 2], -r * u1[k + 3]);
        *reinterpret_cast<float4*>(myst + JP + k) =
            make_float4(u2[j][k], u2[j][k + 1], u2[j][k + 2], u2[j][k + 3]);
        *reinterpret_cast<float4*>(myst + 2 * JP + k) =
            make_float4(u3[j][k], u3[j][k + 1], u3[j][k + 2], u3[j][k + 3]);
      }
    }
    __syncwarp();

    // ---- core gradient of the warp's 32*E entries on the tensor cores ----
#pragma unroll
    for (int j = 0; j < E; ++j)
      core_grad_mma<J, JP, SW, AB, L::NT, L::MT>(stg + j * 32 * SW, dGw, g8, t4);
    __syncwarp();  // the staging rows are free: start the next group's gathers
    issue_rows(rc1, nsl, e0 + E);

    // ---- matrix entries due by this iteration (interleaved) ----
    matrix_entries_until<J, JP>(a, sm, mpos, mrn, mlo + msched.step(), mhi, lane);

#pragma unroll
    for (int j = 0; j < E; ++j) {
      rc[j] = rc1[j];
      rc1[j] = rc2[j];
#pragma unroll
      for (int n = 0; n < 3; ++n) {
        sl[j][n] = nsl[j][n];
        rg[j][n] = nrg[j][n];
      }
    }

    // ---- periodic core push / refresh (block-level, every core_every) ----
    // The warps' private accumulators are summed inside the block so only
    // one damped push per block reaches the global core (same-address
    // atomics serialise in L2; 8x fewer of them than per-warp pushes).
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
        float* dG0 = sm + L::G_FLOATS;
        // fire-and-forget REDs; the shared copy becomes the global core as
        // of the previous push plus this delta, and the global value is
        // re-read now for the next push (no wait on an atomic's return)
#pragma unroll
        for (int k = 0; k < (AB * J + NW * 32 - 1) / (NW * 32); ++k) {
          const int e = threadIdx.x + k * NW * 32;
          if (e < AB * J) {
            const int ab = e / J, c = e - (e / J) * J;
            const int o = ab * JP + c;
            float sum = 0.f;
#pragma unroll
            for (int q = 0; q < NW; ++q) {
              float* dq = dG0 + q * (L::DG_FLOATS + L::STAGE_FLOATS) + o;
              sum += *dq;
              *dq = 0.f;
            }
            const float delta = s * fmaf(kb * a.core_reg, Gs[o], sum);
            if (a.nonneg) {
              Gs[o] = atomic_add_clamp0(a.G + e, delta);
            } else {
              // fire-and-forget RED; the shared copy is refreshed from the
              // global core asynchronously (the read follows our RED to the
              // same address; warps see the old or the new value)
              red_add_f32(a.G + e, delta);
              cp_async4(Gs + o, a.G + e);
            }
          }
        }
      }
      __syncthreads();
    }
    cp_async_commit();  // core refresh group (possibly empty)
    // ---- periodic hot-row merges: all warps in the same iteration, each a
    // 1/NW share (the core push already aligns the warps; a staggered flush
    // would make one warp late at every core-push barrier) ----
    if ((it + 1) % (uint64_t)a.flush_every == 0 || it + 1 == iters)
      flush_all_hot<J, JP, NW>(a, sm, w, lane);
  }
  // remaining matrix entries (rounding) and the final hot flush of everything
  matrix_entries_until<J, JP>(a, sm, mpos, mrn, mhi, mhi, lane);
  cp_async_wait_all();
  __syncthreads();
  flush_all_hot<J, JP, NW>(a, sm, w, lane);
}

}  // namespace cmtfb
