// hog3.cuh -- specialised order-3 S^3CMTF Hogwild sweep and eval pass.
//
// One thread = one SGD worker walking a contiguous chunk of the COO sorted
// by the "cached" mode CM (the row of mode CM stays on chip while its index
// repeats and is written back when it changes).  All threads of a block
// advance in lock step, one entry per iteration, so the block can reduce
// the core gradient of its BT entries in shared memory once per iteration.
//
// Per entry (indices a,b,c of modes 1,2,3; core G row-major, c fastest):
//   OPT (Algorithm 3, reuse of intermediates):
//     one walk over G, each G[a,b,c] (a shared-memory broadcast) feeds two
//     FMAs: t_ab += G*u3[c]  and  g3[c] += G*(u1[a]u2[b]); then
//     W1[a] += t_ab*u2[b], g2[b] += t_ab*u1[a].  x_hat = sum_a W1[a]u1[a].
//     Row gradients -r*{W1,g2,g3} + (lambda/count)*u  (src/gradients.cpp:73-79)
//   NAIVE (Algorithm 2): separate walks for x_hat and for
//     each mode's leave-one-out contraction (src/gradients.cpp:83-128).
//   Core gradient (both): dG[a,b,c] = sum_e -r_e u1[a]u2[b]u3[c]: the
//     entries' (-r u1, u2, u3) are staged in shared memory and re-read by
//     "tile" threads that own a (a,b) pair and J3 accumulators; the block's
//     sum is applied to the global core with one atomic per element
//     (+ k * lambda/|Omega| * G, k = entries this iteration), and the
//     atomic's return value refreshes the block's shared core.
#pragma once

#include "common.cuh"

namespace cmtfb {

struct Hog3Args {
  const uint4* rec;  // sorted records {i1, i2, i3, float_bits(x)}
  uint64_t nnz;
  float* U[3];
  const float* reg[3];
  float* G;          // global core, J1*J2*J3, row-major
  float eta;
  float eta_core;
  float core_reg;    // lambda / nnz_total
  int nonneg;
  uint32_t* visits;  // debug_count_visits (null: off)
};

template <int J1, int J2, int J3>
struct Hog3Layout {
  static constexpr int J1P = round_up4(J1), J2P = round_up4(J2),
                       J3P = round_up4(J3);
  static constexpr int TILES = J1 * J2;
  static constexpr int SW = J1P + J2P + J3P;  // stage row width (floats)
  template <int BT>
  struct B {
    static constexpr int NG = TILES >= BT ? 1 : BT / TILES;  // entry groups
    static constexpr int G_FLOATS = J1 * J2 * J3P;
    static constexpr int PART_FLOATS = round_up4((NG - 1) * TILES * J3);
    static constexpr int U1_FLOATS = J1P * BT;   // per-thread mode-1 row
    static constexpr int W1_FLOATS = J1 * BT;    // per-thread W1
    static constexpr int STAGE_FLOATS = SW * BT;
    static constexpr size_t bytes() {
      return sizeof(float) *
             (size_t)(G_FLOATS + PART_FLOATS + U1_FLOATS + W1_FLOATS +
                      STAGE_FLOATS);
    }
  };
};

template <int N>
__device__ __forceinline__ void load_row_regs(const float* p, float* r) {
#pragma unroll
  for (int k = 0; k < N; k += 4) {
    const float4 q = ld_row4(p + k);
    r[k] = q.x; r[k + 1] = q.y; r[k + 2] = q.z; r[k + 3] = q.w;
  }
}
template <int N>
__device__ __forceinline__ void store_row_regs(float* p, const float* r) {
#pragma unroll
  for (int k = 0; k < N; k += 4)
    st_row4(p + k, make_float4(r[k], r[k + 1], r[k + 2], r[k + 3]));
}

template <int J1, int J2, int J3, bool OPT, int CM, int BT>
__global__ void __launch_bounds__(BT)
hog3_kernel(Hog3Args a) {
  using L = Hog3Layout<J1, J2, J3>;
  using LB = typename L::template B<BT>;
  constexpr int J1P = L::J1P, J2P = L::J2P, J3P = L::J3P;
  extern __shared__ __align__(16) float sm[];
  float* Gs = sm;                               // [J1*J2][J3P]
  float* part = Gs + LB::G_FLOATS;              // [(NG-1)][TILES][J3]
  float* u1s = part + LB::PART_FLOATS;          // [J1P][BT]
  float* w1s = u1s + LB::U1_FLOATS;             // [J1][BT]
  float* stage = w1s + LB::W1_FLOATS;           // [BT][SW]

  const int t = threadIdx.x;
  const uint64_t W = (uint64_t)gridDim.x * BT;
  const uint64_t gt = (uint64_t)blockIdx.x * BT + t;
  const uint64_t lo = a.nnz * gt / W, hi = a.nnz * (gt + 1) / W;
  const uint64_t iters = (a.nnz + W - 1) / W;

  for (int q = t; q < J1 * J2 * J3P; q += BT) {
    const int c = q % J3P, ab = q / J3P;
    Gs[q] = c < J3 ? a.G[ab * J3 + c] : 0.f;
  }

  float* U1 = a.U[0];
  float* U2 = a.U[1];
  float* U3 = a.U[2];
  uint32_t cur = 0xffffffffu;  // cached-mode row index held on chip
  float creg = 0.f;            // its lambda/count
  float u2[J2P], u3[J3P];
#pragma unroll
  for (int k = 0; k < J2P; ++k) u2[k] = 0.f;
#pragma unroll
  for (int k = 0; k < J3P; ++k) u3[k] = 0.f;

  uint4 nrec = make_uint4(0, 0, 0, 0);
  if (lo < hi) nrec = __ldg(a.rec + lo);
  __syncthreads();

  for (uint64_t it = 0; it < iters; ++it) {
    const uint64_t e = lo + it;
    const bool active = e < hi;
    if (active && a.visits) atomicAdd(a.visits + e, 1u);
    const uint4 rc = nrec;
    if (e + 1 < hi) nrec = __ldg(a.rec + e + 1);
    float r = 0.f;
    if (active) {
      const uint32_t i1 = rc.x, i2 = rc.y, i3 = rc.z;
      const uint32_t ic = CM == 0 ? i1 : (CM == 1 ? i2 : i3);
      // ---- gather rows (cached mode only on change) ----
      if (ic != cur) {
        if (cur != 0xffffffffu) {  // write back the cached row
          if (CM == 0) {
#pragma unroll
            for (int k = 0; k < J1P; k += 4)
              st_row4(U1 + (uint64_t)cur * J1P + k,
                      make_float4(u1s[k * BT + t], u1s[(k + 1) * BT + t],
                                  u1s[(k + 2) * BT + t], u1s[(k + 3) * BT + t]));
          } else if (CM == 1) {
            store_row_regs<J2P>(U2 + (uint64_t)cur * J2P, u2);
          } else {
            store_row_regs<J3P>(U3 + (uint64_t)cur * J3P, u3);
          }
        }
        cur = ic;
        creg = __ldg(a.reg[CM] + ic);
        if (CM == 1) load_row_regs<J2P>(U2 + (uint64_t)i2 * J2P, u2);
        if (CM == 2) load_row_regs<J3P>(U3 + (uint64_t)i3 * J3P, u3);
        if (CM == 0) {
#pragma unroll
          for (int k = 0; k < J1P; k += 4) {
            const float4 q = ld_row4(U1 + (uint64_t)i1 * J1P + k);
            u1s[k * BT + t] = q.x; u1s[(k + 1) * BT + t] = q.y;
            u1s[(k + 2) * BT + t] = q.z; u1s[(k + 3) * BT + t] = q.w;
          }
        }
      }
      if (CM != 0) {
#pragma unroll
        for (int k = 0; k < J1P; k += 4) {
          const float4 q = ld_row4(U1 + (uint64_t)i1 * J1P + k);
          u1s[k * BT + t] = q.x; u1s[(k + 1) * BT + t] = q.y;
          u1s[(k + 2) * BT + t] = q.z; u1s[(k + 3) * BT + t] = q.w;
        }
      }
      if (CM != 1) load_row_regs<J2P>(U2 + (uint64_t)i2 * J2P, u2);
      if (CM != 2) load_row_regs<J3P>(U3 + (uint64_t)i3 * J3P, u3);
      const float reg1 = CM == 0 ? creg : __ldg(a.reg[0] + i1);
      const float reg2 = CM == 1 ? creg : __ldg(a.reg[1] + i2);
      const float reg3 = CM == 2 ? creg : __ldg(a.reg[2] + i3);

      // ---- contractions ----
      float g2[J2], g3[J3];
#pragma unroll
      for (int k = 0; k < J2; ++k) g2[k] = 0.f;
#pragma unroll
      for (int k = 0; k < J3; ++k) g3[k] = 0.f;
      float xh = 0.f;
      if (OPT) {
#pragma unroll 1
        for (int ia = 0; ia < J1; ++ia) {
          const float ua = u1s[ia * BT + t];
          const float* grow = Gs + ia * J2 * J3P;
          float w = 0.f;
#pragma unroll
          for (int ib = 0; ib < J2; ++ib) {
            float gv[J3P];
#pragma unroll
            for (int c = 0; c < J3P; c += 4) {
              const float4 q = *reinterpret_cast<const float4*>(grow + ib * J3P + c);
              gv[c] = q.x; gv[c + 1] = q.y; gv[c + 2] = q.z; gv[c + 3] = q.w;
            }
            float t0 = 0.f, t1 = 0.f;
#pragma unroll
            for (int c = 0; c < J3; ++c) {
              if (c & 1) t1 = fmaf(gv[c], u3[c], t1);
              else t0 = fmaf(gv[c], u3[c], t0);
            }
            const float p = ua * u2[ib];
#pragma unroll
            for (int c = 0; c < J3; ++c) g3[c] = fmaf(gv[c], p, g3[c]);
            const float tab = t0 + t1;
            w = fmaf(tab, u2[ib], w);
            g2[ib] = fmaf(tab, ua, g2[ib]);
          }
          w1s[ia * BT + t] = w;
          xh = fmaf(w, ua, xh);
        }
      } else {
        // Algorithm 2: x_hat walk (predict_entry)
#pragma unroll 1
        for (int ia = 0; ia < J1; ++ia) {
          const float ua = u1s[ia * BT + t];
          const float* grow = Gs + ia * J2 * J3P;
#pragma unroll
          for (int ib = 0; ib < J2; ++ib) {
            float tab = 0.f;
#pragma unroll
            for (int c = 0; c < J3; ++c) tab = fmaf(grow[ib * J3P + c], u3[c], tab);
            xh = fmaf(tab * u2[ib], ua, xh);
          }
        }
        asm volatile("" ::: "memory");
        // contract_all_but, mode 1
#pragma unroll 1
        for (int ia = 0; ia < J1; ++ia) {
          const float* grow = Gs + ia * J2 * J3P;
          float w = 0.f;
#pragma unroll
          for (int ib = 0; ib < J2; ++ib) {
            float tab = 0.f;
#pragma unroll
            for (int c = 0; c < J3; ++c) tab = fmaf(grow[ib * J3P + c], u3[c], tab);
            w = fmaf(tab, u2[ib], w);
          }
          w1s[ia * BT + t] = w;
        }
        asm volatile("" ::: "memory");
        // contract_all_but, mode 2
#pragma unroll 1
        for (int ia = 0; ia < J1; ++ia) {
          const float ua = u1s[ia * BT + t];
          const float* grow = Gs + ia * J2 * J3P;
#pragma unroll
          for (int ib = 0; ib < J2; ++ib) {
            float tab = 0.f;
#pragma unroll
            for (int c = 0; c < J3; ++c) tab = fmaf(grow[ib * J3P + c], u3[c], tab);
            g2[ib] = fmaf(tab, ua, g2[ib]);
          }
        }
        asm volatile("" ::: "memory");
        // contract_all_but, mode 3
#pragma unroll 1
        for (int ia = 0; ia < J1; ++ia) {
          const float ua = u1s[ia * BT + t];
          const float* grow = Gs + ia * J2 * J3P;
#pragma unroll
          for (int ib = 0; ib < J2; ++ib) {
            const float p = ua * u2[ib];
#pragma unroll
            for (int c = 0; c < J3; ++c) g3[c] = fmaf(grow[ib * J3P + c], p, g3[c]);
          }
        }
      }
      r = __uint_as_float(rc.w) - xh;

      // ---- stage (-r u1, u2, u3) at pre-update values for the core ----
      float* st = stage + t * L::SW;
#pragma unroll
      for (int k = 0; k < J1P; k += 4)
        *reinterpret_cast<float4*>(st + k) =
            make_float4(-r * u1s[k * BT + t], -r * u1s[(k + 1) * BT + t],
                        -r * u1s[(k + 2) * BT + t], -r * u1s[(k + 3) * BT + t]);
#pragma unroll
      for (int k = 0; k < J2P; k += 4)
        *reinterpret_cast<float4*>(st + J1P + k) =
            make_float4(u2[k], u2[k + 1], u2[k + 2], u2[k + 3]);
#pragma unroll
      for (int k = 0; k < J3P; k += 4)
        *reinterpret_cast<float4*>(st + J1P + J2P + k) =
            make_float4(u3[k], u3[k + 1], u3[k + 2], u3[k + 3]);

      // ---- row steps: u <- u - eta * (-r*c + reg*u)  (clamped if nonneg)
#pragma unroll 1
      for (int ia = 0; ia < J1; ++ia) {
        const float ua = u1s[ia * BT + t];
        float v = ua - a.eta * fmaf(-r, w1s[ia * BT + t], reg1 * ua);
        if (a.nonneg) v = fmaxf(v, 0.f);
        u1s[ia * BT + t] = v;
      }
#pragma unroll
      for (int k = 0; k < J2; ++k) {
        float v = u2[k] - a.eta * fmaf(-r, g2[k], reg2 * u2[k]);
        if (a.nonneg) v = fmaxf(v, 0.f);
        u2[k] = v;
      }
#pragma unroll
      for (int k = 0; k < J3; ++k) {
        float v = u3[k] - a.eta * fmaf(-r, g3[k], reg3 * u3[k]);
        if (a.nonneg) v = fmaxf(v, 0.f);
        u3[k] = v;
      }
      if (CM != 0) {
#pragma unroll
        for (int k = 0; k < J1P; k += 4)
          st_row4(U1 + (uint64_t)i1 * J1P + k,
                  make_float4(u1s[k * BT + t], u1s[(k + 1) * BT + t],
                              u1s[(k + 2) * BT + t], u1s[(k + 3) * BT + t]));
      }
      if (CM != 1) store_row_regs<J2P>(U2 + (uint64_t)i2 * J2P, u2);
      if (CM != 2) store_row_regs<J3P>(U3 + (uint64_t)i3 * J3P, u3);
    } else {
      float* st = stage + t * L::SW;
#pragma unroll
      for (int k = 0; k < L::SW; k += 4)
        *reinterpret_cast<float4*>(st + k) = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    const int kact = __syncthreads_count(active);

    // ---- block-local core-gradient reduction over the staged entries ----
    constexpr int NG = LB::NG;
    const int grp = t / L::TILES;
    float acc[J3];
    for (int tile = (NG == 1 ? t : t % L::TILES); tile < L::TILES && grp < NG;
         tile += BT) {
      const int ia = tile / J2, ib = tile % J2;
#pragma unroll
      for (int c = 0; c < J3; ++c) acc[c] = 0.f;
      const int e0 = NG == 1 ? 0 : grp * BT / NG;
      const int e1 = NG == 1 ? BT : (grp + 1) * BT / NG;
      for (int s = e0; s < e1; ++s) {
        const float* sr = stage + s * L::SW;
        const float p = sr[ia] * sr[J1P + ib];
#pragma unroll
        for (int c = 0; c < J3P; c += 4) {
          const float4 q = *reinterpret_cast<const float4*>(sr + J1P + J2P + c);
          if (c + 0 < J3) acc[c + 0] = fmaf(p, q.x, acc[c + 0]);
          if (c + 1 < J3) acc[c + 1] = fmaf(p, q.y, acc[c + 1]);
          if (c + 2 < J3) acc[c + 2] = fmaf(p, q.z, acc[c + 2]);
          if (c + 3 < J3) acc[c + 3] = fmaf(p, q.w, acc[c + 3]);
        }
      }
      if (NG > 1) {
        if (grp > 0) {
#pragma unroll
          for (int c = 0; c < J3; ++c)
            part[((grp - 1) * L::TILES + tile) * J3 + c] = acc[c];
        }
      } else {
        // NG == 1: apply directly
#pragma unroll
        for (int c = 0; c < J3; ++c) {
          const float gv = Gs[tile * J3P + c];
          const float delta = -a.eta_core * fmaf((float)kact * a.core_reg, gv, acc[c]);
          float nv = atomicAdd(a.G + tile * J3 + c, delta) + delta;
          if (a.nonneg) nv = fmaxf(nv, 0.f);
          Gs[tile * J3P + c] = nv;
        }
      }
    }
    if (NG > 1) {
      __syncthreads();
      if (grp == 0) {
        const int tile = t;
#pragma unroll
        for (int c = 0; c < J3; ++c) {
          float s = acc[c];
          for (int g = 1; g < NG; ++g) s += part[((g - 1) * L::TILES + tile) * J3 + c];
          const float gv = Gs[tile * J3P + c];
          const float delta = -a.eta_core * fmaf((float)kact * a.core_reg, gv, s);
          float nv = atomicAdd(a.G + tile * J3 + c, delta) + delta;
          if (a.nonneg) nv = fmaxf(nv, 0.f);
          Gs[tile * J3P + c] = nv;
        }
      }
    }
    __syncthreads();
  }
  // final write-back of the cached row
  if (cur != 0xffffffffu) {
    if (CM == 0) {
#pragma unroll
      for (int k = 0; k < J1P; k += 4)
        st_row4(U1 + (uint64_t)cur * J1P + k,
                make_float4(u1s[k * BT + t], u1s[(k + 1) * BT + t],
                            u1s[(k + 2) * BT + t], u1s[(k + 3) * BT + t]));
    } else if (CM == 1) {
      store_row_regs<J2P>(U2 + (uint64_t)cur * J2P, u2);
    } else {
      store_row_regs<J3P>(U3 + (uint64_t)cur * J3P, u3);
    }
  }
}

// Eval pass for order 3: thread per entry, fixed 1024-entry blocks
// (src/eval.cpp:10-65), double accumulation, deterministic order.
template <int J1, int J2, int J3>
__global__ void __launch_bounds__(256, 2)
eval3_kernel(const uint4* rec, uint64_t nnz, const float* U1, const float* U2,
             const float* U3, const float* G, double* partial) {
  constexpr int J1P = round_up4(J1), J2P = round_up4(J2), J3P = round_up4(J3);
  constexpr int BT = 256;
  extern __shared__ __align__(16) float sm[];
  float* Gs = sm;
  float* u1s = Gs + J1 * J2 * J3P;
  __shared__ double acc_s[BT / 32];
  const int t = threadIdx.x;
  for (int q = t; q < J1 * J2 * J3P; q += BT) {
    const int c = q % J3P, ab = q / J3P;
    Gs[q] = c < J3 ? G[ab * J3 + c] : 0.f;
  }
  __syncthreads();
  const uint64_t lo = (uint64_t)blockIdx.x * kEvalBlock;
  const uint64_t hi = lo + kEvalBlock < nnz ? lo + kEvalBlock : nnz;
  // the block's 1024 entries, 4 per thread at once: every core row read from
  // shared memory (one broadcast LDS.128 per 4 values) feeds 4 entries
  constexpr int EV = kEvalBlock / BT;
  static_assert(EV == 4, "eval: 4 entries per thread");
  uint4 rc[EV];
  float u2[EV][J2P], u3[EV][J3P], xh[EV];
#pragma unroll
  for (int q = 0; q < EV; ++q) {
    const uint64_t e = lo + t + (uint64_t)q * BT;
    rc[q] = e < hi ? __ldg(rec + e) : make_uint4(0, 0, 0, 0);
    xh[q] = 0.f;
  }
#pragma unroll
  for (int q = 0; q < EV; ++q) {
    load_row_regs<J2P>(U2 + (uint64_t)rc[q].y * J2P, u2[q]);
    load_row_regs<J3P>(U3 + (uint64_t)rc[q].z * J3P, u3[q]);
#pragma unroll
    for (int k = 0; k < J1P; k += 4) {
      const float4 v = ld_row4(U1 + (uint64_t)rc[q].x * J1P + k);
      u1s[((q * J1P) + k) * BT + t] = v.x; u1s[((q * J1P) + k + 1) * BT + t] = v.y;
      u1s[((q * J1P) + k + 2) * BT + t] = v.z; u1s[((q * J1P) + k + 3) * BT + t] = v.w;
    }
  }
#pragma unroll 1
  for (int ia = 0; ia < J1; ++ia) {
    const float* grow = Gs + ia * J2 * J3P;
    float w[EV];
#pragma unroll
    for (int q = 0; q < EV; ++q) w[q] = 0.f;
#pragma unroll
    for (int ib = 0; ib < J2; ++ib) {
      float gv[J3P];
#pragma unroll
      for (int c = 0; c < J3P; c += 4) {
        const float4 g4 = *reinterpret_cast<const float4*>(grow + ib * J3P + c);
        gv[c] = g4.x; gv[c + 1] = g4.y; gv[c + 2] = g4.z; gv[c + 3] = g4.w;
      }
#pragma unroll
      for (int q = 0; q < EV; ++q) {
        float t0 = 0.f, t1 = 0.f;
#pragma unroll
        for (int c = 0; c < J3; ++c) {
          if (c & 1) t1 = fmaf(gv[c], u3[q][c], t1);
          else t0 = fmaf(gv[c], u3[q][c], t0);
        }
        w[q] = fmaf(t0 + t1, u2[q][ib], w[q]);
      }
    }
#pragma unroll
    for (int q = 0; q < EV; ++q) xh[q] = fmaf(w[q], u1s[(q * J1P + ia) * BT + t], xh[q]);
  }
  double acc = 0.0;
#pragma unroll
  for (int q = 0; q < EV; ++q) {
    if (lo + t + (uint64_t)q * BT < hi) {
      const double r = (double)__uint_as_float(rc[q].w) - (double)xh[q];
      acc += r * r;
    }
  }
  acc = warp_sum_d(acc);
  if ((t & 31) == 0) acc_s[t >> 5] = acc;
  __syncthreads();
  if (t == 0) {
    double s = 0.0;
    for (int i = 0; i < BT / 32; ++i) s += acc_s[i];
    partial[blockIdx.x] = s;
  }
}

}  // namespace cmtfb
