// generic.cuh -- order-generic S^3CMTF device kernels (any N <= kMaxOrder,
// any ranks <= kMaxRank, prod(J) <= kMaxCore).  They serve the per-entry
// probe, the serial-parity epoch, the generic Hogwild sweep, the matrix
// sweep, the evaluation pass for shapes without a specialised kernel, and
// the non-finite scan.
//
// Entry math ("team" = a warp or a block cooperating on ONE tensor entry):
//   opt   (Algorithm 3, src/gradients.cpp:130-223): one walk over the core
//         computes the full product G_d * prod_n u_n[j_n] (x_hat) and, by
//         prefix/suffix products, every leave-one-out term of every mode --
//         the intermediate tensor is reused without the division by u_n the
//         reference uses (no divisor fallback is needed).
//   naive (Algorithm 2, src/gradients.cpp:83-128): one walk for x_hat
//         (predict_entry, src/tucker.cpp:96-127), then one walk per mode
//         (contract_all_but, src/tucker.cpp:129-165), then the core walk.
#pragma once

#include "common.cuh"

namespace cmtfb {

constexpr int kMaxCore = 8192;

struct CoreShape {
  int order;
  uint32_t J[kMaxOrder];
  uint32_t off[kMaxOrder + 1];  // offsets of each mode's row in a concat
  uint32_t size;                // prod J
  // CP / hyper-diagonal core (CoreStructure::HyperDiagonalCp, equal ranks):
  // stored densely with zero off-diagonal elements -- every contraction is
  // then exactly the CP one -- and only the superdiagonal (d % dstep == 0,
  // dstep = 1 + J + ... + J^(N-1)) is ever updated
  int cp;
  uint32_t dstep;
};

// Core element d takes steps (every element; CP: the superdiagonal only).
__device__ __forceinline__ bool core_active(const CoreShape& cs, uint32_t d) {
  return !cs.cp || d % cs.dstep == 0;
}

// Decode a linear core index (last mode fastest) into digits.
__device__ __forceinline__ void decode(const CoreShape& cs, uint32_t d,
                                       uint32_t* j) {
  for (int n = cs.order - 1; n >= 0; --n) {
    j[n] = d % cs.J[n];
    d /= cs.J[n];
  }
}

// Team computation of x_hat and the unregularised row contractions
// c_n[k] = (G x_{-n} {u})[k] into cont (smem, zeroed by the caller, concat
// layout cs.off).  u: smem rows (concat layout).  Returns the team-partial
// x_hat of this thread (caller reduces).
template <bool OPT>
__device__ float team_contract(const CoreShape& cs, const float* G,
                               const float* u, float* cont, int t, int T) {
  float xh = 0.f;
  uint32_t j[kMaxOrder];
  if (OPT) {
    for (uint32_t d = t; d < cs.size; d += T) {
      decode(cs, d, j);
      float pre[kMaxOrder + 1];
      pre[0] = G[d];
      for (int n = 0; n < cs.order; ++n) pre[n + 1] = pre[n] * u[cs.off[n] + j[n]];
      xh += pre[cs.order];
      float suf = 1.f;
      for (int n = cs.order - 1; n >= 0; --n) {
        atomicAdd(&cont[cs.off[n] + j[n]], pre[n] * suf);
        suf *= u[cs.off[n] + j[n]];
      }
    }
  } else {
    for (uint32_t d = t; d < cs.size; d += T) {  // predict_entry walk
      decode(cs, d, j);
      float p = G[d];
      for (int n = 0; n < cs.order; ++n) p *= u[cs.off[n] + j[n]];
      xh += p;
    }
    for (int s = 0; s < cs.order; ++s)  // one contract_all_but walk per mode
      for (uint32_t d = t; d < cs.size; d += T) {
        decode(cs, d, j);
        float p = G[d];
        for (int n = 0; n < cs.order; ++n)
          if (n != s) p *= u[cs.off[n] + j[n]];
        atomicAdd(&cont[cs.off[s] + j[s]], p);
      }
  }
  return xh;
}

__device__ __forceinline__ float block_sum(float v, float* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float s = 0.f;
  const int nw = (blockDim.x + 31) >> 5;
  for (int i = 0; i < nw; ++i) s += red[i];
  return s;
}

// ---------------------------------------------------------------------
// Per-entry probe: compute_gradient(_opt) at a frozen model, one warp per
// entry.  Rows come either from the factor tables (training ids mapped to
// sorted positions through pos[]) or from an explicit dense row block.
// ---------------------------------------------------------------------
struct ProbeArgs {
  CoreShape cs;
  const float* G;
  // source A: training entries
  const uint32_t* rec;  // sorted records, (order+1) words each
  const uint32_t* pos;  // training id -> sorted position
  const uint64_t* ids;
  ModeTables mt;
  // source B: explicit rows (stateless compute_gradient)
  const float* rows;    // n x sumJ
  const float* x;
  const uint32_t* counts;  // n x order
  float lambda;
  uint64_t n;
  float core_reg;  // lambda / nnz_total
  int with_core;
  // outputs (device, f32)
  float* xhat;
  float* resid;
  float* grow;   // n x sumJ
  float* gcore;  // n x size
};

template <bool OPT>
__global__ void probe_kernel(ProbeArgs a) {
  extern __shared__ float sm[];
  const int warps = blockDim.x >> 5;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const CoreShape& cs = a.cs;
  const uint32_t sumJ = cs.off[cs.order];
  float* u = sm + w * 2 * sumJ;
  float* cont = u + sumJ;
  __shared__ float reg_s[32][kMaxOrder];
  __shared__ float x_s[32];
  for (uint64_t e = (uint64_t)blockIdx.x * warps + w; e < a.n;
       e += (uint64_t)gridDim.x * warps) {
    if (a.rows) {
      for (uint32_t k = l; k < sumJ; k += 32) u[k] = a.rows[e * sumJ + k];
      if (l < cs.order) reg_s[w][l] = a.lambda / (float)a.counts[e * cs.order + l];
      if (l == 0) x_s[w] = a.x[e];
    } else {
      const uint32_t p = a.pos[a.ids[e]];
      const uint32_t* r = a.rec + (uint64_t)p * (cs.order + 1);
      for (int n = 0; n < cs.order; ++n) {
        const uint32_t i = r[n];
        for (uint32_t k = l; k < cs.J[n]; k += 32)
          u[cs.off[n] + k] = a.mt.U[n][(uint64_t)i * a.mt.JP[n] + k];
        if (l == 0) reg_s[w][n] = a.mt.reg[n][i];
      }
      if (l == 0) x_s[w] = __uint_as_float(r[cs.order]);
    }
    for (uint32_t k = l; k < sumJ; k += 32) cont[k] = 0.f;
    __syncwarp();
    float xh = warp_sum(team_contract<OPT>(cs, a.G, u, cont, l, 32));
    __syncwarp();
    const float r = x_s[w] - xh;
    if (l == 0) {
      if (a.xhat) a.xhat[e] = xh;
      if (a.resid) a.resid[e] = r;
    }
    for (int n = 0; n < cs.order; ++n)
      for (uint32_t k = l; k < cs.J[n]; k += 32) {
        const uint32_t q = cs.off[n] + k;
        a.grow[e * sumJ + q] = fmaf(-r, cont[q], reg_s[w][n] * u[q]);
      }
    if (a.with_core && a.gcore) {
      uint32_t j[kMaxOrder];
      for (uint32_t d = l; d < cs.size; d += 32) {
        decode(cs, d, j);
        float p = 1.f;
        for (int n = 0; n < cs.order; ++n) p *= u[cs.off[n] + j[n]];
        a.gcore[e * cs.size + d] = fmaf(-r, p, a.core_reg * a.G[d]);
      }
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------
// Matrix entry gradients (src/gradients.cpp:225-248), batched probe.
// ---------------------------------------------------------------------
__global__ void matrix_probe_kernel(uint64_t n, uint32_t J, const float* y,
                                    const float* u, const float* v,
                                    float lambda_m, float lambda,
                                    const uint32_t* col_count, float* du,
                                    float* dv, float* resid) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const float* ur = u + e * J;
    const float* vr = v + e * J;
    float yh = 0.f;
    for (uint32_t k = 0; k < J; ++k) yh = fmaf(ur[k], vr[k], yh);
    const float r = y[e] - yh;
    const float reg = lambda_m * lambda / (float)col_count[e];
    for (uint32_t k = 0; k < J; ++k) {
      du[e * J + k] = -lambda_m * r * vr[k];
      dv[e * J + k] = fmaf(-lambda_m * r, ur[k], reg * vr[k]);
    }
    resid[e] = r;
  }
}

// ---------------------------------------------------------------------
// Serial-parity epoch: ONE block replays the reference schedule in order
// with P=1 semantics (src/trainer.cpp:166-237 with workers=1): per tensor
// entry all gradients from pre-update values, rows stepped mode by mode,
// then the core with step eta; per matrix entry both gradients first, then
// the interleaved u/v steps (src/trainer.cpp:220-235).
// ---------------------------------------------------------------------
struct MatDev {
  int mode;
  uint32_t rows, cols;
  uint64_t nnz;
  const uint32_t* rec;   // sorted by row: (row, col, val bits)
  const uint32_t* pos;   // matrix entry id -> sorted position
  float* V;              // cols x JP
  const float* vreg;     // lambda_m * lambda / count_col (0 if count 0)
  const uint32_t* count;
  float weight;
};

constexpr int kMaxMats = 8;

struct SerialArgs {
  CoreShape cs;
  float* G;              // global core, updated at the end
  const uint32_t* rec;   // tensor records (sorted)
  const uint32_t* pos;   // training id -> sorted position
  ModeTables mt;
  uint64_t nnz;
  int n_mat;
  MatDev mats[kMaxMats];
  uint64_t mat_base[kMaxMats + 1];  // schedule id offsets, [0] = nnz
  const uint64_t* sched;
  uint64_t n_sched;
  float eta;
  float eta_core;  // eta * workers (designated-worker rule); P=1 -> eta
  float core_reg;
  int nonneg;
};

template <bool OPT>
__global__ void serial_epoch_kernel(SerialArgs a) {
  extern __shared__ float sm[];
  const CoreShape& cs = a.cs;
  const uint32_t sumJ = cs.off[cs.order];
  float* Gs = sm;                  // cs.size
  float* u = Gs + cs.size;         // sumJ
  float* cont = u + sumJ;          // sumJ
  float* red = cont + sumJ;        // 32
  __shared__ uint32_t idx_s[kMaxOrder];
  __shared__ float x_s;
  const int t = threadIdx.x, T = blockDim.x;
  for (uint32_t d = t; d < cs.size; d += T) Gs[d] = a.G[d];
  __syncthreads();
  for (uint64_t s = 0; s < a.n_sched; ++s) {
    const uint64_t id = a.sched[s];
    if (id < a.nnz) {
      if (t == 0) {
        const uint32_t* r = a.rec + (uint64_t)a.pos[id] * (cs.order + 1);
        for (int n = 0; n < cs.order; ++n) idx_s[n] = r[n];
        x_s = __uint_as_float(r[cs.order]);
      }
      __syncthreads();
      for (int n = 0; n < cs.order; ++n)
        for (uint32_t k = t; k < cs.J[n]; k += T) {
          u[cs.off[n] + k] = a.mt.U[n][(uint64_t)idx_s[n] * a.mt.JP[n] + k];
          cont[cs.off[n] + k] = 0.f;
        }
      __syncthreads();
      const float xh = block_sum(team_contract<OPT>(cs, Gs, u, cont, t, T), red);
      __syncthreads();
      const float r = x_s - xh;
      // core step (uses pre-update rows and core)
      uint32_t j[kMaxOrder];
      for (uint32_t d = t; d < cs.size; d += T) {
        if (!core_active(cs, d)) continue;
        decode(cs, d, j);
        float p = 1.f;
        for (int n = 0; n < cs.order; ++n) p *= u[cs.off[n] + j[n]];
        const float g = fmaf(-r, p, a.core_reg * Gs[d]);
        float v = Gs[d] - a.eta_core * g;
        if (a.nonneg && v < 0.f) v = 0.f;
        Gs[d] = v;
      }
      // row steps
      for (int n = 0; n < cs.order; ++n)
        for (uint32_t k = t; k < cs.J[n]; k += T) {
          const uint32_t q = cs.off[n] + k;
          const float reg = a.mt.reg[n][idx_s[n]];
          const float g = fmaf(-r, cont[q], reg * u[q]);
          float v = u[q] - a.eta * g;
          if (a.nonneg && v < 0.f) v = 0.f;
          a.mt.U[n][(uint64_t)idx_s[n] * a.mt.JP[n] + k] = v;
        }
      __syncthreads();
    } else {
      int m = 0;
      while (id >= a.mat_base[m + 1]) ++m;
      const MatDev& M = a.mats[m];
      const uint64_t e = id - a.mat_base[m];
      const uint32_t* rr = M.rec + (uint64_t)M.pos[e] * 3;
      const uint32_t i1 = rr[0], i2 = rr[1];
      const float y = __uint_as_float(rr[2]);
      const uint32_t J = cs.J[M.mode];
      const uint32_t JP = a.mt.JP[M.mode];
      float* ur = a.mt.U[M.mode] + (uint64_t)i1 * JP;
      float* vr = M.V + (uint64_t)i2 * JP;
      if (t < 32) {
        float part = 0.f;
        for (uint32_t k = t; k < J; k += 32) part = fmaf(ur[k], vr[k], part);
        const float yh = warp_sum(part);
        const float r = y - yh;
        const float reg = M.vreg[i2];
        for (uint32_t k = t; k < J; k += 32) {
          const float uk = ur[k], vk = vr[k];
          const float du = -M.weight * r * vk;
          const float dv = fmaf(-M.weight * r, uk, reg * vk);
          float a1 = uk - a.eta * du;
          float b1 = vk - a.eta * dv;
          if (a.nonneg) {
            a1 = a1 < 0.f ? 0.f : a1;
            b1 = b1 < 0.f ? 0.f : b1;
          }
          ur[k] = a1;
          vr[k] = b1;
        }
      }
      __syncthreads();
    }
  }
  for (uint32_t d = t; d < cs.size; d += T) a.G[d] = Gs[d];
}

// ---------------------------------------------------------------------
// Generic Hogwild sweep: one warp per entry, each warp walks a contiguous
// chunk of the sorted COO.  Rows are read/written with relaxed (L2)
// accesses; the core gradient is accumulated block-locally in shared memory
// over one block-iteration (one entry per warp) and then applied to the
// global core with atomics, the block's core copy being refreshed from the
// atomics' return values.
// ---------------------------------------------------------------------
struct HogArgs {
  CoreShape cs;
  float* G;
  const uint32_t* rec;
  uint64_t nnz;
  ModeTables mt;
  float eta;
  float core_reg;
  int nonneg;
  uint32_t* visits;  // debug_count_visits (null: off)
};

template <bool OPT>
__global__ void hogwild_generic_kernel(HogArgs a) {
  extern __shared__ float sm[];
  const CoreShape& cs = a.cs;
  const uint32_t sumJ = cs.off[cs.order];
  const int warps = blockDim.x >> 5;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  float* Gs = sm;
  float* dG = Gs + cs.size;
  float* u = dG + cs.size + w * 2 * sumJ;
  float* cont = u + sumJ;
  const uint64_t W = (uint64_t)gridDim.x * warps;
  const uint64_t gw = (uint64_t)blockIdx.x * warps + w;
  const uint64_t lo = a.nnz * gw / W, hi = a.nnz * (gw + 1) / W;
  const uint64_t iters = (a.nnz + W - 1) / W;
  for (uint32_t d = threadIdx.x; d < cs.size; d += blockDim.x) {
    Gs[d] = a.G[d];
    dG[d] = 0.f;
  }
  __syncthreads();
  for (uint64_t it = 0; it < iters; ++it) {
    const uint64_t e = lo + it;
    const bool active = e < hi;
    uint32_t idx[kMaxOrder];
    float r = 0.f;
    if (active) {
      if (a.visits && l == 0) atomicAdd(a.visits + e, 1u);
      const uint32_t* rp = a.rec + e * (cs.order + 1);
      for (int n = 0; n < cs.order; ++n) idx[n] = rp[n];
      const float x = __uint_as_float(rp[cs.order]);
      for (int n = 0; n < cs.order; ++n)
        for (uint32_t k = l; k < cs.J[n]; k += 32) {
          u[cs.off[n] + k] = ld_row1(&a.mt.U[n][(uint64_t)idx[n] * a.mt.JP[n] + k]);
          cont[cs.off[n] + k] = 0.f;
        }
      __syncwarp();
      const float xh = warp_sum(team_contract<OPT>(cs, Gs, u, cont, l, 32));
      __syncwarp();
      r = x - xh;
      // block-local core gradient accumulation (pre-update rows)
      uint32_t j[kMaxOrder];
      for (uint32_t d = l; d < cs.size; d += 32) {
        if (!core_active(cs, d)) continue;  // CP: off-diagonal elements stay 0
        decode(cs, d, j);
        float p = 1.f;
        for (int n = 0; n < cs.order; ++n) p *= u[cs.off[n] + j[n]];
        atomicAdd(&dG[d], -r * p);
      }
      for (int n = 0; n < cs.order; ++n) {
        const float reg = a.mt.reg[n][idx[n]];
        for (uint32_t k = l; k < cs.J[n]; k += 32) {
          const uint32_t q = cs.off[n] + k;
          const float g = fmaf(-r, cont[q], reg * u[q]);
          float v = u[q] - a.eta * g;
          if (a.nonneg && v < 0.f) v = 0.f;
          st_row1(&a.mt.U[n][(uint64_t)idx[n] * a.mt.JP[n] + k], v);
        }
      }
    }
    const int k_active = __syncthreads_count(active && l == 0);
    for (uint32_t d = threadIdx.x; d < cs.size; d += blockDim.x) {
      const float g = dG[d] + (float)k_active * a.core_reg * Gs[d];
      const float delta = -a.eta * g;
      float nv = atomicAdd(&a.G[d], delta) + delta;
      if (a.nonneg && nv < 0.f) nv = 0.f;
      Gs[d] = nv;
      dG[d] = 0.f;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------
// Coupled-matrix sweep (src/trainer.cpp:220-235 per entry): each thread
// walks a contiguous chunk of the row-sorted matrix COO, keeping the
// coupled-mode row u in registers while the row index repeats (written back
// on change), V rows gathered/scattered Hogwild-style.
// ---------------------------------------------------------------------
template <int JP>
__global__ void __launch_bounds__(256)
matrix_sweep_kernel(const uint32_t* rec, uint64_t nnz, float* U,
                    float* V, const float* vreg, float weight, float eta,
                    int nonneg, uint32_t* visits) {
  const uint64_t W = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t lo = nnz * t / W, hi = nnz * (t + 1) / W;
  if (lo >= hi) return;
  uint32_t cur = 0xffffffffu;
  float u[JP];
  for (uint64_t e = lo; e < hi; ++e) {
    if (visits) atomicAdd(visits + e, 1u);
    const uint3 rr = *reinterpret_cast<const uint3*>(rec + 3 * e);
    if (rr.x != cur) {
      if (cur != 0xffffffffu) {
#pragma unroll
        for (int k = 0; k < JP; k += 4)
          st_row4(U + (uint64_t)cur * JP + k,
                  make_float4(u[k], u[k + 1], u[k + 2], u[k + 3]));
      }
      cur = rr.x;
#pragma unroll
      for (int k = 0; k < JP; k += 4) {
        const float4 q = ld_row4(U + (uint64_t)cur * JP + k);
        u[k] = q.x; u[k + 1] = q.y; u[k + 2] = q.z; u[k + 3] = q.w;
      }
    }
    float v[JP];
#pragma unroll
    for (int k = 0; k < JP; k += 4) {
      const float4 q = ld_row4(V + (uint64_t)rr.y * JP + k);
      v[k] = q.x; v[k + 1] = q.y; v[k + 2] = q.z; v[k + 3] = q.w;
    }
    float yh = 0.f;
#pragma unroll
    for (int k = 0; k < JP; ++k) yh = fmaf(u[k], v[k], yh);  // padding is 0
    const float r = __uint_as_float(rr.z) - yh;
    const float reg = __ldg(vreg + rr.y);
    const float wr = weight * r;
#pragma unroll
    for (int k = 0; k < JP; ++k) {
      const float du = -wr * v[k];
      const float dv = fmaf(-wr, u[k], reg * v[k]);
      float a1 = u[k] - eta * du;
      float b1 = v[k] - eta * dv;
      if (nonneg) {
        a1 = fmaxf(a1, 0.f);
        b1 = fmaxf(b1, 0.f);
      }
      u[k] = a1;
      v[k] = b1;
    }
#pragma unroll
    for (int k = 0; k < JP; k += 4)
      st_row4(V + (uint64_t)rr.y * JP + k,
              make_float4(v[k], v[k + 1], v[k + 2], v[k + 3]));
  }
#pragma unroll
  for (int k = 0; k < JP; k += 4)
    st_row4(U + (uint64_t)cur * JP + k,
            make_float4(u[k], u[k + 1], u[k + 2], u[k + 3]));
}

// ---------------------------------------------------------------------
// Evaluation (src/eval.cpp:14-97).  Per 1024-entry block a fixed-order
// double partial is produced; the host combines the partials pairwise
// exactly as blocked_sum (src/eval.cpp:46-48), so results are deterministic.
// ---------------------------------------------------------------------
__global__ void eval_generic_kernel(CoreShape cs, const float* G,
                                    const uint32_t* rec, uint64_t nnz,
                                    ModeTables mt, double* partial) {
  extern __shared__ float sm[];
  const uint32_t sumJ = cs.off[cs.order];
  const int warps = blockDim.x >> 5;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  float* Gs = sm;
  float* u = Gs + cs.size + w * sumJ;
  __shared__ double acc_s[32];
  for (uint32_t d = threadIdx.x; d < cs.size; d += blockDim.x) Gs[d] = G[d];
  __syncthreads();
  const uint64_t b = blockIdx.x;
  const uint64_t lo = b * kEvalBlock;
  const uint64_t hi = lo + kEvalBlock < nnz ? lo + kEvalBlock : nnz;
  double acc = 0.0;
  uint32_t j[kMaxOrder];
  for (uint64_t e = lo + w; e < hi; e += warps) {
    const uint32_t* rp = rec + e * (cs.order + 1);
    for (int n = 0; n < cs.order; ++n)
      for (uint32_t k = l; k < cs.J[n]; k += 32)
        u[cs.off[n] + k] = mt.U[n][(uint64_t)rp[n] * mt.JP[n] + k];
    __syncwarp();
    float xh = 0.f;
    for (uint32_t d = l; d < cs.size; d += 32) {
      decode(cs, d, j);
      float p = Gs[d];
      for (int n = 0; n < cs.order; ++n) p *= u[cs.off[n] + j[n]];
      xh += p;
    }
    xh = warp_sum(xh);
    const double r = (double)__uint_as_float(rp[cs.order]) - (double)xh;
    acc += r * r;
    __syncwarp();
  }
  if (l == 0) acc_s[w] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < warps; ++i) s += acc_s[i];
    partial[b] = s;
  }
}

// Matrix SSE partials, fixed 1024-entry blocks.
__global__ void eval_matrix_kernel(const uint32_t* rec, uint64_t nnz,
                                   const float* U, const float* V, uint32_t J,
                                   uint32_t JP, double* partial) {
  __shared__ double acc_s[32];
  const uint64_t b = blockIdx.x;
  const uint64_t lo = b * kEvalBlock;
  const uint64_t hi = lo + kEvalBlock < nnz ? lo + kEvalBlock : nnz;
  double acc = 0.0;
  for (uint64_t e = lo + threadIdx.x; e < hi; e += blockDim.x) {
    const uint32_t* rp = rec + 3 * e;
    const float* ur = U + (uint64_t)rp[0] * JP;
    const float* vr = V + (uint64_t)rp[1] * JP;
    float yh = 0.f;
    for (uint32_t k = 0; k < J; ++k) yh = fmaf(ur[k], vr[k], yh);
    const double r = (double)__uint_as_float(rp[2]) - (double)yh;
    acc += r * r;
  }
  acc = warp_sum_d(acc);
  if ((threadIdx.x & 31) == 0) acc_s[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += acc_s[i];
    partial[b] = s;
  }
}

// Sum of squared row norms over rows with count > 0 (src/eval.cpp:84-97),
// one double partial per block.
__global__ void row_norms_kernel(const float* F, uint32_t rows, uint32_t J,
                                 uint32_t JP, const uint32_t* count,
                                 double* partial) {
  __shared__ double acc_s[32];
  double acc = 0.0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < rows;
       i += (uint64_t)gridDim.x * blockDim.x) {
    if (count && count[i] == 0) continue;
    double s = 0.0;
    for (uint32_t k = 0; k < J; ++k) {
      const double v = F[i * JP + k];
      s += v * v;
    }
    acc += s;
  }
  acc = warp_sum_d(acc);
  if ((threadIdx.x & 31) == 0) acc_s[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += acc_s[i];
    partial[blockIdx.x] = s;
  }
}

// First non-finite element (flat index over the logical J columns) of a
// padded parameter array; result is an atomicMin into *first.
__global__ void nonfinite_kernel(const float* F, uint64_t rows, uint32_t J,
                                 uint32_t JP, unsigned long long* first) {
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
       q < rows * JP; q += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t k = (uint32_t)(q % JP);
    if (k >= J) continue;
    if (!isfinite(F[q]))
      atomicMin(first, (unsigned long long)((q / JP) * J + k));
  }
}

}  // namespace cmtfb
