// stateless64.cuh -- the stateless per-entry gradient API
// (cmtf_gpu_compute_gradient: compute_gradient / compute_gradient_opt,
// include/cmtf/gradients.hpp:59-74) in f64 on the device.
//
// The API's arguments and results are double precision and carry no model
// state, so it computes at the precision of its signature: one warp per
// entry, f64 shared-memory rows and contractions, the reference's
// algorithms term for term (src/gradients.cpp:83-223):
//   naive: x_hat by the predict_entry walk, one contract_all_but walk per
//          mode, core gradient -r * prod u + core_reg * g;
//   opt:   the intermediate tensor S[d] = g_d prod_n u_n[j_n], x_hat = sum S,
//          row gradient collapse(S, n)[k] / u_n[k] (direct contraction where
//          |u_n[k]| < 1e-12), core gradient -r * S[d] / g_d (direct product
//          where |g_d| < 1e-12) -- S is returned as KernelWorkspace::s.
// The epoch kernels are fp32; this path exists for the reference's
// stateless kernel API and its unit tests.
#pragma once

#include "generic.cuh"

namespace cmtfb {

constexpr double kDivisorFloor64 = 1e-12;  // src/gradients.cpp:15

struct Probe64Args {
  CoreShape cs;
  const double* G;       // dense core (CP: zero off the superdiagonal)
  const double* rows;    // n x sumJ
  const double* x;
  const uint32_t* counts;  // n x order
  double lambda;
  uint64_t n;
  double core_reg;       // lambda / nnz_total
  int with_core;
  double* resid;
  double* grow;          // n x sumJ
  double* gcore;         // n x size (dense)
  double* inter;         // n x size (opt: the intermediate tensor S), may be null
};

__device__ __forceinline__ double warp_sum64(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// One warp per entry; smem per warp: u[sumJ] + cont[sumJ] + csum[sumJ] (f64)
template <bool OPT>
__global__ void probe64_kernel(Probe64Args a) {
  extern __shared__ double sm64[];
  const int warps = blockDim.x >> 5;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const CoreShape& cs = a.cs;
  const uint32_t sumJ = cs.off[cs.order];
  double* u = sm64 + (uint64_t)w * 3 * sumJ;
  double* cont = u + sumJ;  // naive: contract_all_but; opt: collapse(S, n)
  for (uint64_t e = (uint64_t)blockIdx.x * warps + w; e < a.n;
       e += (uint64_t)gridDim.x * warps) {
    for (uint32_t k = l; k < sumJ; k += 32) {
      u[k] = a.rows[e * sumJ + k];
      cont[k] = 0.0;
    }
    __syncwarp();
    uint32_t j[kMaxOrder];
    double xh = 0.0;
    if (OPT) {
      for (uint32_t d = l; d < cs.size; d += 32) {
        if (cs.cp && d % cs.dstep) {
          if (a.inter) a.inter[e * cs.size + d] = 0.0;
          continue;
        }
        decode(cs, d, j);
        double p = a.G[d];
        for (int n = 0; n < cs.order; ++n) p *= u[cs.off[n] + j[n]];
        if (a.inter) a.inter[e * cs.size + d] = p;
        xh += p;
        for (int n = 0; n < cs.order; ++n) atomicAdd(&cont[cs.off[n] + j[n]], p);
      }
    } else {
      for (uint32_t d = l; d < cs.size; d += 32) {  // predict_entry walk
        decode(cs, d, j);
        double p = a.G[d];
        for (int n = 0; n < cs.order; ++n) p *= u[cs.off[n] + j[n]];
        xh += p;
      }
    }
    xh = warp_sum64(xh);
    __syncwarp();
    const double r = a.x[e] - xh;
    if (l == 0 && a.resid) a.resid[e] = r;
    for (int n = 0; n < cs.order; ++n) {
      const double reg = a.lambda / (double)a.counts[e * cs.order + n];
      // opt: the mode divides out its own row only if no component is below
      // the floor (src/gradients.cpp:168-186); else the direct contraction
      bool divisible = OPT;
      for (uint32_t k = 0; k < cs.J[n]; ++k)
        if (fabs(u[cs.off[n] + k]) < kDivisorFloor64) divisible = false;
      for (uint32_t k = l; k < cs.J[n]; k += 32) {
        const uint32_t q = cs.off[n] + k;
        double c;
        if (divisible) {
          c = cont[q] / u[q];  // collapse / own row component
        } else {
          // contract_all_but component k of mode n (the naive kernel, and
          // the opt kernel's near-zero-divisor fallback)
          c = 0.0;
          for (uint32_t d = 0; d < cs.size; ++d) {
            decode(cs, d, j);
            if (j[n] != k) continue;
            double p = a.G[d];
            for (int m = 0; m < cs.order; ++m)
              if (m != n) p *= u[cs.off[m] + j[m]];
            c += p;
          }
        }
        a.grow[e * sumJ + q] = -r * c + reg * u[q];  // finish_row_gradient
      }
    }
    if (a.with_core && a.gcore) {
      for (uint32_t d = l; d < cs.size; d += 32) {
        decode(cs, d, j);
        const double g = a.G[d];
        double p;
        if (OPT && fabs(g) >= kDivisorFloor64) {
          p = g;
          for (int n = 0; n < cs.order; ++n) p *= u[cs.off[n] + j[n]];
          p /= g;  // S[d] / g_d
        } else {
          p = 1.0;
          for (int n = 0; n < cs.order; ++n) p *= u[cs.off[n] + j[n]];
        }
        a.gcore[e * cs.size + d] = -r * p + a.core_reg * g;
      }
    }
    __syncwarp();
  }
}

// matrix_entry_gradients (src/gradients.cpp:225-248) in f64: y_hat = u . v,
// r = y - y_hat, du = -lambda_m r v (no regulariser on u),
// dv = -lambda_m r u + (lambda_m lambda / count_col) v
__global__ void matrix_probe64_kernel(uint64_t n, uint32_t J, const double* y, const double* u,
                                      const double* v, double lambda_m, double lambda,
                                      const uint32_t* col_count, double* du, double* dv,
                                      double* resid) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const double* ur = u + e * J;
    const double* vr = v + e * J;
    double yh = 0.0;
    for (uint32_t k = 0; k < J; ++k) yh += ur[k] * vr[k];
    const double r = y[e] - yh;
    const double reg = lambda_m * lambda / (double)col_count[e];
    for (uint32_t k = 0; k < J; ++k) {
      du[e * J + k] = -lambda_m * r * vr[k];
      dv[e * J + k] = -lambda_m * r * ur[k] + reg * vr[k];
    }
    resid[e] = r;
  }
}

// collapse (src/gradients.cpp:35-60): out[k] = sum of the intermediate
// tensor's elements whose mode-`mode` index is k (CP: the identity)
__global__ void collapse64_kernel(CoreShape cs, const double* s, int mode, double* out) {
  const uint32_t jn = cs.J[mode];
  uint64_t stride = 1;
  for (int n = cs.order - 1; n > mode; --n) stride *= cs.J[n];
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < jn; k += gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (uint64_t base = 0; base < cs.size; base += stride * jn)
      for (uint64_t t = 0; t < stride; ++t) acc += s[base + k * stride + t];
    out[k] = acc;
  }
}

}  // namespace cmtfb
