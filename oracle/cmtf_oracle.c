/*
 * cmtf_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, double-precision restatement of the reference S^3CMTF hot path
 * (/root/reference/proj/core, read-only).  It is the CHECKER for the CUDA
 * product path: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  Nothing in
 * paper_1708_08640_b200/ links or calls it.
 *
 * Parity pin: every function below is checked against vectors produced by
 * the reference itself (oracle/_ref, built from the reference sources by
 * oracle/Makefile) and committed under tests/golden/ by
 * tests/golden/make_golden.py; see tests/test_oracle_golden.py.
 *
 * Each function names the reference file:line it restates (paths relative
 * to /root/reference/proj/core).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_MAX_ORDER 16
#define ORC_DIVISOR_FLOOR 1e-12 /* src/gradients.cpp:13 */

/* ------------------------------------------------------------------ */
/* mt19937_64 + the reference's stream mixing (include/cmtf/rng.hpp,   */
/* src/rng.cpp:8-26).  The generator itself is the standard 64-bit     */
/* Mersenne Twister (std::mt19937_64), restated here.                  */
/* ------------------------------------------------------------------ */
typedef struct {
  uint64_t mt[312];
  int mti;
} orc_mt;

void orc_mt_seed(orc_mt *g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) +
               (uint64_t)i;
  g->mti = 312;
}

uint64_t orc_mt_next(orc_mt *g) {
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  const uint64_t A = 0xB5026F5AA96619E9ULL;
  if (g->mti >= 312) {
    int i;
    for (i = 0; i < 312 - 156; ++i) {
      uint64_t x = (g->mt[i] & UM) | (g->mt[i + 1] & LM);
      g->mt[i] = g->mt[i + 156] ^ (x >> 1) ^ ((x & 1ULL) ? A : 0ULL);
    }
    for (; i < 311; ++i) {
      uint64_t x = (g->mt[i] & UM) | (g->mt[i + 1] & LM);
      g->mt[i] = g->mt[i + (156 - 312)] ^ (x >> 1) ^ ((x & 1ULL) ? A : 0ULL);
    }
    uint64_t x = (g->mt[311] & UM) | (g->mt[0] & LM);
    g->mt[311] = g->mt[155] ^ (x >> 1) ^ ((x & 1ULL) ? A : 0ULL);
    g->mti = 0;
  }
  uint64_t x = g->mt[g->mti++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

static uint64_t splitmix64(uint64_t *state) { /* src/rng.cpp:8-14 */
  *state += 0x9e3779b97f4a7c15ULL;
  uint64_t z = *state;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* make_rng: src/rng.cpp:17-26.  Streams: Init=1 Shuffle=2 Split=3 Synth=4
 * Bench=5 (include/cmtf/rng.hpp:11-17). */
void orc_make_rng(orc_mt *g, uint64_t seed, uint64_t stream, uint64_t index) {
  uint64_t state = seed;
  uint64_t mixed = splitmix64(&state);
  state ^= stream * 0xd1b54a32d192ed03ULL;
  mixed ^= splitmix64(&state);
  state ^= index * 0x9e3779b97f4a7c15ULL;
  mixed ^= splitmix64(&state);
  orc_mt_seed(g, mixed);
}

/* include/cmtf/rng.hpp:24-26 */
static double uniform01(orc_mt *g) {
  return (double)(orc_mt_next(g) >> 11) * 0x1.0p-53;
}
/* include/cmtf/rng.hpp:33-36 */
static uint64_t bounded(orc_mt *g, uint64_t n) {
  return (uint64_t)(((unsigned __int128)orc_mt_next(g) * n) >> 64);
}

/* ------------------------------------------------------------------ */
/* Problem description passed in from ctypes.                          */
/* ------------------------------------------------------------------ */
typedef struct {
  int32_t order;
  int32_t cp; /* 1: hyper-diagonal CP core (superdiagonal stored) */
  const uint32_t *dims;
  const uint32_t *ranks;
  uint64_t nnz;
  const uint32_t *idx; /* AoS, order per entry, 0-based */
  const double *vals;
  int32_t n_mat;
  const int32_t *mat_mode;
  const uint32_t *mat_cols;
  const uint64_t *mat_nnz;
  const uint32_t *const *mat_idx; /* pairs (row, col) */
  const double *const *mat_vals;
  const double *mat_weight;
} orc_bundle;

typedef struct {
  double *core;
  double *const *factors;   /* [order] row-major I_n x J_n */
  double *const *couplings; /* [n_mat] row-major cols x J_mode */
} orc_model;

static uint64_t dense_size(int order, const uint32_t *ranks) {
  uint64_t s = 1;
  for (int n = 0; n < order; ++n) s *= ranks[n];
  return s;
}
static uint64_t stored_size(int order, const uint32_t *ranks, int cp) {
  return cp ? ranks[0] : dense_size(order, ranks);
}

/* Digit-counter advance, last mode fastest (src/tucker.cpp:49-54,114-125) */
static void advance(uint32_t *j, int order, const uint32_t *ranks) {
  for (int n = order - 1; n >= 0; --n) {
    if (++j[n] < ranks[n]) return;
    j[n] = 0;
  }
}

/* predict_entry: src/tucker.cpp:96-127 */
double orc_predict(int order, const uint32_t *ranks, int cp, const double *g,
                   const double *const *rows) {
  double acc = 0.0;
  if (cp) {
    for (uint32_t k = 0; k < ranks[0]; ++k) {
      double p = g[k];
      for (int n = 0; n < order; ++n) p *= rows[n][k];
      acc += p;
    }
    return acc;
  }
  uint32_t j[ORC_MAX_ORDER] = {0};
  uint64_t size = dense_size(order, ranks);
  for (uint64_t d = 0; d < size; ++d) {
    double p = g[d];
    for (int n = 0; n < order; ++n) p *= rows[n][j[n]];
    acc += p;
    advance(j, order, ranks);
  }
  return acc;
}

/* contract_all_but: src/tucker.cpp:129-165 */
void orc_contract_all_but(int order, const uint32_t *ranks, int cp,
                          const double *g, const double *const *rows,
                          int skip, double *out) {
  for (uint32_t k = 0; k < ranks[skip]; ++k) out[k] = 0.0;
  if (cp) {
    for (uint32_t k = 0; k < ranks[0]; ++k) {
      double p = g[k];
      for (int n = 0; n < order; ++n)
        if (n != skip) p *= rows[n][k];
      out[k] += p;
    }
    return;
  }
  uint32_t j[ORC_MAX_ORDER] = {0};
  uint64_t size = dense_size(order, ranks);
  for (uint64_t d = 0; d < size; ++d) {
    double p = g[d];
    for (int n = 0; n < order; ++n)
      if (n != skip) p *= rows[n][j[n]];
    out[j[skip]] += p;
    advance(j, order, ranks);
  }
}

/* finish_row_gradient: src/gradients.cpp:73-79 */
static void finish_row(const double *c, double r, const double *u,
                       double lambda, uint32_t count, uint32_t jn,
                       double *out) {
  const double reg = lambda / (double)count;
  for (uint32_t k = 0; k < jn; ++k) out[k] = -r * c[k] + reg * u[k];
}

/*
 * compute_gradient (opt=0): src/gradients.cpp:83-128 (Algorithm 2).
 * compute_gradient_opt (opt=1): src/gradients.cpp:130-223 (Algorithm 3),
 * including the near-zero divisor fallbacks (:168-186, :207-222).
 * grow is the concatenation of the N row gradients (J_1 + ... + J_N).
 */
void orc_compute_gradient(int opt, double x, int order, const uint32_t *ranks,
                          int cp, const double *g, const double *const *rows,
                          double lambda, const uint32_t *counts,
                          uint64_t nnz_total, int with_core, double *grow,
                          double *gcore, double *residual) {
  const uint64_t stored = stored_size(order, ranks, cp);
  double buf[1024];
  double *s = NULL;
  double r;
  if (!opt) {
    r = x - orc_predict(order, ranks, cp, g, rows);
    double *out = grow;
    for (int n = 0; n < order; ++n) {
      orc_contract_all_but(order, ranks, cp, g, rows, n, buf);
      finish_row(buf, r, rows[n], lambda, counts[n], ranks[n], out);
      out += ranks[n];
    }
    if (with_core) {
      const double core_reg = lambda / (double)nnz_total;
      if (cp) {
        for (uint32_t k = 0; k < ranks[0]; ++k) {
          double p = 1.0;
          for (int n = 0; n < order; ++n) p *= rows[n][k];
          gcore[k] = -r * p + core_reg * g[k];
        }
      } else {
        uint32_t j[ORC_MAX_ORDER] = {0};
        for (uint64_t d = 0; d < stored; ++d) {
          double p = 1.0;
          for (int n = 0; n < order; ++n) p *= rows[n][j[n]];
          gcore[d] = -r * p + core_reg * g[d];
          advance(j, order, ranks);
        }
      }
    }
    *residual = r;
    return;
  }

  /* Algorithm 3: intermediate tensor S and x_hat in one walk (:143-164). */
  s = (double *)malloc(sizeof(double) * stored);
  double xhat = 0.0;
  if (cp) {
    for (uint32_t k = 0; k < ranks[0]; ++k) {
      double p = g[k];
      for (int n = 0; n < order; ++n) p *= rows[n][k];
      s[k] = p;
      xhat += p;
    }
  } else {
    uint32_t j[ORC_MAX_ORDER] = {0};
    for (uint64_t d = 0; d < stored; ++d) {
      double p = g[d];
      for (int n = 0; n < order; ++n) p *= rows[n][j[n]];
      s[d] = p;
      xhat += p;
      advance(j, order, ranks);
    }
  }
  r = x - xhat;

  uint64_t strides[ORC_MAX_ORDER];
  {
    uint64_t acc = 1;
    for (int n = order - 1; n >= 0; --n) {
      strides[n] = acc;
      acc *= ranks[n];
    }
  }
  double *out = grow;
  for (int n = 0; n < order; ++n) {
    const double *u = rows[n];
    int divisible = 1;
    for (uint32_t k = 0; k < ranks[n]; ++k)
      if (fabs(u[k]) < ORC_DIVISOR_FLOOR) {
        divisible = 0;
        break;
      }
    if (divisible) {
      /* collapse: src/gradients.cpp:35-60 */
      if (cp) {
        for (uint32_t k = 0; k < ranks[0]; ++k) buf[k] = s[k];
      } else {
        for (uint32_t k = 0; k < ranks[n]; ++k) buf[k] = 0.0;
        const uint64_t stride = strides[n];
        const uint64_t block = stride * ranks[n];
        for (uint64_t base = 0; base < stored; base += block)
          for (uint32_t k = 0; k < ranks[n]; ++k) {
            double acc = 0.0;
            const double *p = s + base + k * stride;
            for (uint64_t t = 0; t < stride; ++t) acc += p[t];
            buf[k] += acc;
          }
      }
      for (uint32_t k = 0; k < ranks[n]; ++k) buf[k] /= u[k];
    } else {
      orc_contract_all_but(order, ranks, cp, g, rows, n, buf);
    }
    finish_row(buf, r, u, lambda, counts[n], ranks[n], out);
    out += ranks[n];
  }

  if (with_core) {
    const double core_reg = lambda / (double)nnz_total;
    uint32_t j[ORC_MAX_ORDER] = {0};
    for (uint64_t d = 0; d < stored; ++d) {
      const double gd = g[d];
      double p;
      if (fabs(gd) < ORC_DIVISOR_FLOOR) {
        p = 1.0;
        for (int n = 0; n < order; ++n)
          p *= rows[n][cp ? (uint32_t)d : j[n]];
      } else {
        p = s[d] / gd;
      }
      gcore[d] = -r * p + core_reg * gd;
      if (!cp) advance(j, order, ranks);
    }
  }
  free(s);
  *residual = r;
}

/* matrix_entry_gradients: src/gradients.cpp:225-248 */
void orc_matrix_entry_gradients(double y, const double *u, const double *v,
                                uint32_t j, double lambda_m, double lambda,
                                uint32_t col_count, double *du, double *dv,
                                double *residual) {
  double yhat = 0.0;
  for (uint32_t k = 0; k < j; ++k) yhat += u[k] * v[k];
  const double r = y - yhat;
  const double reg = lambda_m * lambda / (double)col_count;
  for (uint32_t k = 0; k < j; ++k) {
    du[k] = -lambda_m * r * v[k];
    dv[k] = -lambda_m * r * u[k] + reg * v[k];
  }
  *residual = r;
}

/* ------------------------------------------------------------------ */
/* Counts, init, split, schedule                                       */
/* ------------------------------------------------------------------ */

/* count_mode_occurrences: src/sparse_data.cpp:344-362.  out holds the
 * per-mode tensor counts concatenated (sum dims) followed by the per-matrix
 * column counts concatenated (sum cols). */
void orc_count_modes(const orc_bundle *b, uint32_t *out) {
  uint64_t total = 0;
  for (int n = 0; n < b->order; ++n) total += b->dims[n];
  for (int m = 0; m < b->n_mat; ++m) total += b->mat_cols[m];
  memset(out, 0, sizeof(uint32_t) * total);
  uint32_t *base[ORC_MAX_ORDER];
  uint32_t *p = out;
  for (int n = 0; n < b->order; ++n) {
    base[n] = p;
    p += b->dims[n];
  }
  for (uint64_t e = 0; e < b->nnz; ++e)
    for (int n = 0; n < b->order; ++n) ++base[n][b->idx[e * b->order + n]];
  for (int m = 0; m < b->n_mat; ++m) {
    for (uint64_t e = 0; e < b->mat_nnz[m]; ++e) ++p[b->mat_idx[m][2 * e + 1]];
    p += b->mat_cols[m];
  }
}

/* random_model: src/trainer.cpp:30-58, rng = make_rng(seed, Init)
 * (src/trainer.cpp:100).  Draw order: core, factors by mode, couplings. */
void orc_initialize(const orc_bundle *b, double scale, uint64_t seed,
                    orc_model *m) {
  orc_mt g;
  orc_make_rng(&g, seed, 1, 0);
  const uint64_t stored = stored_size(b->order, b->ranks, b->cp);
  for (uint64_t d = 0; d < stored; ++d) m->core[d] = scale * uniform01(&g);
  for (int n = 0; n < b->order; ++n) {
    const double hi = scale / sqrt((double)b->ranks[n]);
    const uint64_t cnt = (uint64_t)b->dims[n] * b->ranks[n];
    for (uint64_t i = 0; i < cnt; ++i)
      m->factors[n][i] = 0.0 + (hi - 0.0) * uniform01(&g);
  }
  for (int c = 0; c < b->n_mat; ++c) {
    const uint32_t jn = b->ranks[b->mat_mode[c]];
    const double hi = scale / sqrt((double)jn);
    const uint64_t cnt = (uint64_t)b->mat_cols[c] * jn;
    for (uint64_t i = 0; i < cnt; ++i)
      m->couplings[c][i] = 0.0 + (hi - 0.0) * uniform01(&g);
  }
}

/* split_train_test permutation: src/sparse_data.cpp:311-342.  After the
 * call ids[0, n_test) are the test entries and ids[n_test, nnz) the training
 * entries, in this order. Returns n_test = llround(f * nnz). */
uint64_t orc_split_perm(uint64_t nnz, double test_fraction, uint64_t seed,
                        uint64_t *ids) {
  for (uint64_t i = 0; i < nnz; ++i) ids[i] = i;
  orc_mt g;
  orc_make_rng(&g, seed, 3, 0);
  for (uint64_t i = nnz - 1; i > 0; --i) {
    uint64_t k = bounded(&g, i + 1);
    uint64_t t = ids[i];
    ids[i] = ids[k];
    ids[k] = t;
  }
  return (uint64_t)llround(test_fraction * (double)nnz);
}

/* build_schedule: src/trainer.cpp:114-120 */
void orc_build_schedule(uint64_t *s, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) s[i] = i;
}

/* shuffle_schedule: src/trainer.cpp:122-128 (applied to the persisted
 * array, so shuffles accumulate across epochs). */
void orc_shuffle(uint64_t *s, uint64_t n, uint64_t seed, int32_t epoch) {
  orc_mt g;
  orc_make_rng(&g, seed, 2, (uint64_t)epoch);
  for (uint64_t i = n; i > 1; --i) {
    uint64_t k = bounded(&g, i);
    uint64_t t = s[i - 1];
    s[i - 1] = s[k];
    s[k] = t;
  }
}

/* ------------------------------------------------------------------ */
/* One epoch: src/trainer.cpp:166-237 (sweep) and :267-316 (run_epoch). */
/* workers > 1 is serialised chunk by chunk (chunk 0 designated, core   */
/* step eta*P, src/trainer.cpp:211-219) -- one admissible interleaving  */
/* of the reference's Hogwild execution.  Returns 0, or 2 on a          */
/* non-finite parameter (src/trainer.cpp:312-315).                      */
/* ------------------------------------------------------------------ */
int orc_run_epoch_counts(const orc_bundle *b, orc_model *m, uint64_t *schedule,
                         int32_t epoch, uint64_t seed, double eta, double lambda,
                         int32_t kernel_opt, int32_t workers, int32_t nonneg,
                         int32_t do_shuffle, const uint32_t *given_counts,
                         uint64_t nnz_global, uint64_t n_sched);

int orc_run_epoch(const orc_bundle *b, orc_model *m, uint64_t *schedule,
                  int32_t epoch, uint64_t seed, double eta, double lambda,
                  int32_t kernel_opt, int32_t workers, int32_t nonneg,
                  int32_t do_shuffle) {
  return orc_run_epoch_counts(b, m, schedule, epoch, seed, eta, lambda, kernel_opt,
                              workers, nonneg, do_shuffle, NULL, 0, 0);
}

/* As orc_run_epoch, with externally supplied (global) counts and the global
 * training nnz for the core regulariser -- the per-stratum sweep of the
 * DSGD test oracle. */
int orc_run_epoch_counts(const orc_bundle *b, orc_model *m, uint64_t *schedule,
                         int32_t epoch, uint64_t seed, double eta, double lambda,
                         int32_t kernel_opt, int32_t workers, int32_t nonneg,
                         int32_t do_shuffle, const uint32_t *given_counts,
                         uint64_t nnz_global, uint64_t n_sched) {
  const int order = b->order;
  uint64_t total = b->nnz;
  for (int c = 0; c < b->n_mat; ++c) total += b->mat_nnz[c];
  if (n_sched) total = n_sched; /* a sub-schedule (one DSGD stratum) */
  if (do_shuffle) orc_shuffle(schedule, total, seed, epoch);

  uint64_t cnt_total = 0;
  for (int n = 0; n < order; ++n) cnt_total += b->dims[n];
  for (int c = 0; c < b->n_mat; ++c) cnt_total += b->mat_cols[c];
  uint32_t *counts = (uint32_t *)malloc(sizeof(uint32_t) * cnt_total);
  if (given_counts)
    memcpy(counts, given_counts, sizeof(uint32_t) * cnt_total);
  else
    orc_count_modes(b, counts);
  const uint64_t nnz_core = nnz_global ? nnz_global : b->nnz;
  const uint32_t *tcount[ORC_MAX_ORDER];
  const uint32_t *mcount[64];
  {
    const uint32_t *p = counts;
    for (int n = 0; n < order; ++n) {
      tcount[n] = p;
      p += b->dims[n];
    }
    for (int c = 0; c < b->n_mat; ++c) {
      mcount[c] = p;
      p += b->mat_cols[c];
    }
  }

  uint64_t sum_j = 0;
  for (int n = 0; n < order; ++n) sum_j += b->ranks[n];
  const uint64_t stored = stored_size(order, b->ranks, b->cp);
  double *grow = (double *)malloc(sizeof(double) * sum_j);
  double *gcore = (double *)malloc(sizeof(double) * stored);
  double du[1024], dv[1024];

  for (int w = 0; w < workers; ++w) {
    const uint64_t lo = total * (uint64_t)w / (uint64_t)workers;
    const uint64_t hi = total * (uint64_t)(w + 1) / (uint64_t)workers;
    const int designated = (w == 0);
    for (uint64_t i = lo; i < hi; ++i) {
      const uint64_t id = schedule[i];
      if (id < b->nnz) {
        const double *rows[ORC_MAX_ORDER];
        uint32_t cn[ORC_MAX_ORDER];
        for (int n = 0; n < order; ++n) {
          const uint32_t ix = b->idx[id * order + n];
          rows[n] = m->factors[n] + (uint64_t)ix * b->ranks[n];
          cn[n] = tcount[n][ix];
        }
        double r;
        orc_compute_gradient(kernel_opt, b->vals[id], order, b->ranks, b->cp,
                             m->core, rows, lambda, cn, nnz_core, designated,
                             grow, gcore, &r);
        const double *gp = grow;
        for (int n = 0; n < order; ++n) {
          double *u = (double *)rows[n];
          for (uint32_t k = 0; k < b->ranks[n]; ++k) {
            double v = u[k] - eta * gp[k];
            if (nonneg && v < 0) v = 0;
            u[k] = v;
          }
          gp += b->ranks[n];
        }
        if (designated) {
          const double eta_p = eta * (double)workers;
          for (uint64_t d = 0; d < stored; ++d) {
            double v = m->core[d] - eta_p * gcore[d];
            if (nonneg && v < 0) v = 0;
            m->core[d] = v;
          }
        }
      } else {
        uint64_t e = id - b->nnz;
        int c = 0;
        while (e >= b->mat_nnz[c]) {
          e -= b->mat_nnz[c];
          ++c;
        }
        const uint32_t j1 = b->mat_idx[c][2 * e];
        const uint32_t j2 = b->mat_idx[c][2 * e + 1];
        const uint32_t jn = b->ranks[b->mat_mode[c]];
        double *u = m->factors[b->mat_mode[c]] + (uint64_t)j1 * jn;
        double *v = m->couplings[c] + (uint64_t)j2 * jn;
        double r;
        orc_matrix_entry_gradients(b->mat_vals[c][e], u, v, jn,
                                   b->mat_weight[c], lambda, mcount[c][j2], du,
                                   dv, &r);
        for (uint32_t k = 0; k < jn; ++k) {
          double a = u[k] - eta * du[k];
          if (nonneg && a < 0) a = 0;
          u[k] = a;
          double bb = v[k] - eta * dv[k];
          if (nonneg && bb < 0) bb = 0;
          v[k] = bb;
        }
      }
    }
  }
  free(grow);
  free(gcore);
  free(counts);

  /* find_non_finite: src/trainer.cpp:239-263 */
  for (uint64_t d = 0; d < stored; ++d)
    if (!isfinite(m->core[d])) return 2;
  for (int n = 0; n < order; ++n)
    for (uint64_t i = 0; i < (uint64_t)b->dims[n] * b->ranks[n]; ++i)
      if (!isfinite(m->factors[n][i])) return 2;
  for (int c = 0; c < b->n_mat; ++c)
    for (uint64_t i = 0; i < (uint64_t)b->mat_cols[c] * b->ranks[b->mat_mode[c]];
         ++i)
      if (!isfinite(m->couplings[c][i])) return 2;
  return 0;
}

/* ------------------------------------------------------------------ */
/* Evaluation: src/eval.cpp:10-144                                     */
/* ------------------------------------------------------------------ */
#define ORC_KBLOCK 1024 /* src/eval.cpp:10 */

/* blocked_sum: fixed 1024-entry blocks, then pairwise over the block sums
 * (src/eval.cpp:14-50). */
static double blocked_sum_finish(double *partial, uint64_t n_blocks) {
  for (uint64_t width = 1; width < n_blocks; width *= 2)
    for (uint64_t i = 0; i + width < n_blocks; i += 2 * width)
      partial[i] += partial[i + width];
  return partial[0];
}

/* tensor_sse: src/eval.cpp:52-65 */
double orc_tensor_sse(int order, const uint32_t *ranks, int cp,
                      const double *core, double *const *factors, uint64_t nnz,
                      const uint32_t *idx, const double *vals) {
  if (nnz == 0) return 0.0;
  const uint64_t nb = (nnz + ORC_KBLOCK - 1) / ORC_KBLOCK;
  double *partial = (double *)calloc(nb, sizeof(double));
  const double *rows[ORC_MAX_ORDER];
  for (uint64_t bidx = 0; bidx < nb; ++bidx) {
    const uint64_t lo = bidx * ORC_KBLOCK;
    const uint64_t hi = (lo + ORC_KBLOCK < nnz) ? lo + ORC_KBLOCK : nnz;
    double acc = 0.0;
    for (uint64_t e = lo; e < hi; ++e) {
      for (int n = 0; n < order; ++n)
        rows[n] = factors[n] + (uint64_t)idx[e * order + n] * ranks[n];
      const double r = vals[e] - orc_predict(order, ranks, cp, core, rows);
      acc += r * r;
    }
    partial[bidx] = acc;
  }
  double s = blocked_sum_finish(partial, nb);
  free(partial);
  return s;
}

/* matrix_sse: src/eval.cpp:67-81 */
double orc_matrix_sse(uint32_t j, const double *u, const double *v,
                      uint64_t nnz, const uint32_t *idx, const double *vals) {
  if (nnz == 0) return 0.0;
  const uint64_t nb = (nnz + ORC_KBLOCK - 1) / ORC_KBLOCK;
  double *partial = (double *)calloc(nb, sizeof(double));
  for (uint64_t bidx = 0; bidx < nb; ++bidx) {
    const uint64_t lo = bidx * ORC_KBLOCK;
    const uint64_t hi = (lo + ORC_KBLOCK < nnz) ? lo + ORC_KBLOCK : nnz;
    double acc = 0.0;
    for (uint64_t e = lo; e < hi; ++e) {
      const double *ur = u + (uint64_t)idx[2 * e] * j;
      const double *vr = v + (uint64_t)idx[2 * e + 1] * j;
      double yhat = 0.0;
      for (uint32_t k = 0; k < j; ++k) yhat += ur[k] * vr[k];
      const double r = vals[e] - yhat;
      acc += r * r;
    }
    partial[bidx] = acc;
  }
  double s = blocked_sum_finish(partial, nb);
  free(partial);
  return s;
}

/* observed_row_norms: src/eval.cpp:84-97 */
static double observed_row_norms(const double *f, uint32_t rows, uint32_t cols,
                                 const uint32_t *counts) {
  double acc = 0.0;
  for (uint32_t i = 0; i < rows; ++i)
    if (counts[i] > 0) {
      double s = 0.0;
      for (uint32_t k = 0; k < cols; ++k) s += f[(uint64_t)i * cols + k] * f[(uint64_t)i * cols + k];
      acc += s;
    }
  return acc;
}

/* epoch_stats: src/eval.cpp:120-144 */
void orc_epoch_stats(const orc_bundle *b, const orc_model *m, double lambda,
                     double *train_rmse, double *objective) {
  const int order = b->order;
  const double sse = orc_tensor_sse(order, b->ranks, b->cp, m->core,
                                    m->factors, b->nnz, b->idx, b->vals);
  uint64_t cnt_total = 0;
  for (int n = 0; n < order; ++n) cnt_total += b->dims[n];
  for (int c = 0; c < b->n_mat; ++c) cnt_total += b->mat_cols[c];
  uint32_t *counts = (uint32_t *)malloc(sizeof(uint32_t) * cnt_total);
  orc_count_modes(b, counts);

  const uint64_t stored = stored_size(order, b->ranks, b->cp);
  double gn = 0.0;
  for (uint64_t d = 0; d < stored; ++d) gn += m->core[d] * m->core[d];
  double f_t = sse + lambda * gn;
  const uint32_t *p = counts;
  for (int n = 0; n < order; ++n) {
    f_t += lambda * observed_row_norms(m->factors[n], b->dims[n], b->ranks[n], p);
    p += b->dims[n];
  }
  double obj = 0.5 * f_t;
  for (int c = 0; c < b->n_mat; ++c) {
    const uint32_t jn = b->ranks[b->mat_mode[c]];
    double f_m = orc_matrix_sse(jn, m->factors[b->mat_mode[c]], m->couplings[c],
                                b->mat_nnz[c], b->mat_idx[c], b->mat_vals[c]);
    f_m += lambda * observed_row_norms(m->couplings[c], b->mat_cols[c], jn, p);
    p += b->mat_cols[c];
    obj += 0.5 * b->mat_weight[c] * f_m;
  }
  free(counts);
  *train_rmse = b->nnz ? sqrt(sse / (double)b->nnz) : 0.0;
  *objective = obj;
}
