// TEST INFRASTRUCTURE ONLY -- extern "C" wrapper around the UNMODIFIED
// reference library (/root/reference/proj/core), compiled together with the
// reference sources into oracle/_ref/libcmtf_ref.so by oracle/Makefile.
// Used to (a) generate the golden fixtures in tests/golden/ that pin the
// C restatement (oracle/cmtf_oracle.c), and (b) time the reference's own
// multi-threaded CPU path for bench.py's cpu_baseline / --impl reference.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <span>
#include <vector>

#include "cmtf/errors.hpp"
#include "cmtf/eval.hpp"
#include "cmtf/gradients.hpp"
#include "cmtf/model_io.hpp"
#include "cmtf/sparse_data.hpp"
#include "cmtf/synth.hpp"
#include "cmtf/trainer.hpp"
#include "cmtf/tucker.hpp"

using namespace cmtf;

extern "C" {

struct ref_config {
  int32_t order;
  const uint32_t* ranks;
  double eta0, mu, lambda_reg;
  int32_t workers, max_epochs;
  double rel_tol;
  uint64_t seed;
  int32_t kernel_opt, cp, nonnegative;
  double init_scale;
  int32_t eval_threads;
};

static thread_local char g_err[512];
const char* ref_last_error() { return g_err; }

static int fail(const std::exception& e, int code) {
  std::snprintf(g_err, sizeof g_err, "%s", e.what());
  return code;
}

static TrainConfig to_config(const ref_config* c) {
  TrainConfig t;
  t.ranks.assign(c->ranks, c->ranks + c->order);
  t.eta0 = c->eta0;
  t.mu = c->mu;
  t.lambda_reg = c->lambda_reg;
  t.workers = c->workers;
  t.max_epochs = c->max_epochs;
  t.rel_tol = c->rel_tol;
  t.seed = c->seed;
  t.kernel = c->kernel_opt ? GradientKernel::Opt : GradientKernel::Naive;
  t.core_structure =
      c->cp ? CoreStructure::HyperDiagonalCp : CoreStructure::DenseTucker;
  t.nonnegative = c->nonnegative != 0;
  t.init_scale = c->init_scale;
  t.eval_threads = c->eval_threads;
  return t;
}

void* ref_bundle_new(int32_t order, const uint32_t* dims, uint64_t nnz,
                     const uint32_t* idx, const double* vals, int32_t n_mat,
                     const int32_t* mat_mode, const uint32_t* mat_cols,
                     const uint64_t* mat_nnz, const uint32_t* const* mat_idx,
                     const double* const* mat_vals, const double* weights) {
  try {
    SparseTensor t(std::vector<uint32_t>(dims, dims + order),
                   std::vector<uint32_t>(idx, idx + nnz * order),
                   std::vector<double>(vals, vals + nnz));
    std::vector<CoupledMatrix> mats;
    for (int m = 0; m < n_mat; ++m)
      mats.emplace_back(mat_mode[m], dims[mat_mode[m]], mat_cols[m],
                        std::vector<uint32_t>(mat_idx[m],
                                              mat_idx[m] + 2 * mat_nnz[m]),
                        std::vector<double>(mat_vals[m],
                                            mat_vals[m] + mat_nnz[m]),
                        weights[m]);
    return new DataBundle(make_bundle(std::move(t), std::move(mats)));
  } catch (const std::exception& e) {
    fail(e, 1);
    return nullptr;
  }
}

void ref_bundle_free(void* b) { delete static_cast<DataBundle*>(b); }

void* ref_state_new(void* bundle, const ref_config* c) {
  try {
    return new TrainState(
        make_state(to_config(c), *static_cast<DataBundle*>(bundle)));
  } catch (const std::exception& e) {
    fail(e, 1);
    return nullptr;
  }
}

void ref_state_free(void* s) { delete static_cast<TrainState*>(s); }

int ref_run_epoch(void* state, void* bundle, const ref_config* c) {
  try {
    run_epoch(*static_cast<TrainState*>(state),
              *static_cast<DataBundle*>(bundle), to_config(c));
    return 0;
  } catch (const DivergenceError& e) {
    return fail(e, 2);
  } catch (const std::exception& e) {
    return fail(e, 1);
  }
}

static void copy_model_out(const FactorModel& m, double* core,
                           double* const* factors, double* const* couplings) {
  if (core) std::memcpy(core, m.core.stored().data(),
                        m.core.stored().size() * sizeof(double));
  if (factors)
    for (std::size_t n = 0; n < m.factors.size(); ++n)
      std::memcpy(factors[n], m.factors[n].data().data(),
                  m.factors[n].data().size() * sizeof(double));
  if (couplings)
    for (std::size_t c = 0; c < m.couplings.size(); ++c)
      std::memcpy(couplings[c], m.couplings[c].factor.data().data(),
                  m.couplings[c].factor.data().size() * sizeof(double));
}

static void copy_model_in(FactorModel& m, const double* core,
                          const double* const* factors,
                          const double* const* couplings) {
  if (core) std::memcpy(m.core.stored().data(), core,
                        m.core.stored().size() * sizeof(double));
  if (factors)
    for (std::size_t n = 0; n < m.factors.size(); ++n)
      std::memcpy(m.factors[n].data().data(), factors[n],
                  m.factors[n].data().size() * sizeof(double));
  if (couplings)
    for (std::size_t c = 0; c < m.couplings.size(); ++c)
      std::memcpy(m.couplings[c].factor.data().data(), couplings[c],
                  m.couplings[c].factor.data().size() * sizeof(double));
}

void ref_state_get_model(void* state, double* core, double* const* factors,
                         double* const* couplings) {
  copy_model_out(static_cast<TrainState*>(state)->model, core, factors,
                 couplings);
}

void ref_state_set_model(void* state, const double* core,
                         const double* const* factors,
                         const double* const* couplings) {
  copy_model_in(static_cast<TrainState*>(state)->model, core, factors,
                couplings);
}

void ref_state_info(void* state, int32_t* epoch, double* eta) {
  auto* s = static_cast<TrainState*>(state);
  *epoch = s->epoch;
  *eta = s->eta;
}

void ref_state_get_schedule(void* state, uint64_t* out) {
  auto* s = static_cast<TrainState*>(state);
  std::memcpy(out, s->schedule.data(), s->schedule.size() * sizeof(uint64_t));
}

void ref_epoch_stats(void* state, void* bundle, double lambda_reg,
                     int32_t threads, double* rmse, double* objective) {
  EpochStats st = epoch_stats(static_cast<TrainState*>(state)->model,
                              *static_cast<DataBundle*>(bundle), lambda_reg,
                              threads);
  *rmse = st.train_rmse;
  *objective = st.objective;
}

int ref_test_rmse(void* state, int32_t order, const uint32_t* dims,
                  uint64_t nnz, const uint32_t* idx, const double* vals,
                  int32_t threads, double* out) {
  try {
    SparseTensor t(std::vector<uint32_t>(dims, dims + order),
                   std::vector<uint32_t>(idx, idx + nnz * order),
                   std::vector<double>(vals, vals + nnz));
    *out = test_rmse(static_cast<TrainState*>(state)->model, t, threads);
    return 0;
  } catch (const std::exception& e) {
    return fail(e, 1);
  }
}

// The tail of train() (src/trainer.cpp:342-345) applied in place to the
// state's model: apply_nonnegative_projection when nonneg, else
// finalize_orthogonalize (QR through oracle/eigen_shim).
int ref_state_finalize(void* state, int32_t nonneg) {
  try {
    FactorModel& m = static_cast<TrainState*>(state)->model;
    if (nonneg)
      apply_nonnegative_projection(m);
    else
      finalize_orthogonalize(m);
    return 0;
  } catch (const std::exception& e) {
    return fail(e, 1);
  }
}

// train(): convergence loop + finalization. log holds 4 doubles per epoch
// (epoch, train_rmse, objective, seconds).
int ref_train(void* bundle, const ref_config* c, double* core,
              double* const* factors, double* const* couplings, double* log,
              int32_t* n_log) {
  try {
    TrainResult r = train(*static_cast<DataBundle*>(bundle), to_config(c));
    copy_model_out(r.model, core, factors, couplings);
    *n_log = static_cast<int32_t>(r.log.size());
    for (std::size_t i = 0; i < r.log.size(); ++i) {
      log[4 * i + 0] = r.log[i].epoch;
      log[4 * i + 1] = r.log[i].train_rmse;
      log[4 * i + 2] = r.log[i].objective;
      log[4 * i + 3] = r.log[i].seconds;
    }
    return 0;
  } catch (const DivergenceError& e) {
    return fail(e, 2);
  } catch (const std::exception& e) {
    return fail(e, 1);
  }
}

int ref_compute_gradient(int32_t opt, double x, int32_t order,
                         const uint32_t* ranks, int32_t cp, const double* core,
                         const double* const* rows, double lambda_reg,
                         const uint32_t* counts, uint64_t nnz_total,
                         int32_t with_core, double* grow, double* gcore,
                         double* residual) {
  try {
    std::vector<uint32_t> rk(ranks, ranks + order);
    std::size_t stored = 1;
    for (auto j : rk) stored *= j;
    if (cp) stored = rk[0];
    CoreTensor g(rk, cp ? CoreStructure::HyperDiagonalCp
                        : CoreStructure::DenseTucker,
                 std::vector<double>(core, core + stored));
    KernelWorkspace ws(g);
    std::span<const double* const> r(rows, order);
    std::span<const uint32_t> cn(counts, order);
    if (opt)
      compute_gradient_opt(x, g, r, lambda_reg, cn, nnz_total, ws,
                           with_core != 0);
    else
      compute_gradient(x, g, r, lambda_reg, cn, nnz_total, ws, with_core != 0);
    double* out = grow;
    for (int n = 0; n < order; ++n) {
      std::memcpy(out, ws.grad.rows[n].data(), ranks[n] * sizeof(double));
      out += ranks[n];
    }
    if (with_core)
      std::memcpy(gcore, ws.grad.core.data(), stored * sizeof(double));
    *residual = ws.grad.residual;
    return 0;
  } catch (const std::exception& e) {
    return fail(e, 1);
  }
}

void ref_matrix_entry_gradients(double y, const double* u, const double* v,
                                uint32_t j, double lambda_m, double lambda_reg,
                                uint32_t col_count, double* du, double* dv,
                                double* residual) {
  MatrixEntryGradient g;
  matrix_entry_gradients(y, {u, j}, {v, j}, lambda_m, lambda_reg, col_count, g);
  std::memcpy(du, g.du.data(), j * sizeof(double));
  std::memcpy(dv, g.dv.data(), j * sizeof(double));
  *residual = g.residual;
}

void ref_shuffle(uint64_t* s, uint64_t n, uint64_t seed, int32_t epoch) {
  std::vector<uint64_t> v(s, s + n);
  shuffle_schedule(v, seed, epoch);
  std::memcpy(s, v.data(), n * sizeof(uint64_t));
}

// split_train_test: writes train then test entries (idx AoS + vals).
int ref_split(int32_t order, const uint32_t* dims, uint64_t nnz,
              const uint32_t* idx, const double* vals, double frac,
              uint64_t seed, uint32_t* train_idx, double* train_vals,
              uint32_t* test_idx, double* test_vals, uint64_t* n_test) {
  try {
    SparseTensor t(std::vector<uint32_t>(dims, dims + order),
                   std::vector<uint32_t>(idx, idx + nnz * order),
                   std::vector<double>(vals, vals + nnz));
    auto [tr, te] = split_train_test(t, frac, seed);
    std::memcpy(train_idx, tr.indices().data(),
                tr.indices().size() * sizeof(uint32_t));
    std::memcpy(train_vals, tr.values().data(), tr.nnz() * sizeof(double));
    std::memcpy(test_idx, te.indices().data(),
                te.indices().size() * sizeof(uint32_t));
    std::memcpy(test_vals, te.values().data(), te.nnz() * sizeof(double));
    *n_test = te.nnz();
    return 0;
  } catch (const std::exception& e) {
    return fail(e, 1);
  }
}

// The reference's own planted-model generator (src/synth.cpp:100-171).
// Returns a bundle; tensor/matrix arrays are copied out by ref_bundle_get.
void* ref_generate(int32_t order, const uint32_t* dims, uint64_t n_entries,
                   const uint32_t* ranks, double noise, uint64_t seed,
                   int32_t with_matrix, double matrix_ratio,
                   int32_t coupled_mode, uint32_t matrix_cols,
                   double matrix_weight) {
  try {
    SynthSpec s;
    s.dims.assign(dims, dims + order);
    s.n_entries = n_entries;
    s.ranks.assign(ranks, ranks + order);
    s.noise_stddev = noise;
    s.seed = seed;
    s.with_matrix = with_matrix != 0;
    s.matrix_ratio = matrix_ratio;
    s.coupled_mode = coupled_mode;
    s.matrix_cols = matrix_cols;
    s.matrix_weight = matrix_weight;
    return new DataBundle(generate(s).bundle);
  } catch (const std::exception& e) {
    fail(e, 1);
    return nullptr;
  }
}

void ref_bundle_sizes(void* bundle, uint64_t* nnz, int32_t* n_mat,
                      uint64_t* mat_nnz, uint32_t* mat_cols) {
  auto* b = static_cast<DataBundle*>(bundle);
  *nnz = b->tensor.nnz();
  *n_mat = static_cast<int32_t>(b->matrices.size());
  for (std::size_t m = 0; m < b->matrices.size(); ++m) {
    if (mat_nnz) mat_nnz[m] = b->matrices[m].nnz();
    if (mat_cols) mat_cols[m] = b->matrices[m].cols();
  }
}

void ref_bundle_get(void* bundle, uint32_t* idx, double* vals,
                    uint32_t* const* mat_idx, double* const* mat_vals) {
  auto* b = static_cast<DataBundle*>(bundle);
  std::memcpy(idx, b->tensor.indices().data(),
              b->tensor.indices().size() * sizeof(uint32_t));
  std::memcpy(vals, b->tensor.values().data(),
              b->tensor.nnz() * sizeof(double));
  for (std::size_t m = 0; m < b->matrices.size(); ++m) {
    if (mat_idx)
      std::memcpy(mat_idx[m], b->matrices[m].indices().data(),
                  b->matrices[m].indices().size() * sizeof(uint32_t));
    if (mat_vals)
      std::memcpy(mat_vals[m], b->matrices[m].values().data(),
                  b->matrices[m].nnz() * sizeof(double));
  }
}

// ---- text formats (src/sparse_data.cpp:124-311, src/model_io.cpp) ----
// error code: 1 ParseError, 2 ValidationError, 3 anything else
static int classify(const std::exception& e) {
  if (dynamic_cast<const ParseError*>(&e)) return 1;
  if (dynamic_cast<const ValidationError*>(&e)) return 2;
  return 3;
}

void* ref_load_tensor(const char* path, int32_t* code) {
  try {
    *code = 0;
    return new SparseTensor(load_tensor(path));
  } catch (const std::exception& e) {
    *code = fail(e, classify(e));
    return nullptr;
  }
}

void* ref_load_matrix(const char* path, int32_t coupled_mode, double weight, int32_t order,
                      const uint32_t* dims, int32_t* code) {
  try {
    *code = 0;
    SparseTensor t(std::vector<uint32_t>(dims, dims + order), {}, {});
    return new CoupledMatrix(load_matrix(path, coupled_mode, weight, t));
  } catch (const std::exception& e) {
    *code = fail(e, classify(e));
    return nullptr;
  }
}

void ref_coo_info(void* obj, int32_t is_matrix, int32_t* order, uint32_t* dims, uint64_t* nnz) {
  if (is_matrix) {
    auto* m = static_cast<CoupledMatrix*>(obj);
    *order = 2;
    dims[0] = m->rows();
    dims[1] = m->cols();
    *nnz = m->nnz();
  } else {
    auto* t = static_cast<SparseTensor*>(obj);
    *order = t->order();
    for (int n = 0; n < t->order(); ++n) dims[n] = t->dims()[n];
    *nnz = t->nnz();
  }
}

void ref_coo_get(void* obj, int32_t is_matrix, uint32_t* idx, double* vals) {
  const std::vector<uint32_t>& i = is_matrix ? static_cast<CoupledMatrix*>(obj)->indices()
                                             : static_cast<SparseTensor*>(obj)->indices();
  const std::vector<double>& v = is_matrix ? static_cast<CoupledMatrix*>(obj)->values()
                                           : static_cast<SparseTensor*>(obj)->values();
  std::memcpy(idx, i.data(), i.size() * sizeof(uint32_t));
  std::memcpy(vals, v.data(), v.size() * sizeof(double));
}

void ref_coo_free(void* obj, int32_t is_matrix) {
  if (is_matrix) delete static_cast<CoupledMatrix*>(obj);
  else delete static_cast<SparseTensor*>(obj);
}

int ref_save_tensor(const char* path, int32_t order, const uint32_t* dims, uint64_t nnz,
                    const uint32_t* idx, const double* vals) {
  try {
    SparseTensor t(std::vector<uint32_t>(dims, dims + order),
                   std::vector<uint32_t>(idx, idx + nnz * order),
                   std::vector<double>(vals, vals + nnz));
    save_tensor(path, t);
    return 0;
  } catch (const std::exception& e) {
    return fail(e, classify(e));
  }
}

// load_model: 0 ok (ranks / number of factors / couplings returned), else the
// error class with the message in ref_last_error()
int ref_load_model(const char* path, int32_t* order, int32_t* n_factors, int32_t* n_coupled) {
  try {
    FactorModel m = load_model(path);
    *order = m.core.order();
    *n_factors = (int32_t)m.factors.size();
    *n_coupled = (int32_t)m.couplings.size();
    return 0;
  } catch (const std::exception& e) {
    return fail(e, classify(e));
  }
}

int ref_save_model(const char* path, int32_t order, const uint32_t* ranks, int32_t cp,
                   const double* core, const uint32_t* factor_rows, const double* const* factors,
                   int32_t n_coupled, const int32_t* coupled_modes, const uint32_t* coupled_rows,
                   const double* const* couplings) {
  try {
    std::vector<uint32_t> rk(ranks, ranks + order);
    size_t cs = 1;
    for (auto j : rk) cs *= j;
    const size_t stored = cp ? rk[0] : cs;
    FactorModel m{CoreTensor(rk, cp ? CoreStructure::HyperDiagonalCp : CoreStructure::DenseTucker,
                             std::vector<double>(core, core + stored)),
                  {}, {}};
    for (int n = 0; n < order; ++n)
      m.factors.emplace_back(factor_rows[n], rk[n],
                             std::vector<double>(factors[n], factors[n] + (size_t)factor_rows[n] * rk[n]));
    for (int c = 0; c < n_coupled; ++c) {
      const uint32_t J = rk[coupled_modes[c]];
      m.couplings.push_back(Coupling{coupled_modes[c],
                                     FactorMatrix(coupled_rows[c], J,
                                                  std::vector<double>(couplings[c],
                                                                      couplings[c] + (size_t)coupled_rows[c] * J))});
    }
    save_model(path, m);
    return 0;
  } catch (const std::exception& e) {
    return fail(e, classify(e));
  }
}

}  // extern "C"
