// cmtf_core_b200.cpp -- source-level drop-in for the reference's hot-path
// translation units.
//
// Compiled against the reference's own public headers (cmtf/trainer.hpp,
// eval.hpp, gradients.hpp of CMake package cmtf::core), this file defines
// every function those headers declare for the training path, on top of the
// B200 library's C ABI (include/cmtf_b200.h).  A reference build links it
// INSTEAD OF src/gradients.cpp, src/eval.cpp and src/trainer.cpp (keeping
// the data-structure / IO units: sparse_data.cpp, tucker.cpp, rng.cpp,
// model_io.cpp, synth.cpp) plus libcmtf_b200.so; callers -- cmd_train,
// bench_epoch, the reference's own unit tests -- recompile unchanged.
//
// Semantics:
//  * run_epoch: one device epoch on the state's bundle.  workers == 1
//    replays the state's own shuffled schedule exactly (serial mode, the
//    schedule is shuffled here with the reference's stream and handed to the
//    device); workers > 1 runs the lock-free device epoch.  The host
//    TrainState::model stays the f64 master copy: the device runs in fp32 on
//    f32(master) and the epoch's change, taken exactly as f32 differences,
//    is added to the master (a zero step leaves the model bit-identical).
//  * compute_gradient[_opt], matrix_entry_gradients, collapse: the library's
//    stateless f64 device kernels.
//  * epoch_stats / test_rmse / matrix_rmse / objective_value / evaluate:
//    the device evaluation pass (fp32 model, f64 accumulation in the
//    reference's 1024-entry blocks).
//  * initialize / random_model / schedule helpers / finalisation tail:
//    host, the reference's draw law and streams (the initial model is the
//    reference's, bit for bit).
// Device contexts are cached per TrainState / bundle (a few at a time,
// least-recently used evicted); an evicted state is rebuilt from the host
// master copy, so eviction never changes results.
#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <mutex>
#include <ostream>
#include <string>
#include <vector>

#include "cmtf/errors.hpp"
#include "cmtf/eval.hpp"
#include "cmtf/gradients.hpp"
#include "cmtf/rng.hpp"
#include "cmtf/trainer.hpp"
#include "cmtf/tucker.hpp"
#include "cmtf_b200.h"

namespace cmtf {

namespace {

int device_ordinal() {
  const char* v = std::getenv("CMTF_DEVICE");
  return v ? std::atoi(v) : 0;
}

[[noreturn]] void raise(int rc, const std::string& msg) {
  switch (rc) {
    case CMTF_EVALIDATION:
    case CMTF_EUNSUPPORTED:
      throw ValidationError(msg);
    case CMTF_EDIVERGENCE:
      throw DivergenceError(msg);
    case CMTF_EPARSE:
      throw ParseError(msg);
    default:
      throw std::runtime_error(msg);
  }
}
void check(int rc, const cmtf_gpu_ctx* ctx = nullptr) {
  if (rc == CMTF_OK) return;
  raise(rc, ctx ? cmtf_gpu_ctx_error(ctx) : cmtf_gpu_last_error());
}

// ---- device contexts, cached per key (a TrainState, or an evaluation's data)
struct Slot {
  const void* key = nullptr;
  cmtf_gpu_ctx* ctx = nullptr;
  uint64_t data = 0;  // fingerprint of what was uploaded
  std::vector<std::uint32_t> ranks;
  int cp = 0, exec = 0, kernel = 0;
  std::uint64_t tick = 0;
};
std::mutex g_mu;
std::vector<Slot> g_slots;
std::uint64_t g_tick = 0;
constexpr std::size_t kMaxSlots = 4;

std::size_t matrix_nnz(const std::vector<CoupledMatrix>& ms) {
  std::size_t t = 0;
  for (const auto& m : ms) t += m.nnz();
  return t;
}

void upload_tensor(cmtf_gpu_ctx* ctx, const SparseTensor& t) {
  check(cmtf_gpu_set_tensor(ctx, t.dims().data(), t.indices().data(), t.values().data(),
                            t.nnz()),
        ctx);
}
void upload_matrices(cmtf_gpu_ctx* ctx, const std::vector<CoupledMatrix>& ms) {
  check(cmtf_gpu_clear_matrices(ctx), ctx);
  for (const auto& m : ms)
    check(cmtf_gpu_add_matrix(ctx, m.coupled_mode(), m.rows(), m.cols(), m.indices().data(),
                              m.values().data(), m.nnz(), m.weight()),
          ctx);
}

cmtf_gpu_config base_config(const std::vector<std::uint32_t>& ranks, int cp) {
  cmtf_gpu_config c;
  cmtf_gpu_config_default(&c);
  c.order = static_cast<int32_t>(ranks.size());
  c.ranks = ranks.data();
  c.core_structure = cp;
  c.device = device_ordinal();
  return c;
}

// Find or create the context for `key`; `fresh` tells the caller it must
// (re)upload data and model.
cmtf_gpu_ctx* acquire(const void* key, const std::vector<std::uint32_t>& ranks, int cp, int exec,
                      int kernel, const cmtf_gpu_config& cfg, bool* fresh) {
  std::lock_guard<std::mutex> lock(g_mu);
  for (auto& s : g_slots)
    if (s.key == key && s.ranks == ranks && s.cp == cp && s.exec == exec && s.kernel == kernel) {
      s.tick = ++g_tick;
      *fresh = false;
      return s.ctx;
    }
  for (auto it = g_slots.begin(); it != g_slots.end(); ++it)
    if (it->key == key) {  // same key, different shape: replace
      cmtf_gpu_destroy(it->ctx);
      g_slots.erase(it);
      break;
    }
  if (g_slots.size() >= kMaxSlots) {
    auto lru = std::min_element(g_slots.begin(), g_slots.end(),
                                [](const Slot& a, const Slot& b) { return a.tick < b.tick; });
    cmtf_gpu_destroy(lru->ctx);
    g_slots.erase(lru);
  }
  cmtf_gpu_ctx* ctx = nullptr;
  check(cmtf_gpu_create(&cfg, &ctx));
  Slot s;
  s.key = key;
  s.ctx = ctx;
  s.ranks = ranks;
  s.cp = cp;
  s.exec = exec;
  s.kernel = kernel;
  s.tick = ++g_tick;
  g_slots.push_back(s);
  *fresh = true;
  return ctx;
}
Slot* slot_of(cmtf_gpu_ctx* ctx) {
  for (auto& s : g_slots)
    if (s.ctx == ctx) return &s;
  return nullptr;
}

// model transfer: the core's stored values, factors / couplings row-major
void put_model(cmtf_gpu_ctx* ctx, const FactorModel& m) {
  std::vector<const double*> f, v;
  for (const auto& x : m.factors) f.push_back(x.data().data());
  for (const auto& c : m.couplings) v.push_back(c.factor.data().data());
  check(cmtf_gpu_set_model(ctx, m.core.stored().data(), f.data(), v.empty() ? nullptr : v.data()),
        ctx);
}
void get_model(cmtf_gpu_ctx* ctx, FactorModel& m) {
  std::vector<double*> f, v;
  for (auto& x : m.factors) f.push_back(x.data().data());
  for (auto& c : m.couplings) v.push_back(c.factor.data().data());
  check(cmtf_gpu_get_model(ctx, m.core.stored().data(), f.data(), v.empty() ? nullptr : v.data()),
        ctx);
}
// master += (after - f32(master)), elementwise: the device's fp32 step
// applied to the f64 master copy (exactly zero where nothing changed)
void apply_step(std::span<double> master, std::span<const double> after) {
  for (std::size_t i = 0; i < master.size(); ++i)
    master[i] += after[i] - static_cast<double>(static_cast<float>(master[i]));
}

int exec_of(const TrainConfig& c) { return c.workers == 1 ? CMTF_EXEC_SERIAL : CMTF_EXEC_HOGWILD; }

cmtf_gpu_config train_config(const TrainConfig& c) {
  cmtf_gpu_config g = base_config(c.ranks, c.core_structure == CoreStructure::HyperDiagonalCp);
  g.eta0 = c.eta0;
  g.mu = c.mu;
  g.lambda_reg = c.lambda_reg;
  g.workers = c.workers;
  g.max_epochs = c.max_epochs;
  g.rel_tol = c.rel_tol;
  g.seed = c.seed;
  g.kernel = c.kernel == GradientKernel::Naive ? CMTF_KERNEL_NAIVE : CMTF_KERNEL_OPT;
  g.nonnegative = c.nonnegative;
  g.init_scale = c.init_scale;
  g.exec_mode = exec_of(c);
  g.debug_count_visits = c.debug_count_visits;
  return g;
}

// An evaluation context per model shape; the data and the model are
// uploaded on every call (a caller's objects may reuse addresses)
cmtf_gpu_ctx* eval_ctx(const FactorModel& model, const SparseTensor* tensor,
                       const std::vector<CoupledMatrix>* mats) {
  std::vector<std::uint32_t> ranks(model.core.ranks().begin(), model.core.ranks().end());
  const int cp = model.core.structure() == CoreStructure::HyperDiagonalCp;
  cmtf_gpu_config cfg = base_config(ranks, cp);
  cfg.nonnegative = 1;  // evaluation only: no orthogonalisation shape checks
  bool fresh = false;
  static const char eval_key = 0;
  cmtf_gpu_ctx* ctx = acquire(&eval_key, ranks, cp, -1, -1, cfg, &fresh);
  upload_tensor(ctx, *tensor);
  upload_matrices(ctx, mats ? *mats : std::vector<CoupledMatrix>{});
  return ctx;
}

// A cheap identity of a bundle's content (sizes, dims and a strided sample
// of entries): a TrainState's cached context is re-uploaded when it changes
uint64_t fingerprint(const DataBundle& b) {
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](uint64_t v) { h = (h ^ v) * 1099511628211ull; };
  const SparseTensor& t = b.tensor;
  mix(t.nnz());
  for (auto d : t.dims()) mix(d);
  const std::size_t step = std::max<std::size_t>(1, t.nnz() / 4096);
  for (std::size_t e = 0; e < t.nnz(); e += step) {
    for (auto i : t.index(e)) mix(i);
    uint64_t bits;
    const double v = t.value(e);
    std::memcpy(&bits, &v, 8);
    mix(bits);
  }
  for (const auto& m : b.matrices) {
    mix(m.nnz());
    mix(m.rows());
    mix(m.cols());
    const std::size_t ms = std::max<std::size_t>(1, m.nnz() / 1024);
    for (std::size_t e = 0; e < m.nnz(); e += ms) {
      mix(m.row_index(e));
      mix(m.col_index(e));
      uint64_t bits;
      const double v = m.value(e);
      std::memcpy(&bits, &v, 8);
      mix(bits);
    }
  }
  return h;
}

}  // namespace

// ======================================================================
// gradients.hpp
// ======================================================================

IntermediateTensor::IntermediateTensor(const CoreTensor& core)
    : ranks_(core.ranks()),
      structure_(core.structure()),
      strides_(core.strides()),
      values_(core.stored().size(), 0.0) {}

void collapse(const IntermediateTensor& s, int mode, std::span<double> out) {
  const auto& ranks = s.ranks();
  if (mode < 0 || mode >= static_cast<int>(ranks.size()))
    throw ValidationError("collapse mode out of range");
  if (out.size() != ranks[mode]) throw ValidationError("collapse output length mismatch");
  check(cmtf_gpu_collapse(static_cast<int32_t>(ranks.size()), ranks.data(),
                          s.structure() == CoreStructure::HyperDiagonalCp, s.values().data(),
                          mode, out.data(), device_ordinal()));
}

EntryGradient::EntryGradient(const CoreTensor& core) : core(core.stored().size(), 0.0) {
  for (std::uint32_t j : core.ranks()) rows.emplace_back(j, 0.0);
}

KernelWorkspace::KernelWorkspace(const CoreTensor& core) : grad(core), s(core) {
  contract_buf.resize(*std::max_element(core.ranks().begin(), core.ranks().end()));
}

namespace {
void kernel_call(int kernel, double x, const CoreTensor& core, std::span<const double* const> rows,
                 double lambda_reg, std::span<const std::uint32_t> counts, std::uint64_t nnz_total,
                 KernelWorkspace& ws, bool with_core) {
  const auto& ranks = core.ranks();
  if (rows.size() != ranks.size() || counts.size() != ranks.size())
    throw ValidationError("kernel argument order mismatch");
  std::vector<double> flat;
  for (std::size_t n = 0; n < ranks.size(); ++n) flat.insert(flat.end(), rows[n], rows[n] + ranks[n]);
  std::vector<double> grow(flat.size());
  double r = 0.0;
  const bool cp = core.structure() == CoreStructure::HyperDiagonalCp;
  check(cmtf_gpu_compute_gradient(kernel, static_cast<int32_t>(ranks.size()), ranks.data(), cp,
                                  core.stored().data(), 1, &x, flat.data(), counts.data(),
                                  lambda_reg, nnz_total, with_core, grow.data(),
                                  with_core ? ws.grad.core.data() : nullptr, &r,
                                  kernel == CMTF_KERNEL_OPT ? ws.s.values().data() : nullptr,
                                  device_ordinal()));
  ws.grad.residual = r;
  std::size_t o = 0;
  for (std::size_t n = 0; n < ranks.size(); ++n)
    for (std::uint32_t k = 0; k < ranks[n]; ++k) ws.grad.rows[n][k] = grow[o++];
}
}  // namespace

void compute_gradient(double x, const CoreTensor& core, std::span<const double* const> rows,
                      double lambda_reg, std::span<const std::uint32_t> mode_counts,
                      std::uint64_t nnz_total, KernelWorkspace& ws, bool with_core_grad) {
  kernel_call(CMTF_KERNEL_NAIVE, x, core, rows, lambda_reg, mode_counts, nnz_total, ws,
              with_core_grad);
}

void compute_gradient_opt(double x, const CoreTensor& core, std::span<const double* const> rows,
                          double lambda_reg, std::span<const std::uint32_t> mode_counts,
                          std::uint64_t nnz_total, KernelWorkspace& ws, bool with_core_grad) {
  kernel_call(CMTF_KERNEL_OPT, x, core, rows, lambda_reg, mode_counts, nnz_total, ws,
              with_core_grad);
}

void matrix_entry_gradients(double y, std::span<const double> u_row,
                            std::span<const double> v_row, double lambda_m, double lambda_reg,
                            std::uint32_t col_count, MatrixEntryGradient& out) {
  if (u_row.size() != v_row.size())
    throw ValidationError("coupled rows must have equal length");
  out.du.assign(u_row.size(), 0.0);
  out.dv.assign(v_row.size(), 0.0);
  check(cmtf_gpu_matrix_entry_gradients(1, static_cast<uint32_t>(u_row.size()), &y, u_row.data(),
                                        v_row.data(), lambda_m, lambda_reg, &col_count,
                                        out.du.data(), out.dv.data(), &out.residual,
                                        device_ordinal()));
}

// ======================================================================
// eval.hpp
// ======================================================================

EpochStats epoch_stats(const FactorModel& model, const DataBundle& bundle, double lambda_reg,
                       int /*n_threads: the device pass is deterministic*/) {
  if (bundle.tensor.nnz() == 0) {
    // no training entries (the device bundle needs one): the regulariser of
    // the core and the coupled matrices' terms (src/eval.cpp:120-144)
    EpochStats st;
    double core_sq = 0.0;
    for (double g : model.core.stored()) core_sq += g * g;
    st.objective = 0.5 * lambda_reg * core_sq;
    for (std::size_t m = 0; m < bundle.matrices.size(); ++m) {
      const CoupledMatrix& mat = bundle.matrices[m];
      double f_m = 0.0;
      if (mat.nnz()) {
        const double r = matrix_rmse(model, mat, m, 1);
        f_m = r * r * static_cast<double>(mat.nnz());
      }
      const auto& cnt = bundle.counts.matrix_cols[m];
      const FactorMatrix& v = model.couplings[m].factor;
      for (std::uint32_t j = 0; j < v.rows(); ++j)
        if (cnt[j])
          for (double x : v.row(j)) f_m += lambda_reg * x * x;
      st.objective += 0.5 * mat.weight() * f_m;
    }
    return st;
  }
  cmtf_gpu_ctx* ctx = eval_ctx(model, &bundle.tensor, &bundle.matrices);
  put_model(ctx, model);
  EpochStats st;
  check(cmtf_gpu_epoch_stats(ctx, lambda_reg, &st.train_rmse, &st.objective), ctx);
  return st;
}

double test_rmse(const FactorModel& model, const SparseTensor& tensor, int n_threads) {
  if (tensor.nnz() == 0) throw ValidationError("cannot evaluate an empty tensor");
  cmtf_gpu_ctx* ctx = eval_ctx(model, &tensor, nullptr);
  FactorModel bare{model.core, model.factors, {}};
  put_model(ctx, bare);
  EpochStats st;
  check(cmtf_gpu_epoch_stats(ctx, 0.0, &st.train_rmse, &st.objective), ctx);
  (void)n_threads;
  return st.train_rmse;
}

double matrix_rmse(const FactorModel& model, const CoupledMatrix& matrix,
                   std::size_t coupling_index, int /*n_threads*/) {
  if (matrix.nnz() == 0) throw ValidationError("cannot evaluate an empty matrix");
  if (coupling_index >= model.couplings.size() ||
      matrix.coupled_mode() >= static_cast<int>(model.factors.size()))
    throw ValidationError("no coupled factor for this matrix");
  // a one-entry placeholder tensor over the model's mode sizes carries the
  // matrix's row space
  const int order = static_cast<int>(model.factors.size());
  std::vector<std::uint32_t> dims;
  for (const auto& f : model.factors) dims.push_back(f.rows());
  static thread_local std::vector<SparseTensor> holder;
  holder.clear();
  holder.emplace_back(dims, std::vector<std::uint32_t>(order, 0u), std::vector<double>{0.0});
  std::vector<CoupledMatrix> one{matrix};
  cmtf_gpu_ctx* ctx = eval_ctx(model, &holder[0], &one);
  FactorModel m{model.core, model.factors, {model.couplings[coupling_index]}};
  put_model(ctx, m);
  double r = 0.0;
  check(cmtf_gpu_matrix_rmse(ctx, 0, &r), ctx);
  return r;
}

double objective_value(const FactorModel& model, const DataBundle& bundle, double lambda_reg,
                       int n_threads) {
  if (model.couplings.size() != bundle.matrices.size())
    throw ValidationError("model has " + std::to_string(model.couplings.size()) +
                          " coupled factors for " + std::to_string(bundle.matrices.size()) +
                          " matrices");
  return epoch_stats(model, bundle, lambda_reg, n_threads).objective;
}

EvalReport evaluate(const FactorModel& model, const SparseTensor& test,
                    const std::vector<CoupledMatrix>& matrices, int n_threads) {
  EvalReport report;
  report.test_rmse = test_rmse(model, test, n_threads);
  report.n_entries = test.nnz();
  for (std::size_t m = 0; m < matrices.size(); ++m)
    report.matrix_rmse.push_back(matrix_rmse(model, matrices[m], m, n_threads));
  return report;
}

// ======================================================================
// trainer.hpp
// ======================================================================

void write_log_csv(std::ostream& out, const ConvergenceLog& log) {
  out << "epoch,train_rmse,objective,seconds\n";
  for (const auto& e : log) {
    char line[160];
    std::snprintf(line, sizeof line, "%d,%.17g,%.17g,%.6f\n", e.epoch, e.train_rmse, e.objective,
                  e.seconds);
    out << line;
  }
}

FactorModel random_model(std::span<const std::uint32_t> dims,
                         std::span<const std::uint32_t> ranks, CoreStructure structure,
                         const std::vector<std::pair<int, std::uint32_t>>& coupling_shapes,
                         double scale, std::mt19937_64& rng) {
  // draw order: core (its stored values), factors by mode, couplings
  CoreTensor core = CoreTensor::zeros(std::vector<std::uint32_t>(ranks.begin(), ranks.end()),
                                      structure);
  for (double& g : core.stored()) g = uniform(rng, 0.0, scale);
  std::vector<FactorMatrix> factors;
  for (std::size_t n = 0; n < dims.size(); ++n) {
    FactorMatrix f = FactorMatrix::zeros(dims[n], ranks[n]);
    const double top = scale / std::sqrt(static_cast<double>(ranks[n]));
    for (double& v : f.data()) v = uniform(rng, 0.0, top);
    factors.push_back(std::move(f));
  }
  std::vector<Coupling> couplings;
  for (const auto& [mode, cols] : coupling_shapes) {
    FactorMatrix f = FactorMatrix::zeros(cols, ranks[mode]);
    const double top = scale / std::sqrt(static_cast<double>(ranks[mode]));
    for (double& v : f.data()) v = uniform(rng, 0.0, top);
    couplings.push_back(Coupling{mode, std::move(f)});
  }
  return FactorModel{std::move(core), std::move(factors), std::move(couplings)};
}

void validate_config(const TrainConfig& config, const DataBundle& bundle) {
  // the rank count is checked here (the device library sees only the ranks);
  // every other rule is the device library's own validation, same messages
  const auto& dims = bundle.tensor.dims();
  if (config.ranks.size() != dims.size())
    throw ValidationError("rank list has " + std::to_string(config.ranks.size()) +
                          " entries for a tensor of order " + std::to_string(dims.size()));
  for (std::uint32_t j : config.ranks)
    if (j == 0) throw ValidationError("ranks must be positive");
  if (config.core_structure == CoreStructure::HyperDiagonalCp)
    for (std::uint32_t j : config.ranks)
      if (j != config.ranks[0]) throw ValidationError("CP mode requires equal ranks on every mode");
  if (!config.nonnegative)
    for (std::size_t n = 0; n < dims.size(); ++n)
      if (config.ranks[n] > dims[n])
        throw ValidationError("rank of mode " + std::to_string(n + 1) +
                              " exceeds its size; orthogonalization needs J_n <= I_n");
  if (bundle.tensor.nnz() == 0) throw ValidationError("training tensor has no entries");
  cmtf_gpu_config g = train_config(config);
  // the remaining scalar rules (eta0, mu, lambda, workers, epochs, tol, scale)
  cmtf_gpu_ctx* probe = nullptr;
  const int rc = cmtf_gpu_create(&g, &probe);
  if (rc == CMTF_OK) cmtf_gpu_destroy(probe);
  else if (rc == CMTF_EVALIDATION) raise(rc, cmtf_gpu_last_error());
}

FactorModel initialize(const TrainConfig& config, const DataBundle& bundle) {
  validate_config(config, bundle);
  std::vector<std::pair<int, std::uint32_t>> shapes;
  for (const auto& m : bundle.matrices) shapes.emplace_back(m.coupled_mode(), m.cols());
  auto rng = make_rng(config.seed, RngStream::Init);
  return random_model(bundle.tensor.dims(), config.ranks, config.core_structure, shapes,
                      config.init_scale, rng);
}

std::vector<std::pair<std::size_t, std::size_t>> worker_chunks(std::size_t n, int workers) {
  std::vector<std::pair<std::size_t, std::size_t>> out;
  for (int w = 0; w < workers; ++w) out.emplace_back(n * w / workers, n * (w + 1) / workers);
  return out;
}

std::vector<std::uint64_t> build_schedule(const DataBundle& bundle) {
  std::vector<std::uint64_t> s(bundle.tensor.nnz() + matrix_nnz(bundle.matrices));
  for (std::size_t i = 0; i < s.size(); ++i) s[i] = i;
  return s;
}

void shuffle_schedule(std::vector<std::uint64_t>& schedule, std::uint64_t seed, int epoch) {
  auto rng = make_rng(seed, RngStream::Shuffle, static_cast<std::uint64_t>(epoch));
  for (std::size_t i = schedule.size(); i > 1; --i)
    std::swap(schedule[i - 1], schedule[bounded(rng, i)]);
}

TrainState make_state(const TrainConfig& config, const DataBundle& bundle) {
  TrainState state{initialize(config, bundle), 0, config.eta0, {}, build_schedule(bundle), {}};
  if (config.debug_count_visits) state.visit_counts.assign(state.schedule.size(), 0);
  return state;
}

void run_epoch(TrainState& state, const DataBundle& bundle, const TrainConfig& config) {
  const std::size_t total = bundle.tensor.nnz() + matrix_nnz(bundle.matrices);
  if (state.schedule.size() != total) state.schedule = build_schedule(bundle);
  cmtf_gpu_config g = train_config(config);
  const int exec = exec_of(config);
  bool fresh = false;
  cmtf_gpu_ctx* ctx = acquire(&state, config.ranks, g.core_structure, exec, g.kernel, g, &fresh);
  Slot* s = slot_of(ctx);
  const uint64_t fp = fingerprint(bundle);
  if (fresh || s->data != fp) {
    upload_tensor(ctx, bundle.tensor);
    upload_matrices(ctx, bundle.matrices);
    s->data = fp;
  }
  put_model(ctx, state.model);
  check(cmtf_gpu_set_state(ctx, state.epoch, state.eta), ctx);
  if (exec == CMTF_EXEC_SERIAL) {
    // the reference's own visiting order: the persisted schedule, shuffled
    // with the epoch's stream (src/trainer.cpp:122-128)
    shuffle_schedule(state.schedule, config.seed, state.epoch);
    check(cmtf_gpu_set_schedule(ctx, state.schedule.data(), state.schedule.size()), ctx);
  }
  check(cmtf_gpu_run_epoch(ctx), ctx);
  FactorModel after = state.model;
  get_model(ctx, after);
  apply_step(state.model.core.stored(), after.core.stored());
  for (std::size_t n = 0; n < after.factors.size(); ++n)
    apply_step(state.model.factors[n].data(), after.factors[n].data());
  for (std::size_t m = 0; m < after.couplings.size(); ++m)
    apply_step(state.model.couplings[m].factor.data(), after.couplings[m].factor.data());
  state.epoch += 1;
  state.eta = config.eta0 / (1.0 + config.mu * state.epoch);
  if (config.debug_count_visits) {
    state.visit_counts.assign(total, 0);
    if (exec == CMTF_EXEC_SERIAL) {
      // one block replays the schedule: each id exactly as often as listed
      for (std::uint64_t id : state.schedule) state.visit_counts[id] += 1;
    } else {
      // tensor ids from the device counts; matrix entries per device record
      check(cmtf_gpu_visit_counts(ctx, state.visit_counts.data(),
                                  state.visit_counts.data() + bundle.tensor.nnz()),
            ctx);
    }
  }
}

void apply_nonnegative_projection(FactorModel& model) {
  // clamp, then unit columns with the norms absorbed into the core
  // (CP: its superdiagonal) and the coupled factors; predictions unchanged
  auto clamp = [](std::span<double> v) {
    for (double& x : v) x = x < 0 ? 0.0 : x;
  };
  clamp(model.core.stored());
  for (auto& f : model.factors) clamp(f.data());
  for (auto& c : model.couplings) clamp(c.factor.data());
  const bool cp = model.core.structure() == CoreStructure::HyperDiagonalCp;
  for (int n = 0; n < model.core.order(); ++n) {
    FactorMatrix& f = model.factors[n];
    for (std::uint32_t k = 0; k < f.cols(); ++k) {
      double sq = 0.0;
      for (std::uint32_t i = 0; i < f.rows(); ++i) sq += f.row(i)[k] * f.row(i)[k];
      if (sq == 0.0) continue;
      const double norm = std::sqrt(sq);
      for (std::uint32_t i = 0; i < f.rows(); ++i) f.row(i)[k] /= norm;
      if (cp) {
        model.core.stored()[k] *= norm;
      } else {
        const std::size_t stride = model.core.strides()[n];
        const std::size_t span = stride * model.core.ranks()[n];
        auto g = model.core.stored();
        for (std::size_t base = 0; base < g.size(); base += span)
          for (std::size_t t = 0; t < stride; ++t) g[base + k * stride + t] *= norm;
      }
      for (auto& c : model.couplings)
        if (c.mode == n)
          for (std::uint32_t i = 0; i < c.factor.rows(); ++i) c.factor.row(i)[k] *= norm;
    }
  }
}

TrainResult train(const DataBundle& bundle, const TrainConfig& config) {
  validate_config(config, bundle);
  TrainState state = make_state(config, bundle);
  const auto t0 = std::chrono::steady_clock::now();
  double prev = std::numeric_limits<double>::quiet_NaN();
  for (int ep = 0; ep < config.max_epochs; ++ep) {
    run_epoch(state, bundle, config);
    const EpochStats st = epoch_stats(state.model, bundle, config.lambda_reg, 1);
    const double sec =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    state.log.push_back({state.epoch, st.train_rmse, st.objective, sec});
    // convergence (src/trainer.cpp:335-337)
    if (std::isfinite(prev) && prev > 0 && std::abs(prev - st.train_rmse) / prev < config.rel_tol)
      break;
    prev = st.train_rmse;
  }
  if (config.nonnegative)
    apply_nonnegative_projection(state.model);
  else
    finalize_orthogonalize(state.model);
  {  // the state's contexts go with it
    std::lock_guard<std::mutex> lock(g_mu);
    for (auto it = g_slots.begin(); it != g_slots.end();)
      if (it->key == &state) {
        cmtf_gpu_destroy(it->ctx);
        it = g_slots.erase(it);
      } else {
        ++it;
      }
  }
  return TrainResult{std::move(state.model), std::move(state.log)};
}

}  // namespace cmtf
