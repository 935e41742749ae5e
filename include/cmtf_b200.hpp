// cmtf_b200.hpp -- header-only C++ layer over the C ABI (cmtf_b200.h) that
// rebuilds the reference's C++ entry points for the training path
// (namespace cmtf, /root/reference/proj/core/include/cmtf/{trainer,eval,
// gradients}.hpp) with the same names, argument meaning and exception types.
//
// A reference user keeps their DataBundle-building code and swaps
//     cmtf::run_epoch(state, bundle, config)
// for
//     cmtf::b200::run_epoch(state, bundle, config)
// where the b200::TrainState owns a device context.
// The bundle types here are plain structs with the reference's layout
// (sparse_data.hpp:17-84): u32 AoS indices, f64 values.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "cmtf_b200.h"

namespace cmtf {

#ifndef CMTF_ERRORS_DEFINED
#define CMTF_ERRORS_DEFINED
// errors.hpp:10-26 (defined here only if the reference header is not used)
class ParseError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class ValidationError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class DivergenceError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
#endif

namespace b200 {

class CudaError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

inline void check(int rc, const cmtf_gpu_ctx* ctx = nullptr) {
  if (rc == CMTF_OK) return;
  const std::string msg = ctx ? cmtf_gpu_ctx_error(ctx) : cmtf_gpu_last_error();
  switch (rc) {
    case CMTF_EVALIDATION:
    case CMTF_EUNSUPPORTED:
      throw ValidationError(msg);
    case CMTF_EDIVERGENCE:
      throw DivergenceError(msg);
    default:
      throw CudaError(msg);
  }
}

// SparseTensor / CoupledMatrix / DataBundle shapes (sparse_data.hpp:17-84).
struct SparseTensor {
  std::vector<uint32_t> dims;
  std::vector<uint32_t> indices;  // nnz * order, 0-based
  std::vector<double> values;
  std::size_t nnz() const { return values.size(); }
  int order() const { return static_cast<int>(dims.size()); }
};
struct CoupledMatrix {
  int coupled_mode;  // 0-based
  uint32_t rows, cols;
  std::vector<uint32_t> indices;  // nnz * 2
  std::vector<double> values;
  double weight;
  std::size_t nnz() const { return values.size(); }
};
struct DataBundle {
  SparseTensor tensor;
  std::vector<CoupledMatrix> matrices;
};

enum class GradientKernel { Naive, Opt };

// TrainConfig (trainer.hpp:18-36) + device fields.
struct TrainConfig {
  std::vector<uint32_t> ranks;
  double eta0 = 1e-3;
  double mu = 0.1;
  double lambda_reg = 0.1;
  int workers = 1;
  int max_epochs = 100;
  double rel_tol = 1e-4;
  uint64_t seed = 0;
  GradientKernel kernel = GradientKernel::Opt;
  bool nonnegative = false;
  double init_scale = 1.0;
  int device = 0;
  bool serial_parity = false;  // replay the reference schedule (P = 1)
  int hog_threads = 0;         // 0 = auto
};

struct FactorModel {
  std::vector<double> core;                  // row-major, last mode fastest
  std::vector<std::vector<double>> factors;  // I_n x J_n row-major
  std::vector<std::vector<double>> couplings;
};

struct EpochStats {
  double train_rmse = 0.0;
  double objective = 0.0;
};

// TrainState (trainer.hpp:49-56): owns the device context and the model.
class TrainState {
 public:
  TrainState(const TrainConfig& config, const DataBundle& bundle) : config_(config) {
    // validate_config (src/trainer.cpp:62-66): the C ABI cannot see the
    // tensor's order, so the rank count is checked here
    if (config.ranks.size() != bundle.tensor.dims.size())
      throw ValidationError("rank list has " + std::to_string(config.ranks.size()) +
                            " entries for a tensor of order " +
                            std::to_string(bundle.tensor.dims.size()));
    cmtf_gpu_config c;
    cmtf_gpu_config_default(&c);
    c.order = static_cast<int32_t>(config.ranks.size());
    c.ranks = config_.ranks.data();
    c.eta0 = config.eta0;
    c.mu = config.mu;
    c.lambda_reg = config.lambda_reg;
    c.workers = config.workers;
    c.max_epochs = config.max_epochs;
    c.rel_tol = config.rel_tol;
    c.seed = config.seed;
    c.kernel = config.kernel == GradientKernel::Opt ? CMTF_KERNEL_OPT : CMTF_KERNEL_NAIVE;
    c.nonnegative = config.nonnegative;
    c.init_scale = config.init_scale;
    c.device = config.device;
    c.exec_mode = config.serial_parity ? CMTF_EXEC_SERIAL : CMTF_EXEC_HOGWILD;
    c.hog_threads = config.hog_threads;
    check(cmtf_gpu_create(&c, &ctx_));
    upload(bundle);
    check(cmtf_gpu_make_state(ctx_), ctx_);
  }
  ~TrainState() {
    if (ctx_) cmtf_gpu_destroy(ctx_);
  }
  TrainState(const TrainState&) = delete;
  TrainState& operator=(const TrainState&) = delete;

  void upload(const DataBundle& b) {
    check(cmtf_gpu_clear_matrices(ctx_), ctx_);
    check(cmtf_gpu_set_tensor(ctx_, b.tensor.dims.data(), b.tensor.indices.data(),
                              b.tensor.values.data(), b.tensor.nnz()),
          ctx_);
    for (const auto& m : b.matrices)
      check(cmtf_gpu_add_matrix(ctx_, m.coupled_mode, m.rows, m.cols, m.indices.data(),
                                m.values.data(), m.nnz(), m.weight),
            ctx_);
    dims_ = b.tensor.dims;
    mat_shapes_.clear();
    for (const auto& m : b.matrices) mat_shapes_.emplace_back(m.coupled_mode, m.cols);
  }

  // finalized == true: the tail of train() (src/trainer.cpp:342-345) applied
  // to the copy -- finalize_orthogonalize or the nonnegative projection.
  FactorModel model(bool finalized = false) const {
    FactorModel m;
    std::size_t size = 1;
    for (auto j : config_.ranks) size *= j;
    m.core.resize(size);
    std::vector<double*> fp, vp;
    for (std::size_t n = 0; n < dims_.size(); ++n) {
      m.factors.emplace_back(static_cast<std::size_t>(dims_[n]) * config_.ranks[n]);
      fp.push_back(m.factors.back().data());
    }
    for (auto& s : mat_shapes_) {
      m.couplings.emplace_back(static_cast<std::size_t>(s.second) * config_.ranks[s.first]);
      vp.push_back(m.couplings.back().data());
    }
    double* const* vpp = vp.empty() ? nullptr : vp.data();
    if (finalized)
      check(cmtf_gpu_finalize_model(ctx_, m.core.data(), fp.data(), vpp), ctx_);
    else
      check(cmtf_gpu_get_model(ctx_, m.core.data(), fp.data(), vpp), ctx_);
    return m;
  }
  int epoch() const {
    int32_t e = 0;
    check(cmtf_gpu_get_state(ctx_, &e, nullptr), ctx_);
    return e;
  }
  double eta() const {
    double v = 0;
    check(cmtf_gpu_get_state(ctx_, nullptr, &v), ctx_);
    return v;
  }
  cmtf_gpu_ctx* ctx() const { return ctx_; }

 private:
  TrainConfig config_;
  cmtf_gpu_ctx* ctx_ = nullptr;
  std::vector<uint32_t> dims_;
  std::vector<std::pair<int, uint32_t>> mat_shapes_;
};

// run_epoch (trainer.hpp:78-79): the bundle must be the one the state holds
// (re-upload with state.upload(bundle) when it changes).
inline void run_epoch(TrainState& state, const DataBundle&, const TrainConfig&) {
  check(cmtf_gpu_run_epoch(state.ctx()), state.ctx());
}

// epoch_stats (eval.hpp:38-39)
inline EpochStats epoch_stats(const TrainState& state, double lambda_reg) {
  EpochStats s;
  check(cmtf_gpu_epoch_stats(state.ctx(), lambda_reg, &s.train_rmse, &s.objective),
        state.ctx());
  return s;
}

// test_rmse (eval.hpp:20-21)
inline double test_rmse(const TrainState& state, const SparseTensor& t) {
  double r = 0;
  check(cmtf_gpu_test_rmse(state.ctx(), t.indices.data(), t.values.data(), t.nnz(), &r),
        state.ctx());
  return r;
}

struct ConvergenceLogEntry {
  int epoch;
  double train_rmse;
  double objective;
  double seconds;
};

// train (trainer.hpp:89): epochs until convergence, then the reference's
// finalisation (src/trainer.cpp:342-345) of the returned model.
inline std::pair<FactorModel, std::vector<ConvergenceLogEntry>> train(const DataBundle& bundle,
                                                                       const TrainConfig& config) {
  TrainState state(config, bundle);
  std::vector<double> log(4 * static_cast<std::size_t>(config.max_epochs > 0 ? config.max_epochs : 1));
  int32_t n = 0;
  check(cmtf_gpu_train(state.ctx(), log.data(), config.max_epochs, &n), state.ctx());
  std::vector<ConvergenceLogEntry> out;
  for (int32_t i = 0; i < n && i < config.max_epochs; ++i)
    out.push_back({static_cast<int>(log[4 * i]), log[4 * i + 1], log[4 * i + 2], log[4 * i + 3]});
  return {state.model(true), out};
}

}  // namespace b200
}  // namespace cmtf
