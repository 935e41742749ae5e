// Drop-in usage of the C++ layer (include/cmtf_b200.hpp): a reference-style
// training loop on a small planted bundle.  Exit 0 = trained, 3 = no GPU.
#include <cmath>
#include <cstdio>
#include <random>

#include "cmtf_b200.hpp"

int main() {
  using namespace cmtf::b200;
  std::mt19937_64 rng(7);
  std::uniform_real_distribution<double> U(0.0, 1.0);
  DataBundle b;
  b.tensor.dims = {30, 20, 10};
  for (uint32_t i = 0; i < 30; ++i)
    for (uint32_t j = 0; j < 20; ++j)
      for (uint32_t k = 0; k < 10; k += 3) {
        b.tensor.indices.insert(b.tensor.indices.end(), {i, j, k});
        b.tensor.values.push_back(1.0 + 0.1 * U(rng));
      }
  CoupledMatrix m{0, 30, 5, {}, {}, 10.0};
  for (uint32_t i = 0; i < 30; ++i) {
    m.indices.insert(m.indices.end(), {i, i % 5});
    m.values.push_back(0.5);
  }
  b.matrices.push_back(m);
  TrainConfig cfg;
  cfg.ranks = {2, 2, 2};
  cfg.eta0 = 0.01;
  cfg.max_epochs = 3;
  try {
    auto [model, log] = train(b, cfg);
    if (log.empty() || !std::isfinite(log.back().train_rmse)) return 1;
    std::printf("trained %zu epochs, train_rmse %.5f, core[0] %.5f\n", log.size(),
                log.back().train_rmse, model.core[0]);
    try {
      TrainConfig bad = cfg;
      bad.ranks = {2, 2};
      TrainState s(bad, b);
      return 1;
    } catch (const cmtf::ValidationError&) {
    }
    return 0;
  } catch (const CudaError& e) {
    std::printf("no GPU: %s\n", e.what());
    return 3;
  }
}
