"""B200-native S^3CMTF (arXiv 1708.08640) training path.

Drop-in for the reference's factorization entry points (cmtf::train,
run_epoch, epoch_stats, test_rmse, compute_gradient(_opt),
matrix_entry_gradients): the compute runs in hand-written CUDA kernels for
sm_100a behind the C ABI in include/cmtf_b200.h; this package is the thin
host binding plus the synthetic-data generator used by the benchmark.
"""
from .api import (  # noqa: F401
    CoupledMatrix, DataBundle, DivergenceError, EpochStats, FactorModel, ParseError,
    SparseTensor, TrainConfig, TrainResult, TrainState, UnsupportedError,
    ValidationError, compute_gradient, compute_gradient_opt, entry_grads, epoch_stats,
    make_bundle, make_state, matrix_entry_gradients, matrix_rmse, run_epoch,
    test_rmse, train)
from ._abi import build, lib  # noqa: F401
from .io import (  # noqa: F401
    check_entries, load_matrix, load_model, load_tensor, save_matrix, save_model, save_tensor,
    split_train_test)
