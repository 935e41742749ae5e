"""ctypes binding of the C ABI declared in include/cmtf_b200.h.

The shared library is built in-tree (paper_1708_08640_b200/libcmtf_b200.so,
see csrc/Makefile).  There is no fallback: if the library is missing and
cannot be built, importing the API raises.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CMTF_B200_LIB") or os.path.join(_HERE, "libcmtf_b200.so")
_lock = threading.Lock()
_lib = None

OK, EVALIDATION, EDIVERGENCE, ECUDA, ENCCL, EUNSUPPORTED, EPARSE = 0, 1, 2, 3, 4, 5, 6
KERNEL_NAIVE, KERNEL_OPT = 0, 1
EXEC_HOGWILD, EXEC_SERIAL = 0, 1


class cmtf_gpu_config(C.Structure):
    _fields_ = [
        ("order", C.c_int32),
        ("ranks", C.POINTER(C.c_uint32)),
        ("eta0", C.c_double),
        ("mu", C.c_double),
        ("lambda_reg", C.c_double),
        ("workers", C.c_int32),
        ("max_epochs", C.c_int32),
        ("rel_tol", C.c_double),
        ("seed", C.c_uint64),
        ("kernel", C.c_int32),
        ("core_structure", C.c_int32),
        ("nonnegative", C.c_int32),
        ("init_scale", C.c_double),
        ("device", C.c_int32),
        ("exec_mode", C.c_int32),
        ("hog_threads", C.c_int32),
        ("sort_mode", C.c_int32),
        ("force_generic", C.c_int32),
        ("order_policy", C.c_int32),
        ("hot_tau", C.c_float),
        ("kappa", C.c_float),
        ("flush_every", C.c_int32),
        ("kernel_version", C.c_int32),
        ("core_flush_every", C.c_int32),
        ("kappa_core", C.c_float),
        ("debug_count_visits", C.c_int32),
    ]


P = C.c_void_p
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
f64p = C.POINTER(C.c_double)
i32p = C.POINTER(C.c_int32)
f64pp = C.POINTER(f64p)

# (name, restype, argtypes) for every symbol include/cmtf_b200.h declares.
SIGNATURES = [
    ("cmtf_gpu_config_default", None, [C.POINTER(cmtf_gpu_config)]),
    ("cmtf_gpu_last_error", C.c_char_p, []),
    ("cmtf_gpu_ctx_error", C.c_char_p, [P]),
    ("cmtf_gpu_abi_version", C.c_int32, []),
    ("cmtf_gpu_create", C.c_int, [C.POINTER(cmtf_gpu_config), C.POINTER(P)]),
    ("cmtf_gpu_destroy", C.c_int, [P]),
    ("cmtf_gpu_set_tensor", C.c_int, [P, u32p, u32p, f64p, C.c_uint64]),
    ("cmtf_gpu_add_matrix", C.c_int,
     [P, C.c_int32, C.c_uint32, C.c_uint32, u32p, f64p, C.c_uint64, C.c_double]),
    ("cmtf_gpu_clear_matrices", C.c_int, [P]),
    ("cmtf_gpu_make_state", C.c_int, [P]),
    ("cmtf_gpu_set_model", C.c_int, [P, f64p, f64pp, f64pp]),
    ("cmtf_gpu_get_model", C.c_int, [P, f64p, f64pp, f64pp]),
    ("cmtf_gpu_finalize_model", C.c_int, [P, f64p, f64pp, f64pp]),
    ("cmtf_gpu_get_state", C.c_int, [P, i32p, f64p]),
    ("cmtf_gpu_set_state", C.c_int, [P, C.c_int32, C.c_double]),
    ("cmtf_gpu_run_epoch", C.c_int, [P]),
    ("cmtf_gpu_epoch_stats", C.c_int, [P, C.c_double, f64p, f64p]),
    ("cmtf_gpu_test_rmse", C.c_int, [P, u32p, f64p, C.c_uint64, f64p]),
    ("cmtf_gpu_matrix_rmse", C.c_int, [P, C.c_int32, f64p]),
    ("cmtf_gpu_train", C.c_int, [P, f64p, C.c_int32, i32p]),
    ("cmtf_gpu_entry_grads", C.c_int, [P, u64p, C.c_uint64, f64p, f64p, f64p, f64p]),
    ("cmtf_gpu_kernel_probe", C.c_int, [P, f64p, f64p, f64p, f64p]),
    ("cmtf_gpu_compute_gradient", C.c_int,
     [C.c_int32, C.c_int32, u32p, C.c_int32, f64p, C.c_uint64, f64p, f64p, u32p, C.c_double,
      C.c_uint64, C.c_int32, f64p, f64p, f64p, f64p, C.c_int32]),
    ("cmtf_gpu_matrix_entry_gradients", C.c_int,
     [C.c_uint64, C.c_uint32, f64p, f64p, f64p, C.c_double, C.c_double, u32p, f64p,
      f64p, f64p, C.c_int32]),
    ("cmtf_gpu_sweep_range", C.c_int, [P, C.c_uint64, C.c_uint64, u64p, u64p]),
    ("cmtf_gpu_end_epoch", C.c_int, [P]),
    ("cmtf_gpu_set_shared", C.c_int, [P, C.c_int32, C.c_uint32, C.c_uint32, C.c_uint64]),
    ("cmtf_gpu_set_counts", C.c_int, [P, C.c_int32, u32p, C.c_uint32]),
    ("cmtf_gpu_comm_unique_id", C.c_int, [C.c_void_p]),
    ("cmtf_gpu_comm_init", C.c_int, [P, C.c_int32, C.c_int32, C.c_void_p]),
    ("cmtf_gpu_sync", C.c_int, [P, C.c_uint32, C.c_uint32, C.c_int32]),
    ("cmtf_gpu_exchange_rows", C.c_int, [P, C.c_int32, C.c_uint32, C.c_uint32, C.c_int32,
                                         C.c_uint32, C.c_uint32, C.c_int32]),
    ("cmtf_gpu_broadcast_rows", C.c_int, [P, C.c_int32, C.c_int32, u32p, u32p]),
    ("cmtf_gpu_exchange_rows_local", C.c_int, [P, P, C.c_int32, C.c_uint32, C.c_uint32]),
    ("cmtf_gpu_sync_local", C.c_int, [C.POINTER(P), C.c_int32, C.c_uint32, C.c_uint32,
                                      C.c_int32]),
    ("cmtf_gpu_mark", C.c_int, [P, C.c_int32]),
    ("cmtf_gpu_elapsed_ms", C.c_int, [P, C.c_int32, C.c_int32, f64p]),
    ("cmtf_gpu_last_epoch_timing", C.c_int, [P, f64p, i32p]),
    ("cmtf_gpu_kernel_info", C.c_int, [P, i32p, i32p, i32p]),
    ("cmtf_gpu_order_blocks", C.c_int, [P, i32p, u32p]),
    ("cmtf_gpu_visit_counts", C.c_int, [P, u32p, u32p]),
    ("cmtf_gpu_collapse", C.c_int, [C.c_int32, u32p, C.c_int32, f64p, C.c_int32, f64p,
                                    C.c_int32]),
    ("cmtf_gpu_set_schedule", C.c_int, [P, u64p, C.c_uint64]),
    # text formats and host-side data preparation (io.cpp)
    ("cmtf_coo_parse", C.c_int, [C.c_char_p, C.c_int32, C.c_int32, C.POINTER(P)]),
    ("cmtf_coo_order", C.c_int32, [P]),
    ("cmtf_coo_nnz", C.c_uint64, [P]),
    ("cmtf_coo_has_header", C.c_int32, [P]),
    ("cmtf_coo_dims", u32p, [P]),
    ("cmtf_coo_indices", u32p, [P]),
    ("cmtf_coo_values", f64p, [P]),
    ("cmtf_coo_free", None, [P]),
    ("cmtf_coo_write", C.c_int, [C.c_char_p, C.c_int32, u32p, u32p, f64p, C.c_uint64,
                                 C.c_int32]),
    ("cmtf_gpu_check_entries", C.c_int, [C.c_int32, C.c_int32, u32p, u32p, f64p, C.c_uint64,
                                         C.c_int32]),
    ("cmtf_split_train_test", C.c_int, [C.c_int32, u32p, f64p, C.c_uint64, C.c_double,
                                        C.c_uint64, u32p, f64p, u32p, f64p, u64p, C.c_int32]),
    ("cmtf_model_save", C.c_int, [C.c_char_p, C.c_int32, u32p, C.c_int32, f64p, u32p, f64pp,
                                  C.c_int32, i32p, u32p, f64pp]),
    ("cmtf_model_load", C.c_int, [C.c_char_p, C.POINTER(P)]),
    ("cmtf_model_order", C.c_int32, [P]),
    ("cmtf_model_ranks", u32p, [P]),
    ("cmtf_model_core", f64p, [P]),
    ("cmtf_model_factor_rows", C.c_uint32, [P, C.c_int32]),
    ("cmtf_model_factor", f64p, [P, C.c_int32]),
    ("cmtf_model_n_coupled", C.c_int32, [P]),
    ("cmtf_model_coupled_mode", C.c_int32, [P, C.c_int32]),
    ("cmtf_model_coupled_rows", C.c_uint32, [P, C.c_int32]),
    ("cmtf_model_coupled", f64p, [P, C.c_int32]),
    ("cmtf_model_free", None, [P]),
]


def build(verbose: bool = False) -> None:
    """Compile the CUDA library for sm_100a (nvcc cross-compiles; no GPU needed)."""
    cmd = ["make", "-C", os.path.join(_HERE, "csrc")]
    out = subprocess.run(cmd, capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("building libcmtf_b200.so failed:\n" + out.stdout + out.stderr)
    if verbose:
        print(out.stdout)


def lib():
    """Load (building first if absent) the in-tree CUDA library."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                build()
            L = C.CDLL(LIB_PATH)
            for name, res, args in SIGNATURES:
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
        return _lib
