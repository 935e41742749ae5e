"""The C-ABI library loads and exports every symbol include/cmtf_b200.h
declares; host-side validation behaves like the reference (no GPU needed)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import ROOT
from paper_1708_08640_b200 import _abi
from paper_1708_08640_b200.api import TrainConfig, ValidationError, UnsupportedError

HEADER = os.path.join(ROOT, "include", "cmtf_b200.h")


def header_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(cmtf_(?:gpu|coo|model|split)\w*)\s*\(", src)))


def test_header_declares_the_boundary():
    syms = header_symbols()
    for s in ("cmtf_gpu_create", "cmtf_gpu_set_tensor", "cmtf_gpu_add_matrix",
              "cmtf_gpu_run_epoch", "cmtf_gpu_epoch_stats", "cmtf_gpu_entry_grads",
              "cmtf_gpu_compute_gradient", "cmtf_gpu_matrix_entry_gradients",
              "cmtf_gpu_train", "cmtf_gpu_test_rmse", "cmtf_gpu_destroy"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    L = _abi.lib()
    missing = [s for s in header_symbols() if not hasattr(L, s)]
    assert not missing, missing
    bound = {name for name, _, _ in _abi.SIGNATURES}
    assert set(header_symbols()) <= bound


def test_library_is_sm100a():
    # the cubin inside the .so must be sm_100a (cross-compiled here)
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _abi.LIB_PATH],
                         capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_abi_version_and_defaults():
    L = _abi.lib()
    assert L.cmtf_gpu_abi_version() == 2
    c = _abi.cmtf_gpu_config()
    L.cmtf_gpu_config_default(C.byref(c))
    # TrainConfig member initialisers (include/cmtf/trainer.hpp:18-36)
    assert (c.eta0, c.mu, c.lambda_reg, c.workers, c.max_epochs, c.rel_tol) == (
        1e-3, 0.1, 0.1, 1, 100, 1e-4)
    assert c.kernel == _abi.KERNEL_OPT and c.init_scale == 1.0


def _create(cfg: TrainConfig):
    L = _abi.lib()
    c, keep = cfg.to_c()
    h = C.c_void_p()
    rc = L.cmtf_gpu_create(C.byref(c), C.byref(h))
    msg = L.cmtf_gpu_last_error().decode()
    if rc == 0:
        L.cmtf_gpu_destroy(h)
    return rc, msg


@pytest.mark.parametrize("cfg,needle", [
    (TrainConfig(ranks=[2]), "order"),
    (TrainConfig(ranks=[2, 0, 2]), "ranks must be positive"),
    (TrainConfig(ranks=[2, 2, 2], eta0=-1.0), "eta0 must be nonnegative"),
    (TrainConfig(ranks=[2, 2, 2], mu=-1.0), "mu must be nonnegative"),
    (TrainConfig(ranks=[2, 2, 2], lambda_reg=-0.1), "lambda_reg must be nonnegative"),
    (TrainConfig(ranks=[2, 2, 2], workers=0), "workers must be >= 1"),
    (TrainConfig(ranks=[2, 2, 2], max_epochs=-1), "max_epochs must be nonnegative"),
    (TrainConfig(ranks=[2, 2, 2], init_scale=0.0), "init_scale must be positive"),
])
def test_config_validation_matches_reference_messages(cfg, needle):
    # validate_config, src/trainer.cpp:60-92 -- checked before touching a device
    rc, msg = _create(cfg)
    assert rc == _abi.EVALIDATION
    assert needle in msg


def test_unsupported_shapes_are_refused_loudly():
    rc, msg = _create(TrainConfig(ranks=[100, 2, 2]))
    assert rc == _abi.EUNSUPPORTED and "rank" in msg
    # CP cores run on the device; validate_config's equal-rank rule
    # (src/trainer.cpp:69-72) is checked before touching a device
    rc, msg = _create(TrainConfig(ranks=[2, 3, 2], core_structure="cp"))
    assert rc == _abi.EVALIDATION and msg == "CP mode requires equal ranks on every mode"


def test_no_cpu_fallback_without_device():
    # On a machine without a GPU the product path must fail, not fall back.
    import subprocess
    has_gpu = subprocess.run(["bash", "-lc", "nvidia-smi -L"], capture_output=True).returncode == 0
    if has_gpu:
        pytest.skip("GPU present")
    rc, msg = _create(TrainConfig(ranks=[2, 2, 2]))
    assert rc == _abi.ECUDA and "CUDA" in msg


def test_python_raises_typed_errors():
    from paper_1708_08640_b200 import api
    with pytest.raises(ValidationError):
        api._raise(_abi.EVALIDATION, "x")
    with pytest.raises(api.DivergenceError):
        api._raise(_abi.EDIVERGENCE, "y")
    with pytest.raises(UnsupportedError):
        api._raise(_abi.EUNSUPPORTED, "z")
