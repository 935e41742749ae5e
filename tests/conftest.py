import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")


def load_npz(name):
    return dict(np.load(os.path.join(GOLDEN, name)))


def bundle_from(d, prefix):
    from paper_1708_08640_b200.api import CoupledMatrix, DataBundle, SparseTensor
    t = SparseTensor(list(d[prefix + "dims"]), d[prefix + "idx"], d[prefix + "vals"])
    mats = []
    for k in range(int(d.get(prefix + "n_mat", 0))):
        mode, rows, cols = (int(v) for v in d[f"{prefix}m{k}_meta"])
        mats.append(CoupledMatrix(mode, rows, cols, d[f"{prefix}m{k}_idx"],
                                  d[f"{prefix}m{k}_vals"], float(d[f"{prefix}m{k}_w"])))
    return DataBundle(t, mats)


def model_from(d, prefix, n_factors, n_couplings):
    from paper_1708_08640_b200.api import FactorModel
    return FactorModel(d[prefix + "core"], [d[f"{prefix}U{n}"] for n in range(n_factors)],
                       [d[f"{prefix}V{c}"] for c in range(n_couplings)])


@pytest.fixture(scope="session")
def cuda_ok():
    try:
        import torch
        ok = torch.cuda.is_available()
    except Exception:
        ok = False
    if not ok:
        pytest.skip("no CUDA device")
    return True
