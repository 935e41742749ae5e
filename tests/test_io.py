"""Text formats and host-side data preparation
against the reference's own outcomes (tests/golden/io_cases.json, produced
by the unmodified reference: tests/golden/make_io_golden.py).

CPU tests: the parser (every ParseError path, line numbers in the parallel
chunked parse), the writers byte for byte, split_train_test against the
reference's split (tests/golden/split.npz), model round trips.  GPU tests:
the constructor checks (check_entries: range, duplicates) on the device.
"""
import json
import os

import numpy as np
import pytest

from paper_1708_08640_b200 import api, io
from paper_1708_08640_b200.api import ParseError, ValidationError

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
CASES = json.load(open(os.path.join(GOLDEN, "io_cases.json")))

# Outcomes decided by the SparseTensor / CoupledMatrix constructor checks,
# which run on the device (cmtf_gpu_check_entries)
DEVICE_CHECKED = {"duplicate", "duplicate_two", "out_of_range", "matrix_duplicate"}


def _write(tmp_path, name, text):
    p = tmp_path / name
    with open(p, "w", newline="") as f:
        f.write(text)
    return str(p)


def _expect_ok(c, obj):
    assert obj.dims == c["dims"] if hasattr(obj, "dims") else True
    idx = np.array(c["idx"], dtype=np.uint32)
    assert np.array_equal(obj.indices.reshape(-1), idx)
    vals = np.array([float.fromhex(v) for v in c["vals"]])
    assert np.array_equal(obj.values.view(np.uint64), vals.view(np.uint64))


@pytest.mark.parametrize("c", [c for c in CASES["tensor"] if c["name"] not in DEVICE_CHECKED],
                         ids=lambda c: c["name"])
def test_load_tensor_matches_reference(tmp_path, c):
    path = _write(tmp_path, c["name"] + ".tns", c["text"])
    if "error" in c:
        cls = ParseError if c["error"] == "ParseError" else ValidationError
        with pytest.raises(cls) as ei:
            io.load_tensor(path, check=False)
        assert str(ei.value) == c["message"].replace("{path}", path)
    else:
        t = io.load_tensor(path, check=False)
        assert t.dims == c["dims"]
        _expect_ok(c, t)


@pytest.mark.parametrize("c", [c for c in CASES["matrix"] if c["name"] not in DEVICE_CHECKED],
                         ids=lambda c: c["name"])
def test_load_matrix_matches_reference(tmp_path, c):
    path = _write(tmp_path, c["name"] + ".mat", c["text"])
    td = c["tensor_dims"]
    t = api.SparseTensor(td, np.zeros((0, len(td)), np.uint32), np.zeros(0))
    if "error" in c:
        cls = ParseError if c["error"] == "ParseError" else ValidationError
        with pytest.raises(cls) as ei:
            io.load_matrix(path, c["mode"], c["weight"], t, check=False)
        assert str(ei.value) == c["message"].replace("{path}", path)
    else:
        m = io.load_matrix(path, c["mode"], c["weight"], t, check=False)
        assert [m.rows, m.cols] == c["dims"]
        assert m.coupled_mode == c["mode"] - 1 and m.weight == c["weight"]
        _expect_ok(c, m)


@pytest.mark.parametrize("c", CASES["big"], ids=lambda c: f"seed{c['seed']}")
@pytest.mark.parametrize("threads", [1, 7])
def test_parallel_parse_of_a_large_file(tmp_path, c, threads):
    """Multi-megabyte files parsed in line-aligned chunks by several threads:
    identical entries (sha256 of the arrays), and the first error in file
    order with the reference's line number."""
    import hashlib
    import sys
    sys.path.insert(0, GOLDEN)
    from make_io_golden import big_text
    path = _write(tmp_path, "big.tns", big_text(c["seed"], bad_line=c["bad_line"]))
    if "error" in c:
        with pytest.raises(ParseError) as ei:
            io.load_tensor(path, threads=threads, check=False)
        assert str(ei.value) == c["message"].replace("{path}", path)
        return
    t = io.load_tensor(path, threads=threads, check=False)
    assert t.dims == c["dims"] and t.nnz == c["nnz"]
    assert hashlib.sha256(t.indices.tobytes()).hexdigest() == c["idx_sha"]
    assert hashlib.sha256(t.values.tobytes()).hexdigest() == c["vals_sha"]


def test_save_tensor_byte_for_byte(tmp_path):
    s = CASES["save"]["tensor"]
    t = api.SparseTensor(s["dims"], np.array(s["idx"], np.uint32),
                         np.array([float.fromhex(v) for v in s["vals"]]))
    p = str(tmp_path / "t.tns")
    io.save_tensor(p, t)
    assert open(p).read() == s["text"]
    back = io.load_tensor(p, check=False)  # %.17g round-trips exactly
    assert back.dims == t.dims and np.array_equal(back.values, t.values)
    assert np.array_equal(back.indices, t.indices)


def test_save_matrix_round_trip(tmp_path):
    m = api.CoupledMatrix(1, 5, 4, np.array([[0, 0], [4, 3], [2, 1]], np.uint32),
                          np.array([0.5, -2.0, 1e-7]), 3.0)
    p = str(tmp_path / "m.mat")
    io.save_matrix(p, m)
    assert open(p).read().splitlines()[0] == "5 4"
    t = api.SparseTensor([9, 5, 3], np.zeros((0, 3), np.uint32), np.zeros(0))
    back = io.load_matrix(p, 2, 3.0, t, check=False)
    assert (back.rows, back.cols) == (5, 4)
    assert np.array_equal(back.indices, m.indices) and np.array_equal(back.values, m.values)


def _model_from(s):
    ranks = s["ranks"]
    facs = [np.array([float.fromhex(v) for v in f]).reshape(r, j)
            for f, r, j in zip(s["factors"], s["rows"], ranks)]
    core = np.array([float.fromhex(v) for v in s["core"]])
    cps = [np.array([float.fromhex(v) for v in c]).reshape(r, ranks[m])
           for c, r, m in zip(s.get("couplings", []), s.get("coupling_rows", []),
                              s.get("coupling_modes", []))]
    return core, facs, cps


def test_save_model_byte_for_byte(tmp_path):
    s = CASES["save"]["model"]
    core, facs, cps = _model_from(s)
    m = api.FactorModel(core.reshape(s["ranks"]), facs, cps, s["coupling_modes"])
    p = str(tmp_path / "model.txt")
    io.save_model(p, m)
    assert open(p).read() == s["text"]
    back = io.load_model(p)
    assert np.array_equal(back.core.reshape(-1), core)
    for a, b in zip(back.factors, facs):
        assert np.array_equal(a, b)
    assert back.coupling_modes == s["coupling_modes"]
    assert np.array_equal(back.couplings[0], cps[0])


def test_save_model_cp_core_is_written_densely(tmp_path):
    s = CASES["save"]["model_cp"]
    core, facs, _ = _model_from(s)
    p = str(tmp_path / "model_cp.txt")
    io.save_model(p, api.FactorModel(core, facs), cp=True)
    assert open(p).read() == s["text"]
    back = io.load_model(p)  # load_model returns a dense core
    dense = np.zeros((3, 3, 3))
    for k in range(3):
        dense[k, k, k] = core[k]
    assert np.array_equal(back.core, dense)


@pytest.mark.parametrize("c", CASES["model_errors"], ids=lambda c: repr(c["text"][:24]))
def test_load_model_matches_reference(tmp_path, c):
    """load_model's ParseError / ValidationError paths (src/model_io.cpp:128-179,
    validate_model src/tucker.cpp:208-224) and accepted oddities (stoul's
    trailing characters, hex values, CRLF), as the reference decides them."""
    p = _write(tmp_path, "m.txt", c["text"])
    if "error" in c:
        cls = ParseError if c["error"] == "ParseError" else ValidationError
        with pytest.raises(cls) as ei:
            io.load_model(p)
        assert str(ei.value) == c["message"].replace("{path}", p)
    else:
        m = io.load_model(p)
        assert (m.core.ndim, len(m.factors), len(m.couplings)) == \
            (c["order"], c["n_factors"], c["n_coupled"])


def test_split_matches_reference_split():
    """split_train_test vs the reference's own split (tests/golden/split.npz)."""
    g = np.load(os.path.join(GOLDEN, "split.npz"))
    t = api.SparseTensor(list(g["src_dims"]), g["src_idx"], g["src_vals"])
    tr, te = io.split_train_test(t, 0.2, 3)  # make_golden.py: ref_split(..., 0.2, 3)
    assert np.array_equal(tr.indices, g["train_idx"]) and np.array_equal(tr.values, g["train_vals"])
    assert np.array_equal(te.indices, g["test_idx"]) and np.array_equal(te.values, g["test_vals"])


def test_split_errors():
    t = api.SparseTensor([3, 3], np.zeros((0, 2), np.uint32), np.zeros(0))
    with pytest.raises(ValidationError, match="cannot split an empty tensor"):
        io.split_train_test(t, 0.1, 0)
    t = api.SparseTensor([3, 3], np.array([[0, 0]], np.uint32), np.ones(1))
    for f in (0.0, 1.0, -0.5, float("nan")):
        with pytest.raises(ValidationError, match="test fraction must be in"):
            io.split_train_test(t, f, 0)


# ---------------------------------------------------------------- GPU ----
@pytest.mark.gpu
@pytest.mark.parametrize("c", [c for c in CASES["tensor"] + CASES["matrix"]
                               if c["name"] in DEVICE_CHECKED or "error" not in c],
                         ids=lambda c: c["name"])
def test_constructor_checks_on_device(tmp_path, c):
    """load_tensor / load_matrix with the constructor's check_entries on the
    device: duplicates and out-of-range indices rejected with the
    reference's message; valid files accepted."""
    is_matrix = "mode" in c
    path = _write(tmp_path, c["name"] + (".mat" if is_matrix else ".tns"), c["text"])
    def load():
        if is_matrix:
            td = c["tensor_dims"]
            t = api.SparseTensor(td, np.zeros((0, len(td)), np.uint32), np.zeros(0))
            return io.load_matrix(path, c["mode"], c["weight"], t)
        return io.load_tensor(path)
    if "error" in c:
        with pytest.raises(ValidationError) as ei:
            load()
        assert str(ei.value) == c["message"].replace("{path}", path)
    else:
        load()
