"""The command-line front end (paper_1708_08640_b200/cmtf_b200, built with
the library): the reference CLI's train / eval subcommands
(tools/cmtf_main.cpp:113-239 of the reference) -- options, output files,
printed lines and exit codes (0 ok, 1 error, 2 divergence)."""
import json
import os
import subprocess

import numpy as np
import pytest

from paper_1708_08640_b200 import io, synth

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
CLI = os.path.join(ROOT, "paper_1708_08640_b200", "cmtf_b200")


def run(*args):
    return subprocess.run([CLI, *args], capture_output=True, text=True, timeout=600)


@pytest.fixture(scope="module")
def data(tmp_path_factory):
    d = tmp_path_factory.mktemp("cli")
    spec = synth.config1(literal=False)
    spec.nnz, spec.dims = 6000, [80, 70, 60]
    spec.matrices[0].cols, spec.matrices[0].nnz = 40, 800
    spec.test_fraction = 0.0001
    b, _, _ = synth.generate(spec)
    t = b.tensor
    io.save_tensor(d / "tensor.tns", t)
    io.save_matrix(d / "matrix.mat", b.matrices[0])
    return d


def test_cli_usage_and_errors_before_any_device_work(tmp_path):
    r = run()
    assert r.returncode == 1 and "usage" in r.stderr
    r = run("train", "--tensor", str(tmp_path / "none.tns"), "--rank", "2,2,2")
    assert r.returncode == 1 and r.stderr.strip() == f"error: cannot open '{tmp_path / 'none.tns'}'"
    r = run("train", "--bogus")
    assert r.returncode == 1 and "unknown option '--bogus'" in r.stderr
    (tmp_path / "bad.tns").write_text("1 1 1 0.5\n1 x 1 2\n")
    r = run("train", "--tensor", str(tmp_path / "bad.tns"), "--rank", "2,2,2")
    assert r.returncode == 1
    assert r.stderr.strip() == "error: expected an integer index, got 'x' (line 2)"


@pytest.mark.gpu
def test_cli_train_then_eval(data, tmp_path):
    out = tmp_path / "run"
    r = run("train", "--tensor", str(data / "tensor.tns"), "--rank", "4,4,4", "--split", "0.1",
            "--couple", f"1:{data / 'matrix.mat'}:10", "--eta", "0.01", "--lreg", "0.01",
            "--epochs", "6", "--tol", "0", "--seed", "3", "--workers", "4", "--out", str(out))
    assert r.returncode == 0, r.stderr
    lines = r.stdout.splitlines()
    assert lines[0].startswith("epochs=6 train_rmse=")
    assert lines[1].startswith("test_rmse=") and lines[2] == f"model={out}/model.txt"
    for f in ("model.txt", "log.csv", "test.tns", "manifest.json"):
        assert (out / f).exists(), f
    log = (out / "log.csv").read_text().splitlines()
    assert log[0] == "epoch,train_rmse,objective,seconds" and len(log) == 7
    man = json.loads((out / "manifest.json").read_text())
    assert man["command"] == "train" and man["config"]["ranks"] == [4, 4, 4]
    assert man["inputs"]["couples"][0]["mode"] == 1
    m = io.load_model(out / "model.txt")
    assert len(m.factors) == 3 and m.coupling_modes == [0]
    for f in m.factors:  # train() returns orthonormal factors
        np.testing.assert_allclose(f.T @ f, np.eye(4), atol=1e-9)
    # the split is the reference's: 10% of the entries, written with %.17g
    full = io.load_tensor(data / "tensor.tns", check=False)
    test = io.load_tensor(out / "test.tns", check=False)
    _, ref_test = io.split_train_test(full, 0.1, 3)
    assert np.array_equal(test.indices, ref_test.indices)
    assert np.array_equal(test.values, ref_test.values)
    # eval of the saved model on the held-out split reproduces train's line
    r2 = run("eval", "--model", str(out / "model.txt"), "--test", str(out / "test.tns"), "--json")
    assert r2.returncode == 0, r2.stderr
    ev = json.loads(r2.stdout)
    assert ev["n_entries"] == test.nnz and ev["matrix_rmse"] == []
    te = float(lines[1].split("=")[1])
    assert abs(ev["test_rmse"] - te) <= 1e-5 * te
    r3 = run("eval", "--model", str(out / "model.txt"), "--test", str(out / "test.tns"))
    assert r3.stdout.splitlines()[1] == f"n_entries={test.nnz}"


@pytest.mark.gpu
def test_cli_divergence_exits_2(data, tmp_path):
    r = run("train", "--tensor", str(data / "tensor.tns"), "--rank", "4,4,4", "--eta", "1e6",
            "--epochs", "3", "--out", str(tmp_path / "div"))
    assert r.returncode == 2, (r.returncode, r.stderr)
    assert "try a smaller initial learning rate" in r.stderr


@pytest.mark.gpu
def test_cli_validation_errors_exit_1(data, tmp_path):
    r = run("train", "--tensor", str(data / "tensor.tns"), "--rank", "4,4")
    assert r.returncode == 1 and "rank list has 2 entries for a tensor of order 3" in r.stderr
    r = run("train", "--tensor", str(data / "tensor.tns"), "--rank", "4,4,4", "--couple", "1:x")
    assert r.returncode == 1 and "--couple expects MODE:PATH:LAMBDA" in r.stderr
    r = run("train", "--tensor", str(data / "tensor.tns"), "--rank", "4,4,4", "--couple",
            f"5:{data / 'matrix.mat'}:10")
    assert r.returncode == 1 and "coupled mode 5 out of range 1..3" in r.stderr
