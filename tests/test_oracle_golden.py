"""Pins the C restatement (oracle/cmtf_oracle.c) to the reference itself:
every fixture under tests/golden/ was produced by the unmodified reference
(tests/golden/make_golden.py).  CPU only."""
import numpy as np
import pytest

from conftest import bundle_from, load_npz, model_from
from oracle import oracle as O


def test_mt19937_64_known_answer():
    # std::mt19937_64 default-seed 10000th output is 9981545732273789042
    # (C++ standard [rand.predef]); our restatement must match.
    class Mt(O.C.Structure):
        _fields_ = [("mt", O.C.c_uint64 * 312), ("mti", O.C.c_int)]

    g = Mt()
    O.orc().orc_mt_seed(O.C.byref(g), O.C.c_uint64(5489))
    v = 0
    for _ in range(10000):
        v = O.orc().orc_mt_next(O.C.byref(g))
    assert v == 9981545732273789042


def test_shuffle_matches_reference():
    d = load_npz("shuffle.npz")
    k = 0
    while f"shuffle{k}" in d:
        n, seed, ep = (int(v) for v in d[f"shuffle{k}_args"])
        s = np.arange(n, dtype=np.uint64)
        O.shuffle(s, seed, ep)
        np.testing.assert_array_equal(s, d[f"shuffle{k}"])
        k += 1
    assert k >= 5


def test_split_matches_reference():
    d = load_npz("split.npz")
    b = bundle_from(d, "src_")
    ids, n_test = O.split_perm(b.tensor.nnz, 0.2, 3)
    test_ids, train_ids = ids[:n_test], ids[n_test:]
    np.testing.assert_array_equal(b.tensor.indices[test_ids], d["test_idx"])
    np.testing.assert_array_equal(b.tensor.values[test_ids], d["test_vals"])
    np.testing.assert_array_equal(b.tensor.indices[train_ids], d["train_idx"])
    np.testing.assert_array_equal(b.tensor.values[train_ids], d["train_vals"])


@pytest.mark.parametrize("opt", [0, 1])
def test_kernels_match_reference(opt):
    d = load_npz("kernels.npz")
    n = int(d["n_kernel_cases"])
    worst = 0.0
    for rep in range(n):
        ranks = [int(r) for r in d[f"k{rep}_ranks"]]
        flat = d[f"k{rep}_rows"]
        rows, off = [], 0
        for r in ranks:
            rows.append(flat[off:off + r])
            off += r
        x, lam, nnz_total = d[f"k{rep}_scalars"]
        grow, gcore, res = O.compute_gradient(opt, x, d[f"k{rep}_core"], rows, lam,
                                              d[f"k{rep}_counts"], int(nnz_total))
        ref_g = d[f"k{rep}_opt{opt}_grow"]
        ref_c = d[f"k{rep}_opt{opt}_gcore"]
        worst = max(worst, np.max(np.abs(grow - ref_g)), np.max(np.abs(gcore - ref_c)),
                    abs(res - float(d[f"k{rep}_opt{opt}_r"])))
    # same operation order as the reference: bit-identical
    assert worst == 0.0


def test_opt_equals_naive_in_oracle():
    # acceptance.cpp:233-265 (kernel equivalence to 1e-10, planted zeros)
    d = load_npz("kernels.npz")
    for rep in range(int(d["n_kernel_cases"])):
        a = d[f"k{rep}_opt0_grow"], d[f"k{rep}_opt0_gcore"]
        b = d[f"k{rep}_opt1_grow"], d[f"k{rep}_opt1_gcore"]
        for u, v in zip(a, b):
            scale = np.maximum(np.abs(u), np.abs(v))
            rel = np.where(scale > 0, np.abs(u - v) / np.where(scale > 0, scale, 1), 0)
            assert rel.max() <= 1e-10


def test_matrix_gradients_match_reference():
    d = load_npz("kernels.npz")
    rep = 0
    while f"m{rep}_in" in d:
        inp = d[f"m{rep}_in"]
        y, lm, lam, cc = inp[:4]
        j = (inp.shape[0] - 4) // 2
        du, dv, r = O.matrix_entry_gradients(y, inp[4:4 + j], inp[4 + j:], lm, lam, int(cc))
        out = d[f"m{rep}_out"]
        np.testing.assert_array_equal(np.concatenate([[r], du, dv]), out)
        rep += 1


def test_hand_computed_known_answers():
    # test_gradients.cpp:158-170 / SPEC.md:215
    grow, gcore, r = O.compute_gradient(0, 40.0, np.array([[2.0]]), [np.array([3.0]),
                                        np.array([5.0])], 0.0, np.array([1, 1]), 1)
    assert r == 10.0 and grow[0] == -100.0 and grow[1] == -60.0 and gcore[0] == -150.0
    # test_gradients.cpp:322-330 / SPEC.md:241
    du, dv, r = O.matrix_entry_gradients(10.0, np.array([2.0]), np.array([3.0]), 10.0, 0.0, 1)
    assert r == 4.0 and du[0] == -120.0 and dv[0] == -80.0
    # test_tucker.cpp:101-110: core [[1,2],[3,4]], u2 = (1,1) -> (3,7)
    out = np.zeros(2)
    core = np.array([[1.0, 2.0], [3.0, 4.0]])
    rows = [np.array([0.0, 0.0]), np.array([1.0, 1.0])]
    rk = np.array([2, 2], dtype=np.uint32)
    rp = (O.f64p * 2)(*[O._p(r_, O.C.c_double) for r_ in rows])
    O.orc().orc_contract_all_but(2, O._p(rk, O.C.c_uint32), 0,
                                 O._p(core.reshape(-1), O.C.c_double), rp, 0,
                                 O._p(out, O.C.c_double))
    np.testing.assert_array_equal(out, [3.0, 7.0])


@pytest.mark.parametrize("tag,kopt", [("opt1", True), ("naive1", False)])
def test_serial_epochs_bit_identical_to_reference(tag, kopt):
    # test_trainer.cpp:165-205 extended with matrices: the serial oracle
    # reproduces run_epoch(workers=1) bit for bit, including init and stats.
    d = load_npz("epochs.npz")
    b = bundle_from(d, "b_")
    tr = O.SerialTrainer(b, [2, 2, 2], seed=17, eta0=0.01, mu=0.1, lambda_reg=0.1,
                         kernel_opt=kopt)
    ref0 = model_from(d, f"{tag}_init_", 3, len(b.matrices))
    np.testing.assert_array_equal(tr.model.core, ref0.core.reshape(-1))
    for a, c in zip(tr.model.factors + tr.model.couplings, ref0.factors + ref0.couplings):
        np.testing.assert_array_equal(a, c)
    for ep in range(3):
        assert tr.run_epoch() == 0
        np.testing.assert_array_equal(tr.schedule, d[f"{tag}_ep{ep + 1}_sched"])
        ref = model_from(d, f"{tag}_ep{ep + 1}_", 3, len(b.matrices))
        np.testing.assert_array_equal(tr.model.core, ref.core.reshape(-1))
        for a, c in zip(tr.model.factors + tr.model.couplings, ref.factors + ref.couplings):
            np.testing.assert_array_equal(a, c)
        e, eta, rmse, obj = d[f"{tag}_ep{ep + 1}_stats"]
        assert tr.epoch == int(e) and tr.eta == eta
        r2, o2 = O.epoch_stats(b, tr.model, 0.1)
        assert r2 == rmse and o2 == obj


def test_test_rmse_matches_reference():
    d = load_npz("epochs.npz")
    b = bundle_from(d, "b_")
    bt = bundle_from(d, "t_")
    m = O.OracleModel(b, [2, 2, 2]).copy_from(model_from(d, "t_model_", 3, len(b.matrices)))
    assert O.tensor_rmse(bt.tensor, m) == float(d["t_rmse"])


def test_config1_small_two_epochs():
    d = load_npz("config1_small.npz")
    b = bundle_from(d, "c_")
    tr = O.SerialTrainer(b, [5, 5, 5], seed=0, eta0=0.01, mu=0.1, lambda_reg=0.01)
    for ep in range(2):
        tr.run_epoch()
        rmse, obj = O.epoch_stats(b, tr.model, 0.01)
        ref = d[f"c_ep{ep + 1}_stats"]
        assert rmse == ref[0] and obj == ref[1]
