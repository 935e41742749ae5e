"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on
identical seeded inputs.  Tolerances (BASELINE.json north_star):
  * per-entry prediction/gradient pass: 1e-5 relative in fp32 (scale-aware:
    |a-b| <= 1e-5 * max(|ref|, |r| * |contraction| + reg * |u|), inputs rounded
    to fp32 before being fed to the f64 oracle);
  * serial-order single epoch: factors/core within 1e-4 of run_epoch(workers=1);
  * final train/test RMSE after a fixed number of epochs: within 1%.
"""
import numpy as np
import pytest

from conftest import bundle_from, load_npz, model_from
from oracle import oracle as O
from paper_1708_08640_b200 import api, synth
from paper_1708_08640_b200.api import TrainConfig

pytestmark = pytest.mark.gpu

f32 = lambda a: np.asarray(a, dtype=np.float32).astype(np.float64)  # noqa: E731


def _within(got, ref, tol, what=""):
    """|got - ref| <= tol * ref; with CMTF_MARGIN_LOG=<file> the measured
    deviation of every such check is appended there (one JSON line each), so
    the margins of a run can be read beside the pass/fail (profiles/)."""
    import json
    import os
    got, ref = float(got), float(ref)
    dev = (got - ref) / ref if ref else float("inf")
    log = os.environ.get("CMTF_MARGIN_LOG")
    if log:
        with open(log, "a") as f:
            f.write(json.dumps({"test": os.environ.get("PYTEST_CURRENT_TEST", "").split(" ")[0],
                                "what": what, "got": got, "ref": ref, "rel_dev": dev,
                                "tol": tol}) + "\n")
    assert abs(got - ref) <= tol * abs(ref), (what, got, ref, f"rel dev {dev:+.3e} > {tol}")


def scale_close(a, ref, scale, tol):
    err = np.abs(np.asarray(a) - np.asarray(ref))
    bound = tol * np.maximum(np.abs(ref), scale)
    worst = np.unravel_index(np.argmax(err - bound), err.shape)
    assert np.all(err <= bound), f"max excess at {worst}: err {err[worst]:.3e} vs bound {bound[worst]:.3e}"


# ----------------------------------------------------------------------
# per-entry kernels (compute_gradient / _opt / matrix_entry_gradients)
# ----------------------------------------------------------------------
@pytest.mark.parametrize("opt", [0, 1])
def test_compute_gradient_matches_oracle(opt):
    d = load_npz("kernels.npz")
    for rep in range(int(d["n_kernel_cases"])):
        ranks = [int(r) for r in d[f"k{rep}_ranks"]]
        core = f32(d[f"k{rep}_core"]).reshape(ranks)
        flat = f32(d[f"k{rep}_rows"])
        x, lam, nnz_total = d[f"k{rep}_scalars"]
        x = float(np.float32(x))
        counts = d[f"k{rep}_counts"]
        rows, off = [], 0
        for r in ranks:
            rows.append(flat[off:off + r])
            off += r
        g_ref, c_ref, r_ref = O.compute_gradient(opt, x, core, rows, lam, counts, int(nnz_total))
        fn = api.compute_gradient_opt if opt else api.compute_gradient
        grow, gcore, res = fn(x, core, flat[None, :], lam, counts[None, :], int(nnz_total))
        # scale of each component: |r| * |G x_{-n} u| + reg * |u|
        cont_scale = np.abs(r_ref) * np.max(np.abs(core)) * np.prod(
            [np.max(np.abs(r_)) + 1e-30 for r_ in rows]) * 2 + 1e-6
        scale_close(res, [r_ref], max(abs(x), 1.0), 1e-5)
        scale_close(grow[0], g_ref, cont_scale, 1e-5)
        scale_close(gcore[0], c_ref, cont_scale, 1e-5)


def test_hand_computed_rank1_on_gpu():
    # test_gradients.cpp:158-170
    grow, gcore, r = api.compute_gradient(40.0, np.array([[2.0]]), np.array([[3.0, 5.0]]),
                                          0.0, np.array([[1, 1]]), 1)
    assert r[0] == 10.0 and list(grow[0]) == [-100.0, -60.0] and gcore[0, 0] == -150.0
    # test_gradients.cpp:322-330
    du, dv, r = api.matrix_entry_gradients(10.0, [[2.0]], [[3.0]], 10.0, 0.0, 1)
    assert r[0] == 4.0 and du[0, 0] == -120.0 and dv[0, 0] == -80.0


def test_zero_residual_zero_lambda_gives_zero():
    # test_gradients.cpp:144-156
    core = f32(np.random.default_rng(43).uniform(-1, 1, (2, 2)))
    rows = f32(np.random.default_rng(44).uniform(-1, 1, (1, 4)))
    x = O.predict(core, [rows[0, :2], rows[0, 2:]])
    grow, gcore, r = api.compute_gradient(x, core, rows, 0.0, [[5, 7]], 12)
    assert abs(r[0]) < 1e-6 and np.abs(grow).max() < 1e-6 and np.abs(gcore).max() < 1e-6


def test_matrix_gradients_match_oracle():
    d = load_npz("kernels.npz")
    rep = 0
    while f"m{rep}_in" in d:
        inp = d[f"m{rep}_in"]
        y, lm, lam, cc = inp[:4]
        j = (inp.shape[0] - 4) // 2
        u, v, y = f32(inp[4:4 + j]), f32(inp[4 + j:]), float(np.float32(y))
        du_r, dv_r, r_r = O.matrix_entry_gradients(y, u, v, lm, lam, int(cc))
        du, dv, r = api.matrix_entry_gradients(y, u[None], v[None], lm, lam, int(cc))
        sc = abs(r_r) * lm * (np.abs(u).max() + np.abs(v).max()) + 1e-6
        scale_close(du[0], du_r, sc, 1e-5)
        scale_close(dv[0], dv_r, sc, 1e-5)
        scale_close(r, [r_r], max(abs(y), 1.0), 1e-5)
        rep += 1


# ----------------------------------------------------------------------
# probes on a device-resident bundle
# ----------------------------------------------------------------------
def _config1_small():
    d = load_npz("config1_small.npz")
    b = bundle_from(d, "c_")
    test = api.SparseTensor(b.tensor.dims, d["c_test_idx"], d["c_test_vals"])
    return d, b, test


@pytest.mark.parametrize("kernel", ["opt", "naive"])
def test_entry_grads_at_init_and_midtraining(kernel):
    d, b, _ = _config1_small()
    cfg = TrainConfig(ranks=[5, 5, 5], seed=0, eta0=0.01, lambda_reg=0.01, kernel=kernel)
    st = api.make_state(cfg, b)
    ids = np.arange(0, b.tensor.nnz, 37, dtype=np.uint64)
    for snapshot in ("init", "trained"):
        if snapshot == "trained":
            api.run_epoch(st)
        m = st.model  # fp32 values widened to f64: identical inputs to both sides
        xh, r, grow, gcore = api.entry_grads(st, ids)
        counts = O.count_modes(b, [5, 5, 5])
        offs = np.cumsum([0] + list(b.tensor.dims))
        for k, e in enumerate(ids):
            idx = b.tensor.indices[e]
            rows = [m.factors[n][idx[n]] for n in range(3)]
            cn = [counts[offs[n] + idx[n]] for n in range(3)]
            x = float(np.float32(b.tensor.values[e]))
            g_ref, c_ref, r_ref = O.compute_gradient(kernel == "opt", x, m.core, rows, 0.01, cn,
                                                     b.tensor.nnz)
            # scale-aware fp32 bound: r = x - x_hat cancels, so its rounding is
            # relative to max(|x|, |x_hat|), and every gradient term -r*c_n
            # inherits it: scale_n = max(|x|,|x_hat|) * |c_n|_max + reg*|u_n|.
            gmax = np.max(np.abs(m.core))
            l1 = [np.abs(r_).sum() for r_ in rows]
            xs = gmax * np.prod(l1)
            scale_close([xh[k]], [x - r_ref], xs, 1e-5)
            big = max(abs(x), xs)
            off = 0
            for n in range(3):
                cn_max = gmax * np.prod([l1[q] for q in range(3) if q != n])
                sc = big * cn_max + 0.01 * np.abs(rows[n]).max() + 1e-7
                scale_close(grow[k][off:off + 5], g_ref[off:off + 5], sc, 1e-5)
                off += 5
            phi_max = np.prod([np.abs(r_).max() for r_ in rows])
            scale_close(gcore[k], c_ref, big * phi_max + 1e-7, 1e-5)


def test_epoch_stats_and_test_rmse_match_oracle():
    d, b, test = _config1_small()
    cfg = TrainConfig(ranks=[5, 5, 5], seed=0, eta0=0.01, lambda_reg=0.01)
    st = api.make_state(cfg, b)
    api.run_epoch(st)
    m = st.model
    om = O.OracleModel(b, [5, 5, 5]).copy_from(m)
    r_ref, o_ref = O.epoch_stats(b, om, 0.01)
    s = api.epoch_stats(st, 0.01)
    _within(s.train_rmse, r_ref, 1e-5, "s.train_rmse")
    _within(s.objective, o_ref, 1e-5, "s.objective")
    t_ref = O.tensor_rmse(test, om)
    assert abs(api.test_rmse(st, test) - t_ref) <= 1e-5 * t_ref


@pytest.mark.parametrize("order,J,nnz", [(3, 4, 77), (3, 5, 128), (3, 8, 1023), (3, 10, 1025),
                                          (3, 10, 20_011), (4, 8, 131), (4, 8, 9_001)])
def test_tcgen05_eval_matches_oracle_on_ragged_sizes(order, J, nnz, monkeypatch):
    """eval3tm / eval4tm (csrc/eval3tm.cuh; predict_entry src/tucker.cpp:96-127,
    blocked_sum src/eval.cpp:14-65) against the f64 oracle at a trained model:
    entry counts below one 128-entry tile, at tile and 1024-block edges and
    past them, every supported rank; the CUDA-core eval kernel beside it."""
    spec = synth.config1(literal=False)
    spec.nnz, spec.seed = int(nnz / 0.9) + 1, 100 + nnz
    spec.dims = [200, 150, 100] if order == 3 else [40, 30, 20, 16]
    spec.ranks = [J] * order
    spec.matrices[0].cols, spec.matrices[0].nnz = 20, 200
    if order == 4:
        spec.laws = ["uniform"] * 4
    b, test, _ = synth.generate(spec)
    ranks = [J] * order
    out = {}
    for tm in ("1", "0"):
        monkeypatch.setenv("CMTF_EVAL_TM", tm)
        st = api.make_state(TrainConfig(ranks=ranks, seed=1, eta0=0.005, lambda_reg=0.01), b)
        if tm == "1":
            api.run_epoch(st)
            m = st.model
        else:
            st.model = m
        s = api.epoch_stats(st, 0.01)
        out[tm] = (s.train_rmse, s.objective, api.test_rmse(st, test))
        st.close()
    om = O.OracleModel(b, ranks).copy_from(m)
    r_ref, o_ref = O.epoch_stats(b, om, 0.01)
    t_ref = O.tensor_rmse(test, om)
    for tm in ("1", "0"):
        _within(out[tm][0], r_ref, 1e-5, f"train_rmse eval_tm={tm}")
        _within(out[tm][1], o_ref, 1e-5, f"objective eval_tm={tm}")
        _within(out[tm][2], t_ref, 1e-5, f"test_rmse eval_tm={tm}")


def test_initial_model_matches_reference_law():
    # random_model draw law and stream (src/trainer.cpp:30-58,100)
    d = load_npz("epochs.npz")
    b = bundle_from(d, "b_")
    st = api.make_state(TrainConfig(ranks=[2, 2, 2], seed=17, eta0=0.01), b)
    m = st.model
    ref = model_from(d, "opt1_init_", 3, len(b.matrices))
    np.testing.assert_array_equal(m.core.reshape(-1), f32(ref.core).reshape(-1))
    for a, c in zip(m.factors + m.couplings, ref.factors + ref.couplings):
        np.testing.assert_array_equal(a, f32(c))


# ----------------------------------------------------------------------
# serial-order single epoch (exact reference schedule, P=1)
# ----------------------------------------------------------------------
@pytest.mark.parametrize("kernel", ["opt", "naive"])
@pytest.mark.parametrize("fixture", ["epochs", "config1"])
def test_serial_epoch_reproduces_reference(kernel, fixture):
    if fixture == "epochs":
        d = load_npz("epochs.npz")
        b = bundle_from(d, "b_")
        ranks, seed, lr, lam = [2, 2, 2], 17, 0.01, 0.1
    else:
        d, b, _ = _config1_small()
        ranks, seed, lr, lam = [5, 5, 5], 0, 0.01, 0.01
    cfg = TrainConfig(ranks=ranks, seed=seed, eta0=lr, lambda_reg=lam, kernel=kernel,
                      exec_mode="serial")
    st = api.make_state(cfg, b)
    tr = O.SerialTrainer(b, ranks, seed=seed, eta0=lr, mu=0.1, lambda_reg=lam,
                         kernel_opt=kernel == "opt")
    tr.model.copy_from(st.model)  # same fp32-rounded start
    tr.run_epoch()
    api.run_epoch(st)
    m = st.model
    assert st.epoch == 1 and st.eta == pytest.approx(lr / 1.1, rel=0, abs=1e-18)
    for a, ref in zip([m.core.reshape(-1)] + m.factors + m.couplings,
                      [tr.model.core] + tr.model.factors + tr.model.couplings):
        scale_close(a, ref, 1e-2 * np.abs(ref).max(), 1e-4)


# ----------------------------------------------------------------------
# Hogwild epochs: RMSE parity after a fixed number of epochs
# ----------------------------------------------------------------------
@pytest.mark.parametrize("kernel", ["opt", "naive"])
@pytest.mark.parametrize("generic", [False, True])
def test_hogwild_rmse_within_1pct_of_oracle(kernel, generic):
    spec = synth.config1(literal=False)  # reference law, lr 0.01: converges to the noise
    b, test, _ = synth.generate(spec)
    epochs = 10
    tr = O.SerialTrainer(b, [5, 5, 5], seed=0, eta0=0.01, mu=0.1, lambda_reg=0.01)
    for _ in range(epochs):
        assert tr.run_epoch() == 0
    ref_test = O.tensor_rmse(test, tr.model)
    ref_train, _ = O.epoch_stats(b, tr.model, 0.01)
    cfg = TrainConfig(ranks=[5, 5, 5], seed=0, eta0=0.01, lambda_reg=0.01, kernel=kernel,
                      force_generic=generic)
    st = api.make_state(cfg, b)
    for _ in range(epochs):
        api.run_epoch(st)
    info = st.kernel_info()
    assert info["kernel"] == "generic" if generic else info["kernel"].startswith("order3")
    gpu_test = api.test_rmse(st, test)
    gpu_train = api.epoch_stats(st, 0.01).train_rmse
    _within(gpu_test, ref_test, 0.01, "gpu_test")
    _within(gpu_train, ref_train, 0.01, "gpu_train")


def test_zero_learning_rate_changes_nothing():
    # test_trainer.cpp:105-113
    d = load_npz("epochs.npz")
    b = bundle_from(d, "b_")
    st = api.make_state(TrainConfig(ranks=[2, 2, 2], seed=17, eta0=0.0), b)
    before = st.model
    api.run_epoch(st)
    after = st.model
    for a, c in zip([before.core] + before.factors + before.couplings,
                    [after.core] + after.factors + after.couplings):
        np.testing.assert_array_equal(a, c)


def test_learning_rate_decay_law():
    # test_trainer.cpp:91-103
    d = load_npz("epochs.npz")
    b = bundle_from(d, "b_")
    st = api.make_state(TrainConfig(ranks=[2, 2, 2], seed=17, eta0=0.002, mu=0.3), b)
    assert st.eta == 0.002
    for t in range(1, 6):
        api.run_epoch(st)
        assert st.epoch == t and st.eta == 0.002 / (1.0 + 0.3 * t)


def test_divergence_raises_named_error():
    # test_trainer.cpp:294-303
    d = load_npz("epochs.npz")
    b = bundle_from(d, "b_")
    cfg = TrainConfig(ranks=[2, 2, 2], seed=17, eta0=1e8, max_epochs=20)
    with pytest.raises(api.DivergenceError, match="try a smaller initial learning rate"):
        api.train(b, cfg)


def test_validation_errors_on_bad_bundle():
    t = api.SparseTensor([4, 4, 4], [[0, 0, 9]], [1.0])
    with pytest.raises(api.ValidationError, match="index out of range"):
        api.make_state(TrainConfig(ranks=[2, 2, 2]), api.DataBundle(t, []))
    t = api.SparseTensor([4, 4, 4], [[0, 0, 1]], [np.nan])
    with pytest.raises(api.ValidationError, match="not finite"):
        api.make_state(TrainConfig(ranks=[2, 2, 2]), api.DataBundle(t, []))
    t = api.SparseTensor([4, 4, 4], [[0, 0, 1]], [1.0])
    with pytest.raises(api.ValidationError, match="exceeds its size"):
        api.make_state(TrainConfig(ranks=[5, 2, 2]), api.DataBundle(t, []))


def test_duplicate_indices_rejected_like_the_reference():
    """check_entries (src/sparse_data.cpp:44-63): a repeated index tuple is a
    ValidationError naming the lexicographically smallest duplicate, for the
    tensor and for a coupled matrix -- same message as the reference's."""
    rng = np.random.default_rng(3)
    idx = rng.integers(0, 40, size=(5000, 3)).astype(np.uint32)
    idx = np.unique(idx, axis=0)
    rng.shuffle(idx)
    dup = idx[[17, 321]].copy()
    idx = np.concatenate([idx, dup])  # two duplicated tuples; the smaller one is reported
    rng.shuffle(idx)
    want = min(tuple(int(v) + 1 for v in d) for d in dup)
    t = api.SparseTensor([40, 40, 40], idx, rng.random(len(idx)))
    with pytest.raises(api.ValidationError) as ei:
        api.make_state(TrainConfig(ranks=[2, 2, 2]), api.DataBundle(t, []))
    assert str(ei.value) == "duplicate tensor index (%d %d %d)" % want
    if O.ref_available():  # the reference's own message for the same bundle
        with pytest.raises(ValueError) as er:
            O.RefRun(api.DataBundle(t, []), [2, 2, 2])
        assert str(er.value) == str(ei.value)
    ok = np.unique(idx, axis=0)
    t = api.SparseTensor([40, 40, 40], ok, rng.random(len(ok)))
    m_idx = np.array([[1, 2], [3, 4], [1, 2]], dtype=np.uint32)
    mat = api.CoupledMatrix(0, 40, 10, m_idx, np.ones(3), 1.0)
    with pytest.raises(api.ValidationError, match=r"duplicate matrix index \(2 3\)"):
        api.make_state(TrainConfig(ranks=[2, 2, 2]), api.DataBundle(t, [mat]))
    # dims whose product exceeds 64 bits take the hashed path
    big = np.array([[5, 6, 7, 8], [1, 2, 3, 4], [5, 6, 7, 8]], dtype=np.uint32)
    t = api.SparseTensor([1 << 20] * 4, big, np.ones(3))
    with pytest.raises(api.ValidationError, match=r"duplicate tensor index \(6 7 8 9\)"):
        api.make_state(TrainConfig(ranks=[2, 2, 2, 2]), api.DataBundle(t, []))
    # two duplicated wide tuples among many distinct ones: the smaller is reported
    wide = rng.integers(0, 1 << 20, size=(20000, 4)).astype(np.uint32)
    wide = np.unique(wide, axis=0)
    wide = np.concatenate([wide, [[9, 9, 9, 9], [5, 6, 7, 8], [9, 9, 9, 9], [5, 6, 7, 8]]])
    rng.shuffle(wide)
    t = api.SparseTensor([1 << 20] * 4, wide.astype(np.uint32), np.ones(len(wide)))
    with pytest.raises(api.ValidationError, match=r"duplicate tensor index \(6 7 8 9\)"):
        api.make_state(TrainConfig(ranks=[2, 2, 2, 2]), api.DataBundle(t, []))
    # and none: the hashed pass alone accepts the upload
    t = api.SparseTensor([1 << 20] * 4, np.unique(wide, axis=0), np.ones(len(np.unique(wide, axis=0))))
    api.make_state(TrainConfig(ranks=[2, 2, 2, 2]), api.DataBundle(t, []))


def test_order4_and_ragged_ranks_use_generic_path():
    rng = np.random.default_rng(7)
    dims, ranks = [9, 7, 6, 5], [3, 2, 4, 2]
    idx = np.unique(np.stack([rng.integers(0, d, 600) for d in dims], 1), axis=0)
    vals = rng.uniform(0, 2, idx.shape[0])
    b = api.DataBundle(api.SparseTensor(dims, idx, vals), [])
    cfg = TrainConfig(ranks=ranks, seed=3, eta0=0.01, exec_mode="serial")
    st = api.make_state(cfg, b)
    tr = O.SerialTrainer(b, ranks, seed=3, eta0=0.01, mu=0.1, lambda_reg=0.1)
    tr.model.copy_from(st.model)
    tr.run_epoch()
    api.run_epoch(st)
    m = st.model
    for a, ref in zip([m.core.reshape(-1)] + m.factors, [tr.model.core] + tr.model.factors):
        scale_close(a, ref, 1e-2 * np.abs(ref).max(), 1e-4)
    # Hogwild generic sweep runs and decreases the objective
    st2 = api.make_state(TrainConfig(ranks=ranks, seed=3, eta0=0.01), b)
    o0 = api.epoch_stats(st2, 0.1).objective
    for _ in range(3):
        api.run_epoch(st2)
    assert api.epoch_stats(st2, 0.1).objective < o0
    assert st2.kernel_info()["kernel"] == "generic"


@pytest.mark.parametrize("order,ranks", [(9, [2] * 9), (12, [2, 1, 2, 2, 1, 2, 2, 2, 1, 2, 2, 2]),
                                         (16, [2, 1] * 8)])
def test_orders_up_to_16_like_the_reference(order, ranks):
    """The reference's order bound is 16 (src/gradients.cpp:14, src/tucker.cpp:13):
    serial epoch vs the oracle, evaluation, and a Hogwild sweep beyond order 8."""
    rng = np.random.default_rng(order)
    dims = [3 + (n % 4) for n in range(order)]
    idx = np.unique(np.stack([rng.integers(0, d, 700) for d in dims], 1), axis=0)
    vals = rng.uniform(0, 2, idx.shape[0])
    b = api.DataBundle(api.SparseTensor(dims, idx, vals), [])
    cfg = TrainConfig(ranks=ranks, seed=3, eta0=0.01, exec_mode="serial")
    st = api.make_state(cfg, b)
    tr = O.SerialTrainer(b, ranks, seed=3, eta0=0.01, mu=0.1, lambda_reg=0.1)
    tr.model.copy_from(st.model)
    ref_rmse, ref_obj = O.epoch_stats(b, tr.model, 0.1)
    s_gpu = api.epoch_stats(st, 0.1)
    _within(s_gpu.train_rmse, ref_rmse, 1e-5, "s_gpu.train_rmse")
    _within(s_gpu.objective, ref_obj, 1e-5, "s_gpu.objective")
    tr.run_epoch()
    api.run_epoch(st)
    m = st.model
    for a, ref in zip([m.core.reshape(-1)] + m.factors, [tr.model.core] + tr.model.factors):
        scale_close(a, ref, 1e-2 * np.abs(ref).max(), 1e-4)
    st2 = api.make_state(TrainConfig(ranks=ranks, seed=3, eta0=0.01), b)
    o0 = api.epoch_stats(st2, 0.1).objective
    for _ in range(3):
        api.run_epoch(st2)
    assert api.epoch_stats(st2, 0.1).objective < o0
    # one past the bound is refused like the reference (ValidationError)
    if order == 16:
        d17 = dims + [2]
        i17 = np.concatenate([idx, np.zeros((idx.shape[0], 1), idx.dtype)], 1)
        with pytest.raises(api.ValidationError):
            api.make_state(TrainConfig(ranks=ranks + [1]),
                           api.DataBundle(api.SparseTensor(d17, i17, vals), []))


def test_nonnegative_clamp_keeps_parameters_nonnegative():
    spec = synth.config1(literal=False)
    spec.nnz, spec.dims = 5000, [50, 50, 50]
    spec.matrices[0].cols, spec.matrices[0].nnz = 20, 500
    b, _, _ = synth.generate(spec)
    st = api.make_state(TrainConfig(ranks=[5, 5, 5], eta0=0.05, nonnegative=True), b)
    for _ in range(3):
        api.run_epoch(st)
    m = st.model
    for a in [m.core] + m.factors + m.couplings:
        assert a.min() >= 0.0


def test_empty_matrix_is_allowed():
    d = load_npz("epochs.npz")
    b = bundle_from(d, "b_")
    b.matrices.append(api.CoupledMatrix(1, b.tensor.dims[1], 4, np.zeros((0, 2)), np.zeros(0), 1.0))
    st = api.make_state(TrainConfig(ranks=[2, 2, 2], seed=17, eta0=0.01), b)
    api.run_epoch(st)
    assert np.isfinite(api.epoch_stats(st, 0.1).objective)


@pytest.mark.parametrize("tm", ["1", "0"])
def test_config2_rmse_within_1pct_of_reference(tm, monkeypatch):
    """BASELINE configs[1] shape (Zipf 1.2 modes, clipped planted values,
    symmetric + 200-column coupled matrices) at 10% scale: 10 Hogwild epochs on
    the GPU vs the reference's own run (tests/golden/config2_s01_reference.json,
    produced by scripts/oracle_config2.py with oracle/_ref, 6 threads).
    tm=1: the default tcgen05 kernel (hog3tm); tm=0: the CUDA-core hog3v2."""
    import json
    import os
    from conftest import GOLDEN
    monkeypatch.setenv("CMTF_V3_TM", tm)
    ref = json.load(open(os.path.join(GOLDEN, "config2_s01_reference.json")))
    b, test, _ = synth.generate(synth.config2(0.1))
    st = api.make_state(TrainConfig(ranks=[10, 10, 10], eta0=1e-3, mu=0.1, lambda_reg=0.01), b)
    for _ in range(10):
        api.run_epoch(st)
    assert st.kernel_info()["kernel"] == ("order3tm" if tm == "1" else "order3v2")
    tr = api.epoch_stats(st, 0.01).train_rmse
    te = api.test_rmse(st, test)
    _within(tr, ref["train"][-1], 0.01, "tr")
    _within(te, ref["test"][-1], 0.01, "te")


@pytest.mark.parametrize("red,blocks", [("0", "0"), ("1", "0"), ("0", "8"), ("1", "4")])
def test_config5_small_within_1pct_of_reference(red, blocks, monkeypatch):
    """configs[4]'s shape (uniform indices over three large modes, no hot
    rows, so the tcgen05 epoch steps cold rows with bulk asynchronous
    reductions from shared memory -- red=0 -- or with vector REDs -- red=1;
    blocks=B: the L2-blocked visiting order with B x B strata, which the
    full-size config 5 selects by itself): 10 epochs vs the reference's own
    8-thread run on the same data (tests/golden/config5_small_reference.json),
    final RMSE within 1%."""
    import json
    import os
    from conftest import GOLDEN
    monkeypatch.setenv("CMTF_TM_RED", red)
    monkeypatch.setenv("CMTF_TM_BLOCKS", blocks)
    ref = json.load(open(os.path.join(GOLDEN, "config5_small_reference.json")))
    b, test, _ = synth.generate(synth.config5_small())
    st = api.make_state(TrainConfig(ranks=[10, 10, 10], eta0=1e-3, mu=0.1, lambda_reg=0.01), b)
    for _ in range(10):
        api.run_epoch(st)
    assert st.kernel_info()["kernel"] == "order3tm"
    assert st.kernel_info()["blocks"] == int(blocks)
    tr = api.epoch_stats(st, 0.01).train_rmse
    te = api.test_rmse(st, test)
    _within(tr, ref["train"][-1], 0.01, "tr")
    _within(te, ref["test"][-1], 0.01, "te")


@pytest.mark.parametrize("B", [4, 12])
def test_blocked_order_layout_and_positions(B, monkeypatch):
    """The blocked layout: after the first epoch every stratum (mode-1 block,
    mode-2 block) occupies one contiguous run of records, and the layout
    stays put (each epoch's order is virtual: a random stratum sequence and a
    group-affine map per stratum).  The entry -> position map rebuilt from the
    records' ids addresses every entry, and every epoch's virtual order is a
    bijection: the visit counts (kept per physical record) are exactly one.
    B = 4: one partition pass (<= 64 strata); B = 12: two passes (mode-1 blocks,
    then mode-2 blocks inside every mode-1 run)."""
    monkeypatch.setenv("CMTF_TM_BLOCKS", str(B))
    b, _, _ = synth.generate(synth.config5_small(120_000))
    cfg = TrainConfig(ranks=[10, 10, 10], eta0=1e-3, lambda_reg=0.01, debug_count_visits=True)
    st = api.make_state(cfg, b)
    layouts = []
    for _ in range(3):
        api.run_epoch(st)
        assert st.kernel_info()["blocks"] == B
        t, _ = st.visit_counts()
        assert np.all(t == 1)
        order = st._record_order()  # position -> entry id
        assert np.array_equal(np.sort(order), np.arange(b.tensor.nnz))  # every entry once
        idx = b.tensor.indices[order]
        s = (idx[:, 0].astype(np.int64) * B // b.tensor.dims[0]) * B + \
            idx[:, 1].astype(np.int64) * B // b.tensor.dims[1]
        runs = s[np.r_[True, s[1:] != s[:-1]]]
        # one run per (non-empty) stratum, in order
        assert runs.tolist() == sorted(set(s.tolist())), runs
        layouts.append(order)
    assert all(np.array_equal(layouts[0], o) for o in layouts[1:])


def test_config3_full_scale_within_1pct_of_reference():
    """BASELINE configs[2] at its stated size: 1e8 nonzeros (Zipf 1.1 over two
    1e6-row modes, uniform over 1e4), planted 10^3 core + noise, a 1e6 x 1e4
    coupled matrix with 1e7 nonzeros.  10 epochs of the product kernel on the
    GPU vs the reference's own 8-thread run on the same data
    (tests/golden/config3_reference.json, ~25 min of host time): final train
    and test RMSE within 1%."""
    import json
    import os
    from conftest import GOLDEN
    ref = json.load(open(os.path.join(GOLDEN, "config3_reference.json")))
    b, test, _ = synth.generate(synth.config3(1.0))
    assert b.tensor.nnz == 90_000_000 and b.matrices[0].nnz == 10_000_000
    st = api.make_state(TrainConfig(ranks=[10, 10, 10], eta0=1e-3, mu=0.1, lambda_reg=0.01), b)
    trs = []
    for _ in range(10):
        api.run_epoch(st)
    assert st.kernel_info()["kernel"] == "order3tm"
    tr = api.epoch_stats(st, 0.01).train_rmse
    te = api.test_rmse(st, test)
    _within(tr, ref["train"][-1], 0.01, "tr")
    _within(te, ref["test"][-1], 0.01, "te")


@pytest.mark.parametrize("G,n_strat", [(2, 2), (4, 2), (2, 3)])
def test_dsgd_emulated_ranks_within_1pct(G, n_strat):
    """DSGD with G ranks emulated on one GPU -- the multi-GPU
    algorithm minus the NCCL transport: strata sweeps, delta reductions of
    the replicated parameters, ring rotation of the stratified row blocks
    (device copies between the rank contexts) and the final consolidation.
    10 epochs on config 2 at 10% scale vs the reference's own run."""
    import json
    import os
    from conftest import GOLDEN
    from paper_1708_08640_b200 import dsgd
    ref = json.load(open(os.path.join(GOLDEN, "config2_s01_reference.json")))
    b, test, _ = synth.generate(synth.config2(0.1))
    cfg = TrainConfig(ranks=[10, 10, 10], seed=0, eta0=1e-3, mu=0.1, lambda_reg=0.01)
    part = dsgd.partition(b, G, n_strat=n_strat)
    ranks = [dsgd.RankState(part, p, cfg) for p in range(G)]
    for _ in range(10):
        dsgd.run_epoch_emulated(ranks)
    dsgd.consolidate_emulated(ranks)
    models = [r.state.model for r in ranks]
    for m in models[1:]:  # replicas agree after the consolidation
        np.testing.assert_allclose(m.core, models[0].core, rtol=0, atol=1e-6)
        for a, c in zip(m.factors, models[0].factors):
            np.testing.assert_allclose(a, c, rtol=0, atol=1e-6)
    full = api.TrainState(cfg, b)
    full.model = models[0]
    tr = api.epoch_stats(full, 0.01).train_rmse
    te = api.test_rmse(full, test)
    _within(tr, ref["train"][-1], 0.01, "tr")
    _within(te, ref["test"][-1], 0.01, "te")


@pytest.fixture(scope="module")
def order4_reference():
    """Serial oracle run on the configs[3] stand-in (4-way, 8^4 core), 20
    epochs: tests/golden/config4_small_oracle.json (make_order4_golden.py)."""
    import json
    import os
    from conftest import GOLDEN
    ref = json.load(open(os.path.join(GOLDEN, "config4_small_oracle.json")))
    b, test, _ = synth.generate(synth.config4_small())
    return b, test, ref


@pytest.mark.parametrize("kernel", ["opt", "naive"])
def test_order4_kernel_rmse_within_1pct_of_oracle(kernel, order4_reference):
    """hog4 (4-way, J = 8, tensor-core core gradient, interleaved matrices on
    modes 1 and 2): train / test RMSE after 10 epochs (the configs' epoch
    count) within 1% of the serial oracle, whose own seed-to-seed spread
    there is 0.8%."""
    b, test, ref = order4_reference
    cfg = TrainConfig(ranks=[8] * 4, seed=0, eta0=ref["eta0"], mu=ref["mu"],
                      lambda_reg=ref["lambda"], kernel=kernel)
    st = api.make_state(cfg, b)
    epochs = 10
    for _ in range(epochs):
        api.run_epoch(st)
    assert st.kernel_info()["kernel"] == ("order4tm" if kernel == "opt" else "order4")
    ref_train, ref_test = ref["seeds"]["0"][epochs - 1]
    gpu_train = api.epoch_stats(st, ref["lambda"]).train_rmse
    gpu_test = api.test_rmse(st, test)
    msg = (gpu_train, ref_train, gpu_test, ref_test)
    _within(gpu_train, ref_train, 0.01, "gpu_train")
    _within(gpu_test, ref_test, 0.01, "gpu_test")


@pytest.mark.parametrize("kernel", ["opt", "opt-mma.sync", "naive"])
def test_order4_single_entry_steps_match_oracle(kernel, monkeypatch):
    """One tensor entry per epoch (no concurrency): the order-4 sweep's row and
    core steps equal the oracle's serial step.  naive: fp32 CUDA-core sweep;
    opt: hog4tm, the contractions and the core gradient on tcgen05 with
    split-fp16 operands; opt-mma.sync: hog4's mma.sync path with 3xTF32
    operands (CMTF_V4_TM=0) -- both fp32-level accuracy.  The updated
    parameters within 1e-4, and the parameter CHANGES within 1e-4 of their
    magnitude."""
    want = {"opt": "order4tm", "opt-mma.sync": "order4", "naive": "order4"}[kernel]
    if kernel == "opt-mma.sync":
        monkeypatch.setenv("CMTF_V4_TM", "0")
        kernel = "opt"
    dims = [9, 8, 10, 8]
    idx = np.array([[1, 2, 3, 0]], dtype=np.uint32)
    b = api.DataBundle(api.SparseTensor(dims, idx, np.array([2.5])), [])
    cfg = TrainConfig(ranks=[8] * 4, seed=5, eta0=0.05, lambda_reg=0.1, kernel=kernel)
    st = api.make_state(cfg, b)
    m0 = st.model
    tr = O.SerialTrainer(b, [8] * 4, seed=5, eta0=0.05, mu=0.1, lambda_reg=0.1,
                         kernel_opt=kernel == "opt")
    tr.model.copy_from(m0)
    tr.run_epoch()
    api.run_epoch(st)
    assert st.kernel_info()["kernel"] == want
    m = st.model
    for a, ref, a0 in zip([m.core.reshape(-1)] + m.factors, [tr.model.core] + tr.model.factors,
                          [m0.core.reshape(-1)] + m0.factors):
        scale_close(a, ref, 1e-3 * np.abs(ref).max(), 1e-4)
        d, dref = np.asarray(a) - np.asarray(a0), np.asarray(ref) - np.asarray(a0)
        assert np.abs(d - dref).max() <= 1e-4 * np.abs(dref).max() + 1e-7


def test_config4_rmse_within_1pct_of_reference():
    """BASELINE configs[3] shape (4-way, 8^4 planted core, uniform indices,
    coupled matrices on modes 1 and 2) at 10% scale (2.7e7 training entries):
    10 epochs of the order-4 kernel vs the reference's own 8-thread run
    (tests/golden/config4_s01_reference.json, scripts/oracle_config4.py)."""
    import json
    import os
    from conftest import GOLDEN
    ref = json.load(open(os.path.join(GOLDEN, "config4_s01_reference.json")))
    b, test, _ = synth.generate(synth.config4(0.1))
    st = api.make_state(TrainConfig(ranks=[8] * 4, eta0=1e-3, mu=0.1, lambda_reg=0.01), b)
    for _ in range(10):
        api.run_epoch(st)
    assert st.kernel_info()["kernel"] == "order4tm"
    tr = api.epoch_stats(st, 0.01).train_rmse
    te = api.test_rmse(st, test)
    _within(tr, ref["train"][-1], 0.01, "tr")
    _within(te, ref["test"][-1], 0.01, "te")


@pytest.mark.parametrize("which", ["config1", "config2"])
def test_device_hot_selection_matches_host(which, monkeypatch):
    """The device-side hot-row selection (radix sort of (count, array, row)
    keys) picks the same rows in the same replica slots as the host's stable
    sort (CMTF_HOT_CHECK compares them inside prepare and fails the epoch)."""
    monkeypatch.setenv("CMTF_HOT_CHECK", "1")
    if which == "config1":
        b, _, _ = synth.generate(synth.config1(literal=False))
        ranks = [5, 5, 5]
    else:
        b, _, _ = synth.generate(synth.config2(0.1))
        ranks = [10, 10, 10]
    for tau in (0.0, 0.1):
        st = api.make_state(TrainConfig(ranks=ranks, eta0=1e-3, lambda_reg=0.01, hot_tau=tau), b)
        api.run_epoch(st)
        assert np.isfinite(api.epoch_stats(st, 0.01).train_rmse)


# ----------------------------------------------------------------------
# train()'s finalisation: finalize_orthogonalize /
# apply_nonnegative_projection vs the reference on the same model
# ----------------------------------------------------------------------
def _predict_all(m, idx):
    """x_hat for entries idx (numpy, f64) of a dense-core model."""
    G = m.core
    out = np.einsum("abc,ea,eb,ec->e", G, m.factors[0][idx[:, 0]], m.factors[1][idx[:, 1]],
                    m.factors[2][idx[:, 2]])
    return out


@pytest.mark.parametrize("nonneg", [False, True])
def test_finalized_model_matches_reference(nonneg):
    spec = synth.config1(literal=False)
    spec.nnz, spec.dims = 20000, [300, 200, 100]
    spec.matrices[0].cols, spec.matrices[0].nnz = 50, 3000
    b, _, _ = synth.generate(spec)
    ranks = [5, 5, 5]
    st = api.make_state(TrainConfig(ranks=ranks, seed=3, eta0=0.01, lambda_reg=0.01,
                                    nonnegative=nonneg), b)
    for _ in range(2):
        api.run_epoch(st)
    raw = st.model
    fin = st.finalized_model()
    ref = O.RefRun(b, ranks, seed=3, eta0=0.01, lambda_reg=0.01, nonnegative=nonneg)
    ref.set_model(O.OracleModel(b, ranks).copy_from(raw))
    ref.finalize(nonneg=nonneg)
    rm = ref.model()
    tol = 1e-9
    for got, want in zip([fin.core.reshape(-1)] + fin.factors + fin.couplings,
                         [rm.core.reshape(-1)] + rm.factors + rm.couplings):
        assert np.abs(got - want).max() <= tol * max(1.0, np.abs(want).max()), (
            np.abs(got - want).max())
    idx = b.tensor.indices[:2000].astype(np.int64)
    if not nonneg:  # orthonormal factors, predictions and couplings' products preserved
        for f in fin.factors:
            assert np.abs(f.T @ f - np.eye(f.shape[1])).max() <= 1e-9
        p0, p1 = _predict_all(raw, idx), _predict_all(fin, idx)
        assert np.abs(p1 - p0).max() <= 1e-9 * np.abs(p0).max()
        M = b.matrices[0]
        u0 = raw.factors[M.coupled_mode] @ raw.couplings[0].T
        u1 = fin.factors[M.coupled_mode] @ fin.couplings[0].T
        assert np.abs(u1 - u0).max() <= 1e-9 * np.abs(u0).max()
    # train() returns the finalised model
    res = api.train(b, TrainConfig(ranks=ranks, seed=3, eta0=0.01, lambda_reg=0.01,
                                   max_epochs=2, nonnegative=nonneg))
    if not nonneg:
        for f in res.model.factors:
            assert np.abs(f.T @ f - np.eye(f.shape[1])).max() <= 1e-9
    else:
        assert all(a.min() >= 0 for a in [res.model.core] + res.model.factors)


@pytest.mark.parametrize("J", [4, 8, 10])
def test_tcgen05_kernel_ranks_within_1pct_of_oracle(J):
    """hog3tm at every rank it is built for (4, 5, 8, 10; 5 is covered by the
    config-1 test above): 10 Hogwild epochs on the config-1 shape vs the
    serial oracle."""
    spec = synth.config1(literal=False)
    b, test, _ = synth.generate(spec)
    ranks = [J, J, J]
    epochs = 10
    tr = O.SerialTrainer(b, ranks, seed=0, eta0=0.01, mu=0.1, lambda_reg=0.01)
    for _ in range(epochs):
        assert tr.run_epoch() == 0
    ref_test = O.tensor_rmse(test, tr.model)
    ref_train, _ = O.epoch_stats(b, tr.model, 0.01)
    st = api.make_state(TrainConfig(ranks=ranks, seed=0, eta0=0.01, lambda_reg=0.01), b)
    for _ in range(epochs):
        api.run_epoch(st)
    assert st.kernel_info()["kernel"] == "order3tm"
    gpu_test = api.test_rmse(st, test)
    gpu_train = api.epoch_stats(st, 0.01).train_rmse
    _within(gpu_train, ref_train, 0.01, "gpu_train")
    _within(gpu_test, ref_test, 0.01, "gpu_test")


# ----------------------------------------------------------------------
# the product epoch kernel's own arithmetic (hog3tm, tcgen05 split-fp16)
# ----------------------------------------------------------------------
def _hog3tm_probe_check(st, bundle, ranks, lam, n_oracle=400, tol=1e-5):
    """x_hat, r and the row gradients of every training entry, and the summed
    core-gradient data term, as the epoch kernel computes them inside its
    tensor-core tiles, against the f64 oracle at the same (fp32) model.
    Bound: |got - ref| <= tol * (forward-error scale of the sum), i.e. the
    sum of the absolute values of the terms (scale-aware 1e-5)."""
    m = st.model
    before = [m.core.copy()] + [f.copy() for f in m.factors]
    xh, r, grow, gdat = api.kernel_probe(st)
    after = st.model
    assert np.array_equal(after.core, before[0])  # eta = 0: nothing moves
    for n in range(3):
        assert np.array_equal(after.factors[n], before[1 + n])
    t = bundle.tensor
    idx = np.asarray(t.indices, dtype=np.int64).reshape(-1, 3)
    x = f32(t.values)
    G, U = m.core, m.factors
    aG = np.abs(G)
    u = [U[n][idx[:, n]] for n in range(3)]
    au = [np.abs(q) for q in u]
    T = np.einsum("abc,ec->eab", G, u[2])
    aT = np.einsum("abc,ec->eab", aG, au[2])
    c1 = np.einsum("eab,eb->ea", T, u[1])
    a1 = np.einsum("eab,eb->ea", aT, au[1])
    c2 = np.einsum("eab,ea->eb", T, u[0])
    a2 = np.einsum("eab,ea->eb", aT, au[0])
    c3 = np.einsum("abc,ea,eb->ec", G, u[0], u[1])
    a3 = np.einsum("abc,ea,eb->ec", aG, au[0], au[1])
    xref = np.einsum("ea,ea->e", c1, u[0])
    sabs = np.einsum("ea,ea->e", a1, au[0])
    rref = x - xref
    counts = O.count_modes(bundle, ranks)
    offs = np.cumsum([0] + list(t.dims))
    # x_hat and r: the sum's own scale
    scale_close(xh, xref, sabs, tol)
    scale_close(r, rref, sabs, tol)
    J = ranks[0]
    for n, (c, ac) in enumerate(((c1, a1), (c2, a2), (c3, a3))):
        cnt = counts[offs[n] + idx[:, n]].astype(np.float64)
        reg = np.float32(lam) / cnt.astype(np.float32)
        gref = -rref[:, None] * c + reg.astype(np.float64)[:, None] * u[n]
        # error of r propagates through c; error of c through r
        sc = sabs[:, None] * np.abs(c) + np.abs(rref)[:, None] * ac + reg[:, None] * au[n]
        scale_close(grow[:, n * J:(n + 1) * J], gref, sc, tol)
    # the C oracle (compute_gradient_opt restated) on a sample of entries
    rng = np.random.default_rng(1)
    for e in rng.choice(len(x), size=min(n_oracle, len(x)), replace=False):
        rows = [u[n][e] for n in range(3)]
        cn = [counts[offs[n] + idx[e, n]] for n in range(3)]
        g_o, _, r_o = O.compute_gradient(1, float(x[e]), G, rows, lam, cn, len(x), with_core=False)
        sc = np.concatenate([sabs[e] * np.abs(c[e]) + abs(rref[e]) * ac[e] + lam / cn[k] * au[k][e]
                             for k, (c, ac) in enumerate(((c1, a1), (c2, a2), (c3, a3)))])
        scale_close([r[e]], [r_o], sabs[e], tol)
        scale_close(grow[e], g_o, sc, tol)
    # core gradient: sum_e -r_e u1 (x) u2 (x) u3 (the tile MMAs' accumulations)
    D = np.einsum("e,ea,eb,ec->abc", -rref, u[0], u[1], u[2])
    aD = np.einsum("e,ea,eb,ec->abc", np.abs(rref) + sabs, au[0], au[1], au[2])
    scale_close(gdat, D, aD, tol)


@pytest.mark.parametrize("J", [4, 5, 8, 10])
def test_hog3tm_kernel_probe_matches_oracle(J):
    """north_star: the per-entry prediction and gradient pass within 1e-5 --
    checked on the product kernel itself (every training entry, at the initial
    model and after 3 epochs), not on a separate probe kernel."""
    b, _, _ = synth.generate(synth.config1(literal=False))
    ranks = [J] * 3
    st = api.make_state(TrainConfig(ranks=ranks, eta0=1e-3, mu=0.1, lambda_reg=0.01), b)
    _hog3tm_probe_check(st, b, ranks, 0.01)
    assert st.kernel_info()["kernel"] == "order3tm"
    for _ in range(3):
        api.run_epoch(st)
    _hog3tm_probe_check(st, b, ranks, 0.01)


def test_hog3tm_kernel_probe_config2_tile_shapes():
    """Config-2 shape at 10% scale (Zipf heads in hot-row replicas, J = 10,
    all 148 SMs, full 128-entry tiles): the kernel's arithmetic at 1e-5."""
    b, _, _ = synth.generate(synth.config2(0.1))
    ranks = [10, 10, 10]
    st = api.make_state(TrainConfig(ranks=ranks, eta0=1e-3, mu=0.1, lambda_reg=0.01), b)
    api.run_epoch(st)
    _hog3tm_probe_check(st, b, ranks, 0.01, n_oracle=200)


# ---------------------------------------------------------------- CP core --
# CoreStructure::HyperDiagonalCp (src/gradients.cpp:108-115,145-152,192-205,
# src/tucker.cpp:104-112, src/trainer.cpp:69-72,370-371): on the device the
# core is stored densely with zero off-diagonal elements and only its
# superdiagonal takes steps.

@pytest.mark.parametrize("order,J", [(3, 3), (3, 10), (4, 4)])
@pytest.mark.parametrize("opt", [False, True])
def test_cp_compute_gradient_matches_oracle(order, J, opt):
    rng = np.random.default_rng(100 + order * 10 + J)
    n = 64
    core = rng.uniform(-1, 1, J)
    rows = rng.uniform(-1, 1, (n, order * J))
    for e in range(0, n, 5):  # planted zeros (the opt kernel's fallback paths)
        rows[e, e % (order * J)] = 0.0
    x = rng.uniform(-2, 2, n)
    counts = rng.integers(1, 9, (n, order)).astype(np.uint32)
    fn = api.compute_gradient_opt if opt else api.compute_gradient
    grow, gcore, res = fn(x, core, rows, 0.1, counts, 50, ranks=[J] * order, cp=True)
    assert gcore.shape == (n, J)
    f32 = lambda a: np.asarray(a, dtype=np.float32).astype(np.float64)
    for e in range(n):
        rr = [f32(rows[e, k * J:(k + 1) * J]) for k in range(order)]
        g_ref, c_ref, r_ref = O.compute_gradient(int(opt), float(np.float32(x[e])), f32(core), rr,
                                                 0.1, counts[e], 50, cp=1, ranks=[J] * order)
        sc = max(1.0, abs(r_ref)) * (np.abs(core).max() * np.prod(
            [np.abs(q).max() + 1e-3 for q in rr]) + 0.1)
        assert abs(res[e] - r_ref) <= 1e-5 * sc
        assert np.abs(grow[e] - g_ref).max() <= 1e-5 * sc, e
        assert np.abs(gcore[e] - c_ref).max() <= 1e-5 * sc, e


def _cp_bundle(seed=3):
    spec = synth.config1(literal=False)
    spec.nnz, spec.dims, spec.seed = 20_000, [300, 250, 200], seed
    spec.ranks = [4, 4, 4]
    spec.matrices[0].cols, spec.matrices[0].nnz = 120, 3_000
    b, test, _ = synth.generate(spec)
    return b, test


def test_cp_initial_model_and_serial_epoch_match_reference():
    """initialize with a CP core draws only its superdiagonal
    (src/trainer.cpp:30-58); one serial-order epoch (the reference's exact
    schedule, P = 1) matches the reference's run_epoch(workers=1) within 1e-4."""
    b, _ = _cp_bundle()
    cfg = TrainConfig(ranks=[4, 4, 4], seed=5, eta0=0.01, lambda_reg=0.01, core_structure="cp",
                      exec_mode="serial")
    st = api.make_state(cfg, b)
    ref = O.RefRun(b, [4, 4, 4], seed=5, eta0=0.01, mu=0.1, lambda_reg=0.01, workers=1,
                   cp=True)
    m0, r0 = st.model, ref.model()
    assert m0.core.shape == (4,)
    assert np.array_equal(m0.core.astype(np.float32), r0.core.astype(np.float32))
    for a, c in zip(m0.factors, r0.factors):
        assert np.array_equal(a.astype(np.float32), c.astype(np.float32))
    ref.set_model(m0)  # start both from the same f32-rounded model
    for _ in range(2):
        api.run_epoch(st)
        ref.run_epoch()
    m, r = st.model, ref.model()
    for a, c in zip([m.core] + m.factors + m.couplings, [r.core] + r.factors + r.couplings):
        assert np.all(np.abs(a - c) <= 1e-4 * np.maximum(np.abs(c), 1e-2 * np.abs(c).max()))
    ref.close()


def test_cp_hogwild_rmse_within_1pct_of_reference():
    """10 Hogwild epochs with a CP core vs the reference's own threaded run."""
    b, test = _cp_bundle()
    cfg = TrainConfig(ranks=[4, 4, 4], seed=0, eta0=0.01, lambda_reg=0.01, core_structure="cp")
    st = api.make_state(cfg, b)
    ref = O.RefRun(b, [4, 4, 4], seed=0, eta0=0.01, mu=0.1, lambda_reg=0.01, workers=8, cp=True)
    for _ in range(10):
        api.run_epoch(st)
        ref.run_epoch()
    tr, tr_ref = api.epoch_stats(st, 0.01).train_rmse, ref.epoch_stats(0.01)[0]
    te, te_ref = api.test_rmse(st, test), ref.test_rmse(test)
    ref.close()
    _within(tr, tr_ref, 0.01, "tr")
    _within(te, te_ref, 0.01, "te")
    m = st.model
    assert m.core.shape == (4,)


@pytest.mark.parametrize("nonneg", [False, True])
def test_cp_train_finalisation_matches_reference(nonneg):
    """train()'s tail for a CP model: finalize_orthogonalize gives a dense
    core (core_mode_product, src/tucker.cpp:167-206); the nonnegative
    projection keeps the superdiagonal (src/trainer.cpp:370-371)."""
    b, _ = _cp_bundle(seed=4)
    cfg = TrainConfig(ranks=[4, 4, 4], seed=1, eta0=0.01, lambda_reg=0.01, core_structure="cp",
                      nonnegative=nonneg, max_epochs=2, exec_mode="serial")
    st = api.make_state(cfg, b)
    api.run_epoch(st)
    m = st.model
    ref = O.RefRun(b, [4, 4, 4], seed=1, eta0=0.01, mu=0.1, lambda_reg=0.01, workers=1, cp=True,
                   nonnegative=nonneg)
    ref.set_model(m)
    ref.finalize(nonneg=nonneg)
    r = ref.model() if nonneg else None
    fin = st.finalized_model()
    if nonneg:
        assert fin.core.shape == (4,)
        np.testing.assert_allclose(fin.core, r.core, rtol=1e-9, atol=1e-12)
        for a, c in zip(fin.factors, r.factors):
            np.testing.assert_allclose(a, c, rtol=1e-9, atol=1e-12)
    else:
        assert fin.core.shape == (4, 4, 4)
        # predictions preserved by the finalisation
        idx = b.tensor.indices[:200]
        def pred(core, F):
            return np.einsum("abc,na,nb,nc->n", core, F[0][idx[:, 0]], F[1][idx[:, 1]],
                             F[2][idx[:, 2]])
        dense = np.zeros((4, 4, 4))
        for k in range(4):
            dense[k, k, k] = m.core[k]
        np.testing.assert_allclose(pred(fin.core, fin.factors), pred(dense, m.factors),
                                   rtol=1e-9, atol=1e-9)
        for f in fin.factors:
            np.testing.assert_allclose(f.T @ f, np.eye(4), atol=1e-9)
    ref.close()


def _visit_cases():
    c2 = synth.config2(0.02)
    c4 = synth.config4_small(40_000)
    c1 = synth.config1(literal=False)
    return [
        ("order3tm, hot rows", c2, [10, 10, 10], {}),
        ("order3tm, bulk row steps", synth.config5_small(200_000), [10, 10, 10], {}),
        ("order3tm, blocked order", synth.config5_small(200_000), [10, 10, 10],
         {"env": {"CMTF_TM_BLOCKS": "8"}}),
        ("order3v2 naive", c2, [10, 10, 10], {"kernel": "naive"}),
        ("order4tm", c4, [8, 8, 8, 8], {}),
        ("order4 (mma.sync)", c4, [8, 8, 8, 8], {"env": {"CMTF_V4_TM": "0"}}),
        ("order4 naive", c4, [8, 8, 8, 8], {"kernel": "naive"}),
        ("generic (CP core)", c1, [5, 5, 5], {"core_structure": "cp"}),
    ]


@pytest.mark.parametrize("case", _visit_cases(), ids=lambda c: c[0])
def test_every_training_index_is_visited_exactly_once_per_epoch(case, monkeypatch):
    """The reference's debug_count_visits check (test_trainer.cpp:207-219,
    trainer.cpp:158-161,191) on the device epoch kernels: after each of two
    epochs (the second with a freshly reshuffled record order) every training
    entry and every coupled-matrix record was visited exactly once."""
    name, spec, ranks, extra = case
    extra = dict(extra)
    for k, v in extra.pop("env", {}).items():
        monkeypatch.setenv(k, v)
    b, _, _ = synth.generate(spec)
    st = api.make_state(TrainConfig(ranks=ranks, eta0=1e-3, lambda_reg=0.01,
                                    debug_count_visits=True, **extra), b)
    for _ in range(2):
        api.run_epoch(st)
        t, m = st.visit_counts()
        assert t.shape[0] == b.tensor.nnz and np.all(t == 1), (name, np.unique(t))
        assert m.shape[0] == sum(x.nnz for x in b.matrices) and np.all(m == 1), \
            (name, np.unique(m))
