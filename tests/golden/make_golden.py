"""Generate the golden fixtures in tests/golden/ by running the UNMODIFIED
reference (oracle/_ref/libcmtf_ref.so, built from /root/reference by
oracle/Makefile) in this container.  The fixtures pin the C restatement
(oracle/cmtf_oracle.c) in tests/test_oracle_golden.py and travel to the GPU
box, where /root/reference does not exist.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.abspath(os.path.join(HERE, "..", ".."))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_1708_08640_b200.api import CoupledMatrix, DataBundle, SparseTensor  # noqa: E402


def small_bundle(seed, with_matrix=True, dims=(10, 8, 9), ranks=(2, 2, 2), n=300):
    """test_trainer.cpp:36-44 small_bundle, via the reference generator."""
    idx, vals, mats = O.ref_generate(list(dims), n, list(ranks), 0.0, seed,
                                     with_matrix=with_matrix)
    t = SparseTensor(list(dims), idx, vals)
    ms = [CoupledMatrix(m["mode"], m["rows"], m["cols"], m["indices"], m["values"],
                        m["weight"]) for m in mats]
    return DataBundle(t, ms)


def save_bundle(d, prefix, b):
    d[prefix + "dims"] = np.array(b.tensor.dims, dtype=np.uint32)
    d[prefix + "idx"] = b.tensor.indices
    d[prefix + "vals"] = b.tensor.values
    d[prefix + "n_mat"] = np.array(len(b.matrices))
    for k, m in enumerate(b.matrices):
        d[f"{prefix}m{k}_meta"] = np.array([m.coupled_mode, m.rows, m.cols], dtype=np.int64)
        d[f"{prefix}m{k}_w"] = np.array(m.weight)
        d[f"{prefix}m{k}_idx"] = m.indices
        d[f"{prefix}m{k}_vals"] = m.values


def save_model(d, prefix, m):
    d[prefix + "core"] = m.core.copy()
    for n, f in enumerate(m.factors):
        d[f"{prefix}U{n}"] = f.copy()
    for c, v in enumerate(m.couplings):
        d[f"{prefix}V{c}"] = v.copy()


def main():
    O.build()
    rng = np.random.Generator(np.random.PCG64(2024))

    # 1. shuffle streams (src/trainer.cpp:122-128, src/rng.cpp:17-26)
    d = {}
    for k, (n, seed, ep) in enumerate([(37, 0, 0), (37, 17, 3), (1000, 5, 0), (1000, 5, 9),
                                       (1, 1, 1), (2, 123, 0)]):
        s = np.arange(n, dtype=np.uint64)
        O.ref_shuffle(s, seed, ep)
        d[f"shuffle{k}_args"] = np.array([n, seed, ep], dtype=np.uint64)
        d[f"shuffle{k}"] = s
    np.savez_compressed(os.path.join(HERE, "shuffle.npz"), **d)

    # 2. split_train_test (src/sparse_data.cpp:311-342)
    d = {}
    b = small_bundle(11, with_matrix=False, n=200)
    (tri, trv), (tei, tev) = O.ref_split(b.tensor, 0.2, 3)
    save_bundle(d, "src_", b)
    d["train_idx"], d["train_vals"], d["test_idx"], d["test_vals"] = tri, trv, tei, tev
    np.savez_compressed(os.path.join(HERE, "split.npz"), **d)

    # 3. per-entry kernels (src/gradients.cpp:83-248)
    d = {}
    cases = []
    for rep in range(240):
        order = 4 if rep % 6 == 5 else 3
        ranks = [2, 3, 2, 2][:order] if rep % 3 else [3, 2, 4, 2][:order]
        core = rng.uniform(-1.5, 1.5, ranks)
        rows = [rng.uniform(-1.5, 1.5, r) for r in ranks]
        if rep % 4 == 1:  # planted zeros exercise the divisor fallback
            rows[rep % order][int(rng.integers(ranks[rep % order]))] = 0.0
            core.reshape(-1)[int(rng.integers(core.size))] = 0.0
        if rep % 10 == 3:
            rows[1][:] = 0.0
        counts = rng.integers(1, 9, order).astype(np.uint32)
        x = float(rng.uniform(-2, 2))
        lam = 0.1 if rep % 2 else 0.0
        nnz_total = int(rng.integers(1, 50))
        for opt in (0, 1):
            grow, gcore, r = O.ref_compute_gradient(opt, x, core, rows, lam, counts, nnz_total)
            d[f"k{rep}_opt{opt}_grow"] = grow
            d[f"k{rep}_opt{opt}_gcore"] = gcore
            d[f"k{rep}_opt{opt}_r"] = np.array(r)
        d[f"k{rep}_core"] = core
        d[f"k{rep}_rows"] = np.concatenate(rows)
        d[f"k{rep}_ranks"] = np.array(ranks, dtype=np.uint32)
        d[f"k{rep}_counts"] = counts
        d[f"k{rep}_scalars"] = np.array([x, lam, nnz_total])
        cases.append(rep)
    for rep in range(60):
        j = int(rng.integers(1, 12))
        u, v = rng.uniform(-2, 2, j), rng.uniform(-2, 2, j)
        y = float(rng.uniform(-3, 3))
        lm, lam, cc = float(rng.uniform(0.5, 10)), 0.1 if rep % 2 else 0.0, int(rng.integers(1, 6))
        du, dv, r = O.ref_matrix_entry_gradients(y, u, v, lm, lam, cc)
        d[f"m{rep}_in"] = np.concatenate([[y, lm, lam, cc], u, v])
        d[f"m{rep}_out"] = np.concatenate([[r], du, dv])
    d["n_kernel_cases"] = np.array(len(cases))
    np.savez_compressed(os.path.join(HERE, "kernels.npz"), **d)

    # 4. epochs, init, stats (src/trainer.cpp:30-316, src/eval.cpp:120-144)
    d = {}
    b = small_bundle(4, with_matrix=True)
    save_bundle(d, "b_", b)
    for tag, kopt, workers in (("opt1", 1, 1), ("naive1", 0, 1)):
        run = O.RefRun(b, [2, 2, 2], seed=17, eta0=0.01, mu=0.1, lambda_reg=0.1,
                       workers=workers, kernel_opt=bool(kopt))
        save_model(d, f"{tag}_init_", run.model())
        for ep in range(3):
            run.run_epoch()
            e, eta = run.info()
            save_model(d, f"{tag}_ep{ep + 1}_", run.model())
            rmse, obj = run.epoch_stats(0.1)
            d[f"{tag}_ep{ep + 1}_stats"] = np.array([e, eta, rmse, obj])
            d[f"{tag}_ep{ep + 1}_sched"] = run.schedule()
        run.close()
    # test RMSE of the final model on a held-out split of another bundle
    bt = small_bundle(5, with_matrix=False)
    save_bundle(d, "t_", bt)
    run = O.RefRun(b, [2, 2, 2], seed=17, eta0=0.01, mu=0.1, lambda_reg=0.1)
    run.run_epoch()
    d["t_rmse"] = np.array(run.test_rmse(bt.tensor))
    save_model(d, "t_model_", run.model())
    run.close()
    np.savez_compressed(os.path.join(HERE, "epochs.npz"), **d)

    # 5. config-1 shaped planted problem (1000^3, J=5) -- the first parity config
    d = {}
    from paper_1708_08640_b200 import synth
    spec = synth.config1(literal=False)
    spec.nnz, spec.dims = 20_000, [200, 200, 200]
    spec.matrices[0].cols, spec.matrices[0].nnz = 100, 2000
    bundle, test, _ = synth.generate(spec)
    save_bundle(d, "c_", bundle)
    d["c_test_idx"], d["c_test_vals"] = test.indices, test.values
    run = O.RefRun(bundle, [5, 5, 5], seed=0, eta0=0.01, mu=0.1, lambda_reg=0.01)
    for ep in range(2):
        run.run_epoch()
        rmse, obj = run.epoch_stats(0.01)
        d[f"c_ep{ep + 1}_stats"] = np.array([rmse, obj, run.test_rmse(test)])
    save_model(d, "c_ep2_", run.model())
    run.close()
    np.savez_compressed(os.path.join(HERE, "config1_small.npz"), **d)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
