"""Small runs of every device kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool memcheck python scripts/sanitize_run.py [case ...]

Cases: tm (hog3tm with hot-row replicas), tmbulk (hog3tm, bulk row steps),
v2naive (hog3v2), v1 (hog3, J=2), order4 (hog4), cp (generic kernels, CP
core), serial (the serial replay), dsgd (emulated ranks: range sweeps +
delta reductions), probes (stateless f64 kernels, kernel probe), upload
(validation + duplicate check), eval.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_1708_08640_b200 import api, synth
from paper_1708_08640_b200.api import TrainConfig


def run(spec, ranks, epochs=1, **kw):
    b, test, _ = synth.generate(spec)
    st = api.make_state(TrainConfig(ranks=ranks, eta0=1e-3, lambda_reg=0.01, **kw), b)
    for _ in range(epochs):
        api.run_epoch(st)
    s = api.epoch_stats(st, 0.01)
    te = api.test_rmse(st, test)
    print(f"  {st.kernel_info()['kernel']}: train {s.train_rmse:.4f} test {te:.4f}", flush=True)
    return st, b


def c2():
    return synth.config2(0.003)


CASES = {
    "tm": lambda: run(c2(), [10, 10, 10], 2),
    "tmbulk": lambda: run(synth.config5_small(60_000), [10, 10, 10], 2),
    "v2naive": lambda: run(c2(), [10, 10, 10], 1, kernel="naive"),
    "v1": lambda: run(synth.config5_small(20_000, rank=2), [2, 2, 2], 1),
    "order4": lambda: run(synth.config4_small(20_000), [8, 8, 8, 8], 1),
    "cp": lambda: run(synth.config5_small(20_000, rank=4), [4, 4, 4], 1, core_structure="cp"),
    "serial": lambda: run(synth.config5_small(5_000, rank=4), [4, 4, 4], 1, exec_mode="serial"),
}


def dsgd():
    from paper_1708_08640_b200 import dsgd as D
    b, _, _ = synth.generate(c2())
    cfg = TrainConfig(ranks=[10, 10, 10], eta0=1e-3, lambda_reg=0.01)
    part = D.partition(b, 2)
    ranks = [D.RankState(part, p, cfg) for p in range(2)]
    D.run_epoch_emulated(ranks)
    print("  dsgd emulated epoch ok", flush=True)


def probes():
    rng = np.random.default_rng(0)
    core = rng.uniform(-1, 1, (3, 4, 2))
    rows = rng.uniform(-1, 1, (16, 9))
    counts = np.ones((16, 3), np.uint32)
    for f in (api.compute_gradient, api.compute_gradient_opt):
        f(rng.uniform(size=16), core, rows, 0.1, counts, 5)
    api.matrix_entry_gradients(rng.uniform(size=8), rng.uniform(size=(8, 4)),
                               rng.uniform(size=(8, 4)), 10.0, 0.1, np.ones(8, np.uint32))
    st, b = run(synth.config5_small(5_000), [10, 10, 10], 1)
    api.kernel_probe(st)
    print("  probes ok", flush=True)


def upload():
    from paper_1708_08640_b200 import io
    b, _, _ = synth.generate(synth.config5_small(5_000))
    idx = b.tensor.indices.copy()
    idx[7] = idx[3]
    try:
        api.make_state(TrainConfig(ranks=[4, 4, 4]), api.DataBundle(
            api.SparseTensor(b.tensor.dims, idx, b.tensor.values), []))
    except api.ValidationError as e:
        print("  duplicate rejected:", e, flush=True)
    io.check_entries(b.tensor.dims, b.tensor.indices, b.tensor.values)
    print("  upload checks ok", flush=True)


CASES.update({"dsgd": dsgd, "probes": probes, "upload": upload})

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for n in names:
        print(n, flush=True)
        CASES[n]()
    print("done", flush=True)
