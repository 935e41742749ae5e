"""Reference (oracle/_ref, threaded Hogwild) convergence on configs[3] at a
given scale (host generator synth.config4): per-epoch train / test RMSE.
Writes the JSON line used by tests/golden/config4_s01_reference.json.

    python scripts/oracle_config4.py --scale 0.1 --workers 8 --lr 1e-3
"""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O
from paper_1708_08640_b200 import synth
p = argparse.ArgumentParser()
p.add_argument("--scale", type=float, default=0.1)
p.add_argument("--epochs", type=int, default=10)
p.add_argument("--workers", type=int, default=8)
p.add_argument("--lr", type=float, default=1e-3)
p.add_argument("--lam", type=float, default=0.01)
a = p.parse_args()
t0 = time.time()
b, test, _ = synth.generate(synth.config4(a.scale))
print(json.dumps({"generated_sec": time.time() - t0, "nnz": b.tensor.nnz}), flush=True)
out = {"scale": a.scale, "workers": a.workers, "lr": a.lr, "lambda": a.lam, "train": [], "test": []}
run = O.RefRun(b, [8, 8, 8, 8], seed=0, eta0=a.lr, mu=0.1, lambda_reg=a.lam, workers=a.workers)
for ep in range(a.epochs):
    t0 = time.time(); run.run_epoch(); dt = time.time() - t0
    tr, obj = run.epoch_stats(a.lam, threads=a.workers)
    te = run.test_rmse(test, threads=a.workers)
    out["train"].append(tr); out["test"].append(te)
    print(json.dumps({"epoch": ep + 1, "train": tr, "test": te, "sec": dt}), flush=True)
print(json.dumps(out))
