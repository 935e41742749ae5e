"""Oracle convergence targets for config 2 / config 3 (CPU, slow): per-epoch train/test RMSE
of the reference (oracle/_ref, threaded) and/or the C restatement (P=1)."""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O
from paper_1708_08640_b200 import synth
p = argparse.ArgumentParser()
p.add_argument("--scale", type=float, default=1.0)
p.add_argument("--config", default="config2", choices=["config2", "config3", "config5_small"])
p.add_argument("--epochs", type=int, default=10)
p.add_argument("--which", default="ref", choices=["ref", "orc"])
p.add_argument("--workers", type=int, default=8)
p.add_argument("--lr", type=float, default=1e-3)
p.add_argument("--lam", type=float, default=0.01)
a = p.parse_args()
spec = synth.config5_small() if a.config == "config5_small" else getattr(synth, a.config)(a.scale)
b, test, _ = synth.generate(spec)
out = {"config": a.config, "scale": a.scale, "which": a.which, "workers": a.workers, "lr": a.lr, "train": [], "test": []}
if a.which == "ref":
    run = O.RefRun(b, [10, 10, 10], seed=0, eta0=a.lr, mu=0.1, lambda_reg=a.lam, workers=a.workers)
    for ep in range(a.epochs):
        t0 = time.time(); run.run_epoch(); dt = time.time() - t0
        tr, obj = run.epoch_stats(a.lam, threads=a.workers)
        te = run.test_rmse(test, threads=a.workers)
        out["train"].append(tr); out["test"].append(te)
        print(json.dumps({"epoch": ep + 1, "train": tr, "test": te, "sec": dt}), flush=True)
else:
    tr_ = O.SerialTrainer(b, [10, 10, 10], seed=0, eta0=a.lr, mu=0.1, lambda_reg=a.lam)
    for ep in range(a.epochs):
        t0 = time.time(); tr_.run_epoch(); dt = time.time() - t0
        tr, obj = O.epoch_stats(b, tr_.model, a.lam)
        te = O.tensor_rmse(test, tr_.model)
        out["train"].append(tr); out["test"].append(te)
        print(json.dumps({"epoch": ep + 1, "train": tr, "test": te, "sec": dt}), flush=True)
print(json.dumps(out))
