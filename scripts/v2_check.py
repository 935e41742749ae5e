"""Quick v2 check: config-1 convergence vs oracle, config-2 epoch timings."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle as O
from paper_1708_08640_b200 import api, synth

def conv(settings, epochs=10):
    b, test, _ = synth.generate(synth.config1(literal=False))
    tr = O.SerialTrainer(b, [5, 5, 5], seed=0, eta0=0.01, mu=0.1, lambda_reg=0.01)
    ref = []
    for _ in range(epochs):
        tr.run_epoch(); ref.append(O.tensor_rmse(test, tr.model))
    print(json.dumps({"oracle": [round(x, 5) for x in ref]}), flush=True)
    for s in settings:
        st = api.make_state(api.TrainConfig(ranks=[5, 5, 5], seed=0, eta0=0.01, lambda_reg=0.01, **s), b)
        h = []
        for _ in range(epochs):
            api.run_epoch(st); h.append(api.test_rmse(st, test))
        print(json.dumps({"s": s, "info": st.kernel_info(), "gpu": [round(x, 5) for x in h],
                          "rel": round(h[-1] / ref[-1] - 1, 4)}), flush=True)

def timing(scale, settings, epochs=3, uniform=False):
    spec = synth.config2(scale)
    b, test, _ = synth.generate(spec)
    for s in settings:
        st = api.make_state(api.TrainConfig(ranks=[10, 10, 10], eta0=1e-3, lambda_reg=0.01, **s), b)
        t = []
        for _ in range(epochs):
            api.run_epoch(st); t.append(st.last_epoch_timing())
        q = api.epoch_stats(st, 0.01)
        print(json.dumps({"scale": scale, "s": s, "info": st.kernel_info(),
                          "ms": [round(x["total_ms"], 3) for x in t],
                          "train_rmse": q.train_rmse, "test_rmse": api.test_rmse(st, test)}), flush=True)

mode = sys.argv[1] if len(sys.argv) > 1 else "all"
if mode == "grid":
    conv([dict(hog_threads=h, hot_tau=t) for h in (384, 1152, 5376) for t in (0.05, 0.5, 2.0)])
if mode in ("all", "conv"):
    conv([dict(hog_threads=256), dict(hog_threads=1024), dict(), dict(hot_tau=-1),
          dict(kernel_version=1, hog_threads=256)])
if mode in ("all", "time"):
    timing(1.0, [dict(), dict(kernel="naive"), dict(hot_tau=-1), dict(kernel_version=1)], epochs=3)
