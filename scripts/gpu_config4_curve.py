"""GPU convergence on configs[3] at a given scale from the HOST generator
(synth.config4, the same data scripts/oracle_config4.py feeds the reference):
per-epoch train / test RMSE, for a list of config overrides.

    python scripts/gpu_config4_curve.py 0.1 '[{}, {"kernel": "naive"}]' [ref.json]
"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1708_08640_b200 import api, synth
scale = float(sys.argv[1]) if len(sys.argv) > 1 else 0.1
settings = json.loads(sys.argv[2]) if len(sys.argv) > 2 else [{}]
ref = json.load(open(sys.argv[3])) if len(sys.argv) > 3 else None
t0 = time.time()
b, test, _ = synth.generate(synth.config4(scale))
print(json.dumps({"generated_sec": round(time.time() - t0, 1)}), flush=True)
for s in settings:
    cfg = api.TrainConfig(ranks=[8] * 4, seed=0, eta0=1e-3, mu=0.1, lambda_reg=0.01, **s)
    st = api.make_state(cfg, b)
    for ep in range(10):
        api.run_epoch(st)
        tr = api.epoch_stats(st, 0.01).train_rmse
        te = api.test_rmse(st, test)
        line = {"s": s, "epoch": ep + 1, "train": round(tr, 6), "test": round(te, 6),
                "ms": round(st.last_epoch_timing()["total_ms"], 2)}
        if ref:
            line["rel_train"] = round(tr / ref["train"][ep] - 1, 4)
            line["rel_test"] = round(te / ref["test"][ep] - 1, 4)
        print(json.dumps(line), flush=True)
