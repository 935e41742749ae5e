"""Full-scale config-2 convergence sweep vs the reference's run (10 epochs)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1708_08640_b200 import api, synth
scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
REF = ({"train": 0.12004720232059254, "test": 0.12562375225231276} if scale == 1.0 else
       {"train": 0.1907186572058697, "test": 0.21336790418762466})
settings = json.loads(sys.argv[2])
b, test, _ = synth.generate(synth.config2(scale))
for s in settings:
    st = api.make_state(api.TrainConfig(ranks=[10, 10, 10], eta0=1e-3, mu=0.1, lambda_reg=0.01, **s), b)
    ms = []
    for _ in range(10):
        api.run_epoch(st); ms.append(st.last_epoch_timing()["total_ms"])
    tr = api.epoch_stats(st, 0.01).train_rmse; te = api.test_rmse(st, test)
    print(json.dumps({"s": s, "train": round(tr, 5), "test": round(te, 5), "rel_train": round(tr / REF["train"] - 1, 4),
                      "rel_test": round(te / REF["test"] - 1, 4), "ms": round(sorted(ms)[len(ms)//2], 3)}), flush=True)
