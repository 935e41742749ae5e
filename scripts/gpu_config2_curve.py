"""GPU per-epoch train/test RMSE on config 2 (for parity against the oracle logs)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1708_08640_b200 import api, synth
scale = float(sys.argv[1]) if len(sys.argv) > 1 else 0.1
extra = json.loads(sys.argv[2]) if len(sys.argv) > 2 else {}
b, test, _ = synth.generate(synth.config2(scale))
st = api.make_state(api.TrainConfig(ranks=[10, 10, 10], eta0=1e-3, mu=0.1, lambda_reg=0.01, **extra), b)
tr, te = [], []
for ep in range(10):
    api.run_epoch(st)
    tr.append(api.epoch_stats(st, 0.01).train_rmse)
    te.append(api.test_rmse(st, test))
print(json.dumps({"scale": scale, "extra": extra, "info": st.kernel_info(), "train": tr, "test": te}))
