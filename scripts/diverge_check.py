"""Stability check of the Hogwild epoch on config 5 (device-generated):
per-epoch train RMSE and max |core| for a few independent runs."""
import argparse, json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1708_08640_b200 import api, synth_gpu

p = argparse.ArgumentParser()
p.add_argument("--nnz", type=float, default=1e8)
p.add_argument("--rank", type=int, default=10)
p.add_argument("--epochs", type=int, default=12)
p.add_argument("--reps", type=int, default=2)
p.add_argument("--lr", type=float, default=1e-3)
p.add_argument("--kernel", default="opt")
a = p.parse_args()
spec = synth_gpu.config5(a.nnz, a.rank)
bundle, test = synth_gpu.generate(spec, device="cuda:0")
for rep in range(a.reps):
    cfg = api.TrainConfig(ranks=[a.rank] * 3, seed=rep, eta0=a.lr, lambda_reg=0.01, kernel=a.kernel)
    st = api.make_state(cfg, bundle)
    hist = []
    try:
        for ep in range(a.epochs):
            api.run_epoch(st)
            m = st.model
            s = api.epoch_stats(st, 0.01)
            hist.append((round(s.train_rmse, 5), float(np.abs(m.core).max()),
                         float(max(np.abs(f).max() for f in m.factors))))
    except api.CmtfError as e:
        hist.append(str(e))
    print(json.dumps({"rep": rep, "kernel": st.kernel_info()["kernel"],
                      "env_v3_tm": os.environ.get("CMTF_V3_TM"), "hist": hist}), flush=True)
    st.close()
