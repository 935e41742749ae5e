import os, sys, time
sys.path.insert(0, "/root/repo")
import torch
from paper_1708_08640_b200 import api, synth
b, test, _ = synth.generate(synth.config2(1.0))
st = api.make_state(api.TrainConfig(ranks=[10, 10, 10], eta0=1e-3, lambda_reg=0.01), b)
api.run_epoch(st)
for _ in range(5):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    s = api.epoch_stats(st, 0.01)
    t1 = time.perf_counter()
    print(f"epoch_stats {1e3*(t1-t0):.3f} ms", flush=True)
