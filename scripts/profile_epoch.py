"""Small driver for ncu: config2 shapes at a reduced scale, a few epochs."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1708_08640_b200 import api, synth
p = argparse.ArgumentParser()
p.add_argument("--scale", type=float, default=0.1)
p.add_argument("--epochs", type=int, default=3)
p.add_argument("--order", default="random")
p.add_argument("--uniform", action="store_true")
p.add_argument("--kernel", default="opt")
p.add_argument("--nohot", action="store_true")
a = p.parse_args()
spec = synth.config2(a.scale)
if a.uniform:
    spec.laws = ["uniform"] * 3
    for m in spec.matrices:
        m.row_law = m.col_law = "uniform"
if a.nohot:
    spec.dims = [100_000, 100_000, 100_000]
    spec.laws = ["uniform"] * 3
    spec.matrices = []
b, test, _ = synth.generate(spec)
st = api.make_state(api.TrainConfig(ranks=[10, 10, 10], eta0=1e-3, lambda_reg=0.01,
                                    order_policy=a.order, kernel=a.kernel), b)
for _ in range(a.epochs):
    api.run_epoch(st)
    print(st.last_epoch_timing(), flush=True)
