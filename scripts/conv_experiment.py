"""Convergence of the GPU Hogwild sweep vs the CPU oracle (design experiment).
Prints per-epoch test RMSE for several device settings on config-1 shapes."""
import json, sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle as O
from paper_1708_08640_b200 import api, synth

def run(spec_name, lr, epochs, settings):
    spec = synth.config1(literal=(spec_name == "literal"))
    b, test, _ = synth.generate(spec)
    tr = O.SerialTrainer(b, [5, 5, 5], seed=0, eta0=lr, mu=0.1, lambda_reg=0.01)
    ref = []
    for _ in range(epochs):
        tr.run_epoch(); ref.append(O.tensor_rmse(test, tr.model))
    print(json.dumps({"spec": spec_name, "lr": lr, "oracle_P1": [round(x, 5) for x in ref]}), flush=True)
    for s in settings:
        cfg = api.TrainConfig(ranks=[5, 5, 5], seed=0, eta0=lr, lambda_reg=0.01, **s)
        st = api.make_state(cfg, b)
        h = []
        for _ in range(epochs):
            api.run_epoch(st); h.append(api.test_rmse(st, test))
        print(json.dumps({"spec": spec_name, "settings": s, "info": st.kernel_info(),
                          "gpu": [round(x, 5) for x in h],
                          "rel_final": round(h[-1] / ref[-1] - 1, 4)}), flush=True)

settings = []
for order in ("sorted", "random"):
    for ht in (256, 1024, 4096, 0):
        settings.append(dict(order_policy=order, hog_threads=ht))
settings.append(dict(order_policy="random", hog_threads=0, force_generic=True))
settings.append(dict(order_policy="sorted", hog_threads=0, sort_mode=2))
run("ref", 0.01, 10, settings)
run("literal", 1e-3, 10, settings)
