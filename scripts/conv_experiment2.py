"""Isolate the sources of the GPU-vs-oracle convergence gap (design experiment)."""
import json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle as O
from paper_1708_08640_b200 import api, synth

def curves(b, test, lr, epochs, settings, label):
    tr = O.SerialTrainer(b, [5, 5, 5], seed=0, eta0=lr, mu=0.1, lambda_reg=0.01)
    ref = []
    for _ in range(epochs):
        tr.run_epoch(); ref.append(O.tensor_rmse(test, tr.model))
    print(json.dumps({"case": label, "oracle_P1": [round(x, 5) for x in ref]}), flush=True)
    for s in settings:
        st = api.make_state(api.TrainConfig(ranks=[5, 5, 5], seed=0, eta0=lr, lambda_reg=0.01, **s), b)
        h = []
        for _ in range(epochs):
            api.run_epoch(st); h.append(api.test_rmse(st, test))
        print(json.dumps({"case": label, "settings": s, "gpu": [round(x, 5) for x in h],
                          "rel_final": round(h[-1] / ref[-1] - 1, 4)}), flush=True)

spec = synth.config1(literal=False)
b, test, _ = synth.generate(spec)
settings = [dict(order_policy="random", hog_threads=256), dict(order_policy="random", hog_threads=1024),
            dict(exec_mode="serial")]
nomat = api.DataBundle(b.tensor, [])
curves(nomat, test, 0.01, 10, settings, "ref-law no matrix")
curves(b, test, 0.01, 10, settings, "ref-law with matrix")
