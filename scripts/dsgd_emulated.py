"""DSGD with G ranks emulated on one GPU: RMSE vs the reference after 10 epochs."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1708_08640_b200 import api, dsgd, synth
which = sys.argv[1]
Gs = [int(x) for x in sys.argv[2].split(",")]
if which == "c1":
    b, test, _ = synth.generate(synth.config1(literal=False))
    cfg = api.TrainConfig(ranks=[5, 5, 5], seed=0, eta0=0.01, lambda_reg=0.01)
    REF = {"test": 0.10453040901191706}
else:
    scale = float(which[2:])
    b, test, _ = synth.generate(synth.config2(scale))
    cfg = api.TrainConfig(ranks=[10, 10, 10], seed=0, eta0=1e-3, lambda_reg=0.01)
    REF = ({"train": 0.12004720232059254, "test": 0.12562375225231276} if scale == 1.0 else
           {"train": 0.1907186572058697, "test": 0.21336790418762466})
if len(sys.argv) > 3:
    cfg.kappa = float(sys.argv[3])
for G in Gs:
    part = dsgd.partition(b, G)
    ranks = [dsgd.RankState(part, p, cfg) for p in range(G)]
    t0 = time.time()
    for ep in range(10):
        dsgd.run_epoch_emulated(ranks)
    dsgd.consolidate_emulated(ranks)
    el = time.time() - t0
    full = api.TrainState(cfg, b)
    full.model = ranks[0].state.model
    tr = api.epoch_stats(full, cfg.lambda_reg).train_rmse
    te = api.test_rmse(full, test)
    out = {"which": which, "G": G, "train": tr, "test": te, "rel_test": te / REF["test"] - 1,
           "sec": el}
    if "train" in REF:
        out["rel_train"] = tr / REF["train"] - 1
    print(json.dumps(out), flush=True)
