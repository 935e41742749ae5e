"""hog3tm vs hog3v2 parity experiment: config 2 at 10% scale, 10 epochs,
single GPU and DSGD with G ranks emulated, RMSE relative to the reference's
own run (tests/golden/config2_s01_reference.json)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1708_08640_b200 import api, dsgd, synth
ref = json.load(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden",
                                  "config2_s01_reference.json")))
RT, RE = ref["train"][-1], ref["test"][-1]
b, test, _ = synth.generate(synth.config2(0.1))
kw = dict(a.split("=") for a in sys.argv[1:])
def cfg():
    c = api.TrainConfig(ranks=[10, 10, 10], seed=0, eta0=1e-3, mu=0.1, lambda_reg=0.01)
    for k, v in kw.items():
        setattr(c, k, type(getattr(c, k))(v))
    return c
st = api.make_state(cfg(), b)
for _ in range(10):
    api.run_epoch(st)
tr, te = api.epoch_stats(st, 0.01).train_rmse, api.test_rmse(st, test)
out = {"env_tm": os.environ.get("CMTF_V3_TM"), "kw": kw, "kernel": st.kernel_info()["kernel"],
       "single": [round(tr / RT - 1, 5), round(te / RE - 1, 5)]}
for G in (2, 4):
    part = dsgd.partition(b, G)
    ranks = [dsgd.RankState(part, p, cfg()) for p in range(G)]
    for _ in range(10):
        dsgd.run_epoch_emulated(ranks)
    dsgd.consolidate_emulated(ranks)
    full = api.TrainState(cfg(), b)
    full.model = ranks[0].state.model
    tr, te = api.epoch_stats(full, 0.01).train_rmse, api.test_rmse(full, test)
    out[f"G{G}"] = [round(tr / RT - 1, 5), round(te / RE - 1, 5)]
print(json.dumps(out), flush=True)
