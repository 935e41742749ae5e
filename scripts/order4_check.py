"""Order-4 (hog4) kernel vs the oracle on config4_small: per-epoch RMSE of
GPU Hogwild runs beside the serial oracle, for a list of config overrides
(JSON, e.g. '[{"kernel": "opt"}, {"kernel": "opt", "kappa": 1.0}]')."""
import json, os, sys
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
from paper_1708_08640_b200 import api, synth
from paper_1708_08640_b200.api import TrainConfig
import oracle as O

eta, epochs = float(os.environ.get("ETA", 0.01)), 10
settings = json.loads(sys.argv[1]) if len(sys.argv) > 1 else [{"kernel": "opt"}, {"kernel": "naive"}]
verbose = len(sys.argv) > 2
import os
b, test, _ = synth.generate(synth.config4_small(int(os.environ.get('NNZ', 160000))))
tr = O.SerialTrainer(b, [8] * 4, seed=0, eta0=eta, mu=0.1, lambda_reg=0.01)
ref = []
for e in range(epochs):
    tr.run_epoch()
    ref.append((O.epoch_stats(b, tr.model, 0.01)[0], O.tensor_rmse(test, tr.model)))
if verbose:
    for seed in (1, 2):  # the oracle's own spread over seeds
        t2 = O.SerialTrainer(b, [8] * 4, seed=seed, eta0=eta, mu=0.1, lambda_reg=0.01)
        for e in range(epochs):
            t2.run_epoch()
        print("oracle seed", seed, "%.5f %.5f" % (O.epoch_stats(b, t2.model, 0.01)[0],
                                                  O.tensor_rmse(test, t2.model)), flush=True)
for s in settings:
    st = api.make_state(TrainConfig(ranks=[8] * 4, seed=0, eta0=eta, lambda_reg=0.01, **s), b)
    for e in range(epochs):
        api.run_epoch(st)
        if verbose or e == epochs - 1:
            trn = api.epoch_stats(st, 0.01).train_rmse
            tst = api.test_rmse(st, test)
            print(json.dumps(s), e, st.kernel_info()["kernel"],
                  "gpu %.5f %.5f  ref %.5f %.5f  d %+.2f%% %+.2f%%" % (
                      trn, tst, ref[e][0], ref[e][1], 100 * (trn / ref[e][0] - 1),
                      100 * (tst / ref[e][1] - 1)), flush=True)
