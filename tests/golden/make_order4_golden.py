"""Serial oracle trajectory on synth.config4_small() (the configs[3]
stand-in: 4-way, 8^4 core, matrices on modes 1 and 2): per-epoch train /
test RMSE for 10 epochs, seeds 0-2 (the seed spread is the oracle's own
run-to-run variation), and the reference itself (oracle/_ref) with 1 and 6
Hogwild workers, seed 0.  Writes tests/golden/config4_small_oracle.json.

    python tests/golden/make_order4_golden.py
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from paper_1708_08640_b200 import synth  # noqa: E402
import oracle as O  # noqa: E402

EPOCHS, ETA, MU, LAM = 10, 0.01, 0.1, 0.01
b, test, _ = synth.generate(synth.config4_small())
out = {"spec": "synth.config4_small()", "ranks": [8, 8, 8, 8], "eta0": ETA, "mu": MU,
       "lambda": LAM, "epochs": EPOCHS, "seeds": {}}
for seed in (0, 1, 2):
    tr = O.SerialTrainer(b, [8] * 4, seed=seed, eta0=ETA, mu=MU, lambda_reg=LAM)
    traj = []
    for _ in range(EPOCHS):
        assert tr.run_epoch() == 0
        traj.append([O.epoch_stats(b, tr.model, LAM)[0], O.tensor_rmse(test, tr.model)])
    out["seeds"][str(seed)] = traj
    print(seed, traj[9], traj[-1], flush=True)
# the reference itself (oracle/_ref): serial and with 6 Hogwild workers
out["reference"] = {}
for workers in (1, 6):
    run = O.RefRun(b, [8] * 4, seed=0, eta0=ETA, mu=MU, lambda_reg=LAM, workers=workers)
    traj = []
    for _ in range(EPOCHS):
        run.run_epoch()
        tr_rmse, _ = run.epoch_stats(LAM, threads=workers)
        traj.append([tr_rmse, run.test_rmse(test, threads=workers)])
    out["reference"][str(workers)] = traj
    print("reference workers", workers, traj[9], traj[-1], flush=True)
json.dump(out, open(os.path.join(HERE, "config4_small_oracle.json"), "w"), indent=1)
