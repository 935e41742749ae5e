"""Experiment: L2-blocked visiting order for the config-5 epoch.

The record array is laid out stratum-major -- strata = (mode-1 block,
mode-2 block), B x B of them, in a random sequence, random order inside a
stratum -- and the tcgen05 epoch's lanes take strided records
(CMTF_TM_STRIDED=1), so the grid sweeps one stratum at a time and the two
active row blocks (2 x 1/B of U1, U2) stay L2-resident.  Compares epoch time
and training RMSE against the default (random order, contiguous lane chunks)
on the same device-generated data.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1708_08640_b200 import api, synth_gpu
from paper_1708_08640_b200.synth_gpu import DeviceBundle, DeviceTensor

p = argparse.ArgumentParser()
p.add_argument("--nnz", type=float, default=1e8)
p.add_argument("--B", type=int, nargs="+", default=[8, 16])
p.add_argument("--epochs", type=int, default=6)
p.add_argument("--B3", type=int, nargs="*", default=[], help="3-mode blocking (B^3 strata)")
p.add_argument("--skip-default", action="store_true")
a = p.parse_args()
dev = "cuda:0"
spec = synth_gpu.config5(a.nnz, 10)
bundle, test = synth_gpu.generate(spec, device=dev)
t = bundle.tensor
g = torch.Generator(device=dev)
g.manual_seed(1)


def reorder(perm):
    return DeviceBundle(DeviceTensor(t.dims, t.indices[perm].contiguous(),
                                     t.values[perm].contiguous()), bundle.matrices)


def run(name, b, policy, strided):
    os.environ["CMTF_TM_STRIDED"] = "1" if strided else "0"
    cfg = api.TrainConfig(ranks=[10, 10, 10], eta0=1e-3, lambda_reg=0.01, order_policy=policy)
    st = api.make_state(cfg, b)
    ms, rm = [], []
    for ep in range(a.epochs):
        api.run_epoch(st)
        ms.append(st.last_epoch_timing()["total_ms"])
        rm.append(round(api.epoch_stats(st, 0.01).train_rmse, 5))
    te = api.test_rmse(st, test)
    print(json.dumps({"variant": name, "ms": [round(x, 2) for x in ms], "train_rmse": rm,
                      "test_rmse": round(te, 5)}), flush=True)
    st.close()
    torch.cuda.empty_cache()


if not a.skip_default:
    run("default (random, contiguous lanes)", bundle, "random", False)
    perm = torch.randperm(t.nnz, generator=g, device=dev)
    run("random caller order, strided lanes", reorder(perm), "caller", True)
    del perm
for B in a.B:
    i = t.indices.long()
    b1 = i[:, 0] * B // t.dims[0]
    b2 = i[:, 1] * B // t.dims[1]
    seq = torch.randperm(B * B, generator=g, device=dev)  # random stratum sequence
    key = seq[b1 * B + b2] * (1 << 40) + torch.randint(0, 1 << 40, (t.nnz,), generator=g,
                                                         device=dev)
    perm = torch.argsort(key)
    del i, b1, b2, key
    run(f"blocked B={B}, strided lanes", reorder(perm), "caller", True)
    del perm
for B in a.B3:
    i = t.indices.long()
    sid = ((i[:, 0] * B // t.dims[0]) * B + i[:, 1] * B // t.dims[1]) * B + i[:, 2] * B // t.dims[2]
    del i
    seq = torch.randperm(B * B * B, generator=g, device=dev)
    key = seq[sid] * (1 << 40) + torch.randint(0, 1 << 40, (t.nnz,), generator=g, device=dev)
    del sid
    perm = torch.argsort(key)
    del key
    run(f"blocked 3-mode B={B}, strided lanes", reorder(perm), "caller", True)
    del perm
