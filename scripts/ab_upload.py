"""Same-process A/B of upload settings on config 5 (one set of pinned host
buffers, contexts created in turn under each environment):
  python scripts/ab_upload.py 1e9 "CMTF_UP_CHUNKS=4" "CMTF_UP_CHUNKS=16" ..."""
import gc, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1708_08640_b200 import api, synth_gpu
from paper_1708_08640_b200.synth_gpu import DeviceBundle, DeviceMatrix, DeviceTensor
nnz = float(sys.argv[1])
settings = sys.argv[2:]
b, test = synth_gpu.generate(synth_gpu.config5(nnz, 10), device="cuda:0")
pin = lambda a: a.cpu().pin_memory()
t = b.tensor
pb = DeviceBundle(DeviceTensor(t.dims, pin(t.indices), pin(t.values)),
                  [DeviceMatrix(m.coupled_mode, m.rows, m.cols, pin(m.indices), pin(m.values), m.weight)
                   for m in b.matrices])
del b, t, test
gc.collect(); torch.cuda.empty_cache()
keys = set()
for s in settings:
    keys |= {kv.split("=")[0] for kv in s.split(",") if kv}
for rnd in range(2):
    for s in settings:
        for k in keys:
            os.environ.pop(k, None)
        for kv in s.split(","):
            if kv:
                k, v = kv.split("=")
                os.environ[k] = v
        st = api.make_state(api.TrainConfig(ranks=[10, 10, 10], seed=0, eta0=1e-3, lambda_reg=0.01), pb)
        ts, te = [], []
        for _ in range(3):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            st.upload(pb)
            t1 = time.perf_counter()
            api.run_epoch(st)
            t2 = time.perf_counter()
            ts.append(t1 - t0); te.append(t2 - t1)
        print(f"round {rnd} [{s}] upload ms {[round(1e3*x,1) for x in ts]} first epoch ms {[round(1e3*x,1) for x in te]}", flush=True)
        st.close(); del st
        gc.collect(); torch.cuda.empty_cache()
