"""Where an e2e step's time goes at config 5 @1e9 (run with CMTF_PREP_TIMING=1
for the upload phases): raw pinned H2D bandwidth, set_tensor, add_matrix,
run_epoch, epoch_stats."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1708_08640_b200 import api, synth_gpu
from paper_1708_08640_b200.api import _ptr

nnz = float(sys.argv[1]) if len(sys.argv) > 1 else 1e9
b, test = synth_gpu.generate(synth_gpu.config5(nnz, 10), device="cuda:0")
x = torch.empty(1 << 30, dtype=torch.uint8).pin_memory()
y = torch.empty(1 << 30, dtype=torch.uint8, device="cuda:0")
for _ in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter(); y.copy_(x, non_blocking=True)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
print(f"pinned H2D: {1.0 / dt:.1f} GB/s", flush=True)
t = b.tensor
hi, hv = t.indices.cpu().pin_memory(), t.values.cpu().pin_memory()
m = b.matrices[0]
mi, mv = m.indices.cpu().pin_memory(), m.values.cpu().pin_memory()
st = api.make_state(api.TrainConfig(ranks=[10, 10, 10], eta0=1e-3, lambda_reg=0.01), b)
del b, t
torch.cuda.empty_cache()
L, h = st._L, st._h
dims = np.ascontiguousarray(st.bundle.tensor.dims, dtype=np.uint32)
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st._check(L.cmtf_gpu_clear_matrices(h))
    st._check(L.cmtf_gpu_set_tensor(h, _ptr(dims, C.c_uint32), _ptr(hi, C.c_uint32),
                                    _ptr(hv, C.c_double), hv.shape[0]))
    t1 = time.perf_counter()
    st._check(L.cmtf_gpu_add_matrix(h, m.coupled_mode, m.rows, m.cols, _ptr(mi, C.c_uint32),
                                    _ptr(mv, C.c_double), mv.shape[0], m.weight))
    t2 = time.perf_counter()
    api.run_epoch(st)
    t3 = time.perf_counter()
    s = api.epoch_stats(st, 0.01)
    t4 = time.perf_counter()
    print(f"set_tensor {1e3*(t1-t0):.0f} ms  add_matrix {1e3*(t2-t1):.0f} ms  "
          f"run_epoch {1e3*(t3-t2):.0f} ms (device {st.last_epoch_timing()['total_ms']:.0f})  "
          f"epoch_stats {1e3*(t4-t3):.0f} ms", flush=True)
