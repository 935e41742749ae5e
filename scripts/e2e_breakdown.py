import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1708_08640_b200 import api, synth
from paper_1708_08640_b200.api import CoupledMatrix, DataBundle, SparseTensor
b, test, _ = synth.generate(synth.config2(1.0))
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
t = b.tensor
pb = DataBundle(SparseTensor(t.dims, pin(t.indices), pin(t.values)),
                [CoupledMatrix(m.coupled_mode, m.rows, m.cols, pin(m.indices), pin(m.values), m.weight) for m in b.matrices])
st = api.make_state(api.TrainConfig(ranks=[10, 10, 10], eta0=1e-3, lambda_reg=0.01), pb)
api.run_epoch(st)
for k in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    L = st._L
    import ctypes as C
    dims = np.ascontiguousarray(pb.tensor.dims, dtype=np.uint32)
    st._check(L.cmtf_gpu_clear_matrices(st._h)); t1 = time.perf_counter()
    st._check(L.cmtf_gpu_set_tensor(st._h, api._ptr(dims, C.c_uint32), api._ptr(pb.tensor.indices, C.c_uint32), api._ptr(pb.tensor.values, C.c_double), pb.tensor.nnz)); t2 = time.perf_counter()
    for m in pb.matrices:
        st._check(L.cmtf_gpu_add_matrix(st._h, m.coupled_mode, m.rows, m.cols, api._ptr(m.indices, C.c_uint32), api._ptr(m.values, C.c_double), m.nnz, m.weight))
    t3 = time.perf_counter()
    api.run_epoch(st); t4 = time.perf_counter()
    s = api.epoch_stats(st, 0.01); t5 = time.perf_counter()
    api.run_epoch(st); t6 = time.perf_counter()
    print(f"clear {1e3*(t1-t0):.2f} set_tensor {1e3*(t2-t1):.2f} add_matrix {1e3*(t3-t2):.2f} epoch(+prepare) {1e3*(t4-t3):.2f} stats {1e3*(t5-t4):.2f} plain epoch {1e3*(t6-t5):.2f} ms", flush=True)
# raw pinned H2D bandwidth for the same bytes
x = torch.empty(int(t.indices.nbytes + t.values.nbytes), dtype=torch.uint8).pin_memory()
y = torch.empty_like(x, device="cuda")
for _ in range(3):
    torch.cuda.synchronize(); a0 = time.perf_counter()
    y.copy_(x, non_blocking=True); torch.cuda.synchronize(); a1 = time.perf_counter()
    print(f"raw pinned H2D {x.numel()/1e6:.0f} MB: {1e3*(a1-a0):.2f} ms = {x.numel()/(a1-a0)/1e9:.1f} GB/s", flush=True)
