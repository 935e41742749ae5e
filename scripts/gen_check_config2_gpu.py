import sys, time, numpy as np
sys.path.insert(0, '.')
import torch
from paper_1708_08640_b200 import synth_gpu, api
t0=time.time()
b, test = synth_gpu.generate(synth_gpu.config2(1.0), device="cuda:0")
print("gen", time.time()-t0, b.tensor.nnz, [m.nnz for m in b.matrices])
m = b.matrices[0]
ij = m.indices.long()
keys = ij[:,0]*m.rows + ij[:,1]
print("sym dup", keys.numel() - torch.unique(keys).numel(), "self", int((ij[:,0]==ij[:,1]).sum()))
st = api.make_state(api.TrainConfig(ranks=[10,10,10], eta0=1e-3, lambda_reg=0.01), b)
for e in range(10): api.run_epoch(st)
print("rmse", api.epoch_stats(st, 0.01).train_rmse, api.test_rmse(st, test.to_host()))
