"""epoch_stats / test_rmse time and value with the tcgen05 eval (default) and
the CUDA-core eval3_kernel (CMTF_EVAL_TM=0) on one workload, same model:
  python scripts/stats_ab.py config5 1e9 | config4 [scale] | config3 | config2"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1708_08640_b200 import api, synth, synth_gpu
which = sys.argv[1] if len(sys.argv) > 1 else "config5"
if which == "config5":
    spec = synth_gpu.config5(float(sys.argv[2]) if len(sys.argv) > 2 and "=" not in sys.argv[2] else 1e9, 10)
    b, test = synth_gpu.generate(spec, device="cuda:0")
elif which == "config3":
    b, test = synth_gpu.generate(synth_gpu.config3(1.0), device="cuda:0")
elif which == "config4":
    b, test = synth_gpu.generate(synth_gpu.config4(float(sys.argv[2]) if len(sys.argv) > 2 and "=" not in sys.argv[2] else 1.0), device="cuda:0")
else:
    b, test, _ = synth.generate(synth.config2(1.0))
out = {}
settings = [a for a in sys.argv[2:] if "=" in a] or ["CMTF_EVAL_TM=1", "CMTF_EVAL_TM=0"]
for tm in settings:
    for a in settings:
        os.environ.pop(a.split("=")[0], None)
    os.environ[tm.split("=")[0]] = tm.split("=")[1]
    st = api.make_state(api.TrainConfig(ranks=([8] * 4 if which == "config4" else [10, 10, 10]), seed=0, eta0=1e-3, lambda_reg=0.01), b)
    api.run_epoch(st)
    ts = []
    for _ in range(4):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        s = api.epoch_stats(st, 0.01)
        ts.append(time.perf_counter() - t0)
    t0 = time.perf_counter(); te = api.test_rmse(st, test); t1 = time.perf_counter()
    out[tm] = (s.train_rmse, s.objective, te)
    print(f"{which} {tm}: epoch_stats {1e3*min(ts):.2f} ms (min of 4), test_rmse {1e3*(t1-t0):.2f} ms; "
          f"train_rmse {s.train_rmse:.9f} objective {s.objective:.9e} test_rmse {te:.9f}", flush=True)
    st.close(); del st
