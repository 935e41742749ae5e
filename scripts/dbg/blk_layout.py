import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
os.environ["CMTF_TM_BLOCKS"] = "4"
import numpy as np
from paper_1708_08640_b200 import api, synth
from paper_1708_08640_b200.api import TrainConfig
b, _, _ = synth.generate(synth.config5_small(120_000))
for pre in (False, True):
    st = api.make_state(TrainConfig(ranks=[10, 10, 10], eta0=1e-3, lambda_reg=0.01), b)
    if pre:
        st._record_order()
    for ep in range(3):
        api.run_epoch(st)
        order = st._record_order()
        idx = b.tensor.indices[order]
        s = (idx[:, 0].astype(np.int64) * 4 // b.tensor.dims[0]) * 4 + idx[:, 1].astype(np.int64) * 4 // b.tensor.dims[1]
        runs = s[np.r_[True, s[1:] != s[:-1]]]
        print("pre" if pre else "closed", ep, st.kernel_info()["blocks"], len(runs), runs[:20], flush=True)
    st.close()
