"""First-order epoch check of the Hogwild epoch kernels: with a tiny step the
model moves by -eta * (sum of all per-entry gradients at the initial model),
whatever the visit order, so the epoch delta of every row / the core must
match that sum computed in float64 (numpy restatement of
src/gradients.cpp:130-248 at a frozen model).  Usage:
  CMTF_V3_TM=1 python scripts/tm_firstorder.py [scale]"""
import json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1708_08640_b200 import api, synth

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 0.02
spec = synth.config2(scale)
if os.environ.get("UNIFORM", "1") == "1":  # first order holds when no row is hit too often
    spec.laws = ["uniform"] * 3
    for M in spec.matrices:
        M.row_law = M.col_law = "uniform"
b, test, _ = synth.generate(spec)
J, lam, eta = 10, 0.01, float(os.environ.get("ETA", "1e-5"))
cfg = api.TrainConfig(ranks=[J] * 3, seed=0, eta0=eta, mu=0.1, lambda_reg=lam)
for kv in sys.argv[2:]:
    k, v = kv.split("=")
    setattr(cfg, k, type(getattr(cfg, k))(v))
st = api.make_state(cfg, b)
m0 = st.model
api.run_epoch(st)
m1 = st.model
G = m0.core.astype(np.float64).reshape(J, J, J)
U = [f.astype(np.float64) for f in m0.factors]
V = [v.astype(np.float64) for v in m0.couplings]
idx = b.tensor.indices.astype(np.int64)
x = b.tensor.values.astype(np.float32).astype(np.float64)
nnz = len(x)
cnt = [np.bincount(idx[:, n], minlength=b.tensor.dims[n]) for n in range(3)]
dU = [np.zeros_like(u) for u in U]
dV = [np.zeros_like(v) for v in V]
dG = np.zeros_like(G)
for s in range(0, nnz, 200000):
    i, j, k = idx[s:s + 200000].T
    u1, u2, u3 = U[0][i], U[1][j], U[2][k]
    T = np.einsum("abc,ec->eab", G, u3)
    W1 = np.einsum("eab,eb->ea", T, u2)
    g2 = np.einsum("eab,ea->eb", T, u1)
    g3 = np.einsum("abc,ea,eb->ec", G, u1, u2)
    r = x[s:s + 200000] - np.einsum("ea,ea->e", W1, u1)
    for n, (ii, gr, u) in enumerate(((i, W1, u1), (j, g2, u2), (k, g3, u3))):
        grad = -r[:, None] * gr + (lam / cnt[n][ii])[:, None] * u
        np.add.at(dU[n], ii, grad)
    dG += np.einsum("e,ea,eb,ec->abc", -r, u1, u2, u3)
dG += nnz * (lam / nnz) * G
for mi, M in enumerate(b.matrices):
    rr, cc = M.indices[:, 0].astype(np.int64), M.indices[:, 1].astype(np.int64)
    y = M.values.astype(np.float32).astype(np.float64)
    ccnt = np.bincount(cc, minlength=M.cols)
    u, v = U[M.coupled_mode][rr], V[mi][cc]
    res = y - np.einsum("ek,ek->e", u, v)
    np.add.at(dU[M.coupled_mode], rr, -M.weight * res[:, None] * v)
    np.add.at(dV[mi], cc, -M.weight * res[:, None] * u + (M.weight * lam / ccnt[cc])[:, None] * v)
out = {"kernel": st.kernel_info()["kernel"], "eta": eta, "nnz": nnz}
def cmp(name, got, want):
    want = -eta * want
    err = np.abs(got - want)
    sc = np.abs(want).max()
    out[name] = {"max_err_rel_to_max": float(err.max() / sc), "rel_l2": float(np.linalg.norm(err) / np.linalg.norm(want))}
cmp("core", m1.core.reshape(J, J, J) - m0.core.reshape(J, J, J), dG)
for n in range(3):
    cmp(f"U{n + 1}", m1.factors[n].astype(np.float64) - U[n], dU[n])
for mi in range(len(V)):
    cmp(f"V{mi + 1}", m1.couplings[mi].astype(np.float64) - V[mi], dV[mi])
print(json.dumps(out))
