"""TEST INFRASTRUCTURE ONLY -- ctypes bindings for the CPU oracle.

Two libraries:
  * liboracle.so      -- the plain-C restatement (oracle/cmtf_oracle.c), always
                         available (built here and on the GPU box by make);
  * _ref/libcmtf_ref.so -- the UNMODIFIED reference sources + ref_shim.cpp,
                         built from /root/reference by oracle/Makefile in this
                         container; it travels to the GPU box prebuilt.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl
reference) may import this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libcmtf_ref.so")

u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
f64p = C.POINTER(C.c_double)
i32p = C.POINTER(C.c_int32)


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


def build():
    r = subprocess.run(["make", "-f", os.path.join(HERE, "Makefile")],
                       capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + r.stdout + r.stderr)


_orc = None
_ref = None


def orc():
    global _orc
    if _orc is None:
        if not os.path.exists(ORACLE_SO):
            build()
        _orc = C.CDLL(ORACLE_SO)
        _orc.orc_predict.restype = C.c_double
        _orc.orc_tensor_sse.restype = C.c_double
        _orc.orc_split_perm.restype = C.c_uint64
        _orc.orc_run_epoch.restype = C.c_int
        _orc.orc_mt_next.restype = C.c_uint64
    return _orc


def ref_available() -> bool:
    return os.path.exists(REF_SO) or os.path.isdir("/root/reference/proj/core/src")


def ref():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            build()
        if not os.path.exists(REF_SO):
            raise RuntimeError("reference oracle unavailable (no /root/reference and no "
                               "prebuilt oracle/_ref/libcmtf_ref.so)")
        _ref = C.CDLL(REF_SO)
        _ref.ref_last_error.restype = C.c_char_p
        for n in ("ref_bundle_new", "ref_state_new", "ref_generate"):
            getattr(_ref, n).restype = C.c_void_p
        for n in ("ref_bundle_free", "ref_state_free", "ref_run_epoch", "ref_state_get_model",
                  "ref_state_set_model", "ref_state_info", "ref_epoch_stats",
                  "ref_test_rmse", "ref_train", "ref_bundle_sizes", "ref_bundle_get",
                  "ref_state_get_schedule", "ref_state_finalize"):
            getattr(_ref, n).argtypes = None
        _ref.ref_bundle_free.argtypes = [C.c_void_p]
        _ref.ref_state_free.argtypes = [C.c_void_p]
    return _ref


# ----------------------------------------------------------------------
# Structures for the C restatement
# ----------------------------------------------------------------------
class OrcBundle(C.Structure):
    _fields_ = [("order", C.c_int32), ("cp", C.c_int32), ("dims", u32p), ("ranks", u32p),
                ("nnz", C.c_uint64), ("idx", u32p), ("vals", f64p), ("n_mat", C.c_int32),
                ("mat_mode", i32p), ("mat_cols", u32p), ("mat_nnz", u64p),
                ("mat_idx", C.POINTER(u32p)), ("mat_vals", C.POINTER(f64p)),
                ("mat_weight", f64p)]


class OrcModel(C.Structure):
    _fields_ = [("core", f64p), ("factors", C.POINTER(f64p)), ("couplings", C.POINTER(f64p))]


class _Keep:
    """Holds numpy arrays alive while C structs point into them."""

    def __init__(self):
        self.items = []

    def __call__(self, a):
        self.items.append(a)
        return a


def _bundle_struct(bundle, ranks, cp=0):
    keep = _Keep()
    t = bundle.tensor
    dims = keep(np.ascontiguousarray(t.dims, dtype=np.uint32))
    rk = keep(np.ascontiguousarray(ranks, dtype=np.uint32))
    idx = keep(np.ascontiguousarray(t.indices, dtype=np.uint32))
    vals = keep(np.ascontiguousarray(t.values, dtype=np.float64))
    mats = bundle.matrices
    nm = len(mats)
    mode = keep(np.array([m.coupled_mode for m in mats] or [0], dtype=np.int32))
    cols = keep(np.array([m.cols for m in mats] or [0], dtype=np.uint32))
    mnnz = keep(np.array([m.nnz for m in mats] or [0], dtype=np.uint64))
    w = keep(np.array([m.weight for m in mats] or [0], dtype=np.float64))
    mi = [keep(np.ascontiguousarray(m.indices, dtype=np.uint32)) for m in mats]
    mv = [keep(np.ascontiguousarray(m.values, dtype=np.float64)) for m in mats]
    mip = keep((u32p * max(1, nm))(*[_p(a, C.c_uint32) for a in mi]))
    mvp = keep((f64p * max(1, nm))(*[_p(a, C.c_double) for a in mv]))
    b = OrcBundle(len(t.dims), cp, _p(dims, C.c_uint32), _p(rk, C.c_uint32), t.nnz,
                  _p(idx, C.c_uint32), _p(vals, C.c_double), nm, _p(mode, C.c_int32),
                  _p(cols, C.c_uint32), _p(mnnz, C.c_uint64), mip, mvp, _p(w, C.c_double))
    return b, keep


class OracleModel:
    """A double-precision model the C oracle updates in place."""

    def __init__(self, bundle, ranks, cp=0):
        ranks = [int(r) for r in ranks]
        self.ranks = ranks
        t = bundle.tensor
        self.core = np.zeros(ranks[0] if cp else int(np.prod(ranks)))
        self.factors = [np.zeros((t.dims[n], ranks[n])) for n in range(t.order)]
        self.couplings = [np.zeros((m.cols, ranks[m.coupled_mode])) for m in bundle.matrices]

    def struct(self):
        keep = _Keep()
        fp = keep((f64p * max(1, len(self.factors)))(*[_p(f, C.c_double) for f in self.factors]))
        vp = keep((f64p * max(1, len(self.couplings)))(
            *[_p(v, C.c_double) for v in self.couplings]))
        return OrcModel(_p(self.core, C.c_double), fp, vp), keep

    def copy_from(self, m):
        self.core[:] = np.asarray(m.core).reshape(-1)
        for a, b in zip(self.factors, m.factors):
            a[:] = b
        for a, b in zip(self.couplings, m.couplings):
            a[:] = b
        return self


def mt_stream(seed, stream, index, n):
    """First n outputs of make_rng(seed, stream, index) (src/rng.cpp:17-26)."""

    class Mt(C.Structure):
        _fields_ = [("mt", C.c_uint64 * 312), ("mti", C.c_int)]

    g = Mt()
    orc().orc_make_rng(C.byref(g), C.c_uint64(seed), C.c_uint64(stream), C.c_uint64(index))
    return np.array([orc().orc_mt_next(C.byref(g)) for _ in range(n)], dtype=np.uint64)


def initialize(bundle, ranks, seed, scale=1.0, cp=0):
    b, k1 = _bundle_struct(bundle, ranks, cp)
    m = OracleModel(bundle, ranks, cp)
    ms, k2 = m.struct()
    orc().orc_initialize(C.byref(b), C.c_double(scale), C.c_uint64(seed), C.byref(ms))
    return m


def split_perm(nnz, frac, seed):
    ids = np.zeros(nnz, dtype=np.uint64)
    n_test = orc().orc_split_perm(C.c_uint64(nnz), C.c_double(frac), C.c_uint64(seed),
                                  _p(ids, C.c_uint64))
    return ids, int(n_test)


def shuffle(schedule, seed, epoch):
    orc().orc_shuffle(_p(schedule, C.c_uint64), C.c_uint64(schedule.shape[0]),
                      C.c_uint64(seed), C.c_int32(epoch))


def count_modes(bundle, ranks):
    b, k = _bundle_struct(bundle, ranks)
    total = sum(bundle.tensor.dims) + sum(m.cols for m in bundle.matrices)
    out = np.zeros(total, dtype=np.uint32)
    orc().orc_count_modes(C.byref(b), _p(out, C.c_uint32))
    return out


def predict(core, rows, cp=0):
    core = np.ascontiguousarray(core, dtype=np.float64)
    ranks = np.array(core.shape if not cp else [core.shape[0]] * len(rows), dtype=np.uint32)
    rows = [np.ascontiguousarray(r, dtype=np.float64) for r in rows]
    rp = (f64p * len(rows))(*[_p(r, C.c_double) for r in rows])
    return orc().orc_predict(len(rows), _p(ranks, C.c_uint32), cp,
                             _p(core.reshape(-1), C.c_double), rp)


def compute_gradient(opt, x, core, rows, lambda_reg, counts, nnz_total, with_core=True,
                     cp=0, ranks=None):
    core = np.ascontiguousarray(core, dtype=np.float64).reshape(-1)
    if ranks is None:
        ranks = [len(r) for r in rows]
    rk = np.ascontiguousarray(ranks, dtype=np.uint32)
    rows = [np.ascontiguousarray(r, dtype=np.float64) for r in rows]
    rp = (f64p * len(rows))(*[_p(r, C.c_double) for r in rows])
    cnt = np.ascontiguousarray(counts, dtype=np.uint32)
    grow = np.zeros(int(rk.sum()))
    gcore = np.zeros(core.shape[0])
    res = C.c_double()
    orc().orc_compute_gradient(C.c_int(opt), C.c_double(x), C.c_int(len(rows)),
                               _p(rk, C.c_uint32), C.c_int(cp), _p(core, C.c_double), rp,
                               C.c_double(lambda_reg), _p(cnt, C.c_uint32),
                               C.c_uint64(nnz_total), C.c_int(int(with_core)),
                               _p(grow, C.c_double), _p(gcore, C.c_double), C.byref(res))
    return grow, gcore, res.value


def matrix_entry_gradients(y, u, v, lambda_m, lambda_reg, col_count):
    u = np.ascontiguousarray(u, dtype=np.float64)
    v = np.ascontiguousarray(v, dtype=np.float64)
    j = u.shape[0]
    du, dv, r = np.zeros(j), np.zeros(j), C.c_double()
    orc().orc_matrix_entry_gradients(C.c_double(y), _p(u, C.c_double), _p(v, C.c_double),
                                     C.c_uint32(j), C.c_double(lambda_m),
                                     C.c_double(lambda_reg), C.c_uint32(col_count),
                                     _p(du, C.c_double), _p(dv, C.c_double), C.byref(r))
    return du, dv, r.value


def run_epoch(bundle, model: OracleModel, schedule, epoch, seed, eta, lambda_reg,
              kernel_opt=True, workers=1, nonneg=False, shuffle=True):
    b, k1 = _bundle_struct(bundle, model.ranks)
    ms, k2 = model.struct()
    return orc().orc_run_epoch(C.byref(b), C.byref(ms), _p(schedule, C.c_uint64),
                               C.c_int32(epoch), C.c_uint64(seed), C.c_double(eta),
                               C.c_double(lambda_reg), C.c_int32(int(kernel_opt)),
                               C.c_int32(workers), C.c_int32(int(nonneg)),
                               C.c_int32(int(shuffle)))


def epoch_stats(bundle, model: OracleModel, lambda_reg):
    b, k1 = _bundle_struct(bundle, model.ranks)
    ms, k2 = model.struct()
    r, o = C.c_double(), C.c_double()
    orc().orc_epoch_stats(C.byref(b), C.byref(ms), C.c_double(lambda_reg), C.byref(r),
                          C.byref(o))
    return r.value, o.value


def tensor_rmse(tensor, model: OracleModel):
    ranks = np.ascontiguousarray(model.ranks, dtype=np.uint32)
    fp = (f64p * len(model.factors))(*[_p(f, C.c_double) for f in model.factors])
    sse = orc().orc_tensor_sse(tensor.order, _p(ranks, C.c_uint32), 0,
                               _p(model.core, C.c_double), fp, C.c_uint64(tensor.nnz),
                               _p(tensor.indices, C.c_uint32),
                               _p(tensor.values, C.c_double))
    return float(np.sqrt(sse / tensor.nnz))


class SerialTrainer:
    """The reference's train loop at workers=P, serialised (oracle)."""

    def __init__(self, bundle, ranks, seed, eta0, mu, lambda_reg, kernel_opt=True,
                 workers=1, init_scale=1.0):
        self.bundle, self.seed = bundle, seed
        self.eta0, self.mu, self.lam = eta0, mu, lambda_reg
        self.kernel_opt, self.workers = kernel_opt, workers
        self.model = initialize(bundle, ranks, seed, init_scale)
        total = bundle.tensor.nnz + sum(m.nnz for m in bundle.matrices)
        self.schedule = np.arange(total, dtype=np.uint64)
        self.epoch, self.eta = 0, eta0

    def run_epoch(self):
        rc = run_epoch(self.bundle, self.model, self.schedule, self.epoch, self.seed,
                       self.eta, self.lam, self.kernel_opt, self.workers)
        self.epoch += 1
        self.eta = self.eta0 / (1.0 + self.mu * self.epoch)
        return rc


# ----------------------------------------------------------------------
# The reference itself (oracle/_ref), for golden vectors and the CPU arm
# ----------------------------------------------------------------------
class RefConfig(C.Structure):
    _fields_ = [("order", C.c_int32), ("ranks", u32p), ("eta0", C.c_double), ("mu", C.c_double),
                ("lambda_reg", C.c_double), ("workers", C.c_int32), ("max_epochs", C.c_int32),
                ("rel_tol", C.c_double), ("seed", C.c_uint64), ("kernel_opt", C.c_int32),
                ("cp", C.c_int32), ("nonnegative", C.c_int32), ("init_scale", C.c_double),
                ("eval_threads", C.c_int32)]


class RefRun:
    """A reference DataBundle + TrainState, driven through ref_shim.cpp."""

    def __init__(self, bundle, ranks, seed=0, eta0=1e-3, mu=0.1, lambda_reg=0.1, workers=1,
                 kernel_opt=True, max_epochs=100, rel_tol=1e-4, init_scale=1.0,
                 nonnegative=False, eval_threads=0, cp=False):
        L = ref()
        self.cp = bool(cp)
        self.L = L
        self.bundle = bundle
        self._keep = _Keep()
        t = bundle.tensor
        k = self._keep
        dims = k(np.ascontiguousarray(t.dims, dtype=np.uint32))
        idx = k(np.ascontiguousarray(t.indices, dtype=np.uint32))
        vals = k(np.ascontiguousarray(t.values, dtype=np.float64))
        mats = bundle.matrices
        nm = len(mats)
        mode = k(np.array([m.coupled_mode for m in mats] or [0], dtype=np.int32))
        cols = k(np.array([m.cols for m in mats] or [0], dtype=np.uint32))
        mnnz = k(np.array([m.nnz for m in mats] or [0], dtype=np.uint64))
        w = k(np.array([m.weight for m in mats] or [0], dtype=np.float64))
        mi = [k(np.ascontiguousarray(m.indices, dtype=np.uint32)) for m in mats]
        mv = [k(np.ascontiguousarray(m.values, dtype=np.float64)) for m in mats]
        mip = k((u32p * max(1, nm))(*[_p(a, C.c_uint32) for a in mi]))
        mvp = k((f64p * max(1, nm))(*[_p(a, C.c_double) for a in mv]))
        L.ref_bundle_new.argtypes = [C.c_int32, u32p, C.c_uint64, u32p, f64p, C.c_int32, i32p,
                                     u32p, u64p, C.POINTER(u32p), C.POINTER(f64p), f64p]
        self.b = L.ref_bundle_new(len(t.dims), _p(dims, C.c_uint32), t.nnz,
                                  _p(idx, C.c_uint32), _p(vals, C.c_double), nm,
                                  _p(mode, C.c_int32), _p(cols, C.c_uint32),
                                  _p(mnnz, C.c_uint64), mip, mvp, _p(w, C.c_double))
        if not self.b:
            raise ValueError(L.ref_last_error().decode())
        self.ranks = k(np.ascontiguousarray(ranks, dtype=np.uint32))
        self.cfg = RefConfig(len(ranks), _p(self.ranks, C.c_uint32), eta0, mu, lambda_reg,
                             workers, max_epochs, rel_tol, seed, int(kernel_opt), int(cp),
                             int(nonnegative), init_scale, eval_threads)
        L.ref_state_new.argtypes = [C.c_void_p, C.POINTER(RefConfig)]
        self.s = L.ref_state_new(self.b, C.byref(self.cfg))
        if not self.s:
            raise ValueError(L.ref_last_error().decode())

    def run_epoch(self):
        self.L.ref_run_epoch.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(RefConfig)]
        rc = self.L.ref_run_epoch(self.s, self.b, C.byref(self.cfg))
        if rc == 2:
            raise ArithmeticError(self.L.ref_last_error().decode())
        if rc:
            raise ValueError(self.L.ref_last_error().decode())

    def model(self):
        m = OracleModel(self.bundle, list(self.ranks))
        fp = (f64p * len(m.factors))(*[_p(f, C.c_double) for f in m.factors])
        vp = (f64p * max(1, len(m.couplings)))(*[_p(v, C.c_double) for v in m.couplings])
        self.L.ref_state_get_model.argtypes = [C.c_void_p, f64p, C.POINTER(f64p),
                                               C.POINTER(f64p)]
        self.L.ref_state_get_model(self.s, _p(m.core, C.c_double), fp, vp)
        if self.cp:  # CoreTensor::stored() of a CP core: the superdiagonal
            m.core = np.ascontiguousarray(m.core.reshape(-1)[: int(self.ranks[0])])
        return m

    def set_model(self, m):
        fp = (f64p * len(m.factors))(*[_p(f, C.c_double) for f in m.factors])
        vp = (f64p * max(1, len(m.couplings)))(*[_p(v, C.c_double) for v in m.couplings])
        self.L.ref_state_set_model.argtypes = [C.c_void_p, f64p, C.POINTER(f64p),
                                               C.POINTER(f64p)]
        core = np.ascontiguousarray(m.core, dtype=np.float64).reshape(-1)
        self.L.ref_state_set_model(self.s, _p(core, C.c_double), fp, vp)

    def finalize(self, nonneg=False):
        """The tail of the reference's train() on the state's model, in place."""
        self.L.ref_state_finalize.argtypes = [C.c_void_p, C.c_int32]
        rc = self.L.ref_state_finalize(self.s, int(nonneg))
        if rc != 0:
            raise RuntimeError(self.L.ref_last_error().decode())

    def info(self):
        e, eta = C.c_int32(), C.c_double()
        self.L.ref_state_info.argtypes = [C.c_void_p, i32p, f64p]
        self.L.ref_state_info(self.s, C.byref(e), C.byref(eta))
        return e.value, eta.value

    def schedule(self):
        total = self.bundle.tensor.nnz + sum(m.nnz for m in self.bundle.matrices)
        out = np.zeros(total, dtype=np.uint64)
        self.L.ref_state_get_schedule.argtypes = [C.c_void_p, u64p]
        self.L.ref_state_get_schedule(self.s, _p(out, C.c_uint64))
        return out

    def epoch_stats(self, lambda_reg, threads=1):
        r, o = C.c_double(), C.c_double()
        self.L.ref_epoch_stats.argtypes = [C.c_void_p, C.c_void_p, C.c_double, C.c_int32,
                                           f64p, f64p]
        self.L.ref_epoch_stats(self.s, self.b, lambda_reg, threads, C.byref(r), C.byref(o))
        return r.value, o.value

    def test_rmse(self, tensor, threads=1):
        out = C.c_double()
        dims = np.ascontiguousarray(tensor.dims, dtype=np.uint32)
        self.L.ref_test_rmse.argtypes = [C.c_void_p, C.c_int32, u32p, C.c_uint64, u32p, f64p,
                                         C.c_int32, f64p]
        rc = self.L.ref_test_rmse(self.s, len(tensor.dims), _p(dims, C.c_uint32), tensor.nnz,
                                  _p(tensor.indices, C.c_uint32),
                                  _p(tensor.values, C.c_double), threads, C.byref(out))
        if rc:
            raise ValueError(self.L.ref_last_error().decode())
        return out.value

    def close(self):
        if getattr(self, "s", None):
            self.L.ref_state_free(self.s)
            self.s = None
        if getattr(self, "b", None):
            self.L.ref_bundle_free(self.b)
            self.b = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def ref_compute_gradient(opt, x, core, rows, lambda_reg, counts, nnz_total, with_core=True,
                         cp=0, ranks=None):
    L = ref()
    core = np.ascontiguousarray(core, dtype=np.float64).reshape(-1)
    if ranks is None:
        ranks = [len(r) for r in rows]
    rk = np.ascontiguousarray(ranks, dtype=np.uint32)
    rows = [np.ascontiguousarray(r, dtype=np.float64) for r in rows]
    rp = (f64p * len(rows))(*[_p(r, C.c_double) for r in rows])
    cnt = np.ascontiguousarray(counts, dtype=np.uint32)
    grow = np.zeros(int(rk.sum()))
    gcore = np.zeros(core.shape[0])
    res = C.c_double()
    L.ref_compute_gradient.argtypes = [C.c_int32, C.c_double, C.c_int32, u32p, C.c_int32,
                                       f64p, C.POINTER(f64p), C.c_double, u32p, C.c_uint64,
                                       C.c_int32, f64p, f64p, f64p]
    rc = L.ref_compute_gradient(int(opt), x, len(rows), _p(rk, C.c_uint32), cp,
                                _p(core, C.c_double), rp, lambda_reg, _p(cnt, C.c_uint32),
                                nnz_total, int(with_core), _p(grow, C.c_double),
                                _p(gcore, C.c_double), C.byref(res))
    if rc:
        raise ValueError(L.ref_last_error().decode())
    return grow, gcore, res.value


def ref_matrix_entry_gradients(y, u, v, lambda_m, lambda_reg, col_count):
    L = ref()
    u = np.ascontiguousarray(u, dtype=np.float64)
    v = np.ascontiguousarray(v, dtype=np.float64)
    j = u.shape[0]
    du, dv, r = np.zeros(j), np.zeros(j), C.c_double()
    L.ref_matrix_entry_gradients.argtypes = [C.c_double, f64p, f64p, C.c_uint32, C.c_double,
                                             C.c_double, C.c_uint32, f64p, f64p, f64p]
    L.ref_matrix_entry_gradients(y, _p(u, C.c_double), _p(v, C.c_double), j, lambda_m,
                                 lambda_reg, col_count, _p(du, C.c_double),
                                 _p(dv, C.c_double), C.byref(r))
    return du, dv, r.value


def ref_shuffle(schedule, seed, epoch):
    L = ref()
    L.ref_shuffle.argtypes = [u64p, C.c_uint64, C.c_uint64, C.c_int32]
    L.ref_shuffle(_p(schedule, C.c_uint64), schedule.shape[0], seed, epoch)


def ref_split(tensor, frac, seed):
    L = ref()
    nnz, order = tensor.nnz, tensor.order
    tr_i = np.zeros((nnz, order), dtype=np.uint32)
    tr_v = np.zeros(nnz)
    te_i = np.zeros((nnz, order), dtype=np.uint32)
    te_v = np.zeros(nnz)
    n_test = C.c_uint64()
    dims = np.ascontiguousarray(tensor.dims, dtype=np.uint32)
    L.ref_split.argtypes = [C.c_int32, u32p, C.c_uint64, u32p, f64p, C.c_double, C.c_uint64,
                            u32p, f64p, u32p, f64p, u64p]
    rc = L.ref_split(order, _p(dims, C.c_uint32), nnz, _p(tensor.indices, C.c_uint32),
                     _p(tensor.values, C.c_double), frac, seed, _p(tr_i, C.c_uint32),
                     _p(tr_v, C.c_double), _p(te_i, C.c_uint32), _p(te_v, C.c_double),
                     C.byref(n_test))
    if rc:
        raise ValueError(L.ref_last_error().decode())
    nt = n_test.value
    return (tr_i[: nnz - nt], tr_v[: nnz - nt]), (te_i[:nt], te_v[:nt])


def ref_generate(dims, n_entries, ranks, noise, seed, with_matrix=True, matrix_ratio=0.1,
                 coupled_mode=0, matrix_cols=0, matrix_weight=10.0):
    """The reference's own planted generator (src/synth.cpp:100-171)."""
    L = ref()
    d = np.ascontiguousarray(dims, dtype=np.uint32)
    rk = np.ascontiguousarray(ranks, dtype=np.uint32)
    L.ref_generate.argtypes = [C.c_int32, u32p, C.c_uint64, u32p, C.c_double, C.c_uint64,
                               C.c_int32, C.c_double, C.c_int32, C.c_uint32, C.c_double]
    h = L.ref_generate(len(dims), _p(d, C.c_uint32), n_entries, _p(rk, C.c_uint32), noise,
                       seed, int(with_matrix), matrix_ratio, coupled_mode, matrix_cols,
                       matrix_weight)
    if not h:
        raise ValueError(L.ref_last_error().decode())
    nnz, nm = C.c_uint64(), C.c_int32()
    mn = np.zeros(8, dtype=np.uint64)
    mc = np.zeros(8, dtype=np.uint32)
    L.ref_bundle_sizes.argtypes = [C.c_void_p, u64p, i32p, u64p, u32p]
    L.ref_bundle_sizes(h, C.byref(nnz), C.byref(nm), _p(mn, C.c_uint64), _p(mc, C.c_uint32))
    idx = np.zeros((nnz.value, len(dims)), dtype=np.uint32)
    vals = np.zeros(nnz.value)
    mi = [np.zeros((int(mn[m]), 2), dtype=np.uint32) for m in range(nm.value)]
    mv = [np.zeros(int(mn[m])) for m in range(nm.value)]
    mip = (u32p * max(1, nm.value))(*[_p(a, C.c_uint32) for a in mi])
    mvp = (f64p * max(1, nm.value))(*[_p(a, C.c_double) for a in mv])
    L.ref_bundle_get.argtypes = [C.c_void_p, u32p, f64p, C.POINTER(u32p), C.POINTER(f64p)]
    L.ref_bundle_get(h, _p(idx, C.c_uint32), _p(vals, C.c_double), mip, mvp)
    L.ref_bundle_free(h)
    mats = [dict(mode=coupled_mode, rows=int(dims[coupled_mode]), cols=int(mc[m]),
                 indices=mi[m], values=mv[m], weight=matrix_weight) for m in range(nm.value)]
    return idx, vals, mats


def run_epoch_counts(bundle, model: OracleModel, schedule, eta, lambda_reg, counts_concat,
                     nnz_global, kernel_opt=True):
    """One serial sweep over `schedule` with given GLOBAL counts (DSGD stratum)."""
    b, k1 = _bundle_struct(bundle, model.ranks)
    ms, k2 = model.struct()
    cc = np.ascontiguousarray(counts_concat, dtype=np.uint32)
    orc().orc_run_epoch_counts.restype = C.c_int
    return orc().orc_run_epoch_counts(
        C.byref(b), C.byref(ms), _p(schedule, C.c_uint64), C.c_int32(0), C.c_uint64(0),
        C.c_double(eta), C.c_double(lambda_reg), C.c_int32(int(kernel_opt)), C.c_int32(1),
        C.c_int32(0), C.c_int32(0), _p(cc, C.c_uint32), C.c_uint64(nnz_global),
        C.c_uint64(len(schedule)))


# ----------------------------------------------------------------------
# The reference's text formats (test infrastructure: golden fixtures)
# ----------------------------------------------------------------------
def ref_load(path, is_matrix=False, coupled_mode=1, weight=10.0, dims=None):
    """load_tensor / load_matrix of the reference.  Returns ("ok", dims,
    idx, vals) or (kind, message) with kind ParseError / ValidationError."""
    L = ref()
    code = C.c_int32()
    if is_matrix:
        d = np.ascontiguousarray(dims, dtype=np.uint32)
        L.ref_load_matrix.restype = C.c_void_p
        L.ref_load_matrix.argtypes = [C.c_char_p, C.c_int32, C.c_double, C.c_int32, u32p,
                                      C.POINTER(C.c_int32)]
        h = L.ref_load_matrix(os.fsencode(str(path)), coupled_mode, weight, len(d),
                              _p(d, C.c_uint32), C.byref(code))
    else:
        L.ref_load_tensor.restype = C.c_void_p
        L.ref_load_tensor.argtypes = [C.c_char_p, C.POINTER(C.c_int32)]
        h = L.ref_load_tensor(os.fsencode(str(path)), C.byref(code))
    if not h:
        kind = {1: "ParseError", 2: "ValidationError"}.get(code.value, "Error")
        return kind, L.ref_last_error().decode()
    order = C.c_int32()
    dd = np.zeros(64, dtype=np.uint32)
    nnz = C.c_uint64()
    L.ref_coo_info.argtypes = [C.c_void_p, C.c_int32, C.POINTER(C.c_int32), u32p,
                               C.POINTER(C.c_uint64)]
    L.ref_coo_info(h, int(is_matrix), C.byref(order), _p(dd, C.c_uint32), C.byref(nnz))
    idx = np.zeros(max(1, nnz.value * order.value), dtype=np.uint32)
    vals = np.zeros(max(1, nnz.value))
    L.ref_coo_get.argtypes = [C.c_void_p, C.c_int32, u32p, f64p]
    L.ref_coo_get(h, int(is_matrix), _p(idx, C.c_uint32), _p(vals, C.c_double))
    L.ref_coo_free.argtypes = [C.c_void_p, C.c_int32]
    L.ref_coo_free(h, int(is_matrix))
    n = nnz.value
    return ("ok", [int(x) for x in dd[: order.value]],
            idx[: n * order.value].reshape(n, order.value), vals[:n])


def ref_save_tensor(path, dims, idx, vals):
    L = ref()
    d = np.ascontiguousarray(dims, dtype=np.uint32)
    i = np.ascontiguousarray(idx, dtype=np.uint32)
    v = np.ascontiguousarray(vals, dtype=np.float64)
    L.ref_save_tensor.argtypes = [C.c_char_p, C.c_int32, u32p, C.c_uint64, u32p, f64p]
    rc = L.ref_save_tensor(os.fsencode(str(path)), len(d), _p(d, C.c_uint32), v.shape[0],
                           _p(i, C.c_uint32), _p(v, C.c_double))
    if rc:
        raise ValueError(L.ref_last_error().decode())


def ref_save_model(path, core, factors, couplings=(), coupling_modes=(), cp=False):
    L = ref()
    ranks = np.ascontiguousarray([f.shape[1] for f in factors], dtype=np.uint32)
    c = np.ascontiguousarray(core, dtype=np.float64).reshape(-1)
    fs = [np.ascontiguousarray(f, dtype=np.float64) for f in factors]
    rows = np.ascontiguousarray([f.shape[0] for f in fs], dtype=np.uint32)
    fp = (f64p * len(fs))(*[_p(f, C.c_double) for f in fs])
    cs = [np.ascontiguousarray(v, dtype=np.float64) for v in couplings]
    cm = np.ascontiguousarray(list(coupling_modes), dtype=np.int32)
    cr = np.ascontiguousarray([v.shape[0] for v in cs], dtype=np.uint32)
    cpp = (f64p * max(1, len(cs)))(*[_p(v, C.c_double) for v in cs])
    L.ref_save_model.argtypes = [C.c_char_p, C.c_int32, u32p, C.c_int32, f64p, u32p,
                                 C.POINTER(f64p), C.c_int32, C.POINTER(C.c_int32), u32p,
                                 C.POINTER(f64p)]
    rc = L.ref_save_model(os.fsencode(str(path)), len(ranks), _p(ranks, C.c_uint32), int(cp),
                          _p(c, C.c_double), _p(rows, C.c_uint32), fp, len(cs),
                          _p(cm, C.c_int32), _p(cr, C.c_uint32), cpp)
    if rc:
        raise ValueError(L.ref_last_error().decode())


def ref_load_model(path):
    """load_model of the reference: ("ok", order, n_factors, n_coupled) or
    (kind, message)."""
    L = ref()
    o, nf, nc = C.c_int32(), C.c_int32(), C.c_int32()
    L.ref_load_model.argtypes = [C.c_char_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                 C.POINTER(C.c_int32)]
    rc = L.ref_load_model(os.fsencode(str(path)), C.byref(o), C.byref(nf), C.byref(nc))
    if rc:
        return {1: "ParseError", 2: "ValidationError"}.get(rc, "Error"), L.ref_last_error().decode()
    return "ok", o.value, nf.value, nc.value
