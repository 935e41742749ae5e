"""Reference-shaped host API over the C ABI.

Mirrors the reference's C++ entry points (namespace cmtf,
/root/reference/proj/core/include/cmtf/*.hpp): the same names, argument
meaning and error behaviour, so parity tests read like the reference's own
tests.  All compute goes through libcmtf_b200.so (CUDA, sm_100a); there is
no CPU path here.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _abi


class CmtfError(RuntimeError):
    pass


class ParseError(CmtfError):
    """errors.hpp:10-14"""


class ValidationError(CmtfError):
    """errors.hpp:16-20"""


class DivergenceError(CmtfError):
    """errors.hpp:22-26"""


class CudaError(CmtfError):
    pass


class UnsupportedError(ValidationError):
    pass


def _raise(rc: int, msg: str):
    if rc == _abi.OK:
        return
    cls = {
        _abi.EVALIDATION: ValidationError,
        _abi.EDIVERGENCE: DivergenceError,
        _abi.ECUDA: CudaError,
        _abi.ENCCL: CudaError,
        _abi.EUNSUPPORTED: UnsupportedError,
        _abi.EPARSE: ParseError,
    }.get(rc, CmtfError)
    raise cls(msg)


def _ptr(a, t):
    """Pointer to a numpy array (host) or a contiguous torch tensor (host or
    device; the C ABI resolves device pointers through UVA)."""
    if hasattr(a, "data_ptr"):
        return C.cast(C.c_void_p(a.data_ptr()), C.POINTER(t))
    return a.ctypes.data_as(C.POINTER(t))


# ----------------------------------------------------------------------
# Boundary types (include/cmtf/sparse_data.hpp:17-84)
# ----------------------------------------------------------------------
@dataclass
class SparseTensor:
    dims: Sequence[int]
    indices: np.ndarray  # (nnz, order) uint32, 0-based
    values: np.ndarray  # (nnz,) float64

    def __post_init__(self):
        self.dims = [int(d) for d in self.dims]
        self.indices = np.ascontiguousarray(self.indices, dtype=np.uint32).reshape(
            -1, len(self.dims))
        self.values = np.ascontiguousarray(self.values, dtype=np.float64).reshape(-1)
        if self.indices.shape[0] != self.values.shape[0]:
            raise ValidationError("index/value length mismatch")

    @property
    def order(self) -> int:
        return len(self.dims)

    @property
    def nnz(self) -> int:
        return int(self.values.shape[0])


@dataclass
class CoupledMatrix:
    coupled_mode: int  # 0-based
    rows: int
    cols: int
    indices: np.ndarray  # (nnz, 2) uint32
    values: np.ndarray
    weight: float = 10.0

    def __post_init__(self):
        self.indices = np.ascontiguousarray(self.indices, dtype=np.uint32).reshape(-1, 2)
        self.values = np.ascontiguousarray(self.values, dtype=np.float64).reshape(-1)

    @property
    def nnz(self) -> int:
        return int(self.values.shape[0])


@dataclass
class DataBundle:
    tensor: SparseTensor
    matrices: List[CoupledMatrix] = field(default_factory=list)


def make_bundle(tensor: SparseTensor, matrices: Sequence[CoupledMatrix] = ()) -> DataBundle:
    """make_bundle (src/sparse_data.cpp:364-375); counts are derived on the device."""
    for m in matrices:
        if m.coupled_mode >= tensor.order:
            raise ValidationError("coupled mode out of range")
        if m.rows != tensor.dims[m.coupled_mode]:
            raise ValidationError(
                f"coupled matrix row space does not match mode {m.coupled_mode + 1}")
    return DataBundle(tensor, list(matrices))


@dataclass
class TrainConfig:
    """TrainConfig (include/cmtf/trainer.hpp:18-36) + device fields."""
    ranks: Sequence[int] = ()
    eta0: float = 1e-3
    mu: float = 0.1
    lambda_reg: float = 0.1
    workers: int = 1
    max_epochs: int = 100
    rel_tol: float = 1e-4
    seed: int = 0
    kernel: str = "opt"  # "naive" | "opt"
    core_structure: str = "dense"
    nonnegative: bool = False
    init_scale: float = 1.0
    # device fields
    device: int = 0
    exec_mode: str = "hogwild"  # "hogwild" | "serial"
    hog_threads: int = 0
    sort_mode: int = -1
    force_generic: bool = False
    order_policy: str = "random"  # "random" | "sorted" | "caller"
    hot_tau: float = 0.0  # 0 = default 0.5, < 0 disables hot-row replicas
    kappa: float = 0.0  # 0 = default 0.5
    flush_every: int = 0  # 0 = default: 32 (tcgen05 kernel), 16 (others)
    kernel_version: int = 0  # 0 = auto (v2), 1 = v1
    core_flush_every: int = 0  # 0 = default: 1; 2 for the tcgen05 kernel on long sweeps (>= 2048 iterations per lane)
    kappa_core: float = 0.0  # 0 = default 2.0
    debug_count_visits: bool = False  # TrainConfig::debug_count_visits (trainer.hpp:31-32)

    def to_c(self):
        c = _abi.cmtf_gpu_config()
        _abi.lib().cmtf_gpu_config_default(C.byref(c))
        ranks = np.ascontiguousarray(self.ranks, dtype=np.uint32)
        c.order = len(ranks)
        c.ranks = _ptr(ranks, C.c_uint32)
        c.eta0, c.mu, c.lambda_reg = self.eta0, self.mu, self.lambda_reg
        c.workers, c.max_epochs, c.rel_tol = self.workers, self.max_epochs, self.rel_tol
        c.seed = self.seed
        c.kernel = _abi.KERNEL_OPT if self.kernel == "opt" else _abi.KERNEL_NAIVE
        c.core_structure = 0 if self.core_structure == "dense" else 1
        c.nonnegative = int(self.nonnegative)
        c.init_scale = self.init_scale
        c.device = self.device
        c.exec_mode = _abi.EXEC_SERIAL if self.exec_mode == "serial" else _abi.EXEC_HOGWILD
        c.hog_threads = self.hog_threads
        c.sort_mode = self.sort_mode
        c.force_generic = int(self.force_generic)
        c.order_policy = {"random": 1, "caller": 2}.get(self.order_policy, 0)
        c.hot_tau, c.kappa = self.hot_tau, self.kappa
        c.flush_every, c.kernel_version = self.flush_every, self.kernel_version
        c.core_flush_every = self.core_flush_every
        c.debug_count_visits = int(self.debug_count_visits)
        c.kappa_core = self.kappa_core
        return c, ranks


@dataclass
class FactorModel:
    """FactorModel (include/cmtf/tucker.hpp:103-107); core is row-major."""
    core: np.ndarray
    factors: List[np.ndarray]
    couplings: List[np.ndarray] = field(default_factory=list)
    coupling_modes: List[int] = field(default_factory=list)  # Coupling::mode (0-based)

    def copy(self) -> "FactorModel":
        return FactorModel(self.core.copy(), [f.copy() for f in self.factors],
                           [c.copy() for c in self.couplings], list(self.coupling_modes))


@dataclass
class EpochStats:
    train_rmse: float
    objective: float


# ----------------------------------------------------------------------
# Device state (TrainState, include/cmtf/trainer.hpp:49-56)
# ----------------------------------------------------------------------
class TrainState:
    """Owns a device context holding the bundle and the model."""

    def __init__(self, config: TrainConfig, bundle: DataBundle):
        if len(config.ranks) != bundle.tensor.order:  # src/trainer.cpp:62-66
            raise ValidationError(f"rank list has {len(config.ranks)} entries for a tensor "
                                  f"of order {bundle.tensor.order}")
        L = _abi.lib()
        self._L = L
        self.config = config
        self.bundle = bundle
        c, self._ranks = config.to_c()
        h = C.c_void_p()
        _raise(L.cmtf_gpu_create(C.byref(c), C.byref(h)),
               L.cmtf_gpu_last_error().decode())
        self._h = h
        self.upload(bundle)

    # -- bundle --------------------------------------------------------
    def _check(self, rc):
        if rc != _abi.OK:
            _raise(rc, self._L.cmtf_gpu_ctx_error(self._h).decode())

    def upload(self, bundle: DataBundle):
        t = bundle.tensor
        dims = np.ascontiguousarray(t.dims, dtype=np.uint32)
        self._check(self._L.cmtf_gpu_clear_matrices(self._h))
        self._check(self._L.cmtf_gpu_set_tensor(
            self._h, _ptr(dims, C.c_uint32), _ptr(t.indices, C.c_uint32),
            _ptr(t.values, C.c_double), t.nnz))
        for m in bundle.matrices:
            self._check(self._L.cmtf_gpu_add_matrix(
                self._h, m.coupled_mode, m.rows, m.cols, _ptr(m.indices, C.c_uint32),
                _ptr(m.values, C.c_double), m.nnz, m.weight))
        self.bundle = bundle

    def initialize(self):
        """make_state's initial model (src/trainer.cpp:94-103,130-137)."""
        self._check(self._L.cmtf_gpu_make_state(self._h))

    # -- model ---------------------------------------------------------
    def _shapes(self):
        ranks = [int(r) for r in self.config.ranks]
        t = self.bundle.tensor
        fac = [(t.dims[n], ranks[n]) for n in range(t.order)]
        cpl = [(m.cols, ranks[m.coupled_mode]) for m in self.bundle.matrices]
        return ranks, fac, cpl

    @property
    def _cp(self) -> bool:
        return self.config.core_structure != "dense"

    @property
    def model(self) -> FactorModel:
        """The model; a CP core comes back as its ranks[0] superdiagonal
        values (CoreTensor::stored() of a HyperDiagonalCp core)."""
        ranks, fac, cpl = self._shapes()
        core = np.zeros(ranks[0] if self._cp else int(np.prod(ranks)), dtype=np.float64)
        F = [np.zeros(s, dtype=np.float64) for s in fac]
        V = [np.zeros(s, dtype=np.float64) for s in cpl]
        fp = (f64p_t * max(1, len(F)))(*[_ptr(f, C.c_double) for f in F])
        vp = (f64p_t * max(1, len(V)))(*[_ptr(v, C.c_double) for v in V])
        self._check(self._L.cmtf_gpu_get_model(self._h, _ptr(core, C.c_double), fp, vp))
        return FactorModel(core if self._cp else core.reshape(ranks), F, V,
                           [m.coupled_mode for m in self.bundle.matrices])

    def finalized_model(self) -> FactorModel:
        """The tail of train() (src/trainer.cpp:342-345) on the current model:
        finalize_orthogonalize (src/tucker.cpp:226-283), or
        apply_nonnegative_projection in nonnegative mode.  Output only."""
        ranks, fac, cpl = self._shapes()
        core = np.zeros(int(np.prod(ranks)), dtype=np.float64)
        F = [np.zeros(s, dtype=np.float64) for s in fac]
        V = [np.zeros(s, dtype=np.float64) for s in cpl]
        fp = (f64p_t * max(1, len(F)))(*[_ptr(f, C.c_double) for f in F])
        vp = (f64p_t * max(1, len(V)))(*[_ptr(v, C.c_double) for v in V])
        self._check(self._L.cmtf_gpu_finalize_model(self._h, _ptr(core, C.c_double), fp, vp))
        if self._cp and self.config.nonnegative:  # the projection keeps the CP structure
            return FactorModel(core[: ranks[0]].copy(), F, V,
                               [m.coupled_mode for m in self.bundle.matrices])
        return FactorModel(core.reshape(ranks), F, V,
                           [m.coupled_mode for m in self.bundle.matrices])

    @model.setter
    def model(self, m: FactorModel):
        core = np.ascontiguousarray(m.core, dtype=np.float64).reshape(-1)
        F = [np.ascontiguousarray(f, dtype=np.float64) for f in m.factors]
        V = [np.ascontiguousarray(v, dtype=np.float64) for v in m.couplings]
        fp = (f64p_t * max(1, len(F)))(*[_ptr(f, C.c_double) for f in F])
        vp = (f64p_t * max(1, len(V)))(*[_ptr(v, C.c_double) for v in V])
        self._check(self._L.cmtf_gpu_set_model(self._h, _ptr(core, C.c_double), fp, vp))

    @property
    def epoch(self) -> int:
        e, eta = C.c_int32(), C.c_double()
        self._check(self._L.cmtf_gpu_get_state(self._h, C.byref(e), C.byref(eta)))
        return e.value

    @property
    def eta(self) -> float:
        e, eta = C.c_int32(), C.c_double()
        self._check(self._L.cmtf_gpu_get_state(self._h, C.byref(e), C.byref(eta)))
        return eta.value

    def set_state(self, epoch: int, eta: float):
        self._check(self._L.cmtf_gpu_set_state(self._h, epoch, eta))

    # -- introspection -------------------------------------------------
    def last_epoch_timing(self):
        ms = np.zeros(4)
        n = C.c_int32()
        self._check(self._L.cmtf_gpu_last_epoch_timing(self._h, _ptr(ms, C.c_double),
                                                        C.byref(n)))
        return {"tensor_ms": ms[0], "matrix_ms": ms[1], "scan_ms": ms[2],
                "total_ms": ms[3], "launches": n.value}

    def visit_counts(self):
        """TrainState::visit_counts of the last epoch: (per training entry in
        the caller's order, per record of the merged matrix stream)."""
        t = np.zeros(self.bundle.tensor.nnz, dtype=np.uint32)
        m = np.zeros(max(1, sum(x.nnz for x in self.bundle.matrices)), dtype=np.uint32)
        self._check(self._L.cmtf_gpu_visit_counts(self._h, _ptr(t, C.c_uint32),
                                                  _ptr(m, C.c_uint32)))
        return t, m[: sum(x.nnz for x in self.bundle.matrices)]

    def kernel_info(self):
        w, t, s = C.c_int32(), C.c_int32(), C.c_int32()
        self._check(self._L.cmtf_gpu_kernel_info(self._h, C.byref(w), C.byref(t),
                                                  C.byref(s)))
        return {"kernel": ["generic", "order3", "order4", "order3v2", "(retired)", "order3tm", "order4tm"][w.value],
                "hog_threads": t.value, "sort_mode": s.value, "blocks": self._blocks()}

    def _blocks(self):
        b = C.c_int32()
        self._check(self._L.cmtf_gpu_order_blocks(self._h, C.byref(b), None))
        return b.value

    def _record_order(self):
        """Entry ids in the current record order (introspection for tests)."""
        b = C.c_int32()
        pos = np.zeros(self.bundle.tensor.nnz, dtype=np.uint32)
        self._check(self._L.cmtf_gpu_order_blocks(self._h, C.byref(b), _ptr(pos, C.c_uint32)))
        order = np.empty_like(pos)
        order[pos] = np.arange(pos.size, dtype=np.uint32)
        return order

    def close(self):
        if getattr(self, "_h", None):
            self._L.cmtf_gpu_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


f64p_t = C.POINTER(C.c_double)


# ----------------------------------------------------------------------
# Free functions with the reference's names
# ----------------------------------------------------------------------
def make_state(config: TrainConfig, bundle: DataBundle) -> TrainState:
    """make_state (include/cmtf/trainer.hpp:72)."""
    s = TrainState(config, bundle)
    s.initialize()
    return s


def run_epoch(state: TrainState, bundle: Optional[DataBundle] = None,
              config: Optional[TrainConfig] = None) -> None:
    """run_epoch (include/cmtf/trainer.hpp:78-79, src/trainer.cpp:267-316)."""
    if bundle is not None and bundle is not state.bundle:
        state.upload(bundle)
    state._check(state._L.cmtf_gpu_run_epoch(state._h))


def epoch_stats(state: TrainState, lambda_reg: float) -> EpochStats:
    """epoch_stats (include/cmtf/eval.hpp:38-39, src/eval.cpp:120-144)."""
    r, o = C.c_double(), C.c_double()
    state._check(state._L.cmtf_gpu_epoch_stats(state._h, lambda_reg, C.byref(r),
                                               C.byref(o)))
    return EpochStats(r.value, o.value)


def test_rmse(state: TrainState, tensor: SparseTensor) -> float:
    """test_rmse (include/cmtf/eval.hpp:20-21, src/eval.cpp:101-107)."""
    out = C.c_double()
    state._check(state._L.cmtf_gpu_test_rmse(
        state._h, _ptr(tensor.indices, C.c_uint32), _ptr(tensor.values, C.c_double),
        tensor.nnz, C.byref(out)))
    return out.value


test_rmse.__test__ = False  # not a pytest test


def matrix_rmse(state: TrainState, coupling_index: int) -> float:
    out = C.c_double()
    state._check(state._L.cmtf_gpu_matrix_rmse(state._h, coupling_index, C.byref(out)))
    return out.value


@dataclass
class TrainResult:
    model: FactorModel
    log: List[tuple]
    state: TrainState


def train(bundle: DataBundle, config: TrainConfig) -> TrainResult:
    """train (src/trainer.cpp:318-346): epochs until convergence, then the
    reference's finalisation (orthogonalised factors, or the nonnegative
    projection); `state` keeps the un-finalised device model."""
    s = TrainState(config, bundle)
    cap = max(1, config.max_epochs)
    log = np.zeros(4 * cap)
    n = C.c_int32()
    s._check(s._L.cmtf_gpu_train(s._h, _ptr(log, C.c_double), cap, C.byref(n)))
    entries = [(int(log[4 * i]), log[4 * i + 1], log[4 * i + 2], log[4 * i + 3])
               for i in range(min(n.value, cap))]
    return TrainResult(s.finalized_model(), entries, s)


def entry_grads(state: TrainState, ids, with_core: bool = True):
    """Per-entry probe at the frozen device model (compute_gradient(_opt))."""
    ids = np.ascontiguousarray(ids, dtype=np.uint64)
    n = ids.shape[0]
    ranks = [int(r) for r in state.config.ranks]
    sumj, size = sum(ranks), int(np.prod(ranks))
    xhat, r = np.zeros(n), np.zeros(n)
    grow = np.zeros((n, sumj))
    gcore = np.zeros((n, size)) if with_core else None
    state._check(state._L.cmtf_gpu_entry_grads(
        state._h, _ptr(ids, C.c_uint64), n, _ptr(xhat, C.c_double), _ptr(r, C.c_double),
        _ptr(grow, C.c_double), _ptr(gcore, C.c_double) if with_core else None))
    return xhat, r, grow, gcore


def kernel_probe(state: TrainState):
    """The epoch kernel's own per-entry arithmetic at the frozen device model
    (order 3 opt, tcgen05 kernel): one eta = 0 sweep; returns x_hat [nnz],
    r [nnz], the row gradients [nnz, 3 J] and the summed core-gradient data
    term sum_e -r_e u1 (x) u2 (x) u3 [J, J, J].  Entries in caller order."""
    ranks = [int(r) for r in state.config.ranks]
    n = int(state.bundle.tensor.nnz)
    xhat, r = np.zeros(n), np.zeros(n)
    grow = np.zeros((n, sum(ranks)))
    gcore = np.zeros(ranks)
    state._check(state._L.cmtf_gpu_kernel_probe(
        state._h, _ptr(xhat, C.c_double), _ptr(r, C.c_double), _ptr(grow, C.c_double),
        _ptr(gcore, C.c_double)))
    return xhat, r, grow, gcore


def _compute_gradient(kernel: int, x, core, rows, lambda_reg, counts, nnz_total,
                      with_core=True, device=0, ranks=None, cp=False):
    core = np.ascontiguousarray(core, dtype=np.float64)
    if ranks is None:
        ranks = core.shape
    ranks = np.array(ranks, dtype=np.uint32)
    x = np.ascontiguousarray(np.atleast_1d(x), dtype=np.float64)
    n = x.shape[0]
    rows = np.ascontiguousarray(rows, dtype=np.float64).reshape(n, -1)
    counts = np.ascontiguousarray(counts, dtype=np.uint32).reshape(n, -1)
    sumj = int(ranks.sum())
    size = int(ranks[0]) if cp else int(np.prod(ranks))
    grow = np.zeros((n, sumj))
    gcore = np.zeros((n, size))
    res = np.zeros(n)
    L = _abi.lib()
    rc = L.cmtf_gpu_compute_gradient(
        kernel, len(ranks), _ptr(ranks, C.c_uint32), int(cp), _ptr(core, C.c_double), n,
        _ptr(x, C.c_double), _ptr(rows, C.c_double), _ptr(counts, C.c_uint32),
        lambda_reg, nnz_total, int(with_core), _ptr(grow, C.c_double),
        _ptr(gcore, C.c_double), _ptr(res, C.c_double), None, device)
    _raise(rc, L.cmtf_gpu_last_error().decode())
    return grow, gcore, res


def compute_gradient(x, core, rows, lambda_reg, counts, nnz_total, with_core=True,
                     device=0, ranks=None, cp=False):
    """Batched compute_gradient (include/cmtf/gradients.hpp:59-64).

    x: (n,), rows: (n, sum J) concatenated mode rows, counts: (n, N).
    cp: a CP core given as its superdiagonal (with `ranks`).
    Returns (row_grads (n, sumJ), core_grads (n, prod J | J), residuals (n,))."""
    return _compute_gradient(_abi.KERNEL_NAIVE, x, core, rows, lambda_reg, counts,
                             nnz_total, with_core, device, ranks, cp)


def compute_gradient_opt(x, core, rows, lambda_reg, counts, nnz_total, with_core=True,
                         device=0, ranks=None, cp=False):
    """Batched compute_gradient_opt (include/cmtf/gradients.hpp:69-74)."""
    return _compute_gradient(_abi.KERNEL_OPT, x, core, rows, lambda_reg, counts,
                             nnz_total, with_core, device, ranks, cp)


def matrix_entry_gradients(y, u, v, lambda_m, lambda_reg, col_count, device=0):
    """Batched matrix_entry_gradients (include/cmtf/gradients.hpp:83-86)."""
    y = np.ascontiguousarray(np.atleast_1d(y), dtype=np.float64)
    n = y.shape[0]
    u = np.ascontiguousarray(u, dtype=np.float64).reshape(n, -1)
    v = np.ascontiguousarray(v, dtype=np.float64).reshape(n, -1)
    j = u.shape[1]
    cc = np.ascontiguousarray(np.broadcast_to(col_count, (n,)), dtype=np.uint32)
    du, dv, r = np.zeros((n, j)), np.zeros((n, j)), np.zeros(n)
    L = _abi.lib()
    rc = L.cmtf_gpu_matrix_entry_gradients(
        n, j, _ptr(y, C.c_double), _ptr(u, C.c_double), _ptr(v, C.c_double), lambda_m,
        lambda_reg, _ptr(cc, C.c_uint32), _ptr(du, C.c_double), _ptr(dv, C.c_double),
        _ptr(r, C.c_double), device)
    _raise(rc, L.cmtf_gpu_last_error().decode())
    return du, dv, r
