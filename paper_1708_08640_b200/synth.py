"""Deterministic planted-model generator for the BASELINE.json configurations.

The reference's own generator (src/synth.cpp:100-171) cannot express the
benchmark configs (no Zipf indices, clipping, symmetric or multiple coupled
matrices), so this one is written for them: seeded numpy PCG64 streams,
distinct coordinates by draw / de-duplicate / redraw, planted Tucker values
+ Gaussian noise (+ optional clipping), planted coupled matrices
y = u_i . w_j (+ noise).  The same arrays feed the GPU path and the CPU
oracle.  Host-side harness code, not part of the training path.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from .api import CoupledMatrix, DataBundle, SparseTensor


@dataclass
class MatrixSpec:
    mode: int  # 0-based coupled mode
    cols: int
    nnz: int
    weight: float = 10.0
    symmetric: bool = False  # cols == rows; store (i,j) and (j,i), planted u_i.u_j
    row_law: object = "uniform"  # "uniform" | ("zipf", s)
    col_law: object = "uniform"
    noise: float = 0.1


@dataclass
class PlantedSpec:
    dims: Sequence[int]
    nnz: int  # total observed tensor entries before the train/test split
    ranks: Sequence[int]  # planted ranks
    laws: Sequence[object] = ()  # per mode "uniform" | ("zipf", s)
    factor_law: str = "ref"  # "ref": U(0, 1/sqrt(J)) (src/trainer.cpp:43); "unit": U(0,1)
    noise: float = 0.1
    clip: Optional[Tuple[float, float]] = None
    matrices: List[MatrixSpec] = field(default_factory=list)
    test_fraction: float = 0.1
    seed: int = 0


def _sampler(law, dim: int, rng: np.random.Generator):
    if law == "uniform" or law is None:
        return lambda n: rng.integers(0, dim, n, dtype=np.int64)
    kind, s = law
    assert kind == "zipf"
    w = np.arange(1, dim + 1, dtype=np.float64) ** (-float(s))
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    return lambda n: np.minimum(np.searchsorted(cdf, rng.random(n), side="right"),
                                dim - 1).astype(np.int64)


def _keys(idx: np.ndarray, dims: Sequence[int]):
    total = 1
    for d in dims:
        total *= int(d)
    if total < (1 << 63):
        k = np.zeros(idx.shape[0], dtype=np.uint64)
        for n, d in enumerate(dims):
            k = k * np.uint64(d) + idx[:, n].astype(np.uint64)
        return k
    a = np.ascontiguousarray(idx.astype(np.uint32))
    return a.view(np.dtype((np.void, 4 * a.shape[1]))).reshape(-1)


def distinct_coords(n: int, dims: Sequence[int], laws: Sequence[object],
                    rng: np.random.Generator) -> np.ndarray:
    """Exactly n distinct coordinate tuples (draw, de-duplicate, redraw)."""
    samplers = [_sampler(laws[i] if i < len(laws) else "uniform", int(d), rng)
                for i, d in enumerate(dims)]
    have = np.zeros((0, len(dims)), dtype=np.int64)
    for _ in range(200):
        need = n - have.shape[0]
        if need <= 0:
            break
        m = int(need * 1.25) + 1024
        draw = np.stack([s(m) for s in samplers], axis=1)
        allc = np.concatenate([have, draw])
        _, first = np.unique(_keys(allc, dims), return_index=True)
        first.sort()  # keep the earlier draws first: deterministic and stable
        have = allc[first]
    if have.shape[0] < n:
        raise ValueError("could not draw enough distinct coordinates")
    keep = np.sort(rng.permutation(have.shape[0])[:n])
    return have[keep]


def planted_values(core: np.ndarray, factors: List[np.ndarray], idx: np.ndarray,
                   chunk: int = 1 << 20) -> np.ndarray:
    """x = G x_1 u1 x_2 u2 ... for each coordinate (factored, chunked)."""
    out = np.empty(idx.shape[0])
    N = len(factors)
    for lo in range(0, idx.shape[0], chunk):
        hi = min(idx.shape[0], lo + chunk)
        t = core.reshape(core.shape[0], -1)  # (J1, rest)
        acc = factors[0][idx[lo:hi, 0]] @ t  # (n, rest)
        for n in range(1, N):
            j = core.shape[n]
            acc = acc.reshape(hi - lo, j, -1)
            acc = np.einsum("nj,njr->nr", factors[n][idx[lo:hi, n]], acc)
        out[lo:hi] = acc.reshape(-1)
    return out


def generate(spec: PlantedSpec):
    """Returns (train DataBundle, test SparseTensor, truth dict)."""
    rng = np.random.Generator(np.random.PCG64(spec.seed))
    dims = [int(d) for d in spec.dims]
    ranks = [int(r) for r in spec.ranks]
    core = rng.random(ranks)
    if spec.factor_law == "unit":
        factors = [rng.random((d, r)) for d, r in zip(dims, ranks)]
    else:
        factors = [rng.random((d, r)) / np.sqrt(r) for d, r in zip(dims, ranks)]
    idx = distinct_coords(spec.nnz, dims, spec.laws, rng)
    vals = planted_values(core, factors, idx)
    if spec.noise:
        vals = vals + rng.normal(0.0, spec.noise, vals.shape[0])
    if spec.clip is not None:
        vals = np.clip(vals, spec.clip[0], spec.clip[1])
    perm = rng.permutation(idx.shape[0])
    n_test = int(round(spec.test_fraction * idx.shape[0]))
    test_ids, train_ids = perm[:n_test], perm[n_test:]
    train = SparseTensor(dims, idx[train_ids].astype(np.uint32), vals[train_ids])
    test = SparseTensor(dims, idx[test_ids].astype(np.uint32), vals[test_ids])

    mats = []
    truth_w = []
    for ms in spec.matrices:
        rows = dims[ms.mode]
        if ms.symmetric:
            if ms.cols != rows:
                raise ValueError("symmetric matrix must be square")
            # unordered pairs i < j, distinct, then mirrored: no duplicates
            half = np.zeros((0, 2), dtype=np.int64)
            need = ms.nnz // 2
            for _ in range(50):
                if half.shape[0] >= need:
                    break
                c = distinct_coords(2 * (need - half.shape[0]) + 64, [rows, rows],
                                    [ms.row_law, ms.col_law], rng)
                c = c[c[:, 0] != c[:, 1]]
                c = np.sort(c, axis=1)
                allc = np.concatenate([half, c])
                _, first = np.unique(allc[:, 0] * rows + allc[:, 1], return_index=True)
                half = allc[np.sort(first)]
            half = half[:need]
            w = factors[ms.mode]
            y = np.einsum("nj,nj->n", factors[ms.mode][half[:, 0]], w[half[:, 1]])
            if ms.noise:
                y = y + rng.normal(0.0, ms.noise, y.shape[0])
            ij = np.concatenate([half, half[:, ::-1]])
            y = np.concatenate([y, y])
        else:
            if spec.factor_law == "unit":
                w = rng.random((ms.cols, ranks[ms.mode]))
            else:
                w = rng.random((ms.cols, ranks[ms.mode])) / np.sqrt(ranks[ms.mode])
            ij = distinct_coords(ms.nnz, [rows, ms.cols], [ms.row_law, ms.col_law], rng)
            y = np.einsum("nj,nj->n", factors[ms.mode][ij[:, 0]], w[ij[:, 1]])
            if ms.noise:
                y = y + rng.normal(0.0, ms.noise, y.shape[0])
        truth_w.append(w)
        mats.append(CoupledMatrix(ms.mode, rows, ms.cols, ij.astype(np.uint32), y, ms.weight))
    bundle = DataBundle(train, mats)
    return bundle, test, {"core": core, "factors": factors, "couplings": truth_w}


# ----------------------------------------------------------------------
# BASELINE.json configurations (synthetic stand-ins)
# ----------------------------------------------------------------------
def config1(literal: bool = True) -> PlantedSpec:
    """configs[0]: 1000^3, 1e5 uniform nnz, core 5^3, factors U(0,1) (literal) or
    the reference law U(0,1/sqrt J); 1000x500 matrix on mode 1 with 1e4 nnz."""
    return PlantedSpec(dims=[1000, 1000, 1000], nnz=100_000, ranks=[5, 5, 5],
                       laws=["uniform"] * 3, factor_law="unit" if literal else "ref",
                       noise=0.1, matrices=[MatrixSpec(0, 500, 10_000, weight=10.0)],
                       test_fraction=0.1, seed=0)


def config2(scale: float = 1.0) -> PlantedSpec:
    """configs[1]: 1e5 x 1e5 x 1e3, 1e7 nnz, Zipf(1.2) on modes 1/2, planted 10^3,
    clipped to [1,5]; symmetric 1e5 x 1e5 (1e6 nnz) on mode 1 and 1e5 x 200
    (2e6 nnz) on mode 2.  `scale` shrinks every count for quick runs."""
    n = int(10_000_000 * scale)
    return PlantedSpec(
        dims=[100_000, 100_000, 1000], nnz=n, ranks=[10, 10, 10],
        laws=[("zipf", 1.2), ("zipf", 1.2), "uniform"], factor_law="ref", noise=0.1,
        clip=(1.0, 5.0),
        matrices=[MatrixSpec(0, 100_000, int(1_000_000 * scale), symmetric=True),
                  MatrixSpec(1, 200, int(2_000_000 * scale))],
        test_fraction=0.1, seed=0)


def config4_small(nnz: int = 160_000) -> PlantedSpec:
    """A CPU-oracle-sized stand-in for configs[3] (4-way, planted 8^4 core,
    uniform indices, coupled matrices on modes 1 and 2) used by the parity
    tests of the order-4 kernel: the same laws, dimensions shrunk so that a
    block sees about the same number of concurrent updates per row of the
    small modes as at full size (configs[3], mode 4: ~2.6 per iteration) and
    modes 1 / 2 keep ~9 / ~36 observations per row."""
    k = nnz / 40_000
    return PlantedSpec(dims=[int(4000 * k), int(1000 * k), 200, 100], nnz=nnz, ranks=[8, 8, 8, 8],
                       laws=["uniform"] * 4, factor_law="ref", noise=0.1,
                       matrices=[MatrixSpec(0, 200, nnz // 10), MatrixSpec(1, 200, nnz // 10)],
                       test_fraction=0.1, seed=0)


def config4(scale: float = 1.0) -> PlantedSpec:
    """configs[3] on the host (numpy): 4-way 1e6 x 1e5 x 1e3 x 100, 3e8 * scale
    uniform nonzeros, planted 8^4 core + N(0, 0.1); coupled matrices on modes 1
    and 2 (1e4 columns each, unspecified in BASELINE) with 3e7 * scale nonzeros
    each.  Used at scale 0.1 for the reference-vs-GPU parity run; the bench
    generates full size on the device (synth_gpu.config4)."""
    return PlantedSpec(dims=[1_000_000, 100_000, 1000, 100], nnz=int(3e8 * scale),
                       ranks=[8, 8, 8, 8], laws=["uniform"] * 4, factor_law="ref", noise=0.1,
                       matrices=[MatrixSpec(0, 10_000, int(3e7 * scale)),
                                 MatrixSpec(1, 10_000, int(3e7 * scale))],
                       test_fraction=0.1, seed=0)


def config3(scale: float = 1.0) -> PlantedSpec:
    """configs[2] on the host (numpy): 1e6 x 1e6 x 1e4, 1e8 * scale nonzeros
    with Zipf(1.1) mode-1/mode-2 indices and uniform mode 3, planted 10^3 core
    + N(0, 0.1) noise (no clipping is stated); one coupled 1e6 x 1e4 matrix on
    mode 1 with 1e7 * scale nonzeros.  The full-size run of the reference
    (scripts/oracle_config2.py --config config3) pins the GPU's 10-epoch RMSE;
    the bench generates the same laws on the device (synth_gpu.config3)."""
    return PlantedSpec(dims=[1_000_000, 1_000_000, 10_000], nnz=int(1e8 * scale),
                       ranks=[10, 10, 10], laws=[("zipf", 1.1), ("zipf", 1.1), "uniform"],
                       factor_law="ref", noise=0.1,
                       matrices=[MatrixSpec(0, 10_000, int(1e7 * scale))],
                       test_fraction=0.1, seed=0)


def config5_small(nnz: int = 1_000_000, rank: int = 10) -> PlantedSpec:
    """A CPU-reference-sized stand-in for configs[4] (uniform indices on three
    large modes, planted core + N(0, 0.1), one coupled matrix on mode 1 with
    10% of the tensor nonzeros): every row has ~nnz / 50_000 observations, so
    no row is hot and the tcgen05 epoch takes its bulk row-step path, as at
    full size.  Pins the config-5 kernel path against the reference's own
    threaded run (tests/golden/config5_small_reference.json)."""
    return PlantedSpec(dims=[50_000, 50_000, 50_000], nnz=int(nnz), ranks=[rank] * 3,
                       laws=["uniform"] * 3, factor_law="ref", noise=0.1,
                       matrices=[MatrixSpec(0, 5_000, int(nnz) // 10)],
                       test_fraction=0.1, seed=0)
