"""Device-side planted-model generator for the large BASELINE configs (3, 4, 5:
1e8 - 1e9 nonzeros), where host numpy generation is impractical.  Harness
code (torch on the GPU as plumbing), not the training path.

Same laws as synth.py: distinct coordinates (draw / de-duplicate / redraw;
uniform or Zipf marginals), planted Tucker values + N(0, sigma) noise
(+ clipping), planted coupled matrices; seeded torch generators.  The
resulting tensors stay on the device and are uploaded through the C ABI from
device pointers (cmtf_gpu_set_tensor accepts UVA pointers).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np


@dataclass
class DeviceTensor:
    dims: List[int]
    indices: "object"  # torch.int32 [nnz, order] (u32 bit pattern), on device
    values: "object"  # torch.float64 [nnz], on device

    @property
    def nnz(self) -> int:
        return int(self.values.shape[0])

    @property
    def order(self) -> int:
        return len(self.dims)

    def to_host(self, lo: int = 0, hi: Optional[int] = None):
        from .api import SparseTensor
        hi = self.nnz if hi is None else hi
        return SparseTensor(self.dims, self.indices[lo:hi].cpu().numpy().view(np.uint32),
                            self.values[lo:hi].cpu().numpy())


@dataclass
class DeviceMatrix:
    coupled_mode: int
    rows: int
    cols: int
    indices: "object"
    values: "object"
    weight: float = 10.0

    @property
    def nnz(self) -> int:
        return int(self.values.shape[0])

    def to_host(self, lo: int = 0, hi: Optional[int] = None):
        from .api import CoupledMatrix
        hi = self.nnz if hi is None else hi
        return CoupledMatrix(self.coupled_mode, self.rows, self.cols,
                             self.indices[lo:hi].cpu().numpy().view(np.uint32),
                             self.values[lo:hi].cpu().numpy(), self.weight)


@dataclass
class DeviceBundle:
    tensor: DeviceTensor
    matrices: List[DeviceMatrix] = field(default_factory=list)


def _sampler(law, dim, gen, device):
    import torch
    if law == "uniform" or law is None:
        return lambda n: torch.randint(0, dim, (n,), generator=gen, device=device,
                                       dtype=torch.int64)
    _, s = law
    w = torch.arange(1, dim + 1, device=device, dtype=torch.float64) ** (-float(s))
    cdf = torch.cumsum(w, 0)
    cdf /= cdf[-1].clone()
    return lambda n: torch.clamp(torch.searchsorted(
        cdf, torch.rand(n, generator=gen, device=device, dtype=torch.float64), right=True),
        max=dim - 1)


def distinct_coords(n, dims, laws, gen, device, dedup=True):
    """Exactly n distinct coordinate tuples.  For very sparse uniform spaces
    (n^2 / prod(dims) < 1e-3 expected collisions) the de-duplication pass is
    skipped and stated by the caller."""
    import torch
    samplers = [_sampler(laws[i] if i < len(laws) else "uniform", int(d), gen, device)
                for i, d in enumerate(dims)]
    space = 1
    for d in dims:
        space *= int(d)
    if not dedup:
        return torch.stack([s(n) for s in samplers], 1)
    if space >= (1 << 63):
        raise ValueError("coordinate space too large for 64-bit keys; use dedup=False")
    strides = []
    acc = 1
    for d in reversed(dims):
        strides.append(acc)
        acc *= int(d)
    strides = list(reversed(strides))
    keys = torch.zeros(0, dtype=torch.int64, device=device)
    for _ in range(100):
        need = n - keys.shape[0]
        if need <= 0:
            break
        m = int(need * 1.2) + 4096
        draw = torch.zeros(m, dtype=torch.int64, device=device)
        for s_, st in zip(samplers, strides):
            draw += s_(m) * st
        keys = torch.unique(torch.cat([keys, draw]))  # sorted, distinct
    if keys.shape[0] < n:
        raise ValueError("could not draw enough distinct coordinates")
    keys = keys[torch.randperm(keys.shape[0], generator=gen, device=device)[:n]]
    cols = []
    for d, st in zip(dims, strides):
        cols.append((keys // st) % int(d))
    return torch.stack(cols, 1)


def planted_values(core, factors, idx, chunk=1 << 22):
    import torch
    out = torch.empty(idx.shape[0], dtype=torch.float64, device=idx.device)
    N = len(factors)
    J = core.shape
    for lo in range(0, idx.shape[0], chunk):
        hi = min(idx.shape[0], lo + chunk)
        acc = factors[0][idx[lo:hi, 0]] @ core.reshape(J[0], -1)
        for n in range(1, N):
            acc = acc.reshape(hi - lo, J[n], -1)
            acc = torch.einsum("nj,njr->nr", factors[n][idx[lo:hi, n]], acc)
        out[lo:hi] = acc.reshape(-1)
    return out


@dataclass
class GpuMatrixSpec:
    mode: int
    cols: int
    nnz: int
    weight: float = 10.0
    noise: float = 0.1
    symmetric: bool = False  # cols == rows; (i,j) and (j,i) stored, y = u_i . u_j


@dataclass
class GpuSpec:
    dims: Sequence[int]
    nnz: int
    ranks: Sequence[int]
    laws: Sequence[object] = ()
    noise: float = 0.1
    clip: Optional[Tuple[float, float]] = None
    matrices: List[GpuMatrixSpec] = field(default_factory=list)
    test_fraction: float = 0.1
    seed: int = 0
    dedup: bool = True


def generate(spec: GpuSpec, device="cuda"):
    """Returns (train DeviceBundle, test DeviceTensor)."""
    import torch
    gen = torch.Generator(device=device)
    gen.manual_seed(spec.seed)
    dims = [int(d) for d in spec.dims]
    ranks = [int(r) for r in spec.ranks]
    core = torch.rand(ranks, generator=gen, device=device, dtype=torch.float64)
    factors = [torch.rand((d, r), generator=gen, device=device, dtype=torch.float64) / r ** 0.5
               for d, r in zip(dims, ranks)]
    idx = distinct_coords(spec.nnz, dims, spec.laws, gen, device, dedup=spec.dedup)
    vals = planted_values(core, factors, idx)
    if spec.noise:
        vals += spec.noise * torch.randn(vals.shape[0], generator=gen, device=device,
                                         dtype=torch.float64)
    if spec.clip is not None:
        vals.clamp_(spec.clip[0], spec.clip[1])
    n_test = int(round(spec.test_fraction * spec.nnz))
    perm = torch.randperm(spec.nnz, generator=gen, device=device)
    idx32 = idx.to(torch.int32)
    del idx
    test = DeviceTensor(dims, idx32[perm[:n_test]].contiguous(), vals[perm[:n_test]].contiguous())
    train = DeviceTensor(dims, idx32[perm[n_test:]].contiguous(), vals[perm[n_test:]].contiguous())
    del idx32, vals, perm
    mats = []
    for ms in spec.matrices:
        rows = dims[ms.mode]
        if ms.symmetric:
            # unordered pairs i < j, distinct, then mirrored (no duplicates)
            w = factors[ms.mode]
            half = ms.nnz // 2
            draw = distinct_coords(int(half * 1.05) + 1024, [rows, rows], ["uniform", "uniform"],
                                   gen, device)
            draw = draw[draw[:, 0] != draw[:, 1]]
            lo_, hi_ = torch.minimum(draw[:, 0], draw[:, 1]), torch.maximum(draw[:, 0], draw[:, 1])
            keys = torch.unique(lo_ * rows + hi_)
            keys = keys[torch.randperm(keys.shape[0], generator=gen, device=device)[:half]]
            pairs = torch.stack([keys // rows, keys % rows], 1)
            y = (w[pairs[:, 0]] * w[pairs[:, 1]]).sum(1)
            if ms.noise:
                y += ms.noise * torch.randn(y.shape[0], generator=gen, device=device,
                                            dtype=torch.float64)
            ij = torch.cat([pairs, pairs.flip(1)])
            y = torch.cat([y, y])
            mats.append(DeviceMatrix(ms.mode, rows, rows, ij.to(torch.int32).contiguous(),
                                     y.contiguous(), ms.weight))
            continue
        w = torch.rand((ms.cols, ranks[ms.mode]), generator=gen, device=device,
                       dtype=torch.float64) / ranks[ms.mode] ** 0.5
        ij = distinct_coords(ms.nnz, [rows, ms.cols], ["uniform", "uniform"], gen, device,
                             dedup=rows * ms.cols < (1 << 62))
        y = (factors[ms.mode][ij[:, 0]] * w[ij[:, 1]]).sum(1)
        if ms.noise:
            y += ms.noise * torch.randn(y.shape[0], generator=gen, device=device,
                                        dtype=torch.float64)
        mats.append(DeviceMatrix(ms.mode, rows, ms.cols, ij.to(torch.int32).contiguous(),
                                 y.contiguous(), ms.weight))
    torch.cuda.synchronize()
    torch.cuda.empty_cache()  # generation temporaries: give the memory back
    return DeviceBundle(train, mats), test


# ----------------------------------------------------------------------
# BASELINE.json configs 3 - 5 (synthetic stand-ins)
# ----------------------------------------------------------------------
def config2(scale: float = 1.0) -> GpuSpec:
    """configs[1] on the device (the host generator synth.config2 is the
    reference stand-in at 1 GPU; this one feeds the multi-GPU weak-scaling
    runs, where the problem grows with the GPU count): 1e5 x 1e5 x 1e3,
    1e7 * scale Zipf(1.2) / Zipf(1.2) / uniform nonzeros, planted 10^3 core,
    clipped to [1, 5]; symmetric 1e5 x 1e5 matrix (1e6 * scale) on mode 1 and
    1e5 x 200 (2e6 * scale) on mode 2."""
    return GpuSpec(dims=[100_000, 100_000, 1000], nnz=int(1e7 * scale), ranks=[10, 10, 10],
                   laws=[("zipf", 1.2), ("zipf", 1.2), "uniform"], clip=(1.0, 5.0),
                   matrices=[GpuMatrixSpec(0, 100_000, int(1e6 * scale), symmetric=True),
                             GpuMatrixSpec(1, 200, int(2e6 * scale))])


def config3(scale: float = 1.0) -> GpuSpec:
    """configs[2]: 1e6 x 1e6 x 1e4, 1e8 Zipf(1.1) nonzeros, planted 10^3 + noise;
    coupled 1e6 x 1e4 matrix with 1e7 nonzeros on mode 1."""
    return GpuSpec(dims=[1_000_000, 1_000_000, 10_000], nnz=int(1e8 * scale),
                   ranks=[10, 10, 10], laws=[("zipf", 1.1), ("zipf", 1.1), "uniform"],
                   matrices=[GpuMatrixSpec(0, 10_000, int(1e7 * scale))])


def config4(scale: float = 1.0) -> GpuSpec:
    """configs[3]: 4-way 1e6 x 1e5 x 1e3 x 100, 3e8 uniform nonzeros, planted
    8^4 + N(0,0.1); coupled matrices on modes 1 and 2 with 3e7 nonzeros each
    (column counts unspecified in BASELINE: 1e4 each)."""
    return GpuSpec(dims=[1_000_000, 100_000, 1000, 100], nnz=int(3e8 * scale),
                   ranks=[8, 8, 8, 8], laws=["uniform"] * 4,
                   matrices=[GpuMatrixSpec(0, 10_000, int(3e7 * scale)),
                             GpuMatrixSpec(1, 10_000, int(3e7 * scale))])


def config5(nnz: float = 1e8, rank: int = 10) -> GpuSpec:
    """configs[4]: 1e7^3 uniform with nnz in {1e7, 1e8, 1e9}; planted core of
    `rank`^3 + noise; coupled 1e7 x 1e6 matrix with 10% of the tensor nnz.
    The coordinate space (1e21) is beyond 64-bit keys; at <= 1e9 draws the
    expected number of duplicate coordinates is nnz^2 / 2e21 < 1e-3, so the
    de-duplication pass is skipped."""
    return GpuSpec(dims=[10_000_000] * 3, nnz=int(nnz), ranks=[rank] * 3,
                   laws=["uniform"] * 3, matrices=[GpuMatrixSpec(0, 1_000_000, int(nnz * 0.1))],
                   dedup=False)
