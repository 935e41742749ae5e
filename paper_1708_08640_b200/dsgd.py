"""DSGD across GPUs (BASELINE.json north_star).

Stratification: mode-1 and mode-2 index ranges are split into G blocks
balanced by observation count.  Rank p owns mode-1 block p; in sub-epoch t it
sweeps the stratum (p, (p+t) mod G), so concurrently processed strata touch
disjoint U1 and U2 rows.  The core, the remaining ("shared") modes and the
coupled factors are replicated; after every sub-epoch the ranks all-reduce
the deltas of the replicated parameters and of the rotating U2 blocks
(NCCL over NVLink, inside the C library), and U1 at the end of the epoch.

Coupled matrices: entries of a matrix on mode 1 follow the mode-1 owner
(spread over its sub-epochs), entries of a matrix on mode 2 are processed by
whoever holds their U2 block in one sub-epoch, entries of matrices on other
modes are spread over ranks and sub-epochs.

This module is host logic only: the sweeps, the delta reductions and the
NCCL calls run in libcmtf_b200.so (cmtf_gpu_sweep_range, cmtf_gpu_sync,
cmtf_gpu_sync_local).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Sequence, Tuple

import numpy as np

from . import _abi
from .api import (CoupledMatrix, DataBundle, SparseTensor, TrainConfig, TrainState, _ptr,
                  _raise)


def balanced_blocks(counts: np.ndarray, G: int) -> np.ndarray:
    """Block id per row: G contiguous index ranges with ~equal total count."""
    counts = np.asarray(counts, dtype=np.float64)
    total = counts.sum()
    if total <= 0 or G == 1:
        return np.zeros(counts.shape[0], dtype=np.int64)
    cum = np.cumsum(counts) - counts / 2.0
    return np.minimum((cum * G / total).astype(np.int64), G - 1)


def _hash(x: np.ndarray, salt: int) -> np.ndarray:
    v = (x.astype(np.uint64) + np.uint64(salt)) * np.uint64(0x9E3779B97F4A7C15)
    v ^= v >> np.uint64(31)
    return v


@dataclass
class RankPlan:
    """Rank-local bundle grouped by stratum (caller order) and its ranges."""
    rank: int
    world: int
    bundle: DataBundle
    t_ranges: List[Tuple[int, int]]  # per sub-epoch t: [lo, hi) of tensor records
    m_ranges: List[List[Tuple[int, int]]]  # per sub-epoch t, per matrix m
    shared_modes: int  # damping mask: replicated modes updated concurrently
    sync_modes: int  # synced after every sub-epoch
    end_modes: int  # synced at the end of the epoch
    mat_mask: int


@dataclass
class Partition:
    world: int
    block1: np.ndarray
    block2: np.ndarray
    counts: List[np.ndarray]  # global tensor counts per mode
    col_counts: List[np.ndarray]  # global column counts per matrix
    nnz: int
    plans: List[RankPlan] = field(default_factory=list)


def partition(bundle: DataBundle, G: int, seed: int = 0) -> Partition:
    t = bundle.tensor
    N = t.order
    if N < 2:
        raise ValueError("DSGD needs order >= 2")
    counts = [np.bincount(t.indices[:, n], minlength=t.dims[n]).astype(np.uint32)
              for n in range(N)]
    col_counts = [np.bincount(m.indices[:, 1], minlength=m.cols).astype(np.uint32)
                  for m in bundle.matrices]
    b1 = balanced_blocks(counts[0], G)
    b2 = balanced_blocks(counts[1], G)
    part = Partition(G, b1, b2, counts, col_counts, t.nnz)
    eb1 = b1[t.indices[:, 0]]
    eb2 = b2[t.indices[:, 1]]
    estr = (eb2 - eb1) % G  # sub-epoch at which the owner of eb1 sweeps it
    rng = np.random.Generator(np.random.PCG64(seed + 12345))
    shuffle_key = rng.random(t.nnz)
    shared = 0
    for n in range(2, N):
        shared |= 1 << n
    mat_mask = (1 << len(bundle.matrices)) - 1
    for p in range(G):
        sel = np.nonzero(eb1 == p)[0]
        order = np.lexsort((shuffle_key[sel], estr[sel]))
        sel = sel[order]
        tb = np.bincount(estr[sel], minlength=G)
        tcut = np.concatenate([[0], np.cumsum(tb)])
        t_ranges = [(int(tcut[s]), int(tcut[s + 1])) for s in range(G)]
        mats, m_ranges = [], [[] for _ in range(G)]
        for mi, m in enumerate(bundle.matrices):
            e = np.arange(m.nnz)
            h = _hash(e, 7919 * (mi + 1))
            if m.coupled_mode == 0:
                keep = b1[m.indices[:, 0]] == p
                sub = (h % np.uint64(G)).astype(np.int64)
            elif m.coupled_mode == 1:
                q = b2[m.indices[:, 0]]  # the matrix rows index mode 2
                part_t = (h % np.uint64(G)).astype(np.int64)
                keep = (q - part_t) % G == p  # block q, part t -> rank (q - t) mod G
                sub = part_t
            else:
                keep = (h % np.uint64(G)).astype(np.int64) == p
                sub = ((h // np.uint64(G)) % np.uint64(G)).astype(np.int64)
            idx = np.nonzero(keep)[0]
            mkey = rng.random(m.nnz)
            o = np.lexsort((mkey[idx], sub[idx]))
            idx = idx[o]
            sb = np.bincount(sub[idx], minlength=G)
            cut = np.concatenate([[0], np.cumsum(sb)])
            for s in range(G):
                m_ranges[s].append((int(cut[s]), int(cut[s + 1])))
            mats.append(CoupledMatrix(m.coupled_mode, m.rows, m.cols, m.indices[idx],
                                      m.values[idx], m.weight))
        local = DataBundle(SparseTensor(t.dims, t.indices[sel], t.values[sel]), mats)
        part.plans.append(RankPlan(p, G, local, t_ranges, m_ranges, shared,
                                   sync_modes=shared | 0b10, end_modes=0b1,
                                   mat_mask=mat_mask))
    return part


class RankState:
    """A rank's device context: local bundle, global counts, shared set."""

    def __init__(self, part: Partition, p: int, config: TrainConfig):
        plan = part.plans[p]
        cfg = TrainConfig(**{**config.__dict__, "order_policy": "caller"})
        self.plan = plan
        self.state = TrainState(cfg, plan.bundle)
        self._set_counts(part)
        self.state.initialize()  # same seed on every rank: identical replicas
        L, h = self.state._L, self.state._h
        self.state._check(L.cmtf_gpu_set_shared(h, plan.world, plan.shared_modes,
                                                plan.mat_mask, part.nnz))

    def _set_counts(self, part: Partition):
        L, h = self.state._L, self.state._h
        for n, c in enumerate(part.counts):
            c = np.ascontiguousarray(c)
            self.state._check(L.cmtf_gpu_set_counts(h, n, _ptr(c, C.c_uint32), c.shape[0]))
        for m, c in enumerate(part.col_counts):
            c = np.ascontiguousarray(c)
            self.state._check(L.cmtf_gpu_set_counts(h, 100 + m, _ptr(c, C.c_uint32), c.shape[0]))

    def reupload(self, part: Partition):
        """Upload the local bundle again from host memory (keeps the model)."""
        self.state.upload(self.plan.bundle)
        self._set_counts(part)

    def sweep(self, t: int):
        lo, hi = self.plan.t_ranges[t]
        nm = len(self.plan.m_ranges[t])
        mlo = np.array([r[0] for r in self.plan.m_ranges[t]] or [0], dtype=np.uint64)
        mhi = np.array([r[1] for r in self.plan.m_ranges[t]] or [0], dtype=np.uint64)
        L, h = self.state._L, self.state._h
        self.state._check(L.cmtf_gpu_sweep_range(
            h, lo, hi, _ptr(mlo, C.c_uint64) if nm else None,
            _ptr(mhi, C.c_uint64) if nm else None))


def run_epoch_emulated(ranks: Sequence[RankState]):
    """One DSGD epoch with all G ranks on ONE device (sequential sweeps; the
    ranks never wait on each other), deltas reduced in-process."""
    G = len(ranks)
    L = ranks[0].state._L
    arr = (C.c_void_p * G)(*[r.state._h for r in ranks])
    plan = ranks[0].plan
    for t in range(G):
        for r in ranks:
            r.sweep(t)
        _raise(L.cmtf_gpu_sync_local(arr, G, plan.sync_modes, plan.mat_mask, 1),
               L.cmtf_gpu_last_error().decode())
    _raise(L.cmtf_gpu_sync_local(arr, G, plan.end_modes, 0, 0), L.cmtf_gpu_last_error().decode())
    for r in ranks:
        r.state._check(L.cmtf_gpu_end_epoch(r.state._h))


def _map_torch_nccl():
    """The C library resolves NCCL at first use from whatever libnccl.so.2 the
    process has mapped; importing torch first makes that PyTorch's copy."""
    import torch  # noqa: F401


def comm_init(rank_state: RankState, world: int, rank: int, unique_id: bytes):
    _map_torch_nccl()
    L, h = rank_state.state._L, rank_state.state._h
    buf = C.create_string_buffer(unique_id, 128)
    rank_state.state._check(L.cmtf_gpu_comm_init(h, world, rank, buf))


def new_unique_id() -> bytes:
    _map_torch_nccl()
    buf = C.create_string_buffer(128)
    L = _abi.lib()
    _raise(L.cmtf_gpu_comm_unique_id(buf), L.cmtf_gpu_last_error().decode())
    return buf.raw


def run_epoch_nccl(rank_state: RankState):
    """One DSGD epoch on this rank (one process per GPU); NCCL inside."""
    L, h = rank_state.state._L, rank_state.state._h
    plan = rank_state.plan
    for t in range(plan.world):
        rank_state.sweep(t)
        rank_state.state._check(L.cmtf_gpu_sync(h, plan.sync_modes, plan.mat_mask, 1))
    rank_state.state._check(L.cmtf_gpu_sync(h, plan.end_modes, 0, 0))
    rank_state.state._check(L.cmtf_gpu_end_epoch(h))
