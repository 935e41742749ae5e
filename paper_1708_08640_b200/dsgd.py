"""DSGD across GPUs (BASELINE.json north_star).

Stratification: the index ranges of the first `n_strat` modes (2: modes 1
and 2; 3: modes 1, 2 and 3 -- configs[4], whose three modes all have 1e7
rows) are cut into G contiguous blocks balanced by observation count.  Rank p
owns mode-1 block p for the whole epoch.  A step visits one stratum per rank,
and the strata of one step touch pairwise disjoint rows of every stratified
mode:

    n_strat = 2: G steps;  step t:      rank p sweeps (p, (p+t) % G)
    n_strat = 3: G^2 steps; step a*G+c: rank p sweeps (p, (p+a) % G, (p+c) % G)

Blocks move instead of being reduced: after each step the mode-2 (n_strat 2)
or mode-3 (n_strat 3) block a rank just updated goes to rank p-1 and the one
it needs next comes from rank p+1 (ncclSend / ncclRecv over NVLink,
cmtf_gpu_exchange_rows); for n_strat 3 the mode-2 block moves the same way
once every G steps.  After a full epoch every block is back with its
owner.  Only the replicated parameters -- the core, the modes that are not
stratified and the coupled factors -- are delta all-reduced
(cmtf_gpu_sync), every `sync_every` steps and at the end of the epoch.
consolidate() broadcasts every block from its owner so that all ranks hold
the whole model (evaluation, checkpoints).

Coupled matrices: entries of a matrix on a stratified mode are processed by
whichever rank holds their row's block at the step chosen by a hash of the
entry; entries of a matrix on a replicated mode are spread over ranks and
steps.  The damping of the replicated parameters counts the `world` ranks
updating them concurrently (cmtf_gpu_set_shared).

Partitioning runs where the data is: partition() on host numpy bundles (the
tests), partition_rank() with torch on the device for device-resident
bundles (the 1e9-entry bench: each rank keeps only its own entries).  This
module is host logic only: sweeps, reductions, rotations and NCCL calls run
in libcmtf_b200.so.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

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


def block_cuts(block: np.ndarray, G: int) -> List[int]:
    """Row ranges [cut[b], cut[b+1]) of contiguous blocks."""
    counts = np.bincount(block, minlength=G)
    return [0] + np.cumsum(counts).astype(np.int64).tolist()


def _hash(x, salt: int):
    v = (x.astype(np.uint64) + np.uint64(salt)) * np.uint64(0x9E3779B97F4A7C15)
    v ^= v >> np.uint64(31)
    return v


@dataclass
class Schedule:
    """The step structure shared by every rank."""
    world: int
    n_strat: int

    @property
    def steps(self) -> int:
        return self.world ** (self.n_strat - 1)

    def block(self, p: int, mode: int, step: int) -> int:
        """Block of stratified `mode` that rank p holds during `step`."""
        G = self.world
        if mode == 0:
            return p
        if self.n_strat == 2:
            return (p + step) % G
        a, c = divmod(step, G)
        return (p + (a if mode == 1 else c)) % G

    def rotations_after(self, step: int) -> List[int]:
        """Stratified modes whose blocks move to rank p-1 after `step`."""
        if self.n_strat == 2:
            return [1]
        out = [2]
        if step % self.world == self.world - 1:
            out.append(1)
        return out

    def step_of(self, p: int, blocks: Sequence[int]) -> int:
        """The step at which rank p holds `blocks` (of modes 1..n_strat-1)."""
        G = self.world
        if self.n_strat == 2:
            return (blocks[0] - p) % G
        return ((blocks[0] - p) % G) * G + (blocks[1] - p) % G


@dataclass
class RankPlan:
    """Rank-local bundle grouped by step (caller order) and its ranges."""
    rank: int
    world: int
    bundle: DataBundle
    t_ranges: List[Tuple[int, int]]  # per step: [lo, hi) of tensor records
    m_ranges: List[List[Tuple[int, int]]]  # per step, per matrix
    shared_modes: int  # replicated modes (damping + delta sync)
    mat_mask: int  # replicated coupled factors
    schedule: Schedule = None
    cuts: List[List[int]] = field(default_factory=list)  # per stratified mode

    # compatibility names
    @property
    def sync_modes(self) -> int:
        return self.shared_modes

    @property
    def end_modes(self) -> int:
        return 0


@dataclass
class Partition:
    world: int
    block1: np.ndarray
    block2: np.ndarray
    counts: List[np.ndarray]  # global tensor counts per mode
    col_counts: List[np.ndarray]  # global column counts per matrix
    nnz: int
    plans: List[RankPlan] = field(default_factory=list)
    n_strat: int = 2
    cuts: List[List[int]] = field(default_factory=list)
    blocks: List[np.ndarray] = field(default_factory=list)


def _matrix_assignment(schedule: Schedule, blocks: List[np.ndarray], m: CoupledMatrix, mi: int,
                       xp=np):
    """(rank, step) of every entry of matrix m (numpy or torch arrays)."""
    G, S = schedule.world, schedule.steps
    n = m.nnz
    if xp is np:
        e = np.arange(n, dtype=np.uint64)
        h = (_hash(e, 7919 * (mi + 1)) >> np.uint64(2)).astype(np.int64)
        rows = m.indices[:, 0].astype(np.int64)
    else:
        import torch
        e = torch.arange(n, device=m.indices.device, dtype=torch.int64)
        h = (e + 7919 * (mi + 1)) * 0x9E3779B9 % (1 << 31)
        rows = m.indices[:, 0].long()
    mode = m.coupled_mode
    if mode == 0:
        rank = blocks[0][rows]
        step = h % S
    elif mode < schedule.n_strat:
        q = blocks[mode][rows]
        if schedule.n_strat == 2:
            t = h % G
            rank = (q - t) % G
            step = t
        else:
            a, c = h % G, (h // G) % G
            if mode == 1:
                rank = (q - a) % G
            else:
                rank = (q - c) % G
            step = a * G + c
    else:
        rank = h % G
        step = (h // G) % S
    if xp is np:
        return rank.astype(np.int64), step.astype(np.int64)
    return rank, step


def _shared_masks(N: int, n_mat: int, n_strat: int) -> Tuple[int, int]:
    shared = 0
    for n in range(n_strat, N):
        shared |= 1 << n
    return shared, (1 << n_mat) - 1


def partition(bundle: DataBundle, G: int, seed: int = 0, n_strat: int = 2) -> Partition:
    """Host partition of a (numpy) bundle for all G ranks."""
    t = bundle.tensor
    N = t.order
    if N < n_strat:
        raise ValueError(f"stratifying {n_strat} modes needs order >= {n_strat}")
    counts = [np.bincount(t.indices[:, n], minlength=t.dims[n]).astype(np.uint32)
              for n in range(N)]
    col_counts = [np.bincount(m.indices[:, 1], minlength=m.cols).astype(np.uint32)
                  for m in bundle.matrices]
    blocks = [balanced_blocks(counts[n], G) for n in range(n_strat)]
    cuts = [block_cuts(b, G) for b in blocks]
    sch = Schedule(G, n_strat)
    part = Partition(G, blocks[0], blocks[1], counts, col_counts, t.nnz, n_strat=n_strat,
                     cuts=cuts, blocks=blocks)
    eb = [blocks[n][t.indices[:, n]] for n in range(n_strat)]
    if n_strat == 2:
        estep = (eb[1] - eb[0]) % G
    else:
        estep = ((eb[1] - eb[0]) % G) * G + (eb[2] - eb[0]) % G
    rng = np.random.Generator(np.random.PCG64(seed + 12345))
    shuffle_key = rng.random(t.nnz)
    shared, mat_mask = _shared_masks(N, len(bundle.matrices), n_strat)
    massign = [_matrix_assignment(sch, blocks, m, mi) for mi, m in enumerate(bundle.matrices)]
    mkeys = [rng.random(m.nnz) for m in bundle.matrices]
    S = sch.steps
    for p in range(G):
        sel = np.nonzero(eb[0] == p)[0]
        order = np.lexsort((shuffle_key[sel], estep[sel]))
        sel = sel[order]
        tb = np.bincount(estep[sel], minlength=S)
        tcut = np.concatenate([[0], np.cumsum(tb)])
        t_ranges = [(int(tcut[s]), int(tcut[s + 1])) for s in range(S)]
        mats, m_ranges = [], [[] for _ in range(S)]
        for mi, m in enumerate(bundle.matrices):
            rank, step = massign[mi]
            idx = np.nonzero(rank == p)[0]
            o = np.lexsort((mkeys[mi][idx], step[idx]))
            idx = idx[o]
            sb = np.bincount(step[idx], minlength=S)
            cut = np.concatenate([[0], np.cumsum(sb)])
            for s in range(S):
                m_ranges[s].append((int(cut[s]), int(cut[s + 1])))
            mats.append(CoupledMatrix(m.coupled_mode, m.rows, m.cols, m.indices[idx],
                                      m.values[idx], m.weight))
        local = DataBundle(SparseTensor(t.dims, t.indices[sel], t.values[sel]), mats)
        part.plans.append(RankPlan(p, G, local, t_ranges, m_ranges, shared, mat_mask, sch, cuts))
    return part


def partition_rank(bundle, G: int, p: int, seed: int = 0, n_strat: int = 2):
    """Device partition (torch) of a device-resident bundle
    (synth_gpu.DeviceBundle) for rank p only: returns (RankPlan with a
    device-resident local bundle, global counts, global column counts)."""
    import torch
    from .synth_gpu import DeviceBundle, DeviceMatrix, DeviceTensor
    t = bundle.tensor
    dev = t.indices.device
    N = len(t.dims)
    idx = t.indices
    counts = [torch.bincount(idx[:, n].long(), minlength=t.dims[n]) for n in range(N)]
    col_counts = [torch.bincount(m.indices[:, 1].long(), minlength=m.cols)
                  for m in bundle.matrices]
    blocks, cuts = [], []
    for n in range(n_strat):
        c = counts[n].double()
        tot = float(c.sum())
        cum = torch.cumsum(c, 0) - c / 2.0
        b = torch.clamp((cum * G / max(tot, 1.0)).long(), max=G - 1) if G > 1 else \
            torch.zeros_like(c, dtype=torch.long)
        blocks.append(b)
        cuts.append([0] + torch.cumsum(torch.bincount(b, minlength=G), 0).tolist())
    sch = Schedule(G, n_strat)
    S = sch.steps
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed + 12345 + p)
    eb0 = blocks[0][idx[:, 0].long()]
    sel = torch.nonzero(eb0 == p).squeeze(1)
    del eb0
    loc = idx[sel].long()
    eb = [blocks[n][loc[:, n]] for n in range(1, n_strat)]
    if n_strat == 2:
        step = (eb[0] - p) % G
    else:
        step = ((eb[0] - p) % G) * G + (eb[1] - p) % G
    key = step * (1 << 40) + torch.randint(0, 1 << 40, (sel.shape[0],), generator=gen, device=dev)
    o = torch.argsort(key)
    sel = sel[o]
    step = step[o]
    del key, o, loc, eb
    tb = torch.bincount(step, minlength=S)
    tcut = [0] + torch.cumsum(tb, 0).tolist()
    t_ranges = [(int(tcut[s]), int(tcut[s + 1])) for s in range(S)]
    local_t = DeviceTensor(t.dims, idx[sel].contiguous(), t.values[sel].contiguous())
    del sel, step
    mats, m_ranges = [], [[] for _ in range(S)]
    for mi, m in enumerate(bundle.matrices):
        rank, mstep = _matrix_assignment(sch, blocks, m, mi, xp=torch)
        ms = torch.nonzero(rank == p).squeeze(1)
        mstep = mstep[ms]
        k2 = mstep * (1 << 40) + torch.randint(0, 1 << 40, (ms.shape[0],), generator=gen,
                                                device=dev)
        o = torch.argsort(k2)
        ms, mstep = ms[o], mstep[o]
        sb = torch.bincount(mstep, minlength=S)
        cut = [0] + torch.cumsum(sb, 0).tolist()
        for s in range(S):
            m_ranges[s].append((int(cut[s]), int(cut[s + 1])))
        mats.append(DeviceMatrix(m.coupled_mode, m.rows, m.cols, m.indices[ms].contiguous(),
                                 m.values[ms].contiguous(), m.weight))
    shared, mat_mask = _shared_masks(N, len(bundle.matrices), n_strat)
    plan = RankPlan(p, G, DeviceBundle(local_t, mats), t_ranges, m_ranges, shared, mat_mask, sch,
                    cuts)
    hc = [c.to(torch.int64).cpu().numpy().astype(np.uint32) for c in counts]
    hcc = [c.to(torch.int64).cpu().numpy().astype(np.uint32) for c in col_counts]
    return plan, hc, hcc, int(t.nnz)


class RankState:
    """A rank's device context: local bundle, global counts, shared set."""

    def __init__(self, part_or_plan, p: int, config: TrainConfig, counts=None, col_counts=None,
                 nnz: Optional[int] = None):
        if isinstance(part_or_plan, Partition):
            plan = part_or_plan.plans[p]
            counts, col_counts, nnz = (part_or_plan.counts, part_or_plan.col_counts,
                                       part_or_plan.nnz)
        else:
            plan = part_or_plan
        cfg = TrainConfig(**{**config.__dict__, "order_policy": "caller"})
        self.plan = plan
        self.counts, self.col_counts, self.nnz = counts, col_counts, nnz
        self.state = TrainState(cfg, plan.bundle)
        self._set_counts()
        self.state.initialize()  # same seed on every rank: identical replicas
        L, h = self.state._L, self.state._h
        self.state._check(L.cmtf_gpu_set_shared(h, plan.world, plan.shared_modes,
                                                plan.mat_mask, nnz))

    def _set_counts(self):
        L, h = self.state._L, self.state._h
        for n, c in enumerate(self.counts):
            c = np.ascontiguousarray(c, dtype=np.uint32)
            self.state._check(L.cmtf_gpu_set_counts(h, n, _ptr(c, C.c_uint32), c.shape[0]))
        for m, c in enumerate(self.col_counts):
            c = np.ascontiguousarray(c, dtype=np.uint32)
            self.state._check(L.cmtf_gpu_set_counts(h, 100 + m, _ptr(c, C.c_uint32), c.shape[0]))

    def reupload(self, part=None):
        """Upload the local bundle again (keeps the model)."""
        self.state.upload(self.plan.bundle)
        self._set_counts()

    def sweep(self, t: int):
        lo, hi = self.plan.t_ranges[t]
        nm = len(self.plan.m_ranges[t])
        mlo = np.array([r[0] for r in self.plan.m_ranges[t]] or [0], dtype=np.uint64)
        mhi = np.array([r[1] for r in self.plan.m_ranges[t]] or [0], dtype=np.uint64)
        L, h = self.state._L, self.state._h
        self.state._check(L.cmtf_gpu_sweep_range(
            h, lo, hi, _ptr(mlo, C.c_uint64) if nm else None,
            _ptr(mhi, C.c_uint64) if nm else None))

    def block_rows(self, mode: int, b: int) -> Tuple[int, int]:
        c = self.plan.cuts[mode]
        return int(c[b]), int(c[b + 1])


def _sync_due(step: int, steps: int, sync_every: int) -> bool:
    return (step + 1) % sync_every == 0 or step + 1 == steps


def run_epoch_emulated(ranks: Sequence[RankState], sync_every: int = 1):
    """One DSGD epoch with all G ranks on ONE device (sequential sweeps; the
    ranks never wait on each other): replicated deltas reduced in-process,
    block rotations as device copies between the contexts."""
    G = len(ranks)
    L = ranks[0].state._L
    arr = (C.c_void_p * G)(*[r.state._h for r in ranks])
    plan = ranks[0].plan
    sch = plan.schedule
    for step in range(sch.steps):
        for r in ranks:
            r.sweep(step)
        if _sync_due(step, sch.steps, sync_every):
            _raise(L.cmtf_gpu_sync_local(arr, G, plan.shared_modes, plan.mat_mask, 1),
                   L.cmtf_gpu_last_error().decode())
        for mode in sch.rotations_after(step):
            # rank p's current block goes to rank p-1 (its next block)
            for p, r in enumerate(ranks):
                b = sch.block(p, mode, step)
                lo, hi = r.block_rows(mode, b)
                dst = ranks[(p - 1) % G]
                _raise(L.cmtf_gpu_exchange_rows_local(r.state._h, dst.state._h, mode, lo, hi),
                       L.cmtf_gpu_last_error().decode())
    for r in ranks:
        r.state._check(L.cmtf_gpu_end_epoch(r.state._h))


def consolidate_emulated(ranks: Sequence[RankState]):
    """Every rank gets every block of the stratified modes from its owner."""
    G = len(ranks)
    L = ranks[0].state._L
    sch = ranks[0].plan.schedule
    for mode in range(sch.n_strat):
        for b in range(G):
            lo, hi = ranks[b].block_rows(mode, b)
            for q in range(G):
                if q != b:
                    _raise(L.cmtf_gpu_exchange_rows_local(ranks[b].state._h, ranks[q].state._h,
                                                          mode, lo, hi),
                           L.cmtf_gpu_last_error().decode())


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


def run_epoch_nccl(rank_state: RankState, sync_every: int = 1):
    """One DSGD epoch on this rank (one process per GPU): stratum sweeps,
    replicated-delta all-reduces and block rotations (ncclSend / ncclRecv),
    all enqueued on the context's stream."""
    L, h = rank_state.state._L, rank_state.state._h
    plan = rank_state.plan
    sch = plan.schedule
    G, p = plan.world, plan.rank
    for step in range(sch.steps):
        rank_state.sweep(step)
        if _sync_due(step, sch.steps, sync_every):
            rank_state.state._check(L.cmtf_gpu_sync(h, plan.shared_modes, plan.mat_mask, 1))
        if G > 1:
            for mode in sch.rotations_after(step):
                slo, shi = rank_state.block_rows(mode, sch.block(p, mode, step))
                # the block arriving from rank p+1 is the one it holds now,
                # which is the one this rank needs next
                rb = sch.block((p + 1) % G, mode, step)
                rlo, rhi = rank_state.block_rows(mode, rb)
                rank_state.state._check(L.cmtf_gpu_exchange_rows(
                    h, mode, slo, shi, (p - 1) % G, rlo, rhi, (p + 1) % G))
    rank_state.state._check(L.cmtf_gpu_end_epoch(h))


def consolidate_nccl(rank_state: RankState):
    """Broadcast every block of the stratified modes from its owner."""
    L, h = rank_state.state._L, rank_state.state._h
    plan = rank_state.plan
    G = plan.world
    for mode in range(plan.schedule.n_strat):
        lo = np.array([plan.cuts[mode][b] for b in range(G)], dtype=np.uint32)
        hi = np.array([plan.cuts[mode][b + 1] for b in range(G)], dtype=np.uint32)
        rank_state.state._check(L.cmtf_gpu_broadcast_rows(h, mode, G, _ptr(lo, C.c_uint32),
                                                          _ptr(hi, C.c_uint32)))
