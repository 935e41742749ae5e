"""DSGD host logic on CPU: partition invariants, and the
2-rank schedule + delta all-reduce run with gloo, the C oracle standing in
for the device sweep of each stratum."""
import os
import socket

import numpy as np
import pytest

from paper_1708_08640_b200 import dsgd, synth


def small_problem(n=6000, dims=(60, 50, 12)):
    spec = synth.config1(literal=False)
    spec.nnz, spec.dims = n, list(dims)
    spec.matrices = [synth.MatrixSpec(0, 30, 600), synth.MatrixSpec(1, 20, 500),
                     synth.MatrixSpec(2, 8, 60)]
    return synth.generate(spec)


@pytest.mark.parametrize("G", [1, 2, 3, 4])
@pytest.mark.parametrize("n_strat", [2, 3])
def test_partition_covers_every_entry_once_and_strata_are_disjoint(G, n_strat):
    b, _, _ = small_problem()
    part = dsgd.partition(b, G, n_strat=n_strat)
    sch = part.plans[0].schedule
    assert sch.steps == G ** (n_strat - 1)
    t = b.tensor
    # every tensor entry exactly once over all ranks
    keys = np.concatenate([p.bundle.tensor.indices.astype(np.int64) @ np.array([1 << 40, 1 << 20, 1])
                           for p in part.plans])
    full = t.indices.astype(np.int64) @ np.array([1 << 40, 1 << 20, 1])
    assert np.array_equal(np.sort(keys), np.sort(full))
    # in every step the strata touch disjoint rows of every stratified mode,
    # and those rows are in the block the rank holds at that step
    for s in range(sch.steps):
        for n in range(n_strat):
            seen = set()
            for p in part.plans:
                lo, hi = p.t_ranges[s]
                rows = set(p.bundle.tensor.indices[lo:hi, n].tolist())
                assert not (rows & seen)
                seen |= rows
                assert all(part.blocks[n][i] == sch.block(p.rank, n, s) for i in rows)
    # every matrix entry exactly once; entries of a matrix on a stratified
    # mode follow that block's holder
    for mi, m in enumerate(b.matrices):
        tot = sum(p.bundle.matrices[mi].nnz for p in part.plans)
        assert tot == m.nnz
        if m.coupled_mode < n_strat:
            for p in part.plans:
                for s in range(sch.steps):
                    lo, hi = p.m_ranges[s][mi]
                    rws = p.bundle.matrices[mi].indices[lo:hi, 0]
                    assert all(part.blocks[m.coupled_mode][r] ==
                               sch.block(p.rank, m.coupled_mode, s) for r in rws)


@pytest.mark.parametrize("G", [2, 3, 4])
@pytest.mark.parametrize("n_strat", [2, 3])
def test_rotation_schedule_brings_every_block_home(G, n_strat):
    """Simulated ring: after each step every rank sends its current block to
    p-1; the block it receives from p+1 is the one the schedule gives it next,
    and after a full epoch every rank holds its own block again."""
    sch = dsgd.Schedule(G, n_strat)
    for mode in range(1, n_strat):
        held = [sch.block(p, mode, 0) for p in range(G)]
        for s in range(sch.steps):
            assert held == [sch.block(p, mode, s) for p in range(G)]
            if mode in sch.rotations_after(s):
                held = [held[(p + 1) % G] for p in range(G)]
        assert held == list(range(G))


def test_balanced_blocks_balance_counts():
    rng = np.random.default_rng(0)
    counts = (1000 * rng.pareto(1.2, 5000)).astype(np.int64) + 1
    for G in (2, 4, 8):
        b = dsgd.balanced_blocks(counts, G)
        assert b.min() == 0 and b.max() == G - 1
        assert np.all(np.diff(b) >= 0)  # contiguous ranges
        loads = np.bincount(b, weights=counts, minlength=G)
        assert loads.max() <= loads.sum() / G + counts.max()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, out, n_strat):
    """One DSGD rank on CPU (gloo): the oracle sweeps the rank's strata, the
    replicated parameters are delta all-reduced after every step, the
    stratified blocks rotate along the ring (send to p-1, receive from p+1)
    exactly as run_epoch_nccl schedules them, and consolidate broadcasts
    every block from its owner at the end."""
    import torch
    import torch.distributed as dist
    from oracle import oracle as O
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b, test, _ = small_problem()
    part = dsgd.partition(b, world, n_strat=n_strat)
    plan = part.plans[rank]
    sch = plan.schedule
    ranks = [5, 5, 5]
    model = O.initialize(b, ranks, seed=0)  # identical replicas (same seed)
    loc = O.OracleModel(plan.bundle, ranks)
    loc.copy_from(model)
    counts = np.concatenate(part.counts + part.col_counts)
    eta, lam = 0.01, 0.01
    shared = [loc.factors[n] for n in range(3) if (plan.shared_modes >> n) & 1]
    shared += [loc.couplings[m] for m in range(3) if (plan.mat_mask >> m) & 1] + [loc.core]
    base = {id(a): a.copy() for a in shared}

    def sync():
        for a in shared:
            d = torch.from_numpy(a - base[id(a)])
            dist.all_reduce(d)
            a[...] = base[id(a)] + d.numpy()
            base[id(a)] = a.copy()

    def rows(mode, blk):
        return part.cuts[mode][blk], part.cuts[mode][blk + 1]

    for ep in range(6):
        for s in range(sch.steps):
            lo, hi = plan.t_ranges[s]
            sched = np.arange(lo, hi, dtype=np.uint64)
            moff = plan.bundle.tensor.nnz
            for mi, m in enumerate(plan.bundle.matrices):
                mlo, mhi = plan.m_ranges[s][mi]
                sched = np.concatenate([sched, np.arange(moff + mlo, moff + mhi, dtype=np.uint64)])
                moff += m.nnz
            np.random.default_rng(ep * 100 + s).shuffle(sched)
            assert O.run_epoch_counts(plan.bundle, loc, sched, eta, lam, counts, b.tensor.nnz) == 0
            sync()
            for mode in sch.rotations_after(s):
                slo, shi = rows(mode, sch.block(rank, mode, s))
                rlo, rhi = rows(mode, sch.block((rank + 1) % world, mode, s))
                F = loc.factors[mode]
                send = torch.from_numpy(np.ascontiguousarray(F[slo:shi]))
                recv = torch.zeros((rhi - rlo, F.shape[1]), dtype=torch.float64)
                reqs = [dist.isend(send, (rank - 1) % world), dist.irecv(recv, (rank + 1) % world)]
                for r in reqs:
                    r.wait()
                F[rlo:rhi] = recv.numpy()
        eta = 0.01 / (1.0 + 0.1 * (ep + 1))
    # every block is home again: broadcast from the owners
    for mode in range(n_strat):
        for blk in range(world):
            lo, hi = rows(mode, blk)
            t = torch.from_numpy(np.ascontiguousarray(loc.factors[mode][lo:hi]))
            dist.broadcast(t, src=blk)
            loc.factors[mode][lo:hi] = t.numpy()
    if rank == 0:
        full = O.OracleModel(b, ranks).copy_from(loc)
        out.put((O.epoch_stats(b, full, lam)[0], O.tensor_rmse(test, full)))
    # every rank ends with the same model
    chk = torch.tensor([float(np.sum(loc.core)), float(np.sum(loc.factors[1])),
                        float(np.sum(loc.factors[0]))], dtype=torch.float64)
    g = [torch.zeros_like(chk) for _ in range(world)]
    dist.all_gather(g, chk)
    assert torch.allclose(g[0], g[-1])
    dist.destroy_process_group()


@pytest.mark.parametrize("n_strat", [2, 3])
def test_dsgd_two_ranks_gloo_matches_serial_sgd(n_strat):
    import torch.multiprocessing as mp
    from oracle import oracle as O
    b, test, _ = small_problem()
    tr = O.SerialTrainer(b, [5, 5, 5], seed=0, eta0=0.01, mu=0.1, lambda_reg=0.01)
    for _ in range(6):
        tr.run_epoch()
    ref_train, _ = O.epoch_stats(b, tr.model, 0.01)
    ref_test = O.tensor_rmse(test, tr.model)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, q, n_strat)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(600)
        assert p.exitcode == 0
    train, testr = q.get(timeout=10)
    # DSGD (strata + summed deltas) vs sequential SGD after 6 epochs
    # raw summed deltas of the shared parameters (no damping on this CPU path)
    assert abs(train - ref_train) <= 0.05 * ref_train, (train, ref_train)
    assert abs(testr - ref_test) <= 0.05 * ref_test, (testr, ref_test)
