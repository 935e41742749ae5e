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
def test_partition_covers_every_entry_once_and_strata_are_disjoint(G):
    b, _, _ = small_problem()
    part = dsgd.partition(b, G)
    t = b.tensor
    # every tensor entry exactly once over all ranks
    keys = np.concatenate([p.bundle.tensor.indices.astype(np.int64) @ np.array([1 << 40, 1 << 20, 1])
                           for p in part.plans])
    full = t.indices.astype(np.int64) @ np.array([1 << 40, 1 << 20, 1])
    assert np.array_equal(np.sort(keys), np.sort(full))
    # in every sub-epoch the G strata touch disjoint mode-1 and mode-2 rows
    for s in range(G):
        seen1, seen2 = set(), set()
        for p in part.plans:
            lo, hi = p.t_ranges[s]
            i1 = set(p.bundle.tensor.indices[lo:hi, 0].tolist())
            i2 = set(p.bundle.tensor.indices[lo:hi, 1].tolist())
            assert not (i1 & seen1) and not (i2 & seen2)
            seen1 |= i1
            seen2 |= i2
            # and the rows are the rank's own mode-1 block / the rotating mode-2 block
            assert all(part.block1[i] == p.rank for i in i1)
            assert all(part.block2[i] == (p.rank + s) % G for i in i2)
    # every matrix entry exactly once; mode-2 matrix entries follow the U2 block holder
    for mi, m in enumerate(b.matrices):
        tot = sum(p.bundle.matrices[mi].nnz for p in part.plans)
        assert tot == m.nnz
        if m.coupled_mode == 1:
            for p in part.plans:
                for s in range(G):
                    lo, hi = p.m_ranges[s][mi]
                    rows = p.bundle.matrices[mi].indices[lo:hi, 0]
                    assert all(part.block2[r] == (p.rank + s) % G for r in rows)
        if m.coupled_mode == 0:
            for p in part.plans:
                rows = p.bundle.matrices[mi].indices[:, 0]
                assert all(part.block1[r] == p.rank for r in rows)


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


def _rank_main(rank, world, port, out):
    import torch
    import torch.distributed as dist
    from oracle import oracle as O
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b, test, _ = small_problem()
    part = dsgd.partition(b, world)
    plan = part.plans[rank]
    ranks = [5, 5, 5]
    model = O.initialize(b, ranks, seed=0)  # identical replicas (same seed)
    loc = O.OracleModel(plan.bundle, ranks)
    loc.copy_from(model)
    counts = np.concatenate(part.counts + part.col_counts)
    eta, lam = 0.01, 0.01

    def arrays(mask_modes, mask_mats, core):
        out_ = [loc.factors[n] for n in range(3) if (mask_modes >> n) & 1]
        out_ += [loc.couplings[m] for m in range(3) if (mask_mats >> m) & 1]
        if core:
            out_.append(loc.core)
        return out_

    def sync(mask_modes, mask_mats, core, base):
        for a, key in zip(arrays(mask_modes, mask_mats, core), range(100)):
            d = torch.from_numpy(a - base[id(a)])
            dist.all_reduce(d)
            a[...] = base[id(a)] + d.numpy()
            base[id(a)] = a.copy()

    allarr = loc.factors + loc.couplings + [loc.core]
    base = {id(a): a.copy() for a in allarr}
    for ep in range(6):
        for s in range(world):
            lo, hi = plan.t_ranges[s]
            sched = np.arange(lo, hi, dtype=np.uint64)
            moff = plan.bundle.tensor.nnz
            for mi, m in enumerate(plan.bundle.matrices):
                mlo, mhi = plan.m_ranges[s][mi]
                sched = np.concatenate([sched, np.arange(moff + mlo, moff + mhi, dtype=np.uint64)])
                moff += m.nnz
            np.random.default_rng(ep * 100 + s).shuffle(sched)
            assert O.run_epoch_counts(plan.bundle, loc, sched, eta, lam, counts, b.tensor.nnz) == 0
            sync(plan.sync_modes, plan.mat_mask, 1, base)
        sync(plan.end_modes, 0, 0, base)
        eta = 0.01 / (1.0 + 0.1 * (ep + 1))
    if rank == 0:
        full = O.OracleModel(b, ranks).copy_from(loc)
        out.put((O.epoch_stats(b, full, lam)[0], O.tensor_rmse(test, full)))
    # every rank ends with the same model
    chk = torch.tensor([float(np.sum(loc.core)), float(np.sum(loc.factors[1]))], dtype=torch.float64)
    g = [torch.zeros_like(chk) for _ in range(world)]
    dist.all_gather(g, chk)
    assert torch.allclose(g[0], g[-1])
    dist.destroy_process_group()


def test_dsgd_two_ranks_gloo_matches_serial_sgd():
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
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, q)) for r in range(2)]
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
