"""Multi-GPU sharding logic on CPU (gloo, world_size 2): the unit planner and the final gather
to rank 0 (paper_2503_16080_b200/shard.py).  Each rank computes its units with the oracle, so
the test checks exactly the host-side plumbing a multi-GPU run uses (plan, per-unit outputs,
point-to-point gather, placement in the [L][d3][rows] layout)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2503_16080_b200.shard import (Unit, choose_gather, gathered_bytes, plan_units, primes_needed,  # noqa: E402
                                         run_and_gather)


@pytest.mark.parametrize("L,d3,world", [(8, 32768, 8), (8, 32768, 2), (3, 16384, 8), (2, 4096, 8), (4, 4096, 8),
                                        (1, 7, 3), (5, 3, 4), (3, 10, 2), (4, 10, 2), (1, 1, 1)])
def test_plan_covers_each_pair_once_and_balances(L, d3, world):
    plan = plan_units(L, d3, world)
    assert len(plan) == world
    seen = np.zeros((L, d3), dtype=np.int64)
    cols = []
    for units in plan:
        n = 0
        for u in units:
            assert 0 <= u.l < L and 0 <= u.c0 < u.c1 <= d3
            seen[u.l, u.c0:u.c1] += 1
            n += u.ncols
        cols.append(n)
        assert len(primes_needed(units)) <= -(-L // world) + 1
    assert (seen == 1).all()
    assert max(cols) - min(cols) <= 1  # equal residue-MACs up to one column
    if L % world == 0:
        assert all(u.c0 == 0 and u.c1 == d3 for units in plan for u in units)  # whole primes


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cfg, out_path, use_into=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import ctgen
    import oracle

    fmt, N, k, d2, d3, L = cfg
    d1 = N * k
    ra = oracle.rows_A(fmt, N, d1)
    ps = ctgen.primes(L)
    plan = plan_units(L, d3, world)
    U = ctgen.U_matrix(2, d2, d3, 8)
    cts = {l: ctgen.encrypt(fmt, N, d1, d2, 2, 20, [ps[l]]) for l in primes_needed(plan[rank])}

    def compute(u: Unit):
        ct = cts[u.l]
        A, B = oracle.format_matrices(fmt, N, d1, ct.a_polys[0], ct.b_polys[0])
        cols = np.arange(u.c0, u.c1)
        au = oracle.modmatmul(np.ascontiguousarray(A.T), U, ps[u.l], cols=cols)
        bu = oracle.modmatmul(np.ascontiguousarray(B.T), U, ps[u.l], cols=cols)
        return torch.from_numpy(au.view(np.int32)), torch.from_numpy(bu.view(np.int32))

    def compute_into(u: Unit, au_dst, bu_dst):
        au, bu = compute(u)
        au_dst.copy_(au)
        bu_dst.copy_(bu)

    out_AU = torch.full((L, d3, ra), -1, dtype=torch.int32) if rank == 0 else None
    out_BU = torch.full((L, d3, d1), -1, dtype=torch.int32) if rank == 0 else None
    log = []
    run_and_gather(plan, rank, compute, out_AU, out_BU, gather=True, compute_into=compute_into if use_into else None,
                   log=log)
    if rank == 0:
        np.savez(out_path, AU=out_AU.numpy().view(np.uint32), BU=out_BU.numpy().view(np.uint32),
                 log=np.array([e[0] for e in log]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("use_into", [False, True], ids=["copy", "into"])
@pytest.mark.parametrize("cfg", [(2, 16, 2, 24, 10, 3),   # L=3 over 2 ranks: column-split units
                                 (1, 8, 2, 20, 9, 4)],    # L=4 over 2 ranks: whole primes
                         ids=["column_split", "prime_split"])
def test_gloo_world2_gather_matches_single_process(cfg, use_into, tmp_path):
    import ctgen
    import oracle

    out = str(tmp_path / "gathered.npz")
    mp.spawn(_worker, args=(2, _free_port(), cfg, out, use_into), nprocs=2, join=True)
    got = np.load(out)
    # rank 0 posted every remote receive before computing any of its own units (the transfers of
    # the senders' units overlap rank 0's compute instead of queueing behind it)
    log = list(got["log"])
    assert "compute" in log and "post_recv" in log
    assert log.index("compute") > max(i for i, e in enumerate(log) if e == "post_recv")
    fmt, N, k, d2, d3, L = cfg
    d1 = N * k
    ps = ctgen.primes(L)
    U = ctgen.U_matrix(2, d2, d3, 8)
    for l, p in enumerate(ps):
        ct = ctgen.encrypt(fmt, N, d1, d2, 2, 20, [p])
        A, B = oracle.format_matrices(fmt, N, d1, ct.a_polys[0], ct.b_polys[0])
        assert np.array_equal(got["AU"][l], oracle.modmatmul(np.ascontiguousarray(A.T), U, p))
        assert np.array_equal(got["BU"][l], oracle.modmatmul(np.ascontiguousarray(B.T), U, p))


def _choose_worker(rank, world, port, flags, out_path, want):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mode = choose_gather(want, world, flags[rank])
    with open(f"{out_path}.{rank}", "w") as f:
        f.write(mode)
    dist.destroy_process_group()


@pytest.mark.parametrize("flags,want,expect", [((True, True), "auto", "ipc"),    # every rank reaches rank 0's GPU
                                               ((True, False), "auto", "nccl"),  # one rank cannot: NCCL for all
                                               ((True, True), "nccl", "nccl"),
                                               ((False, False), "ipc", "ipc")])
def test_gloo_world2_gather_choice(flags, want, expect, tmp_path):
    """choose_gather: the fused IPC gather only when EVERY rank's device can access rank 0's (peer
    access), otherwise the NCCL gather; all ranks agree."""
    out = str(tmp_path / "mode")
    mp.spawn(_choose_worker, args=(2, _free_port(), flags, out, want), nprocs=2, join=True)
    modes = {open(f"{out}.{r}").read() for r in range(2)}
    assert modes == {expect}


def test_gather_choice_single_rank_and_bytes():
    assert choose_gather("auto", 1, False) == "none"
    plan = plan_units(3, 16384, 8)
    # c3 over 8 ranks: 7/8 of the outputs cross into rank 0 (4·d3·(rows_A + d1) bytes per prime)
    assert gathered_bytes(plan, 4096, 16384) == sum(4 * u.ncols * 20480 for us in plan[1:] for u in us)
    assert gathered_bytes(plan, 4096, 16384) == 4 * 20480 * (3 * 16384 - sum(u.ncols for u in plan[0]))
