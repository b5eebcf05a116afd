"""The fused compute + gather path (paper_2503_16080_b200/shard.py: share_gather_buffers,
run_fused_gather) on one B200: two processes, both on cuda:0, gloo for the handle exchange and
the barrier.  Rank 1's GEMM epilogues store its units' residues straight into rank 0's output
buffer through a CUDA IPC mapping opened on rank 1's current device (ctpt_ipc_open, peer access
enabled as needed) — the same code path that, on a multi-GPU node, writes over NVLink into rank
0's HBM.  No kernel waits on another process (only a host barrier after both
finished), so sharing one GPU is safe.  The gathered result must equal the oracle everywhere."""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cfg, out_path):
    import torch
    import torch.distributed as dist

    sys.path.insert(0, ROOT)
    import ctgen
    from paper_2503_16080_b200.shard import gpu_compute_into_fn, plan_units, run_fused_gather, share_gather_buffers

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    fmt, N, k, d2, d3, L = cfg
    d1 = N * k
    ps = ctgen.primes(L)
    U = ctgen.U_matrix(5, d2, d3, 8)
    ra = d1 if fmt == ctgen.SHARED_S else N
    plan = plan_units(L, d3, world)
    out_AU = torch.full((L, d3, ra), -1, dtype=torch.int32, device="cuda") if rank == 0 else None
    out_BU = torch.full((L, d3, d1), -1, dtype=torch.int32, device="cuda") if rank == 0 else None
    peers = share_gather_buffers(out_AU, out_BU, rank, L, d3, ra, d1)

    def cts(l):
        ct = ctgen.encrypt(fmt, N, d1, d2, 5, 20, [ps[l]])
        return ct.a_polys[0], ct.b_polys[0]

    compute_into = gpu_compute_into_fn(fmt, N, d1, d2, d3, ps, cts, U, "cuda")
    run_fused_gather(plan, rank, compute_into, peers)
    if rank == 0:
        np.savez(out_path, AU=out_AU.cpu().numpy().view(np.uint32), BU=out_BU.cpu().numpy().view(np.uint32))
    peers.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("cfg", [(2, 64, 2, 300, 600, 3),   # L = 3 over 2 ranks: column-split units
                                 (1, 32, 4, 130, 40, 2),    # whole primes, d3 <= 32 + fused kernels
                                 (0, 128, 1, 520, 300, 1)],  # one prime split by columns
                         ids=["column_split", "prime_split_skinny", "one_prime"])
def test_fused_gather_two_processes_one_gpu(cfg, tmp_path):
    import torch.multiprocessing as mp

    import ctgen
    import oracle

    out = str(tmp_path / "gathered.npz")
    mp.spawn(_worker, args=(2, _free_port(), cfg, out), nprocs=2, join=True)
    got = np.load(out)
    fmt, N, k, d2, d3, L = cfg
    d1 = N * k
    ps = ctgen.primes(L)
    U = ctgen.U_matrix(5, d2, d3, 8)
    for l, p in enumerate(ps):
        ct = ctgen.encrypt(fmt, N, d1, d2, 5, 20, [p])
        A, B = oracle.format_matrices(fmt, N, d1, ct.a_polys[0], ct.b_polys[0])
        assert np.array_equal(got["AU"][l], oracle.modmatmul(np.ascontiguousarray(A.T), U, p)), f"A·U prime {l}"
        assert np.array_equal(got["BU"][l], oracle.modmatmul(np.ascontiguousarray(B.T), U, p)), f"B·U prime {l}"
