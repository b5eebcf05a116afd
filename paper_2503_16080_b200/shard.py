"""Multi-GPU sharding of CP-MM — planner, per-rank execution, final gather.

The path partitions naturally: the residue products of different RNS primes are independent
(one Mod-PP-MM per prime, the structure of Strategy 3), and so are different
column blocks of U (output column j is output ciphertext j).  A *unit* is
(prime index l, U columns [c0, c1)).  There is no exchange inside the computation; the only
communication is the optional final gather of every unit's (A·U, B·U) block to rank 0, issued
as point-to-point sends right after each unit is computed so the transfer of unit i overlaps
the compute of unit i+1 (NCCL runs its sends on its own stream).

Layout of the gathered result on rank 0 (the single-GPU layout of ctpt_matmul):
    AU [L][d3][rows_A], BU [L][d3][d1]; a unit is the contiguous block AU[l, c0:c1].
"""
from __future__ import annotations

import dataclasses

from dataclasses import dataclass
from typing import Callable


@dataclass(frozen=True)
class Unit:
    l: int   # prime index
    c0: int  # first U column
    c1: int  # one past the last U column

    @property
    def ncols(self) -> int:
        return self.c1 - self.c0


def plan_units(L: int, d3: int, world: int) -> list[list[Unit]]:
    """Per-rank unit lists covering every (prime, column) pair exactly once, with equal
    residue-MAC counts up to one column.
    * world | L: rank r takes primes [r·L/world, (r+1)·L/world), all columns (no U split);
    * otherwise: the (prime, column) pairs in prime-major order are cut into `world` contiguous
      slices; a rank touches at most ⌈L/world⌉ + 1 primes."""
    if world < 1 or L < 1 or d3 < 1:
        raise ValueError("world, L, d3 must be >= 1")
    if L % world == 0:
        per = L // world
        return [[Unit(l, 0, d3) for l in range(r * per, (r + 1) * per)] for r in range(world)]
    total = L * d3
    out = []
    for r in range(world):
        a, b = total * r // world, total * (r + 1) // world
        units = []
        while a < b:
            l, c = divmod(a, d3)
            c1 = min(d3, c + (b - a))
            units.append(Unit(l, c, c1))
            a += c1 - c
        out.append(units)
    return out


def primes_needed(units: list[Unit]) -> list[int]:
    return sorted({u.l for u in units})


def run_and_gather(units_per_rank: list[list[Unit]], rank: int, compute: Callable[[Unit], tuple],
                   out_AU=None, out_BU=None, gather: bool = True, group=None):
    """Compute this rank's units with `compute(unit) -> (AU_blk [ncols][rows_A], BU_blk [ncols][d1])`
    (torch tensors on the communication device) and, if `gather`, send them to rank 0, which
    writes every rank's blocks into out_AU [L][d3][rows_A] / out_BU [L][d3][d1].
    Returns the list of (unit, AU_blk, BU_blk) computed locally."""
    import torch.distributed as dist

    mine = []
    reqs = []
    for u in units_per_rank[rank]:
        au, bu = compute(u)
        mine.append((u, au, bu))
        if gather and rank != 0:
            reqs.append(dist.isend(au.contiguous(), dst=0, group=group))
            reqs.append(dist.isend(bu.contiguous(), dst=0, group=group))
    if gather and rank == 0:
        for (u, au, bu) in mine:
            out_AU[u.l, u.c0:u.c1].copy_(au)
            out_BU[u.l, u.c0:u.c1].copy_(bu)
        for src in range(1, len(units_per_rank)):
            for u in units_per_rank[src]:
                dist.recv(out_AU[u.l, u.c0:u.c1], src=src, group=group)
                dist.recv(out_BU[u.l, u.c0:u.c1], src=src, group=group)
    for r in reqs:
        r.wait()
    return mine


def gpu_compute_fn(fmt: int, N: int, d1: int, d2: int, d3: int, primes: list, get_ciphertexts: Callable,
                   U, device):
    """compute(unit) for one GPU: ctpt_layout + ctpt_plain_precompute + ctpt_matmul on a one-prime,
    one-column-block Spec.  get_ciphertexts(l) -> (a_polys_l, b_polys_l) of prime l (host numpy or
    device tensors); prime l's layout is cached across its units."""
    import torch

    from . import ctpt
    from .engine import CpmmEngine

    cache = {}

    def compute(u: Unit):
        key = u.l
        if key not in cache:
            cache.clear()
            eng = CpmmEngine(ctpt.Spec(fmt, N, d1, d2, d3, [primes[u.l]]), device)
            a, b = get_ciphertexts(u.l)
            eng.layout(a, b)
            eng.precompute(U)
            cache[key] = eng
        base = cache[key]
        # the unit's column block of the base problem (keeps the plane mode: kU, u_unsigned, u_offset)
        spec = dataclasses.replace(base.spec, col_begin=u.c0, col_end=u.c1)
        sizes = ctpt.query_sizes(spec)
        AU = torch.empty(sizes.out_AU_bytes // 4, dtype=torch.int32, device=device)
        BU = torch.empty(sizes.out_BU_bytes // 4, dtype=torch.int32, device=device)
        if base.ws.numel() < sizes.workspace_bytes:  # a narrow unit (<= 32 columns) takes the raw-byte kernel
            base.ws = torch.empty(sizes.workspace_bytes, dtype=torch.uint8, device=device)
        ctpt.matmul(spec, base.ctmat, base.plain, AU, BU, base.ws)
        return AU.view(u.ncols, sizes.rows_A), BU.view(u.ncols, d1)

    return compute


# ----------------------------------------------------------------------------------------------
# Fused compute + gather over peer memory (NVLink / NVSwitch on one node)
# ----------------------------------------------------------------------------------------------
def share_gather_buffers(out_AU, out_BU, rank: int, group=None):
    """Rank 0's output buffers mapped into every rank's address space (CUDA IPC through torch's
    tensor-sharing reductions; on one node with NVLink the mapping is peer memory).  Rank 0 passes
    its tensors, the others pass None; every rank gets (AU, BU) tensors aliasing rank 0's memory."""
    import torch.distributed as dist
    from torch.multiprocessing.reductions import reduce_tensor

    obj = [None]
    if rank == 0:
        obj[0] = (reduce_tensor(out_AU), reduce_tensor(out_BU))
    dist.broadcast_object_list(obj, src=0, group=group)
    if rank == 0:
        return out_AU, out_BU
    (fa, aa), (fb, ab) = obj[0]
    return fa(*aa), fb(*ab)


def run_fused_gather(units_per_rank: list[list[Unit]], rank: int, compute_into: Callable, peer_AU, peer_BU,
                     group=None):
    """Every rank computes its units with `compute_into(unit, AU_dst, BU_dst)`, whose kernels'
    epilogues store the reduced residues DIRECTLY into rank 0's gathered layout
    (peer_AU [L][d3][rows_A], peer_BU [L][d3][d1], mapped by share_gather_buffers): the transfer
    over NVLink is the GEMM's own stores, tile by tile, with no staging copy and no collective.
    A unit's block peer_AU[l, c0:c1] is contiguous, so it is a plain output pointer for
    ctpt_matmul.  Ends with a device sync and a barrier, after which rank 0 holds the result."""
    import torch
    import torch.distributed as dist

    for u in units_per_rank[rank]:
        compute_into(u, peer_AU[u.l, u.c0:u.c1], peer_BU[u.l, u.c0:u.c1])
    torch.cuda.synchronize()
    dist.barrier(group=group)


def gpu_compute_into_fn(fmt: int, N: int, d1: int, d2: int, d3: int, primes: list, get_ciphertexts: Callable, U,
                        device):
    """compute_into(unit, AU_dst, BU_dst) for one GPU: ctpt_layout + precompute once per prime,
    then ctpt_matmul on the unit's column block writing into the (possibly peer-mapped)
    destination blocks."""
    import torch

    from . import ctpt
    from .engine import CpmmEngine

    cache = {}

    def compute_into(u: Unit, AU_dst, BU_dst):
        if u.l not in cache:
            cache.clear()
            eng = CpmmEngine(ctpt.Spec(fmt, N, d1, d2, d3, [primes[u.l]]), device)
            a, b = get_ciphertexts(u.l)
            eng.layout(a, b)
            eng.precompute(U)
            cache[u.l] = eng
        base = cache[u.l]
        spec = dataclasses.replace(base.spec, col_begin=u.c0, col_end=u.c1)
        sizes = ctpt.query_sizes(spec)
        if base.ws.numel() < sizes.workspace_bytes:
            base.ws = torch.empty(sizes.workspace_bytes, dtype=torch.uint8, device=device)
        ctpt.matmul(spec, base.ctmat, base.plain, AU_dst, BU_dst, base.ws)

    return compute_into
