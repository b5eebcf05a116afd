"""Multi-GPU sharding of CP-MM — planner, per-rank execution, final gather.

The path partitions naturally: the residue products of different RNS primes are independent
(one Mod-PP-MM per prime, the structure of Strategy 3), and so are different
column blocks of U (output column j is output ciphertext j).  A *unit* is
(prime index l, U columns [c0, c1)).  There is no exchange inside the computation; the only
communication is the final gather of every unit's (A·U, B·U) block to rank 0.

Layout of the gathered result on rank 0 (the single-GPU layout of ctpt_matmul):
    AU [L][d3][rows_A], BU [L][d3][d1]; a unit is the contiguous block AU[l, c0:c1].

Two gathers:
  * "ipc" (the fused compute + gather): rank 0's buffers are mapped into every rank's CURRENT
    device by CUDA IPC (ctpt_ipc_open, peer access enabled as needed), and each rank's
    ctpt_matmul gets the unit's block in rank 0's buffer as its output pointer — the GEMM
    epilogues' stores ARE the transfer over NVLink / NVSwitch, tile by tile, overlapped with the
    MMAs of the next tiles; no staging, no collective, one barrier at the end.
  * "nccl" (fallback when a rank's GPU has no peer access to rank 0's): rank 0 posts every
    remote receive (irecv straight into the gathered layout) BEFORE computing its own units, so
    each sender's transfer of unit i overlaps its compute of unit i+1 and rank 0's own compute;
    the compute kernels leave SMs to the NCCL kernels (ctpt_problem.max_ctas).
choose_gather picks "ipc" when every rank's device can access rank 0's, else "nccl".
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


def gathered_bytes(units_per_rank: list[list[Unit]], rows_A: int, d1: int) -> int:
    """Output bytes that cross into rank 0 per gather (every unit not computed on rank 0)."""
    return sum(4 * u.ncols * (rows_A + d1) for units in units_per_rank[1:] for u in units)


# ----------------------------------------------------------------------------------------------
# Choice of gather
# ----------------------------------------------------------------------------------------------
def choose_gather(want: str, world: int, can_reach_rank0: bool, group=None) -> str:
    """'none' for one rank; want = 'ipc' / 'nccl' as asked; 'auto' = 'ipc' if EVERY rank's device
    can access rank 0's device (can_reach_rank0, e.g. ctpt.peer_access(dev, dev_of_rank0)), else
    'nccl'.  Collective over the process group (every rank must call it)."""
    if world == 1:
        return "none"
    if want in ("ipc", "nccl"):
        return want
    if want != "auto":
        raise ValueError(f"unknown gather {want!r}")
    import torch.distributed as dist

    flags = [None] * world
    dist.all_gather_object(flags, bool(can_reach_rank0), group=group)
    return "ipc" if all(flags) else "nccl"


# ----------------------------------------------------------------------------------------------
# NCCL (or gloo) point-to-point gather
# ----------------------------------------------------------------------------------------------
def run_and_gather(units_per_rank: list[list[Unit]], rank: int, compute: Callable[[Unit], tuple],
                   out_AU=None, out_BU=None, gather: bool = True, group=None,
                   compute_into: Callable | None = None, log: list | None = None):
    """Compute this rank's units and gather them into rank 0's out_AU [L][d3][rows_A] /
    out_BU [L][d3][d1].

    Rank 0 first POSTS every remote receive (irecv into the unit's block of the gathered layout),
    then computes its own units — with `compute_into(unit, AU_blk, BU_blk)` straight into the
    gathered layout if given, else `compute(unit)` + a copy — and finally waits for the receives.
    Every other rank computes its units in order with `compute(unit) -> (AU_blk [ncols][rows_A],
    BU_blk [ncols][d1])` and sends each one (isend) as soon as it is computed, so the transfer of
    unit i overlaps the compute of unit i+1.  `log` (tests) records the order of posts and
    computes.  Returns the list of (unit, AU_blk, BU_blk) computed locally (blocks of the gathered
    layout on rank 0)."""
    import torch.distributed as dist

    mine = []
    reqs = []
    if gather and rank == 0:
        for src in range(1, len(units_per_rank)):
            for u in units_per_rank[src]:
                reqs.append(dist.irecv(out_AU[u.l, u.c0:u.c1], src=src, group=group))
                reqs.append(dist.irecv(out_BU[u.l, u.c0:u.c1], src=src, group=group))
                if log is not None:
                    log.append(("post_recv", src, u))
    for u in units_per_rank[rank]:
        if log is not None:
            log.append(("compute", rank, u))
        if gather and rank == 0 and compute_into is not None:
            au, bu = out_AU[u.l, u.c0:u.c1], out_BU[u.l, u.c0:u.c1]
            compute_into(u, au, bu)
        else:
            au, bu = compute(u)
            if gather and rank == 0:
                out_AU[u.l, u.c0:u.c1].copy_(au)
                out_BU[u.l, u.c0:u.c1].copy_(bu)
        mine.append((u, au, bu))
        if gather and rank != 0:
            reqs.append(dist.isend(au.contiguous(), dst=0, group=group))
            reqs.append(dist.isend(bu.contiguous(), dst=0, group=group))
    for r in reqs:
        r.wait()
    return mine


def gpu_compute_fn(fmt: int, N: int, d1: int, d2: int, d3: int, primes: list, get_ciphertexts: Callable,
                   U, device, max_ctas: int = 0):
    """compute(unit) for one GPU: ctpt_layout + ctpt_plain_precompute + ctpt_matmul on a one-prime,
    one-column-block Spec.  get_ciphertexts(l) -> (a_polys_l, b_polys_l) of prime l (host numpy or
    device tensors); prime l's layout is cached across its units."""
    import torch

    from . import ctpt

    into = gpu_compute_into_fn(fmt, N, d1, d2, d3, primes, get_ciphertexts, U, device, max_ctas)

    def compute(u: Unit):
        ra = d1 if fmt == ctpt.SHARED_S else (0 if fmt == ctpt.STRUCT_A else N)
        AU = torch.empty((u.ncols, max(ra, 0)), dtype=torch.int32, device=device)
        BU = torch.empty((u.ncols, d1), dtype=torch.int32, device=device)
        into(u, AU, BU)
        return AU, BU

    return compute


def gpu_compute_into_fn(fmt: int, N: int, d1: int, d2: int, d3: int, primes: list, get_ciphertexts: Callable, U,
                        device, max_ctas: int = 0):
    """compute_into(unit, AU_dst, BU_dst) for one GPU: ctpt_layout + precompute once per prime,
    then ctpt_matmul on the unit's column block writing into the destination blocks (torch tensors
    or raw device addresses — e.g. rank 0's buffers mapped by PeerGather)."""
    import torch

    from . import ctpt
    from .engine import CpmmEngine

    cache = {}

    def compute_into(u: Unit, AU_dst, BU_dst):
        if u.l not in cache:
            cache.clear()
            eng = CpmmEngine(ctpt.Spec(fmt, N, d1, d2, d3, [primes[u.l]], max_ctas=max_ctas), device)
            a, b = get_ciphertexts(u.l)
            eng.layout(a, b)
            eng.precompute(U)
            cache[u.l] = eng
        base = cache[u.l]
        spec = dataclasses.replace(base.spec, col_begin=u.c0, col_end=u.c1)
        sizes = ctpt.query_sizes(spec)
        if base.ws.numel() < sizes.workspace_bytes:  # a narrow unit (<= 32 columns) takes the raw-byte kernel
            base.ws = torch.empty(sizes.workspace_bytes, dtype=torch.uint8, device=device)
        ctpt.matmul(spec, base.ctmat, base.plain, AU_dst, BU_dst, base.ws)

    return compute_into


# ----------------------------------------------------------------------------------------------
# Fused compute + gather over peer memory (NVLink / NVSwitch on one node)
# ----------------------------------------------------------------------------------------------
class PeerGather:
    """Rank 0's gathered output buffers as device addresses usable by THIS rank's current device:
    rank 0's own tensors on rank 0, CUDA IPC mappings opened on this rank's device elsewhere
    (ctpt_ipc_open: peer access to rank 0's GPU is enabled as needed, so this device's kernels
    store over NVLink).  block(u) gives the unit's contiguous (AU, BU) block addresses."""

    def __init__(self, au_addr: int, bu_addr: int, L: int, d3: int, rows_A: int, d1: int, bases=()):
        self.au, self.bu = au_addr, bu_addr
        self.L, self.d3, self.rows_A, self.d1 = L, d3, rows_A, d1
        self._bases = list(bases)

    def block(self, u: Unit) -> tuple[int, int]:
        au = self.au + 4 * (u.l * self.d3 + u.c0) * self.rows_A if self.rows_A else 0
        bu = self.bu + 4 * (u.l * self.d3 + u.c0) * self.d1
        return au, bu

    def close(self):
        from . import ctpt

        for b in self._bases:
            ctpt.ipc_close(b)
        self._bases = []


def share_gather_buffers(out_AU, out_BU, rank: int, L: int, d3: int, rows_A: int, d1: int,
                         group=None) -> PeerGather:
    """Rank 0 passes its gathered output tensors (AU may be None when rows_A = 0), the others None;
    the IPC handles travel over the process group and every other rank opens them on its current
    device (torch.cuda.set_device first)."""
    import torch.distributed as dist

    from . import ctpt

    obj = [None]
    if rank == 0:
        obj[0] = (ctpt.ipc_export(out_AU) if out_AU is not None and rows_A else None, ctpt.ipc_export(out_BU))
    dist.broadcast_object_list(obj, src=0, group=group)
    if rank == 0:
        return PeerGather(out_AU.data_ptr() if out_AU is not None and rows_A else 0, out_BU.data_ptr(), L, d3,
                          rows_A, d1)
    (ha, hb) = obj[0]
    bases = []
    au = 0
    if ha is not None:
        base, au = ctpt.ipc_open(*ha)
        bases.append(base)
    base, bu = ctpt.ipc_open(*hb)
    bases.append(base)
    return PeerGather(au, bu, L, d3, rows_A, d1, bases)


def run_fused_gather(units_per_rank: list[list[Unit]], rank: int, compute_into: Callable, peers: PeerGather,
                     group=None):
    """Every rank computes its units with `compute_into(unit, AU_addr, BU_addr)` whose kernels'
    epilogues store the reduced residues DIRECTLY into rank 0's gathered layout: the transfer over
    NVLink is the GEMM's own stores, tile by tile, with no staging copy and no collective.  Ends
    with a device sync and a barrier, after which rank 0 holds the result."""
    import torch
    import torch.distributed as dist

    for u in units_per_rank[rank]:
        compute_into(u, *peers.block(u))
    torch.cuda.synchronize()
    dist.barrier(group=group)
