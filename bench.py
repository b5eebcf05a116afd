#!/usr/bin/env python
"""Benchmark of the CP-MM hot path (Algorithm 6 step 1) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl ours|reference]

One "step" = ctpt_matmul over one batch of synthetic input: every RNS prime of the
configuration, i.e. (A·U mod p, B·U mod p) for all L primes, with the limb split inside
the step (SURVEY.md §8(a) note 2).  Default workload: config c3 (shared-a, N = 4096,
k = 4, d1 = d2 = d3 = 16384, L = 3) — the configuration BASELINE.json's metric ("at
d = 16384") is quoted on.  Prints ONE JSON line on rank 0.

Multi-GPU (torchrun, one rank per GPU): every rank runs its own independent c3 problem
(seed = rank); there is no collective on the data path, so "scaling" is "weak" and
value = all ranks' residue-MACs ÷ the max-over-ranks device time.

--impl reference: the CPU oracle (oracle/, schoolbook modular matmul, 128-bit
accumulation) as it stands, on the host cores, on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
import types

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ct-pt matmul residue-MACs/s at d=16384 and % of B200 dense INT8 TC peak"
UNIT = "residue-MAC/s"
INT8_DATASHEET_MACS = 2.25e15  # dense INT8 4.5 POPS, in MAC/s
# configs whose device-resident single-problem step does not fit one GPU (c5: 68.7 GB of laid-out
# inputs + 68.7 GB of outputs + the raw ciphertexts during layout): even at N = 1 they run as
# per-prime units with the primes streamed sequentially (BASELINE.json configs[4])
STREAMED_CONFIGS = {"c5"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c3")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--overlap", action="store_true",
                    help="experiment: run prime l+1's limb split on a side stream during prime l's GEMM "
                         "(measured slower; default off)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--split-overlap", default="auto", choices=["auto", "on", "off"],
                    help="split + GEMM path: split prime l+1 inside prime l's GEMM kernel (ctpt_gemm_next); "
                         "measured +2.2 %% (c4) and +1.6 %% (c2, both d3 = 4096) but +0.3 %% (noise) on c3 "
                         "(d3 = 16384, the split is 3 %% of the step) at a 4 %% lower GEMM roofline fraction, "
                         "so auto = on for d3 <= 8192 (profiles/r01/split_in_gemm)")
    ap.add_argument("--graph", default="auto", choices=["auto", "on", "off"],
                    help="replay each step as one CUDA graph (auto: launch-bound workloads, < 1e9 residue MACs)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target seconds of oracle work per sample")
    ap.add_argument("--rescale", action="store_true",
                    help="Algorithm 6 with step 2 (SURVEY.md §8(f) row 3): U real uniform[-1,1) encoded at "
                         "Δ_U = the last prime (per-prime residues, kU = 4), RNS Rescale by that prime "
                         "fused into the other primes' epilogues")
    ap.add_argument("--raster-group", type=int, default=0,
                    help="k_gemm_tc raster group in j-tiles (ctpt_problem.raster_group; 0 = the library's choice)")
    ap.add_argument("--max-ctas", type=int, default=0,
                    help="cap on the persistent grids (ctpt_problem.max_ctas; 0 = one CTA per SM)")
    ap.add_argument("--mode", default="auto", choices=["auto", "strong", "weak"],
                    help="auto: ONE problem strong-scaled over the ranks (N > 1, or a config whose inputs and "
                         "outputs do not fit one device-resident problem, i.e. c5: the primes stream through "
                         "per-prime units); at N = 1 the device-resident single-problem step.  strong: always "
                         "the per-unit sharded path.  weak: every rank runs its own independent problem "
                         "(no data-path collective)")
    ap.add_argument("--gather", default="auto", choices=["auto", "ipc", "nccl"],
                    help="strong mode, N > 1: how the units' outputs reach rank 0 inside the timed region. "
                         "ipc = the GEMM epilogues store into rank 0's buffers through CUDA IPC peer mappings "
                         "(NVLink); nccl = point-to-point, rank 0 posts its receives before computing; auto = ipc "
                         "when every rank's GPU has peer access to rank 0's, else nccl")
    return ap.parse_args()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            mp = json.load(f)
        return mp, "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def config_for(c, world: int, mode: str) -> dict:
    """The `config` object of the JSON line — the same for our arm and the reference (oracle) arm:
    the workload, its L2 footprint and the parallelism."""
    l2 = c.L * c.R * ((c.d2 + 15) // 16 * 16) * 4
    par = {"strong": f"strong: ONE problem's (prime, U-column) units sharded over {world} GPU(s) "
                     f"(shard.plan_units), outputs gathered into rank 0 inside the timed region",
           "weak": f"weak: {world} independent problem(s), one per GPU, no data-path collective"}[mode]
    return dict(workload_desc(c), l2=f"inputs {l2 / 2**30:.2f} GiB per step > 126 MB L2 (no flush needed)",
                parallelism=par)


def workload_desc(c) -> dict:
    import ctgen

    return {"workload": f"{c.name}: {ctgen.FORMAT_NAMES[c.fmt]} N={c.N} k={c.k} d1={c.d1} d2={c.d2} d3={c.d3} "
                        f"L={c.L} Δ=2^{c.log_delta} U∈[-{c.u_bound},{c.u_bound}]",
            "format": ctgen.FORMAT_NAMES[c.fmt], "N": c.N, "d1": c.d1, "d2": c.d2, "d3": c.d3, "L": c.L,
            "rows_stacked_R": c.R, "seed": c.seed}


# ------------------------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, dev):
        """dev: the torch CUDA device whose clocks to sample — selected by UUID, since NVML's indices
        need not follow CUDA's device order (CUDA_VISIBLE_DEVICES, PCI ordering)."""
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        gid = gpu_uuid_of(dev) or str(getattr(dev, "index", dev) or 0)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                       "-lms", "100", "-i", gid], stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = []
        with open(self.f.name) as fh:
            raw = fh.read()
        for line in raw.splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        if os.environ.get("CTPT_CLOCK_LOG"):
            with open(os.environ["CTPT_CLOCK_LOG"], "w") as fh:
                fh.write(self.FIELDS + "\n" + raw)
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None

        sm = [num(r[1]) for r in rows if num(r[1]) is not None]
        smax = [num(r[2]) for r in rows if num(r[2]) is not None]
        pw = [num(r[3]) for r in rows if num(r[3]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "power_w_max": max(pw) if pw else None, "power_w_median": statistics.median(pw) if pw else None,
                "samples": len(rows), "reasons": reasons}


# ------------------------------------------------------------------------------------ CPU oracle
def cpu_oracle_rate(c, ct, U, target_s: float, gpu_out=None):
    """Residue-MAC/s of the oracle's schoolbook on a bounded sample of workload c: output
    columns of prime 0 over all R stacked rows and the full d2 contraction.  With gpu_out =
    (AU [d3][rows_A], BU [d3][d1]) of prime 0 from the timed run, the same oracle outputs also give
    a parity verdict on the sampled columns (every entry compared)."""
    import oracle

    cores = os.cpu_count() or 1
    p = ct.primes[0]
    ra = c.rows_A
    Ac = ct.a_polys[0].reshape(c.d2, ra) if ra else None  # structured-A: only B·U (Algorithm 7)
    Bc = ct.b_polys[0].reshape(c.d2, c.d1)
    ncols = max(1, min(cores, c.d3))
    t0 = time.perf_counter()
    if Ac is not None:
        oracle.modmatmul(Ac, U, p, cols=np.arange(ncols), nthreads=cores)
    oracle.modmatmul(Bc, U, p, cols=np.arange(ncols), nthreads=cores)
    dt = time.perf_counter() - t0
    # scale the sample to ~target_s of work
    ncols2 = int(min(c.d3, max(ncols, ncols * target_s / max(dt, 1e-3))))
    ncols2 = max(cores, (ncols2 // cores) * cores) if ncols2 >= cores else ncols2
    t0 = time.perf_counter()
    wa = oracle.modmatmul(Ac, U, p, cols=np.arange(ncols2), nthreads=cores) if Ac is not None else None
    wb = oracle.modmatmul(Bc, U, p, cols=np.arange(ncols2), nthreads=cores)
    dt = time.perf_counter() - t0
    macs = c.R * c.d2 * ncols2
    # single-thread rate (the paper's setting) on a slab: one output column of B·U
    t1 = time.perf_counter()
    oracle.modmatmul(Bc, U, p, cols=np.arange(1), nthreads=1)
    st_rate = c.d1 * c.d2 / (time.perf_counter() - t1)
    out = {"value": macs / dt, "unit": UNIT, "cores": cores, "kind": "oracle", "host": host_description(),
           "single_thread_value": st_rate,
           "sample": f"prime 0, {ncols2} of {c.d3} output columns x all {c.R} stacked rows x d2={c.d2} "
                     f"({macs:.3e} residue-MACs, {dt:.1f} s, schoolbook __int128, OpenMP {cores} threads)"}
    if gpu_out is not None:
        ga, gb = gpu_out
        bad = int(np.count_nonzero(gb[:ncols2] != wb))
        if wa is not None:
            bad += int(np.count_nonzero(ga[:ncols2] != wa))
        out["parity_on_sample"] = {"entries": int(ncols2 * c.R), "mismatches": bad,
                                   "verdict": "bit-exact" if bad == 0 else "MISMATCH"}
    return out


def host_description() -> str:
    """lscpu model, sockets × cores × threads per core."""
    try:
        txt = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
    except (OSError, subprocess.SubprocessError):
        return f"{os.cpu_count()} logical CPUs"
    kv = {}
    for line in txt.splitlines():
        if ":" in line:
            k, v = line.split(":", 1)
            kv[k.strip()] = v.strip()
    return (f"{kv.get('Model name', '?')}; {kv.get('Socket(s)', '?')} socket(s) x {kv.get('Core(s) per socket', '?')} "
            f"cores x {kv.get('Thread(s) per core', '?')} threads = {os.cpu_count()} logical CPUs")


def precision_on_sample(c, ps, AU, BU, U, cols, nthreads: int):
    """Decrypt and decode sampled output columns of the timed run (all primes) and compare with
    M·U in float64 — the paper's precision metric prec = log2‖M·U‖∞ − log2‖dec − M·U‖∞
     and the relative error the north star bounds by 1e-6 (reading Q15).  Oracle
    code only (decryption, exact CRT); AU / BU: device outputs [L][d3][rows_A], [L][d3][d1]."""
    import ctgen
    import oracle

    nk = c.k if c.fmt == ctgen.SHARED_A else 1
    sks = [ctgen.sk(c.seed, t, c.N) for t in range(nk)]
    ra = c.rows_A
    mu = np.zeros((c.d1, len(cols)), dtype=np.float64)
    Uc = U[:, cols].astype(np.float64)
    kb = 2048
    for k0 in range(0, c.d2, kb):
        n = min(kb, c.d2 - k0)
        mu += ctgen.msg_block(c.seed, c.d1, 0, c.d1, k0, n, nthreads=nthreads).dot(Uc[k0:k0 + n])
    worst_prec, worst_rel, worst_abs = float("inf"), 0.0, 0.0
    for ci, j in enumerate(cols):
        decs = []
        for l, p in enumerate(ps):
            a_col = AU[l, j].cpu().numpy().view(np.uint32) if ra else None
            b_col = BU[l, j].cpu().numpy().view(np.uint32)
            decs.append(oracle.decrypt_col(c.fmt, c.N, c.d1, sks, a_col, b_col, p, nthreads=nthreads))
        cen = oracle.crt_centred_array(np.stack(decs), ps)
        dec = np.array([float(v) for v in cen]) / 2.0 ** c.log_delta
        worst_prec = min(worst_prec, oracle.precision_bits(mu[:, ci], dec))
        worst_rel = max(worst_rel, float(np.abs(dec - mu[:, ci]).max() / np.abs(mu[:, ci]).max()))
        worst_abs = max(worst_abs, float(np.abs(dec - mu[:, ci]).max()))
    # reading Q16: |Dec/Δ − M·U| ≤ ‖U‖∞·d2·(B_e + ½)/Δ with B_e = 20; reading Q15: the 1e-6
    # relative bound applies to c2–c5 (c1's Δ = 2^20 cannot meet it)
    q16 = c.u_bound * c.d2 * 20.5 / 2.0 ** c.log_delta
    rel_ok = worst_rel <= 1e-6 or c.name == "c1"
    return {"columns": [int(j) for j in cols], "precision_bits": worst_prec, "rel_err_inf": worst_rel,
            "abs_err_inf": worst_abs, "q16_abs_bound": q16, "rel_bound": None if c.name == "c1" else 1e-6,
            "verdict": "ok" if (worst_abs <= q16 and rel_ok) else "OUT OF BOUND"}


# ------------------------------------------------------------------------------------ inputs
def make_inputs(c, seed: int, nthreads: int):
    import ctgen

    ps = ctgen.primes(c.L)
    t0 = time.perf_counter()
    ct = ctgen.encrypt(c.fmt, c.N, c.d1, c.d2, seed, c.log_delta, ps, nthreads=nthreads)
    U = ctgen.U_matrix(seed, c.d2, c.d3, c.u_bound, nthreads=nthreads)
    return ps, ct, U, time.perf_counter() - t0


# ------------------------------------------------------------------------------------ reference arm
def arm_mode(args, world: int) -> str:
    """'strong' or 'weak': the parallelism both arms report (main() dispatches on the same rule)."""
    return "weak" if args.mode == "weak" else "strong"


def run_reference(args, rank: int, world: int = 1):
    """The reference arm: the CPU oracle as it stands on the host cores, rank 0 only (the other
    ranks exit without work), on a bounded sample of the same workload and the same `config`."""
    import ctgen

    if rank != 0:
        return
    if args.config == "modmm":  # the oracle's schoolbook on a bounded sample of the Mod-PP-MM workload
        import oracle

        cores = os.cpu_count() or 1
        p = ctgen.primes(1)[0]
        K = M = 16384
        X = ctgen.uniform_residues(9000, p, K * M, nthreads=cores).reshape(K, M)  # col-major [K][M]
        Y = ctgen.uniform_residues(9001, p, K * cores, nthreads=cores).reshape(K, cores).astype(np.int64)
        times = []
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            oracle.modmatmul(X, Y, p, nthreads=cores)
            if i >= args.warmup:
                times.append(time.perf_counter() - t0)
        t = statistics.mean(times)
        v = M * K * cores / t
        print(json.dumps({
            "impl": "reference", "metric": "Mod-PP-MM residue-MACs/s (full residues both sides, 16384^3 x 3 primes)",
            "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u128 (schoolbook residues)", "data": "synthetic", "config": {"workload": "modmm"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"per step: one prime, {cores} output columns x {M} rows x K={K}"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))
        return
    c = ctgen.CONFIGS[args.config]
    cores = os.cpu_count() or 1
    ps = ctgen.primes(c.L)
    # only prime 0's ciphertexts: the sample never touches the others (c5: 8.6 GB instead of 69 GB)
    ct = ctgen.encrypt(c.fmt, c.N, c.d1, c.d2, c.seed, c.log_delta, ps[:1], nthreads=cores)
    U = ctgen.U_matrix(c.seed, c.d2, c.d3, c.u_bound, nthreads=cores)
    import oracle

    p = ps[0]
    Ac = ct.a_polys[0].reshape(c.d2, c.rows_A) if c.rows_A else None
    Bc = ct.b_polys[0].reshape(c.d2, c.d1)
    # size each step to ~ (a few minutes / (steps + warmup)) of CPU work
    budget = min(20.0, 150.0 / max(1, args.steps + args.warmup))
    t0 = time.perf_counter()
    if Ac is not None:
        oracle.modmatmul(Ac, U, p, cols=np.arange(cores), nthreads=cores)
    oracle.modmatmul(Bc, U, p, cols=np.arange(cores), nthreads=cores)
    per_col = (time.perf_counter() - t0) / cores
    ncols = int(max(1, min(c.d3, budget / max(per_col, 1e-6))))
    times = []
    for i in range(args.warmup + args.steps):
        j0 = (i * ncols) % max(1, c.d3 - ncols + 1)
        cols = np.arange(j0, j0 + ncols)
        t0 = time.perf_counter()
        if Ac is not None:
            oracle.modmatmul(Ac, U, p, cols=cols, nthreads=cores)
        oracle.modmatmul(Bc, U, p, cols=cols, nthreads=cores)
        if i >= args.warmup:
            times.append(time.perf_counter() - t0)
    macs = c.R * c.d2 * ncols
    t = statistics.mean(times)
    v = macs / t
    sample = (f"per step: prime 0, {ncols} of {c.d3} output columns x all {c.R} stacked rows x d2={c.d2} "
              f"({macs:.3e} residue-MACs)")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": arm_mode(args, world),
        "vs_baseline": None, "dtype": "u128 (schoolbook residues)", "data": "synthetic",
        "config": config_for(c, world, arm_mode(args, world)),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


# ------------------------------------------------------------------------------------ our arm
def run_ours(args, rank: int, world: int, local_rank: int, scaling: str = "strong"):
    """The device-resident single-problem step (every prime in one ctpt_problem): at N = 1 the
    default (the strong-scaling curve's N = 1 point); with --mode weak every rank runs its own
    independent problem (seed = rank), no data-path collective."""
    import torch

    import ctgen
    from paper_2503_16080_b200 import ctpt
    from paper_2503_16080_b200.engine import CpmmEngine

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    c = ctgen.CONFIGS[args.config]
    cores = os.cpu_count() or 1
    seed = c.seed + rank
    ps, ct, U, gen_s = make_inputs(c, seed, max(1, cores // world))

    want = args.split_overlap == "on" or (args.split_overlap == "auto" and c.d3 <= 8192)
    # only the split + GEMM path has a split pass to hide (d3 <= 256 runs the fused kernels)
    inkernel_split = want and not args.rescale and len(ps) >= 2 and not args.overlap and c.d3 > 256
    eng = CpmmEngine(ctpt.Spec(c.fmt, c.N, c.d1, c.d2, c.d3, ps, rescale=int(args.rescale),
                               split_overlap=int(inkernel_split), raster_group=args.raster_group,
                               max_ctas=args.max_ctas), dev)
    a_dev = torch.from_numpy(ct.a_polys.view(np.int32)).to(dev)
    b_dev = torch.from_numpy(ct.b_polys.view(np.int32)).to(dev)
    eng.layout(a_dev, b_dev, validate=True)
    if args.rescale:
        _, U0 = ctgen.U_real(seed, c.d2, c.d3, ps[-1], nthreads=cores)
        kU = eng.precompute_rns(np.stack([(U0 % int(p)).astype(np.uint32) for p in ps]))
        del U0
    else:
        kU = eng.precompute(U)
    AU, BU = eng.alloc_outputs()
    spec, sizes = eng.spec, eng.sizes
    stream = torch.cuda.current_stream(dev)
    d3l, ra = sizes.d3_loc, sizes.rows_A
    # the library's automatic kernel choice (include/ctpt.h ctpt_kernel), stage by stage
    fused = d3l <= 256 and kU == 1 and not args.rescale  # the fused / raw-byte kernels (no limb split pass)
    n_ev = 1 if args.rescale else len(ps)

    mv = fused and kernel_path(d3l, kU, spec.u_unsigned, spec.u_offset, c.R) == "mv"
    # Split/GEMM overlap (split path): the limb split of prime l+1 runs on a side stream into the
    # other of two workspaces while prime l's GEMM runs (the split needs no shared memory and
    # little SM time, so it co-resides with the persistent GEMM); gemm(l) waits on split(l).
    # Measured (profiles/r01/split_overlap_experiment): with the overlap the GEMM slows from 14.05 to
    # 16.05 ms per launch — the co-resident split costs it far more than the 0.45 ms it hides —
    # so it is off unless asked for (--overlap).
    overlap = (not fused) and (not args.rescale) and args.overlap
    ws2 = [eng.ws, torch.empty_like(eng.ws)] if overlap else [eng.ws]
    side = torch.cuda.Stream(dev) if overlap else stream
    ev_split = [torch.cuda.Event() for _ in range(2)]
    ev_free = [torch.cuda.Event() for _ in range(2)]
    counter = [0]
    # Launch-bound workloads (c1: one 64-row tile per prime, ~5 µs of kernel against ~40 µs of
    # host-side argument checks + TMA descriptor encoding per call) replay the step as one CUDA
    # graph (the descriptors are kernel parameters, baked in at capture; tools/bench_graph.py).
    use_graph = args.graph == "on" or (args.graph == "auto" and c.residue_macs < 1e9)
    use_graph = use_graph and not overlap

    def step(ev_pairs=None, stream=stream):
        if args.rescale:  # the whole ctpt_matmul: last prime first, Rescale in the others' epilogues
            if ev_pairs is not None:
                ev_pairs[0][0].record(stream)
            ctpt.matmul(spec, eng.ctmat, eng.plain, AU, BU, eng.ws, stream=stream)
            if ev_pairs is not None:
                ev_pairs[0][1].record(stream)
            return
        for l in range(len(ps)):
            au, bu = AU[l * d3l * ra:], BU[l * d3l * c.d1:]
            if not fused and inkernel_split:  # prime l+1's split rides inside prime l's GEMM
                if l == 0:
                    ctpt.split(spec, 0, eng.ctmat, eng.ws, stream=stream)
                if ev_pairs is not None:
                    ev_pairs[l][0].record(stream)
                ctpt.gemm_next(spec, l, eng.ctmat, eng.ws, eng.plain, au, bu, stream=stream)
                if ev_pairs is not None:
                    ev_pairs[l][1].record(stream)
                continue
            if not fused:
                b = counter[0] % len(ws2)
                counter[0] += 1
                if overlap:
                    side.wait_event(ev_free[b])  # the GEMM that last read ws2[b] has finished
                ctpt.split(spec, l, eng.ctmat, ws2[b], stream=side if overlap else stream)
                if overlap:
                    ev_split[b].record(side)
                    stream.wait_event(ev_split[b])
            if ev_pairs is not None:
                ev_pairs[l][0].record(stream)
            if mv:
                ctpt.gemm_mv(spec, l, eng.ctmat, eng.plain, au, bu, eng.ws, stream=stream)
            elif fused:
                ctpt.gemm_fused(spec, l, eng.ctmat, eng.plain, au, bu, stream=stream)
            else:
                ctpt.gemm(spec, l, ws2[b], eng.plain, au, bu, stream=stream)
                if overlap:
                    ev_free[b].record(stream)
            if ev_pairs is not None:
                ev_pairs[l][1].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    graph = None
    if use_graph:
        cap = torch.cuda.Stream(dev)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=cap):
            step(stream=cap)
        for _ in range(args.warmup):
            graph.replay()
        torch.cuda.synchronize(dev)

    # ------------------------------------------------ timed region (device-resident inputs)
    gemm_ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n_ev)]
               for _ in range(args.steps)]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(dev)
    clk = ClockSampler(dev)
    time.sleep(0.3)  # let the sampler start
    t_start.record(stream)
    if overlap:
        side.wait_event(t_start)  # the first split belongs to the timed region
    step_ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    step_ev[0].record(stream)
    for s in range(args.steps):
        if graph is not None:
            graph.replay()
        else:
            step(gemm_ev[s])
        step_ev[s + 1].record(stream)
    t_end.record(stream)
    torch.cuda.synchronize(dev)
    clocks = clk.stop()
    if world > 1:
        torch.distributed.barrier()
    elapsed_ms = t_start.elapsed_time(t_end)
    step_ms = [step_ev[i].elapsed_time(step_ev[i + 1]) for i in range(args.steps)]
    if graph is not None:  # no events inside the graph: one replay = the step's n_ev launches
        gemm_ms = [t / n_ev for t in step_ms for _ in range(n_ev)]
    else:
        gemm_ms = [a.elapsed_time(b) for row in gemm_ev for (a, b) in row]
    if world > 1:
        t = torch.tensor([elapsed_ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        elapsed_ms = float(t.item())

    macs_rank = c.residue_macs  # per step
    value = world * macs_rank * args.steps / (elapsed_ms / 1e3)
    ms_per_step = elapsed_ms / args.steps

    # ------------------------------------------------ roofline of the dominant kernel (k_gemm_tc)
    mp, which = peaks()
    gemm_avg_s = statistics.mean(gemm_ms) / 1e3
    limb_macs_launch = 4 * kU * c.R * c.d2 * c.d3 * (len(ps) if args.rescale else 1)
    achieved_tops = 2 * limb_macs_launch / gemm_avg_s / 1e12
    # int8 = 2 x bf16 (the guide's nominal ratio).  Burst peak for a timed region well short of
    # MEASURED_PEAKS' 4-s sustained loop (< 1.5 s: the clocks have not settled at the power cap yet),
    # sustained peak for longer runs (c4's 20 steps take ~2.0 s: a 2-s cut flipped box to box).
    peak_key = "bf16_tflops" if elapsed_ms < 1500.0 else "bf16_tflops_sustained"
    peak_tops = 2 * float(mp[peak_key])
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "gemm_dram_bytes.json")) as f:
            traffic = json.load(f).get(c.name + ("_side_split" if inkernel_split else ""))
    except OSError:
        pass

    # ------------------------------------------------ the untimed stages, each timed on its own
    setup = setup_stage_rates(c, eng, a_dev, b_dev, U, dev, stream) if not args.rescale else None
    del a_dev, b_dev

    # ------------------------------------------------ end to end through the ABI (host buffers)
    e2e = ({"value": None, "note": "skipped (--e2e-steps 0)"} if args.e2e_steps <= 0 else
           run_e2e(args, c, ps, ct, eng, dev, stream, world) if not args.rescale else
           {"value": None, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
            "note": "ctpt_matmul_host does not Rescale; no host-buffer path for this workload"})

    gemm_share = sum(gemm_ms) / elapsed_ms
    result = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": scaling,
        "vs_baseline": None, "dtype": "int8", "data": "synthetic",
        # per-step device times (the paper reports the mean of 10 runs)
        "step_ms_stats": {"mean": statistics.mean(step_ms), "median": statistics.median(step_ms),
                          "min": min(step_ms), "max": max(step_ms)},
        "config": config_for(c, world, scaling),
        "kernel_config": {"kU": kU, "limb_macs_per_residue_mac": 4 * kU,
                          "u_plane": (f"u8: U+{eng.spec.u_offset} (ctpt_plain_precompute_unsigned)" if eng.spec.u_unsigned
                                      else "s8 balanced digits")},
        "pct_int8_datasheet": 100.0 * value * 4 * kU / world / INT8_DATASHEET_MACS,
        "rescale": bool(args.rescale),
        "vs_cublaslt_int8": cublaslt_ratio(value * 4 * kU / world, elapsed_ms),
        # % of the clock-normalised peak 148 SMs × 8192 int8 MAC/clk × the median
        # SM clock sampled during the timed region (how busy the tensor pipe is per clock)
        "pct_int8_clock_normalised": (100.0 * value * 4 * kU / world / (148 * 8192 * clocks["sm_mhz"] * 1e6)
                                      if clocks.get("sm_mhz") else None),
        "roofline": roofline_fused(c, d3l, gemm_avg_s, gemm_share, mp, which,
                                   "k_gemm_mv" if mv else "k_gemm_fused_t")
        if fused else {
                     "bound": "tensor", "achieved": achieved_tops, "peak": peak_tops, "unit": "TOP/s",
                     "frac": achieved_tops / peak_tops, "traffic": traffic if not args.rescale else None,
                     "kernel": ("ctpt_matmul: k_split + kU passes of k_gemm_tc per prime, Rescale epilogue"
                                if args.rescale else "k_gemm_tc"),
                     "peak_source": f"{which}: 2 x {peak_key} (int8/bf16 nominal 2x; timed region "
                                    f"{elapsed_ms / 1e3:.2f} s)",
                     "per_launch": (f"{limb_macs_launch:.4e} limb MACs (4·kU·R·d2·d3 · L, whole step)" if args.rescale
                                    else f"{limb_macs_launch:.4e} limb MACs (4·kU·R·d2·d3, one prime)"),
                     "avg_launch_ms": gemm_avg_s * 1e3, "share_of_step": gemm_share,
                     # achieved DRAM GB/s of that kernel (ncu bytes per launch ÷ the
                     # live per-launch time) against the measured copy bandwidth
                     "vs_int8_mma_ceiling": mma_ceiling_ratio(achieved_tops) if not args.rescale else None,
                     "dram_gbs": (traffic / gemm_avg_s / 1e9) if traffic and not args.rescale else None,
                     "dram_frac": (traffic / gemm_avg_s / 1e9 / float(mp["hbm_gbs"]))
                     if traffic and not args.rescale else None},
        "e2e": e2e,
        # per prime: k_split[_rows] + kU x k_gemm_tc, or one k_gemm_fused_t / k_gemm_mv (+ k_expand_u)
        "gpu_launches": ((1 + kU * len(ps)) if inkernel_split else
                         (2 if mv else 1 if fused else 1 + kU) * len(ps)) * args.steps,
        "split_overlap": overlap,
        "split_in_gemm": inkernel_split,
        "cuda_graph": graph is not None,
        "setup_stages": setup,
        "clocks": clocks,
        "input_generation_s": gen_s,
    }
    if rank == 0 and not args.no_cpu_baseline:
        gpu0 = None
        if not args.rescale:  # prime 0's outputs of the last timed step, for the sampled parity verdict
            n0 = d3l * ra
            gpu0 = (AU[:n0].cpu().numpy().view(np.uint32).reshape(d3l, ra),
                    BU[:d3l * c.d1].cpu().numpy().view(np.uint32).reshape(d3l, c.d1))
        result["cpu_baseline"] = cpu_oracle_rate(c, ct, U, args.cpu_seconds, gpu0)
        if not args.rescale and c.fmt != ctgen.STRUCT_A:  # decode a few columns of the timed run
            t0 = time.perf_counter()
            AUv = AU.view(len(ps), d3l, ra) if ra else None
            BUv = BU.view(len(ps), d3l, c.d1)
            pr = precision_on_sample(c, ps, AUv, BUv, U, [0, d3l - 1], cores)
            pr["seconds"] = time.perf_counter() - t0
            result["cpu_baseline"]["decoded_on_sample"] = pr
    if rank == 0:
        print(json.dumps(result))


def setup_stage_rates(c, eng, a_dev, b_dev, U, dev, stream, reps: int = 3) -> dict:
    """ctpt_layout (a1) and ctpt_plain_precompute (a2) are not in `value`; time
    each on its own (CUDA events, mean of `reps` calls, device-resident inputs) and report GB/s of
    their algorithmic bytes: layout reads every ciphertext residue and writes X (4 + 4 B per
    residue); precompute reads U as int64 and writes its digit plane(s) (8 + kU B per entry).
    The precompute call synchronises its stream once (it reads max|U| back, include/ctpt.h)."""
    import torch

    def timed(fn):
        fn()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        return e0.elapsed_time(e1) / reps / 1e3

    sz = eng.sizes
    n_in = (a_dev.numel() if sz.rows_A else 0) + b_dev.numel()
    lay_bytes = 4 * n_in + 4 * c.L * c.R * sz.d2p
    t_lay = timed(lambda: eng.layout(a_dev, b_dev, validate=False))
    U_dev = torch.from_numpy(np.ascontiguousarray(U, dtype=np.int64)).to(dev)
    mode = (eng.spec.kU, eng.spec.u_unsigned, eng.spec.u_offset)
    pre_bytes = 8 * c.d2 * c.d3 + eng.spec.kU * c.d3 * sz.d2p
    t_pre = timed(lambda: eng.precompute(U_dev))
    assert (eng.spec.kU, eng.spec.u_unsigned, eng.spec.u_offset) == mode
    mp, _ = peaks()
    hbm = float(mp["hbm_gbs"])
    return {"layout": {"ms": t_lay * 1e3, "bytes": lay_bytes, "gbs": lay_bytes / t_lay / 1e9,
                       "frac_hbm": lay_bytes / t_lay / 1e9 / hbm, "kernel": "k_layout (all primes)"},
            "plain_precompute": {"ms": t_pre * 1e3, "bytes": pre_bytes, "gbs": pre_bytes / t_pre / 1e9,
                                 "frac_hbm": pre_bytes / t_pre / 1e9 / hbm,
                                 "kernel": "k_minmax_i64 + read-back + k_plain"}}


def mma_ceiling_ratio(achieved_tops: float):
    """Achieved per-launch TOP/s ÷ the measured power-limited INT8 tensor ceiling for k_gemm_tc's
    MMA shape and operand statistics (tools/mma_ceiling.py: MMAs only, operands resident in shared
    memory; profiles/r01/int8_mma_ceiling.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r01", "int8_mma_ceiling.json")) as f:
            mc = json.load(f)
    except OSError:
        return None
    return {"frac": achieved_tops / float(mc["gemm_like_tops"]), "ceiling_tops": mc["gemm_like_tops"],
            "ceiling_sm_mhz": mc["gemm_like_sm_mhz"], "ceiling_kind": "sustained (~3 s at the power cap)",
            "source": "profiles/r01/int8_mma_ceiling.json"}


def cublaslt_ratio(limb_macs_per_s: float, elapsed_ms: float):
    """Our limb-MAC rate ÷ the measured cuBLASLt int8 GEMM rate (torch._int_mm 16384³,
    profiles/r01/int8_cublaslt_probe.json, tools/int8_probe.py): burst for short timed regions,
    sustained (4 s back to back) for long ones — the "measured INT8 ceiling" of SURVEY.md §8(d)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r01", "int8_cublaslt_probe.json")) as f:
            pr = json.load(f)
    except OSError:
        return None
    key = "burst_tops" if elapsed_ms < 1500.0 else "sustained_tops"
    return {"ratio": 2 * limb_macs_per_s / 1e12 / float(pr[key]), "cublaslt_tops": pr[key], "which": key}


def roofline_fused(c, d3l, launch_s, share, mp, which, kernel="k_gemm_fused_t"):
    """HBM roofline of the skinny kernels (k_gemm_fused_t, k_gemm_mv): algorithmic bytes per launch (one prime) = 4·R·d2
    (X int32, read once) + d3·d2 (U digits) + 4·R·d3 (outputs)."""
    alg = 4 * c.R * c.d2 + d3l * c.d2 + 4 * c.R * d3l
    gbs = alg / launch_s / 1e9
    return {"bound": "hbm", "achieved": gbs, "peak": float(mp["hbm_gbs"]), "unit": "GB/s",
            "frac": gbs / float(mp["hbm_gbs"]), "traffic": None, "kernel": kernel,
            "peak_source": f"{which}: hbm_gbs", "per_launch": f"{alg} algorithmic bytes (4·R·d2 + d3·d2 + 4·R·d3)",
            "avg_launch_ms": launch_s * 1e3, "share_of_step": share}


def pcie_bandwidth(dev, nbytes: int = 1 << 30) -> dict:
    """Pinned host<->device copy bandwidth (GB/s): each direction alone and both at once on
    two streams — the floor of the e2e path, whose every step moves its inputs and outputs."""
    import torch

    h_src = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    h_dst = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d_a = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    d_b = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def timed(fn_list):
        evs = []
        torch.cuda.synchronize(dev)
        for s, fn in fn_list:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(s):
                e0.record(s)
                fn()
                e1.record(s)
            evs.append((e0, e1))
        torch.cuda.synchronize(dev)
        return [a.elapsed_time(b) / 1e3 for a, b in evs]

    h2d = lambda: d_a.copy_(h_src, non_blocking=True)  # noqa: E731
    d2h = lambda: h_dst.copy_(d_b, non_blocking=True)  # noqa: E731
    timed([(s1, h2d), (s2, d2h)])  # warm
    t_h = min(timed([(s1, h2d)])[0] for _ in range(3))
    t_d = min(timed([(s2, d2h)])[0] for _ in range(3))
    tc = [timed([(s1, h2d), (s2, d2h)]) for _ in range(3)]
    th_c = min(t[0] for t in tc)
    td_c = min(t[1] for t in tc)
    del h_src, h_dst, d_a, d_b
    return {"h2d_gbs": nbytes / t_h / 1e9, "d2h_gbs": nbytes / t_d / 1e9,
            "h2d_concurrent_gbs": nbytes / th_c / 1e9, "d2h_concurrent_gbs": nbytes / td_c / 1e9}


def run_e2e(args, c, ps, ct, eng, dev, stream, world: int = 1):
    """Same metric through the public ABI with HOST buffers: every step is one ctpt_matmul_host
    call, which copies the ciphertexts from pinned host memory chunk by chunk, lays them out,
    splits, multiplies and copies the outputs back, with copies and compute overlapped.  With
    N ranks: barrier, every rank's own problem, max over ranks; value = N problems ÷ that time."""
    import torch

    from paper_2503_16080_b200 import ctpt

    a_h = torch.from_numpy(ct.a_polys.view(np.int32)).pin_memory()
    b_h = torch.from_numpy(ct.b_polys.view(np.int32)).pin_memory()
    AU_h = torch.empty(max(1, eng.sizes.out_AU_bytes // 4), dtype=torch.int32).pin_memory()
    BU_h = torch.empty(eng.sizes.out_BU_bytes // 4, dtype=torch.int32).pin_memory()
    # free the device-resident copies of the first leg; the host path stages chunks itself
    eng.ctmat = None
    torch.cuda.empty_cache()
    chunk = int(os.environ.get("CTPT_E2E_CHUNK", "0"))  # rows of X per pipeline chunk (0: library default)
    hws = torch.empty(ctpt.host_workspace_bytes(eng.spec, chunk), dtype=torch.uint8, device=dev)

    def step():
        ctpt.matmul_host(eng.spec, a_h, b_h, eng.plain, AU_h, BU_h, hws, chunk_rows=chunk, stream=stream)

    step()
    torch.cuda.synchronize(dev)
    if world > 1:
        torch.distributed.barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(args.e2e_steps):
        step()
    t1.record(stream)
    torch.cuda.synchronize(dev)
    ms = t0.elapsed_time(t1) / args.e2e_steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    h2d = (a_h.numel() * 4 if eng.sizes.rows_A else 0) + b_h.numel() * 4  # structured-A: Ã is not read
    d2h = eng.sizes.out_AU_bytes + eng.sizes.out_BU_bytes
    bw = pcie_bandwidth(dev)
    floor_ms = max(h2d / bw["h2d_concurrent_gbs"], d2h / bw["d2h_concurrent_gbs"]) / 1e6
    return {"value": world * c.residue_macs / (ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d * world,
            "d2h_bytes_per_step": d2h * world,
            "ms_per_step": ms, "steps": args.e2e_steps,
            "pcie": dict(bw, floor_ms=floor_ms, frac_of_floor=floor_ms / ms),
            "path": "ctpt_matmul_host: pinned host ciphertexts -> chunked H2D || layout+split+GEMM || D2H "
                    "(3 streams) -> pinned host outputs"}


def gpu_uuid_of(dev) -> str | None:
    """nvidia-smi id of the CUDA device `dev` (its UUID: NVML indices need not follow CUDA's order)."""
    import torch

    try:
        return f"GPU-{torch.cuda.get_device_properties(dev).uuid}"
    except (RuntimeError, AttributeError):
        return None


def kernel_path(d3_loc: int, kU: int, u_unsigned: int, u_offset: int, R: int = 1 << 30, sms: int = 148) -> str:
    """The library's automatic kernel choice for one prime (include/ctpt.h ctpt_kernel; ctpt.cu
    choose_path): the raw-byte kernel for d3_loc <= 32 with fewer 64-row tiles than SMs (and no
    unsigned-U row correction), the limbs-in-TMEM skinny kernel up to 256 columns (it forms the u8
    plane's row sums itself), else split + GEMM."""
    if kU != 1 or d3_loc > 256:
        return "split_gemm"
    if d3_loc <= 32 and not (u_unsigned and u_offset) and (R + 63) // 64 < sms:
        return "mv"
    return "fused"


def launch_unit(spec_u, eng, au, bu, stream, ev=None):
    """One (prime, column-block) unit through the stage entry points: the limb split + k_gemm_tc
    (ev brackets the GEMM), or the fused / raw-byte kernel (ev brackets it).  Returns #launches."""
    from paper_2503_16080_b200 import ctpt

    sz = eng.unit_sizes[(spec_u.col_begin, spec_u.col_end)]
    path = kernel_path(sz.d3_loc, spec_u.kU, spec_u.u_unsigned, spec_u.u_offset, sz.R)
    if path == "split_gemm":
        ctpt.split(spec_u, 0, eng.ctmat, eng.ws, stream=stream)
    if ev is not None:
        ev[0].record(stream)
    if path == "mv":
        ctpt.gemm_mv(spec_u, 0, eng.ctmat, eng.plain, au, bu, eng.ws, stream=stream)
    elif path == "fused":
        ctpt.gemm_fused(spec_u, 0, eng.ctmat, eng.plain, au, bu, stream=stream)
    else:
        ctpt.gemm(spec_u, 0, eng.ws, eng.plain, au, bu, stream=stream)
    if ev is not None:
        ev[1].record(stream)
    return (1 + spec_u.kU) if path == "split_gemm" else (2 if path == "mv" else 1)


def run_strong(args, rank: int, world: int, local_rank: int):
    """ONE problem strong-scaled over the ranks: the (prime, U-column) units of
    shard.plan_units (whole primes when world | L, else prime-major column slices), each rank's
    inputs device-resident (one laid-out X per prime it needs, prime by prime), and the GATHER of
    every unit's (A·U, B·U) block into rank 0's [L][d3][rows] buffers INSIDE the timed region:
    ipc = the GEMM epilogues store straight into rank 0's buffers through CUDA IPC mappings opened
    on each rank's own device (NVLink / NVSwitch peer stores, overlapped tile by tile with the
    MMAs); nccl = rank 0 posts every receive before computing its own units, senders isend each
    unit as soon as it is computed.  One step = every rank's units + the gather; timed with CUDA
    events on each rank from a barrier to its last kernel / receive, max over ranks; value = the
    whole problem's residue MACs ÷ that time.  At N = 1 the primes stream through one GPU."""
    import torch
    import torch.distributed as dist

    import ctgen
    from paper_2503_16080_b200 import ctpt
    from paper_2503_16080_b200.engine import CpmmEngine
    from paper_2503_16080_b200.shard import (PeerGather, choose_gather, gathered_bytes, plan_units, primes_needed,
                                             share_gather_buffers)

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    c = ctgen.CONFIGS[args.config]
    cores = os.cpu_count() or 1
    nthreads = max(1, cores // world)
    ps = ctgen.primes(c.L)
    plan = plan_units(c.L, c.d3, world)
    mine = plan[rank]
    ra = c.rows_A
    sms = torch.cuda.get_device_properties(dev).multi_processor_count

    # ---------------------------------------------------------------- which gather
    can_reach = True
    if world > 1:
        ids = [None] * world
        dist.all_gather_object(ids, torch.cuda.get_device_properties(dev).pci_bus_id)
        bus0 = ids[0]
        idx0 = next((i for i in range(torch.cuda.device_count())
                     if torch.cuda.get_device_properties(i).pci_bus_id == bus0), None)
        can_reach = idx0 is not None and ctpt.peer_access(local_rank, idx0)
    gather = choose_gather(args.gather, world, can_reach)
    # the NCCL gather's kernels need SMs of their own while the persistent GEMMs run
    max_ctas = sms - 8 if gather == "nccl" else 0

    # ---------------------------------------------------------------- inputs, prime by prime
    t0 = time.perf_counter()
    U = ctgen.U_matrix(c.seed, c.d2, c.d3, c.u_bound, nthreads=nthreads)
    engines, host_ct = {}, {}
    shared_ws = None
    want_e2e = args.e2e_steps > 0
    for l in primes_needed(mine):
        ct = ctgen.encrypt(c.fmt, c.N, c.d1, c.d2, c.seed, c.log_delta, [ps[l]], nthreads=nthreads)
        eng = CpmmEngine(ctpt.Spec(c.fmt, c.N, c.d1, c.d2, c.d3, [ps[l]], max_ctas=max_ctas), dev,
                         alloc_ws=shared_ws is None)
        if shared_ws is None:
            shared_ws = eng.ws
        eng.ws = shared_ws
        a_dev = torch.from_numpy(ct.a_polys.view(np.int32)).to(dev) if ra else None
        b_dev = torch.from_numpy(ct.b_polys.view(np.int32)).to(dev)
        eng.layout(a_dev, b_dev, validate=True)
        del a_dev, b_dev
        if not engines:
            eng.precompute(U)
        else:  # the same U for every prime: share the first engine's digit plane(s)
            first = next(iter(engines.values()))
            eng.plain = first.plain
            eng.spec = dataclasses.replace(eng.spec, kU=first.spec.kU, u_unsigned=first.spec.u_unsigned,
                                           u_offset=first.spec.u_offset)
            eng.sizes = ctpt.query_sizes(eng.spec)
        engines[l] = eng
        if want_e2e:  # the host-buffer leg reads the same per-column ciphertexts from pinned memory
            host_ct[l] = (torch.from_numpy(ct.a_polys.view(np.int32)).pin_memory() if ra else None,
                          torch.from_numpy(ct.b_polys.view(np.int32)).pin_memory())
        del ct
        torch.cuda.empty_cache()
    gen_s = time.perf_counter() - t0
    specs = []
    for u in mine:
        eng = engines[u.l]
        sp = dataclasses.replace(eng.spec, col_begin=u.c0, col_end=u.c1)
        sz = ctpt.query_sizes(sp)
        eng.unit_sizes = getattr(eng, "unit_sizes", {})
        eng.unit_sizes[(u.c0, u.c1)] = sz
        if shared_ws.numel() < sz.workspace_bytes:
            shared_ws = torch.empty(sz.workspace_bytes, dtype=torch.uint8, device=dev)
        specs.append(sp)
    for eng in engines.values():
        eng.ws = shared_ws
    kU = next(iter(engines.values())).spec.kU
    stream = torch.cuda.current_stream(dev)

    # ---------------------------------------------------------------- outputs and the gather
    out_AU = torch.empty((c.L, c.d3, max(ra, 1)), dtype=torch.int32, device=dev) if rank == 0 else None
    out_BU = torch.empty((c.L, c.d3, c.d1), dtype=torch.int32, device=dev) if rank == 0 else None
    if gather == "ipc":
        peers = share_gather_buffers(out_AU, out_BU, rank, c.L, c.d3, ra, c.d1)
    elif rank == 0:
        peers = PeerGather(out_AU.data_ptr() if ra else 0, out_BU.data_ptr(), c.L, c.d3, ra, c.d1)
    else:
        peers = None
    # per-unit local buffers: the NCCL senders' staging, and every rank's "no gather" pass
    local = [(torch.empty((u.ncols, max(ra, 1)), dtype=torch.int32, device=dev),
              torch.empty((u.ncols, c.d1), dtype=torch.int32, device=dev)) for u in mine] if world > 1 else []

    def dst(i, u, to_local):
        if to_local or (gather == "nccl" and rank != 0):
            return local[i][0].data_ptr() if ra else 0, local[i][1].data_ptr()
        return peers.block(u)

    def step(evs=None, to_local=False):
        n = 0
        reqs = []
        if gather == "nccl" and not to_local and rank == 0:
            for src in range(1, world):  # every remote receive posted before rank 0 computes
                for u in plan[src]:
                    if ra:
                        reqs.append(dist.irecv(out_AU[u.l, u.c0:u.c1], src=src))
                    reqs.append(dist.irecv(out_BU[u.l, u.c0:u.c1], src=src))
        for i, (u, sp) in enumerate(zip(mine, specs)):
            au, bu = dst(i, u, to_local)
            n += launch_unit(sp, engines[u.l], au, bu, stream, None if evs is None else evs[i])
            if gather == "nccl" and not to_local and rank != 0:
                if ra:
                    reqs.append(dist.isend(local[i][0], dst=0))
                reqs.append(dist.isend(local[i][1], dst=0))
        for r in reqs:
            r.wait()  # NCCL: the current stream waits for the transfer
        return n

    def timed(steps, to_local=False, with_events=False):
        evs = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in mine]
               for _ in range(steps)] if with_events else None
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        clk = ClockSampler(dev) if with_events else None
        if clk:
            time.sleep(0.3)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        launches = 0
        for st_i in range(steps):
            launches += step(None if evs is None else evs[st_i], to_local)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        clocks = clk.stop() if clk else None
        if world > 1:
            dist.barrier()  # every rank's stores into rank 0's buffers have landed
        ms = e0.elapsed_time(e1) / steps
        if world > 1:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        gemm = [a.elapsed_time(b) for row in evs for (a, b) in row] if evs else []
        return ms, gemm, launches, clocks

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    ms, gemm_ms, launches, clocks = timed(args.steps, with_events=True)
    ms_local, _, _, _ = timed(args.steps, to_local=True) if world > 1 else (ms, None, None, None)

    # ---------------------------------------------------------------- roofline (rank-0 unit launches)
    mp, which = peaks()
    macs = c.residue_macs
    value = macs / (ms / 1e3)
    paths = {kernel_path(engines[u.l].unit_sizes[(u.c0, u.c1)].d3_loc, kU, engines[u.l].spec.u_unsigned,
                         engines[u.l].spec.u_offset, c.R) for u in mine}
    unit_limb_macs = [4 * kU * c.R * c.d2 * u.ncols for u in mine]
    if paths == {"split_gemm"}:
        tops = [2 * m / (t / 1e3) / 1e12 for m, t in zip(unit_limb_macs * args.steps, gemm_ms)]
        peak_key = "bf16_tflops" if ms * args.steps < 1500.0 else "bf16_tflops_sustained"
        ach = 2 * sum(unit_limb_macs) * args.steps / (sum(gemm_ms) / 1e3) / 1e12
        roof = {"bound": "tensor", "achieved": ach, "peak": 2 * float(mp[peak_key]), "unit": "TOP/s",
                "frac": ach / (2 * float(mp[peak_key])), "traffic": None, "kernel": "k_gemm_tc",
                "peak_source": f"{which}: 2 x {peak_key} (int8/bf16 nominal 2x)",
                "per_launch": "4·kU·R·d2·ncols limb MACs per unit launch (rank 0's units)",
                "avg_launch_ms": statistics.mean(gemm_ms), "min_unit_tops": min(tops),
                "share_of_step": sum(gemm_ms) / args.steps / ms,
                "vs_int8_mma_ceiling": mma_ceiling_ratio(ach)}
    else:
        alg = sum(4 * c.R * c.d2 + u.ncols * c.d2 + 4 * c.R * u.ncols for u in mine) * args.steps
        gbs = alg / (sum(gemm_ms) / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": gbs, "peak": float(mp["hbm_gbs"]), "unit": "GB/s",
                "frac": gbs / float(mp["hbm_gbs"]), "traffic": None, "kernel": "/".join(sorted(paths)),
                "peak_source": f"{which}: hbm_gbs", "avg_launch_ms": statistics.mean(gemm_ms),
                "share_of_step": sum(gemm_ms) / args.steps / ms}
    gbytes = gathered_bytes(plan, ra, c.d1) if world > 1 else 0
    link = 770.0  # measured NVLink peer copy, GB/s per direction (B200_PROFILING.md)
    compute_floor_ms = 4 * kU * macs / world / (2 * float(mp["bf16_tflops"]) * 1e12 / 2) * 1e3
    gather_info = {
        "mode": gather, "bytes_into_rank0_per_step": gbytes,
        "rank0_ingest_gbs": gbytes / (ms / 1e3) / 1e9 if gbytes else 0.0,
        "link_gbs_measured_peer_copy": link,
        "gather_floor_ms": gbytes / (link * 1e9) * 1e3,
        "compute_floor_ms": compute_floor_ms,
        "frac_of_max_floor": max(gbytes / (link * 1e9) * 1e3, compute_floor_ms) / ms,
        "no_gather_ms": ms_local,
        "max_ctas": max_ctas or sms,
    }

    # ---------------------------------------------------------------- end to end from host buffers
    e2e = {"value": None, "note": "skipped (--e2e-steps 0)"}
    if want_e2e:
        for eng in engines.values():
            eng.ctmat = None
        torch.cuda.empty_cache()
        outs = []
        for u in mine:
            sz = engines[u.l].unit_sizes[(u.c0, u.c1)]
            outs.append((torch.empty(max(1, sz.out_AU_bytes // 4), dtype=torch.int32).pin_memory(),
                         torch.empty(sz.out_BU_bytes // 4, dtype=torch.int32).pin_memory()))
        hws = torch.empty(ctpt.host_workspace_bytes_units(specs, 0), dtype=torch.uint8, device=dev)
        h_a = [host_ct[u.l][0] for u in mine]
        h_b = [host_ct[u.l][1] for u in mine]
        h_plain = [engines[u.l].plain for u in mine]

        def hstep():  # every unit of this rank in ONE copy / compute pipeline (ctpt_matmul_host_units)
            ctpt.matmul_host_units(specs, h_a, h_b, h_plain, [o[0] for o in outs], [o[1] for o in outs], hws,
                                   stream=stream)

        hstep()
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.e2e_steps):
            hstep()
        f1.record(stream)
        torch.cuda.synchronize(dev)
        hms = f0.elapsed_time(f1) / args.e2e_steps
        h2d = sum((host_ct[u.l][0].numel() * 4 if ra else 0) + host_ct[u.l][1].numel() * 4 for u in mine)
        d2h = sum(au.numel() * 4 * (ra > 0) + bu.numel() * 4 for au, bu in outs)
        vals = torch.tensor([hms, h2d, d2h], dtype=torch.float64, device=dev)
        if world > 1:
            mx = vals.clone()
            dist.all_reduce(mx, op=dist.ReduceOp.MAX)
            dist.all_reduce(vals, op=dist.ReduceOp.SUM)
            hms = float(mx[0].item())
        h2d, d2h = int(vals[1].item()), int(vals[2].item())
        e2e = {"value": macs / (hms / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": hms, "steps": args.e2e_steps,
               "path": "per rank: pinned host ciphertexts -> ctpt_matmul_host_units over the rank's units (one "
                       "chunked H2D || layout + split + GEMM || D2H pipeline) -> pinned host outputs (the sharded "
                       "result in host memory)"}

    # ---------------------------------------------------------------- gather parity on sampled columns
    sample = None
    if rank == 0 and world > 1 and not args.no_cpu_baseline:
        sample = gather_parity(c, ps, plan, U, out_AU, out_BU, cores)

    result = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "int8", "data": "synthetic",
        "config": config_for(c, world, "strong"),
        "kernel_config": {"kU": kU, "limb_macs_per_residue_mac": 4 * kU,
                          "u_plane": "u8 (U + u_offset)" if next(iter(engines.values())).spec.u_unsigned else "s8",
                          "units_per_rank": [[(u.l, u.c0, u.c1) for u in us] for us in plan]},
        "pct_int8_datasheet": 100.0 * value * 4 * kU / world / INT8_DATASHEET_MACS,
        "roofline": roof, "gather": gather_info, "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clocks, "input_generation_s": gen_s,
    }
    if sample is not None:
        result["gather_parity_on_sample"] = sample
    if rank == 0 and world == 1 and not args.no_cpu_baseline and 0 in host_ct:
        ct0 = types.SimpleNamespace(primes=ps, a_polys=host_ct[0][0].numpy().view(np.uint32)[None] if ra else None,
                                    b_polys=host_ct[0][1].numpy().view(np.uint32)[None])
        gpu0 = None
        if out_AU is not None:
            gpu0 = (out_AU[0].cpu().numpy().view(np.uint32).reshape(c.d3, max(ra, 1)),
                    out_BU[0].cpu().numpy().view(np.uint32).reshape(c.d3, c.d1))
        result["cpu_baseline"] = cpu_oracle_rate(c, ct0, U, args.cpu_seconds, gpu0)
    if gather == "ipc" and rank != 0:
        peers.close()
    if rank == 0:
        print(json.dumps(result))


def gather_parity(c, ps, plan, U, out_AU, out_BU, cores):
    """After the timed run: in rank 0's GATHERED buffers, one sampled output column of the first unit
    of rank 1 and of the last rank (so at least one block that arrived through the gather) against
    the oracle's schoolbook over all R rows and the full d2 (every entry of those columns)."""
    import ctgen
    import oracle

    picks = []
    for r in sorted({1, len(plan) - 1}):
        u = plan[r][0]
        picks.append((r, u.l, u.c0))
    ra = c.rows_A
    bad, n = 0, 0
    for r, l, j in picks:
        ct = ctgen.encrypt(c.fmt, c.N, c.d1, c.d2, c.seed, c.log_delta, [ps[l]], nthreads=cores)
        cols = np.array([j])
        wb = oracle.modmatmul(ct.b_polys[0].reshape(c.d2, c.d1), U, ps[l], cols=cols, nthreads=cores)
        gb = out_BU[l, j].cpu().numpy().view(np.uint32)
        bad += int(np.count_nonzero(gb != wb[0]))
        n += gb.size
        if ra:
            wa = oracle.modmatmul(ct.a_polys[0].reshape(c.d2, ra), U, ps[l], cols=cols, nthreads=cores)
            ga = out_AU[l, j].cpu().numpy().view(np.uint32)
            bad += int(np.count_nonzero(ga != wa[0]))
            n += ga.size
        del ct
    return {"columns": [{"from_rank": r, "prime": l, "column": j} for r, l, j in picks], "entries": n,
            "mismatches": bad, "verdict": "bit-exact" if bad == 0 else "MISMATCH"}


def run_modmm(args, rank: int, world: int, local_rank: int):
    """SURVEY.md §8(f) row 4 under the bench contract: the Mod-PP-MM stage that CC-MM (Alg. 8,
    P:1843–1845) and the RGSW product (Alg. 9) reduce to — Z = X·Y mod p for 3 primes
    with FULL residues on both sides (16384³), through ctpt_modmatmul: Y's 4 balanced digit
    planes precomputed once (outside the timed region, as for a reused operand), then per prime
    the limb split of X and 4 GEMM passes (16 limb MACs per residue MAC) accumulating in the
    epilogue.  Inputs: seeded uniform residues (ctgen), device-resident; weak scaling."""
    import torch

    import ctgen
    from paper_2503_16080_b200 import ctpt

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    M = K = Nc = 16384
    L = 3
    ps = ctgen.primes(L)
    cores = os.cpu_count() or 1
    seed = 9 + rank
    ldx, plain_bytes, ws_bytes = ctpt.modmatmul_sizes(ps, M, K, Nc)
    t0 = time.perf_counter()
    Xh = np.zeros((L, M, ldx), np.uint32)
    Yh = np.empty((L, K, Nc), np.uint32)
    for l, p in enumerate(ps):
        Xh[l, :, :K] = ctgen.uniform_residues(seed * 1000 + 2 * l, p, M * K, nthreads=max(1, cores // world)).reshape(M, K)
        Yh[l] = ctgen.uniform_residues(seed * 1000 + 2 * l + 1, p, K * Nc, nthreads=max(1, cores // world)).reshape(K, Nc)
    gen_s = time.perf_counter() - t0
    X = torch.from_numpy(Xh.view(np.int32)).to(dev)
    Y = torch.from_numpy(Yh.view(np.int32)).to(dev)
    plain = torch.empty(plain_bytes, dtype=torch.uint8, device=dev)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    ZT = torch.empty((L, Nc, M), dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev)
    ctpt.modmatmul_precompute(ps, M, K, Nc, Y, plain, stream=stream)
    del Y
    for _ in range(args.warmup):
        ctpt.modmatmul(ps, M, K, Nc, X, ldx, plain, ZT, ws, stream=stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        torch.distributed.barrier()
    clk = ClockSampler(dev)
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        ctpt.modmatmul(ps, M, K, Nc, X, ldx, plain, ZT, ws, stream=stream)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    clocks = clk.stop()
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    macs = L * M * K * Nc
    value = world * macs / (ms / 1e3)
    mp, which = peaks()
    tops = 2 * 16 * macs / (ms / 1e3) / 1e12
    peak_key = "bf16_tflops" if ms * args.steps < 1500.0 else "bf16_tflops_sustained"
    result = {
        "metric": "Mod-PP-MM residue-MACs/s (full residues both sides, 16384^3 x 3 primes)", "value": value,
        "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int8", "data": "synthetic",
        "config": {"workload": "modmm: Z = X.Y mod p, X 16384x16384, Y 16384x16384 uniform residues, 3 primes < 2^31 "
                               "(SURVEY.md §8(f) row 4)", "M": M, "K": K, "N": Nc, "L": L,
                   "limb_macs_per_residue_mac": 16, "l2": "inputs 3 GiB per step > L2"},
        "pct_int8_datasheet": 100.0 * 16 * macs / (ms / 1e3) / INT8_DATASHEET_MACS,
        "roofline": {"bound": "tensor", "achieved": tops, "peak": 2 * float(mp[peak_key]), "unit": "TOP/s",
                     "frac": tops / (2 * float(mp[peak_key])), "traffic": None,
                     "kernel": "k_split + 4 passes of k_gemm_tc per prime (whole step)",
                     "vs_int8_mma_ceiling": mma_ceiling_ratio(tops)},
        "e2e": {"value": None, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
                "note": "device-resident workload (no host-buffer entry point for Mod-PP-MM)"},
        "gpu_launches": (1 + 4) * L * args.steps, "clocks": clocks, "input_generation_s": gen_s,
    }
    if rank == 0 and not args.no_cpu_baseline:
        import oracle

        p = ps[0]
        Xc = np.ascontiguousarray(Xh[0, :, :K].T)  # col-major [K][M] view of X for the oracle
        Yi = Yh[0].astype(np.int64)
        ncols = max(1, cores)
        t0 = time.perf_counter()
        want = oracle.modmatmul(Xc, Yi, p, cols=np.arange(ncols), nthreads=cores)
        dt = time.perf_counter() - t0
        got = ZT[0, :ncols].cpu().numpy().view(np.uint32)
        bad = int(np.count_nonzero(got != want))
        result["cpu_baseline"] = {"value": M * K * ncols / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
                                  "host": host_description(),
                                  "sample": f"prime 0, {ncols} output columns x {M} rows x K={K} (schoolbook __int128)",
                                  "parity_on_sample": {"entries": int(got.size), "mismatches": bad,
                                                       "verdict": "bit-exact" if bad == 0 else "MISMATCH"}}
    if rank == 0:
        print(json.dumps(result))


def relaunch_under_torchrun(args) -> int:
    """`python bench.py --gpus N` (N > 1) outside torchrun: re-run this command as N ranks under
    torch.distributed.run on this node (rendezvous on 127.0.0.1)."""
    import socket

    with socket.socket() as sock:
        sock.bind(("127.0.0.1", 0))
        port = sock.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch_under_torchrun(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: refusing to run a different "
                         f"number of ranks than asked\n")
        sys.exit(2)
    # Test hook for the multi-rank code path on a one-GPU box: CTPT_BENCH_ONE_DEVICE=1 puts every
    # rank on cuda:0 (no kernel waits on another rank's) and CTPT_DIST_BACKEND=gloo replaces NCCL
    # (which refuses two ranks on one device).  Never set by the driver; the numbers of such a run
    # are not a scaling measurement.
    if os.environ.get("CTPT_BENCH_ONE_DEVICE") == "1":
        local_rank = 0
    backend = os.environ.get("CTPT_DIST_BACKEND", "nccl")
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch

        torch.cuda.set_device(local_rank)
        if backend == "nccl":
            torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            torch.distributed.init_process_group(backend)
    try:
        if args.config == "modmm":
            run_modmm(args, rank, world, local_rank)
        elif args.mode == "weak" or args.rescale:  # Rescale needs every prime of an element: no prime units
            run_ours(args, rank, world, local_rank, scaling="weak" if world > 1 else "strong")
        elif args.mode == "strong" or world > 1 or args.config in STREAMED_CONFIGS:
            run_strong(args, rank, world, local_rank)
        else:
            run_ours(args, rank, world, local_rank, scaling="strong")
    finally:
        if world > 1:
            import torch

            torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
