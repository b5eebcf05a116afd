"""bench.py's multi-rank strong-scaling path on ONE B200 (the verdict's acceptance check for
SURVEY.md §8(e)): `bench.py --gpus N` with no launcher re-runs itself under torchrun as N ranks;
CTPT_BENCH_ONE_DEVICE=1 puts every rank on cuda:0 and CTPT_DIST_BACKEND=gloo replaces NCCL (which
refuses two ranks on one device).  The line must report n_gpus = N, strong scaling, a non-zero
gather into rank 0 through the fused IPC path, and bit-exact gathered columns (rank 0 checks
every entry of a column that came from another rank against the oracle).  No kernel waits on
another rank's, so sharing one GPU is safe; the timings of such a run are not a scaling number."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("config,gpus", [("c1", 2), ("c2", 2), ("c2", 3)])
def test_bench_gpus_n_strong_scaling_one_device(config, gpus, tmp_path):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env.update(CTPT_BENCH_ONE_DEVICE="1", CTPT_DIST_BACKEND="gloo")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(gpus), "--config", config,
                        "--steps", "2", "--warmup", "1", "--e2e-steps", "1"],
                       capture_output=True, text=True, env=env, timeout=900, cwd=str(tmp_path))
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = lines[0]
    assert d["n_gpus"] == gpus and d["scaling"] == "strong"
    assert d["gather"]["mode"] == "ipc" and d["gather"]["bytes_into_rank0_per_step"] > 0
    assert d["gather_parity_on_sample"]["verdict"] == "bit-exact", d["gather_parity_on_sample"]
    assert d["gpu_launches"] > 0 and d["e2e"]["value"] > 0
