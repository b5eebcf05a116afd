"""The C ABI from plain C (tests/c/ctpt_client.c): no torch, no Python between the caller and
libctpt.so.  CPU: the client compiles against include/ctpt.h, links the library and gets every
documented size and refusal from ctpt_query_sizes.  GPU: the client runs layout → plain
precompute → ctpt_matmul on its own cudaMalloc'd buffers and its outputs equal the oracle's."""
import os
import shutil
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(__file__))
LIBDIR = os.path.join(ROOT, "paper_2503_16080_b200")
CUDA = "/usr/local/cuda"


def _build(tmp_path):
    cc = shutil.which("gcc")
    if cc is None or not os.path.exists(os.path.join(LIBDIR, "libctpt.so")):
        pytest.skip("gcc or libctpt.so missing")
    exe = str(tmp_path / "ctpt_client")
    cmd = [cc, "-O1", "-Wall", "-Werror", "-o", exe, os.path.join(ROOT, "tests", "c", "ctpt_client.c"),
           "-I", os.path.join(ROOT, "include"), "-I", f"{CUDA}/include", "-L", LIBDIR, "-lctpt",
           f"-Wl,-rpath,{LIBDIR}", "-L", f"{CUDA}/lib64", "-lcudart", f"-Wl,-rpath,{CUDA}/lib64"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_client_sizes_and_refusals(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe, "sizes"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all refusals as documented" in r.stdout
    assert "c3: R=20480 d2p=16384" in r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(1, 64, 1, 64, 64, 1), (2, 64, 3, 200, 300, 2), (0, 256, 1, 130, 17, 2),
                                   (3, 32, 4, 96, 140, 1)],
                         ids=lambda s: "f%d_N%d_k%d_d2%d_d3%d_L%d" % s)
def test_c_client_matmul_matches_oracle(tmp_path, shape):
    import ctgen
    from gpu_helpers import oracle_outputs

    exe = _build(tmp_path)
    fmt, N, k, d2, d3, L = shape
    d1 = N * k
    ps = ctgen.primes(L)
    ct = ctgen.encrypt(fmt, N, d1, d2, 31, 20, ps)
    U = ctgen.U_matrix(31, d2, d3, 8)
    inp, out = tmp_path / "in.bin", tmp_path / "out.bin"
    with open(inp, "wb") as f:
        f.write(np.array([fmt, L], np.int32).tobytes())
        f.write(np.array([N, d1, d2, d3], np.int64).tobytes())
        f.write(np.array(ps, np.uint32).tobytes())
        if fmt != ctgen.STRUCT_A:
            f.write(np.ascontiguousarray(ct.a_polys, np.uint32).tobytes())
        f.write(np.ascontiguousarray(ct.b_polys, np.uint32).tobytes())
        f.write(np.ascontiguousarray(U, np.int64).tobytes())
    r = subprocess.run([exe, "run", str(inp), str(out)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    ra = ctgen.rows_A_of(fmt, N, d1)
    raw = np.fromfile(out, dtype=np.uint32)
    AU = raw[:L * d3 * ra].reshape(L, d3, ra)
    BU = raw[L * d3 * ra:].reshape(L, d3, d1)
    for l, p in enumerate(ps):
        wa, wb = oracle_outputs(fmt, N, d1, ct.a_polys[l], ct.b_polys[l], U, p)
        assert np.array_equal(AU[l], wa) and np.array_equal(BU[l], wb), l
