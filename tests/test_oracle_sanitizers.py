"""The oracle's C code (oracle/oracle.c) under AddressSanitizer + UndefinedBehaviorSanitizer
(SURVEY.md §5): a small C driver exercises every exported routine on tiny inputs (including
ragged sizes and negative U entries) and must exit cleanly with no sanitizer report."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

DRIVER = r"""
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include "oracle.c"

int main(void) {
  const uint32_t p = 2147352577u;
  enum { ROWS = 37, D2 = 19, D3 = 5, N = 8 };
  uint32_t* X = malloc(sizeof(uint32_t) * ROWS * D2);
  int64_t* U = malloc(sizeof(int64_t) * D2 * D3);
  uint32_t* out = malloc(sizeof(uint32_t) * ROWS * D3);
  for (int i = 0; i < ROWS * D2; ++i) X[i] = (uint32_t)((1103515245u * (unsigned)i + 12345u) % p);
  for (int i = 0; i < D2 * D3; ++i) U[i] = (i % 17) - 8;
  int64_t cols[D3] = {4, 0, 3, 1, 2};
  orc_modmatmul_cols(X, ROWS, D2, U, D3, cols, D3, p, out, 2);
  int64_t r_idx[3] = {0, 36, 17}, j_idx[3] = {4, 0, 2};
  uint32_t e[3];
  orc_modmatmul_entries(X, ROWS, D2, U, D3, r_idx, j_idx, 3, p, e, 2);
  uint32_t* C = malloc(sizeof(uint32_t) * ROWS * D3);
  int64_t all[D3] = {0, 1, 2, 3, 4};
  orc_modmatmul_cols(X, ROWS, D2, U, D3, all, D3, p, C, 1);
  uint64_t v[D3] = {1, 2, 3, 4, 5};
  uint32_t lhs[ROWS], rhs[ROWS];
  int64_t bad = orc_freivalds(X, ROWS, D2, U, D3, C, p, v, lhs, rhs, 2);
  uint32_t a[N], o[N];
  int64_t s[N];
  for (int i = 0; i < N; ++i) { a[i] = (uint32_t)(i * 977u % p); s[i] = (i % 3) - 1; }
  orc_negacyclic_mul(a, s, N, p, o);
  uint32_t acol[2 * N], bcol[2 * N], dec[2 * N];
  for (int i = 0; i < 2 * N; ++i) { acol[i] = (uint32_t)(i * 31u); bcol[i] = (uint32_t)(i * 7u); }
  int64_t keys[2 * N];
  for (int i = 0; i < 2 * N; ++i) keys[i] = (i % 3) - 1;
  int rc = 0;
  for (int fmt = 0; fmt < 4; ++fmt) rc |= orc_decrypt_col(fmt, N, fmt == 0 ? N : 2 * N, keys, acol, bcol, p, dec, 2);
  printf("%lld %u %u %d\n", (long long)bad, e[0], o[0], rc);
  free(X); free(U); free(out); free(C);
  return (bad != 0 || rc != 0) ? 1 : 0;
}
"""


@pytest.mark.skipif(shutil.which("gcc") is None, reason="gcc not available")
def test_oracle_c_under_asan_ubsan(tmp_path):
    src = tmp_path / "driver.c"
    src.write_text(DRIVER)
    exe = tmp_path / "driver"
    cmd = ["gcc", "-O1", "-g", "-fopenmp", "-fsanitize=address,undefined", "-fno-sanitize-recover=all",
           "-I", os.path.join(ROOT, "oracle"), "-o", str(exe), str(src)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0 and "sanitize" in (r.stderr or ""):
        pytest.skip("sanitizer runtime not available: " + r.stderr[-200:])
    assert r.returncode == 0, r.stderr
    env = dict(os.environ, ASAN_OPTIONS="detect_leaks=1:abort_on_error=1", UBSAN_OPTIONS="print_stacktrace=1")
    run = subprocess.run([str(exe)], capture_output=True, text=True, env=env, timeout=120)
    assert run.returncode == 0, run.stdout + run.stderr
    assert "ERROR" not in run.stderr and "runtime error" not in run.stderr, run.stderr


GEN_DRIVER = r"""
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include "ctgen.c"

int main(void) {
  uint32_t ps[2];
  if (ctgen_primes(2, ps) != 2) return 2;
  const int64_t N = 16, d2 = 5;
  int rc = 0;
  for (int fmt = 0; fmt < 4; ++fmt) {
    const int64_t k = fmt == 0 ? 1 : 3, d1 = N * k;
    const int64_t n_a = fmt == 1 ? d2 * k : (fmt == 3 ? k : d2);
    uint32_t* a = malloc(sizeof(uint32_t) * 2 * n_a * N);
    uint32_t* b = malloc(sizeof(uint32_t) * 2 * d2 * k * N);
    rc |= ctgen_encrypt(fmt, N, d1, d2, 7, 20, 2, ps, 0, d2, a, b, 2);
    free(a); free(b);
  }
  int64_t U[6 * 4];
  ctgen_U(1, 6, 4, 8, U, 2);
  double ur[6 * 4];
  int64_t ue[6 * 4];
  ctgen_U_real(1, 6, 4, ps[1], ur, ue, 2);
  printf("%d %lld %lld\n", rc, (long long)U[0], (long long)ue[0]);
  return rc != 0;
}
"""


@pytest.mark.skipif(shutil.which("gcc") is None, reason="gcc not available")
def test_generator_c_under_asan_ubsan(tmp_path):
    src = tmp_path / "gen_driver.c"
    src.write_text(GEN_DRIVER)
    exe = tmp_path / "gen_driver"
    cmd = ["gcc", "-O1", "-g", "-fopenmp", "-fsanitize=address,undefined", "-fno-sanitize-recover=all",
           "-I", os.path.join(ROOT, "ctgen"), "-o", str(exe), str(src), "-lm"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0 and "sanitize" in (r.stderr or ""):
        pytest.skip("sanitizer runtime not available: " + r.stderr[-200:])
    assert r.returncode == 0, r.stderr
    run = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120,
                         env=dict(os.environ, ASAN_OPTIONS="detect_leaks=1:abort_on_error=1"))
    assert run.returncode == 0, run.stdout + run.stderr
    assert "runtime error" not in run.stderr, run.stderr
