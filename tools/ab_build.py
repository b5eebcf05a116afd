#!/usr/bin/env python
"""Build a variant of libctpt.so for an A/B measurement against the default build:

    python tools/ab_build.py OUT.so [--src=CSRC_COPY] -DCTPT_NO_TMA_STORE ...

The bench and tests load it with CTPT_LIB=OUT.so (paper_2503_16080_b200/ctpt.py); the library
itself reads no environment variables.  The same nvcc flags as __graft_entry__.build_ctpt."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__ as g  # noqa: E402

out, defs = sys.argv[1], sys.argv[2:]
src = g.CSRC
if defs and defs[0].startswith("--src="):  # another copy of csrc/ (e.g. with an older kernel header)
    src, defs = defs[0][len("--src="):], defs[1:]
cmd = [g._nvcc()] + g.NVCC_FLAGS + [f'-DCTPT_SRC_HASH="{g.source_hash()}"'] + defs + \
      ["-o", out, os.path.join(src, "ctpt.cu")]
r = subprocess.run(cmd, capture_output=True, text=True)
if r.returncode:
    sys.stderr.write(r.stderr)
sys.exit(r.returncode)
