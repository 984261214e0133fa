"""A short run of every random-input checker under tools/ (each compares the CUDA path with the CPU oracle,
or two equivalent public paths bitwise, on seeded random shapes): the long runs are in
profiles/r02_fuzz_summary.txt, this keeps them from rotting and catches state-dependent regressions that the
fixed-shape tests cannot (a replayed graph reading a freed tensor, a download racing a clone, a shape without
a compiled kernel were all found this way)."""
import os
import re
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("tool,args", [
    ("fuzz_vs_oracle.py", ["250", "7"]),
    ("fuzz_vs_oracle.py", ["20", "8", "72", "260"]),
    ("fuzz_batches.py", ["80", "7"]),
    ("fuzz_pipeline.py", ["60", "7"]),
    ("fuzz_more.py", ["24", "7"]),
    ("fuzz_inputs.py", ["60", "7"]),
    ("fuzz_gemm.py", ["60", "7"]),
    ("fuzz_harness.py", ["40", "7"]),
])
def test_random_inputs(cuda, oracle_lib, tool, args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", tool)] + args, capture_output=True, text=True,
                         timeout=900, cwd=ROOT)
    text = out.stdout + out.stderr
    assert out.returncode in (0, 1), text[-2000:]
    counts = re.findall(r"(\d+) failures", text)
    assert counts, text[-2000:]
    assert all(int(c) == 0 for c in counts), text[-3000:]
