"""A fixed slice of the randomized parity sweep (tests/_fuzz_parity.py, seed 31: 35/35 within
tolerance when recorded): random beams, sub-ray layouts, N_s up to 512, widths, depths up to 7,
combines, jitter, fp32 verify and ragged batches through both training paths, each against the
fp64 oracle.  Run in a subprocess (the sweep creates and destroys many contexts)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_fuzz_slice_within_tolerance():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "_fuzz_parity.py"), "16", "31"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, (out.stdout[-4000:], out.stderr[-2000:])
    assert "16/16 cases within tolerance" in out.stdout
