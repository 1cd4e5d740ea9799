"""A slice of the randomized parity sweep (tests/_fuzz_parity.py) with a FRESH seed every run
(printed, and appended to gpurun_out/fuzz_seeds.log, so a failure can be replayed with
`python tests/_fuzz_parity.py 24 <seed>`): random beams, sub-ray layouts, N_s up to 512, widths,
depths within the advertised envelope (include/dinr.h), combines, jitter, fp32 verify and ragged
batches through every training path, each against the fp64 oracle.  Run in a subprocess (the sweep
creates and destroys many contexts).  DINR_FUZZ_SEED pins the seed."""
import os
import subprocess
import sys
import time

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_fuzz_slice_within_tolerance():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    seed = int(os.environ.get("DINR_FUZZ_SEED", str(int(time.time() * 1000) % 1_000_000_007)))
    print(f"fuzz seed {seed}")
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "fuzz_seeds.log"), "a") as fh:
        fh.write(f"{seed}\n")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "_fuzz_parity.py"), "24", str(seed)],
                         capture_output=True, text=True, timeout=1200, cwd=ROOT)
    assert out.returncode == 0, (seed, out.stdout[-4000:], out.stderr[-2000:])
    assert "24/24 cases within tolerance" in out.stdout
