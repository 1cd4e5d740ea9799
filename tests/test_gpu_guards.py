"""Out-of-bounds write check of every kernel family (the GPU pool has no compute-sanitizer): the
library built as usual but run with DINR_GUARDS=1 surrounds each scratch buffer with a 4 KB guard
band of 0xA5 bytes, and dinr_get_device_status reports DINR_EDEVICE if any band changed.  Each path
runs in a fresh process (the switches are read once): tools/sanitize_driver.py drives the fused
kernels (k_fused2 + k_dw01, H = 64 per-stream loss mode), Adam, the N1 sampler and loop, N2, N4,
the H = 256 split path (k_tc_fwd3, K3, K5 and the opt-in variants), the one-tile K2 / K3 and fp32 verify."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("part,extra", [("fused", {}), ("split", {}), ("split", {"DINR_ZALL": "1"}),
                                        ("split", {"DINR_NO_BWD3": "1"}), ("verify", {})],
                         ids=["fused", "split", "split-zall", "split-k3", "verify"])
def test_no_out_of_bounds_scratch_writes(part, extra):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, DINR_GUARDS="1", **extra)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_driver.py"), part], env=env,
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, (out.stdout[-2000:], out.stderr[-3000:])
    assert "ok" in out.stdout
