"""Gradient parity (bf16 tolerance 1e-2, north_star) of every alternative training path, each in a
fresh process because the library reads its DINR_* path switches once:
  DINR_FUSED_V1  the one-stream fused kernel k_fused instead of k_fused2
  DINR_NO_DW01   K5 (stash + feature recompute) instead of k_dw01 for the two unfused layers
  DINR_NO_FUSED  the split path (K2 / K4 / K3 / K5) at H = 128
  DINR_NO_FWD2   the one-tile K2 (k_tc_mlp MODE 1) instead of k_tc_fwd2 at H = 256
  DINR_BWD2      the two-stream K3 experiment k_tc_bwd2 instead of k_tc_mlp MODE 2 at H = 256
  DINR_NO_BWD3   the one-tile K3 k_tc_mlp MODE 2 instead of the CTA-pair k_tc_bwd3
  DINR_ZALL      the y-only stash experiment (k_tc_fwd3 zall, k_tc_mlp MODE 3, k_tc_dwz)
  DINR_NO_FWD3   k_tc_fwd2 instead of the CTA-pair K2 k_tc_fwd3
plus the default paths for reference."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = os.path.join(ROOT, "tests", "_path_parity_child.py")

FAN = ("fan512", {}, {}, 9)
CONE256 = ("cone512", {"n_s": 32}, {}, 5)
# (switches, case, expected fused-kernel kind from dinr_train_path: 0 split, 1 k_fused, 2 k_fused2)
CASES = [
    ({}, FAN, 2),
    ({"DINR_FUSED_V1": "1"}, FAN, 1),
    ({"DINR_NO_DW01": "1"}, FAN, 2),
    ({"DINR_NO_FUSED": "1"}, FAN, 0),
    ({}, CONE256, 0),
    ({"DINR_NO_FWD2": "1"}, CONE256, 0),
    ({"DINR_BWD2": "1"}, CONE256, 0),
    ({"DINR_NO_BWD3": "1"}, CONE256, 0),
    ({"DINR_ZALL": "1"}, CONE256, 0),
    ({"DINR_NO_FWD3": "1"}, CONE256, 0),
]


@pytest.mark.parametrize("env,case,kind", CASES, ids=[",".join(e) or "default" for e, _, _ in CASES])
def test_path_gradient_parity(env, case, kind):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    name, over, fover, n = case
    e = dict(os.environ)
    for k in ("DINR_FUSED_V1", "DINR_NO_DW01", "DINR_NO_FUSED", "DINR_NO_FWD2", "DINR_BWD2", "DINR_NO_BWD3", "DINR_ZALL", "DINR_NO_FWD3"):
        e.pop(k, None)
    e.update(env)
    out = subprocess.run([sys.executable, CHILD, name, json.dumps(over), json.dumps(fover), str(n)], env=e,
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    r = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert r["path"][0] == kind, r
    assert r["max_err"] <= 1e-2, r
    assert r["loss_rel"] <= 1e-2, r
