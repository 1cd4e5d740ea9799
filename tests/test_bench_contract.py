"""bench.py's JSON-line contract (the task's bench rules and SURVEY 8(d)): the reference arm on
the host (CPU test) and our arm on the GPU (gpu test), each one short run parsed and checked key
by key."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def common_keys(d):
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "e2e", "cpu_baseline"):
        assert k in d, k
    assert d["metric"] == "ray-samples/sec fwd+bwd" and d["unit"] == "samples/s"
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["higher_is_better"] is True
    assert "workload" in d["config"]
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in d["e2e"], k
    for k in ("value", "unit", "cores", "kind", "sample"):
        assert k in d["cpu_baseline"], k
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1


def test_reference_arm_line():
    d = run_bench("--impl", "reference", "--workload", "parallel64", "--steps", "1", "--warmup", "1",
                  "--ref-seconds", "2")
    common_keys(d)
    assert d["impl"] == "reference" and d["dtype"] == "f64" and d["n_gpus"] == 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["e2e"]["value"] == d["value"] == d["cpu_baseline"]["value"]


@pytest.mark.gpu
def test_our_arm_line():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    d = run_bench("--steps", "3", "--warmup", "3", "--cpu-baseline-seconds", "1")
    common_keys(d)
    assert d["config"]["workload"] == "cone4d2048" and d["n_gpus"] == 1 and d["scaling"] == "weak"
    assert d["dtype"] == "bf16" and d["data"] == "synthetic" and "l2" in d["config"]
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert r["bound"] in ("tensor", "hbm", "alu") and 0 < r["frac"] < 1
    assert abs(r["achieved"] / r["peak"] - r["frac"]) < 1e-9
    b = d["binding_roofline"]
    assert b["bound"] in b["samples_per_s"] and 0 < b["frac"] < 1
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert 0 < d["e2e"]["value"] <= 1.5 * d["value"]
    assert d["gpu_launches"] > 0
    for k in ("sm_mhz", "sm_max_mhz", "reasons"):
        assert k in d["clocks"], k
    assert d["replicas_equal"] is True
    st = d["stash_roofline"]  # the split path's HBM view: 4 L H bytes per sample for K2, K3, K5
    assert st["bytes_per_sample"] == 4 * 5 * 256
    for k in ("forward", "backward", "dw"):
        assert 0 < st["frac"][k] < 1.2 and abs(st["achieved_gbs"][k] / st["peak_gbs"] - st["frac"][k]) < 1e-9


def test_launcher_spawns_one_rank_per_gpu():
    """`bench.py --gpus 2` without torchrun re-executes itself under torch.distributed.run with
    two ranks (dry run: each rank reports its RANK / WORLD_SIZE and exits, no GPU needed)."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--launch-dry-run"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    ranks = [json.loads(ln) for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert sorted(r["rank"] for r in ranks) == [0, 1]
    assert all(r["world"] == 2 for r in ranks)


def test_world_mismatch_fails_loudly():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2"], capture_output=True,
                         text=True, timeout=300, cwd=ROOT, env=env)
    assert out.returncode != 0 and "WORLD_SIZE" in out.stderr


def test_profiled_traffic_lookup():
    """roofline.traffic comes from the committed ncu --set full captures (profiles/traffic.json, one
    entry per workload): the dominant kernel of each bench workload has a capture, and a workload
    or kernel class without one reads as None (the line then says traffic: null)."""
    sys.path.insert(0, ROOT)
    import bench

    with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
        tr = json.load(fh)["workloads"]
    assert bench.profiled_traffic("cone4d2048", "forward", 0) in tr["cone4d2048"]["kernels"].values()
    assert bench.profiled_traffic("cone4d2048", "backward", 0) in tr["cone4d2048"]["kernels"].values()
    assert bench.profiled_traffic("fan512", "backward", 2) in tr["fan512"]["kernels"].values()
    assert bench.profiled_traffic("cone4d2048", "forward", 0) > 1e10  # the stash writes: ~21 GB per launch
    assert bench.profiled_traffic("no-such-workload", "forward", 0) is None
    assert bench.profiled_traffic("cone4d2048", "no-such-class", 0) is None


def test_reference_arm_under_two_ranks_uses_all_host_cores():
    """The driver launches the reference arm like ours (torchrun for N > 1): rank 0 alone times the
    oracle and prints one line, the other rank exits 0; torchrun's OMP_NUM_THREADS=1 must not pin
    the oracle to one core (the line's cores = the oracle's OpenMP threads)."""
    d = run_bench("--impl", "reference", "--gpus", "2", "--workload", "parallel64", "--steps", "1", "--warmup", "1",
                  "--ref-seconds", "2")
    assert d["impl"] == "reference" and d["n_gpus"] == 2
    assert d["cpu_baseline"]["cores"] == (os.cpu_count() or 1)
