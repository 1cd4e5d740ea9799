#!/usr/bin/env python
"""bench.py -- ray-samples/s (forward + backward) of the DINR training step on 1..8 B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload fan512] [--impl ours|reference]

One step = the whole north_star hot path over one per-GPU batch of B_px pixels (BASELINE
workload, synthetic seeded inputs resident in HBM): ray setup (K1), fused forward MLP
projection (K2), combine + loss (K4), fused recomputed forward + backward dX chain (K3), dW
GEMM (K5), gradient assembly, NCCL all-reduce of the gradient (ncclAvg), and the Adam update
fused with the re-pack of the bf16 weight images (NEXT row N1).  For pixel groups that fit two
128-sample tiles (fan512, parallel64) the forward, loss and backward run as one fused kernel.  Multi-GPU: launched by torchrun, one rank per GPU, views
sharded round-robin (weak scaling: B_px fixed per GPU).

Timing: L2 is flushed (256 MiB write) before every step outside the timed intervals; each
step is bracketed by CUDA events on the launching stream; K steps are bracketed by a barrier
+ synchronize; the reported time is the max over ranks.  Kernel durations for the roofline
come from a second, instrumented pass (library events around each launch).  The e2e number
goes through dinr_project_and_grad_host with pinned host buffers (H2D inputs and D2H
gradient inside the timed region).  cpu_baseline / --impl reference time the fp64 oracle on
this host's cores on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2404_19075_b200 import synth  # noqa: E402

METRIC = "ray-samples/sec fwd+bwd"
UNIT = "samples/s"


def flops_per_sample(L, H):
    """Algorithmic work of one sample, forward + backward: 2 (3L - 1) H^2."""
    return 2 * (3 * L - 1) * H * H


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return p["bf16_tflops"], p.get("bf16_tflops_sustained"), p["hbm_gbs"], "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback"


def profiled_traffic(workload, kernel_class, path_kind):
    """DRAM bytes per launch of the dominant kernel from the committed ncu --set full captures
    (profiles/traffic.json, one entry per workload, written by tools/ncu_summary.py traffic), or
    None if no capture holds this workload / kernel."""
    names = {"backward": {0: ("k_tc_bwd", "k_tc_mlp"), 1: ("k_fused<",), 2: ("k_fused2<",)}.get(path_kind, ()),
             "dw": ("k_tc_dw", "k_dw01"), "forward": ("k_tc_fwd", "k_tc_mlp"), "rays": ("k_ray_setup",),
             "loss": ("k_loss",)}
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            tr = json.load(fh)
    except Exception:
        return None
    kern = tr.get("workloads", {}).get(workload, {}).get("kernels", {})
    for want in names.get(kernel_class, ()):  # the first candidate the capture holds
        for k, v in kern.items():
            if want in k:
                return v
    return None


# ---------------------------------------------------------------------------- clocks
class ClockSampler:
    """Polls nvidia-smi (one query every ~200 ms) in a background thread."""
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap", "power.draw", "power.limit"]
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device_index):
        import threading

        self.dev = str(device_index)
        self.rows = []
        self.window = None
        self.stop_evt = threading.Event()
        self.th = threading.Thread(target=self._run, daemon=True)
        self.th.start()

    def _run(self):
        while not self.stop_evt.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", self.dev, "--query-gpu=" + ",".join(self.FIELDS),
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout
                parts = [x.strip() for x in out.strip().split(",")]
                if len(parts) == len(self.FIELDS):
                    self.rows.append((time.perf_counter(), parts))
            except Exception:
                pass
            self.stop_evt.wait(0.2)

    def mark(self, start, end):
        self.window = (start, end)

    def stop(self):
        self.stop_evt.set()
        self.th.join(timeout=10)
        rows = self.rows
        if self.window:
            w = [r for r in rows if self.window[0] <= r[0] <= self.window[1]]
            rows = w if w else rows
        sm, mx, pw, lim, reasons = [], [], [], [], set()
        for _, parts in rows:
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for flag, name in zip(parts[2:6], self.NAMES):
                if flag.lower() == "active":
                    reasons.add(name)
            try:
                pw.append(float(parts[6]))
                lim.append(float(parts[7]))
            except (ValueError, IndexError):
                pass
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w": statistics.median(pw) if pw else None, "power_limit_w": max(lim) if lim else None}


# ---------------------------------------------------------------------------- oracle timing
def oracle_rate(name, budget_s=15.0, max_pixels=1 << 20):
    """fp64 oracle (test infrastructure) on this host's cores, adaptive bounded sample."""
    from oracle import oracle as O

    O.lib()
    g = synth.geometry(name)
    th, t = synth.views(name)
    f = synth.field(name)
    B = synth.grff_matrix(f["C"], f["sigma_t"], f["sigma_s"])
    prm = synth.init_params(f["C"], f["L"])
    S, ns = g["sub_x"] * g["sub_z"], g["n_s"]
    max_pixels = min(max_pixels, len(th) * g["n_rows"] * g["n_cols"])  # (the whole dataset at most)
    n, last = 1, None
    while n <= max_pixels:
        idx = synth.pixel_batch(name, n, seed=99)
        y = synth.synthetic_y(n, 1.0)
        t0 = time.perf_counter()
        O.project_and_grad(g, th, t, f, B, prm, idx, y)
        dt = time.perf_counter() - t0
        last = (n, dt)
        if dt >= budget_s / 3:
            break
        n *= 2
    n, dt = last
    return n * S * ns / dt, n, dt


def cores():
    """Threads the oracle's OpenMP loops use: the "cores" of a host timing."""
    from oracle import oracle as O

    return O.max_threads()


# ---------------------------------------------------------------------------- reference arm
def run_reference(args, rank, world):
    if rank != 0:
        return 0
    # torch.distributed.run sets OMP_NUM_THREADS=1 for every rank; rank 0 alone runs the oracle
    # here, on all of the host's cores (set before the oracle's OpenMP runtime starts)
    if world > 1 and os.environ.get("OMP_NUM_THREADS") == "1":
        os.environ["OMP_NUM_THREADS"] = str(os.cpu_count() or 1)
    name = args.workload
    g = synth.geometry(name)
    S, ns = g["sub_x"] * g["sub_z"], g["n_s"]
    from oracle import oracle as O

    O.lib()
    th, t = synth.views(name)
    f = synth.field(name)
    B = synth.grff_matrix(f["C"], f["sigma_t"], f["sigma_s"])
    prm = synth.init_params(f["C"], f["L"])
    # bounded per-step sample, sized so W + K steps finish in about a minute
    rate, _, _ = oracle_rate(name, budget_s=min(6.0, args.ref_seconds / 4))
    per_step_samples = max(S * ns, int(rate * args.ref_seconds / max(1, args.steps + args.warmup)))
    n = max(1, per_step_samples // (S * ns))
    times = []
    for it in range(args.warmup + args.steps):
        idx = synth.pixel_batch(name, n, seed=200 + it)
        y = synth.synthetic_y(n, 1.0, seed=it)
        t0 = time.perf_counter()
        O.project_and_grad(g, th, t, f, B, prm, idx, y)
        if it >= args.warmup:
            times.append(time.perf_counter() - t0)
    ms = 1e3 * sum(times) / len(times)
    value = n * S * ns / (ms / 1e3)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": name, "pixels_per_step": n, "samples_per_pixel": S * ns, "parallelism": "host cores"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores(), "kind": "oracle",
                         "sample": f"{n} pixels x {S * ns} samples per step of the {name} workload"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------- launcher
def free_port():
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def launch_ranks(args):
    """`bench.py --gpus N` run without torchrun: re-execute this script under
    torch.distributed.run, one rank per GPU on this node (the launch the driver uses for N > 1),
    and return its exit code.  Fails loudly when fewer than N devices are visible (the reference
    arm runs the oracle on the host: rank 0 alone works, so it needs no device)."""
    if not args.launch_dry_run and args.impl != "reference":
        import torch

        have = torch.cuda.device_count()
        if have < args.gpus:
            print(f"bench.py --gpus {args.gpus}: only {have} CUDA device(s) visible", file=sys.stderr)
            return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


# ---------------------------------------------------------------------------- our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="cone4d2048", choices=list(synth.WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=0, help="pixels per GPU per step (default: workload's)")
    ap.add_argument("--cpu-baseline-seconds", type=float, default=15.0)
    ap.add_argument("--ref-seconds", type=float, default=50.0,
                    help="--impl reference: host time budget of the W + K oracle steps")
    ap.add_argument("--combine", default="beer", choices=["beer", "linear"])
    ap.add_argument("--strong", action="store_true",
                    help="strong scaling: the workload's batch is the global batch, split over the ranks")
    ap.add_argument("--full-step", action="store_true",
                    help="time the N1 epoch loop's iteration (sampler + gather + step + all-reduce + Adam at the "
                         "epoch's lr) through dinr_train_iterations on a resident view-sharded y")
    ap.add_argument("--launch-dry-run", action="store_true",
                    help="spawn the ranks, have each print its rank and world size, and exit (no GPU work)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return launch_ranks(args)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.launch_dry_run:
        print(json.dumps({"rank": rank, "world": world, "local_rank": local}), flush=True)
        return 0
    if world != args.gpus:
        print(f"bench.py --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist

    from paper_2404_19075_b200 import _lib as D
    from paper_2404_19075_b200 import build
    from paper_2404_19075_b200 import dist as pdist

    if rank == 0:
        build.build()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=dev)
        dist.barrier()

    name = args.workload
    g = synth.geometry(name)
    th, t = synth.views(name)
    f = synth.field(name, combine=args.combine)
    C_, L = f["C"], f["L"]
    H = 2 * C_
    S, ns = g["sub_x"] * g["sub_z"], g["n_s"]
    n = args.batch or synth.WORKLOADS[name]["batch"]
    if args.strong:
        n = max(1, (n + world - 1) // world)  # fixed global batch (SURVEY 8(e) strong scaling)
    P = synth.param_count(C_, L)
    B = torch.tensor(synth.grff_matrix(C_, f["sigma_t"], f["sigma_s"]), device=dev)
    params = torch.tensor(synth.init_params(C_, L), device=dev)

    ctx = D.create(local)
    D.set_geometry(ctx, g, th, t)
    stream = torch.cuda.current_stream(dev)
    D.set_field_weights(ctx, f, B, params, stream=stream)
    pdist.init_comm(ctx, rank, world)
    path_kind, path_nf = D.train_path(ctx, n)
    gemm_layers = D.train_gemm_layers(ctx, n)

    # inputs resident in HBM: a pool of distinct per-step batches from this rank's view shard
    pool = 4
    idx_pool = [torch.tensor(pdist.shard_batch(name, n, rank, world, seed=1000 + 17 * q), device=dev)
                for q in range(pool)]
    # measured data: exact line integrals of the workload phantom + 0.1 % transmission-space noise
    # (N2), synthesised on the GPU by the library before the timed region
    y_pool = []
    for q in range(pool):
        yq = torch.zeros(n, device=dev)
        D.phantom_project(ctx, synth.phantom(name), idx_pool[q], yq, combine=args.combine, noise_frac=1e-3, seed=q,
                          stream=stream)
        y_pool.append(yq)
    grad = torch.zeros(P + 1, device=dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)

    adam_m = torch.zeros(P, device=dev)
    adam_v = torch.zeros(P, device=dev)
    adam_t = [0]

    full = None
    if args.full_step:
        # N1 epoch loop (R27): every step samples this rank's pixels from its view
        # shard without replacement (per-epoch permutation), gathers y from the resident shard,
        # then local loss + gradient, all-reduce, Adam at lr0 0.95^epoch -- one dinr_train_iterations
        # call.  y shard: seeded uniform values (the work does not depend on them), view by view.
        M_, N_ = len(th), g["n_rows"] * g["n_cols"]
        nv = len(range(rank, M_, world))
        y_shard = torch.empty(nv * N_, device=dev)
        y_shard.uniform_(0.0, 1.0, generator=torch.Generator(device=dev).manual_seed(77 + rank))
        desc = D.train_desc(seed=2024, batch=n, rank=rank, world=world, sharding="views")
        full = dict(y=y_shard, desc=desc, loss=torch.zeros(1, device=dev), g=[0],
                    ipe=D.iterations_per_epoch(ctx, desc))

    def step(q):
        if full is not None:
            D.train_iterations(ctx, full["desc"], full["g"][0], 1, full["y"], params, adam_m, adam_v, grad, full["loss"],
                               stream=stream)
            full["g"][0] += 1
            return
        # one training step: local loss + gradient, gradient average across the
        # ranks, then Adam (lr 1e-3) fused with the re-pack of the bf16 weight images
        D.project_and_grad(ctx, idx_pool[q % pool], y_pool[q % pool], grad, stream=stream)
        D.allreduce_grads(ctx, grad, stream=stream)
        adam_t[0] += 1
        D.adam_step(ctx, params, grad, adam_m, adam_v, lr=1e-3, step=adam_t[0], stream=stream)

    clk = ClockSampler(local)
    time.sleep(0.5)
    for q in range(args.warmup):
        step(q)
    torch.cuda.synchronize()

    def timed_pass(instrument):
        D.set_timing(ctx, instrument)
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        l0 = D.launch_count(ctx)
        for q in range(args.steps):
            flush.fill_(q & 0xFF)
            evs[q][0].record(stream)
            step(q)
            evs[q][1].record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        launches = D.launch_count(ctx) - l0
        D.set_timing(ctx, False)
        return sum(a.elapsed_time(b) for a, b in evs), launches

    t_start = time.perf_counter()
    total_ms, launches = timed_pass(False)
    # keep the GPU under the same load for >= 1.5 s so the clock record covers the regime
    soak = 0
    while time.perf_counter() - t_start < 1.5 and soak < 2000:
        step(soak)
        soak += 1
        if soak % 20 == 0:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    clk.mark(t_start, time.perf_counter())
    clocks = clk.stop()
    # instrumented pass: per-kernel device time (events on the launching stream)
    for k in D.TIMERS:
        D.read_timing(ctx, k, reset=True)
    _, _ = timed_pass(True)
    ktimes = {k: D.read_timing(ctx, k, reset=True) for k in D.TIMERS}

    # e2e through the host-buffer entry point (pinned buffers, H2D + D2H inside the timed region)
    idx_h = [x.cpu().pin_memory() for x in idx_pool]
    y_h = [x.cpu().pin_memory() for x in y_pool]
    g_h = torch.zeros(P + 1, dtype=torch.float32).pin_memory()
    for q in range(2):
        D.project_and_grad_host(ctx, idx_h[q % pool], y_h[q % pool], g_h, allreduce=True, stream=stream)
    e2e_ms = []
    if world > 1:
        dist.barrier()
    for q in range(args.steps):
        flush.fill_(q & 0xFF)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        D.project_and_grad_host(ctx, idx_h[q % pool], y_h[q % pool], g_h, allreduce=True, stream=stream)
        e2e_ms.append(1e3 * (time.perf_counter() - t0))
    e2e_total = sum(e2e_ms)

    # replicas stay identical after allreduce + Adam: compare the parameters
    replicas_equal = True
    if world > 1:
        gathered = [torch.empty_like(params) for _ in range(world)]
        dist.all_gather(gathered, params)
        replicas_equal = all(torch.equal(gathered[0], x) for x in gathered[1:])

    # max over ranks
    vals = torch.tensor([total_ms, e2e_total], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    total_ms, e2e_total = vals.tolist()
    samples_per_step = n * S * ns * world
    ms_per_step = total_ms / args.steps
    value = samples_per_step / (ms_per_step / 1e3)
    e2e_value = samples_per_step / (e2e_total / args.steps / 1e3)

    if rank == 0:
        tf_burst, tf_sust, hbm, peak_src = peaks()
        fps = flops_per_sample(L, H)
        # per-kernel algorithmic work per launch
        nsamp = n * S * ns
        # algorithmic H x H GEMMs per sample of each kernel class on this path, from the library
        # (dinr_train_gemm_layers: forward L, dX L - 1, dW L in total; recomputes not counted)
        gl = gemm_layers
        assert sum(gl.values()) == 3 * L - 1, gl
        alg = {k: ("tensor", 2.0 * gl[k] * H * H * nsamp) for k in ("forward", "backward", "dw") if gl[k] > 0}
        alg.update({
            "rays": ("hbm", n * (8 + S * 36.0)),
            "loss": ("hbm", n * (4 + 4 + S * (4 + 4.0 * (ns // 32)) + S * 4)),
        })
        shares = {k: v[0] for k, v in ktimes.items()}
        dom = max((k for k in alg), key=lambda k: shares.get(k, 0.0))
        ms_k, n_k = ktimes[dom]
        avg_s = (ms_k / max(1, n_k)) / 1e3
        bound, work = alg[dom]
        if bound == "tensor":
            achieved = work / avg_s / 1e12
            roof = {"bound": "tensor", "achieved": achieved, "peak": tf_burst, "unit": "TFLOP/s",
                    "frac": achieved / tf_burst, "traffic": profiled_traffic(name, dom, path_kind), "kernel": dom,
                    "peak_source": f"{peak_src} bf16 dense (burst)"}
        else:
            achieved = work / avg_s / 1e9
            roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                    "traffic": profiled_traffic(name, dom, path_kind), "kernel": dom, "peak_source": f"{peak_src} HBM copy"}
        # split path (H = 256): each of K2, K3, K5 moves 4 L H bytes of stash per sample (DESIGN.md
        # section 11: h and s2 written / s2 read and delta written / h and delta read, 2 H bytes per
        # sample and layer each); their HBM view beside the tensor one
        stash = None
        if path_kind == 0 and not os.environ.get("DINR_ZALL"):
            bps = 4.0 * L * H
            stash = {"bytes_per_sample": bps, "peak_gbs": hbm, "peak_source": f"{peak_src} HBM copy",
                     "achieved_gbs": {}, "frac": {}}
            for k in ("forward", "backward", "dw"):
                ms_k2, n_k2 = ktimes.get(k, (0.0, 0))
                if n_k2 > 0 and ms_k2 > 0:
                    gbs = bps * nsamp / ((ms_k2 / n_k2) / 1e3) / 1e9
                    stash["achieved_gbs"][k] = gbs
                    stash["frac"][k] = gbs / hbm
        step_tflops = value * fps / 1e12
        # configs with small H can be bound by the MUFU (tanh per activation, sin/cos per
        # frequency: L*H + 2C per sample forward) or the FP32/FMA pipe (~10 epilogue ops per
        # activation fwd+bwd) rather than the tensor core.  Unit rates per SM per clock: MUFU 16,
        # FMA 128; clocks.max.sm 1965 MHz, 148 SMs (B200_PROFILING.md) -- DESIGN.md "Binding roofline".
        sm_rate = 148 * 1.965e9 * world
        C = H // 2
        rates = {"tensor": tf_burst * 1e12 * world / fps, "mufu": 16 * sm_rate / (L * H + 2 * C),
                 "fma": 128 * sm_rate / (10.0 * L * H)}
        bind = min(rates, key=rates.get)
        binding = {"bound": bind, "samples_per_s": {k: v for k, v in rates.items()}, "frac": value / rates[bind]}
        base_rate, base_px, base_dt = (None, 0, 0.0)
        if args.cpu_baseline_seconds > 0 and world == 1:
            base_rate, base_px, base_dt = oracle_rate(name, budget_s=args.cpu_baseline_seconds)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong" if args.strong else "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": name, "pixels_per_gpu": n, "sub_rays": S, "samples_per_ray": ns,
                       "mlp": f"{L}x{H}", "params": P, "samples_per_step": samples_per_step,
                       "combine": args.combine, "l2": "flushed (256 MiB write) before every timed step",
                       "parallelism": f"dp{world}",
                       "step": ("N1 epoch-loop iteration: sample + gather + project_and_grad + allreduce + Adam"
                                f" (dinr_train_iterations, {full['ipe']} iterations/epoch)" if full is not None else
                                "project_and_grad + allreduce + Adam on resident batches")},
            "roofline": roof,
            "step_roofline": {"flop_per_sample": fps, "achieved_tflops": step_tflops,
                              "frac_burst": step_tflops / tf_burst,
                              "frac_sustained": step_tflops / tf_sust if tf_sust else None},
            "binding_roofline": binding,
            "stash_roofline": stash,
            "kernel_ms_per_step": {k: v[0] / args.steps for k, v in ktimes.items()},
            "cpu_baseline": ({"value": base_rate, "unit": UNIT, "cores": cores(), "kind": "oracle",
                              "sample": f"{base_px} pixels ({base_px * S * ns} samples) of {name}, "
                                        f"project_and_grad in fp64, {base_dt:.1f} s"}
                             if base_rate else None),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": n * (8 + 4),
                    "d2h_bytes_per_step": (P + 1) * 4},
            "gpu_launches": launches,
            "clocks": clocks,
            "replicas_equal": replicas_equal,
        }
        print(json.dumps(line), flush=True)
    D.destroy(ctx)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
