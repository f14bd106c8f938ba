#!/usr/bin/env python
"""Benchmark: directed message updates/s of synchronous banded BP on B200.

Default workload (N=1): BASELINE config C4 -- 2048x1536 grid, M=128,
truncated linear alpha=0.5 T=8 (m=15, reference nnz=1864), sum-product,
fp32, 100 synchronous iterations, seeded synthetic stereo.  One "step" is
one full run of the hot path over the grid: message reset, 100 iterations,
MAP labels.  For N>1 (torchrun) the grid is split into row strips with an
NCCL halo-row exchange per iteration (strong scaling: total work fixed).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line on rank 0.  ``--impl reference`` times the CPU oracle
(the f64 C restatement of the reference arithmetic, OpenMP over all host
cores) on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

FP32_NOMINAL_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12   # 74.4 TF/s at the max SM clock
FALLBACK_HBM_GBS = 6650.0                               # B200_PROFILING.md fallback


def fp32_peak():
    """FP32 ceilings (T op/s) from the committed microbenchmark record
    (profiles/fp32_peaks.json): the measured FFMA rate -- the roofline
    denominator of both domains -- and, for max-sum, the measured rate of the
    band's own FADD2 + FMNMX3 instruction stream (one add and one max per
    band candidate), reported beside it; else the nominal FFMA peak."""
    p = ROOT / "profiles" / "fp32_peaks.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"ffma": float(d["ffma_tflops"]), "add_max": float(d["add_max_tops"]),
                "source": f"measured ({p.name}: {d.get('how', '')})"}
    return {"ffma": FP32_NOMINAL_TFLOPS, "add_max": FP32_NOMINAL_TFLOPS,
            "source": "nominal 148 SM x 128 lanes x 2 x 1.965 GHz"}


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def tensor_tf32_peak():
    """Dense tf32 tensor-core peak in TFLOP/s: half the measured bf16 rate
    (MEASURED_PEAKS.json bf16_tflops, burst), else half the nominal 2250."""
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return float(json.loads(p.read_text()).get("bf16_tflops", 2250.0)) / 2
    return 1125.0


def algorithmic(cfg, pot):
    """Bytes / FLOPs per synchronous iteration: read every unary
    and every directed message once, write every directed message once;
    2*(nnz + 2M) flops per directed update (reference madd counter x2)."""
    H, W, M = cfg.height, cfg.width, cfg.M
    N = H * W
    E = cfg.n_directed
    B = 4 * M * (N + 2 * E)
    F = E * 2 * (pot.nnz + 2 * M)
    return B, F


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks.mem,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        rows = []
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) != 8:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), parts[4:], float(parts[2]),
                             float(parts[3])))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, _, r, _, _ in rows for i, v in enumerate(r)
                          if v.lower() == "active"})
        return {"sm_mhz": float(np.median([r[0] for r in rows])),
                "sm_max_mhz": max(r[1] for r in rows), "reasons": reasons,
                "mem_mhz": float(np.median([r[3] for r in rows])),
                "power_w": float(np.median([r[4] for r in rows])),
                "samples": len(rows)}


def sustained_copy_gbs(torch, dev, seconds: float = 2.0) -> float:
    """Copy bandwidth (read + write bytes) held for `seconds` of back-to-back
    1 GiB device copies -- the same sustained, power-capped regime as the
    timed message kernels (MEASURED_PEAKS.json holds a best-of-10 burst)."""
    a = torch.empty(1 << 29, dtype=torch.float16, device=dev)
    b = torch.empty_like(a)
    b.copy_(a)
    torch.cuda.synchronize()
    n, t0 = 0, time.perf_counter()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    while time.perf_counter() - t0 < seconds:
        for _ in range(20):
            b.copy_(a)
        n += 20
        torch.cuda.synchronize()
    ev1.record()
    torch.cuda.synchronize()
    return 2 * a.numel() * a.element_size() * n / (ev0.elapsed_time(ev1) / 1e3) / 1e9


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def traffic_for(kernel_name: str):
    """Per-launch DRAM bytes of the kernel from the committed ncu summary."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    if not p.exists():
        return None
    d = json.loads(p.read_text())
    return d.get(kernel_name)


# ---------------------------------------------------------------------------
# CPU baseline / reference arm: the oracle on the host cores
# ---------------------------------------------------------------------------

def cpu_sample(cfg, domain: str, min_seconds: float = 10.0, max_iters: int = 3):
    """Time synchronous iterations of the full grid with the f64 C oracle on
    all host cores; returns (updates/s, cores, sample description)."""
    import oracle
    from paper_1010_0012_b200 import synth
    model = synth.build_config_model(cfg)
    H, W = model.grid_shape
    M = model.M
    cores = os.cpu_count() or 1
    values = model.unaries if domain == "sum" else model.log_unaries
    ori = oracle.oriented_pots(model, domain, "fast")
    a = oracle.init_msgs(H, W, M, domain)
    b = a.copy()
    oracle.sync_iterate_local(H, W, M, 0, H, 1, 2, domain, "fast", values, a, b, ori, cores)
    its, t0 = 0, time.perf_counter()
    while its < max_iters:
        oracle.sync_iterate_local(H, W, M, 0, H, 1, H + 1, domain, "fast", values, a, b, ori,
                                  cores)
        a, b = b, a
        its += 1
        if time.perf_counter() - t0 >= min_seconds:
            break
    dt = time.perf_counter() - t0
    ups = cfg.n_directed * its / dt
    return ups, cores, f"{its} synchronous iteration(s) of the full {H}x{W} M={M} grid, f64"


def reference_run_sweeps_sample(cfg, domain: str, rows: int = 64, sweeps: int = 3):
    """The as-shipped reference ``sparsebp.run_sweeps`` (its default: the
    canonical in-place sequential schedule, numba, one thread by design,
    SPEC.md:264) on a bounded sample -- the first ``rows`` rows of the same
    seeded stereo pair -- timed on this host (BASELINE.md section 3 item 1,
    reference bench.py:67-77: min over sweeps).  The reference is installed
    unmodified under baseline/_ref (pip --target, git-ignored); returns None
    if it is absent."""
    ref_dir = ROOT / "baseline" / "_ref"
    if not (ref_dir / "sparsebp").exists():
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/sbp_numba_cache")
    if str(ref_dir) not in sys.path:
        sys.path.insert(0, str(ref_dir))
    import sparsebp
    from paper_1010_0012_b200 import synth
    left, right, _ = synth.noisy_stereo_pair(cfg.height, cfg.width, cfg.M, cfg.sigma, 0)
    params = sparsebp.StereoParams(M=cfg.M, alpha=cfg.alpha, T_b=cfg.T if cfg.potential == "linear"
                                   else 2.0, beta=cfg.beta, T_u=cfg.T_u)
    u, lu = sparsebp.stereo_unary_field(sparsebp.GrayImage(left[:rows]),
                                        sparsebp.GrayImage(right[:rows]), params)
    if cfg.potential == "linear":
        pot = sparsebp.truncated_linear_potential(cfg.M, cfg.alpha, cfg.T)
    else:
        d = np.abs(np.arange(cfg.M)[:, None] - np.arange(cfg.M)[None, :]).astype(np.float64)
        table = np.exp(-cfg.alpha * np.minimum(d * d, cfg.T))
        pot = sparsebp.sparse_from_dense(table, fbar=table[0, -1])
    model = sparsebp.build_grid_mrf(rows, cfg.width, cfg.M, u, pot, log_unary_provider=lu)
    warm = sparsebp.build_grid_mrf(2, 3, cfg.M, u[:6], pot, log_unary_provider=lu[:6])
    sparsebp.run_sweeps(warm, 1, kernel="fast", domain=domain)      # numba JIT / cache load
    store = sparsebp.run_sweeps(model, sweeps, kernel="fast", domain=domain)
    per_sweep = 2 * model.n_edges
    best = min(store.stats.sweep_seconds)
    return {"value": per_sweep / best, "unit": "updates/s", "cores": 1,
            "kind": "reference",
            "sample": f"sparsebp.run_sweeps(kernel='fast', domain='{domain}') as shipped "
                      f"(sequential schedule, numba, 1 thread) on rows 0..{rows - 1} of the "
                      f"{cfg.height}x{cfg.width} M={cfg.M} grid; min of {sweeps} sweeps",
            "sec_per_sweep": best}


def run_reference(args, cfg):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import oracle
    from paper_1010_0012_b200 import synth
    model = synth.build_config_model(cfg)
    H, W = model.grid_shape
    M = model.M
    cores = os.cpu_count() or 1
    values = model.unaries if args.domain == "sum" else model.log_unaries
    ori = oracle.oriented_pots(model, args.domain, "fast")
    a = oracle.init_msgs(H, W, M, args.domain)
    b = a.copy()
    # one step = one synchronous iteration of the full grid (bounded sample of
    # the 100-iteration workload; the per-iteration cost is constant)
    for _ in range(args.warmup):
        oracle.sync_iterate_local(H, W, M, 0, H, 1, H + 1, args.domain, "fast", values, a, b,
                                  ori, cores)
        a, b = b, a
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.sync_iterate_local(H, W, M, 0, H, 1, H + 1, args.domain, "fast", values, a, b,
                                  ori, cores)
        a, b = b, a
    dt = time.perf_counter() - t0
    ups = cfg.n_directed * args.steps / dt
    sample = (f"{args.steps} timed synchronous iteration(s) (after {args.warmup} warm-up) of "
              f"the full {H}x{W} M={M} grid, f64 C oracle (port of the reference bodies)")
    line = {
        "impl": "reference", "metric": "directed_message_updates_per_s", "value": ups,
        "unit": "updates/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(cfg, args, world),
        "cpu_baseline": {"value": ups, "unit": "updates/s", "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": ups, "unit": "updates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "as_shipped_run_sweeps": reference_run_sweeps_sample(cfg, args.domain),
    }
    print(json.dumps(line), flush=True)


def config_dict(cfg, args, world):
    return {"workload": f"{cfg.name}: {cfg.width}x{cfg.height} grid, M={cfg.M}, "
                        f"{cfg.potential} alpha={cfg.alpha} T={cfg.T}, {args.domain}-product, "
                        f"{args.iters} synchronous iterations",
            "grid": [cfg.height, cfg.width], "M": cfg.M, "iterations": args.iters,
            "domain": args.domain, "potential": cfg.potential, "alpha": cfg.alpha, "T": cfg.T,
            "parallelism": f"row-strips x{world}" if world > 1 else "single GPU",
            "l2": f"inputs larger than L2 (~{algorithmic(cfg, cfg.build_potential())[0] / 1e9:.1f} GB "
                  "read+written per iteration vs 126 MB L2)"}


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    from paper_1010_0012_b200 import synth
    from paper_1010_0012_b200.engine import GridEngine
    from paper_1010_0012_b200.strips import GpuStrip, partition_rows, run_rank

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    r0, rows = partition_rows(cfg.height, world)[rank]
    smodel = synth.StripModel(cfg)
    values = synth.config_values(cfg, args.domain, seed=0, r0=r0, rows=rows)
    if world > 1:
        strip = GpuStrip(smodel, r0, rows, args.domain, "fast", device=dev, values=values)
        eng = strip.engine
        interior = torch.cuda.Stream(device=dev)
    else:
        eng = GridEngine(smodel, args.domain, "fast", device=dev, values=values)
    torch.cuda.synchronize()
    iter_events: list = []
    strip_timing: list = []
    host_s: list = []

    def step(record):
        eng.reset()
        if world > 1:
            if record:
                ev0 = torch.cuda.Event(enable_timing=True)
                ev0.record()
            strip_timing.clear()
            h0 = time.perf_counter()
            run_rank(strip, args.iters, rank, world, interior_stream=interior,
                     timing=strip_timing if record else None)
            host_s.append(time.perf_counter() - h0)
            if record:
                ev1 = torch.cuda.Event(enable_timing=True)
                ev1.record()
                iter_events.append((ev0, ev1, args.iters))
        else:
            evs = [] if record else None
            eng.step(args.iters, events=evs)
            if record:
                # iteration 0 reads no messages (SBP_ITER_FIRST): the roofline
                # is taken over the steady-state launches 1..iters-1
                iter_events.extend(evs[1:])
        return eng.labels()

    for _ in range(args.warmup):
        step(False)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        start.record()
        for _ in range(args.steps):
            step(True)
        stop.record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    eng.raise_if_degenerate()
    ms = start.elapsed_time(stop)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    per_rank = None
    if world > 1:
        from paper_1010_0012_b200.strips import summarize_timing
        mine = summarize_timing(strip_timing)      # last timed step, medians
        mine.update(rank=rank, rows=rows,
                    host_enqueue_ms_per_iteration=float(np.median(host_s)) / args.iters * 1e3)
        gathered = [None] * world
        dist.all_gather_object(gathered, mine)
        per_rank = gathered
    # message-kernel launches: (ms, iterations in the launch).  A fused launch
    # (temporal blocking) runs `levels` iterations and moves the algorithmic
    # bytes B once; the roofline is taken over the full-length launches.
    launches = [(a.elapsed_time(b), n) for a, b, n in iter_events]
    kern_ms = sum(t for t, _ in launches) / max(1, sum(n for _, n in launches))
    levels = max((n for _, n in launches), default=1) if world == 1 else 1
    full = [t for t, n in launches if n == levels] or [kern_ms * levels]
    launch_ms = sum(full) / len(full)

    sus = sustained_copy_gbs(torch, dev) if rank == 0 else None
    E = cfg.n_directed
    value = E * args.iters * args.steps / (ms / 1e3)
    pot = smodel.shared_potential
    B, F = algorithmic(cfg, pot)
    hbm_peak, peak_src = peaks()
    achieved = (B / world) / (launch_ms / 1e3) / 1e9
    kernel_launches = -(-args.iters // levels) if world == 1 else args.iters * 3
    launches_per_step = kernel_launches + 1   # message kernels + labels

    # e2e through the public API with host buffers; CPU baseline at N=1 only
    e2e = None
    cpu = None
    others = None
    if world == 1 and not args.kernel_only and not args.no_configs:
        others = configs_block_isolated()
    if not args.kernel_only:
        if world == 1:
            e2e = e2e_public_api(args, cfg, torch)
            ups, cores, sample = cpu_sample(cfg, args.domain)
            cpu = {"value": ups, "unit": "updates/s", "cores": cores, "kind": "port",
                   "sample": sample,
                   "as_shipped_run_sweeps": reference_run_sweeps_sample(cfg, args.domain)}
        else:
            e2e = e2e_strips(args, cfg, torch, rank, world, dev)
    if rank != 0:
        return
    line = {
        "metric": "directed_message_updates_per_s", "value": value, "unit": "updates/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": f"synthetic (seeded random-dot stereo, 8-rectangle disparity, sigma={cfg.sigma:g} noise)",
        "config": config_dict(cfg, args, world),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak,
                     # ncu DRAM bytes per launch, measured on the C4 workload only
                     "traffic": traffic_for(eng.kernel_name.split("<")[0]) if cfg.name == "C4" else None,
                     "peak_source": peak_src, "kernel": eng.kernel_name,
                     "kernel_ms": launch_ms, "iterations_per_launch": levels,
                     "ms_per_iteration": kern_ms,
                     "algorithmic_bytes_per_launch": B / world,
                     "l2_bytes_per_launch": B * levels / world,
                     "l2_gbs": (B * levels / world) / (launch_ms / 1e3) / 1e9,
                     "flops_per_launch": F * levels / world,
                     "fp32_frac_nominal": (F / world) / (kern_ms / 1e3) / 1e12 / FP32_NOMINAL_TFLOPS,
                     "fp32_frac_measured": (F / world) / (kern_ms / 1e3) / 1e12 / fp32_peak()["ffma"],
                     "sustained_copy_gbs": sus,
                     "frac_of_sustained_copy": achieved / sus if sus else None},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clocks.summary(),
        "configs": others,
        "per_rank": per_rank,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def configs_block(args, torch, dev):
    """The other BASELINE configs, measured in the same run (driver-visible):
    C3 (max-product, 100 iterations) and the C5 band-width sweep (M=256,
    T in {2,5,9,17,33}, both domains, 20 iterations) with the banded kernel
    against the dense O(M^2) comparison kernel on identical unaries.  Per
    entry: median device ms per synchronous iteration (CUDA events on the
    launching stream, steady state), directed updates/s, the roofline
    max(B / HBM peak, F / FP32 peak) it is measured against, and the clocks
    sampled while it ran."""
    from paper_1010_0012_b200 import _lib, synth
    from paper_1010_0012_b200.engine import GridEngine
    hbm, _ = peaks()
    fp = fp32_peak()
    out = {"hbm_peak_gbs": hbm, "fp32_peak_tflops": fp["ffma"],
           "max_sum_band_ceiling_tops": fp["add_max"],
           "fp32_peak_source": fp["source"], "entries": []}

    def measure(eng, iters, cfg, domain, kernel):
        eng.reset()
        eng.step(2)
        torch.cuda.synchronize()
        evs: list = []
        # runs of `iters` iterations from the initial messages, repeated for
        # at least 0.5 s so the clock sampler sees the kernel under load
        with ClockSampler(dev.index) as clk:
            t0 = time.perf_counter()
            while True:
                eng.reset()
                eng.step(iters, events=evs)
                torch.cuda.synchronize()
                if time.perf_counter() - t0 >= 0.5:
                    break
        eng.raise_if_degenerate()
        per = sorted(a.elapsed_time(b) / k for a, b, k in evs)
        ms = per[len(per) // 2]
        pot = eng.model.shared_potential
        B, F = algorithmic(cfg, pot)
        if kernel == "standard":
            F = cfg.n_directed * 2 * cfg.M * cfg.M
        t_hbm = B / (hbm * 1e9) * 1e3
        t_fp = F / (fp["ffma"] * 1e12) * 1e3
        bound = "hbm" if t_hbm >= t_fp else "fp32"
        roof = {"bound": bound, "ms": max(t_hbm, t_fp), "frac": max(t_hbm, t_fp) / ms,
                "hbm_frac": t_hbm / ms, "fp32_frac": t_fp / ms}
        if "dense_tc_kernel" in eng.kernel_name:
            # 3xTF32 on the tensor cores: three tf32 MMA passes over the padded
            # table; tf32 dense peak = half the measured bf16 rate
            tf32 = tensor_tf32_peak()
            Ms = eng.grid.Ms
            t_tc = 3 * cfg.n_directed * 2 * Ms * Ms / (tf32 * 1e12) * 1e3
            bound = "hbm" if t_hbm >= t_tc else "tensor"
            roof = {"bound": bound, "ms": max(t_hbm, t_tc), "frac": max(t_hbm, t_tc) / ms,
                    "hbm_frac": t_hbm / ms, "tensor_frac": t_tc / ms, "tf32_peak_tflops": tf32,
                    "mma_passes": 3}
        if domain == "max" and kernel == "fast":
            # the max-sum band issues one FADD2 half + one FMNMX3 half per
            # candidate; its own instruction stream peaks below FFMA
            t_im = F / (fp["add_max"] * 1e12) * 1e3
            roof["band_ceiling_frac"] = max(t_hbm, t_im) / ms
        return {"config": cfg.name, "domain": domain, "kernel": kernel,
                "kernel_name": eng.kernel_name, "iterations": iters,
                "ms_per_iteration": ms, "updates_per_s": cfg.n_directed / ms * 1e3,
                "bytes_per_iteration": B, "flops_per_iteration": F,
                "roofline": roof, "clocks": clk.summary()}

    cfg = synth.CONFIGS["C3"]
    eng = GridEngine(synth.StripModel(cfg), "max", "fast", device=dev,
                     values=synth.config_values(cfg, "max"))
    out["entries"].append(measure(eng, cfg.iters, cfg, "max", "fast"))
    del eng
    torch.cuda.empty_cache()
    for domain in ("sum", "max"):
        vals = synth.config_values(synth.CONFIGS["C5_T2"], domain)
        for T in (2, 5, 9, 17, 33):
            cfg = synth.CONFIGS[f"C5_T{T}"]
            band = None
            # dense arms: the default (sum-product: 3xTF32 on the tensor cores,
            # max-sum: tiled SIMT) and, for sum-product, the SIMT kernel too
            arms = [("fast", None), ("standard", None)]
            if domain == "sum":
                arms.append(("standard", "0"))
            for kernel, tc in arms:
                if tc is not None:
                    os.environ["SBP_DENSE_TC"] = tc
                    _lib.lib().sbp_reload_config()
                try:
                    eng = GridEngine(synth.StripModel(cfg), domain, kernel, device=dev, values=vals)
                    e = measure(eng, cfg.iters if kernel == "fast" else 6, cfg, domain, kernel)
                finally:
                    if tc is not None:
                        del os.environ["SBP_DENSE_TC"]
                        _lib.lib().sbp_reload_config()
                if kernel == "fast":
                    band = e
                else:
                    key = "dense" if tc is None else "dense_simt"
                    band[key] = {k: e[k] for k in ("kernel_name", "ms_per_iteration",
                                                   "updates_per_s", "roofline")}
                    if tc is None:
                        band["speedup_band_over_dense"] = e["ms_per_iteration"] / band["ms_per_iteration"]
                    else:
                        band["speedup_band_over_dense_simt"] = e["ms_per_iteration"] / band["ms_per_iteration"]
                del eng
                torch.cuda.empty_cache()
            out["entries"].append(band)
        del vals
    return out


def configs_block_isolated():
    """configs_block in a child process (`bench.py --configs-only`): its
    kernels (tensor cores, CTA pairs, every band width) get their own CUDA
    context, so a failure there is reported in the line instead of taking the
    headline measurement down with it."""
    try:
        r = subprocess.run([sys.executable, str(Path(__file__).resolve()), "--configs-only"],
                           capture_output=True, text=True, timeout=1200)
        lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
        if r.returncode == 0 and lines:
            return json.loads(lines[-1])
        return {"error": f"configs child rc={r.returncode}: {r.stderr.strip()[-300:]}"}
    except Exception as e:   # timeout, spawn failure
        return {"error": f"configs child: {type(e).__name__}: {e}"}


def e2e_public_api(args, cfg, torch):
    """End to end through the public API with host buffers, two ways:

    * stereo pipeline (the reference's ``sparsebp stereo`` path, cli.py:121-136):
      pinned uint8 image pair -> ``build_stereo_mrf`` -> ``run_sweeps`` ->
      ``map_labels``; unaries are built on the device from the images;
    * model unaries: a model holding pinned f64 unaries -> ``run_sweeps`` ->
      ``map_labels`` (3.2 GB of f64 unaries cross PCIe each run).
    H2D inputs and the D2H labels are inside both timed regions.
    """
    import paper_1010_0012_b200 as sbp
    from paper_1010_0012_b200 import synth
    reps = max(1, min(args.steps, 3))

    def timed(fn):
        # median of the per-run wall times: one run in three can take 100 ms
        # longer on the host side (page-locked 3.2 GB source, allocator)
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            out = fn()
            ts.append(time.perf_counter() - t0)
        return sorted(ts)[len(ts) // 2], out

    left, right, _ = synth.noisy_stereo_pair(cfg.height, cfg.width, cfg.M, cfg.sigma, 0)
    imgs = []
    for img in (left, right):
        t = torch.empty(img.shape, dtype=torch.uint8, pin_memory=True)
        t.numpy()[...] = img
        imgs.append(t.numpy())
    params = sbp.StereoParams(M=cfg.M, alpha=cfg.alpha, T_b=cfg.T, beta=cfg.beta, T_u=cfg.T_u)

    # the reference stereo builder fixes a truncated-linear smoothness term;
    # other configs (C3: quadratic) wrap the same image pair with their own
    # potential (the unaries are still built on the device from the images)
    if cfg.potential == "linear":
        stereo_api = "build_stereo_mrf(left, right)"

        def stereo_model():
            return sbp.build_stereo_mrf(imgs[0], imgs[1], params)
    else:
        from paper_1010_0012_b200.stereo import StereoMrf
        stereo_api = f"StereoMrf(left, right, {cfg.potential} potential)"

        def stereo_model():
            return StereoMrf(imgs[0], imgs[1], params, cfg.build_potential())

    def stereo_once():
        model = stereo_model()
        store = sbp.run_sweeps(model, args.iters, domain=args.domain, schedule="synchronous")
        return sbp.map_labels(store)

    dt_s, labels = timed(stereo_once)

    values = synth.config_values(cfg, args.domain)
    pinned = torch.empty(values.shape, dtype=torch.float64, pin_memory=True)
    pinned.numpy()[...] = values
    del values
    host = pinned.numpy()
    if args.domain == "sum":
        model = sbp.GridMrf(cfg.height, cfg.width, cfg.M, host, cfg.build_potential())
    else:
        model = sbp.GridMrf(cfg.height, cfg.width, cfg.M, np.exp(host), cfg.build_potential(),
                            log_unaries=host)

    def unary_once():
        store = sbp.run_sweeps(model, args.iters, domain=args.domain, schedule="synchronous")
        return sbp.map_labels(store)

    dt_u, labels_u = timed(unary_once)
    assert (labels_u == labels).mean() > 0.999   # same problem, two input routes
    E = cfg.n_directed * args.iters
    return {"value": E / dt_s, "unit": "updates/s",
            "h2d_bytes_per_step": int(imgs[0].nbytes + imgs[1].nbytes),
            "d2h_bytes_per_step": int(labels.size * 4), "ms_per_step": dt_s * 1e3,
            "api": stereo_api + " + run_sweeps(schedule='synchronous') + "
                   "map_labels; unaries built on the device",
            "model_unaries": {"value": E / dt_u, "unit": "updates/s",
                              "h2d_bytes_per_step": int(host.nbytes),
                              "d2h_bytes_per_step": int(labels_u.size * 4),
                              "ms_per_step": dt_u * 1e3,
                              "api": "run_sweeps(GridMrf with pinned f64 unaries) + map_labels"}}


def e2e_strips(args, cfg, torch, rank, world, dev):
    """N>1 end to end: every rank uploads its rows of the pinned image pair,
    builds its unaries on its GPU, runs the strip iterations (NCCL halos) and
    the labels are gathered to rank 0's host.  Wall time, max over ranks."""
    import torch.distributed as dist

    import paper_1010_0012_b200 as sbp
    from paper_1010_0012_b200 import synth
    from paper_1010_0012_b200.distributed import gather_labels, run_sweeps_strips
    left, right, _ = synth.noisy_stereo_pair(cfg.height, cfg.width, cfg.M, cfg.sigma, 0)
    imgs = []
    for img in (left, right):
        t = torch.empty(img.shape, dtype=torch.uint8, pin_memory=True)
        t.numpy()[...] = img
        imgs.append(t.numpy())
    params = sbp.StereoParams(M=cfg.M, alpha=cfg.alpha, T_b=cfg.T, beta=cfg.beta, T_u=cfg.T_u)

    def once():
        model = sbp.build_stereo_mrf(imgs[0], imgs[1], params)
        eng = run_sweeps_strips(model, args.iters, domain=args.domain, device=dev)
        return gather_labels(eng)

    once()
    reps = max(1, min(args.steps, 3))
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(reps):
        labels = once()
    torch.cuda.synchronize()
    dt = torch.tensor([(time.perf_counter() - t0) / reps], dtype=torch.float64, device=dev)
    dist.all_reduce(dt, op=dist.ReduceOp.MAX)
    dt = float(dt.item())
    rows = cfg.height // world + 1
    return {"value": cfg.n_directed * args.iters / dt, "unit": "updates/s",
            "h2d_bytes_per_step": int(2 * rows * cfg.width),
            "d2h_bytes_per_step": int(cfg.height * cfg.width * 4) if rank == 0 else 0,
            "ms_per_step": dt * 1e3, "n_labels": None if labels is None else int(labels.size),
            "api": "build_stereo_mrf + distributed.run_sweeps_strips + gather_labels"}


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="C4")
    ap.add_argument("--domain", default=None)
    ap.add_argument("--iters", type=int, default=None)
    ap.add_argument("--kernel-only", action="store_true",
                    help="skip the e2e, CPU-baseline and other-config legs (kernel A/B runs)")
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the other-config block (C3, C5 band-width sweep)")
    ap.add_argument("--configs-only", action="store_true",
                    help="print the other-config block (C3, C5 sweep) as one JSON line and exit")
    args = ap.parse_args()
    if args.configs_only:
        import torch
        torch.cuda.set_device(0)
        print(json.dumps(configs_block(args, torch, torch.device("cuda", 0))))
        return
    from paper_1010_0012_b200 import synth
    cfg = synth.CONFIGS[args.config]
    args.domain = args.domain or cfg.domains[0]
    args.iters = args.iters or cfg.iters
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
