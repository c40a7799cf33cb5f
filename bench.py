#!/usr/bin/env python3
"""Benchmark of the B200 ALS-HOSVD hot path (arXiv 2004.02583 / tenkit).

Metric (BASELINE.json): ALS-sweep effective HBM GB/s and t/st-HOSVD-ALS
time-to-solution. One *step* = one call of the public decomposition API
(t_hosvd for configs 1/3, st_hosvd for 2/4/5) on one synthetic tensor of the
config's shape. `value` = algorithmic bytes of the step's tensor passes
(init + k right + (k-1) left updates per mode, core TTM chain / st shrink;
8 bytes x (|A| + F r + I r) per contraction) / step time, with
the tensor resident in HBM; `e2e` = the same bytes / step time through the
API with a pinned host tensor (H2D of the tensor and D2H of core + factors
inside the timed region).

  python bench.py [--config 3] [--steps K] [--warmup W] [--gpus N] [--impl b200|reference]

Under torchrun (N > 1) the ranks decompose ONE tensor of the config's shape
split along its last mode (paper_2004_02583_b200.dist, NCCL): strong
scaling, `value` = the step's algorithmic bytes / the max-over-ranks step
time.
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

CONFIGS = {
    1: dict(kind="t", dims=[256, 256, 256], ranks=[10, 10, 10], alpha=0.0, nu=1e-3, eta=1e-8,
            seed=2004025831, sample_dims=[256, 256, 256]),
    2: dict(kind="st", dims=[96, 96, 96, 96], ranks=[10, 10, 10, 10], alpha=0.0, nu=1e-3,
            eta=1e-8, seed=2004025832, sample_dims=[96, 96, 96, 96]),
    3: dict(kind="t", dims=[1024, 1024, 1024], ranks=[32, 32, 32], alpha=1.0, nu=1e-4, eta=1e-8,
            seed=2004025833, sample_dims=[1024, 1024, 128]),
    4: dict(kind="st", dims=[2048, 2048, 512], ranks=[64, 64, 32], alpha=1.5, nu=1e-3, eta=1e-8,
            seed=2004025834, sample_dims=[2048, 2048, 64]),
    5: dict(kind="st", dims=[200, 200, 200, 200], ranks=[50, 50, 50, 50], alpha=0.0, nu=1e-2,
            eta=1e-10, seed=2004025835, sample_dims=[200, 200, 200, 64]),
}
ALS_SEED = 7
MAX_ITERS = 50
L2_BYTES = 126 * 2**20


def workload_name(c, dims=None):
    dims = dims or c["dims"]
    drv = "t-HOSVD-ALS" if c["kind"] == "t" else "st-HOSVD-ALS"
    return (f"{drv} {'x'.join(map(str, dims))} fp64, ranks ({','.join(map(str, c['ranks']))}), "
            f"tol {c['eta']:g}, max {MAX_ITERS} iters, ALS seed {ALS_SEED}")


# ---- algorithmic work, shared by both arms --------------------
def contraction_bytes(count, I, r):
    F = count // I
    return 8 * (count + F * r + I * r)


def step_bytes(kind, dims, ranks, per_mode):
    """per_mode: [(mode, iterations)] in processing order."""
    dims = list(dims)
    total = 0
    if kind == "t":
        count = int(np.prod(dims))
        for mode, k in per_mode:
            total += 2 * k * contraction_bytes(count, dims[mode - 1], ranks[mode - 1])
        cur = list(dims)
        for n in range(len(dims)):  # core TTM chain, ascending modes
            total += contraction_bytes(int(np.prod(cur)), cur[n], ranks[n])
            cur[n] = ranks[n]
    else:
        cur = list(dims)
        for mode, k in per_mode:
            count = int(np.prod(cur))
            I, r = cur[mode - 1], ranks[mode - 1]
            total += 2 * k * contraction_bytes(count, I, r)
            total += 8 * 2 * (count // I) * r  # shrink: read R, write the r-extent tensor
            cur[mode - 1] = r
    return total


def step_flops(kind, dims, ranks, per_mode):
    dims = list(dims)
    total = 0
    if kind == "t":
        count = int(np.prod(dims))
        for mode, k in per_mode:
            total += 2 * k * 2 * count * ranks[mode - 1]
        cur = list(dims)
        for n in range(len(dims)):
            total += 2 * int(np.prod(cur)) * ranks[n]
            cur[n] = ranks[n]
    else:
        cur = list(dims)
        for mode, k in per_mode:
            count = int(np.prod(cur))
            total += 2 * k * 2 * count * ranks[mode - 1]
            cur[mode - 1] = ranks[mode - 1]
    return total


# ---- helpers -----------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.proc = None
        self.index = index

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.2)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                out = ""
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            p = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(p[0]))
                smax.append(float(p[1]))
            except (ValueError, IndexError):
                continue
            for name, v in zip(names, p[4:8]):
                if v.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(smax),
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def load_peaks():
    peaks = {"hbm_gbs": 6650.0, "hbm_src": "fallback (B200_PROFILING.md)",
             "fp64_tflops": None, "fp64_src": None}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mp = json.load(f)
        peaks["hbm_gbs"] = float(mp["hbm_gbs"])
        peaks["hbm_src"] = "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        pass
    try:
        with open(os.path.join(ROOT, "profiles", "microbench_fp64.json")) as f:
            mb = json.load(f)
        peaks["fp64_tflops"] = float(mb["dmma_m8n8k4_tflops"])
        peaks["fp64_src"] = "measured FP64 DMMA peak on this pool's B200 (profiles/microbench_fp64.json)"
    except Exception:
        peaks["fp64_tflops"] = 37.2
        peaks["fp64_src"] = "datasheet FP64 (no microbench file)"
    return peaks


def ncu_traffic(config_id, cls):
    """DRAM bytes per launch of the kernel class `cls` ("fc" / "fr") on this
    config, from one ncu --set full capture (profiles/ncu_traffic.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f)
        return d.get(str(config_id), {}).get(cls)
    except Exception:
        return None


def make_tensor(c, dims, pinned):
    import paper_2004_02583_b200 as tk
    n = int(np.prod(dims))
    if pinned:
        import torch
        buf = torch.empty(n, dtype=torch.float64, pin_memory=True)
        arr = buf.numpy()
    else:
        buf = None
        arr = np.empty(n)
    tk.synth_tucker(dims, c["ranks"], c["alpha"], c["nu"], c["seed"], out=arr)
    return arr.reshape(dims, order="F"), buf


# ---- reference arm (the compiled reference on the host cores) -----------------
def write_config_tnsr(config_id, dims, path):
    """Synthesise the config's tensor (dims may be a slab shape) and write it
    as TNSR v1 (io.cpp:19-24,131-139). Runs in a CHILD process of the
    reference arm, so the arm's own process maps only oracle/_ref."""
    c = CONFIGS[config_id]
    a, _ = make_tensor(c, dims, pinned=False)
    flat = a.reshape(-1, order="F")
    with open(path, "wb") as f:
        f.write(b"TNSR")
        f.write(np.array([1, len(dims)], dtype="<u4").tobytes())
        f.write(np.array(dims, dtype="<u8").tobytes())
        step = 1 << 26
        for s in range(0, flat.size, step):
            f.write(flat[s:s + step].astype("<f8", copy=False).tobytes())


def tnsr_outside(config_id, dims, tmpdir):
    path = os.path.join(tmpdir, f"bench_ref_c{config_id}_{'x'.join(map(str, dims))}_{os.getpid()}.tnsr")
    subprocess.check_call([sys.executable, os.path.abspath(__file__), "--config", str(config_id),
                           "--write-tnsr", path, "--tnsr-dims", ",".join(map(str, dims))],
                          stdout=subprocess.DEVNULL)
    return path


def run_reference_tnsr(c, path, dims, steps, threads):
    """K decompositions of the tensor in `path` by the compiled, unmodified
    reference (oracle/_ref: its own read_tnsr, then tenkit::t_hosvd /
    st_hosvd, hosvd.cpp:74-191) with `threads` OpenMP threads. The timed
    quantity is the decomposition call (the relative residual included, as
    the API computes it; reading the file excluded: the tensor is resident in
    host RAM, as the B200 arm's is in HBM)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracles import Ref
    ref = Ref()
    ref.set_threads(threads)
    times, res = [], None
    for _ in range(steps):
        res, call_s = ref.hosvd_als_tnsr(path, dims, c["ranks"], sequential=(c["kind"] == "st"),
                                         eta=c["eta"], max_iters=MAX_ITERS, seed=ALS_SEED)
        times.append(call_s)
    per_mode = [(m.mode, m.iterations) for m in res.per_mode]
    nbytes = step_bytes(c["kind"], dims, c["ranks"], per_mode)
    t = sum(times) / len(times)
    return {"value": nbytes / t / 1e9, "seconds": t, "tts_s": res.seconds, "threads": threads,
            "iterations": per_mode, "dims": list(dims), "rel_err": res.relative_residual,
            "bytes": nbytes}


def run_reference_sample(c, steps=1, warmup=0):
    """The bounded CPU sample of the B200 arm's cpu_baseline: the same
    decomposition on the config's slab (`sample_dims`), in-process."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracles import Ref
    ref = Ref()
    threads = os.cpu_count() or 1
    ref.set_threads(threads)
    dims = c["sample_dims"]
    a, _ = make_tensor(c, dims, pinned=False)
    times, res = [], None
    for s in range(warmup + steps):
        t0 = time.perf_counter()
        res = ref.hosvd_als(a, c["ranks"], sequential=(c["kind"] == "st"), eta=c["eta"],
                            max_iters=MAX_ITERS, seed=ALS_SEED)
        dt = time.perf_counter() - t0
        if s >= warmup:
            times.append(dt)
    per_mode = [(m.mode, m.iterations) for m in res.per_mode]
    nbytes = step_bytes(c["kind"], dims, c["ranks"], per_mode)
    t = sum(times) / len(times)
    return {"value": nbytes / t / 1e9, "seconds": t, "tts_s": res.seconds, "threads": threads,
            "iterations": per_mode, "dims": dims, "rel_err": res.relative_residual,
            "bytes": nbytes}


def full_size_cpu(config_id):
    """Full-size CPU time to solution of the compiled reference on this pool's
    GPU box, from tools/parity_full.py (profiles/parity_full_r02.jsonl)."""
    try:
        with open(os.path.join(ROOT, "profiles", "parity_full_r02.jsonl")) as f:
            for line in f:
                d = json.loads(line)
                if d.get("config") == config_id and d.get("scale", 1.0) == 1.0:
                    return {"time_to_solution_s": d["cpu"]["report_seconds"],
                            "call_s": d["cpu"]["call_s"], "threads": d["cpu"]["threads"],
                            "cpu_model": d["cpu"]["cpu_model"],
                            "source": "profiles/parity_full_r02.jsonl (tools/parity_full.py: the "
                                      "compiled reference on the full config tensor, same bytes as "
                                      "the GPU run, on this pool's GPU box)"}
    except (OSError, ValueError, KeyError):
        pass
    return None


def reference_arm(args, c, world, rank):
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    tmpdir = os.environ.get("TKG_BENCH_TMP", "/tmp")
    dims = c["dims"]
    # warm-up steps on the slab sample (thread pool, page faults of the code);
    # the K timed steps decompose the FULL config tensor
    paths = []
    try:
        if args.warmup > 0:
            paths.append(tnsr_outside(args.config, c["sample_dims"], tmpdir))
            run_reference_tnsr(c, paths[-1], c["sample_dims"], args.warmup, threads)
        paths.append(tnsr_outside(args.config, dims, tmpdir))
        r = run_reference_tnsr(c, paths[-1], dims, args.steps, threads)
    finally:
        for p in paths:
            try:
                os.unlink(p)
            except OSError:
                pass
    sample = (f"full {workload_name(c)} via the reference's read_tnsr + tenkit::{c['kind']}_hosvd "
              f"(oracle/_ref, unmodified reference sources), {threads} threads; the TNSR was written "
              f"by a child process, so this process maps only oracle/_ref; warm-up steps on a "
              f"{'x'.join(map(str, c['sample_dims']))} slab")
    line = {
        "metric": f"ALS-sweep effective HBM GB/s ({workload_name(c)})",
        "value": r["value"], "unit": "GB/s", "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["seconds"] * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded Tucker model, SURVEY §8(d))",
        "config": {"workload": workload_name(c), "config_id": args.config,
                   "iterations": r["iterations"]},
        "value_basis": VALUE_BASIS,
        "time_to_solution_s": r["tts_s"],
        "relative_residual": r["rel_err"],
        "cpu_baseline": {"value": r["value"], "unit": "GB/s", "cores": threads,
                         "kind": "reference", "sample": sample},
        "e2e": {"value": r["value"], "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    emit(line)
    return 0


VALUE_BASIS = ("effective: algorithmic bytes of the REFERENCE algorithm's tensor passes for the run's "
               "iteration counts (init + k right + (k-1) left per mode, t: core TTM chain over A, "
               "st: shrink; 8(|A| + F r + I r) per contraction, SURVEY §8(d)) / step time; the same "
               "byte count for both arms. The B200 t-HOSVD path skips the first core TTM pass over A "
               "(DESIGN §3); its relative residual is the closed form ||A||^2 - ||G||^2, or below rel 5e-5 a fused "
               "expansion pass the count does not credit (DESIGN §5)")


# ---- B200 arm ------------------------------------------------------------------------
def b200_arm(args, c, world, rank, local):
    import paper_2004_02583_b200 as tk
    from paper_2004_02583_b200 import dist as tkd
    import torch
    dims, ranks = c["dims"], c["ranks"]
    sharded = world > 1 or args.shard
    if sharded:
        # one rank per GPU, tensor split along its last mode (BASELINE north star)
        uid = tkd.broadcast_unique_id(rank) if world > 1 else tkd.nccl_unique_id()
        sc = tkd.ShardedContext.nccl(local, rank, world, uid)
        ctx = sc.ctx
        b0, nl = tkd.shard_range(dims[-1], rank, world)
    else:
        ctx = tk.Context(local)
        b0, nl = 0, dims[-1]
    ldims = list(dims[:-1]) + [nl]
    n = int(np.prod(ldims))
    host_buf = torch.empty(n, dtype=torch.float64, pin_memory=True)

    def combine(sq):  # per-slice sums of every rank's slab (exact: x + 0)
        if world == 1:
            return sq
        import torch.distributed as dist
        full = torch.zeros((dims[-1], 2), dtype=torch.float64,
                           device=f"cuda:{local}" if dist.get_backend() == "nccl" else "cpu")
        full[b0:b0 + nl] = torch.from_numpy(sq).to(full.device)
        dist.all_reduce(full)
        return full.cpu().numpy()

    tk.synth_tucker_slab(dims, ranks, c["alpha"], c["nu"], c["seed"], b0, nl, out=host_buf.numpy(),
                         combine=combine)
    host = host_buf.numpy().reshape(ldims, order="F")
    dev = torch.empty(n, dtype=torch.float64, device=f"cuda:{local}")
    dev.copy_(host_buf)
    torch.cuda.synchronize()
    dt = tk.DeviceTensor.from_torch(dev, ldims)
    eng = tk.FactorEngine.with_als(tk.AlsConfig(eta=c["eta"], max_iters=MAX_ITERS, seed=ALS_SEED))
    flush = n * 8 < 4 * L2_BYTES

    def call(x):
        if sharded:
            if c["kind"] == "t":
                return sc.t_hosvd(x, dims, tk.Truncation(ranks), eng)
            return sc.st_hosvd(x, dims, tk.Truncation(ranks), None, eng)
        if c["kind"] == "t":
            return ctx.t_hosvd(x, tk.Truncation(ranks), eng)
        return ctx.st_hosvd(x, tk.Truncation(ranks), None, eng)

    for _ in range(args.warmup):
        call(dt)
    # device-resident timed region (no per-launch instrumentation)
    barrier(world)
    total_ms, launches, reps = 0.0, 0, []
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            if flush:
                ctx.flush_l2()
            ctx.timer_start()
            tkr, rep = call(dt)
            total_ms += ctx.timer_stop()
            launches += rep.kernel_launches
            reps.append(rep)
    barrier(world)
    # the same steps again with CUDA events around every launch: per-class
    # device times for the roofline of the dominant kernel
    ctx.set_profiling(True)
    ctx.kernel_stats()  # reset
    for _ in range(args.steps):
        if flush:
            ctx.flush_l2()
        call(dt)
    stats = ctx.kernel_stats()
    ctx.set_profiling(False)
    barrier(world)
    total_ms = max_over_ranks(total_ms, world)
    ms_step = total_ms / args.steps
    rep = reps[-1]
    per_mode = [(m.mode, m.als.iterations) for m in rep.per_mode]
    nbytes = step_bytes(c["kind"], dims, ranks, per_mode)
    nflops = step_flops(c["kind"], dims, ranks, per_mode)
    # the whole job decomposes ONE tensor of the config's shape (strong scaling)
    value = nbytes / (ms_step * 1e-3) / 1e9

    # end-to-end through the API with the pinned host tensor
    for _ in range(1):
        call(host)
    barrier(world)
    e2e_ms = 0.0
    for _ in range(args.steps):
        ctx.timer_start()
        _, rep_e = call(host)
        e2e_ms += ctx.timer_stop()
    e2e_ms = max_over_ranks(e2e_ms, world) / args.steps
    # job totals: every rank uploads its slab and reads back core + factors
    h2d = int(np.prod(dims)) * 8
    d2h = world * 8 * (int(np.prod(ranks)) + sum(dims[k] * ranks[k] for k in range(len(dims))))

    if rank != 0:
        return 0

    peaks = load_peaks()
    # dominant kernel class over the timed region
    cls = max(("fc", "fr", "sweep"), key=lambda k: stats.get(k, {"ms": 0.0})["ms"])
    st = stats[cls]
    per_launch_ms = st["ms"] / max(1, st["launches"])
    ai = st["flops"] / max(1.0, st["bytes"])
    ridge = peaks["fp64_tflops"] * 1e12 / (peaks["hbm_gbs"] * 1e9)
    if ai >= ridge:
        achieved = st["flops"] / (st["ms"] * 1e-3) / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": peaks["fp64_tflops"],
                "unit": "TFLOP/s", "frac": achieved / peaks["fp64_tflops"],
                "peak_source": peaks["fp64_src"] + "; FP64 runs on the DMMA tensor pipe"}
    else:
        achieved = st["bytes"] / (st["ms"] * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / peaks["hbm_gbs"], "peak_source": peaks["hbm_src"]}
    roof.update({"kernel": {"fc": "FC fiber contraction (ALS right update A_(n)^T L')",
                            "fr": "FR fiber reduction (left update A_(n) R, init A_(n) S)",
                            "sweep": "fused sweep pass (right update, R^T R and left-update sum from one read)"}[cls],
                 "traffic": (ncu_traffic(args.config, cls) or {}).get("dram_bytes_per_launch"),
                 "traffic_source": ncu_traffic(args.config, cls), "launch_ms": per_launch_ms,
                 "arith_intensity_flop_per_byte": ai, "ridge_flop_per_byte": ridge,
                 "share_of_step": st["ms"] / (ms_step * args.steps),
                 "hbm_frac_of_dominant": (st["bytes"] / (st["ms"] * 1e-3) / 1e9) / peaks["hbm_gbs"],
                 "per_class_ms": {k: v["ms"] / args.steps for k, v in stats.items()}})

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        r = run_reference_sample(c, steps=1, warmup=0)
        cpu = {"value": r["value"], "unit": "GB/s", "cores": r["threads"], "kind": "reference",
               "sample": (f"bounded sample: tenkit::{c['kind']}_hosvd (oracle/_ref, unmodified reference sources) "
                          f"on a {'x'.join(map(str, r['dims']))} tensor from the same generator, "
                          f"{r['threads']} host threads, 1 run of {r['seconds']:.1f} s"),
               "time_to_solution_s": r["tts_s"], "full_size": full_size_cpu(args.config)}

    line = {
        "metric": f"ALS-sweep effective HBM GB/s ({workload_name(c)})",
        "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded Tucker model, SURVEY §8(d); counter-based generator csrc/synth.cpp)",
        "config": {"workload": workload_name(c), "config_id": args.config,
                   "parallelism": (f"shard{world} along mode {len(dims)} (NCCL allreduce of the I_n x R_n / "
                                   f"R_n x R_n partials, one all-to-all for the last mode)"
                                   if sharded else "single GPU"),
                   "l2": "flushed between steps" if flush else "tensor larger than L2 (%.1f GiB)" % (n * 8 / 2**30),
                   "iterations": per_mode},
        "value_basis": VALUE_BASIS,
        "time_to_solution_s": rep.seconds,
        "tflops": nflops / (ms_step * 1e-3) / 1e12,
        "relative_residual": rep.relative_residual,
        "e2e": {"value": nbytes / (e2e_ms * 1e-3) / 1e9, "unit": "GB/s",
                "ms_per_step": e2e_ms, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "roofline": roof,
        "cpu_baseline": cpu,
        "gpu_launches": launches,
        "clocks": clocks.summary(),
        "device": torch.cuda.get_device_name(local),
    }
    emit(line)
    return 0


_JSON_OUT = None


def emit(line):
    """The one JSON line goes to the real stdout; everything native code
    prints (NCCL's banner, for instance) was moved to stderr in main()."""
    out = _JSON_OUT if _JSON_OUT is not None else sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def main():
    global _JSON_OUT
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", type=int, default=3, choices=sorted(CONFIGS))
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--shard", action="store_true",
                   help="use the sharded (NCCL) path even on one GPU")
    p.add_argument("--write-tnsr", default=None, help=argparse.SUPPRESS)
    p.add_argument("--tnsr-dims", default=None, help=argparse.SUPPRESS)
    args = p.parse_args()
    if args.write_tnsr:  # child of the reference arm: synthesise + write, nothing else
        dims = [int(x) for x in args.tnsr_dims.split(",")] if args.tnsr_dims else CONFIGS[args.config]["dims"]
        write_config_tnsr(args.config, dims, args.write_tnsr)
        return 0
    args.warmup = max(args.warmup, 3) if args.impl == "b200" else args.warmup
    c = CONFIGS[args.config]
    world, rank, local = dist_setup()
    try:
        if args.impl == "reference":
            return reference_arm(args, c, world, rank)
        return b200_arm(args, c, world, rank, local)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
