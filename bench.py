#!/usr/bin/env python
"""CP-ALS-QR (ALS-QR-BRE) sweeps/s on B200 -- the BASELINE.json metric.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

A step is one ALS-QR-BRE sweep (every factor updated once through the
dimension-tree TTM chain with branch reuse and Q0 extrapolation) of the
BASELINE config (default c2: 512^3, R=32, 1e-3 noise -- configs[1], the
single-GPU TTM roofline case).  N>1 shards X along mode 1 over N GPUs (one
process per GPU, NCCL all-reduce of the partial sums of TTMs that contract the
sharded mode); total work is fixed -> "scaling": "strong".

value      K sweeps / device time of those K sweeps (CUDA events on the solve
           stream; inputs already in HBM; max over ranks).
e2e        the same metric through the public C ABI with host buffers: H2D of X
           from pinned memory, the K-sweep solve, D2H of the model, wall clock.
roofline   the root TTM (X x_c Q_c^T), the dominant kernel: algorithmic FLOPs
           and bytes per launch / average launch time (CUDA events).
cpu_baseline  the reference itself (oracle/_ref: the unmodified reference
           headers compiled -O3 -DNDEBUG) on 1 host core, a bounded sample of
           the same workload (rank 0, N=1).
"""
from __future__ import annotations

import argparse
import json
import os

# every kernel of libcpdb loaded when the module loads, not on its first
# launch (a variant first used mid-run, e.g. the dual V-GEMM when the beta gate
# opens, would otherwise pay module loading inside the timed sweeps)
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "CP-ALS-QR sweeps/sec and root-TTM FP64 TFLOPS (% of roofline) at 1/2/4/8 B200"
CONFIGS = {
    "c1": dict(kind=0, dims=(100, 100, 100), rank=10, rho=1e-2, sweeps=50),
    "c2": dict(kind=0, dims=(512, 512, 512), rank=32, rho=1e-3, sweeps=100),
    "c3": dict(kind=0, dims=(128, 128, 128, 128), rank=16, rho=1e-2, sweeps=100),
    "c4": dict(kind=1, dims=(256, 256, 256), rank=20, rho=1e-4, sweeps=500),
    "c5": dict(kind=0, dims=(256, 256, 256, 256), rank=64, rho=1e-3, sweeps=50),
}
CPU_BASELINE_MAX_ELEMS = 1 << 28  # 2 GB of f64: larger X has no bounded reference sample
TRUTH_SEED = {"c1": 20250001, "c2": 20250002, "c3": 20250003, "c4": 20250004, "c5": 20250005}
INIT_SEED = 7


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    hbm, src = 6650.0, "fallback (B200_PROFILING.md)"
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        try:
            hbm, src = float(json.load(open(p))["hbm_gbs"]), "MEASURED_PEAKS.json"
        except Exception:
            pass
    fp = json.load(open(os.path.join(ROOT, "profiles", "fp64_peak.json")))
    return hbm, src, float(fp["dmma_m8n8k4_tflops"])


def workload_name(cfg_name, c):
    d = "x".join(str(v) for v in c["dims"])
    kind = "iid N(0,1) factors" if c["kind"] == 0 else "congruence-0.9 log-scaled factors"
    return f"{cfg_name}: {d} FP64, R={c['rank']}, {kind}, {c['rho']:g} rel. noise, ALS-QR-BRE"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons around the timed region (the recipe's
    clocks line).  nvidia-smi is started BEFORE the warm-up (its start-up takes
    driver locks that would stall the timed sweeps) and `mark()`/`stop()`
    bracket the timed window; samples stamped inside it are summarised (the
    nearest ones when the window is shorter than the sampling period)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device, period_ms=20):
        self.device, self.period, self.lines, self.proc = device, period_ms, [], None
        self.t0 = self.t1 = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", str(self.period)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            deadline = time.perf_counter() + 10.0
            while not self.lines and time.perf_counter() < deadline:
                time.sleep(0.02)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.perf_counter(), line.strip()))

    def mark(self):
        self.t0 = time.perf_counter()

    def stop(self):
        self.t1 = time.perf_counter()
        if self.proc:
            time.sleep(max(0.05, 2 * self.period / 1e3))
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        t0, t1 = self.t0 or 0.0, self.t1 or float("inf")
        inside = [l for t, l in self.lines if t0 <= t <= t1 + self.period / 1e3]
        if not inside and self.lines:  # window shorter than the period: nearest samples
            after = [l for t, l in self.lines if t >= t0]
            inside = after[:2] if after else [self.lines[-1][1]]
        for line in inside:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def init_dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        # NCCL's communicator set-up lines (rank / nranks per comm) in the log
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("gloo", rank=rank, world_size=world)
    return rank, world, local


def barrier(world):
    """Barrier across the ranks with a device synchronisation on both sides
    (the session keeps the next sweep's first update in flight between run()
    calls: the synchronisation drains it before the other ranks are met)."""
    import torch
    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        torch.cuda.synchronize()


def allmax(world, v):
    if world <= 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(v)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def cpu_reference_rate(x, c, max_sweeps):
    """The reference's own ALS-QR-BRE (oracle/_ref) on this host: 1 + n sweeps,
    steady rate from the trace's wall clock (the first, dim-tree sweep excluded)."""
    from oracle.pyoracle import Oracle, available
    kind = "reference" if available("reference") else "port"
    o = Oracle(kind)
    n = max(2, max_sweeps)
    t0 = time.perf_counter()
    r = o.solve(x, c["rank"], 1 + n, extrapolate=True, seed=INIT_SEED)
    wall = time.perf_counter() - t0
    w = [t["wall_seconds"] for t in r.trace]
    rate = n / (w[-1] - w[0])
    return rate, kind, n, wall


def bench_config(args, c, world):
    """The workload description both arms print (the reference arm runs the
    device arm's config, so the two dicts are identical)."""
    dims = list(c["dims"])
    return {"workload": workload_name(args.config, c), "dims": dims, "rank": c["rank"],
            "parallelism": f"mode-1 shards x{world}" + (
                f", reductions: {os.environ.get('CPDB_SHARD_POLICY', 'auto')} "
                "(eager all-reduce / reduce-scatter / lazy at V, per step)"
                if world > 1 else ""),
            "l2": (f"X = {np.prod(dims) * 8 / 1e9:.2f} GB > 126 MB L2: every sweep "
                   f"streams X from HBM, no flush needed"
                   if np.prod(dims) * 8 > 126e6 else
                   f"X = {np.prod(dims) * 8 / 1e6:.0f} MB fits the 126 MB L2: the job itself "
                   f"re-reads the same X every sweep, so the timed sweeps are L2-resident as "
                   f"in a real run (no flush: it would time a different job)")}


def run_reference(args, c, rank, world):
    """--impl reference: the reference's own CPU path of this workload."""
    if rank != 0:
        return 0
    from oracle.pyoracle import Oracle, available
    kind = "reference" if available("reference") else "port"
    if int(np.prod(c["dims"])) > CPU_BASELINE_MAX_ELEMS:
        print(json.dumps({"impl": "reference", "unavailable":
                          f"one single-threaded reference sweep of {workload_name(args.config, c)} "
                          "takes >= 10 min on a host core (SURVEY 8d): no bounded sample"}),
              flush=True)
        return 0
    o = Oracle(kind)
    t0 = time.perf_counter()
    x = o.synth_baseline(c["kind"], c["dims"], c["rank"], c["rho"], TRUTH_SEED[args.config])
    gen = time.perf_counter() - t0
    # The same W warm-up + K timed sweeps as the device arm when that fits the
    # time budget (a 3-sweep probe measures the sweep time first); otherwise as
    # many timed sweeps as the budget allows after the W warm-up sweeps.
    W = max(1, args.warmup)
    probe = o.solve(x, c["rank"], 3, extrapolate=True, seed=INIT_SEED)
    pw = [t["wall_seconds"] for t in probe.trace]
    per = max((pw[-1] - pw[0]) / 2.0, 1e-9)
    budget = float(args.ref_budget_s)
    k = int(max(2, min(args.steps, budget / per - W)))
    r = o.solve(x, c["rank"], W + k, extrapolate=True, seed=INIT_SEED)
    w = [t["wall_seconds"] for t in r.trace]
    rate = k / (w[-1] - w[W - 1])
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": "sweeps/s",
        "n_gpus": args.gpus, "steps": k, "warmup": W, "ms_per_step": 1e3 / rate,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generator cpd::Rng, BASELINE construction; the device "
                "arm's counter-based generator draws other values of the same distribution: "
                "throughput-neutral)",
        "config": bench_config(args, c, max(world, args.gpus)),
        "cpu_baseline": {"value": rate, "unit": "sweeps/s", "cores": 1, "kind": kind,
                         "sample": f"{k} ALS-QR-BRE sweeps after {W} warm-up sweeps (the first "
                                   f"is the dim-tree sweep) on the same config; the reference "
                                   f"is single-threaded; time budget {budget:.0f}s"},
        "e2e": {"value": rate, "unit": "sweeps/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "notes": f"input generation {gen:.1f}s untimed",
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-baseline-sweeps", type=int, default=2)
    ap.add_argument("--ref-max-sweeps", type=int, default=8)  # (kept for old command lines)
    ap.add_argument("--ref-budget-s", type=float, default=150.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    c = CONFIGS[args.config]
    rank, world, local = init_dist()
    if args.impl == "reference":
        return run_reference(args, c, rank, world)

    import paper_2503_18759_b200 as cpd

    W, K = args.warmup, args.steps
    nccl_id = None
    if world > 1:
        import torch.distributed as dist
        obj = [cpd.Context.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    ctx = cpd.Context(local, rank=rank, world=world, nccl_id=nccl_id)
    dims = list(c["dims"])
    ctx.synth_tensor(c["kind"], dims, c["rank"], c["rho"], TRUTH_SEED[args.config])
    ctx.norm_sq()
    cfg = cpd.SolverConfig(rank=c["rank"], max_iterations=W + K, seed=INIT_SEED)

    # ---- device-timed K sweeps after W warm-up sweeps ---------------------------
    # (torch's CUDA state is set up here, outside the timed window: the
    # barriers below call torch.cuda.synchronize())
    import torch
    torch.cuda.set_device(local)
    torch.cuda.synchronize()
    clocks = ClockSampler(local).start()
    sess = ctx.session(cfg, extrapolate=True)
    warm = sess.run(W)
    p0 = ctx.profile()
    barrier(world)
    clocks.mark()
    rows = sess.run(K)
    clocks.stop()
    barrier(world)
    p1 = ctx.profile()
    model = sess.end()
    sess.close()
    dt = rows[-1].wall_seconds - warm[-1].wall_seconds
    dt = allmax(world, dt)
    value = K / dt
    d = {k: p1[k] - p0[k] for k in ("root_ttms", "root_ttm_ms", "root_ttm_flops",
                                     "root_ttm_bytes", "branch_ttm_ms", "mode_update_ms",
                                     "comm_ms", "kernel_launches")}
    # ---- the root TTM kernel alone (roofline): same config, overlap off ------
    # In the timed run the sweep's root TTM shares the GPU with the preceding
    # update (low-priority stream), so its launch-to-end time is not the
    # kernel's speed.  A short run with the overlap off times it alone.
    ctx.set_options(timing=True, overlap=False)
    iso_n = 20 if np.prod(dims) < (1 << 30) else 6  # C5: 6 sweeps of ~40 ms
    iso = ctx.session(cpd.SolverConfig(rank=c["rank"], max_iterations=W + iso_n, seed=INIT_SEED),
                      extrapolate=True)
    iso.run(W)
    q0 = ctx.profile()
    iso.run(iso_n)
    q1 = ctx.profile()
    iso.close()
    ctx.set_options(timing=True, overlap=True)
    iso_roots = max(q1["root_ttms"] - q0["root_ttms"], 1)
    iso_ms = (q1["root_ttm_ms"] - q0["root_ttm_ms"]) / iso_roots
    hbm, hbm_src, p64 = peaks()
    n_root = max(d["root_ttms"], 1)
    overlapped_ms = d["root_ttm_ms"] / n_root
    t_launch = iso_ms * 1e-3
    f_launch = d["root_ttm_flops"] / n_root
    b_launch = d["root_ttm_bytes"] / n_root
    ridge = p64 * 1e12 / (hbm * 1e9)
    if f_launch / b_launch >= ridge:
        roof = {"bound": "tensor", "achieved": f_launch / t_launch / 1e12, "peak": p64,
                "unit": "TFLOP/s", "peak_source": "profiles/fp64_peak.json (measured DMMA f64)"}
    else:
        roof = {"bound": "hbm", "achieved": b_launch / t_launch / 1e9, "peak": hbm,
                "unit": "GB/s", "peak_source": hbm_src}
    roof["frac"] = roof["achieved"] / roof["peak"]
    traffic = None
    tp = os.path.join(ROOT, "profiles", f"ncu_root_ttm_{args.config}.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    roof["traffic"] = traffic
    roof["kernel"] = "ttm_tma_kernel (root TTM X x_c Q_c^T, TMA-staged DMMA)"
    roof["algorithmic_flops_per_launch"] = f_launch
    roof["algorithmic_bytes_per_launch"] = b_launch
    roof["avg_launch_ms"] = t_launch * 1e3
    roof["timing"] = (f"kernel alone (overlap off, {iso_n} sweeps after the timed run, CUDA "
                      "events on its stream); in the timed run it overlaps the previous update")
    roof["overlapped_avg_launch_ms"] = overlapped_ms
    roof["share_of_step"] = d["root_ttm_ms"] / (dt * 1e3)
    roof["fp64_tflops"] = f_launch / t_launch / 1e12
    roof["hbm_gbs"] = b_launch / t_launch / 1e9
    roof["roofline_frac"] = (max(f_launch / (p64 * 1e12), b_launch / (hbm * 1e9))) / t_launch
    # the same launches inside the timed run (sharing the GPU with the update
    # the root overlaps): launch-to-end time on its stream
    roof["frac_in_timed_run"] = (max(f_launch / (p64 * 1e12), b_launch / (hbm * 1e9))
                                 / (overlapped_ms * 1e-3))

    # ---- e2e through the C ABI with host buffers ---------------------------------
    e2e = None
    x_host = None
    local_dims = [dims[0] // world] + dims[1:]
    need_cpu = (rank == 0 and world == 1 and not args.no_cpu_baseline
                and np.prod(dims) <= CPU_BASELINE_MAX_ELEMS)
    if not args.no_e2e or need_cpu:
        x_host = ctx.get_tensor(local_dims)
    if not args.no_e2e:
        try:
            import torch
            pinned = torch.empty(x_host.size, dtype=torch.float64, pin_memory=True).numpy()
            pinned[:] = x_host.ravel()
            xh = pinned.reshape(local_dims)
        except Exception:
            xh = x_host
        ctx2 = ctx
        if world > 1:
            # a second communicator needs its own NCCL unique id (an id
            # bootstraps exactly one communicator)
            import torch.distributed as dist
            obj = [cpd.Context.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            ctx2 = cpd.Context(local, rank=rank, world=world, nccl_id=obj[0])
        cfg2 = cpd.SolverConfig(rank=c["rank"], max_iterations=K, seed=INIT_SEED)
        # (untimed: the same upload once, synchronously, for the copy's own time)
        tc = time.perf_counter()
        ctx2.set_tensor(xh, dims)
        t_h2d = time.perf_counter() - tc
        barrier(world)
        t0 = time.perf_counter()
        # the job: queue the H2D from pinned memory (cpdb_tensor_set_async), set
        # the solver up under it (the first synchronisation inside waits for it)
        ctx2.set_tensor(xh, dims, wait=False)
        s2 = ctx2.session(cfg2, extrapolate=True)
        t_begin = time.perf_counter()
        r2 = s2.run(K)
        t_run = time.perf_counter()
        m2 = s2.end()
        t1 = time.perf_counter()
        s2.close()
        barrier(world)
        et = allmax(world, t1 - t0)
        h2d = xh.size * 8
        d2h = (sum(f.size for f in m2.factors) + m2.lam.size) * 8 + len(r2) * 128
        e2e = {"value": K / et, "unit": "sweeps/s", "h2d_bytes_per_step": h2d / K,
               "d2h_bytes_per_step": d2h / K, "h2d_ms": t_h2d * 1e3,
               "upload_and_begin_ms": (t_begin - t0) * 1e3,
               "sweeps_ms": (t_run - t_begin) * 1e3, "end_ms": (t1 - t_run) * 1e3,
               "h2d_gbs": h2d / t_h2d / 1e9,
               "rest_ms": (et - t_h2d) * 1e3,
               "note": "one job: H2D of X from pinned memory (queued, cpdb_tensor_set_async; "
                       "h2d_ms is the same copy timed alone before the job) with the solver "
                       "set-up under it + K sweeps + D2H of the model, bytes amortised over "
                       "the K sweeps"}

    # ---- CPU baseline: the reference itself, bounded sample ---------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        if np.prod(dims) > CPU_BASELINE_MAX_ELEMS:
            # one reference sweep of C5's 34 GB tensor takes >= 10 min on a
            # host core: no bounded sample of this workload exists
            cpu = {"value": None, "unit": "sweeps/s", "cores": 1, "kind": "reference",
                   "sample": "skipped: one single-threaded reference sweep of this tensor "
                             "takes >= 10 min (SURVEY 8d)"}
        else:
            rate, kind, n, wall = cpu_reference_rate(x_host, c, args.cpu_baseline_sweeps)
            cpu = {"value": rate, "unit": "sweeps/s", "cores": 1, "kind": kind,
                   "sample": f"{n} steady ALS-QR-BRE sweeps (after the untimed dim-tree sweep) "
                             f"on the same tensor, single-threaded reference, {wall:.1f}s wall"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "sweeps/s", "n_gpus": world,
            "steps": K, "warmup": W, "ms_per_step": dt / K * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (device generator, BASELINE construction)",
            "config": bench_config(args, c, world),
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clocks.summary(),
            "gpu_launches": int(d["kernel_launches"]),
            # device time per step summed by kernel class (CUDA events per
            # launch).  Classes run concurrently on several streams (the root
            # under the previous update, Z-QR beside the chain), so the sum
            # exceeds the wall time by the overlap: concurrency = sum / wall.
            # mode_update (Z-QR, V-GEMM, finisher) is 0 unless CPDB_TIME_TAILS=1
            # (its events cost ~5% of the sweep rate); profiles/ has its share.
            "kernel_ms_per_step": {
                "root_ttm": d["root_ttm_ms"] / K, "branch_ttm": d["branch_ttm_ms"] / K,
                "mode_update": d["mode_update_ms"] / K, "comm": d["comm_ms"] / K,
                "sum": (d["root_ttm_ms"] + d["branch_ttm_ms"] + d["mode_update_ms"]
                        + d["comm_ms"]) / K,
                "wall": dt / K * 1e3,
                "concurrency": (d["root_ttm_ms"] + d["branch_ttm_ms"] + d["mode_update_ms"]
                                + d["comm_ms"]) / (dt * 1e3)},
            "final_fitness": rows[-1].fitness,
        }
        print(json.dumps(line), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
