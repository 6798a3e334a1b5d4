#!/usr/bin/env python
"""Benchmark of the integrator hot path (BASELINE.json metric: time-to-epsrel and FP64 integrand
evaluations per second, beside the reference's CPU path).

    python bench.py --gpus N --steps K --warmup W [--workload config1..config4] [--impl reference]

A *step* is one complete run of the workload through the public API:
  config1  PAGANI  f4 d=5 rel_tol 1e-3            refine() to tolerance          (BASELINE configs[0])
  config2  m-Cubes f2 d=6 n=1e6/iteration 1e-3     run() to tolerance (<=15 its)  (configs[1]; default at N=1)
  config3  PAGANI  f1 d=8 rel_tol 1e-6             refine() to the region cap     (configs[2], one GPU)
  config4  m-Cubes f3 d=8 n=1e9/iteration 1e-6     run() to epsrel 1e-6 (~170 iterations of 8.6e8 samples), sub-cubes
           sharded over the ranks, NCCL all-gather/all-reduce per iteration (configs[3]; default at N>1)
  config4_fixed  the same pass, 4 iterations of fixed work (sampler throughput; round-1 figure)
With --gpus N > 1 and no torchrun environment the script re-executes itself under torch.distributed.run
with N ranks (one per GPU); it never prints n_gpus = N from fewer than N ranks.
Units are integrand evaluations: regions_processed * f_eval(d) for PAGANI, m*p per m-Cubes iteration.

`value` is evaluations/s over the CUDA-event time of the K steps (max over ranks); `e2e` is the same
count over the wall-clock of the public Python API calls, host buffers in and out.  `roofline` times
the dominant kernel with CUDA events on its launching stream over the same K steps run a second time
(event pairs between back-to-back kernels would perturb the steps `value` is timed on); the FP64 peak
is a DFMA micro-benchmark run live (MEASURED_PEAKS.json has no FP64 entry).  `cpu_baseline` and
`--impl reference` time the numpy restatement of the reference (oracle/) on the host cores.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

F_EVAL = {d: 2**d + 2 * d * d + 2 * d + 1 for d in range(1, 13)}
# formula flops per evaluation: PAGANI F + 2d + 10, m-Cubes F + 10d + 4
FORMULA_FLOPS = {"f1": lambda d: 2 * d, "f2": lambda d: 5 * d - 1, "f3": lambda d: 2 * d + 1, "f4": lambda d: 3 * d + 1,
                 "f5": lambda d: 2 * d + 1, "f6": lambda d: 2 * d, "sum": lambda d: d - 1}

WORKLOADS = {
    "config1": dict(kind="pagani", family="f4", d=5, rel_tol=1e-3,
                    label="config1: PAGANI f4 (Gaussian) d=5 rel_tol=1e-3, refine() to tolerance"),
    "config2": dict(kind="mcubes", family="f2", d=6, n=10**6, rel_tol=1e-3, max_iterations=15, seed=0,
                    label="config2: m-Cubes f2 (product peak) d=6 n=1e6/iteration epsrel=1e-3 seed=0, run() to tolerance"),
    "config3": dict(kind="pagani", family="f1", d=8, rel_tol=1e-6,
                    label="config3: PAGANI f1 (oscillatory) d=8 rel_tol=1e-6, refine() to the 2^26 region cap"),
    "config4": dict(kind="mcubes", family="f3", d=8, n=10**9, rel_tol=1e-6, max_iterations=600, seed=0,
                    label="config4: m-Cubes f3 (corner peak) d=8 n=1e9/iteration epsrel=1e-6 seed=0, run() to tolerance, sub-cubes sharded"),
    "config4_fixed": dict(kind="mcubes", family="f3", d=8, n=10**9, rel_tol=None, max_iterations=4, seed=0,
                          label="config4_fixed: m-Cubes f3 (corner peak) d=8 n=1e9/iteration, 4 iterations of fixed work"),
}


# dram__bytes_read.sum + dram__bytes_write.sum of the dominant kernel, from the committed `ncu --set full` capture of
# the same kernel at the same size (scripts/collect_profiles.sh writes profiles/<round>_ncu_*.txt)
TRAFFIC_PROFILE = {"config2": "ncu_vsample_config2.txt", "config4": "ncu_vsample_config4.txt",
                   "config4_fixed": "ncu_vsample_config4.txt",
                   "config3": "ncu_pagani_lanes_f1_d8.txt", "config1": "ncu_pagani_warp_f4_d5_small.txt"}
PROFILE_ROUNDS = ("r2", "r1")   # newest committed capture wins


def _profile_path(workload):
    name = TRAFFIC_PROFILE.get(workload)
    if not name:
        return None, None
    for rnd in PROFILE_ROUNDS:
        path = os.path.join(ROOT, "profiles", f"{rnd}_{name}")
        if os.path.exists(path):
            return path, f"profiles/{rnd}_{name}"
    return None, None


def dram_traffic_bytes(workload):
    """(bytes per launch, source file) of the dominant kernel, or (None, None) when no capture is committed."""
    path, shown = _profile_path(workload)
    if not path:
        return None, None
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    total, seen = 0.0, 0
    for line in open(path):
        line = line.strip()
        if line.startswith(("dram__bytes_read.sum", "dram__bytes_write.sum")):
            unit = line[line.index("[") + 1:line.index("]")]
            total += float(line.split("=")[1]) * scale.get(unit, 1.0)
            seen += 1
    return (total, shown) if seen == 2 else (None, None)


def ncu_pipe_figures(workload):
    """FP64-pipe and issue-slot utilisation (%) of the dominant kernel from the same committed capture, or {}."""
    path, _ = _profile_path(workload)
    out = {}
    if path:
        keys = {"sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_busy_pct",
                "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_slots_busy_pct"}
        for line in open(path):
            line = line.strip()
            for k, label in keys.items():
                if line.startswith(k):
                    out[label] = round(float(line.split("=")[1]), 1)
    return out


def flops_per_eval(w):
    d = w["d"]
    return FORMULA_FLOPS[w["family"]](d) + (2 * d + 10 if w["kind"] == "pagani" else 10 * d + 4)


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clock and throttle reasons through NVML while the timed region runs."""

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._thread = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001
            self._nv = None

    def _loop(self):
        nv = self._nv
        names = {"hw_slowdown": 0x8, "sw_power_cap": 0x4, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
                 "hw_power_brake": 0x80, "sync_boost": 0x10, "applications_clocks": 0x2}
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                try:
                    mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                except Exception:  # noqa: BLE001
                    mask = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
                for k, bit in names.items():
                    if mask & bit:
                        self.reasons.add(k)
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(0.02)

    def __enter__(self):
        if self._nv is not None:
            self._thread = threading.Thread(target=self._loop, daemon=True)
            self._thread.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._thread is not None:
            self._thread.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ----------------------------------------------------------------------------- CPU reference arm
def reference_rule(d):
    """The reference's own rule table for dimension d <= 8, from the fixtures oracle/make_golden.py wrote with the
    unmodified reference (tests/golden/rules.npz + golden.json).  The reference arm imports nothing of the product."""
    z = np.load(os.path.join(ROOT, "tests", "golden", "rules.npz"))
    with open(os.path.join(ROOT, "tests", "golden", "golden.json")) as fh:
        m = json.load(fh)["rules"][str(d)]
    return dict(generators=z[f"gen{d}"], weights=z[f"w{d}"], axial_indices=z[f"ax{d}"],
                split_weights=np.array([float.fromhex(v) for v in m["split"]]),
                null_degrees=tuple(m["null_degrees"]), null_scales=tuple(m["null_scales"]))


def oracle_step(w, workers):
    """One step of the workload on the host cores with the numpy restatement of the reference.
    Returns (evaluations, seconds, description)."""
    from oracle import parcube_oracle as po

    d = w["d"]
    rd = reference_rule(d) if w["kind"] == "pagani" else None   # input data, loaded outside the timed region
    t0 = time.perf_counter()
    if w["kind"] == "pagani":
        budget = None if w["family"] == "f4" else 20.0
        out = po.pagani_refine(w["family"], d, rd, rel_tol=w["rel_tol"], workers=workers, time_budget_s=budget)
        evals = out["regions_processed"] * F_EVAL[d]
        what = (f"refine() {'to completion' if budget is None or out['reason'] != 'oracle time budget' else 'cut at a 20 s budget'}: "
                f"{out['iterations']} iterations, {out['regions_processed']} regions")
    else:
        n = w["n"] if w["n"] <= 10**7 else 10**7   # bounded sample of the sampler on the CPU
        its = w["max_iterations"] if w["n"] <= 10**7 else 2
        out = po.mcubes_run(w["family"], n, d, its, seed=w["seed"], workers=workers, rel_tol=w["rel_tol"])
        done = len(out["iterations"])
        evals = done * out["plan"]["m"] * out["plan"]["p"]
        what = f"run() n={n:.0e}/iteration, {done} iterations" + ("" if n == w["n"] else f" (workload n={w['n']:.0e} is bounded to n=1e7 x 2 its on the CPU)")
    return evals, time.perf_counter() - t0, what


def run_reference_arm(args, w, rank):
    if rank != 0:
        return
    workers = os.cpu_count() or 1
    times, evals, what = [], 0, ""
    for i in range(args.warmup + args.steps):
        e, t, what = oracle_step(w, workers)
        if i >= args.warmup:
            times.append(t)
            evals += e
    total = sum(times)
    value = evals / total
    line = {"impl": "reference", "metric": "integrand_evals_per_s", "value": value, "unit": "evals/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / len(times), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (Genz integrand, counter-hash samples)",
            "config": {"workload": w["label"]},
            "cpu_baseline": {"value": value, "unit": "evals/s", "cores": workers, "kind": "port", "sample": what},
            "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "time_to_epsrel_s": total / len(times)}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- launch
def spawn_ranks(n):
    """Re-execute this script under torch.distributed.run with n ranks on this node; returns its exit status."""
    import socket
    import subprocess

    import torch

    have = torch.cuda.device_count()
    if have < n:
        print(json.dumps({"error": f"--gpus {n} requested, {have} CUDA device(s) visible; nothing measured"}), flush=True)
        return 2
    with socket.socket() as sock:
        sock.bind(("127.0.0.1", 0))
        port = sock.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


# ----------------------------------------------------------------------------- B200 arm
def b200_step(w, pb, comm=None):
    """One step through the public API. Returns (evaluations, device_seconds, info, h2d_bytes, d2h_bytes)."""
    from paper_2302_05730_b200 import _native, sharded

    d = w["d"]
    f = pb.get_integrand(w["family"], d)
    if w["kind"] == "pagani" and comm is not None and comm.world > 1:
        # region list sharded over the ranks, per-iteration rebalancing (sharded.py)
        t0 = time.perf_counter()
        res = sharded.pagani_refine_sharded(f, pb.PaganiConfig(rel_tol=w["rel_tol"]), comm)
        secs = time.perf_counter() - t0
        evals = int(res.regions_processed) * F_EVAL[d]
        info = dict(estimate=res.estimate, errorest=res.errorest, iterations=res.iterations,
                    regions_processed=int(res.regions_processed), reason=res.reason)
        return evals, secs, info, 312 + 352 + 40, 40 * (res.iterations + 1) + 56
    ctx = _native.context()
    if w["kind"] == "pagani":
        # the call a user makes: refine() of the reference's API (rule table built/cached by the package)
        res = pb.refine(f, pb.PaganiConfig(rel_tol=w["rel_tol"]))
        evals = int(res.regions_processed) * F_EVAL[d]
        info = dict(estimate=res.estimate, errorest=res.errorest, iterations=res.iterations,
                    regions_processed=int(res.regions_processed), reason=res.reason)
        # in: integrand + rule + config structs; out: one progress record per iteration + the result struct
        return evals, ctx.last_device_seconds, info, 312 + 352 + 40, 40 * len(res.history) + 56
    if comm is not None and comm.world > 1:
        # sub-cubes sharded over the ranks; device-resident loop, NCCL collectives on the library's buffers (sharded.py)
        res = sharded.mcubes_run_sharded(f, w["n"], d, w["max_iterations"], comm, seed=w["seed"], rel_tol=w["rel_tol"])
        secs = ctx.last_device_seconds     # CUDA events around this rank's whole run
    else:
        # the call a user makes: mcubes_run() of the reference's API (per-iteration contribution tables included)
        res = pb.mcubes_run(f, w["n"], d, w["max_iterations"], seed=w["seed"], rel_tol=w["rel_tol"])
        secs = ctx.last_device_seconds
    n_it = len(res.iterations)
    evals = n_it * res.plan.n_actual
    info = dict(estimate=res.estimate, errorest=res.errorest, chi2_per_dof=res.chi2_per_dof, iterations=n_it,
                samples_per_iteration=res.plan.n_actual,
                rel_error_reached=res.errorest / abs(res.estimate) if res.estimate else None)
    grid_bytes = d * 501 * 8
    return evals, secs, info, 312 + 40 + grid_bytes, n_it * (32 + d * 500 * 8) + grid_bytes


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=None)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="auto", choices=["auto", *WORKLOADS])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the secondary-workload measurements")
    args = ap.parse_args()

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl != "reference":
        # launched plainly with --gpus N: become N ranks, one per GPU (the launch the driver's torchrun line makes)
        sys.exit(spawn_ranks(args.gpus))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl != "reference" and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but the launch has {world} rank(s); refusing to report n_gpus={args.gpus}")
    name = args.workload if args.workload != "auto" else ("config2" if args.gpus == 1 else "config4")
    w = WORKLOADS[name]
    heavy = name in ("config3", "config4", "config4_fixed")
    if args.steps is None:
        args.steps = (2 if name == "config4" else 5) if heavy else 200
    if args.warmup is None:
        args.warmup = 3 if heavy else 20
    args.warmup = max(args.warmup, 3)

    if args.impl == "reference":
        if rank != 0:
            return                      # under torchrun the other ranks exit 0 without work
        if args.steps > 20:
            args.steps, args.warmup = 5, 1  # each CPU step takes seconds
        run_reference_arm(args, w, rank)
        return

    import torch

    import paper_2302_05730_b200 as pb
    from paper_2302_05730_b200 import _native, sharded

    comm = None
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        comm = sharded.Comm(device=local_rank)
    os.environ.setdefault("PARCUBE_B200_DEVICE", str(local_rank))
    ctx = _native.context(local_rank)
    dev_name, sms, _ = ctx.device_info()
    peak = ctx.measure_fp64_peak()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local_rank}")  # > 126 MB L2

    def sync_all():
        torch.cuda.synchronize()
        if comm is not None:
            comm.barrier()
            torch.cuda.synchronize()

    t0 = time.perf_counter()
    cold = b200_step(w, pb, comm)           # first call of the process: allocations, kernel attributes, module load
    cold_wall_s, cold_dev_s = time.perf_counter() - t0, cold[1]
    for _ in range(args.warmup - 1):
        b200_step(w, pb, comm)
    sync_all()
    launches0 = ctx.launch_count()
    dev_s = wall_s = 0.0
    evals = 0
    info = {}
    h2d = d2h = 0
    with ClockSampler(local_rank) as clocks:
        t_region = time.perf_counter()
        for _ in range(args.steps):
            flush.zero_()               # flush L2 between steps
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            e, s, info, h2d, d2h = b200_step(w, pb, comm)
            wall_s += time.perf_counter() - t0
            dev_s += s
            evals += e
        sync_all()
        region_s = time.perf_counter() - t_region
    launches = ctx.launch_count() - launches0
    # Roofline leg: the same K steps once more, now with a CUDA-event pair around every launch of the dominant
    # kernel on its launching stream.  The event records sit between back-to-back kernels (they end the
    # programmatic overlap of a launch with the tail of its predecessor), so they stay out of the steps that
    # `value` and `e2e` are timed on; this leg's own step time is reported next to the kernel time.
    kind = 0 if w["kind"] == "pagani" else 1
    ctx.profile_begin()
    span_dev_s = 0.0
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        span_dev_s += b200_step(w, pb, comm)[1]
    sync_all()
    k_ms, k_launches, k_units = ctx.profile_end(kind)

    # max over ranks of the timed durations (device seconds and API wall-clock)
    if comm is not None:
        agg = np.max(np.stack(comm.allgather(np.array([dev_s, wall_s, k_ms, span_dev_s]))), axis=0)
        dev_s, wall_s, k_ms, span_dev_s = (float(x) for x in agg)
        k_units *= 1  # per-rank units; the roofline below is per GPU
    fpe = flops_per_eval(w)
    traffic, traffic_src = dram_traffic_bytes(name)
    evals_per_unit = F_EVAL[w["d"]] if w["kind"] == "pagani" else 1
    achieved = (k_units * evals_per_unit * fpe) / (k_ms * 1e-3) / 1e12 if k_ms > 0 else 0.0

    line = {
        "metric": "integrand_evals_per_s", "value": evals / dev_s, "unit": "evals/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dev_s / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (Genz integrand; samples from the reference counter hash, generated in-kernel)",
        "config": {"workload": w["label"], "l2": "256 MiB buffer written between steps; the path has no HBM-resident input",
                   "device": dev_name, "sms": sms},
        "time_to_epsrel_s": dev_s / args.steps, "result": info,
        "cold_first_call": {"wall_ms": 1e3 * cold_wall_s, "device_ms": 1e3 * cold_dev_s,
                            "note": "first call of the process (buffer reservation, kernel attributes, module load); "
                                    "every later call reuses the context's reserved buffers"},
        "e2e": {"value": evals / wall_s, "unit": "evals/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": 1e3 * wall_s / args.steps,
                "api": "the package's public refine() / mcubes_run() (reference names and result types), host objects in, "
                       "host records + per-iteration tables out"},
        "gpu_launches": int(launches),
        "roofline": {"bound": "fp64",
                     "bound_note": "FP64 vector pipe (DFMA): the path is ~100 flop per HBM byte and is no dense contraction, "
                                   "so neither the HBM nor the tensor roofline binds it (BASELINE.json north_star)",
                     "kernel": ("pagani_eval_lanes_kernel / pagani_eval_mult_kernel (one region per lane / per warp)" if kind == 0
                                else "vsample_kernel"),
                     "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak if peak else None,
                     "traffic": traffic, "traffic_unit": "bytes of DRAM read+write per launch (ncu --set full capture)",
                     "traffic_source": traffic_src, "launches": int(k_launches), "avg_launch_ms": k_ms / max(k_launches, 1),
                     "flops_per_eval": fpe, "evals_per_launch": k_units * evals_per_unit / max(k_launches, 1),
                     "kernel_share_of_step": k_ms * 1e-3 / span_dev_s if span_dev_s else None,
                     "timed_on": "a second leg of the same K steps with a CUDA-event pair around every launch of this kernel",
                     "ms_per_step_with_event_pairs": 1e3 * span_dev_s / args.steps,
                     "peak_source": "DFMA micro-benchmark run live (MEASURED_PEAKS.json has no FP64 entry; nominal 37 TFLOP/s)",
                     # `achieved` counts FORMULA flops (exp/cos/div = 1, the integer hash = 0); what the pipes
                     # executed for them is in the committed ncu capture of the same kernel
                     "ncu": ncu_pipe_figures(name)},
        "clocks": clocks.summary(),
        "timed_region_s": region_s,
    }

    if rank == 0 and not args.no_extras and world == 1:
        extras = {}
        for other in ("config1", "config3", "config4_fixed", "config4"):
            if other == name:
                continue
            ww = WORKLOADS[other]
            t0 = time.perf_counter()
            first = b200_step(ww, pb)
            cold_ms = 1e3 * (time.perf_counter() - t0)
            reps = {"config1": 50, "config4": 1}.get(other, 3)
            t0 = time.perf_counter()
            tot_e = tot_s = 0
            for _ in range(reps):
                e, s, inf, _, _ = b200_step(ww, pb)
                tot_e += e
                tot_s += s
            wall = time.perf_counter() - t0
            # the event pairs around the dominant kernel in a leg of their own, as for the main workload
            # (config4 to tolerance: the leg above is the first call's; one more 6-second run buys nothing)
            if other == "config4":
                ms = nl = units = 0
            else:
                ctx.profile_begin()
                for _ in range(reps):
                    b200_step(ww, pb)
                kk = 0 if ww["kind"] == "pagani" else 1
                ms, nl, units = ctx.profile_end(kk)
            epu = F_EVAL[ww["d"]] if ww["kind"] == "pagani" else 1
            ach = units * epu * flops_per_eval(ww) / (ms * 1e-3) / 1e12 if ms else None
            extras[other] = {"workload": ww["label"], "evals_per_s": tot_e / tot_s, "time_to_epsrel_s": tot_s / reps,
                             "e2e_evals_per_s": tot_e / wall, "e2e_ms": 1e3 * wall / reps, "first_call_wall_ms": cold_ms,
                             "roofline_achieved_tflops": ach, "roofline_frac": ach / peak if ach else None,
                             "result": inf}
        line["other_workloads"] = extras

    if rank == 0 and not args.no_cpu_baseline:
        e, t, what = oracle_step(w, os.cpu_count() or 1)
        line["cpu_baseline"] = {"value": e / t, "unit": "evals/s", "cores": os.cpu_count() or 1, "kind": "port",
                                "sample": what, "seconds": t}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if comm is not None:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
