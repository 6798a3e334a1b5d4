#!/usr/bin/env python
"""Benchmark of the integrator hot path (BASELINE.json metric: time-to-epsrel and FP64 integrand
evaluations per second, beside the reference's CPU path).

    python bench.py --gpus N --steps K --warmup W [--workload config1..config4] [--impl reference]

A *step* is one complete run of the workload through the public API:
  config1  PAGANI  f4 d=5 rel_tol 1e-3            refine() to tolerance          (BASELINE configs[0])
  config2  m-Cubes f2 d=6 n=1e6/iteration 1e-3     run() to tolerance (<=15 its)  (configs[1]; default at N=1)
  config3  PAGANI  f1 d=8 rel_tol 1e-6             refine() to the region cap     (configs[2], one GPU)
  config4  m-Cubes f3 d=8 n=1e9/iteration          4 iterations, sub-cubes sharded over the ranks with
           NCCL all-gather/all-reduce (configs[3]; default at N>1; 1e-6 itself needs ~1e11 samples)
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
    "config4": dict(kind="mcubes", family="f3", d=8, n=10**9, rel_tol=None, max_iterations=4, seed=0,
                    label="config4: m-Cubes f3 (corner peak) d=8 n=1e9/iteration, 4 iterations, sub-cubes sharded"),
}


# dram__bytes_read.sum + dram__bytes_write.sum of the dominant kernel, from the committed `ncu --set full` capture of
# the same kernel at the same size (scripts/collect_profiles.sh writes profiles/<round>_ncu_*.txt)
TRAFFIC_PROFILE = {"config2": "r1_ncu_vsample_config2.txt", "config4": "r1_ncu_vsample_config4.txt",
                   "config3": "r1_ncu_pagani_lanes_f1_d8.txt", "config1": "r1_ncu_pagani_warp_f4_d5_small.txt"}


def dram_traffic_bytes(workload):
    """(bytes per launch, source file) of the dominant kernel, or (None, None) when no capture is committed."""
    name = TRAFFIC_PROFILE.get(workload)
    path = os.path.join(ROOT, "profiles", name) if name else None
    if not path or not os.path.exists(path):
        return None, None
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    total, seen = 0.0, 0
    for line in open(path):
        line = line.strip()
        if line.startswith(("dram__bytes_read.sum", "dram__bytes_write.sum")):
            unit = line[line.index("[") + 1:line.index("]")]
            total += float(line.split("=")[1]) * scale.get(unit, 1.0)
            seen += 1
    return (total, "profiles/" + name) if seen == 2 else (None, None)


def ncu_pipe_figures(workload):
    """FP64-pipe and issue-slot utilisation (%) of the dominant kernel from the same committed capture, or {}."""
    name = TRAFFIC_PROFILE.get(workload)
    path = os.path.join(ROOT, "profiles", name) if name else None
    out = {}
    if path and os.path.exists(path):
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
def oracle_step(w, workers):
    """One step of the workload on the host cores with the numpy restatement of the reference.
    Returns (evaluations, seconds, description)."""
    from oracle import parcube_oracle as po
    import paper_2302_05730_b200 as pb  # rule tables only (host numpy); no device call

    d = w["d"]
    t0 = time.perf_counter()
    if w["kind"] == "pagani":
        rule = pb.build_rule(d)
        rd = dict(generators=rule.generators, weights=rule.weights, axial_indices=rule.axial_indices,
                  split_weights=rule.split_weights, null_degrees=rule.null_degrees, null_scales=rule.null_scales)
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
    if w["kind"] == "pagani":
        cfg = pb.PaganiConfig(rel_tol=w["rel_tol"])
        res, history = _native.pagani_refine(f.device_spec(), pb.rules.orbit_form(pb.build_rule(d)), cfg)
        evals = int(res.regions_processed) * F_EVAL[d]
        info = dict(estimate=res.estimate, errorest=res.errorest, iterations=res.iterations,
                    regions_processed=int(res.regions_processed), reason=_native.STOP_REASONS[res.reason])
        # in: integrand + rule + config structs; out: one progress record per iteration + the result struct
        return evals, res.seconds_device, info, 312 + 352 + 40, 40 * res.n_records + 56
    if comm is not None and comm.world > 1:
        t0 = time.perf_counter()
        res = sharded.mcubes_run_sharded(f, w["n"], d, w["max_iterations"], comm, seed=w["seed"], rel_tol=w["rel_tol"])
        secs = time.perf_counter() - t0
    else:
        plan = pb.make_plan(w["n"], d)
        its, contribs, _b, secs = _native.mcubes_run(f.device_spec(), plan, 500, w["max_iterations"], w["seed"],
                                                     _native.RNG_REFERENCE_HASH, True, 1.5, True,
                                                     0.0 if w["rel_tol"] is None else w["rel_tol"])
        hist = [pb.stratified.McubesIterationResult(r.integral, r.variance, None, r.n_samples, r.clamp_events) for r in its]
        est, err, chi2 = pb.combine_iterations(hist)
        res = pb.MonteCarloResult(est, err, chi2, hist, plan)
    n_it = len(res.iterations)
    evals = n_it * res.plan.n_actual
    info = dict(estimate=res.estimate, errorest=res.errorest, iterations=n_it, samples_per_iteration=res.plan.n_actual)
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

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    name = args.workload if args.workload != "auto" else ("config2" if args.gpus == 1 else "config4")
    w = WORKLOADS[name]
    heavy = name in ("config3", "config4")
    if args.steps is None:
        args.steps = 5 if heavy else 200
    if args.warmup is None:
        args.warmup = 3 if heavy else 20
    args.warmup = max(args.warmup, 3)

    if args.impl == "reference":
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

    for _ in range(args.warmup):
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
        "e2e": {"value": evals / wall_s, "unit": "evals/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": 1e3 * wall_s / args.steps, "api": "refine()/mcubes_run() C-ABI call, host structs in, host records out"},
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
        for other in ("config1", "config3", "config4"):
            if other == name:
                continue
            ww = WORKLOADS[other]
            b200_step(ww, pb)
            reps = 3 if other != "config1" else 50
            t0 = time.perf_counter()
            tot_e = tot_s = 0
            for _ in range(reps):
                e, s, inf, _, _ = b200_step(ww, pb)
                tot_e += e
                tot_s += s
            wall = time.perf_counter() - t0
            # the event pairs around the dominant kernel in a leg of their own, as for the main workload
            ctx.profile_begin()
            for _ in range(reps):
                b200_step(ww, pb)
            kk = 0 if ww["kind"] == "pagani" else 1
            ms, nl, units = ctx.profile_end(kk)
            epu = F_EVAL[ww["d"]] if ww["kind"] == "pagani" else 1
            ach = units * epu * flops_per_eval(ww) / (ms * 1e-3) / 1e12
            extras[other] = {"workload": ww["label"], "evals_per_s": tot_e / tot_s, "time_to_epsrel_s": tot_s / reps,
                             "e2e_evals_per_s": tot_e / wall, "roofline_achieved_tflops": ach, "roofline_frac": ach / peak,
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
