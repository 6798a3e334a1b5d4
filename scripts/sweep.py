"""BASELINE config 5: PAGANI vs m-Cubes over the six Genz families, d = 5..8, epsrel 1e-3..1e-8.

Writes a JSON list and a markdown table (time-to-epsrel on the device, evaluations, outcome).
PAGANI runs `refine` to the tolerance / iteration budget / region cap exactly like the reference;
m-Cubes runs `mcubes_run(n=1e8 per iteration, rel_tol=eps, <= 20 iterations)`.
    python scripts/sweep.py [--quick] --out profiles/r1_sweep_config5
"""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2302_05730_b200 as pb
from paper_2302_05730_b200 import _native

ap = argparse.ArgumentParser()
ap.add_argument("--quick", action="store_true")
ap.add_argument("--out", default="gpurun_out/sweep")
ap.add_argument("--reserve-gib", type=float, default=0.0)
args = ap.parse_args()
fams = ["f1", "f2", "f3", "f4", "f5", "f6"]
dims = [5, 6, 7, 8]
tols = [1e-3, 1e-6] if args.quick else [1e-3, 1e-4, 1e-5, 1e-6, 1e-7, 1e-8]
F = {d: 2**d + 2 * d * d + 2 * d + 1 for d in dims}
rows = []
ctx = _native.context(0)
# one reservation for the whole sweep (pcb_ctx_reserve: physical chunks created once, buffers then grow by mapping
# them): without it the first run that reaches ~6e7 regions pays 100-200 ms for creating its memory inside its clock
t0 = time.perf_counter()
reserved = ctx.reserve(int(args.reserve_gib * 2**30)) if args.reserve_gib > 0 else 0
print(f"reserved {reserved / 2**30:.1f} GiB in {time.perf_counter() - t0:.2f} s", flush=True)
for fam in fams:
    for d in dims:
        f = pb.get_integrand(fam, d)
        truth = pb.reference_value(fam, d).value
        # warm-up: the first launch of a kernel pays CUDA's lazy module loading (tens of ms for the large evaluate
        # kernels); it is not part of a time-to-epsrel
        spec, orbit = f.device_spec(), pb.rules.orbit_form(pb.build_rule(d))
        # (a run to a 40000-region cap walks the short-list kernel, the general path and the lane kernel once)
        _native.pagani_refine(spec, orbit, pb.PaganiConfig(rel_tol=1e-13, region_cap=40000))
        _native.mcubes_run(spec, pb.make_plan(10**8, d), 500, 1, 0, _native.RNG_REFERENCE_HASH, True, 1.5, True, 0.0,
                           keep_contributions=False)
        for tol in tols:
            spec, orbit = f.device_spec(), pb.rules.orbit_form(pb.build_rule(d))
            res, hist = _native.pagani_refine(spec, orbit, pb.PaganiConfig(rel_tol=tol))
            rows.append(dict(integrator="pagani", family=fam, d=d, rel_tol=tol, seconds=res.seconds_device,
                             evals=int(res.regions_processed) * F[d], estimate=res.estimate, errorest=res.errorest,
                             true_rel_err=abs(res.estimate - truth) / abs(truth), converged=bool(res.converged),
                             outcome=_native.STOP_REASONS[res.reason], iterations=res.iterations,
                             regions=int(res.regions_processed)))
            plan = pb.make_plan(10**8, d)
            its, _, _, secs = _native.mcubes_run(spec, plan, 500, 20, 0, _native.RNG_REFERENCE_HASH, True, 1.5, True, tol,
                                                 keep_contributions=False)
            hist = [pb.stratified.McubesIterationResult(r.integral, r.variance, None, r.n_samples, r.clamp_events) for r in its]
            est, err, chi2 = pb.combine_iterations(hist)
            ok = err <= tol * abs(est)
            rows.append(dict(integrator="mcubes", family=fam, d=d, rel_tol=tol, seconds=secs, evals=len(its) * plan.n_actual,
                             estimate=est, errorest=err, true_rel_err=abs(est - truth) / abs(truth), converged=bool(ok),
                             outcome="tolerance met" if ok else "20 iterations", iterations=len(its), chi2_per_dof=chi2))
            print(rows[-2]["integrator"], fam, d, tol, f"{rows[-2]['seconds']:.4f}s", rows[-2]["outcome"], "|",
                  "mcubes", f"{secs:.4f}s", rows[-1]["outcome"], flush=True)
os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
json.dump(rows, open(args.out + ".json", "w"), indent=1)
with open(args.out + ".md", "w") as fh:
    fh.write("# Config 5 sweep on one B200 (device seconds; PAGANI refine vs m-Cubes n=1e8/iteration, <=20 iterations)\n\n")
    fh.write("| family | d | rel_tol | PAGANI s | PAGANI outcome | regions | true rel err | m-Cubes s | m-Cubes outcome | its | true rel err |\n|---|---|---|---|---|---|---|---|---|---|---|\n")
    for i in range(0, len(rows), 2):
        a, b = rows[i], rows[i + 1]
        fh.write(f"| {a['family']} | {a['d']} | {a['rel_tol']:.0e} | {a['seconds']:.4f} | {a['outcome']} | {a['regions']} | {a['true_rel_err']:.1e} | "
                 f"{b['seconds']:.4f} | {b['outcome']} | {b['iterations']} | {b['true_rel_err']:.1e} |\n")
print("wrote", args.out)
