"""First-contact probe on the GPU box: prints parity numbers instead of asserting."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2302_05730_b200 as pb
from paper_2302_05730_b200 import _native
from oracle import parcube_oracle as po

ctx = _native.context(0)
print("device", ctx.device_info(), "fp64 peak TF", ctx.measure_fp64_peak())

def rule_dict(r):
    return dict(generators=r.generators, weights=r.weights, axial_indices=r.axial_indices, split_weights=r.split_weights,
                null_degrees=r.null_degrees, null_scales=r.null_scales)

# functors
rng = np.random.default_rng(1)
for fam in ["f1","f2","f3","f4","f5","f6","sum"]:
    for d in (1, 5, 8, 12):
        pts = rng.random((1000, d))
        got = pb.get_integrand(fam, d).eval_many(pts)
        want = po.genz_eval(fam, d, pts)
        rel = np.max(np.abs(got-want)/np.maximum(np.abs(want),1e-300))
        print("functor", fam, d, "max rel", rel, "exact", np.array_equal(got, want))

# rng
s = np.arange(1000, dtype=np.uint64); c = (np.arange(1000, dtype=np.uint64)*7919)
print("rng exact", np.array_equal(_native.uniforms(12345, s, c), po.uniform(12345, s, c)))

# pagani evaluate
for fam, d, g in [("f4",5,4),("f2",5,4),("sum",5,4),("f1",8,2),("f2",8,2),("f3",6,3),("f6",3,5),("f5",7,2),("sum",1,16),("f2",2,9), ("f4",12,1)]:
    rule = pb.build_rule(d)
    rl = pb.uniform_split(d, g)
    t0=time.perf_counter(); est = pb.pagani_kernel(pb.get_integrand(fam,d), rl, rule); t1=time.perf_counter()
    i,e,k = po.pagani_evaluate(fam, rl.lefts, rl.lengths, rule_dict(rule))
    sc = np.max(np.abs(i))
    print("eval", fam, d, g, "I exact", np.array_equal(est.integrals,i), "maxdev/scale", np.max(np.abs(est.integrals-i))/sc,
          "E exact", np.array_equal(est.errors,e), "E maxrel", np.max(np.abs(est.errors-e)/np.maximum(e,1e-300*1)), "K eq", np.array_equal(est.split_axes,k), f"{(t1-t0)*1e3:.1f} ms")

# refine
for fam, d, tol, kw in [("f4",5,1e-3,{}),("f2",5,1e-3,{}),("f5",5,1e-3,{}),("f3",6,1e-3,{}),("f1",8,1e-6,dict(region_cap=1<<19))]:
    t0=time.perf_counter(); res = pb.refine(pb.get_integrand(fam,d), pb.PaganiConfig(rel_tol=tol, **kw)); t1=time.perf_counter()
    print("refine", fam, d, res.estimate, res.errorest, res.iterations, res.regions_processed, res.reason, f"{(t1-t0)*1e3:.1f} ms")
    print("   leaves", [h[2] for h in res.history])

# mcubes
for fam, d, n in [("f2",6,10**6),("f3",8,10**6),("sum",5,10**5),("f4",5,10**5)]:
    plan = pb.make_plan(n,d); grid = pb.init_grid(d)
    t0=time.perf_counter(); r = pb.mcubes_kernel(pb.get_integrand(fam,d), plan, grid, seed=0); t1=time.perf_counter()
    o = po.vsample(fam, po.make_plan(n,d), grid.boundaries, seed=0, workers=8)
    print("vsample", fam, d, n, "I", r.integral, o["integral"], "rel", abs(r.integral-o["integral"])/abs(o["integral"]),
          "Var rel", abs(r.variance-o["variance"])/o["variance"], "C maxrel", np.max(np.abs(r.contributions.c-o["contributions"]))/np.max(o["contributions"]),
          "clamps", r.clamp_events, o["clamp_events"], f"{(t1-t0)*1e3:.1f} ms")
    nb = pb.refine_grid(grid, r.contributions).boundaries
    ob = po.refine_grid(grid.boundaries, o["contributions"])
    print("   refine_grid max abs dev", np.max(np.abs(nb-ob)))
for fam,d,n,its in [("f2",6,10**6,6),("f3",8,10**6,5)]:
    t0=time.perf_counter(); r = pb.mcubes_run(pb.get_integrand(fam,d), n, d, its, seed=0); t1=time.perf_counter()
    o = po.mcubes_run(fam, n, d, its, seed=0, workers=8)
    print("run", fam, d, r.estimate, o["estimate"], r.errorest, o["errorest"], f"{(t1-t0)*1e3:.1f} ms")
for n in (10**8, 10**9):
    t0=time.perf_counter(); r = pb.mcubes_run(pb.get_integrand("f3",8), n, 8, 2, seed=0); t1=time.perf_counter()
    print("big run f3 d8", n, r.estimate, r.errorest, f"{(t1-t0)*1e3:.1f} ms for 2 its", r.plan.n_actual*2/(t1-t0)/1e9, "Gsamples/s")
t0=time.perf_counter(); res = pb.refine(pb.get_integrand("f1",8), pb.PaganiConfig(rel_tol=1e-6)); t1=time.perf_counter()
print("config3", res.estimate, res.errorest, res.iterations, res.regions_processed, res.reason, f"{(t1-t0):.2f} s", res.regions_processed*401/(t1-t0)/1e9, "Gevals/s")
