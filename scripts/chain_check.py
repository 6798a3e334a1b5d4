"""A/B check of the device-resident short-list chain (PCB_PAGANI_SPECULATE=1/0): stop reasons, schedule widths, callbacks;
prints whether every result, history included, is identical.  python scripts/chain_check.py"""
import os, sys, subprocess, json
sys.path.insert(0, os.getcwd())
if len(sys.argv) > 1:
    import numpy as np
    import paper_2302_05730_b200 as pb
    out = []
    for fam, d, kw in [("f4", 5, dict(rel_tol=1e-3)), ("f4", 5, dict(rel_tol=1e-3, group_size=96)), ("f4", 5, dict(rel_tol=1e-3, group_size=32)),
                       ("f4", 5, dict(rel_tol=1e-6, max_iterations=4)), ("f4", 5, dict(rel_tol=1e-9, region_cap=3000)),
                       ("f2", 3, dict(rel_tol=1e-4, initial_regions=8)), ("f5", 4, dict(rel_tol=1e-5, initial_regions=16)),
                       ("f1", 2, dict(rel_tol=1e-10, max_iterations=30, initial_regions=4)), ("f3", 6, dict(rel_tol=1e-2, err_mode="magnitude" if False else "two-level"))]:
        r = pb.refine(pb.get_integrand(fam, d), pb.PaganiConfig(**kw))
        out.append([fam, d, r.estimate, r.errorest, r.iterations, int(r.regions_processed), r.reason, [list(h) for h in r.history]])
    # abort from the progress callback in the middle of a chain
    seen = []
    def cb(rec):
        seen.append(rec.iteration)
        if rec.iteration == 3: raise KeyboardInterrupt
    try:
        pb.refine(pb.get_integrand("f4", 5), pb.PaganiConfig(rel_tol=1e-6), progress=cb)
        out.append("no abort")
    except BaseException as e:
        out.append(["abort", type(e).__name__, seen])
    r = pb.refine(pb.get_integrand("f4", 5), pb.PaganiConfig(rel_tol=1e-3))      # the context is usable afterwards
    out.append([r.estimate, r.iterations])
    # non-finite inside a chain
    f = pb.get_integrand("f2", 3); f.a2 = 0.0
    try:
        pb.refine(f, pb.PaganiConfig(rel_tol=1e-3, initial_regions=8))
        out.append("no error")
    except pb.GroupTaskError as e:
        out.append(["nonfinite", int(e.cause.region_index), list(map(float, e.cause.point))])
    print(json.dumps(out))
else:
    res = {}
    for spec in ("1", "0"):
        env = dict(os.environ, PCB_PAGANI_SPECULATE=spec)
        p = subprocess.run([sys.executable, __file__, "child"], capture_output=True, text=True, env=env)
        if p.returncode != 0: print(p.stderr[-2000:])
        res[spec] = json.loads(p.stdout.strip().splitlines()[-1])
    same = res["1"] == res["0"]
    print("speculative chain == one-at-a-time:", same)
    if not same:
        for a, b in zip(res["1"], res["0"]):
            if a != b: print("DIFF", str(a)[:300], "|", str(b)[:300])
    for x in res["1"]: print(str(x)[:160])
