"""Small fixed workloads for ncu: `python scripts/profile_target.py eval|vsample|run [family d size]`."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2302_05730_b200 as pb

mode = sys.argv[1]
fam = sys.argv[2] if len(sys.argv) > 2 else ("f1" if mode == "eval" else "f3")
d = int(sys.argv[3]) if len(sys.argv) > 3 else 8
if mode == "eval":
    g = int(sys.argv[4]) if len(sys.argv) > 4 else 4
    rl = pb.uniform_split(d, g)
    rule = pb.build_rule(d)
    for _ in range(3):
        est = pb.pagani_kernel(pb.get_integrand(fam, d), rl, rule)
    print("regions", rl.n, "sum", pb.tree_sum(est.integrals))
elif mode == "run":  # the adaptive run: reduce_kernel and finish_kernel as config 2 launches them (d refinement CTAs)
    n = int(float(sys.argv[4])) if len(sys.argv) > 4 else 10**6
    for _ in range(2):
        r = pb.mcubes_run(pb.get_integrand(fam, d), n, d, 15, seed=0, rel_tol=1e-3)
    print("iterations", len(r.iterations), r.estimate, r.errorest)
else:
    n = int(float(sys.argv[4])) if len(sys.argv) > 4 else 10**8
    plan = pb.make_plan(n, d)
    grid = pb.init_grid(d)
    for _ in range(3):
        r = pb.mcubes_kernel(pb.get_integrand(fam, d), plan, grid, seed=1)
    print("samples", plan.n_actual, r.integral, r.variance)
