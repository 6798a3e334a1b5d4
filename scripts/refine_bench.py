"""Time-to-tolerance of mid-size PAGANI refinements (the config-5 cases whose lists stay between 1e4 and 5e6 regions):
`python scripts/refine_bench.py [reps]` prints device ms per run (best of reps), iterations and regions."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2302_05730_b200 as pb
from paper_2302_05730_b200 import _native

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
cases = [("f4", 5, 1e-4), ("f4", 5, 1e-5), ("f4", 5, 1e-6), ("f4", 5, 1e-7), ("f5", 5, 1e-5), ("f5", 5, 1e-7), ("f3", 5, 1e-7),
         ("f3", 5, 1e-8), ("f2", 5, 1e-3), ("f2", 5, 1e-4), ("f3", 6, 1e-3), ("f3", 7, 1e-3), ("f1", 5, 1e-7), ("f1", 6, 1e-3)]
total = 0.0
for fam, d, tol in cases:
    f = pb.get_integrand(fam, d)
    spec, orbit = f.device_spec(), pb.rules.orbit_form(pb.build_rule(d))
    best = None
    for _ in range(reps + 1):
        res, hist = _native.pagani_refine(spec, orbit, pb.PaganiConfig(rel_tol=tol))
        best = res.seconds_device if best is None else min(best, res.seconds_device)
    total += best
    print(f"{fam} d={d} tol={tol:.0e}: {best * 1e3:8.3f} ms  {res.iterations:3d} iterations  {int(res.regions_processed):9d} regions  "
          f"{best * 1e6 / max(res.iterations, 1):7.1f} us/iteration")
print(f"total {total * 1e3:.3f} ms")
