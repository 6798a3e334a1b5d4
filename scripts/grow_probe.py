import os, sys, time
sys.path.insert(0, os.getcwd())
import paper_2302_05730_b200 as pb
from paper_2302_05730_b200 import _native
ctx = _native.context(0)
f = pb.get_integrand("f1", 5)
for tol in (1e-5, 1e-8, 1e-8):
    t0 = time.perf_counter()
    r = pb.refine(f, pb.PaganiConfig(rel_tol=tol))
    print(f"tol {tol:.0e} wall {1e3*(time.perf_counter()-t0):.2f} ms device {1e3*ctx.last_device_seconds:.2f} ms regions {r.regions_processed}", flush=True)
