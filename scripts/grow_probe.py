"""Debug: where does the first f1 d=5 run to 1e-6 of a process spend its time?  (PCB_DEBUG_MEM=1 prints buffer growth)"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2302_05730_b200 as pb
from paper_2302_05730_b200 import _native
ctx = _native.context(0)
if len(sys.argv) > 1:
    print("reserved", ctx.reserve(int(float(sys.argv[1]) * 2**30)))
f = pb.get_integrand("f1", 5)
spec, orbit = f.device_spec(), pb.rules.orbit_form(pb.build_rule(5))
def run(tol):
    t0 = time.perf_counter()
    res, hist = _native.pagani_refine(spec, orbit, pb.PaganiConfig(rel_tol=tol))
    print(f"tol {tol:.0e} wall {1e3*(time.perf_counter()-t0):.2f} ms device {1e3*res.seconds_device:.3f} ms regions {int(res.regions_processed)} its {res.iterations}", flush=True)
run(1e-5)
_native.mcubes_run(spec, pb.make_plan(10**8, 5), 500, 1, 0, _native.RNG_REFERENCE_HASH, True, 1.5, True, 0.0, keep_contributions=False)
for tol in (1e-3, 1e-4, 1e-5, 1e-6, 1e-6, 1e-7, 1e-7, 1e-8, 1e-8):
    run(tol)
