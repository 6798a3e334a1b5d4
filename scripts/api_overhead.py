"""Host-side cost of the public mcubes_run()/refine() wrappers around the C-ABI call (debug)."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2302_05730_b200 as pb
from paper_2302_05730_b200 import _native
ctx = _native.context(0)
f = pb.get_integrand("f2", 6)
for _ in range(20):
    pb.mcubes_run(f, 10**6, 6, 15, seed=0, rel_tol=1e-3)
n = 300
t0 = time.perf_counter()
for _ in range(n):
    pb.mcubes_run(f, 10**6, 6, 15, seed=0, rel_tol=1e-3)
print("public mcubes_run: %.1f us per call, device %.1f us" % (1e6 * (time.perf_counter() - t0) / n, 1e6 * ctx.last_device_seconds))
plan = pb.make_plan(10**6, 6)
spec = f.device_spec()
t0 = time.perf_counter()
for _ in range(n):
    _native.mcubes_run(spec, plan, 500, 15, 0, _native.RNG_REFERENCE_HASH, True, 1.5, True, 1e-3)
print("_native.mcubes_run: %.1f us per call" % (1e6 * (time.perf_counter() - t0) / n))
pr = cProfile.Profile()
pr.enable()
for _ in range(n):
    pb.mcubes_run(f, 10**6, 6, 15, seed=0, rel_tol=1e-3)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
