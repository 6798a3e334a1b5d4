"""Cold-call cost of refine(): first call of a process, calls that outgrow the pool, and warm calls.
    python scripts/cold_call.py [--reserve GB]
"""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2302_05730_b200 as pb
from paper_2302_05730_b200 import _native

ap = argparse.ArgumentParser()
ap.add_argument("--reserve", type=float, default=0.0)
args = ap.parse_args()
t0 = time.perf_counter()
ctx = _native.context(0)
print(f"context              {1e3 * (time.perf_counter() - t0):9.2f} ms")
if args.reserve:
    t0 = time.perf_counter()
    got = ctx.reserve(int(args.reserve * 2**30))
    print(f"reserve {args.reserve:.1f} GiB      {1e3 * (time.perf_counter() - t0):9.2f} ms -> pool {got / 2**30:.2f} GiB")


def timed(label, fn):
    t0 = time.perf_counter()
    res = fn()
    wall = 1e3 * (time.perf_counter() - t0)
    print(f"{label:34s} wall {wall:9.2f} ms  device {1e3 * ctx.last_device_seconds:9.2f} ms  regions {res.regions_processed}")


f4, f1 = pb.get_integrand("f4", 5), pb.get_integrand("f1", 8)
timed("config1 first call", lambda: pb.refine(f4, pb.PaganiConfig(rel_tol=1e-3)))
timed("config1 warm", lambda: pb.refine(f4, pb.PaganiConfig(rel_tol=1e-3)))
timed("f1 d=8 cap 2^20 first (module load)", lambda: pb.refine(f1, pb.PaganiConfig(rel_tol=1e-6, region_cap=1 << 20)))
timed("f1 d=8 cap 2^20 warm", lambda: pb.refine(f1, pb.PaganiConfig(rel_tol=1e-6, region_cap=1 << 20)))
timed("f1 d=8 cap 2^23 (pool grows)", lambda: pb.refine(f1, pb.PaganiConfig(rel_tol=1e-6, region_cap=1 << 23)))
timed("f1 d=8 cap 2^23 warm", lambda: pb.refine(f1, pb.PaganiConfig(rel_tol=1e-6, region_cap=1 << 23)))
timed("config3 (pool grows)", lambda: pb.refine(f1, pb.PaganiConfig(rel_tol=1e-6)))
timed("config3 warm", lambda: pb.refine(f1, pb.PaganiConfig(rel_tol=1e-6)))
f6 = pb.get_integrand("f1", 6)
for tol in (1e-3, 1e-4, 1e-5, 1e-6):
    timed(f"f1 d=6 rel_tol {tol:.0e}", lambda: pb.refine(f6, pb.PaganiConfig(rel_tol=tol)))
