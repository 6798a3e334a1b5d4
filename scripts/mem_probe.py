import os, sys, time
sys.path.insert(0, "/root/repo")
import paper_2302_05730_b200 as pb
from paper_2302_05730_b200 import _native
ctx = _native.context(0)
f1 = pb.get_integrand("f1", 8)
pb.refine(f1, pb.PaganiConfig(rel_tol=1e-6))
print("=== now f1 d=6 1e-4", file=sys.stderr)
f6 = pb.get_integrand("f1", 6)
t0 = time.perf_counter(); pb.refine(f6, pb.PaganiConfig(rel_tol=1e-4)); print("f1 d=6 1e-4 wall", time.perf_counter() - t0, file=sys.stderr)
t0 = time.perf_counter(); pb.refine(f6, pb.PaganiConfig(rel_tol=1e-4)); print("f1 d=6 1e-4 wall again", time.perf_counter() - t0, file=sys.stderr)
