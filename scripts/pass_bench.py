"""Kernel-only m-Cubes pass timing: `python scripts/pass_bench.py fam d n [reps]` (uniform grid, events on the stream)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2302_05730_b200 as pb
from paper_2302_05730_b200 import _native
fam, d, n = sys.argv[1], int(sys.argv[2]), int(float(sys.argv[3]))
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
plan, grid, f = pb.make_plan(n, d), pb.init_grid(d), pb.get_integrand(fam, d)
ctx = _native.context(0)
pb.mcubes_kernel(f, plan, grid, seed=1)
ctx.profile_begin()
for _ in range(reps):
    pb.mcubes_kernel(f, plan, grid, seed=1)
ms, k, units = ctx.profile_end(1)
print(f"{fam} d={d} samples={plan.n_actual} g={plan.g} p={plan.p}: {ms / k:.3f} ms/pass  {units / (ms * 1e-3):.3e} samples/s")
