"""Kernel-only PAGANI evaluate timing: `python scripts/eval_bench.py fam d g [reps]` prints ms per launch and
evaluations/s for uniform_split(d, g), once per kernel choice (lanes / warp)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2302_05730_b200 as pb
from paper_2302_05730_b200 import _native

fam, d, g = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
rl, rule = pb.uniform_split(d, g), pb.build_rule(d)
f = pb.get_integrand(fam, d)
ctx = _native.context(0)
fe = 2**d + 2 * d * d + 2 * d + 1
for name, lanes_min in (("lanes", "1"), ("warp", str(10**12))):
    os.environ["PCB_PAGANI_LANES_MIN"] = lanes_min
    pb.pagani_kernel(f, rl, rule)
    ctx.profile_begin()
    for _ in range(reps):
        pb.pagani_kernel(f, rl, rule)
    ms, n, units = ctx.profile_end(0)
    print(f"{fam} d={d} regions={rl.n} {name}: {ms / n:.3f} ms/launch  {units * fe / (ms * 1e-3):.3e} evals/s")
