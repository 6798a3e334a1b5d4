"""Where does a cold config-3 refine() spend its time inside a process that also holds torch? (debug)"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2302_05730_b200 as pb
from paper_2302_05730_b200 import _native
mode = sys.argv[1] if len(sys.argv) > 1 else "torch"
ctx = _native.context(0)
if mode == "torch":
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda:0")
    flush.zero_(); torch.cuda.synchronize()
if mode in ("torch", "peak"):
    print("peak", ctx.measure_fp64_peak())
f2 = pb.get_integrand("f2", 6)
for _ in range(5):
    pb.mcubes_run(f2, 10**6, 6, 15, seed=0, rel_tol=1e-3)
pb.refine(pb.get_integrand("f4", 5), pb.PaganiConfig(rel_tol=1e-3))
f1 = pb.get_integrand("f1", 8)
t0 = time.perf_counter()
marks = []
res = pb.refine(f1, pb.PaganiConfig(rel_tol=1e-6), progress=lambda r: marks.append((r["iteration"], time.perf_counter() - t0)))
print("cold config3 wall", time.perf_counter() - t0, "device", ctx.last_device_seconds)
for it, t in marks:
    print(f"  iteration {it:2d} record at {1e3 * t:9.2f} ms")
t0 = time.perf_counter()
pb.refine(f1, pb.PaganiConfig(rel_tol=1e-6))
print("warm config3 wall", time.perf_counter() - t0)
