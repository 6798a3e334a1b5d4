"""Plumbing cost of the sharded drivers on ONE GPU: a one-rank NCCL job runs every collective of the product path
(forced), so wall(sharded, world 1) - wall(single-GPU entry point) is the per-run cost of packing, the NCCL launches on
the library's stream, the global-tree kernels and the host reads; divided by the iteration count it is the per-iteration
plumbing an N-rank run pays on top of compute / N (the collectives' payloads are <= a few hundred KB: latency-bound).
    python scripts/sharded_probe.py            (sets up its own one-rank process group on 127.0.0.1)
"""
import os, socket, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
import paper_2302_05730_b200 as pb
from paper_2302_05730_b200 import _native, sharded

with socket.socket() as s:
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
comm = sharded.Comm(device=0)
ctx = _native.context(0)
ctx.reserve(14 << 30)


def best(fn, reps=3):
    out = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = fn()
        out.append(time.perf_counter() - t0)
    return min(out), res


print("workload | single-GPU wall ms | sharded world=1 (all collectives issued) wall ms | iterations | plumbing per iteration us | projected 8-rank speed-up")
f1 = pb.get_integrand("f1", 8)
for tag, cfg in (("config3 PAGANI f1 d=8 1e-6 (2^26 cap)", pb.PaganiConfig(rel_tol=1e-6)),
                 ("PAGANI f1 d=8 1e-6 cap 2^22", pb.PaganiConfig(rel_tol=1e-6, region_cap=1 << 22))):
    pb.refine(f1, cfg); sharded.pagani_refine_sharded(f1, cfg, comm, force_collectives=True)
    t1, ref = best(lambda: pb.refine(f1, cfg))
    t2, res = best(lambda: sharded.pagani_refine_sharded(f1, cfg, comm, force_collectives=True))
    assert res.history == ref.history
    its = ref.iterations + 1
    per = (t2 - t1) / its
    print(f"{tag} | {1e3 * t1:.2f} | {1e3 * t2:.2f} | {its} | {1e6 * per:.1f} | {t1 / (t1 / 8 + max(per, 0) * its):.2f}")
f3 = pb.get_integrand("f3", 8)
for tag, n, its_max, tol in (("config4_fixed m-Cubes f3 d=8 n=1e9 x 4", 10**9, 4, None), ("m-Cubes f3 d=8 n=1e8 x 8", 10**8, 8, None),
                             ("config2 m-Cubes f2 d=6 n=1e6 to 1e-3", 10**6, 15, 1e-3)):
    f = f3 if "f3" in tag else pb.get_integrand("f2", 6)
    d = f.d
    pb.mcubes_run(f, n, d, its_max, seed=0, rel_tol=tol); sharded.mcubes_run_sharded(f, n, d, its_max, comm, seed=0, rel_tol=tol, force_collectives=True)
    t1, ref = best(lambda: pb.mcubes_run(f, n, d, its_max, seed=0, rel_tol=tol))
    t2, res = best(lambda: sharded.mcubes_run_sharded(f, n, d, its_max, comm, seed=0, rel_tol=tol, force_collectives=True))
    assert res.estimate == ref.estimate
    its = len(ref.iterations)
    per = (t2 - t1) / its
    print(f"{tag} | {1e3 * t1:.2f} | {1e3 * t2:.2f} | {its} | {1e6 * per:.1f} | {t1 / (t1 / 8 + max(per, 0) * its):.2f}")
dist.destroy_process_group()
