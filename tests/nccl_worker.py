"""Worker of tests/test_gpu_nccl.py: one rank of a real NCCL job (torch.distributed, backend nccl) that runs the sharded
drivers with the collectives on the library's device buffers and compares them with the single-GPU runs of the same
process.  Launched by torchrun (world >= 2, needs as many GPUs) or directly with RANK/WORLD_SIZE = 0/1 (one GPU: NCCL
still executes every collective, on a one-rank communicator).  Prints one JSON line per rank."""

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2302_05730_b200 as pb  # noqa: E402
from paper_2302_05730_b200 import sharded  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    os.environ["PARCUBE_B200_DEVICE"] = str(local)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", local))
    out = {"rank": rank, "world": world, "backend": dist.get_backend()}
    try:
        comm = sharded.Comm(device=local)
        # ---- m-Cubes: BASELINE config 2 to its tolerance, and a d = 8 pass with many work-groups
        f = pb.get_integrand("f2", 6)
        want = pb.mcubes_run(f, 10**6, 6, 15, seed=0, rel_tol=1e-3)
        got = sharded.mcubes_run_sharded(f, 10**6, 6, 15, comm, seed=0, rel_tol=1e-3, force_collectives=True)
        out["mcubes_iterations"] = [len(got.iterations), len(want.iterations)]
        out["mcubes_it0_bit_identical"] = bool(got.iterations[0].integral == want.iterations[0].integral
                                               and got.iterations[0].variance == want.iterations[0].variance)
        out["mcubes_all_bit_identical"] = bool(all(a.integral == b.integral and a.variance == b.variance and
                                                   np.array_equal(a.contributions.c, b.contributions.c)
                                                   for a, b in zip(got.iterations, want.iterations)))
        out["mcubes_rel_dev"] = abs(got.estimate - want.estimate) / abs(want.estimate)
        # ---- PAGANI: config 1 (survivors concentrate: rows move between ranks) and the config-3 shape
        for tag, fam, d, kw in (("config1", "f4", 5, dict(rel_tol=1e-3)), ("config3_cap19", "f1", 8, dict(rel_tol=1e-6, region_cap=1 << 19))):
            g = pb.get_integrand(fam, d)
            cfg = pb.PaganiConfig(**kw)
            ref = pb.refine(g, cfg)
            res = sharded.pagani_refine_sharded(g, cfg, comm, force_collectives=True)
            out[f"pagani_{tag}_bit_identical"] = bool(res.history == ref.history and res.reason == ref.reason and
                                                      res.regions_processed == ref.regions_processed)
        # every rank holds the same results
        digest = torch.tensor([got.estimate, got.errorest, res.estimate, res.errorest], dtype=torch.float64, device=f"cuda:{local}")
        parts = [torch.empty_like(digest) for _ in range(world)]
        dist.all_gather(parts, digest)
        out["ranks_agree"] = bool(all(torch.equal(p, parts[0]) for p in parts))
        out["ok"] = True
    except Exception as exc:  # noqa: BLE001
        import traceback
        out["ok"] = False
        out["error"] = f"{type(exc).__name__}: {exc}"
        out["trace"] = traceback.format_exc()[-1500:]
    finally:
        dist.destroy_process_group()
    print("NCCL_WORKER " + json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
