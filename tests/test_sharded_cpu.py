"""Multi-GPU host logic on CPU: world_size-2 gloo runs of the sharded m-Cubes driver with an
oracle-backed compute backend (the product backend is the CUDA library; only the collectives,
shard arithmetic and reduction order are under test here)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import parcube_oracle as po


class OracleBackend:
    """Per-rank compute through the CPU oracle (test infrastructure only)."""

    def sample(self, family, plan, boundaries, seed, thread_range, rng_kind):
        oplan = po.make_plan(plan.n_requested, plan.d, plan.group_size)
        g0, g1 = thread_range[0] // plan.group_size, -(-thread_range[1] // plan.group_size)
        out = po.vsample(family, oplan, boundaries, seed=seed, groups=range(g0, g1))
        return out["group_partials"], out["contributions"], out["clamp_events"]

    def refine(self, boundaries, contrib, alpha, smoothing):
        return po.refine_grid(boundaries, contrib, alpha, smoothing)

    def tree_sum(self, values):
        return po.tree_sum(values)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, family, n, d, iterations, seed, out_dir):
    import torch.distributed as dist

    from paper_2302_05730_b200 import sharded

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = sharded.Comm()
        recs = []
        res = sharded.mcubes_run_sharded(family, n, d, iterations, comm, backend=OracleBackend(), seed=seed,
                                         progress=recs.append)
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), estimate=res.estimate, errorest=res.errorest,
                 integrals=[r.integral for r in res.iterations], variances=[r.variance for r in res.iterations],
                 clamps=[r.clamp_events for r in res.iterations], table=res.iterations[-1].contributions.c,
                 n_progress=len(recs))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("family,n,d,world", [("f3", 60000, 5, 2), ("f2", 40000, 3, 2), ("f5", 30000, 4, 3)])
def test_sharded_mcubes_matches_single_process(tmp_path, family, n, d, world):
    iterations, seed = 3, 5
    mp.spawn(_worker, args=(world, _free_port(), family, n, d, iterations, seed, str(tmp_path)), nprocs=world, join=True)
    ranks = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    want = po.mcubes_run(family, n, d, iterations, seed=seed)
    for r in ranks:
        # every rank holds the same result
        assert r["estimate"] == ranks[0]["estimate"] and np.array_equal(r["table"], ranks[0]["table"])
        assert r["n_progress"] == iterations
        # iteration 0 runs on the same grid: the all-gathered group partials + reference pair tree are bit-exact
        assert r["integrals"][0] == want["iterations"][0]["integral"]
        assert r["variances"][0] == want["iterations"][0]["variance"]
        assert list(r["clamps"]) == [it["clamp_events"] for it in want["iterations"]]
        # later iterations see a grid refined from an all-reduced table (different summation order): 1e-10
        assert abs(r["estimate"] - want["estimate"]) <= 1e-10 * abs(want["estimate"])
        assert abs(r["errorest"] - want["errorest"]) <= 1e-8 * want["errorest"]


def test_group_shards_cover_everything():
    from paper_2302_05730_b200.sharded import group_shards

    for n_groups in (1, 2, 7, 230, 256):
        for world in (1, 2, 3, 8):
            shards = group_shards(n_groups, world)
            assert shards[0][0] == 0 and shards[-1][1] == n_groups
            assert all(a[1] == b[0] for a, b in zip(shards, shards[1:]))
            assert max(b - a for a, b in shards) - min(b - a for a, b in shards) <= 1
