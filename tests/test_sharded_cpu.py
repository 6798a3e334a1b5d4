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


# ================================================================================ PAGANI
class OraclePaganiShard:
    """The shard-step interface of _native.PaganiShard, computed by the CPU oracle (test only)."""

    def __init__(self, family, d, rule, cfg):
        self.family, self.d, self.rule, self.cfg = family, d, rule, cfg
        self.ret_i = self.ret_e = np.empty(0)

    def init(self, g, first, count):
        lefts, lengths = po.uniform_tiling(self.d, g)
        self.lefts, self.lengths = lefts[first:first + count].copy(), lengths[first:first + count].copy()
        self.evaluate()

    def evaluate(self):
        if len(self.lefts):
            self.i, self.e, self.k = po.pagani_evaluate(self.family, self.lefts, self.lengths, self.rule)
        else:
            self.i, self.e, self.k = np.empty(0), np.empty(0), np.empty(0, dtype=np.int64)

    def counts(self):
        return len(self.lefts), len(self.ret_i)

    def reduce(self, which, head):
        a = (self.i, self.e, self.ret_i, self.ret_e)[which]
        h = min(head, len(a))
        nb = (len(a) - h) // 1024
        blocks = np.array([po.tree_sum(a[h + 1024 * b:h + 1024 * (b + 1)]) for b in range(nb)])
        return a[:h].copy(), blocks, a[h + 1024 * nb:].copy()

    def max_error(self):
        return float(self.e.max()) if len(self.e) else 0.0

    def classify(self, budget, mode, emax):
        if mode == 0:
            self.mask = self.e > budget * np.prod(self.lengths, axis=1) if len(self.e) else np.zeros(0, dtype=bool)
        else:
            self.mask = self.e >= emax
        return int(np.count_nonzero(self.mask))

    def split(self):
        m = self.mask
        self.ret_i, self.ret_e = self.i[~m], self.e[~m]
        if m.any():
            self.lefts, self.lengths = po.bisect(self.lefts[m], self.lengths[m], self.k[m])
        else:
            self.lefts, self.lengths = np.empty((0, self.d)), np.empty((0, self.d))

    def export(self, begin, end):
        return self.lefts[begin:end].copy(), self.lengths[begin:end].copy()

    def rebuild(self, keep_begin, keep_end, front, back):
        parts_l, parts_h = [], []
        for rows in (front, (self.lefts[keep_begin:keep_end], self.lengths[keep_begin:keep_end]), back):
            if rows is not None and len(rows[0]):
                parts_l.append(rows[0])
                parts_h.append(rows[1])
        self.lefts = np.concatenate(parts_l) if parts_l else np.empty((0, self.d))
        self.lengths = np.concatenate(parts_h) if parts_h else np.empty((0, self.d))

    def tree_sum(self, values):
        return po.tree_sum(values)


def _rule_from_golden(d):
    import json

    from conftest import GOLDEN
    z = np.load(os.path.join(GOLDEN, "rules.npz"))
    meta = json.load(open(os.path.join(GOLDEN, "golden.json")))["rules"][str(d)]
    return dict(generators=z[f"gen{d}"], weights=z[f"w{d}"], axial_indices=z[f"ax{d}"],
                split_weights=np.array([float.fromhex(v) for v in meta["split"]]),
                null_degrees=tuple(meta["null_degrees"]), null_scales=tuple(meta["null_scales"]))


def _pagani_worker(rank, world, port, family, d, cfg_kw, out_dir):
    import torch.distributed as dist

    from paper_2302_05730_b200 import sharded
    from paper_2302_05730_b200.cubature import PaganiConfig

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys_path_root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    import sys
    sys.path.insert(0, os.path.join(sys_path_root, "tests"))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = sharded.Comm()
        cfg = PaganiConfig(**cfg_kw)
        shard = OraclePaganiShard(family, d, _rule_from_golden(d), cfg)
        recs = []
        res = sharded.pagani_refine_sharded(None, cfg, comm, shard=shard, progress=recs.append)
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), history=np.array(res.history), iterations=res.iterations,
                 processed=res.regions_processed, converged=res.converged, reason=res.reason,
                 active=[r["active"] for r in recs], final_local=len(shard.lefts))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("family,d,cfg_kw,world", [
    ("f2", 3, dict(rel_tol=1e-5), 2),                                   # peaked: survivors concentrate -> rebalancing
    ("f2", 3, dict(rel_tol=1e-3, max_iterations=20, initial_regions=16), 3),  # tiny lists, empty shards, forced progress
    ("f4", 4, dict(rel_tol=1e-4), 3),
    ("sum", 2, dict(rel_tol=1e-16, max_iterations=3), 2),               # everything splits: ragged 1024-block edges
    ("f1", 5, dict(rel_tol=1e-6, region_cap=20000), 2),                 # region cap
])
def test_sharded_pagani_is_bit_identical_to_single_process(tmp_path, family, d, cfg_kw, world):
    mp.spawn(_pagani_worker, args=(world, _free_port(), family, d, cfg_kw, str(tmp_path)), nprocs=world, join=True)
    want = po.pagani_refine(family, d, _rule_from_golden(d), **cfg_kw)
    ranks = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    for r in ranks:
        assert str(r["reason"]) == want["reason"] and bool(r["converged"]) == want["converged"]
        assert int(r["iterations"]) == want["iterations"] and int(r["processed"]) == want["regions_processed"]
        assert list(r["active"]) == want["active_counts"]
        got = [(float(a), float(b), int(c)) for a, b, c in r["history"]]
        assert got == [(a, b, int(c)) for a, b, c in want["history"]]     # bit-identical estimates and errors
    # the final lists are balanced to within one region
    sizes = [int(r["final_local"]) for r in ranks]
    assert max(sizes) - min(sizes) <= 1


# ================================================================================ tensor-level collectives
def _tensor_worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist

    from paper_2302_05730_b200 import sharded

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = sharded.Comm()
        # in-place all-gather: the rank's row sits at its own slot of the target, like the library's packed rows
        n = 7
        gathered = torch.zeros(world * n, dtype=torch.float64)
        row = torch.arange(n, dtype=torch.float64) + 100.0 * rank
        comm.all_gather_into(gathered, row)
        table = torch.full((5,), float(rank + 1), dtype=torch.float64)
        comm.all_reduce_sum_(table)
        peak = torch.tensor([float(rank), -float(rank)], dtype=torch.float64)
        comm.all_reduce_max_(peak)
        # ring exchange of [2][d][n] row blocks of different sizes
        d = 3
        right, left = (rank + 1) % world, (rank - 1) % world
        send = torch.full((2, d, rank + 1), float(rank), dtype=torch.float64)
        recv = torch.empty((2, d, left + 1), dtype=torch.float64)
        comm.exchange_tensors({right: send}, {left: recv})
        np.savez(os.path.join(out_dir, f"t{rank}.npz"), gathered=gathered.numpy(), table=table.numpy(), peak=peak.numpy(),
                 recv=recv.numpy(), left=left)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_comm_tensor_collectives_under_gloo(tmp_path, world):
    """The tensor-level surface the device drivers use (all_gather_into, all_reduce_sum_/max_, exchange_tensors), on CPU
    tensors under gloo: same calls, same semantics as under NCCL on the library's device buffers."""
    mp.spawn(_tensor_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    for rank in range(world):
        z = np.load(tmp_path / f"t{rank}.npz")
        want = np.concatenate([np.arange(7) + 100.0 * r for r in range(world)])
        assert np.array_equal(z["gathered"], want)
        assert np.array_equal(z["table"], np.full(5, world * (world + 1) / 2))
        assert np.array_equal(z["peak"], [world - 1.0, 0.0])
        left = int(z["left"])
        assert z["recv"].shape == (2, 3, left + 1) and np.all(z["recv"] == left)
