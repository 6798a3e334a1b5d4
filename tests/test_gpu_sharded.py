"""The sharded drivers with the real CUDA backend: several ranks emulated on ONE B200 (one library
context per rank, threads + an in-process communicator).  Multi-GPU runs are not possible in this
environment; what is checked here is that sharding changes nothing: histories are bit-identical to the
single-context runs for every family (same kernels, same global pair trees, same classification)."""

import numpy as np
import pytest

import paper_2302_05730_b200 as pb
from helpers import run_ranks
from paper_2302_05730_b200 import _native, rules, sharded

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("family,d,cfg_kw,world", [
    ("f4", 5, dict(rel_tol=1e-3), 2),                       # BASELINE config 1, survivors concentrate -> rebalancing
    ("f2", 5, dict(rel_tol=1e-3), 3),
    ("f3", 6, dict(rel_tol=1e-3), 4),
    ("f1", 8, dict(rel_tol=1e-6, region_cap=1 << 19), 8),   # config 3 shape: every region splits, 8 ranks
    ("f2", 3, dict(rel_tol=1e-3, max_iterations=20, initial_regions=16), 3),   # empty shards + forced progress
])
def test_sharded_pagani_equals_single_context(family, d, cfg_kw, world):
    cfg = pb.PaganiConfig(**cfg_kw)
    f = pb.get_integrand(family, d)
    want = pb.refine(f, cfg)
    orbit = rules.orbit_form(pb.build_rule(d))

    def rank_body(rank, comm):
        ctx = _native.Context(0)
        try:
            shard = _native.PaganiShard(f.device_spec(), orbit, cfg, ctx=ctx)
            return sharded.pagani_refine_sharded(f, cfg, comm, shard=shard)
        finally:
            ctx.close()

    for res in run_ranks(world, rank_body):
        assert res.history == want.history          # bit-identical estimate / errorest / leaf counts
        assert (res.iterations, res.regions_processed, res.converged, res.reason) == \
               (want.iterations, want.regions_processed, want.converged, want.reason)


@pytest.mark.parametrize("family,d,n,world", [("f3", 8, 10**6, 2), ("f2", 6, 10**6, 4), ("f5", 5, 10**5, 3)])
def test_sharded_mcubes_equals_single_context(family, d, n, world, monkeypatch):
    monkeypatch.setenv("PCB_MCUBES_SEGMENTS", "2")   # same per-thread segmentation in every run
    f = pb.get_integrand(family, d)
    want = pb.mcubes_run(f, n, d, 3, seed=4)

    def rank_body(rank, comm):
        return sharded.mcubes_run_sharded(f, n, d, 3, comm, seed=4)

    for res in run_ranks(world, rank_body):
        # iteration 0: identical grid -> bit-identical (I, Var) through the all-gathered group partials
        assert res.iterations[0].integral == want.iterations[0].integral
        assert res.iterations[0].variance == want.iterations[0].variance
        assert [it.clamp_events for it in res.iterations] == [it.clamp_events for it in want.iterations]
        assert abs(res.estimate - want.estimate) <= 1e-10 * abs(want.estimate)
        assert np.allclose(res.iterations[0].contributions.c, want.iterations[0].contributions.c, rtol=1e-12, atol=0)
