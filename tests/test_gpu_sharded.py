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
@pytest.mark.parametrize("host_staged", [False, True])
def test_sharded_pagani_equals_single_context(family, d, cfg_kw, world, host_staged):
    """host_staged = False: the product path (pieces packed on the device, exchanged as device tensors, global trees
    finished on the device); True: the same pieces as host arrays (the path the gloo CPU tests drive)."""
    cfg = pb.PaganiConfig(**cfg_kw)
    f = pb.get_integrand(family, d)
    want = pb.refine(f, cfg)
    orbit = rules.orbit_form(pb.build_rule(d))

    def rank_body(rank, comm):
        ctx = _native.Context(0)
        try:
            shard = _native.PaganiShard(f.device_spec(), orbit, cfg, ctx=ctx)
            return sharded.pagani_refine_sharded(f, cfg, comm, shard=shard, host_staged=host_staged)
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
        ctx = _native.Context(0)    # one library context (stream, buffers, run state) per rank
        try:
            return sharded.mcubes_run_sharded(f, n, d, 3, comm, seed=4, ctx=ctx)
        finally:
            ctx.close()

    for res in run_ranks(world, rank_body):
        # iteration 0: identical grid -> bit-identical (I, Var) through the all-gathered group partials
        assert res.iterations[0].integral == want.iterations[0].integral
        assert res.iterations[0].variance == want.iterations[0].variance
        assert [it.clamp_events for it in res.iterations] == [it.clamp_events for it in want.iterations]
        assert abs(res.estimate - want.estimate) <= 1e-10 * abs(want.estimate)
        assert np.allclose(res.iterations[0].contributions.c, want.iterations[0].contributions.c, rtol=1e-12, atol=0)


def test_sharded_mcubes_single_rank_is_the_single_gpu_run():
    """world = 1 through the shard entry points (pcb_mcubes_shard_*): same kernels, the packed row instead of the group
    buffer -- every iteration bit-identical to pcb_mcubes_run, tables included."""
    f = pb.get_integrand("f2", 6)
    want = pb.mcubes_run(f, 10**6, 6, 15, seed=0, rel_tol=1e-3)
    (got,) = run_ranks(1, lambda rank, comm: sharded.mcubes_run_sharded(f, 10**6, 6, 15, comm, seed=0, rel_tol=1e-3))
    assert len(got.iterations) == len(want.iterations) == 4
    for a, b in zip(got.iterations, want.iterations):
        assert (a.integral, a.variance, a.clamp_events) == (b.integral, b.variance, b.clamp_events)
        assert np.array_equal(a.contributions.c, b.contributions.c)
    assert (got.estimate, got.errorest, got.chi2_per_dof) == (want.estimate, want.errorest, want.chi2_per_dof)


def test_sharded_mcubes_more_ranks_than_groups_and_tolerance_stop():
    """Ranks without a work-group (n_groups = 2 < world = 3) contribute empty rows and tables; the tolerance stop is taken
    on the device from the gathered rows, identically on every rank."""
    f = pb.get_integrand("f4", 3)
    n = 2 * 128 * 4            # m = 8^3 = 512 sub-cubes -> s = 1, 512 threads... two work-groups of 256? (group_size 256)
    want = pb.mcubes_run(f, n, 3, 12, seed=2, rel_tol=5e-2, group_size=256)
    assert want.plan.n_groups == 2

    def rank_body(rank, comm):
        ctx = _native.Context(0)
        try:
            return sharded.mcubes_run_sharded(f, n, 3, 12, comm, seed=2, rel_tol=5e-2, group_size=256, ctx=ctx)
        finally:
            ctx.close()

    for res in run_ranks(3, rank_body):
        assert len(res.iterations) == len(want.iterations)
        assert res.iterations[0].integral == want.iterations[0].integral
        assert abs(res.estimate - want.estimate) <= 1e-10 * abs(want.estimate)


def test_sharded_mcubes_non_finite_raises_on_every_rank():
    """A non-finite sample: the flag travels in the gathered rows, so every rank raises the same error -- the lowest
    offending sub-cube of the WHOLE pass, which lies on rank 0's shard -- instead of hanging in the next collective
    (single-GPU error type and index, mcubes.py:238-241)."""
    f = pb.get_integrand("f2", 2)
    f.a2 = float("nan")          # every sample is NaN: rank 1's own first offender is NOT sub-cube 0
    n = 2 * 10**5
    with pytest.raises(pb.GroupTaskError) as info:
        pb.mcubes_run(f, n, 2, 2, seed=0)
    want = info.value.cause.region_index
    assert want == 0
    errors = []

    def rank_body(rank, comm):
        ctx = _native.Context(0)
        try:
            sharded.mcubes_run_sharded(f, n, 2, 2, comm, seed=0, ctx=ctx)
        except pb.GroupTaskError as exc:
            errors.append((rank, exc.cause.region_index, exc.group_id))
        finally:
            ctx.close()

    run_ranks(2, rank_body)
    assert sorted(errors) == [(0, want, 0), (1, want, 0)]


def test_sharded_pagani_non_finite_raises_on_every_rank():
    """A non-finite evaluation (here: every tile with an axis centred on x = 1/2; the first is tile 1 of the 3^3
    tiling, on rank 0's slice): the flags travel in the packed rows, the lowest owner looks the evaluation up and every
    rank raises the single-GPU GroupTaskError with the GLOBAL region index (pagani.py:206-209)."""
    f = pb.get_integrand("f2", 3)
    f.a2 = 0.0                      # 1/(0 + u^2) is infinite at x = 1/2
    cfg = pb.PaganiConfig(rel_tol=1e-3, initial_regions=27)   # g = 3: the middle third of an axis is centred on 1/2
    with pytest.raises(pb.GroupTaskError) as info:
        pb.refine(f, cfg)
    want = (info.value.cause.region_index, info.value.group_id, tuple(info.value.cause.point))
    assert want[0] == 1
    orbit = rules.orbit_form(pb.build_rule(3))
    seen = []

    def rank_body(rank, comm):
        ctx = _native.Context(0)
        try:
            sharded.pagani_refine_sharded(f, cfg, comm, shard=_native.PaganiShard(f.device_spec(), orbit, cfg, ctx=ctx))
        except pb.GroupTaskError as exc:
            seen.append((rank, exc.cause.region_index, exc.group_id, tuple(exc.cause.point)))
        finally:
            ctx.close()

    run_ranks(3, rank_body)
    assert sorted(seen) == [(r,) + want for r in range(3)]
