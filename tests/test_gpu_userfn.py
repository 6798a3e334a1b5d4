"""Run-time integrand families (userfn.compile_integrand): the functor is compiled from CUDA source against the
library's kernel templates.  Checked (1) against the built-in family it restates, bit for bit, through every kernel
path, and (2) against the oracle evaluating the same function as a numpy callable (the reference's
FunctionIntegrand(vectorized=True), core.py:72-93)."""
import os

import numpy as np
import pytest

import paper_2302_05730_b200 as pb
from oracle import parcube_oracle as po
from helpers import random_boxes
from test_gpu_pagani import rule_dict

pytestmark = pytest.mark.gpu

F2_TERM = "double u = x - 0.5; return 1.0 / (param[0] + u * u);"


def _bump(d):
    """exp(-7 sum (x_j - 0.3)^2): a family the registry does not have."""
    f = pb.compile_integrand(d, term="double u = x - 0.3; return u * u;", finish="return exp(-param[0] * acc);",
                             combine="numpy_sum", params=(7.0,), name="bump")
    return f, (lambda pts: np.exp(-7.0 * np.sum((pts - 0.3) * (pts - 0.3), axis=1)))


def test_restated_family_is_bit_identical_pagani():
    d = 5
    user = pb.compile_integrand(d, F2_TERM, combine="prod", params=(1.0 / 2500.0,), name="f2-restated")
    builtin = pb.get_integrand("f2", d)
    rule = pb.build_rule(d)
    lefts, lengths = random_boxes(d, 3000, 3)
    rl = pb.RegionList(lefts, lengths)
    for lanes_min in ("1", str(10**12)):            # the one-region-per-lane kernel and the warp-per-region kernel
        os.environ["PCB_PAGANI_LANES_MIN"] = lanes_min
        try:
            a, b = pb.pagani_kernel(user, rl, rule), pb.pagani_kernel(builtin, rl, rule)
        finally:
            del os.environ["PCB_PAGANI_LANES_MIN"]
        assert np.array_equal(a.integrals, b.integrals) and np.array_equal(a.errors, b.errors)
        assert np.array_equal(a.split_axes, b.split_axes)
    wide = pb.PaganiConfig(group_size=96)
    assert np.array_equal(pb.pagani_kernel(user, rl, rule, cfg=wide).integrals, pb.pagani_kernel(builtin, rl, rule, cfg=wide).integrals)
    ra, rb = pb.refine(user, pb.PaganiConfig(rel_tol=1e-3), rule=rule), pb.refine(builtin, pb.PaganiConfig(rel_tol=1e-3), rule=rule)
    assert (ra.estimate, ra.errorest, ra.regions_processed, ra.iterations) == (rb.estimate, rb.errorest, rb.regions_processed, rb.iterations)
    pts = np.random.default_rng(0).random((1000, d))
    assert np.array_equal(user.eval_many(pts), builtin.eval_many(pts))
    assert user(pts[0]) == builtin(pts[0])


def test_restated_family_is_bit_identical_mcubes():
    d = 6
    user = pb.compile_integrand(d, F2_TERM, combine="prod", params=(1.0 / 2500.0,))
    builtin = pb.get_integrand("f2", d)
    plan, grid = pb.make_plan(200_000, d), pb.init_grid(d)
    a, b = pb.mcubes_kernel(user, plan, grid, seed=3), pb.mcubes_kernel(builtin, plan, grid, seed=3)
    assert (a.integral, a.variance) == (b.integral, b.variance)
    assert np.allclose(a.contributions.c, b.contributions.c, rtol=1e-12, atol=0)
    ra = pb.mcubes_run(user, 10**6, d, 15, seed=0, rel_tol=1e-3)
    rb = pb.mcubes_run(builtin, 10**6, d, 15, seed=0, rel_tol=1e-3)
    assert len(ra.iterations) == len(rb.iterations)
    assert abs(ra.estimate - rb.estimate) <= 1e-9 * abs(rb.estimate)


@pytest.mark.parametrize("d", [3, 6])
def test_new_family_against_oracle_pagani(d):
    f, fn = _bump(d)
    rule = pb.build_rule(d)
    lefts, lengths = random_boxes(d, 2000, 5)
    want_i, want_e, want_k = po.pagani_evaluate(fn, lefts, lengths, rule_dict(rule))
    got = pb.pagani_kernel(f, pb.RegionList(lefts, lengths), rule)
    assert np.all(np.abs(got.integrals - want_i) <= 1e-12 * np.abs(want_i))
    resolved = want_e > 1e-7 * np.abs(want_i)
    assert np.all(np.abs(got.errors - want_e)[resolved] <= 1e-7 * want_e[resolved])
    assert np.mean(got.split_axes == want_k) >= 0.99
    want = po.pagani_refine(fn, d, rule_dict(rule), rel_tol=1e-4)
    res = pb.refine(f, pb.PaganiConfig(rel_tol=1e-4), rule=rule)
    assert (res.iterations, res.regions_processed, res.converged) == (want["iterations"], want["regions_processed"], want["converged"])
    assert abs(res.estimate - want["estimate"]) <= 1e-10 * abs(want["estimate"])
    # the closed form: prod_j integral of exp(-7 (x - 0.3)^2) over [0, 1]
    from math import erf, pi, sqrt
    exact = (sqrt(pi / 7.0) / 2.0 * (erf(sqrt(7.0) * 0.7) + erf(sqrt(7.0) * 0.3))) ** d
    assert abs(res.estimate - exact) <= 10 * res.errorest


def test_new_family_against_oracle_mcubes():
    d = 4
    f, fn = _bump(d)
    plan = pb.make_plan(50_000, d)
    oplan = po.make_plan(50_000, d)
    grid = pb.init_grid(d)
    got = pb.mcubes_kernel(f, plan, grid, seed=9)
    want = po.vsample(fn, oplan, grid.boundaries, seed=9)
    assert abs(got.integral - want["integral"]) <= 1e-12 * abs(want["integral"])
    assert abs(got.variance - want["variance"]) <= 1e-10 * abs(want["variance"])
    assert np.allclose(got.contributions.c, want["contributions"], rtol=1e-12, atol=0)
    # bounds wrapper over a run-time family, run to a tolerance, against the closed form on [0, 2]^d
    from math import erf, pi, sqrt
    wrapped = pb.scale_to_bounds(f, pb.IntegrationBounds(np.zeros(d), 2.0 * np.ones(d)))
    res = pb.mcubes_run(wrapped, 10**6, d, 10, seed=1, rel_tol=1e-3)
    exact = (sqrt(pi / 7.0) / 2.0 * (erf(sqrt(7.0) * 1.7) + erf(sqrt(7.0) * 0.3))) ** d
    assert abs(res.estimate - exact) <= 4 * res.errorest + 1e-3 * exact


def test_source_errors_and_slot_reuse():
    with pytest.raises(ValueError, match="does not compile"):
        pb.compile_integrand(3, term="return undefined_symbol;")
    with pytest.raises(ValueError):
        pb.compile_integrand(3, term="return x;", combine="median")
    # more families than resident slots: the oldest is replaced and comes back on use
    fams = [pb.compile_integrand(2, term=f"return {k}.0 * x;") for k in range(1, 11)]
    pts = np.array([[0.25, 0.5]])
    for k, f in enumerate(fams, start=1):
        assert f.eval_many(pts)[0] == k * 0.25 + k * 0.5
    assert fams[0].eval_many(pts)[0] == 0.75
    # kernels that need a shared-memory grant, on recycled slots: integral of k (x + y) over the unit square = k
    plan, grid, rule = pb.make_plan(20000, 2), pb.init_grid(2), pb.build_rule(2)
    for k in (10, 1, 9, 2):
        r = pb.mcubes_kernel(fams[k - 1], plan, grid, seed=k)
        assert abs(r.integral - k) <= 5 * r.variance**0.5
        est = pb.pagani_kernel(fams[k - 1], pb.uniform_split(2, 120), rule)      # 14400 regions: the lane kernel
        assert abs(pb.tree_sum(est.integrals) - k) <= 1e-12 * k


def test_bounds_wrapper_pagani_against_oracle():
    d = 3
    f, fn = _bump(d)
    low, high = np.array([-0.5, 0.0, 0.1]), np.array([1.0, 2.0, 0.9])
    wrapped = pb.scale_to_bounds(f, pb.IntegrationBounds(low, high))
    rule = pb.build_rule(d)
    lefts, lengths = random_boxes(d, 1500, 8)
    bounds = (low, high - low, float(np.prod(high - low)))
    want_i, want_e, _ = po.pagani_evaluate(fn, lefts, lengths, rule_dict(rule), bounds=bounds)
    got = pb.pagani_kernel(wrapped, pb.RegionList(lefts, lengths), rule)
    assert np.all(np.abs(got.integrals - want_i) <= 1e-12 * np.abs(want_i))
    want = po.pagani_refine(fn, d, rule_dict(rule), rel_tol=1e-5, bounds=bounds)
    res = pb.refine(wrapped, pb.PaganiConfig(rel_tol=1e-5), rule=rule)
    assert (res.iterations, res.regions_processed, res.converged) == (want["iterations"], want["regions_processed"], want["converged"])
    assert abs(res.estimate - want["estimate"]) <= 1e-10 * abs(want["estimate"])


def test_non_finite_report_of_a_run_time_family():
    """1 / (x_0 - 1/2) is infinite at the centre abscissa of a region centred on 1/2: same report as a built-in family."""
    f = pb.compile_integrand(3, term="return j == 0 ? 1.0 / (x - 0.5) : x;", name="pole")
    lefts = np.array([[0.0, 0.0, 0.0], [0.25, 0.25, 0.25], [0.0, 0.25, 0.25]])
    lengths = np.array([[0.5, 0.5, 0.5], [0.5, 0.5, 0.5], [1.0, 0.5, 0.5]])
    with pytest.raises(pb.GroupTaskError) as info:
        pb.pagani_kernel(f, pb.RegionList(np.tile(lefts, (400, 1)), np.tile(lengths, (400, 1))), pb.build_rule(3))
    cause = info.value.cause
    assert isinstance(cause, pb.NonFiniteEvaluationError)
    assert cause.region_index == 1 and np.array_equal(cause.point, [0.5, 0.5, 0.5]) and np.isinf(cause.value)


def test_sharded_refine_with_a_run_time_family():
    """Two emulated ranks on one device (one library context per rank): same history as the single-device refinement."""
    from paper_2302_05730_b200 import _native, rules, sharded
    from test_gpu_sharded import run_ranks

    d = 3
    f, _ = _bump(d)
    cfg = pb.PaganiConfig(rel_tol=1e-6)
    want = pb.refine(f, cfg)
    orbit = rules.orbit_form(pb.build_rule(d))

    def rank_body(rank, comm):
        ctx = _native.Context(0)
        try:
            shard = _native.PaganiShard(f.device_spec(), orbit, cfg, ctx=ctx)
            return sharded.pagani_refine_sharded(f, cfg, comm, shard=shard)
        finally:
            ctx.close()

    for res in run_ranks(2, rank_body):
        assert res.history == want.history
        assert (res.iterations, res.regions_processed, res.converged) == (want.iterations, want.regions_processed, want.converged)
