"""PAGANI parity on the B200, through the C-ABI (ctypes) behind the reference-named API.

Bars (BASELINE.json north_star): per-region values within 1e-12 relative, final estimates
within 1e-10 relative, region counts identical (integer classification bit-exact).  Families
whose arithmetic has no transcendental (f2, sum) must match the oracle BIT FOR BIT, which
proves the abscissa map, the 64-virtual-thread strided schedule, the pair tree, the error
estimate, the split axis, the filter and the bisection are exact restatements.
"""

import numpy as np
import pytest

import paper_2302_05730_b200 as pb
from conftest import fromhex, golden_rule
from helpers import random_boxes
from oracle import parcube_oracle as po

pytestmark = pytest.mark.gpu

FAMILIES = ["f1", "f2", "f3", "f4", "f5", "f6", "sum"]
EXACT = ("f2", "sum")
REL_I = 1e-12   # per-region integral, relative to max(|I|, region scale)
REL_E = 1e-7    # per-region error estimate where it is above the cancellation floor
REL_EST = 1e-10  # final estimates
# split axes that may differ from the reference over ALL non-exact evaluate fixtures together (ties of the
# fourth-difference indicator broken by rounding noise); measured on the B200: see the printed table
MAX_DIFFERING_AXES = 40


def rule_dict(r):
    return dict(generators=r.generators, weights=r.weights, axial_indices=r.axial_indices,
                split_weights=r.split_weights, null_degrees=r.null_degrees, null_scales=r.null_scales)


def _regions(meta):
    if meta["kind"] == "uniform":
        rl = pb.uniform_split(meta["d"], meta["g"])
        return rl.lefts, rl.lengths
    return random_boxes(meta["d"], meta["n"], meta["seed"])


def _integrand(meta):
    f = pb.get_integrand(meta["family"], meta["d"])
    if "low" in meta:
        f = pb.scale_to_bounds(f, pb.IntegrationBounds(meta["low"], meta["high"]))
    return f


def _check_regions(tag, fam, got, want_i, want_e, want_k, exact, volumes=None):
    if exact:
        assert np.array_equal(got.integrals, want_i), tag
        assert np.array_equal(got.errors, want_e), tag
        assert np.array_equal(got.split_axes, want_k), tag
        return
    # 1e-12 relative to the region's own scale: |I| or, for sign-changing integrands whose I cancels,
    # the largest |I| of a congruent region in the batch
    scale = np.maximum(np.abs(want_i), 1e-3 * np.max(np.abs(want_i)))
    if fam == "f1" and volumes is not None:
        # oscillatory: I cancels inside a region; the natural scale is volume * max|f| = volume
        scale = np.maximum(np.abs(want_i), volumes)
    assert np.all(np.abs(got.integrals - want_i) <= REL_I * scale), (tag, np.max(np.abs(got.integrals - want_i) / scale))
    # the null-rule sums cancel to ~1e-3..1e-10 of |I|; compare E where it is resolved
    resolved = want_e > 1e-7 * np.abs(want_i)
    if resolved.any():
        dev = np.abs(got.errors - want_e)[resolved] / want_e[resolved]
        assert dev.max() <= REL_E, (tag, dev.max())
    assert np.all(got.errors >= 0)


# ------------------------------------------------------------------ device functors
@pytest.mark.parametrize("fam", FAMILIES)
def test_functors_against_oracle(fam):
    rng = np.random.default_rng(7)
    for d in (1, 2, 5, 6, 7, 8, 9, 12):
        pts = rng.random((4096, d))
        got = pb.get_integrand(fam, d).eval_many(pts)
        want = po.genz_eval(fam, d, pts)
        if fam in EXACT:
            assert np.array_equal(got, want)
        elif fam == "f1":  # |cos| <= 1: absolute accuracy (argument rounding of a sum up to 78)
            assert np.max(np.abs(got - want)) <= 4e-14
        else:
            assert np.max(np.abs(got - want) / np.abs(want).clip(1e-300)) <= 4e-14, fam
    f = pb.get_integrand(fam, 3)
    assert f(np.array([0.2, 0.4, 0.6])) == f.eval_many(np.array([[0.2, 0.4, 0.6]]))[0]


def test_f6_threshold_is_strict():
    f = pb.get_integrand("f6", 2)   # thresholds 0.4, 0.5
    pts = np.array([[0.4, 0.1], [np.nextafter(0.4, 0), 0.1], [0.1, 0.5], [0.39, 0.49]])
    got = f.eval_many(pts)
    assert got[0] == 0.0 and got[2] == 0.0 and got[1] > 0 and got[3] > 0
    assert np.allclose(got, po.genz_eval("f6", 2, pts), rtol=1e-15)


# ------------------------------------------------------------------ evaluate vs the reference fixtures
def test_evaluate_matches_reference_fixtures(golden):
    z = golden["_pagani_eval"]
    differing = {}
    for tag, meta in golden["pagani_eval"].items():
        d = meta["d"]
        lefts, lengths = _regions(meta)
        cfg = pb.PaganiConfig(err_mode=meta.get("err_mode", "two-level"))
        got = pb.pagani_kernel(_integrand(meta), pb.RegionList(lefts, lengths), pb.build_rule(d), None, cfg)
        assert got.split_axes.dtype == np.int64 and not got.integrals.flags.writeable
        exact = meta["family"] in EXACT and "low" not in meta
        _check_regions(tag, meta["family"], got, z[f"{tag}_I"], z[f"{tag}_E"], z[f"{tag}_K"].astype(np.int64), exact,
                       volumes=np.prod(lengths, axis=1))
        if not exact:
            # split axis: identical wherever the reference's own indicator is not a numerical tie.  The number of
            # differing axes per fixture is printed (pytest -s / the captured-output section of a failure), so a
            # drift from 99.9 % to 99.1 % shows in the log long before it trips the bar.
            same = got.split_axes == z[f"{tag}_K"]
            differing[tag] = (int((~same).sum()), int(same.size))
            assert same.mean() >= 0.99, (tag, same.mean())
    print("split axes differing from the reference, per fixture (count / regions):")
    for tag, (bad, n) in differing.items():
        print(f"  {tag:24s} {bad:5d} / {n}")
    print(f"  total {sum(b for b, _ in differing.values())} / {sum(n for _, n in differing.values())}")
    # today's state, so that a regression shows as a failure, not only in the log: every fixture but the tie-ridden
    # uniform f4/f5 tilings agrees on every region
    assert sum(b for b, _ in differing.values()) <= MAX_DIFFERING_AXES, differing


@pytest.mark.parametrize("fam", EXACT)
@pytest.mark.parametrize("d", [1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11])
def test_evaluate_bit_exact_random_boxes(fam, d):
    n = 300 if d < 9 else 24
    lefts, lengths = random_boxes(d, n, seed=900 + d)
    rule = pb.build_rule(d)
    got = pb.pagani_kernel(pb.get_integrand(fam, d), pb.RegionList(lefts, lengths), rule)
    i, e, k = po.pagani_evaluate(fam, lefts, lengths, rule_dict(rule))
    _check_regions(f"{fam}{d}", fam, got, i, e, k, exact=True)


@pytest.mark.parametrize("group", [1, 7, 16, 32, 33, 63, 64, 65, 100, 128, 149, 150, 1000])
def test_schedule_width_is_bit_exact(group):
    """Every schedule width the reference accepts (pagani.py:56,66: any G >= 1); f_eval(6) = 149, so 149/150/1000
    cover "one point per virtual thread" and "more virtual threads than points"."""
    d = 6
    lefts, lengths = random_boxes(d, 128, seed=5)
    rule = pb.build_rule(d)
    cfg = pb.PaganiConfig(group_size=group)
    got = pb.pagani_kernel(pb.get_integrand("f2", d), pb.RegionList(lefts, lengths), rule, None, cfg)
    i, e, k = po.pagani_evaluate("f2", lefts, lengths, rule_dict(rule), group=group)
    _check_regions(f"G{group}", "f2", got, i, e, k, exact=True)


@pytest.mark.parametrize("fam", ["f1", "f3", "f4"])
def test_wide_schedule_on_transcendental_families(fam):
    """G > 64 with exp/cos/pow: per-region values to 1e-12 against the oracle at the same width."""
    d, group = 8, 200
    lefts, lengths = random_boxes(d, 96, seed=21)
    rule = pb.build_rule(d)
    got = pb.pagani_kernel(pb.get_integrand(fam, d), pb.RegionList(lefts, lengths), rule, None, pb.PaganiConfig(group_size=group))
    i, e, k = po.pagani_evaluate(fam, lefts, lengths, rule_dict(rule), group=group)
    _check_regions(f"{fam}-G{group}", fam, got, i, e, k, exact=False, volumes=np.prod(lengths, axis=1))


def test_bad_schedule_width_is_an_error():
    with pytest.raises(ValueError):
        pb.PaganiConfig(group_size=0)


@pytest.mark.parametrize("mode", ["two-level", "max-null", "max-pairwise"])
def test_error_modes_bit_exact(mode):
    d = 6
    lefts, lengths = random_boxes(d, 200, seed=11)
    rule = pb.build_rule(d)
    got = pb.pagani_kernel(pb.get_integrand("f2", d), pb.RegionList(lefts, lengths), rule, None, pb.PaganiConfig(err_mode=mode))
    i, e, k = po.pagani_evaluate("f2", lefts, lengths, rule_dict(rule), mode=mode)
    _check_regions(mode, "f2", got, i, e, k, exact=True)


def test_bounded_integrand_bit_exact():
    d = 4
    low, high = np.array([-1.0, 0.25, 0.0, -3.0]), np.array([2.0, 0.75, 3.0, 5.0])
    b = pb.IntegrationBounds(low, high)
    lefts, lengths = random_boxes(d, 200, seed=3)
    rule = pb.build_rule(d)
    for fam in EXACT:
        got = pb.pagani_kernel(pb.scale_to_bounds(pb.get_integrand(fam, d), b), pb.RegionList(lefts, lengths), rule)
        i, e, k = po.pagani_evaluate(fam, lefts, lengths, rule_dict(rule), bounds=(low, high - low, float(np.prod(high - low))))
        _check_regions("bounded-" + fam, fam, got, i, e, k, exact=True)


def test_spec_known_answers():
    from paper_2302_05730_b200.genz import ConstantOne
    est = pb.pagani_kernel(ConstantOne(3), pb.uniform_split(3, 4), pb.build_rule(3))
    assert abs(pb.tree_sum(est.integrals) - 1.0) < 1e-12 and est.errors.max() <= 1e-12 and not est.split_axes.any()
    one = pb.pagani_kernel(pb.get_integrand("sum", 5), pb.RegionList(np.zeros((1, 5)), np.ones((1, 5))), pb.build_rule(5))
    assert abs(one.integrals[0] - 2.5) < 1e-12
    # split axis = k for an integrand varying only along axis k, at any scale
    for k in range(3):
        low, high = np.zeros(3), np.ones(3)
        # f4 restricted: stretch the other axes so that only axis k sees the peak
        width = np.full(3, 1e-6)
        width[k] = 1.0
        f = pb.scale_to_bounds(pb.get_integrand("f4", 3), pb.IntegrationBounds(0.5 - width / 2, 0.5 + width / 2))
        est = pb.pagani_kernel(f, pb.uniform_split(3, 2), pb.build_rule(3))
        assert np.all(est.split_axes == k)


def test_argument_errors():
    rule = pb.build_rule(3)
    with pytest.raises(ValueError):
        pb.pagani_kernel(pb.get_integrand("f4", 4), pb.uniform_split(3, 2), rule)
    with pytest.raises(ValueError):
        pb.pagani_kernel(pb.get_integrand("f4", 3), pb.uniform_split(3, 2), pb.build_rule(4))
    with pytest.raises(TypeError):
        pb.pagani_kernel(pb.FunctionIntegrand(lambda x: 1.0, 3), pb.uniform_split(3, 2), rule)


def test_non_finite_report_matches_reference_convention():
    f = pb.get_integrand("f2", 3)
    f.a2 = 0.0  # 1/(0 + u^2) is infinite at the centre abscissa x = 1/2
    lefts = np.array([[0.0, 0.0, 0.0], [0.25, 0.25, 0.25], [0.0, 0.25, 0.25]])
    lengths = np.array([[0.5, 0.5, 0.5], [0.5, 0.5, 0.5], [1.0, 0.5, 0.5]])
    with pytest.raises(pb.GroupTaskError) as info:
        pb.pagani_kernel(f, pb.RegionList(np.tile(lefts, (400, 1)), np.tile(lengths, (400, 1))), pb.build_rule(3),
                         None, pb.PaganiConfig(chunk=512))
    cause = info.value.cause
    assert isinstance(cause, pb.NonFiniteEvaluationError)
    # first offending (region, point) in row-major order: region 1 (centre 0.5 on every axis), point 0
    assert cause.region_index == 1 and info.value.group_id == 0
    assert np.array_equal(cause.point, [0.5, 0.5, 0.5]) and np.isinf(cause.value)


# ------------------------------------------------------------------ reductions
@pytest.mark.parametrize("n", [1, 2, 3, 63, 64, 1000, 1024, 1025, 4097, 1048577, 3000001])
def test_tree_sum_bit_exact(n):
    a = np.random.default_rng(n).standard_normal(n) * 10.0 ** np.random.default_rng(n + 1).integers(-8, 8, n)
    assert pb.tree_sum(a) == po.tree_sum(a)


def test_tree_sum_edge_cases():
    assert pb.tree_sum([]) == 0.0
    m = np.random.default_rng(0).random((3, 50))
    assert np.array_equal(pb.tree_sum(m, axis=1), po.tree_sum(m, axis=1))
    assert pb.reduce([]) == 0.0 and pb.reduce([1.0, 2.0, 3.0]) == 6.0


# ------------------------------------------------------------------ refine vs the reference
def _sweep_cases():
    import json
    import os
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "sweep_refine.json")
    with open(path) as fh:
        return json.load(fh)["cases"]


@pytest.mark.parametrize("case", _sweep_cases(), ids=lambda c: f"{c['family']}d{c['d']}")
def test_refine_sweep_config5_matches_reference(case):
    """BASELINE config 5: the sweep cases the reference converges on at rel_tol 1e-3 (f1d6, f4d6, f5d6, f3d7, f3d8;
    the d=5 ones and f3d6 are in test_refine_matches_reference).  Up to 15.5 M regions: identical iteration counts,
    per-iteration active/leaf counts, regions_processed and stop reasons; estimates to 1e-10."""
    _check_refine_case(case)


@pytest.mark.parametrize("idx", range(15))
def test_refine_matches_reference(golden, idx):
    _check_refine_case(golden["pagani_refine"][idx])


def _check_refine_case(case):
    recs = []
    res = pb.refine(pb.get_integrand(case["family"], case["d"]), pb.PaganiConfig(rel_tol=case["rel_tol"], **case["cfg"]),
                    progress=recs.append)
    assert res.reason == case["reason"] and res.converged == case["converged"]
    # integer classification bit-exact: same iteration count, same region counts in every iteration
    assert res.iterations == case["iterations"]
    assert res.regions_processed == case["regions_processed"]
    assert [r["active"] for r in recs] == case["active"]
    assert [h[2] for h in res.history] == [h[2] for h in case["history"]]
    assert [r["iteration"] for r in recs] == list(range(len(recs)))
    want_est, want_err = fromhex(case["estimate"]), fromhex(case["errorest"])
    assert abs(res.estimate - want_est) <= REL_EST * abs(want_est)
    assert abs(res.errorest - want_err) <= 1e-6 * want_err
    for (e, r, _), (we, wr, _) in zip(res.history, case["history"]):
        assert abs(e - fromhex(we)) <= REL_EST * abs(fromhex(we))
    if case["family"] in EXACT:
        assert [(float(a).hex(), float(b).hex()) for a, b, _ in res.history] == [(a, b) for a, b, _ in case["history"]]


def test_refine_config3_full_size():
    """BASELINE config 3 at full size: the reference does not converge, it stops on the region cap
    after 53,741,151 regions (reference values measured at survey time)."""
    res = pb.refine(pb.get_integrand("f1", 8), pb.PaganiConfig(rel_tol=1e-6))
    assert (res.reason, res.converged, res.iterations, res.regions_processed) == ("region cap reached", False, 12, 53741151)
    assert [h[2] for h in res.history] == [6561 * 2**k for k in range(13)]
    assert abs(res.estimate - 3.4395582917226246e-05) <= REL_EST * 3.4395582917226246e-05
    assert abs(res.errorest - 2.0412892505107233e-07) <= 1e-6 * 2.0412892505107233e-07


def test_refine_against_live_oracle_with_bounds():
    low, high = np.array([0.2, 0.1, 0.3]), np.array([0.9, 0.8, 0.7])
    f = pb.scale_to_bounds(pb.get_integrand("f2", 3), pb.IntegrationBounds(low, high))
    res = pb.refine(f, pb.PaganiConfig(rel_tol=1e-6, initial_regions=200))
    rule = rule_dict(pb.build_rule(3))
    want = po.pagani_refine("f2", 3, rule, rel_tol=1e-6, initial_regions=200,
                            bounds=(low, high - low, float(np.prod(high - low))))
    assert res.iterations == want["iterations"] and res.regions_processed == want["regions_processed"]
    assert [(a, b, c) for a, b, c in res.history] == want["history"]   # bit-exact, bounds included


def test_refine_budget_and_caps():
    with pytest.raises(pb.BudgetExceededError):
        pb.refine(pb.get_integrand("f4", 5), pb.PaganiConfig(region_cap=1000))
    res = pb.refine(pb.get_integrand("f6", 4), pb.PaganiConfig(rel_tol=1e-9, max_iterations=0))
    assert res.reason == "max iterations reached" and res.iterations == 0 and len(res.history) == 1
    res = pb.refine(pb.get_integrand("f6", 4), pb.PaganiConfig(rel_tol=1e-9, region_cap=5000))
    assert res.reason == "region cap reached" and res.regions_processed <= 5000


def test_refine_force_progress_fallback_bit_exact():
    """When no active region exceeds its budget share, the worst regions (ties included) are split
    (pagani.py:364-365).  f2, d=3 from 16 initial regions enters that path from iteration 15 on."""
    rule = rule_dict(pb.build_rule(3))
    for tol in (1e-3, 1e-6):
        want = po.pagani_refine("f2", 3, rule, rel_tol=tol, max_iterations=25, initial_regions=16)
        assert want["forced_iterations"], "fixture no longer exercises the fallback"
        res = pb.refine(pb.get_integrand("f2", 3), pb.PaganiConfig(rel_tol=tol, max_iterations=25, initial_regions=16))
        assert [(a, b, c) for a, b, c in res.history] == want["history"]
        assert res.regions_processed == want["regions_processed"] and res.reason == want["reason"]


def test_apply_rules_single_region(golden):
    rule = pb.build_rule(5)
    region = pb.Region(np.full(5, 0.25), np.full(5, 0.5))
    est, fx = pb.apply_rules(pb.get_integrand("f2", 5), region, rule)
    pts = region.left + region.length * ((rule.generators + 1.0) / 2.0)
    want_fx = po.genz_eval("f2", 5, pts)
    assert np.array_equal(fx, want_fx)
    want = float(np.prod(region.length)) * po.tree_sum(rule.weights * want_fx[None, :], axis=-1)
    assert np.array_equal(est.values, want)
    assert pb.compute_split_axis(fx, rule, 5) in range(5)
    assert pb.find_max_err(est, 1.0, rule=rule) >= 0


# ------------------------------------------------------------------ one-region-per-lane kernel
@pytest.mark.parametrize("fam", FAMILIES)
@pytest.mark.parametrize("d", [1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 12])
def test_lane_kernel_equals_warp_kernel_bit_for_bit(fam, d, monkeypatch):
    """Long lists run one region per lane, short ones one warp per region (pagani_eval_lanes.cuh vs
    pagani_eval.cuh / pagani_eval_mult.cuh).  The results must not depend on which kernel evaluated
    a region -- otherwise a sharded list would not reproduce the single-GPU tree."""
    n = {1: 1000, 2: 999, 3: 777, 4: 600, 5: 555, 6: 333, 7: 200, 8: 130, 9: 100, 10: 70, 12: 40}[d]
    lefts, lengths = random_boxes(d, n, 1234 + d)
    regions, rule = pb.RegionList(lefts, lengths), pb.build_rule(d)
    for wrap in (False, True):
        f = pb.get_integrand(fam, d)
        if wrap:
            f = pb.scale_to_bounds(f, pb.IntegrationBounds([0.1] * d, [0.9 + 0.01 * j for j in range(d)]))
        monkeypatch.setenv("PCB_PAGANI_LANES_MIN", "1")
        lanes = pb.pagani_kernel(f, regions, rule)
        monkeypatch.setenv("PCB_PAGANI_LANES_MIN", str(10**12))
        warps = pb.pagani_kernel(f, regions, rule)
        assert np.array_equal(lanes.integrals, warps.integrals), (fam, d, wrap)
        assert np.array_equal(lanes.errors, warps.errors), (fam, d, wrap)
        assert np.array_equal(lanes.split_axes, warps.split_axes), (fam, d, wrap)
        if fam in EXACT and not wrap:   # and both are the reference, bit for bit
            i, e, k = po.pagani_evaluate(fam, lefts, lengths, rule_dict(rule))
            assert np.array_equal(lanes.integrals, i) and np.array_equal(lanes.errors, e) and np.array_equal(lanes.split_axes, k)


def test_rule_with_parity_in_another_row_keeps_warp_kernels(monkeypatch):
    """The lane kernels hard-wire WHICH null rule alternates its corner weights with the bit count (row 2,
    quadrature.py:199-203).  A caller-supplied table with that rule in another row must still evaluate
    exactly: the host routes it to the warp-per-region kernels whatever the list length."""
    d = 8
    base = pb.build_rule(d)
    w = np.array(base.weights)
    w[[2, 3]] = w[[3, 2]]
    deg, sc = list(base.null_degrees), list(base.null_scales)
    deg[1], deg[2] = deg[2], deg[1]
    sc[1], sc[2] = sc[2], sc[1]
    rule = pb.RuleTable(d, base.f_eval, base.generators, w, base.split_weights, base.axial_indices, deg, sc)
    lefts, lengths = random_boxes(d, 200, 99)
    regions = pb.RegionList(lefts, lengths)
    f = pb.get_integrand("f2", d)
    i, e, k = po.pagani_evaluate("f2", lefts, lengths, rule_dict(rule))
    for lanes_min in ("1", str(10**12)):
        monkeypatch.setenv("PCB_PAGANI_LANES_MIN", lanes_min)
        est = pb.pagani_kernel(f, regions, rule)
        assert np.array_equal(est.integrals, i) and np.array_equal(est.errors, e) and np.array_equal(est.split_axes, k)


def test_lane_kernel_reports_first_nonfinite(monkeypatch):
    """A non-finite evaluation surfaces exactly as in the warp kernels (pagani.py:206-209)."""
    d = 3
    # the Jacobian 1e160^3 overflows: every evaluation is 0 * inf or finite * inf
    f = pb.scale_to_bounds(pb.get_integrand("f4", d), pb.IntegrationBounds([0.0] * d, [1e160] * d))
    rl = pb.uniform_split(d, 8)
    errs = []
    for lanes_min in ("1", str(10**12)):
        monkeypatch.setenv("PCB_PAGANI_LANES_MIN", lanes_min)
        with pytest.raises(pb.GroupTaskError) as exc:
            pb.pagani_kernel(f, rl, pb.build_rule(d))
        cause = exc.value.cause
        errs.append((cause.region_index, tuple(np.asarray(cause.point).tolist())))
    assert errs[0] == errs[1]


@pytest.mark.parametrize("fam,d,tol,kw", [
    ("f4", 5, 1e-3, {}), ("f2", 5, 1e-3, {}), ("sum", 3, 1e-9, {}), ("f5", 2, 1e-6, {}), ("f1", 3, 1e-8, {}),
    ("f3", 4, 1e-5, {}), ("f6", 3, 1e-4, {"max_iterations": 7}), ("f2", 4, 1e-6, {"region_cap": 3000}),
    ("f4", 6, 1e-3, {"max_iterations": 12}),
])
def test_short_list_iteration_kernel_equals_general_path(fam, d, tol, kw, monkeypatch):
    """Lists of <= 1024 regions run a whole refinement iteration in one CTA (short_iteration_kernel); the
    history must be the general path's, bit for bit, through every transition between the two."""
    f = pb.get_integrand(fam, d)
    cfg = pb.PaganiConfig(rel_tol=tol, **kw)
    monkeypatch.setenv("PCB_PAGANI_SHORT", "1")
    a = pb.refine(f, cfg)
    monkeypatch.setenv("PCB_PAGANI_SHORT", "0")
    b = pb.refine(f, cfg)
    assert a.history == b.history
    assert (a.estimate, a.errorest, a.iterations, a.regions_processed, a.converged, a.reason) == \
           (b.estimate, b.errorest, b.iterations, b.regions_processed, b.converged, b.reason)


@pytest.mark.parametrize("fam,d,rel,absv", [("f2", 4, 1e-12, 1e4), ("sum", 3, 1e-16, 1e-13), ("f4", 5, 1e-9, 1e-11),
                                            ("f5", 3, 1e-12, 1e-6), ("f2", 5, 1e-3, 0.0)])
def test_abs_tol_extension_matches_oracle(fam, d, rel, absv):
    """epsabs (BASELINE.json north_star; the reference has rel_tol only): the target becomes
    max(abs_tol, rel_tol*|estimate|) for the stop test and the split threshold.  abs_tol = 0 is the reference."""
    res = pb.refine(pb.get_integrand(fam, d), pb.PaganiConfig(rel_tol=rel, abs_tol=absv, max_iterations=30))
    want = po.pagani_refine(fam, d, rule_dict(pb.build_rule(d)), rel_tol=rel, abs_tol=absv, max_iterations=30)
    assert (res.iterations, res.regions_processed, res.reason, res.converged) == \
           (want["iterations"], want["regions_processed"], want["reason"], want["converged"])
    if fam in EXACT:
        assert res.history == want["history"]
    else:
        assert abs(res.estimate - want["estimate"]) <= REL_EST * abs(want["estimate"])
    if res.converged:
        assert res.errorest <= max(absv, rel * abs(res.estimate))


def test_progress_exception_stops_the_run_at_once():
    """An exception raised by `progress` ends the refinement at that iteration and propagates (the reference calls
    `progress` inline, pagani.py:341-349); the context stays usable."""
    seen = []

    class Stop(Exception):
        pass

    def cb(rec):
        seen.append(rec["iteration"])
        if rec["iteration"] == 2:
            raise Stop("enough")

    with pytest.raises(Stop):
        pb.refine(pb.get_integrand("f1", 8), pb.PaganiConfig(rel_tol=1e-6, region_cap=1 << 22), progress=cb)
    assert seen == [0, 1, 2]
    seen.clear()
    with pytest.raises(Stop):   # short-list path (<= 1024 regions per iteration)
        pb.refine(pb.get_integrand("f4", 5), pb.PaganiConfig(rel_tol=1e-3), progress=cb)
    assert seen == [0, 1, 2]
    res = pb.refine(pb.get_integrand("f4", 5), pb.PaganiConfig(rel_tol=1e-3))
    assert (res.iterations, res.regions_processed) == (10, 3328)


_REFINE_SNIPPET = r"""
import json
import paper_2302_05730_b200 as pb
out = []
for fam, d, kw in [("f4", 5, dict(rel_tol=1e-5)), ("f2", 5, dict(rel_tol=1e-3)), ("f1", 6, dict(rel_tol=1e-3)),
                   ("f3", 5, dict(rel_tol=1e-6, region_cap=100000)), ("f5", 4, dict(rel_tol=1e-5, initial_regions=16)),
                   ("f4", 5, dict(rel_tol=1e-3, group_size=96)), ("f6", 3, dict(rel_tol=1e-9, max_iterations=9))]:
    r = pb.refine(pb.get_integrand(fam, d), pb.PaganiConfig(**kw))
    out.append([r.estimate, r.errorest, r.iterations, int(r.regions_processed), r.reason, [list(h) for h in r.history]])
print(json.dumps(out))
"""


def test_refine_launch_modes_agree_bit_for_bit():
    """How the refinement is driven is scheduling only: programmatic launches (PCB_NO_PDL=1: plain), scalars through
    pinned memory (PCB_PAGANI_PUBLISH=0: copy + synchronise) and the device-resident short-list chain
    (PCB_PAGANI_SPECULATE=0: one iteration at a time) give the same histories, bit for bit."""
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for extra in ({}, {"PCB_NO_PDL": "1"}, {"PCB_PAGANI_PUBLISH": "0"}, {"PCB_PAGANI_SPECULATE": "0"},
                  {"PCB_NO_PDL": "1", "PCB_PAGANI_PUBLISH": "0", "PCB_PAGANI_SPECULATE": "0"}):
        env = dict(os.environ, PYTHONPATH=root, **extra)
        res = subprocess.run([sys.executable, "-c", _REFINE_SNIPPET], env=env, capture_output=True, text=True, timeout=600)
        assert res.returncode == 0, res.stderr[-2000:]
        outs.append(json.loads(res.stdout.strip().splitlines()[-1]))
    assert all(o == outs[0] for o in outs[1:])
