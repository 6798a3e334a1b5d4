"""Pin the CPU oracle (oracle/parcube_oracle.py) against fixtures generated from the
UNMODIFIED reference by oracle/make_golden.py, plus the SPEC.md known-answer vectors
(SURVEY.md section 4).  CPU only.

Integer RNG vectors must match bit-for-bit anywhere.  Floating-point vectors must match
bit-for-bit on the numpy build that generated them and to 1e-13 (relative to the natural
scale) elsewhere -- numpy's SIMD exp/cos/pow and OpenBLAS gemv differ between builds.
"""

import os

import numpy as np
import pytest

from conftest import fromhex, golden_rule
from helpers import random_boxes, same_numpy_build
from oracle import parcube_oracle as po


def _close(golden, got, want, scale=None, tol=1e-13):
    got, want = np.asarray(got, dtype=float), np.asarray(want, dtype=float)
    if same_numpy_build(golden) and np.array_equal(got, want):
        return
    assert not os.environ.get("ORACLE_STRICT"), "bit-exact match required on the generating build"
    s = np.maximum(np.abs(want), 0 if scale is None else scale)
    assert np.all(np.abs(got - want) <= tol * np.maximum(s, 1e-300)), \
        f"max rel dev {np.max(np.abs(got - want) / np.maximum(s, 1e-300))}"


# ------------------------------------------------------------------ RNG (integer, portable)
def test_rng_integer_vectors(golden):
    g = golden["rng"]
    for z, want in g["mix64"].items():
        assert int(po.mix64(np.uint64(int(z)))) == want
    for key, want in g["stream_key"].items():
        s, t = map(int, key.split(","))
        assert int(po.stream_key(s, np.uint64(t))) == want
    for key, want in g["uniform"].items():
        s, t, c = map(int, key.split(","))
        assert float(po.uniform(s, np.uint64(t), np.uint64(c))).hex() == want
    for key, want in g["derive_seed"].items():
        s, l = map(int, key.split(","))
        assert po.derive_seed(s, l) == want


def test_rng_survey_vectors():
    # SURVEY.md section 4, captured from the reference at survey time
    assert int(po.mix64(np.uint64(1))) == 0x5692161D100B05E5
    assert int(po.stream_key(12345, np.uint64(7))) == 0x5C42A3F59A093334
    assert float(po.uniform(0, np.uint64(0), np.uint64(0))).hex() == "0x1.0606c54beddd8p-2"
    assert float(po.uniform(12345, np.uint64(7), np.uint64(1))) == 0.0712725466492744
    assert po.derive_seed(0, 1) == 0xE220A8397B1DCDAF
    assert po.derive_seed(7, 3) == 0xE6984080BAB12A02


# ------------------------------------------------------------------ SPEC.md known answers
def test_spec_plans():
    p = po.make_plan(10**8, 8)
    assert (p["g"], p["m"], p["p"]) == (9, 43046721, 2)
    p = po.make_plan(32, 2)
    assert (p["g"], p["m"], p["p"]) == (4, 16, 2)
    p = po.make_plan(10**9, 8)
    assert (p["g"], p["m"], p["p"], p["s"]) == (12, 429981696, 2, 13122)


def test_spec_transform():
    x, jac, b = po.grid_transform(np.array([[0.75]]), np.array([[0.0, 0.8, 1.0]]))
    assert abs(x[0, 0] - 0.9) < 1e-15 and abs(jac[0] - 0.4) < 1e-15 and b[0, 0] == 1


def test_spec_rule_properties(golden):
    for d in (2, 3, 5, 8):
        r = golden_rule(golden, d)
        assert r["weights"].shape[1] == 2**d + 2 * d * d + 2 * d + 1
        assert abs(r["weights"][0].sum() - 1.0) < 1e-12
        assert np.all(np.abs(r["weights"][1:].sum(axis=1)) < 1e-12)


def test_spec_constant_and_sum(golden):
    lefts, lengths = po.uniform_tiling(3, 4)
    i, e, k = po.pagani_evaluate("one", lefts, lengths, golden_rule(golden, 3))
    assert abs(po.tree_sum(i) - 1.0) < 1e-12 and e.max() <= 1e-12 and not k.any()
    i, e, k = po.pagani_evaluate("sum", np.zeros((1, 5)), np.ones((1, 5)), golden_rule(golden, 5))
    assert abs(i[0] - 2.5) < 1e-12


def test_spec_error_mode_max_null():
    v = np.array([[1.0, 0.02, -0.05, 0.01, 0.0]])
    assert po.error_estimates(v, None, None, mode="max-null")[0] == 0.05


def test_tree_sum_shape():
    a = np.arange(1.0, 8.0)
    assert po.tree_sum(a) == ((1 + 2.0) + (3 + 4.0)) + ((5 + 6.0) + (7 + 0.0))
    assert po.tree_sum([]) == 0.0


# ------------------------------------------------------------------ PAGANI evaluate
def _regions_for(meta):
    if meta["kind"] == "uniform":
        return po.uniform_tiling(meta["d"], meta["g"])
    return random_boxes(meta["d"], meta["n"], meta["seed"])


def test_pagani_evaluate_matches_reference(golden):
    z = golden["_pagani_eval"]
    for tag, meta in golden["pagani_eval"].items():
        d = meta["d"]
        if d > 8:
            continue  # fixtures carry full rule tables for d <= 8 only
        lefts, lengths = _regions_for(meta)
        bounds = None
        if "low" in meta:
            low, high = np.array(meta["low"]), np.array(meta["high"])
            bounds = (low, high - low, float(np.prod(high - low)))
        i, e, k = po.pagani_evaluate(meta["family"], lefts, lengths, golden_rule(golden, d),
                                     bounds=bounds, mode=meta.get("err_mode", "two-level"))
        scale = np.max(np.abs(z[f"{tag}_I"]))
        _close(golden, i, z[f"{tag}_I"], scale=scale * 1e-3)
        _close(golden, e, z[f"{tag}_E"], scale=scale * 1e-3, tol=1e-9)
        if same_numpy_build(golden):
            assert np.array_equal(k, z[f"{tag}_K"]), tag


# ------------------------------------------------------------------ PAGANI refine
@pytest.mark.parametrize("idx", range(15))
def test_pagani_refine_matches_reference(golden, idx):
    case = golden["pagani_refine"][idx]
    if case["seconds"] > 6:
        pytest.skip("reference run too slow for the CPU suite; covered on the GPU")
    d = case["d"]
    out = po.pagani_refine(case["family"], d, golden_rule(golden, d), rel_tol=case["rel_tol"],
                           workers=4, **case["cfg"])
    assert out["reason"] == case["reason"] and out["converged"] == case["converged"]
    if same_numpy_build(golden):
        assert out["iterations"] == case["iterations"]
        assert out["regions_processed"] == case["regions_processed"]
        assert out["active_counts"] == case["active"]
        assert [[float(a).hex(), float(b).hex(), c] for a, b, c in out["history"]] == case["history"]
    else:
        assert abs(out["estimate"] - fromhex(case["estimate"])) <= 1e-10 * abs(fromhex(case["estimate"]))


# ------------------------------------------------------------------ m-Cubes
def _bounds(meta):
    if "low" not in meta:
        return None
    low, high = np.array(meta["low"]), np.array(meta["high"])
    return low, high - low, float(np.prod(high - low))


def test_vsample_matches_reference(golden):
    z, metas = golden["_mcubes"], golden["mcubes"]
    for tag, meta in metas.items():
        if tag in ("runs", "inj") or meta["n"] > 300000:
            continue
        plan = po.make_plan(meta["n"], meta["d"])
        assert {k: plan[k] for k in "gmps"} == meta["plan"]
        grid = z[f"{meta['grid_from']}_B"] if "grid_from" in meta else po.uniform_grid(meta["d"])
        res = po.vsample(meta["family"], plan, grid, seed=meta["seed"], workers=4, bounds=_bounds(meta))
        _close(golden, res["integral"], fromhex(meta["integral"]), tol=1e-12)
        _close(golden, res["variance"], fromhex(meta["variance"]), tol=1e-11)
        _close(golden, res["contributions"], z[f"{tag}_C"], scale=z[f"{tag}_C"].max() * 1e-6, tol=1e-12)
        assert res["clamp_events"] == meta["clamps"]
        _close(golden, po.refine_grid(grid, res["contributions"]), z[f"{tag}_B"], tol=1e-12)


def test_vsample_injected_uniforms(golden):
    meta, z = golden["mcubes"]["inj"], golden["_mcubes"]
    plan = po.make_plan(meta["n"], meta["d"])
    table = np.random.default_rng(meta["table_seed"]).random(plan["m"] * plan["p"] * plan["d"])
    stride = plan["s"] * plan["p"] * plan["d"]
    res = po.vsample(meta["family"], plan, po.uniform_grid(meta["d"]),
                     uniform_fn=lambda seed, sid, ctr: table[sid.astype(np.int64) * stride + ctr.astype(np.int64)])
    _close(golden, res["integral"], fromhex(meta["integral"]), tol=1e-12)
    _close(golden, res["variance"], fromhex(meta["variance"]), tol=1e-11)
    _close(golden, res["contributions"], z["inj_C"], scale=z["inj_C"].max() * 1e-6, tol=1e-12)


def test_refine_grid_peaked(golden):
    z = golden["_mcubes"]
    got = po.refine_grid(po.uniform_grid(2), z["peaked_C"])
    _close(golden, got, z["peaked_B"], tol=1e-12)
    assert np.all(np.diff(got, axis=1) > 0)


def test_mcubes_run_matches_reference(golden):
    for run in golden["mcubes"]["runs"]:
        if run["n"] > 300000:
            continue
        out = po.mcubes_run(run["family"], run["n"], run["d"], run["iterations"], seed=run["seed"], workers=4)
        _close(golden, out["estimate"], fromhex(run["estimate"]), tol=1e-10)
        _close(golden, out["errorest"], fromhex(run["errorest"]), tol=1e-9)
        for got, want in zip(out["progress"], run["progress"]):
            _close(golden, got["iter_integral"], fromhex(want["iter_integral"]), tol=1e-10)


def _cube_cases():
    import json
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "sample_cube.json")) as fh:
        return json.load(fh)


def test_sample_cube_matches_reference():
    """mcubes.sample_cube (mcubes.py:143-164): RngStream-fed and table-fed sub-cubes from the reference."""
    doc = _cube_cases()
    for c in doc["cases"]:
        plan = po.make_plan(c["n"], c["d"])
        u = np.array([fromhex(v) for v in c["uniforms"]])
        if c["kind"] == "stream":   # the stream position the reference took the uniforms from (integer-exact)
            ctr = (c["cube"] % plan["s"]) * plan["p"] * c["d"] + np.arange(u.size)
            assert np.array_equal(po.uniform(77, np.uint64(c["cube"] // plan["s"]), ctr.astype(np.uint64)), u)
        s1, s2, bins, w = po.sample_cube(c["family"], c["cube"], plan, po.uniform_grid(c["d"]), u)
        assert bins.tolist() == c["bins"]
        want = (fromhex(c["s1"]), fromhex(c["s2"]), np.array([fromhex(v) for v in c["weights"]]))
        if doc["numpy"] == np.__version__:
            assert (s1, s2) == want[:2] and np.array_equal(w, want[2])
        else:
            assert abs(s1 - want[0]) <= 1e-13 * abs(want[0]) and abs(s2 - want[1]) <= 1e-13 * abs(want[1])
            assert np.allclose(w, want[2], rtol=1e-13, atol=0)


def test_update_variance_examples():
    # SPEC.md:386-387 through the same formulas the V-Sample pass uses
    def upd(s1, s2, p, m):
        raw = (s2 - s1 * s1 / p) / (p * (p - 1) * m * m)
        return s1 / (p * m), max(raw, 0.0)
    assert upd(2, 4, 2, 1) == (1.0, 1.0)
    assert upd(2, 2, 2, 4) == (0.25, 0.0)
