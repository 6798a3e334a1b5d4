"""Degree-7 fully symmetric cubature rule tables and their device (orbit) form.

`build_rule(d)` reproduces the reference's `RuleTable` (reference:
pkg/src/parcube/quadrature.py:260-289) -- same generator order
(quadrature.py:87-114), the same two moment solves (quadrature.py:121-171) and
the same SVD/Gram-Schmidt null rules (quadrature.py:174-257) -- so the tables are
bit-identical to the reference's on the same numpy/LAPACK build
(tests/test_rules.py pins this against fixtures generated from the reference).
The table is *input data* for the device: `orbit_form(rule)` verifies that a
table has the fully symmetric orbit structure and compresses it to the 7 distinct
abscissa offsets and 5x5 orbit weights the kernels take by value.

Point order: centre | (+l2,-l2) per axis | (+l3,-l3) per axis | for j<k the sign
pairs (+,+),(-,+),(+,-),(-,-) at l4 | 2^d corners at l5, bit j set => minus.
"""

from __future__ import annotations

import numpy as np

from .domain import Integrand, Region, _Frozen, check_dimension, region_volume

LAMBDA2 = np.sqrt(9.0 / 70.0)
LAMBDA3 = np.sqrt(9.0 / 10.0)
LAMBDA4 = np.sqrt(9.0 / 10.0)
LAMBDA5 = np.sqrt(9.0 / 19.0)
SAFEGUARD_SCALE = 1e-3  # reference: quadrature.py:177

N_ORBITS = 5  # centre, l2-axial, l3-axial, l4-pairs, l5-corners


def f_eval_count(d: int) -> int:
    """2^d + 2d^2 + 2d + 1 points (reference: quadrature.py:37-40)."""
    d = check_dimension(d)
    return (1 << d) + 2 * d * d + 2 * d + 1


class RuleTable(_Frozen):
    """Per-dimension rule data, read-only (reference: quadrature.py:43-70)."""

    __slots__ = ("d", "f_eval", "generators", "weights", "split_weights",
                 "axial_indices", "null_degrees", "null_scales")

    def __init__(self, d, f_eval, generators, weights, split_weights, axial_indices,
                 null_degrees, null_scales):
        self._put("d", int(d))
        self._put("f_eval", int(f_eval))
        for name, arr in (("generators", generators), ("weights", weights),
                          ("split_weights", split_weights)):
            a = np.array(arr, dtype=np.float64, order="C")
            a.setflags(write=False)
            self._put(name, a)
        ai = np.array(axial_indices, dtype=np.int64, order="C")
        ai.setflags(write=False)
        self._put("axial_indices", ai)
        self._put("null_degrees", tuple(null_degrees))
        self._put("null_scales", tuple(null_scales))


class RuleEstimates(_Frozen):
    """Five volume-scaled rule values of one region (reference: quadrature.py:73-84)."""

    __slots__ = ("values",)

    def __init__(self, values):
        v = np.array(values, dtype=np.float64)
        if v.shape != (5,):
            raise ValueError("expected exactly five rule values")
        v.setflags(write=False)
        self._put("values", v)


# --------------------------------------------------------------------------- construction
def _point_set(d: int):
    """(generators (F,d), orbit id per point (F,))."""
    f_eval = f_eval_count(d)
    gen = np.zeros((f_eval, d))
    orb = np.zeros(f_eval, dtype=np.int64)
    row = 1
    for lam, oid in ((LAMBDA2, 1), (LAMBDA3, 2)):
        for j in range(d):
            gen[row, j] = lam
            gen[row + 1, j] = -lam
            orb[row:row + 2] = oid
            row += 2
    for j in range(d):
        for k in range(j + 1, d):
            for sj, sk in ((1, 1), (-1, 1), (1, -1), (-1, -1)):
                gen[row, j] = sj * LAMBDA4
                gen[row, k] = sk * LAMBDA4
                orb[row] = 3
                row += 1
    bits = np.arange(1 << d)[:, None]
    minus = ((bits >> np.arange(d)[None, :]) & 1).astype(bool)
    gen[row:] = np.where(minus, -LAMBDA5, LAMBDA5)
    orb[row:] = 4
    return gen, orb


_POWERS = {"x2": 2, "x4": 4, "x6": 6}


def _moment_table(d: int) -> dict:
    """Orbit sums (unit weight per point) of the even monomials that pin degree 7,
    for the unit-normalised measure on [-1,1]^d (reference: quadrature.py:121-136)."""
    lam = (None, LAMBDA2, LAMBDA3, LAMBDA4, LAMBDA5)
    table = {"1": np.array([1, 2 * d, 2 * d, 2 * d * (d - 1), 2**d], dtype=float)}
    for key, e in _POWERS.items():
        table[key] = np.array([0,
                               2 * lam[1]**e,
                               2 * lam[2]**e,
                               4 * (d - 1) * lam[3]**e,
                               2**d * lam[4]**e])
    if d >= 2:
        table["x2y2"] = np.array([0, 0, 0, 4 * lam[3]**4, 2**d * lam[4]**4])
    return table


def _orbit_solve(table: dict, orbits: tuple, moments: dict) -> np.ndarray:
    cols = list(orbits)
    lhs = np.array([table[k][cols] for k in moments])
    rhs = np.array([moments[k] for k in moments])
    out = np.zeros(N_ORBITS)
    out[cols] = np.linalg.solve(lhs, rhs)
    return out


def _degree7_and_5(d: int, table: dict):
    """Orbit weights of the degree-7 rule and its embedded degree-5 companion
    (reference: quadrature.py:152-171). Moments: E[x^2]=1/3, E[x^4]=1/5,
    E[x^6]=1/7, E[x^2 y^2]=1/9."""
    if d >= 2:
        w7 = _orbit_solve(table, (0, 1, 2, 3, 4),
                          {"1": 1.0, "x2": 1 / 3, "x4": 1 / 5, "x6": 1 / 7, "x2y2": 1 / 9})
        w5 = _orbit_solve(table, (0, 1, 2, 3),
                          {"1": 1.0, "x2": 1 / 3, "x4": 1 / 5, "x2y2": 1 / 9})
    else:
        w7 = _orbit_solve(table, (0, 1, 2, 4), {"1": 1.0, "x2": 1 / 3, "x4": 1 / 5, "x6": 1 / 7})
        w5 = _orbit_solve(table, (0, 1, 2), {"1": 1.0, "x2": 1 / 3, "x4": 1 / 5})
    return w7, w5


def _gram_schmidt(candidates, against: list) -> list:
    kept = []
    for vec in candidates:
        for q in against + kept:
            vec = vec - np.dot(vec, q) * q
        nrm = np.linalg.norm(vec)
        if nrm > 1e-10:
            kept.append(vec / nrm)
    return kept


def _null_rows(d: int, orb: np.ndarray, table: dict, w7: np.ndarray, w5: np.ndarray):
    """Four null rules per point + their degrees and scales (reference: quadrature.py:180-257)."""
    n1 = (w5 - w7)[orb]
    n1_norm = float(np.linalg.norm(n1))
    corners = np.nonzero(orb == 4)[0]

    def rescale(v, factor):
        return v * (factor * n1_norm / np.linalg.norm(v))

    active = [0, 1, 2, 3, 4] if d >= 2 else [0, 1, 2, 4]
    constraint = np.stack([table["1"][active], table["x2"][active]])
    basis = np.linalg.svd(constraint)[2][2:]
    v0 = (w5 - w7)[active]
    v0 = v0 / np.linalg.norm(v0)
    extras = _gram_schmidt(basis, [v0])

    def spread(orbit_vec):
        full = np.zeros(N_ORBITS)
        full[active] = orbit_vec
        return full[orb]

    if d >= 2:
        parity = np.zeros(orb.size)
        odd_bits = np.array([bin(b).count("1") & 1 for b in range(1 << d)], dtype=bool)
        parity[corners] = np.where(odd_bits, -1.0, 1.0)
        parity *= n1_norm / np.linalg.norm(parity)
        n3 = rescale(spread(extras[0]), SAFEGUARD_SCALE)
        n4 = rescale(spread(extras[1]), SAFEGUARD_SCALE)
        return [n1, parity, n3, n4], (5, d - 1, 3, 3), (1.0, 1.0, SAFEGUARD_SCALE, SAFEGUARD_SCALE)

    # d == 1 (reference: quadrature.py:233-257): degree-3 null, a degree-1 null, an odd corner rule
    n2 = rescale(spread(extras[0]), SAFEGUARD_SCALE)
    vt1 = np.linalg.svd(table["1"][active][None, :])[2]
    deg1 = None
    for vec in vt1[1:]:
        got = _gram_schmidt([vec], [v0] + extras)
        if got:
            deg1 = got[0]
            break
    n3 = rescale(spread(deg1), SAFEGUARD_SCALE)
    odd = np.zeros(orb.size)
    odd[corners[0]], odd[corners[1]] = 1.0, -1.0
    n4 = odd * (SAFEGUARD_SCALE * n1_norm / np.linalg.norm(odd))
    return [n1, n2, n3, n4], (5, 3, 1, 0), (1.0, SAFEGUARD_SCALE, SAFEGUARD_SCALE, SAFEGUARD_SCALE)


_RULE_CACHE: dict = {}


def build_rule(d: int) -> RuleTable:
    """Rule table for dimension d (reference: quadrature.py:260-289).

    The table is immutable (read-only arrays), so one instance per dimension is shared: the
    moment solve and the SVD cost ~0.4 ms, more than a whole refine() of a short list on the device.
    """
    d = check_dimension(d)
    hit = _RULE_CACHE.get(d)
    if hit is None:
        hit = _RULE_CACHE[d] = _build_rule(d)
    return hit


def _build_rule(d: int) -> RuleTable:
    gen, orb = _point_set(d)
    table = _moment_table(d)
    w7, w5 = _degree7_and_5(d, table)
    nulls, degrees, scales = _null_rows(d, orb, table, w7, w5)
    weights = np.vstack([w7[orb]] + nulls)
    j = np.arange(d)
    axial = np.stack([1 + 2 * j, 2 + 2 * j, 1 + 2 * d + 2 * j, 2 + 2 * d + 2 * j], axis=1)
    return RuleTable(d, gen.shape[0], gen, weights,
                     np.array([1.0, LAMBDA2**2 / LAMBDA3**2]), axial, degrees, scales)


# --------------------------------------------------------------------------- device form
class OrbitRule(_Frozen):
    """What the kernels take by value: 7 offsets, 5x5 orbit weights, corner sign rule.

    offsets = (1/2, (1+l2)/2, (1-l2)/2, (1+l3)/2, (1-l3)/2, (1+l5)/2, (1-l5)/2) taken from the
    table's own generators via (g + 1.0) / 2.0, the reference's expression
    (quadrature.py:301).  weights[k][o] is rule k's weight on orbit o; rules whose
    corner weights alternate with bit parity carry corner_parity[k] = 1.
    """

    __slots__ = ("d", "f_eval", "offsets", "weights", "corner_parity", "split_weights",
                 "high_mask", "null_scales")


_ORBIT_CACHE: dict = {}


def orbit_form(rule: RuleTable) -> OrbitRule:
    """Compress a RuleTable, verifying it has the canonical fully symmetric layout.

    Raises ValueError for tables whose points or weights are not orbit-structured
    (the device kernels derive abscissae and weights from the point index).
    Verified forms are remembered per table object (tables are immutable).
    """
    hit = _ORBIT_CACHE.get(id(rule))
    if hit is not None and hit[0] is rule:
        return hit[1]
    out = _orbit_form(rule)
    if len(_ORBIT_CACHE) > 64:
        _ORBIT_CACHE.clear()
    _ORBIT_CACHE[id(rule)] = (rule, out)   # the strong reference keeps id(rule) from being reused
    return out


def _orbit_form(rule: RuleTable) -> OrbitRule:
    d = rule.d
    gen_ref, orb = _point_set(d)
    if rule.f_eval != gen_ref.shape[0] or rule.generators.shape != gen_ref.shape:
        raise ValueError("rule table does not have the degree-7 fully symmetric point count")
    g = rule.generators
    # distinct magnitudes come from the table itself, the sign/zero pattern must be canonical
    l2 = g[1, 0]
    l3 = g[1 + 2 * d, 0]
    l5 = g[rule.f_eval - (1 << d), 0]
    l4 = g[1 + 4 * d, 0] if d >= 2 else l3
    if l4 != l3:
        raise ValueError("rule table: pair-orbit magnitude differs from the l3 axial magnitude")
    expect = np.zeros_like(gen_ref)
    for lam_ref, lam in ((LAMBDA2, l2), (LAMBDA5, l5)):
        expect += np.where(np.abs(gen_ref) == lam_ref, np.sign(gen_ref) * lam, 0.0)
    expect += np.where(np.abs(gen_ref) == LAMBDA3, np.sign(gen_ref) * l3, 0.0)
    if not np.array_equal(expect, g):
        raise ValueError("rule table generators are not in the canonical fully symmetric order")

    w = rule.weights
    if w.shape != (5, rule.f_eval):
        raise ValueError("rule table needs five weight rows")
    ow = np.zeros((5, N_ORBITS))
    parity_flag = np.zeros(5, dtype=np.int32)
    corners = np.nonzero(orb == 4)[0]
    odd_bits = np.array([bin(b).count("1") & 1 for b in range(1 << d)], dtype=bool)
    for k in range(5):
        for o in range(N_ORBITS):
            rows = np.nonzero(orb == o)[0]
            if rows.size == 0:
                continue
            vals = w[k, rows]
            if np.all(vals == vals[0]):
                ow[k, o] = vals[0]
            elif o == 4 and np.array_equal(vals, np.where(odd_bits, -vals[0], vals[0])):
                ow[k, o] = vals[0]
                parity_flag[k] = 1
            else:
                raise ValueError(f"rule table row {k} is not constant on orbit {o}")
    if d == 1 and parity_flag.any():
        pass  # d = 1: the odd corner rule is the parity pattern on two corners
    expected_axial = np.stack([1 + 2 * np.arange(d), 2 + 2 * np.arange(d),
                               1 + 2 * d + 2 * np.arange(d), 2 + 2 * d + 2 * np.arange(d)], axis=1)
    if not np.array_equal(rule.axial_indices, expected_axial):
        raise ValueError("rule table axial_indices are not canonical")

    offs = np.array([(0.0 + 1.0) / 2.0, (l2 + 1.0) / 2.0, (-l2 + 1.0) / 2.0, (l3 + 1.0) / 2.0,
                     (-l3 + 1.0) / 2.0, (l5 + 1.0) / 2.0, (-l5 + 1.0) / 2.0])
    degrees = np.array(rule.null_degrees)
    scales = np.array(rule.null_scales, dtype=np.float64)
    out = OrbitRule.__new__(OrbitRule)
    out._put("d", d)
    out._put("f_eval", rule.f_eval)
    out._put("offsets", offs)
    out._put("weights", ow)
    out._put("corner_parity", parity_flag)
    out._put("split_weights", np.array(rule.split_weights, dtype=np.float64))
    out._put("high_mask", (degrees >= 5).astype(np.int32))
    out._put("null_scales", scales)
    return out


# --------------------------------------------------------------------------- small helpers
def eval_point(rule: RuleTable, region: Region, f_id: int) -> np.ndarray:
    """Generator row f_id mapped into the region (reference: quadrature.py:292-296)."""
    if not 0 <= f_id < rule.f_eval:
        raise IndexError(f"point index {f_id} out of range [0, {rule.f_eval})")
    return region.left + region.length * (rule.generators[f_id] + 1.0) / 2.0


def region_points(rule: RuleTable, lefts: np.ndarray, lengths: np.ndarray) -> np.ndarray:
    """(n, f_eval, d) abscissae: left + length * ((g + 1) / 2) (reference: quadrature.py:299-302).

    Index bookkeeping for error reports only; the kernels never materialise this."""
    offsets = (rule.generators + 1.0) / 2.0
    return lefts[:, None, :] + lengths[:, None, :] * offsets[None, :, :]


def apply_rules(f: Integrand, region: Region, rule: RuleTable):
    """Five rule values of one region and the stored evaluations
    (reference: quadrature.py:305-322): unlike the kernel path the sums here are a
    plain pairwise tree over ascending point index. Evaluated on the device."""
    from . import _native

    if rule.d != f.d:
        raise ValueError(f"rule dimension {rule.d} != integrand dimension {f.d}")
    values, fx = _native.apply_rules_single(f.device_spec(), rule, region.left, region.length)
    return RuleEstimates(values), fx
