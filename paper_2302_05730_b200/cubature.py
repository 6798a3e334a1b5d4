"""PAGANI: per-region rule evaluation and the refinement driver, on the B200.

Drop-in mirror of the reference's cubature layer (reference: pkg/src/parcube/pagani.py):
`pagani_kernel` (pagani.py:227-257) and `refine` (pagani.py:300-391) keep their signatures,
result types, stop reasons and error behaviour; the arithmetic runs in
csrc/pagani_eval.cuh / csrc/pagani_driver.cuh through the C-ABI.
"""

from __future__ import annotations

import json

import numpy as np

from . import _native
from .domain import (DEFAULT_REGION_CAP, BudgetExceededError, Integrand, NonFiniteEvaluationError, Region,
                     RegionEstimates, RegionList, _Frozen)
from .execution import ExecConfig, GroupTaskError
from .rules import RuleEstimates, RuleTable, build_rule, orbit_form

ERR_TWO_LEVEL = "two-level"
ERR_MAX_NULL = "max-null"
ERR_MAX_PAIRWISE = "max-pairwise"
TWO_LEVEL_SAFETY = 10.0  # pagani.py:40


class PaganiConfig(_Frozen):
    """Tolerance, budgets and schedule shape (pagani.py:44-69).

    `abs_tol` (epsabs, an extension; 0 = the reference) widens the target to
    max(abs_tol, rel_tol*|estimate|), for the stop test and for the split threshold alike.
    `group_size` (the strided schedule width, any G >= 1 as in the reference) changes floating-point
    association only; `chunk` is accepted for compatibility and only affects which group id a
    non-finite report carries.
    """

    __slots__ = ("rel_tol", "max_iterations", "group_size", "region_cap", "initial_regions", "err_mode",
                 "rel_floor", "chunk", "abs_tol")

    def __init__(self, rel_tol: float = 1e-3, max_iterations: int = 50, group_size: int = 64,
                 region_cap: int = DEFAULT_REGION_CAP, initial_regions: int = 1024, err_mode: str = ERR_TWO_LEVEL,
                 rel_floor: float = 1e-15, chunk: int = 512, abs_tol: float = 0.0):
        if rel_tol <= 0:
            raise ValueError("rel_tol must be > 0")
        if not abs_tol >= 0:
            raise ValueError("abs_tol must be >= 0")
        if group_size < 1 or chunk < 1:
            raise ValueError("group_size and chunk must be >= 1")
        if err_mode not in (ERR_TWO_LEVEL, ERR_MAX_NULL, ERR_MAX_PAIRWISE):
            raise ValueError(f"unknown err_mode {err_mode!r}")
        for k, v in (("rel_tol", float(rel_tol)), ("max_iterations", int(max_iterations)),
                     ("group_size", int(group_size)), ("region_cap", int(region_cap)),
                     ("initial_regions", int(initial_regions)), ("err_mode", err_mode),
                     ("rel_floor", float(rel_floor)), ("chunk", int(chunk)), ("abs_tol", float(abs_tol))):
            self._put(k, v)


class RegionRecord(_Frozen):
    """Evaluation summary of one region (pagani.py:72-86)."""

    __slots__ = ("region", "volume", "integral", "error", "split_axis")

    def __init__(self, region, volume, integral, error, split_axis):
        if error < 0:
            raise ValueError("error must be >= 0")
        if not 0 <= split_axis < region.d:
            raise ValueError("split_axis out of range")
        for k, v in zip(self.__slots__, (region, volume, integral, error, split_axis)):
            self._put(k, v)


class IntegralResult(_Frozen):
    """pagani.py:89-101."""

    __slots__ = ("estimate", "errorest", "iterations", "regions_processed", "converged", "history", "reason")

    def __init__(self, estimate, errorest, iterations, regions_processed, converged, history=None, reason=""):
        if errorest < 0:
            raise ValueError("errorest must be >= 0")
        for k, v in zip(self.__slots__, (estimate, errorest, iterations, regions_processed, converged,
                                         list(history or []), reason)):
            self._put(k, v)


def _device_of(exec_cfg):
    return None if exec_cfg is None else exec_cfg.device


def _raise_nonfinite(exc: _native.NonFiniteStatus, chunk: int):
    cause = NonFiniteEvaluationError(exc.point, exc.value, region_index=int(exc.region_index))
    raise GroupTaskError(int(exc.region_index) // chunk, cause) from cause


def pagani_kernel(f: Integrand, regions: RegionList, rule: RuleTable, exec_cfg: ExecConfig | None = None,
                  cfg: PaganiConfig | None = None) -> RegionEstimates:
    """Integral, error estimate and split axis of every region (pagani.py:227-257)."""
    if regions.n == 0:
        raise ValueError("region list is empty")
    if rule.d != regions.d or rule.d != f.d:
        raise ValueError("rule, regions, and integrand dimensions must agree")
    cfg = cfg or PaganiConfig()
    spec = f.device_spec()
    try:
        i, e, k = _native.pagani_evaluate(spec, orbit_form(rule), cfg, regions.lefts, regions.lengths,
                                          device=_device_of(exec_cfg))
    except _native.NonFiniteStatus as exc:
        _raise_nonfinite(exc, cfg.chunk)
    return RegionEstimates(integrals=i, errors=e, split_axes=k)


def evaluate_region(f: Integrand, region: Region, rule: RuleTable, cfg: PaganiConfig | None = None) -> RegionRecord:
    """Single-region wrapper around the kernel path (pagani.py:260-270)."""
    est = pagani_kernel(f, RegionList(region.left[None, :], region.length[None, :]), rule, None, cfg)
    return RegionRecord(region, float(np.prod(region.length)), float(est.integrals[0]), float(est.errors[0]),
                        int(est.split_axes[0]))


def find_max_err(est: RuleEstimates, volume: float, rel_floor: float = 1e-15, mode: str = ERR_TWO_LEVEL,
                 rule: RuleTable | None = None) -> float:
    """Error estimate of one region from its five rule values (pagani.py:135-154; modes 104-132).

    Five scalars; evaluated inline (the kernels compute the same expression per region)."""
    v = est.values
    if not np.all(np.isfinite(v)):
        raise NonFiniteEvaluationError(np.full(1, np.nan), float(v[np.argmax(~np.isfinite(v))]))
    if mode == ERR_TWO_LEVEL and rule is None:
        raise ValueError("two-level mode needs the rule table for null metadata")
    nulls = [abs(float(x)) for x in v[1:5]]
    if mode == ERR_MAX_NULL:
        err = max(nulls)
    elif mode == ERR_MAX_PAIRWISE:
        err = max(abs(float(a) - float(b)) for a in v[1:5] for b in v[1:5])
    elif mode == ERR_TWO_LEVEL:
        high = [deg >= 5 for deg in rule.null_degrees]
        e_high = max(n for n, h in zip(nulls, high) if h)
        e_low = max(n / s for n, h, s in zip(nulls, high, rule.null_scales) if not h)
        corr = TWO_LEVEL_SAFETY * e_high / e_low if e_low > 0 else 1.0
        err = e_high * min(1.0, corr)
    else:
        raise ValueError(f"unknown err_mode {mode!r}")
    return max(err, rel_floor * abs(float(v[0])))


def compute_split_axis(stored_evals, rule: RuleTable, d: int) -> int:
    """Axis with the largest fourth-difference indicator, lowest index on ties (pagani.py:157-172)."""
    fx = np.asarray(stored_evals, dtype=np.float64)
    if d == 1:
        return 0
    best, best_val = 0, -1.0
    c0, c1 = (float(c) for c in rule.split_weights)
    for j in range(d):
        a0, a1, b0, b1 = (float(fx[i]) for i in rule.axial_indices[j])
        ind = abs(c0 * (a0 + a1 - 2.0 * float(fx[0])) - c1 * (b0 + b1 - 2.0 * float(fx[0])))
        if ind > best_val:
            best, best_val = j, ind
    return best


def refine(f: Integrand, cfg: PaganiConfig | None = None, exec_cfg: ExecConfig | None = None,
           rule: RuleTable | None = None, progress=None) -> IntegralResult:
    """Bisect regions until errorest <= rel_tol*|estimate| (pagani.py:300-391).

    The whole loop -- uniform tiling, evaluation, tree sums, threshold filter, stable
    compaction and bisection -- stays on the device; the host sees one small record per
    iteration, delivered to `progress` before the convergence test exactly like the reference.
    """
    cfg = cfg or PaganiConfig()
    rule = rule or build_rule(f.d)
    if rule.d != f.d:
        raise ValueError("rule, regions, and integrand dimensions must agree")
    spec = f.device_spec()
    try:
        res, history = _native.pagani_refine(spec, orbit_form(rule), cfg, progress, device=_device_of(exec_cfg))
    except _native.NonFiniteStatus as exc:
        _raise_nonfinite(exc, cfg.chunk)
    except _native.BudgetStatus as exc:
        raise BudgetExceededError(str(exc)) from None
    return IntegralResult(estimate=res.estimate, errorest=res.errorest, iterations=res.iterations,
                          regions_processed=int(res.regions_processed), converged=bool(res.converged),
                          history=history, reason=_native.STOP_REASONS[res.reason])


def progress_to_stream(stream):
    """Per-iteration records as line-delimited JSON (pagani.py:394-400)."""

    def emit(record):
        stream.write(json.dumps(record) + "\n")

    return emit
