"""m-Cubes: stratified importance-sampled Monte Carlo, on the B200.

Drop-in mirror of the reference's Monte Carlo layer (reference: pkg/src/parcube/mcubes.py):
`make_plan` (110-129), `mcubes_kernel` (268-308), `run` (332-382), `combine_iterations`
(311-329), the counter-based RNG helpers (31-74).  Sampling, bin accumulation and grid
refinement run in csrc/mcubes_kernels.cuh / csrc/mcubes_aux.cuh through the C-ABI.
"""

from __future__ import annotations

import math

import numpy as np

from . import _native
from .domain import Integrand, NonFiniteEvaluationError, _Frozen, check_dimension
from .execution import ExecConfig, GroupTaskError
from .vegas import BinContributions, GridRefineParams, VegasGrid, check_grid_shape, init_grid

_MASK64 = (1 << 64) - 1
_GOLDEN = 0x9E3779B97F4A7C15
_MIX1 = 0xBF58476D1CE4E5B9
_MIX2 = 0x94D049BB133111EB
_VARIANCE_FLOOR = 1e-30
RNG_KINDS = {"reference-hash": _native.RNG_REFERENCE_HASH, "philox": _native.RNG_PHILOX}


def _mix64_int(z: int) -> int:
    z &= _MASK64
    z = ((z ^ (z >> 30)) * _MIX1) & _MASK64
    z = ((z ^ (z >> 27)) * _MIX2) & _MASK64
    return z ^ (z >> 31)


def derive_seed(seed: int, label: int) -> int:
    """Child seed of iteration `label` (mcubes.py:58-60): integer bookkeeping on the host,
    the same function the device driver applies per iteration."""
    return _mix64_int((seed & _MASK64) + (int(label) * _GOLDEN))


def _uniform(seed: int, stream_id, counter, device=None) -> np.ndarray:
    """U[0,1) draws as a pure function of (seed, stream, counter) (mcubes.py:51-55), on the device."""
    shape = np.broadcast(np.asarray(stream_id), np.asarray(counter)).shape
    return _native.uniforms(int(seed), stream_id, counter, device=device).reshape(shape)


class RngStream:
    """Counter-based stream; state is (seed, stream_id, counter) (mcubes.py:63-74)."""

    def __init__(self, seed: int, stream_id: int, counter: int = 0):
        self.seed, self.stream_id, self.counter = int(seed), int(stream_id), int(counter)

    def take(self, n: int) -> np.ndarray:
        ctr = self.counter + np.arange(n, dtype=np.uint64)
        self.counter += int(n)
        return _uniform(self.seed, np.uint64(self.stream_id), ctr)


class McubesPlan(_Frozen):
    """Sub-cube partition geometry and per-thread batch layout (mcubes.py:77-107)."""

    __slots__ = ("d", "g", "m", "p", "s", "group_size", "n_requested")

    def __init__(self, d, g, m, p, s, group_size=128, n_requested=0):
        if m != g**d:
            raise ValueError("m must equal g^d")
        if p < 2:
            raise ValueError("p must be >= 2")
        if s < 1 or group_size < 1:
            raise ValueError("s and group_size must be >= 1")
        for k, v in zip(self.__slots__, (d, g, m, p, s, group_size, n_requested)):
            self._put(k, int(v))

    @property
    def n_actual(self) -> int:
        return self.m * self.p

    @property
    def n_threads(self) -> int:
        return -(-self.m // self.s)

    @property
    def n_groups(self) -> int:
        return -(-self.n_threads // self.group_size)


def make_plan(n, d: int, group_size: int = 128, target_groups: int = 256) -> McubesPlan:
    """g = largest integer with g^d <= n//2; p = max(2, round(n/g^d)); s batches the sub-cubes
    into ~target_groups work-groups (mcubes.py:110-129).  Plans are immutable: one instance per argument set."""
    key = (int(n), int(d), int(group_size), int(target_groups))
    hit = _PLAN_CACHE.get(key)
    if hit is None:
        if len(_PLAN_CACHE) > 256:
            _PLAN_CACHE.clear()
        hit = _PLAN_CACHE[key] = _make_plan(*key)
    return hit


_PLAN_CACHE: dict = {}


def _make_plan(n: int, d: int, group_size: int, target_groups: int) -> McubesPlan:
    d = check_dimension(d)
    n = int(n)
    if n < 2 ** (d + 1):
        raise ValueError(f"need n >= 2^(d+1) = {2 ** (d + 1)} to give every sub-cube 2 samples")
    half = n // 2
    g = max(1, int((n / 2.0) ** (1.0 / d)))
    while (g + 1) ** d <= half:
        g += 1
    while g > 1 and g**d > half:
        g -= 1
    m = g**d
    p = max(2, int(math.floor(n / m + 0.5)))
    s = max(1, -(-m // (group_size * target_groups)))
    return McubesPlan(d, g, m, p, s, group_size, n)


def cube_coordinates(cube_index, g: int, d: int) -> np.ndarray:
    """Base-g digits, axis 0 most significant (mcubes.py:132-140); index bookkeeping only."""
    rem = np.atleast_1d(np.asarray(cube_index, dtype=np.int64)).copy()
    out = np.empty((rem.size, d), dtype=np.int64)
    for j in range(d - 1, -1, -1):
        out[:, j] = rem % g
        rem //= g
    return out


def sample_cube(f: Integrand, cube_index: int, plan: McubesPlan, grid: VegasGrid, rng):
    """Draw p samples in one sub-cube; returns (S1, S2, bin_hits) (mcubes.py:143-164).

    `rng` is duck-typed like the reference's: anything with `take(n) -> n uniforms in [0, 1)`
    (an `RngStream`, or a table-backed object -- the reference's second injection route,
    SURVEY.md section 0.1).  The stratified map, the grid transform, the integrand and the two
    `tree_sum`s run on the device (pcb_mcubes_sample_cube); `bin_hits` is the reference's list of
    (bin ids of sample k, v_k^2)."""
    if not 0 <= cube_index < plan.m:
        raise IndexError(f"cube index {cube_index} out of range [0, {plan.m})")
    if plan.d != grid.d or plan.d != f.d:
        raise ValueError("plan, grid, and integrand dimensions must agree")
    u = np.asarray(rng.take(plan.p * plan.d), dtype=np.float64).reshape(plan.p, plan.d)
    try:
        s1, s2, bins, weights = _native.mcubes_sample_cube(f.device_spec(), plan, grid.boundaries, int(cube_index), u)
    except _native.NonFiniteStatus as exc:
        raise NonFiniteEvaluationError(exc.point, exc.value) from None
    return s1, s2, [(bins[k], float(weights[k])) for k in range(plan.p)]


def update_variance(s1: float, s2: float, p: int, m: int):
    """Per-cube estimate and clamped variance from sample sums (mcubes.py:167-179).
    Three scalars; the V-Sample kernel evaluates the same expressions per sub-cube."""
    if p < 2:
        raise ValueError("p must be >= 2")
    est = s1 / (p * m)
    raw = (s2 - s1 * s1 / p) / (p * (p - 1) * m * m)
    return (est, 0.0, True) if raw < 0.0 else (est, raw, False)


class McubesIterationResult(_Frozen):
    """mcubes.py:182-192."""

    __slots__ = ("integral", "variance", "contributions", "n_samples", "clamp_events")

    def __init__(self, integral, variance, contributions, n_samples, clamp_events):
        if variance < 0:
            raise ValueError("variance must be >= 0")
        for k, v in zip(self.__slots__, (float(integral), float(variance), contributions, int(n_samples),
                                         int(clamp_events))):
            self._put(k, v)


class MonteCarloResult(_Frozen):
    """Weighted combination of the per-iteration estimates (mcubes.py:195-207)."""

    __slots__ = ("estimate", "errorest", "chi2_per_dof", "iterations", "plan")

    def __init__(self, estimate, errorest, chi2_per_dof, iterations, plan):
        if errorest < 0 or chi2_per_dof < 0:
            raise ValueError("errorest and chi2_per_dof must be >= 0")
        for k, v in zip(self.__slots__, (estimate, errorest, chi2_per_dof, iterations, plan)):
            self._put(k, v)


def _device_of(exec_cfg):
    return None if exec_cfg is None else exec_cfg.device


def _raise_nonfinite(exc: _native.NonFiniteStatus, plan: McubesPlan):
    cube = int(exc.region_index)
    cause = NonFiniteEvaluationError(exc.point, exc.value, region_index=cube)
    raise GroupTaskError(cube // (plan.s * plan.group_size), cause) from cause


def _table(d, n_bins, c) -> BinContributions:
    """A BinContributions over `c` itself when it is a float64 (d, n_bins) array the caller hands over (the per-iteration
    slices of a run's table block), else over a copy."""
    out = BinContributions.__new__(BinContributions)
    out.d, out.n_bins = int(d), int(n_bins)
    if isinstance(c, np.ndarray) and c.dtype == np.float64 and c.shape == (d, n_bins) and c.flags.writeable:
        out.c = c
    else:
        out.c = np.array(c, dtype=np.float64).reshape(d, n_bins)
    return out


def mcubes_kernel(f: Integrand, plan: McubesPlan, grid: VegasGrid, exec_cfg: ExecConfig | None = None, seed: int = 0,
                  squared_weighted: bool = True, rng: str = "reference-hash", injected_uniforms=None,
                  thread_range=None) -> McubesIterationResult:
    """One sampling pass over all sub-cubes (mcubes.py:268-308).

    Extensions (keyword-only in spirit): `rng` selects the reference's counter hash (default,
    bit-identical draws) or Philox4x32-10; `injected_uniforms`, an array of m*p*d values indexed
    (cube*p + k)*d + j, replaces the generator (the reference's `_uniform` monkeypatch hook);
    `thread_range=(t0, t1)` samples only that shard of logical threads (multi-GPU).
    """
    if plan.d != grid.d or plan.d != f.d:
        raise ValueError("plan, grid, and integrand dimensions must agree")
    kind = _native.RNG_INJECTED if injected_uniforms is not None else RNG_KINDS[rng]
    try:
        it, contrib, _ = _native.mcubes_sample(f.device_spec(), plan, grid.boundaries, seed, kind, injected_uniforms,
                                               squared_weighted, thread_range, device=_device_of(exec_cfg))
    except _native.NonFiniteStatus as exc:
        _raise_nonfinite(exc, plan)
    return McubesIterationResult(it.integral, it.variance, _table(plan.d, grid.n_bins, contrib), it.n_samples,
                                 it.clamp_events)


def combine_iterations(iteration_results: list) -> tuple[float, float, float]:
    """Inverse-variance weighted mean, its standard deviation and chi2/dof (mcubes.py:311-329).
    A handful of scalars per run; the device driver applies the same formulas per iteration."""
    if not iteration_results:
        raise ValueError("need at least one iteration")
    w = [1.0 / max(r.variance, _VARIANCE_FLOOR) for r in iteration_results]
    wsum = sum(w)
    est = sum(wi * r.integral for wi, r in zip(w, iteration_results)) / wsum
    err = wsum**-0.5
    chi2 = 0.0
    if len(iteration_results) > 1:
        chi2 = sum(wi * (r.integral - est) ** 2 for wi, r in zip(w, iteration_results)) / (len(iteration_results) - 1)
    return float(est), float(err), float(chi2)


def run(f: Integrand, n, d: int, iterations: int, params: GridRefineParams | None = None, seed: int = 0,
        exec_cfg: ExecConfig | None = None, n_bins: int = 500, group_size: int = 128, target_groups: int = 256,
        adapt: bool = True, progress=None, rel_tol: float | None = None, rng: str = "reference-hash",
        abs_tol: float | None = None) -> MonteCarloResult:
    """Iterate {sample; refine grid} and combine the iteration estimates (mcubes.py:332-382).

    The loop is device-resident (grid, contribution table and partial sums never leave HBM);
    the host receives one (integral, variance) pair per iteration.  `rel_tol` (extension,
    default None = reference behaviour) stops after the first iteration whose cumulative
    errorest/|estimate| is <= rel_tol; `iterations` is then the maximum.  `abs_tol` (epsabs) widens the
    target to max(abs_tol, rel_tol*|estimate|); either one alone may be given.
    """
    if iterations < 1:
        raise ValueError("iterations must be >= 1")
    if f.d != d:
        raise ValueError("plan, grid, and integrand dimensions must agree")
    params = params or GridRefineParams()
    plan = make_plan(n, d, group_size=group_size, target_groups=target_groups)
    check_grid_shape(d, n_bins)  # argument validation as in the reference's init_grid
    try:
        its, contribs, _final_b, _secs = _native.mcubes_run(
            f.device_spec(), plan, n_bins, iterations, seed, RNG_KINDS[rng], adapt, params.alpha, params.smoothing,
            0.0 if rel_tol is None else float(rel_tol), progress, device=_device_of(exec_cfg),
            abs_tol=0.0 if abs_tol is None else float(abs_tol))
    except _native.NonFiniteStatus as exc:
        _raise_nonfinite(exc, plan)
    history = [McubesIterationResult(r.integral, r.variance, _table(d, n_bins, contribs[i]), r.n_samples, r.clamp_events)
               for i, r in enumerate(its)]
    estimate, errorest, chi2 = combine_iterations(history)
    return MonteCarloResult(estimate, errorest, chi2, history, plan)
