"""Multi-GPU drivers: one process per GPU, torch.distributed for the plumbing.

m-Cubes shards the logical threads (hence the sub-cubes) across ranks on work-group
boundaries.  Every draw is uniform(seed, thread, counter) (mcubes.py:224-232), so any
partition reproduces the reference's sample set.  Per iteration the ranks exchange
  * the per-work-group (I, Var) partials -- all-gathered in group order, then every rank
    finishes the reference's pair tree (mcubes.py:292-293): the result is bit-identical for
    any GPU count;
  * the (d x n_bins) contribution table and the clamp counter -- all-reduced (sum);
and then run the identical grid refinement.  Messages are <= 32 KB + 4 KB: latency-bound,
NCCL over NVLink/NVSwitch (or gloo on CPU in the tests).

The compute backend is injectable so the CPU test-suite can drive this logic with the
oracle under gloo; the product backend below is the CUDA library and nothing else.
"""

from __future__ import annotations

import math

import numpy as np

from . import _native
from .stratified import (McubesIterationResult, MonteCarloResult, _table, combine_iterations, derive_seed, make_plan)
from .vegas import GridRefineParams, init_grid


class CudaBackend:
    """Per-rank compute on the local B200 through the C-ABI."""

    def __init__(self, device=None):
        self.device = device

    def sample(self, spec, plan, boundaries, seed, thread_range, rng_kind):
        it, contrib, partials = _native.mcubes_sample(spec, plan, boundaries, seed, rng_kind, None, True, thread_range,
                                                      want_group_partials=True, device=self.device)
        return partials, contrib, int(it.clamp_events)

    def refine(self, boundaries, contrib, alpha, smoothing):
        return _native.grid_refine(boundaries, contrib, alpha, smoothing, device=self.device)

    def tree_sum(self, values):
        return _native.tree_sum_1d(values, device=self.device)


class Comm:
    """Minimal collective surface over torch.distributed (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None, device=None):
        import torch
        import torch.distributed as dist

        self._torch, self._dist, self.group = torch, dist, group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        backend = dist.get_backend(group)
        self.device = torch.device("cuda", device if device is not None else torch.cuda.current_device()) \
            if backend == "nccl" else torch.device("cpu")

    def _to(self, a):
        return self._torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(self.device)

    def allreduce_sum(self, a: np.ndarray) -> np.ndarray:
        t = self._to(a)
        self._dist.all_reduce(t, op=self._dist.ReduceOp.SUM, group=self.group)
        return t.cpu().numpy()

    def allgather(self, a: np.ndarray) -> list:
        """Gather equally-shaped float64 arrays from every rank, in rank order."""
        t = self._to(a)
        out = [self._torch.empty_like(t) for _ in range(self.world)]
        self._dist.all_gather(out, t, group=self.group)
        return [o.cpu().numpy() for o in out]

    def barrier(self):
        self._dist.barrier(group=self.group)


def group_shards(n_groups: int, world: int) -> list:
    """Contiguous, near-equal ranges of work-groups per rank: [(g0, g1), ...]."""
    return [(n_groups * r // world, n_groups * (r + 1) // world) for r in range(world)]


def mcubes_iteration_sharded(spec, plan, boundaries, seed, comm, backend, rng_kind=_native.RNG_REFERENCE_HASH):
    """One V-Sample pass split over comm.world ranks. Returns (integral, variance, contributions, clamps)."""
    shards = group_shards(plan.n_groups, comm.world)
    g0, g1 = shards[comm.rank]
    width = max(b - a for a, b in shards)
    local = np.zeros((width, 2))
    contrib = np.zeros((plan.d, boundaries.shape[1] - 1))
    clamps = 0
    if g1 > g0:
        t0, t1 = g0 * plan.group_size, min(g1 * plan.group_size, plan.n_threads)
        partials, contrib, clamps = backend.sample(spec, plan, boundaries, seed, (t0, t1), rng_kind)
        local[: g1 - g0] = partials
    gathered = comm.allgather(local)
    ordered = np.concatenate([gathered[r][: b - a] for r, (a, b) in enumerate(shards)])
    integral = backend.tree_sum(ordered[:, 0])
    variance = max(backend.tree_sum(ordered[:, 1]), 0.0)
    packed = comm.allreduce_sum(np.concatenate([contrib.ravel(), [float(clamps)]]))
    return integral, variance, packed[:-1].reshape(contrib.shape), int(round(packed[-1]))


def mcubes_run_sharded(f, n, d, iterations, comm, backend=None, params=None, seed=0, n_bins=500, group_size=128,
                       target_groups=256, adapt=True, progress=None, rel_tol=None, rng="reference-hash"):
    """mcubes.run (mcubes.py:332-382) with the sub-cubes sharded over comm.world GPUs.

    Every rank returns the same MonteCarloResult; (integral, variance) per iteration are
    bit-identical to the single-GPU run, the contribution tables agree to summation order.
    """
    from .stratified import RNG_KINDS

    if iterations < 1:
        raise ValueError("iterations must be >= 1")
    backend = backend or CudaBackend()
    params = params or GridRefineParams()
    plan = make_plan(n, d, group_size=group_size, target_groups=target_groups)
    boundaries = np.array(init_grid(d, n_bins).boundaries)
    spec = f.device_spec() if hasattr(f, "device_spec") else f
    history = []
    for it in range(iterations):
        integral, variance, contrib, clamps = mcubes_iteration_sharded(
            spec, plan, boundaries, derive_seed(seed, it), comm, backend, RNG_KINDS[rng])
        history.append(McubesIterationResult(integral, variance, _table(d, n_bins, contrib), plan.n_actual, clamps))
        if adapt:
            boundaries = backend.refine(boundaries, contrib, params.alpha, params.smoothing)
        est, err, chi2 = combine_iterations(history)
        if progress is not None:
            progress({"iteration": it, "estimate": est, "errorest": err, "chi2_per_dof": chi2,
                      "iter_integral": integral, "iter_sd": math.sqrt(variance)})
        if rel_tol is not None and err <= rel_tol * abs(est):
            break
    est, err, chi2 = combine_iterations(history)
    return MonteCarloResult(est, err, chi2, history, plan)
