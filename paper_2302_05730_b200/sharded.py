"""Multi-GPU drivers: one process per GPU, torch.distributed for the plumbing.

PAGANI shards the ordered region list in contiguous slices.  Per iteration the ranks exchange
  * tree-sum pieces of the active (and just-retired) integrals/errors: each rank reduces the
    1024-aligned blocks of the GLOBAL index space that lie inside its slice and ships the ragged
    head/tail elements raw, so every rank finishes engine.tree_sum's pair tree bit-identically
    for any GPU count (estimate and errorest drive the classification, pagani.py:336-365);
  * the split counts (region-cap test is global, pagani.py:367) and, only when nothing exceeds
    its budget, the maximum error;
  * region rows that change owner when the children are rebalanced to equal contiguous slices
    (only rows that move travel; config 3 doubles every slice uniformly and moves nothing).

m-Cubes shards the logical threads (hence the sub-cubes) across ranks on work-group
boundaries.  Every draw is uniform(seed, thread, counter) (mcubes.py:224-232), so any
partition reproduces the reference's sample set.  Per iteration the ranks exchange
  * the per-work-group (I, Var) partials -- all-gathered in group order, then every rank
    finishes the reference's pair tree (mcubes.py:292-293): the result is bit-identical for
    any GPU count;
  * the (d x n_bins) contribution table and the clamp counter -- all-reduced (sum);
and then run the identical grid refinement.  Messages are <= 32 KB + 4 KB: latency-bound,
NCCL over NVLink/NVSwitch (or gloo on CPU in the tests).

Product path: the collectives run on DEVICE buffers of the library, on the library's own stream
(torch.cuda.ExternalStream), so nothing is staged through the host and the m-Cubes loop stays
device-resident -- per iteration one all-gather of a (2*ceil(G/W)+2)-double row and one all-reduce
of the table, enqueued between `pass` and `finish` of pcb_mcubes_shard_*; the host enqueues
iteration it+1 before it polls the record of iteration it.  PAGANI: one all-gather of the packed
tree pieces and one of (split count, max error) per iteration, region rows move rank-to-rank
with NCCL send/recv straight between the device lists.

The compute backend is injectable so the CPU test-suite can drive the partition logic with the
oracle under gloo (host arrays); the product backend is the CUDA library and nothing else.
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

    # ---- tensor-level collectives: operate in place on the tensors given (device buffers of the library under NCCL,
    #      CPU tensors under gloo), ordered on the current torch stream, no host staging
    def all_gather_into(self, out, inp):
        """out[r*n:(r+1)*n] = inp of rank r (n = inp.numel()); out may alias inp at its own slot."""
        if self.world == 1 and out.data_ptr() == inp.data_ptr() and self._dist.get_backend(self.group) != "nccl":
            return
        self._dist.all_gather_into_tensor(out, inp, group=self.group)

    def all_reduce_sum_(self, t):
        self._dist.all_reduce(t, op=self._dist.ReduceOp.SUM, group=self.group)

    def all_reduce_max_(self, t):
        self._dist.all_reduce(t, op=self._dist.ReduceOp.MAX, group=self.group)

    def exchange_tensors(self, sends: dict, recvs: dict):
        """Point-to-point exchange of device tensors: sends[r] = tensor for rank r, recvs[r] = preallocated tensor to
        fill from rank r (NCCL send/recv, one batched group)."""
        dist = self._dist
        ops = [dist.P2POp(dist.isend, t, r, group=self.group) for r, t in sends.items()]
        ops += [dist.P2POp(dist.irecv, t, r, group=self.group) for r, t in recvs.items()]
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()

    def exchange_rows(self, sends: dict, recvs: dict, d: int) -> dict:
        """Point-to-point exchange of region rows: sends[r] = (lefts, lengths) for rank r, recvs[r] = row
        count expected from rank r.  Returns {r: (lefts, lengths)}.  (NCCL send/recv on GPUs, gloo on CPU.)"""
        torch, dist = self._torch, self._dist
        ops, bufs = [], {}
        for r, (lefts, lengths) in sends.items():
            t = self._to(np.stack([lefts, lengths]))
            ops.append(dist.P2POp(dist.isend, t, r, group=self.group))
        for r, n in recvs.items():
            bufs[r] = torch.empty((2, n, d), dtype=torch.float64, device=self.device)
            ops.append(dist.P2POp(dist.irecv, bufs[r], r, group=self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        return {r: (b[0].cpu().numpy(), b[1].cpu().numpy()) for r, b in bufs.items()}


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


def _device_tensor(view, device):
    import torch

    return torch.as_tensor(view, device=torch.device("cuda", device))


def _mcubes_run_device(spec, plan, iterations, comm, params, seed, n_bins, adapt, progress, rel_tol, abs_tol, rng_kind,
                       device, force_collectives, ctx=None):
    """The product path: device-resident loop, collectives on the library's buffers and stream."""
    import torch

    run = _native.McubesShardRun(spec, plan, n_bins, iterations, seed, rng_kind, adapt, params.alpha, params.smoothing,
                                 0.0 if rel_tol is None else float(rel_tol), 0.0 if abs_tol is None else float(abs_tol),
                                 True, comm.rank, comm.world, device=device, ctx=ctx)
    dev = run.ctx.device
    row, gathered, table = (_device_tensor(v, dev) for v in (run.row, run.gathered, run.table))
    collect = comm.world > 1 or force_collectives
    history, records = [], []

    def enqueue(it):
        run.enqueue_pass(it)
        if collect:
            comm.all_gather_into(gathered, row)
            comm.all_reduce_sum_(table)
        run.enqueue_finish(it)

    with torch.cuda.stream(torch.cuda.ExternalStream(run.stream, device=torch.device("cuda", dev))):
        enqueue(0)
        enqueued = 1
        for it in range(iterations):
            if enqueued < iterations:      # the device never waits for the host: iteration it+1 is already queued
                enqueue(enqueued)
                enqueued += 1
            rec, stop = run.wait(it)
            records.append((rec.integral, rec.variance, int(rec.n_samples), int(rec.clamp_events)))
            if progress is not None:
                est, err, chi2 = combine_iterations([McubesIterationResult(i, v, None, ns, c) for i, v, ns, c in records])
                progress({"iteration": it, "estimate": est, "errorest": err, "chi2_per_dof": chi2,
                          "iter_integral": rec.integral, "iter_sd": math.sqrt(rec.variance)})
            if stop:
                break
        contribs, _final_b, _secs = run.end(len(records))
    for k, (i, v, ns, c) in enumerate(records):
        history.append(McubesIterationResult(i, v, _table(plan.d, n_bins, contribs[k]), ns, c))
    est, err, chi2 = combine_iterations(history)
    return MonteCarloResult(est, err, chi2, history, plan)


def mcubes_run_sharded(f, n, d, iterations, comm, backend=None, params=None, seed=0, n_bins=500, group_size=128,
                       target_groups=256, adapt=True, progress=None, rel_tol=None, rng="reference-hash", abs_tol=None,
                       device=None, force_collectives=False, ctx=None):
    """mcubes.run (mcubes.py:332-382) with the sub-cubes sharded over comm.world GPUs.

    Every rank returns the same MonteCarloResult.  (integral, variance) of iteration 0 are bit-identical to the
    single-GPU run for any GPU count (same samples, same per-group partials, same group-order tree); the
    contribution tables agree to summation order (an all-reduce instead of the single-GPU merge order), so the
    refined grids and hence iterations >= 1 agree to rounding.  A non-finite sample raises the same
    GroupTaskError on every rank (the flag travels in the gathered rows).

    `backend=None` is the product path (CUDA library, device-resident loop, collectives on device buffers; `ctx`
    selects the library context, default the process-wide one of `device`; `force_collectives` issues the
    collectives even for one rank); an injected backend (the CPU test-suite's oracle) takes the host-array path below.
    """
    from .stratified import RNG_KINDS, _raise_nonfinite

    if iterations < 1:
        raise ValueError("iterations must be >= 1")
    params = params or GridRefineParams()
    plan = make_plan(n, d, group_size=group_size, target_groups=target_groups)
    spec = f.device_spec() if hasattr(f, "device_spec") else f
    if backend is None:
        try:
            return _mcubes_run_device(spec, plan, iterations, comm, params, seed, n_bins, adapt, progress, rel_tol, abs_tol,
                                      RNG_KINDS[rng], device, force_collectives, ctx)
        except _native.NonFiniteStatus as exc:
            _raise_nonfinite(exc, plan)
    boundaries = np.array(init_grid(d, n_bins).boundaries)
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
        if (rel_tol is not None or abs_tol is not None) and err <= max(abs_tol or 0.0, (rel_tol or 0.0) * abs(est)):
            break
    est, err, chi2 = combine_iterations(history)
    return MonteCarloResult(est, err, chi2, history, plan)


# =============================================================================== PAGANI
TREE_SPAN = 1024


def global_tree_sum(comm, backend_tree_sum, pieces, counts):
    """Finish engine.tree_sum over the concatenation of all ranks' arrays.

    `pieces` = (head_vals, block_sums, tail_vals) of this rank for head = (-offset) mod 1024;
    `counts` = element count of every rank.  Every rank returns the same float, bit-identical to a
    single-device tree over the concatenated array (blocks of 2^10, then a pair tree over the block sums).
    """
    head, blocks, tail = pieces
    width = max(1, max(c // TREE_SPAN + 1 for c in counts))
    packed = np.zeros(3 + 2 * TREE_SPAN + width)
    packed[0], packed[1], packed[2] = len(head), len(blocks), len(tail)
    packed[3:3 + len(head)] = head
    packed[3 + TREE_SPAN:3 + TREE_SPAN + len(tail)] = tail
    packed[3 + 2 * TREE_SPAN:3 + 2 * TREE_SPAN + len(blocks)] = blocks
    sums, carry = [], []
    for part in comm.allgather(packed):
        nh, nb, nt = int(part[0]), int(part[1]), int(part[2])
        carry.extend(part[3:3 + nh])
        if len(carry) == TREE_SPAN:
            sums.append(backend_tree_sum(np.array(carry)))
            carry = []
        sums.extend(part[3 + 2 * TREE_SPAN:3 + 2 * TREE_SPAN + nb])
        if nt:
            assert not carry, "a tail can only follow a completed block"
            carry = list(part[3 + TREE_SPAN:3 + TREE_SPAN + nt])
    if carry:
        sums.append(backend_tree_sum(np.array(carry)))   # last, zero-padded block
    return backend_tree_sum(np.array(sums)) if sums else 0.0


def _offsets(counts):
    out, run = [], 0
    for c in counts:
        out.append(run)
        run += c
    return out, run


def _even_ranges(total, world):
    return [(total * r // world, total * (r + 1) // world) for r in range(world)]


def rebalance(comm, shard, counts):
    """Move region rows so that rank r owns global indices [N*r/W, N*(r+1)/W) of the ordered list."""
    offsets, total = _offsets(counts)
    me, world = comm.rank, comm.world
    target = _even_ranges(total, world)
    my0, my1 = offsets[me], offsets[me] + counts[me]
    t0, t1 = target[me]
    if all(offsets[r] == target[r][0] and counts[r] == target[r][1] - target[r][0] for r in range(world)):
        return counts
    d = shard.d
    sends = {}
    for r in range(world):           # my rows that belong to rank r
        a, b = max(my0, target[r][0]), min(my1, target[r][1])
        if r != me and a < b:
            sends[r] = shard.export(a - my0, b - my0)
    recvs = {}
    for r in range(world):           # rows of rank r that belong to me
        a, b = max(offsets[r], t0), min(offsets[r] + counts[r], t1)
        if r != me and a < b:
            recvs[r] = b - a
    got = comm.exchange_rows(sends, recvs, d)
    keep0, keep1 = max(my0, t0), min(my1, t1)
    front = [got[r] for r in sorted(got) if r < me]
    back = [got[r] for r in sorted(got) if r > me]
    cat = lambda parts: (np.concatenate([p[0] for p in parts]), np.concatenate([p[1] for p in parts])) if parts else None
    if keep0 < keep1:
        shard.rebuild(keep0 - my0, keep1 - my0, cat(front), cat(back))
    else:
        shard.rebuild(0, 0, cat(front), cat(back))
    return [b - a for a, b in target]


def rebalance_device(comm, shard, counts, device):
    """rebalance() with the rows travelling device to device: slices of the local structure-of-arrays list are sent
    as [2][d][n] blocks (lefts, lengths) and the new list is assembled on the device (pcb_pagani_shard_rebuild_dev)."""
    import torch

    offsets, total = _offsets(counts)
    me, world = comm.rank, comm.world
    target = _even_ranges(total, world)
    if all(offsets[r] == target[r][0] and counts[r] == target[r][1] - target[r][0] for r in range(world)):
        return counts
    my0, my1 = offsets[me], offsets[me] + counts[me]
    t0, t1 = target[me]
    d = shard.d
    sends, recvs = {}, {}
    if my1 > my0:
        lv, hv, _n, ld = shard.list_dev()
        lefts = _device_tensor(lv, device).view(d, ld)
        lengths = _device_tensor(hv, device).view(d, ld)
    for r in range(world):           # my rows that belong to rank r
        a, b = max(my0, target[r][0]), min(my1, target[r][1])
        if r != me and a < b:
            sends[r] = torch.stack([lefts[:, a - my0:b - my0], lengths[:, a - my0:b - my0]]).contiguous()
    for r in range(world):           # rows of rank r that belong to me
        a, b = max(offsets[r], t0), min(offsets[r] + counts[r], t1)
        if r != me and a < b:
            recvs[r] = torch.empty((2, d, b - a), dtype=torch.float64, device=torch.device("cuda", device))
    comm.exchange_tensors(sends, recvs)
    keep0, keep1 = max(my0, t0), min(my1, t1)

    def cat(parts):
        if not parts:
            return None
        return parts[0] if len(parts) == 1 else torch.cat(parts, dim=2).contiguous()

    front = cat([recvs[r] for r in sorted(recvs) if r < me])
    back = cat([recvs[r] for r in sorted(recvs) if r > me])
    kb, ke = (keep0 - my0, keep1 - my0) if keep0 < keep1 else (0, 0)
    shard.rebuild_dev(kb, ke, 0 if front is None else front.shape[2], 0 if front is None else front.data_ptr(),
                      0 if back is None else back.shape[2], 0 if back is None else back.data_ptr())
    return [b - a for a, b in target]


def _pagani_refine_device(f, cfg, comm, shard, progress, force_collectives):
    """The product path: every per-iteration exchange is a collective on device buffers of the library, issued on the
    library's stream; the host reads four sums and 2*world small numbers per iteration (the same two round trips the
    single-GPU driver makes)."""
    import torch

    from .cubature import IntegralResult
    from .domain import BudgetExceededError, NonFiniteEvaluationError
    from .execution import GroupTaskError

    d, world, me = shard.d, comm.world, comm.rank
    dev = shard.ctx.device
    collect = world > 1 or force_collectives
    g = 1
    while g**d < cfg.initial_regions:
        g += 1
    n0 = g**d
    if n0 > cfg.region_cap:
        raise BudgetExceededError(f"uniform split needs {n0} regions, cap is {cfg.region_cap}")
    shard.deferred(True)
    first, last = _even_ranges(n0, world)[me]
    counts = [b - a for a, b in _even_ranges(n0, world)]
    fin_i = fin_e = 0.0
    fin_count, processed = 0, n0
    history, converged, reason = [], False, ""
    ret_counts = None
    abs_tol = getattr(cfg, "abs_tol", 0.0)
    stream = None

    stream_ctx = {}

    def on_stream():
        # the library's stream as torch's current one; the wrapper object is built once per stream handle
        ext = stream_ctx.get(stream)
        if ext is None:
            ext = stream_ctx[stream] = torch.cuda.ExternalStream(stream, device=torch.device("cuda", dev))
        return torch.cuda.stream(ext)

    counts_host = torch.empty((world, 2), dtype=torch.float64).pin_memory()   # (split count, max error) of every rank

    try:
        shard.init(g, first, last - first)
        for iteration in range(cfg.max_iterations + 1):
            with_ret = ret_counts is not None
            offs, n_active = _offsets(counts)
            head_a = (-offs[me]) % TREE_SPAN
            head_r = (-_offsets(ret_counts)[0][me]) % TREE_SPAN if with_ret else 0
            width = max(max(counts), max(ret_counts) if with_ret else 0) // TREE_SPAN + 1
            stream, row, gathered = shard.pack(head_a, head_r, with_ret, width, world)
            if collect:
                with on_stream():
                    comm.all_gather_into(_device_tensor(gathered, dev), _device_tensor(row, dev))
            sums, bad_rank = shard.global_sums(world, n_active, sum(ret_counts) if with_ret else 0)
            if bad_rank >= 0:
                # the owner looks the evaluation up; every rank raises the single-GPU error (pagani.py:206-209)
                detail = np.zeros(3 + d)
                if bad_rank == me:
                    region, point, value, x = shard.nonfinite()
                    detail[:3] = offs[me] + region, point, value
                    detail[3:] = x
                detail = comm.allgather(detail)[bad_rank] if world > 1 else detail
                cause = NonFiniteEvaluationError(detail[3:], float(detail[2]), region_index=int(detail[0]))
                raise GroupTaskError(int(detail[0]) // cfg.chunk, cause) from cause
            if with_ret:                                    # fin += tree_sum(act[~mask]) of the last split
                fin_i += sums[2]
                fin_e += sums[3]
                ret_counts = None
            estimate = fin_i + sums[0]
            errorest = fin_e + sums[1]
            history.append((estimate, errorest, fin_count + n_active))
            if progress is not None:
                progress({"iteration": iteration, "n_regions": fin_count + n_active, "active": n_active,
                          "estimate": estimate, "errorest": errorest})
            rel_target = cfg.rel_tol * abs(estimate)
            if errorest <= (abs_tol if abs_tol > rel_target else rel_target):
                converged, reason = True, "tolerance met"
                break
            if iteration == cfg.max_iterations:
                reason = "max iterations reached"
                break
            if n_active == 0:
                reason = "no active regions left"
                break
            budget = 0.8 * abs_tol if abs_tol > rel_target else 0.8 * cfg.rel_tol * abs(estimate)

            def classify(mode, emax):
                rowb, gatheredb = shard.classify_dev(budget, mode, emax, world)
                with on_stream():
                    gt = _device_tensor(gatheredb, dev)
                    if collect:
                        comm.all_gather_into(gt, _device_tensor(rowb, dev))
                    counts_host.copy_(gt.view(world, 2), non_blocking=True)     # pinned target: no staging allocation
                    torch.cuda.current_stream().synchronize()
                    vals = counts_host.numpy()
                return [int(round(v)) for v in vals[:, 0]], float(vals[:, 1].max())

            split_counts, emax = classify(0, 0.0)
            if sum(split_counts) == 0:                      # force progress on the globally worst regions
                split_counts, _ = classify(1, emax)
            n_split = sum(split_counts)
            if processed + 2 * n_split > cfg.region_cap:
                reason = "region cap reached"
                break
            shard.split_dev(split_counts[me])
            ret_counts = [c - s for c, s in zip(counts, split_counts)]
            fin_count += n_active - n_split
            processed += 2 * n_split
            with on_stream():
                counts = rebalance_device(comm, shard, [2 * s for s in split_counts], dev)
            shard.evaluate()
    finally:
        shard.deferred(False)
    return IntegralResult(estimate, errorest, len(history) - 1, processed, converged, history, reason)


def pagani_refine_sharded(f, cfg, comm, shard=None, rule=None, progress=None, force_collectives=False, host_staged=False):
    """refine (pagani.py:300-391) with the region list sharded over comm.world GPUs.

    Every rank returns the same IntegralResult; histories are bit-identical to the single-GPU run
    for any world size (same per-region values, same global pair trees, same classification).  A non-finite
    evaluation raises the single-GPU GroupTaskError on every rank.

    Product path (`shard` a `_native.PaganiShard` or None): collectives on device buffers, see
    `_pagani_refine_device`.  A shard object without the device entry points (the CPU test-suite's oracle shard) or
    `host_staged=True` takes the host-array path below, which exchanges the same pieces as numpy arrays.
    """
    from .cubature import IntegralResult, PaganiConfig
    from .rules import build_rule, orbit_form

    cfg = cfg or PaganiConfig()
    if shard is None:
        shard = _native.PaganiShard(f.device_spec(), orbit_form(rule or build_rule(f.d)), cfg)
    if isinstance(shard, _native.PaganiShard) and not host_staged:
        return _pagani_refine_device(f, cfg, comm, shard, progress, force_collectives)
    d = shard.d
    g = 1
    while g**d < cfg.initial_regions:
        g += 1
    n0 = g**d
    if n0 > cfg.region_cap:
        from .domain import BudgetExceededError
        raise BudgetExceededError(f"uniform split needs {n0} regions, cap is {cfg.region_cap}")
    first, last = _even_ranges(n0, comm.world)[comm.rank]
    shard.init(g, first, last - first)
    counts = [b - a for a, b in _even_ranges(n0, comm.world)]
    fin_i = fin_e = 0.0
    fin_count, processed = 0, n0
    history, converged, reason = [], False, ""
    ret_counts = None

    def tree(which, cnts):
        offs, _ = _offsets(cnts)
        head = (-offs[comm.rank]) % TREE_SPAN
        return global_tree_sum(comm, shard.tree_sum, shard.reduce(which, head), cnts)

    for iteration in range(cfg.max_iterations + 1):
        if ret_counts is not None:                      # fin += tree_sum(act[~mask]) of the last split
            fin_i += tree(2, ret_counts)
            fin_e += tree(3, ret_counts)
            ret_counts = None
        n_active = sum(counts)
        estimate = fin_i + tree(0, counts)
        errorest = fin_e + tree(1, counts)
        history.append((estimate, errorest, fin_count + n_active))
        if progress is not None:
            progress({"iteration": iteration, "n_regions": fin_count + n_active, "active": n_active,
                      "estimate": estimate, "errorest": errorest})
        abs_tol = getattr(cfg, "abs_tol", 0.0)
        rel_target = cfg.rel_tol * abs(estimate)
        if errorest <= (abs_tol if abs_tol > rel_target else rel_target):
            converged, reason = True, "tolerance met"
            break
        if iteration == cfg.max_iterations:
            reason = "max iterations reached"
            break
        if n_active == 0:
            reason = "no active regions left"
            break
        budget = 0.8 * abs_tol if abs_tol > rel_target else 0.8 * cfg.rel_tol * abs(estimate)
        local_split = shard.classify(budget, 0, 0.0)
        split_counts = [int(round(v[0])) for v in comm.allgather(np.array([float(local_split)]))]
        if sum(split_counts) == 0:                      # force progress on the globally worst regions
            emax = max(float(v[0]) for v in comm.allgather(np.array([shard.max_error()])))
            local_split = shard.classify(budget, 1, emax)
            split_counts = [int(round(v[0])) for v in comm.allgather(np.array([float(local_split)]))]
        n_split = sum(split_counts)
        if processed + 2 * n_split > cfg.region_cap:
            reason = "region cap reached"
            break
        shard.split()
        ret_counts = [c - s for c, s in zip(counts, split_counts)]
        fin_count += n_active - n_split
        processed += 2 * n_split
        counts = rebalance(comm, shard, [2 * s for s in split_counts])
        shard.evaluate()
    return IntegralResult(estimate, errorest, len(history) - 1, processed, converged, history, reason)
