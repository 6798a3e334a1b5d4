"""CPU ORACLE -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.

A numpy restatement of the two integrator hot paths of the reference package
`parcube` 0.1.0 (/root/reference/pkg/src/parcube), used ONLY as the checker by
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference`
legs.  Nothing under paper_2302_05730_b200/ imports this file.

Pinning: the reference is pure Python and runs in the build container, so this
restatement is pinned against the *reference itself* -- tests/golden/*.npz were
produced by oracle/make_golden.py importing /root/reference, and
tests/test_oracle_golden.py requires this file to reproduce them (integer RNG
vectors bit-exactly; FP vectors bit-exactly on the generating numpy build and
to 1e-13 elsewhere, because numpy's SIMD exp/cos/pow and OpenBLAS gemv are
build-dependent).  The reference ships no tests of its own;
the SPEC.md known-answer examples are encoded in tests/test_oracle_golden.py.

Third-party arithmetic underneath (not in /root/reference): numpy (>=1.24,
unpinned; container has 2.3.5 + OpenBLAS 0.3.30) for exp/cos/power ufuncs, `@`
(dgemv), bincount, add.reduceat, cumsum, searchsorted.

Each function cites the reference lines it follows.
"""

from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

U64 = np.uint64
GOLDEN = U64(0x9E3779B97F4A7C15)
MIX_A = U64(0xBF58476D1CE4E5B9)
MIX_B = U64(0x94D049BB133111EB)


# =========================================================================== reductions
def tree_sum(values, axis=-1):
    """Adjacent-pair binary tree, odd levels zero-padded (engine.py:69-86)."""
    a = np.moveaxis(np.asarray(values, dtype=np.float64), axis, -1)
    if a.ndim == 1 and a.size == 0:
        return 0.0
    while a.shape[-1] > 1:
        if a.shape[-1] & 1:
            a = np.concatenate([a, np.zeros(a.shape[:-1] + (1,))], axis=-1)
        a = a[..., ::2] + a[..., 1::2]
    a = a[..., 0]
    return float(a) if a.ndim == 0 else a


def _pool_map(n_tasks, task, workers):
    """Static fan-out in task order (engine.py:106-161, failure handling omitted:
    the first exception propagates)."""
    workers = workers or (os.cpu_count() or 1)
    if workers == 1 or n_tasks <= 1:
        return [task(i) for i in range(n_tasks)]
    with ThreadPoolExecutor(max_workers=workers) as pool:
        return list(pool.map(task, range(n_tasks)))


# =========================================================================== integrands
def genz_eval(family: str, d: int, points: np.ndarray, bounds=None) -> np.ndarray:
    """The seven benchmark families in numpy's evaluation order
    (integrands.py:28-128); `bounds=(low, width, jac)` applies core.py:146-148."""
    pts = np.asarray(points, dtype=np.float64)
    if bounds is not None:
        low, width, jac = bounds
        return genz_eval(family, d, low + width * pts) * jac
    if callable(family):  # a vectorised user function, FunctionIntegrand(vectorized=True) (core.py:72-93)
        return np.asarray(family(pts), dtype=np.float64)
    idx = np.arange(1, d + 1, dtype=float)
    if family == "f1":
        return np.cos(pts @ idx)
    if family == "f2":
        u = pts - 0.5
        return np.prod(1.0 / (1.0 / 2500.0 + u * u), axis=1)
    if family == "f3":
        return (1.0 + pts @ idx) ** (-d - 1)
    if family == "f4":
        u = pts - 0.5
        return np.exp(-625.0 * np.sum(u * u, axis=1))
    if family == "f5":
        return np.exp(-10.0 * np.sum(np.abs(pts - 0.5), axis=1))
    if family == "f6":
        coeffs = idx + 4.0
        thresholds = (3.0 + idx) / 10.0
        inside = np.all(pts < thresholds, axis=1)
        out = np.zeros(len(pts))
        if inside.any():
            out[inside] = np.exp(pts[inside] @ coeffs)
        return out
    if family == "sum":
        return np.sum(pts, axis=1)
    if family == "one":  # constant, for the SPEC.md f=1 known answers
        return np.ones(len(pts))
    raise KeyError(family)


class NonFinite(ArithmeticError):
    def __init__(self, point, value, index):
        super().__init__(f"non-finite {value} at {point} in {index}")
        self.point, self.value, self.index = point, value, index


# =========================================================================== PAGANI
def initial_tiling(d: int, target: int = 1024):
    """Smallest g with g^d >= target, lexicographic tiling (pagani.py:273-279, core.py:250-269)."""
    g = max(1, int(round(target ** (1.0 / d))))
    while g**d < target:
        g += 1
    while g > 1 and (g - 1) ** d >= target:
        g -= 1
    return g, uniform_tiling(d, g)


def uniform_tiling(d: int, g: int):
    n = g**d
    idx = np.indices((g,) * d).reshape(d, n).T.astype(np.float64)
    h = 1.0 / g
    return idx * h, np.full((n, d), h)


def error_estimates(values, degrees, scales, mode="two-level", rel_floor=1e-15):
    """pagani.py:104-132."""
    nulls = np.abs(values[:, 1:5])
    if mode == "max-null":
        err = nulls.max(axis=1)
    elif mode == "max-pairwise":
        s = values[:, 1:5]
        err = np.abs(s[:, :, None] - s[:, None, :]).max(axis=(1, 2))
    else:
        high = np.asarray(degrees) >= 5
        sc = np.asarray(scales, dtype=float)
        e_high = nulls[:, high].max(axis=1)
        e_low = (nulls[:, ~high] / sc[~high]).max(axis=1)
        corr = np.ones(len(nulls))
        np.divide(10.0 * e_high, e_low, out=corr, where=e_low > 0)
        err = e_high * np.minimum(1.0, corr)
    return np.maximum(err, rel_floor * np.abs(values[:, 0]))


def strided_sums(products, group=64):
    """(n,5,F) -> (n,5): virtual thread t adds t, t+G, ... then a pair tree (pagani.py:175-192)."""
    n, rows, fe = products.shape
    steps = -(-fe // group)
    if steps * group != fe:
        products = np.concatenate([products, np.zeros((n, rows, steps * group - fe))], axis=2)
    lanes = products.reshape(n, rows, steps, group)
    acc = lanes[:, :, 0, :].copy()
    for s in range(1, steps):
        acc += lanes[:, :, s, :]
    return tree_sum(acc, axis=-1)


def evaluate_chunk(family, lefts, lengths, rule, base=0, group=64, mode="two-level",
                   rel_floor=1e-15, bounds=None):
    """One chunk of regions (pagani.py:195-224). `rule` is a dict with generators,
    weights, axial_indices, split_weights, null_degrees, null_scales."""
    off = (rule["generators"] + 1.0) / 2.0                      # quadrature.py:301
    pts = lefts[:, None, :] + lengths[:, None, :] * off[None]   # quadrature.py:302
    n, fe, d = pts.shape
    fx = genz_eval(family, d, pts.reshape(n * fe, d), bounds).reshape(n, fe)
    bad = ~np.isfinite(fx)
    if bad.any():
        r, i = np.unravel_index(int(np.argmax(bad)), bad.shape)
        raise NonFinite(pts[r, i], float(fx[r, i]), base + int(r))
    vol = np.prod(lengths, axis=1)
    vals = vol[:, None] * strided_sums(rule["weights"][None] * fx[:, None, :], group)
    err = error_estimates(vals, rule["null_degrees"], rule["null_scales"], mode, rel_floor)
    if d > 1:
        f0 = fx[:, :1]
        ax = fx[:, rule["axial_indices"]]
        c0, c1 = rule["split_weights"]
        da = ax[:, :, 0] + ax[:, :, 1] - 2.0 * f0
        db = ax[:, :, 2] + ax[:, :, 3] - 2.0 * f0
        k = np.argmax(np.abs(c0 * da - c1 * db), axis=1)
    else:
        k = np.zeros(n, dtype=np.int64)
    return vals[:, 0], err, k


def pagani_evaluate(family, lefts, lengths, rule, chunk=512, workers=1, **kw):
    """pagani_kernel (pagani.py:227-257): fixed chunks of 512 regions in order."""
    starts = list(range(0, len(lefts), chunk))
    parts = _pool_map(len(starts),
                      lambda i: evaluate_chunk(family, lefts[starts[i]:starts[i] + chunk],
                                               lengths[starts[i]:starts[i] + chunk], rule,
                                               base=starts[i], **kw),
                      workers)
    return (np.concatenate([p[0] for p in parts]), np.concatenate([p[1] for p in parts]),
            np.concatenate([p[2] for p in parts]))


def bisect(lefts, lengths, axes):
    """Children adjacent, lower half first (pagani.py:282-297)."""
    n, d = lefts.shape
    r = np.arange(n)
    half = lengths.copy()
    half[r, axes] *= 0.5
    upper = lefts.copy()
    upper[r, axes] += half[r, axes]
    out_l = np.empty((2 * n, d))
    out_h = np.empty((2 * n, d))
    out_l[0::2], out_l[1::2] = lefts, upper
    out_h[0::2], out_h[1::2] = half, half
    return out_l, out_h


def pagani_refine(family, d, rule, rel_tol=1e-3, max_iterations=50, region_cap=1 << 26,
                  initial_regions=1024, workers=1, bounds=None, time_budget_s=None, abs_tol=0.0, **kw):
    """The refinement driver (pagani.py:300-391). Returns a dict mirroring IntegralResult.
    `time_budget_s` is an oracle-only escape hatch for the bounded CPU baseline."""
    import time

    t_start = time.perf_counter()
    _, (lefts, lengths) = initial_tiling(d, initial_regions)
    act_i, act_e, act_k = pagani_evaluate(family, lefts, lengths, rule, workers=workers,
                                          bounds=bounds, **kw)
    fin_i = fin_e = 0.0
    fin_n = 0
    processed = len(lefts)
    history, active_counts, forced = [], [], []
    converged, reason = False, ""
    for it in range(max_iterations + 1):
        estimate = fin_i + tree_sum(act_i)
        errorest = fin_e + tree_sum(act_e)
        history.append((estimate, errorest, fin_n + act_i.size))
        active_counts.append(int(act_i.size))
        # abs_tol = 0 is the reference (pagani.py:350, 362); abs_tol > 0 is the epsabs extension of the B200 build
        if errorest <= max(abs_tol, rel_tol * abs(estimate)):
            converged, reason = True, "tolerance met"
            break
        if it == max_iterations:
            reason = "max iterations reached"
            break
        if act_i.size == 0:
            reason = "no active regions left"
            break
        if time_budget_s is not None and time.perf_counter() - t_start > time_budget_s:
            reason = "oracle time budget"
            break
        vol = np.prod(lengths, axis=1)
        budget = 0.8 * abs_tol if abs_tol > rel_tol * abs(estimate) else 0.8 * rel_tol * abs(estimate)
        mask = act_e > budget * vol
        if not mask.any():
            mask = act_e >= act_e.max()
            forced.append(it)
        n_split = int(np.count_nonzero(mask))
        if processed + 2 * n_split > region_cap:
            reason = "region cap reached"
            break
        fin_i += tree_sum(act_i[~mask])
        fin_e += tree_sum(act_e[~mask])
        fin_n += act_i.size - n_split
        lefts, lengths = bisect(lefts[mask], lengths[mask], act_k[mask])
        processed += len(lefts)
        act_i, act_e, act_k = pagani_evaluate(family, lefts, lengths, rule, workers=workers,
                                              bounds=bounds, **kw)
    return dict(estimate=estimate, errorest=errorest, iterations=len(history) - 1,
                regions_processed=processed, converged=converged, history=history,
                reason=reason, active_counts=active_counts, forced_iterations=forced)


# =========================================================================== m-Cubes RNG
def mix64(z):
    """mcubes.py:37-42 (wrap-around uint64)."""
    with np.errstate(over="ignore"):
        z = np.asarray(z, dtype=U64)
        z = (z ^ (z >> U64(30))) * MIX_A
        z = (z ^ (z >> U64(27))) * MIX_B
        return z ^ (z >> U64(31))


def stream_key(seed, stream):
    """mcubes.py:45-48."""
    with np.errstate(over="ignore"):
        s = U64(int(seed) & 0xFFFFFFFFFFFFFFFF)
        return mix64(s ^ mix64(np.asarray(stream, dtype=U64) * GOLDEN + U64(1)))


def uniform(seed, stream, counter):
    """mcubes.py:51-55: 53-bit draw in [0,1)."""
    with np.errstate(over="ignore"):
        h = mix64(stream_key(seed, stream) + (np.asarray(counter, dtype=U64) + U64(1)) * GOLDEN)
    return (h >> U64(11)).astype(np.float64) * 2.0**-53


def derive_seed(seed, label):
    """mcubes.py:58-60."""
    with np.errstate(over="ignore"):
        return int(mix64(U64(int(seed) & 0xFFFFFFFFFFFFFFFF) + U64(int(label)) * GOLDEN))


# =========================================================================== m-Cubes
def make_plan(n, d, group_size=128, target_groups=256):
    """mcubes.py:110-129 -> dict(d,g,m,p,s,group_size,n_threads,n_groups)."""
    n = int(n)
    if n < 2 ** (d + 1):
        raise ValueError("n too small")
    half = n // 2
    g = max(1, int((n / 2.0) ** (1.0 / d)))
    while (g + 1) ** d <= half:
        g += 1
    while g > 1 and g**d > half:
        g -= 1
    m = g**d
    p = max(2, int(math.floor(n / m + 0.5)))
    s = max(1, -(-m // (group_size * target_groups)))
    n_threads = -(-m // s)
    return dict(d=d, g=g, m=m, p=p, s=s, group_size=group_size, n_threads=n_threads,
                n_groups=-(-n_threads // group_size))


def cube_coords(cubes, g, d):
    """Base-g digits, axis 0 most significant (mcubes.py:132-140)."""
    rem = np.array(cubes, dtype=np.int64)
    out = np.empty((rem.size, d), dtype=np.int64)
    for j in range(d - 1, -1, -1):
        out[:, j] = rem % g
        rem //= g
    return out


def grid_transform(y, boundaries):
    """vegas_grid.py:99-114."""
    d, nb1 = boundaries.shape
    nb = nb1 - 1
    z = y * nb
    b = z.astype(np.int64)
    frac = z - b
    cols = np.arange(d)
    lo = boundaries[cols, b]
    width = boundaries[cols, b + 1] - lo
    return lo + frac * width, np.prod(nb * width, axis=1), b


def vsample_group(family, plan, boundaries, seed, gid, squared_weighted=True, bounds=None,
                  uniform_fn=None):
    """One work-group of the V-Sample pass (mcubes.py:210-265)."""
    d, g, m, p, s = plan["d"], plan["g"], plan["m"], plan["p"], plan["s"]
    nb = boundaries.shape[1] - 1
    t0 = gid * plan["group_size"]
    t1 = min(t0 + plan["group_size"], plan["n_threads"])
    cubes = np.arange(t0 * s, min(t1 * s, m), dtype=np.int64)
    if cubes.size == 0:
        return 0.0, 0.0, np.zeros((d, nb)), 0, 0
    thr = cubes // s
    loc = cubes - thr * s
    ctr = ((loc[:, None] * p + np.arange(p)[None, :]) * d)[:, :, None] + np.arange(d)[None, None, :]
    draw = uniform_fn or uniform
    u = draw(seed, np.repeat(thr, p * d).astype(U64), ctr.astype(U64).reshape(-1))
    u = u.reshape(cubes.size * p, d)
    y = (np.repeat(cube_coords(cubes, g, d), p, axis=0) + u) / g
    x, jac, bins = grid_transform(y, boundaries)
    fx = np.asarray(genz_eval(family, d, x, bounds), dtype=np.float64)
    bad = ~np.isfinite(fx)
    if bad.any():
        i = int(np.argmax(bad))
        raise NonFinite(x[i], float(fx[i]), int(cubes[i // p]))
    v = fx * jac
    vv = v.reshape(cubes.size, p)
    s1 = vv.sum(axis=1)
    s2 = (vv * vv).sum(axis=1)
    est = s1 / (p * m)
    raw = (s2 - s1 * s1 / p) / (p * (p - 1) * m * m)
    clamps = int(np.count_nonzero(raw < 0))
    var = np.maximum(raw, 0.0)
    seg = np.concatenate(([0], np.nonzero(np.diff(thr))[0] + 1))
    gi = float(tree_sum(np.add.reduceat(est, seg)))
    ge = float(tree_sum(np.add.reduceat(var, seg)))
    w = v * v if squared_weighted else fx * fx
    c = np.empty((d, nb))
    for j in range(d):
        c[j] = np.bincount(bins[:, j], weights=w, minlength=nb)
    return gi, ge, c, clamps, cubes.size


def sample_cube(family, cube_index, plan, boundaries, uniforms, bounds=None):
    """mcubes.sample_cube (mcubes.py:143-164) with the p*d uniforms already taken from the stream:
    returns (S1, S2, bins (p,d), v*v (p))."""
    d, g, p = plan["d"], plan["g"], plan["p"]
    coords = cube_coords([cube_index], g, d)[0]
    u = np.asarray(uniforms, dtype=np.float64).reshape(p, d)
    y = (coords + u) / g
    x, jac, bins = grid_transform(y, boundaries)
    fx = np.asarray(genz_eval(family, d, x, bounds), dtype=np.float64)
    bad = ~np.isfinite(fx)
    if bad.any():
        i = int(np.argmax(bad))
        raise NonFinite(x[i], float(fx[i]), int(cube_index))
    v = fx * jac
    return float(tree_sum(v)), float(tree_sum(v * v)), bins, v * v


def vsample(family, plan, boundaries, seed=0, workers=1, squared_weighted=True, bounds=None,
            uniform_fn=None, groups=None):
    """mcubes_kernel (mcubes.py:268-308), deterministic mode. `groups` restricts the pass
    to a subset of work-groups (used for the sharding tests)."""
    gids = list(range(plan["n_groups"])) if groups is None else list(groups)
    res = _pool_map(len(gids),
                    lambda i: vsample_group(family, plan, boundaries, seed, gids[i],
                                            squared_weighted, bounds, uniform_fn),
                    workers)
    integral = tree_sum([r[0] for r in res]) if res else 0.0
    variance = max(tree_sum([r[1] for r in res]) if res else 0.0, 0.0)
    if len(res) > 1:
        contrib = tree_sum(np.stack([r[2] for r in res], axis=0), axis=0)
    else:
        contrib = res[0][2].copy()
    return dict(integral=integral, variance=variance, contributions=contrib,
                n_samples=plan["m"] * plan["p"], clamp_events=sum(r[3] for r in res),
                group_partials=np.array([[r[0], r[1]] for r in res]))


def uniform_grid(d, n_bins=500):
    """vegas_grid.py:77-84."""
    return np.tile(np.arange(n_bins + 1) / n_bins, (d, 1))


def refine_grid(boundaries, contrib, alpha=1.5, smoothing=True):
    """vegas_grid.py:133-193."""
    d, nb1 = boundaries.shape
    n = nb1 - 1
    new_b = np.array(boundaries)
    for j in range(d):
        c = contrib[j]
        if not np.any(c > 0):
            continue
        if smoothing and n >= 2:
            sm = np.empty_like(c)
            sm[1:-1] = (c[:-2] + c[1:-1] + c[2:]) / 3.0
            sm[0] = (c[0] + c[1]) / 2.0
            sm[-1] = (c[-2] + c[-1]) / 2.0
            c = sm
        r = c / c.sum()
        w = np.zeros(n)
        mid = (r > 0) & (r < 1)
        w[mid] = ((1.0 - r[mid]) / np.log(1.0 / r[mid])) ** alpha
        w[r >= 1.0] = 1.0
        wsum = w.sum()
        if wsum <= 0:
            continue
        cw = np.concatenate(([0.0], np.cumsum(w)))
        cw[-1] = wsum
        targets = wsum * np.arange(1, n) / n
        idx = np.clip(np.searchsorted(cw, targets, side="right") - 1, 0, n - 1)
        seg = cw[idx + 1] - cw[idx]
        frac = np.where(seg > 0, (targets - cw[idx]) / np.where(seg > 0, seg, 1.0), 0.0)
        old = boundaries[j]
        new_b[j, 1:-1] = old[idx] + frac * (old[idx + 1] - old[idx])
        new_b[j, 0], new_b[j, -1] = 0.0, 1.0
        row = new_b[j]
        for k in range(1, n + 1):
            if row[k] <= row[k - 1]:
                row[k] = np.nextafter(row[k - 1], 2.0)
        if row[-1] != 1.0:
            row[-1] = 1.0
            for k in range(n, 0, -1):
                if row[k - 1] >= row[k]:
                    row[k - 1] = np.nextafter(row[k], -1.0)
    return new_b


def combine(integrals, variances):
    """Inverse-variance combination (mcubes.py:311-329)."""
    iv = np.array(integrals, dtype=float)
    var = np.maximum(np.array(variances, dtype=float), 1e-30)
    w = 1.0 / var
    wsum = float(w.sum())
    est = float(np.dot(w, iv) / wsum)
    chi2 = float(np.dot(w, (iv - est) ** 2) / (len(iv) - 1)) if len(iv) > 1 else 0.0
    return est, wsum**-0.5, chi2


def mcubes_run(family, n, d, iterations, seed=0, workers=1, n_bins=500, adapt=True,
               alpha=1.5, smoothing=True, bounds=None, rel_tol=None, abs_tol=None):
    """mcubes.run (mcubes.py:332-382); `rel_tol` adds the time-to-epsrel stop rule of
    BASELINE.md section 3 (stop after the first iteration whose cumulative
    errorest/|estimate| <= rel_tol) -- the reference itself has no tolerance stop."""
    plan = make_plan(n, d)
    grid = uniform_grid(d, n_bins)
    its, progress = [], []
    for it in range(iterations):
        res = vsample(family, plan, grid, seed=derive_seed(seed, it), workers=workers, bounds=bounds)
        its.append(res)
        if adapt:
            grid = refine_grid(grid, res["contributions"], alpha, smoothing)
        est, err, chi2 = combine([r["integral"] for r in its], [r["variance"] for r in its])
        progress.append(dict(iteration=it, estimate=est, errorest=err, chi2_per_dof=chi2,
                             iter_integral=res["integral"], iter_sd=math.sqrt(res["variance"])))
        if (rel_tol is not None or abs_tol is not None) and err <= max(abs_tol or 0.0, (rel_tol or 0.0) * abs(est)):
            break
    est, err, chi2 = combine([r["integral"] for r in its], [r["variance"] for r in its])
    return dict(estimate=est, errorest=err, chi2_per_dof=chi2, iterations=its, plan=plan,
                progress=progress, boundaries=grid)


# =========================================================================== QMC oracle
def oracle_integral(family, d, n_points, n_shifts=16, seed=20260810, bounds=None):
    """integrands.oracle_integral (integrands.py:223-260): randomly shifted Sobol' average; returns
    (value, bound, per-shift estimates).  Third-party generator: scipy.stats.qmc.Sobol (unscrambled)."""
    from scipy.stats import qmc

    if n_points < 2**16:
        raise ValueError("oracle needs n_points >= 2**16")
    if n_shifts < 2:
        raise ValueError("need at least two shifts for an error bound")
    m = max(16, int(math.ceil(math.log2(n_points))))
    shifts = np.random.default_rng(seed).random((n_shifts, d))
    acc = np.zeros(n_shifts)
    engine = qmc.Sobol(d=d, scramble=False)
    remaining = 2**m
    while remaining:
        take = min(2**18, remaining)
        base = engine.random(take)
        for s in range(n_shifts):
            pts = base + shifts[s]
            pts -= np.floor(pts)
            acc[s] += float(np.sum(genz_eval(family, d, pts, bounds)))
        remaining -= take
    estimates = acc / 2**m
    return float(np.mean(estimates)), 3.0 * float(np.std(estimates, ddof=1)) / math.sqrt(n_shifts), estimates
