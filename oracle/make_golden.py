"""Generate tests/golden/* from the UNMODIFIED reference (build container only).

Usage (from the repo root, in the container that has /root/reference):
    PYTHONDONTWRITEBYTECODE=1 python oracle/make_golden.py [--slow]

The reference (`parcube`, pure Python) is imported from /root/reference/pkg/src; it
does not travel to the GPU box, the fixtures written here do.  Floating-point
fixtures record the numpy build that produced them (numpy SIMD exp/cos/pow and
OpenBLAS gemv are build-dependent), integer RNG vectors are portable.
TEST INFRASTRUCTURE -- not imported by the product.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

sys.dont_write_bytecode = True
REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REF_SRC)

import parcube  # noqa: E402
from parcube import mcubes as ref_mc  # noqa: E402
from parcube import pagani as ref_pg  # noqa: E402
from parcube import vegas_grid as ref_vg  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")
FAMILIES = ["f1", "f2", "f3", "f4", "f5", "f6", "sum"]


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def hexf(x) -> str:
    return float(x).hex()


def random_boxes(d, n, seed):
    rng = np.random.default_rng(seed)
    lengths = rng.uniform(0.01, 0.5, size=(n, d))
    lefts = rng.uniform(0.0, 1.0, size=(n, d)) * (1.0 - lengths)
    return lefts, lengths


def gen_rules(out):
    full, digest = {}, {}
    for d in range(1, 13):
        r = parcube.build_rule(d)
        digest[str(d)] = dict(f_eval=r.f_eval, generators=sha(r.generators), weights=sha(r.weights),
                              axial=sha(r.axial_indices), split=[hexf(v) for v in r.split_weights],
                              null_degrees=list(r.null_degrees), null_scales=list(r.null_scales))
        if d <= 8:
            full[f"gen{d}"] = r.generators
            full[f"w{d}"] = r.weights
            full[f"ax{d}"] = r.axial_indices
    np.savez_compressed(os.path.join(out, "rules.npz"), **full)
    return digest


def gen_rng():
    v = {}
    v["mix64"] = {str(z): int(ref_mc._mix64(np.uint64(z))) for z in (0, 1, 2, 0xFFFFFFFFFFFFFFFF, 123456789)}
    v["stream_key"] = {f"{s},{t}": int(ref_mc._stream_key(s, np.uint64(t)))
                       for s, t in ((0, 0), (0, 1), (12345, 7), (2**64 - 1, 2**40), (-3 & (2**64 - 1), 5))}
    v["uniform"] = {f"{s},{t},{c}": hexf(ref_mc._uniform(s, np.uint64(t), np.uint64(c)))
                    for s, t in ((0, 0), (12345, 7), (0xE220A8397B1DCDAF, 32767))
                    for c in (0, 1, 2, 3, 1000003, 2**33 + 5)}
    v["derive_seed"] = {f"{s},{l}": parcube.mcubes.derive_seed(s, l)
                        for s, l in ((0, 0), (0, 1), (0, 2), (7, 3), (2**63 + 11, 9))}
    return v


def gen_pagani_eval(out):
    arrays, meta = {}, {}

    def case(tag, f, lefts, lengths, fam, d, extra=None, cfg=None):
        rule = parcube.build_rule(d)
        est = parcube.pagani_kernel(f, parcube.RegionList(lefts, lengths), rule,
                                    parcube.ExecConfig(workers=1), cfg)
        arrays[f"{tag}_I"], arrays[f"{tag}_E"] = est.integrals, est.errors
        arrays[f"{tag}_K"] = est.split_axes.astype(np.int8)
        meta[tag] = dict(family=fam, d=d, n=len(lefts), **(extra or {}))

    for fam in FAMILIES:
        rl = parcube.uniform_split(5, 4)
        case(f"u5g4_{fam}", parcube.get_integrand(fam, 5), rl.lefts, rl.lengths, fam, 5,
             dict(kind="uniform", g=4))
        rl = parcube.uniform_split(8, 2)
        case(f"u8g2_{fam}", parcube.get_integrand(fam, 8), rl.lefts, rl.lengths, fam, 8,
             dict(kind="uniform", g=2))
    rl = parcube.uniform_split(8, 3)
    case("u8g3_f1", parcube.get_integrand("f1", 8), rl.lefts, rl.lengths, "f1", 8, dict(kind="uniform", g=3))
    for d in (1, 2, 3, 4, 6, 7, 9, 10):
        n = 64 if d < 9 else 8
        lefts, lengths = random_boxes(d, n, seed=100 + d)
        for fam in ("f2", "sum", "f4", "f3", "f6"):
            case(f"r{d}_{fam}", parcube.get_integrand(fam, d), lefts, lengths, fam, d,
                 dict(kind="random", seed=100 + d))
    # bounded integrand (core.py:134-148)
    for fam in ("f4", "f2", "f1"):
        d = 3
        low, high = np.array([-1.0, 0.25, 0.0]), np.array([2.0, 0.75, 3.0])
        f = parcube.scale_to_bounds(parcube.get_integrand(fam, d), parcube.IntegrationBounds(low, high))
        rl = parcube.uniform_split(d, 5)
        case(f"b3g5_{fam}", f, rl.lefts, rl.lengths, fam, d,
             dict(kind="uniform", g=5, low=low.tolist(), high=high.tolist()))
    # other error modes (pagani.py:116-120)
    for mode in ("max-null", "max-pairwise"):
        rl = parcube.uniform_split(6, 2)
        case(f"u6g2_f5_{mode}", parcube.get_integrand("f5", 6), rl.lefts, rl.lengths, "f5", 6,
             dict(kind="uniform", g=2, err_mode=mode), cfg=parcube.PaganiConfig(err_mode=mode))
    np.savez_compressed(os.path.join(out, "pagani_eval.npz"), **arrays)
    return meta


SWEEP_CASES = [("f1", 6, 1e-3), ("f4", 6, 1e-3), ("f5", 6, 1e-3), ("f3", 7, 1e-3), ("f3", 8, 1e-3)]


def run_refine_case(fam, d, tol, kw):
    t0 = time.perf_counter()
    recs = []
    res = parcube.refine(parcube.get_integrand(fam, d), parcube.PaganiConfig(rel_tol=tol, **kw),
                         parcube.ExecConfig(workers=os.cpu_count() or 8), progress=recs.append)
    rec = dict(family=fam, d=d, rel_tol=tol, cfg=kw, estimate=hexf(res.estimate),
               errorest=hexf(res.errorest), iterations=res.iterations,
               regions_processed=res.regions_processed, converged=res.converged,
               reason=res.reason,
               history=[[hexf(a), hexf(b), int(c)] for a, b, c in res.history],
               active=[r["active"] for r in recs],
               seconds=round(time.perf_counter() - t0, 2))
    print("refine", fam, d, tol, kw, res.iterations, res.regions_processed, res.reason, rec["seconds"], flush=True)
    return rec


def gen_sweep(out):
    """BASELINE config 5: the PAGANI cases of the f1..f6 x d=5..8 sweep at rel_tol 1e-3 that the reference converges
    on within ~100 s of CPU and that gen_pagani_refine does not already hold.  Written to
    a file of their own (tests/golden/sweep_refine.json) so the minutes-long cases regenerate independently."""
    recs = [run_refine_case(fam, d, tol, {}) for fam, d, tol in SWEEP_CASES]
    with open(os.path.join(out, "sweep_refine.json"), "w") as fh:
        json.dump(dict(generator="oracle/make_golden.py --sweep", reference="parcube 0.1.0 (/root/reference/pkg)",
                       numpy=np.__version__, cases=recs), fh, indent=1)


def gen_sample_cube(out):
    """mcubes.sample_cube (mcubes.py:143-164) on a few sub-cubes, with an RngStream and with a table-backed
    duck-typed rng (the injection route of SURVEY 0.1); written to tests/golden/sample_cube.json."""
    class TableRng:
        def __init__(self, table):
            self.table, self.pos = table, 0

        def take(self, n):
            out = self.table[self.pos:self.pos + n]
            self.pos += n
            return out

    recs = []
    for fam, d, n, cube, kind in (("f2", 4, 20000, 0, "stream"), ("f3", 5, 100000, 1234, "stream"),
                                  ("f4", 3, 2000, 999, "table"), ("sum", 2, 200, 17, "table"),
                                  ("f5", 8, 10**5, 255, "stream")):
        plan = parcube.make_plan(n, d)
        grid = parcube.init_grid(d)
        if kind == "stream":
            rng = parcube.RngStream(77, cube // plan.s, (cube % plan.s) * plan.p * d)
            u = parcube.RngStream(77, cube // plan.s, (cube % plan.s) * plan.p * d).take(plan.p * d)
        else:
            u = np.random.default_rng(cube).random(plan.p * d)
            rng = TableRng(u)
        s1, s2, hits = ref_mc.sample_cube(parcube.get_integrand(fam, d), cube, plan, grid, rng)
        recs.append(dict(family=fam, d=d, n=n, cube=cube, kind=kind, uniforms=[hexf(v) for v in u], s1=hexf(s1), s2=hexf(s2),
                         bins=[[int(b) for b in h[0]] for h in hits], weights=[hexf(h[1]) for h in hits]))
    with open(os.path.join(out, "sample_cube.json"), "w") as fh:
        json.dump(dict(generator="oracle/make_golden.py --cube", numpy=np.__version__, cases=recs), fh, indent=1)


def gen_pagani_refine(slow):
    cases = [("f4", 5, 1e-3, {}), ("f1", 5, 1e-3, {}), ("f2", 5, 1e-3, {}), ("f3", 5, 1e-3, {}),
             ("f5", 5, 1e-3, {}), ("f6", 5, 1e-3, dict(max_iterations=8)),
             ("sum", 4, 1e-9, {}), ("f3", 6, 1e-3, {}), ("f5", 5, 1e-5, dict(max_iterations=12)),
             ("f1", 8, 1e-6, dict(region_cap=1 << 19)), ("f4", 8, 1e-3, dict(max_iterations=5)),
             ("f2", 6, 1e-3, dict(max_iterations=9)), ("f4", 3, 1e-6, {}), ("f2", 2, 1e-8, {}),
             ("f3", 7, 1e-3, dict(max_iterations=10))]
    if slow:
        cases += [("f1", 6, 1e-3, {}), ("f1", 8, 1e-6, {})]
    out = []
    for fam, d, tol, kw in cases:
        t0 = time.perf_counter()
        recs = []
        res = parcube.refine(parcube.get_integrand(fam, d), parcube.PaganiConfig(rel_tol=tol, **kw),
                             parcube.ExecConfig(workers=8), progress=recs.append)
        out.append(dict(family=fam, d=d, rel_tol=tol, cfg=kw, estimate=hexf(res.estimate),
                        errorest=hexf(res.errorest), iterations=res.iterations,
                        regions_processed=res.regions_processed, converged=res.converged,
                        reason=res.reason,
                        history=[[hexf(a), hexf(b), int(c)] for a, b, c in res.history],
                        active=[r["active"] for r in recs],
                        seconds=round(time.perf_counter() - t0, 2)))
        print("refine", fam, d, tol, kw, res.iterations, res.regions_processed, res.reason,
              out[-1]["seconds"], flush=True)
    return out


def gen_mcubes(out):
    arrays, meta = {}, {}
    ex = parcube.ExecConfig(workers=8)

    def kern(tag, fam, d, n, seed, grid=None, f=None, extra=None):
        f = f or parcube.get_integrand(fam, d)
        plan = parcube.make_plan(n, d)
        grid = grid or parcube.init_grid(d)
        res = parcube.mcubes_kernel(f, plan, grid, ex, seed=seed)
        arrays[f"{tag}_C"] = res.contributions.c
        new = parcube.refine_grid(grid, res.contributions)
        arrays[f"{tag}_B"] = new.boundaries
        meta[tag] = dict(family=fam, d=d, n=n, seed=seed, integral=hexf(res.integral),
                         variance=hexf(res.variance), clamps=res.clamp_events,
                         n_samples=res.n_samples,
                         plan=dict(g=plan.g, m=plan.m, p=plan.p, s=plan.s), **(extra or {}))
        return res, new

    for fam in FAMILIES:
        kern(f"k5_{fam}", fam, 5, 100000, 0)
    kern("k8_f3", "f3", 8, 1000000, 0)
    kern("k6_f2", "f2", 6, 1000000, 0)
    kern("k2_sum", "sum", 2, 32, 3)
    kern("k1_f4", "f4", 1, 1000, 11)
    kern("k3_f5", "f5", 3, 5000, ref_mc.derive_seed(5, 2))
    # second pass on an adapted grid
    _, g1 = kern("k6a_f4", "f4", 6, 200000, 1)
    res2, _ = kern("k6b_f4", "f4", 6, 200000, 2, grid=g1, extra=dict(grid_from="k6a_f4"))
    # bounded
    low, high = np.array([-1.0, 0.25, 0.0, 0.0]), np.array([2.0, 0.75, 3.0, 1.0])
    fb = parcube.scale_to_bounds(parcube.get_integrand("f4", 4), parcube.IntegrationBounds(low, high))
    kern("k4b_f4", "f4", 4, 50000, 4, f=fb, extra=dict(low=low.tolist(), high=high.tolist()))

    # injected uniforms: replace the reference's hash by a table lookup (SURVEY 0.1 last row)
    fam, d, n = "f3", 5, 20000
    plan = parcube.make_plan(n, d)
    table = np.random.default_rng(20230213).random(plan.m * plan.p * d)
    stride = plan.s * plan.p * d
    original = ref_mc._uniform
    ref_mc._uniform = lambda seed, sid, ctr: table[(np.asarray(sid, dtype=np.int64) * stride
                                                    + np.asarray(ctr, dtype=np.int64))]
    try:
        res = parcube.mcubes_kernel(parcube.get_integrand(fam, d), plan, parcube.init_grid(d), ex, seed=0)
    finally:
        ref_mc._uniform = original
    arrays["inj_C"] = res.contributions.c
    meta["inj"] = dict(family=fam, d=d, n=n, table_seed=20230213, integral=hexf(res.integral),
                       variance=hexf(res.variance), clamps=res.clamp_events,
                       plan=dict(g=plan.g, m=plan.m, p=plan.p, s=plan.s))

    runs = []
    for fam, d, n, its, seed in (("f2", 6, 1000000, 6, 0), ("f3", 8, 1000000, 5, 0),
                                 ("f4", 8, 1000000, 10, 0), ("f5", 5, 100000, 10, 3),
                                 ("f1", 5, 100000, 4, 0), ("f6", 6, 200000, 6, 9)):
        recs = []
        res = parcube.mcubes_run(parcube.get_integrand(fam, d), n, d, its, seed=seed, exec_cfg=ex,
                                 progress=recs.append)
        runs.append(dict(family=fam, d=d, n=n, iterations=its, seed=seed, estimate=hexf(res.estimate),
                         errorest=hexf(res.errorest), chi2=hexf(res.chi2_per_dof),
                         progress=[{k: (hexf(v) if isinstance(v, float) else v) for k, v in r.items()}
                                   for r in recs]))
        print("run", fam, d, n, res.estimate, res.errorest, flush=True)
    meta["runs"] = runs
    # standalone refine_grid on a synthetic, very peaked table (exercises the nextafter nudges)
    c = np.zeros((2, 500))
    c[0, 250] = 1.0
    c[1, :] = np.linspace(0.0, 1.0, 500) ** 8
    bc = ref_vg.BinContributions(2, 500)
    bc.c[:] = c
    arrays["peaked_C"] = c
    arrays["peaked_B"] = parcube.refine_grid(parcube.init_grid(2), bc).boundaries
    np.savez_compressed(os.path.join(out, "mcubes.npz"), **arrays)
    return meta


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--slow", action="store_true", help="also run the minutes-long refine cases")
    ap.add_argument("--cube", action="store_true", help="only (re)generate tests/golden/sample_cube.json")
    ap.add_argument("--sweep", action="store_true", help="only (re)generate tests/golden/sweep_refine.json (config 5)")
    args = ap.parse_args()
    os.makedirs(OUT, exist_ok=True)
    if args.sweep:
        gen_sweep(OUT)
        return
    if args.cube:
        gen_sample_cube(OUT)
        return
    meta = dict(generator="oracle/make_golden.py", reference="parcube 0.1.0 (/root/reference/pkg)",
                numpy=np.__version__, blas=str(np.show_config(mode="dicts")["Build Dependencies"]["blas"].get("version")),
                cpu_features=str(np.show_config(mode="dicts").get("SIMD Extensions", {}).get("found")))
    meta["rules"] = gen_rules(OUT)
    meta["rng"] = gen_rng()
    meta["pagani_eval"] = gen_pagani_eval(OUT)
    meta["mcubes"] = gen_mcubes(OUT)
    meta["pagani_refine"] = gen_pagani_refine(args.slow)
    with open(os.path.join(OUT, "golden.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
