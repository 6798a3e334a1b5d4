"""CPU-only checks of the host layer: the C-ABI library loads and exports every declared
symbol, rule tables match the reference fixtures, plans/tilings/seeds follow the reference,
and the product path fails loudly without a GPU (no CPU fallback, no oracle import)."""

import ctypes
import hashlib
import os
import re

import numpy as np
import pytest

import paper_2302_05730_b200 as pb
from conftest import ROOT, golden_rule
from helpers import same_numpy_build
from oracle import parcube_oracle as po
from paper_2302_05730_b200 import _native, rules


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_library_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "parcube_b200.h")).read()
    declared = set(re.findall(r"^(?:pcb_status|void|const char\*|int64_t)\s+(pcb_[a-z0-9_]+)\(", header, flags=re.M))
    assert declared == set(_native.SIGNATURES), declared ^ set(_native.SIGNATURES)
    lib = _native.load_library()
    raw = ctypes.CDLL(_native.LIB_PATH)
    for name in declared:
        assert getattr(raw, name) is not None and getattr(lib, name) is not None


def test_struct_sizes_match_header_layout():
    assert ctypes.sizeof(_native.IntegrandC) == 16 + 8 * (3 * 12 + 1)
    assert ctypes.sizeof(_native.RuleC) == 8 + 8 * 7 + 8 * 25 + 4 * 6 + 16 + 16 + 32
    assert ctypes.sizeof(_native.PaganiConfigC) == 48   # ... rel_floor, abs_tol
    assert ctypes.sizeof(_native.NonFiniteC) == 24 + 96
    assert ctypes.sizeof(_native.McubesPlanC) == 40


def test_build_rule_matches_reference_tables(golden):
    for d in range(1, 13):
        r = pb.build_rule(d)
        meta = golden["rules"][str(d)]
        assert r.f_eval == meta["f_eval"] == pb.f_eval_count(d)
        assert list(r.null_degrees) == meta["null_degrees"] and list(r.null_scales) == meta["null_scales"]
        assert _sha(r.generators) == meta["generators"] and _sha(r.axial_indices) == meta["axial"]
        assert [float(v).hex() for v in r.split_weights] == meta["split"]
        if same_numpy_build(golden):
            assert _sha(r.weights) == meta["weights"], f"d={d}: LAPACK-derived weights differ"
        elif d <= 8:
            assert np.allclose(r.weights, golden_rule(golden, d)["weights"], rtol=1e-12, atol=1e-16)


def test_orbit_form_roundtrip_and_validation(golden):
    for d in (1, 2, 5, 8):
        r = pb.build_rule(d)
        o = rules.orbit_form(r)
        gen, orb = rules._point_set(d)
        # rebuild the full weight table from the orbit form
        odd = np.array([bin(b).count("1") & 1 for b in range(1 << d)], dtype=bool)
        for k in range(5):
            full = o.weights[k][orb].copy()
            if o.corner_parity[k]:
                full[orb == 4] = np.where(odd, -o.weights[k, 4], o.weights[k, 4])
            assert np.array_equal(full, r.weights[k])
        assert np.array_equal(np.unique((r.generators + 1.0) / 2.0), np.unique(o.offsets))
    bad = pb.build_rule(3)
    w = np.array(bad.weights)
    w[0, 5] *= 1.0000001
    broken = rules.RuleTable(3, bad.f_eval, bad.generators, w, bad.split_weights, bad.axial_indices,
                             bad.null_degrees, bad.null_scales)
    with pytest.raises(ValueError):
        rules.orbit_form(broken)


def test_plans_tilings_seeds_follow_reference(golden):
    for n, d in ((10**8, 8), (32, 2), (10**9, 8), (10**6, 6), (10**5, 5), (1000, 1), (3 * 10**9, 8)):
        mine, ref = pb.make_plan(n, d), po.make_plan(n, d)
        assert (mine.g, mine.m, mine.p, mine.s, mine.n_threads, mine.n_groups) == \
               (ref["g"], ref["m"], ref["p"], ref["s"], ref["n_threads"], ref["n_groups"])
    with pytest.raises(ValueError):
        pb.make_plan(100, 8)
    for d, g in ((1, 7), (3, 4), (5, 3)):
        rl = pb.uniform_split(d, g)
        lefts, lengths = po.uniform_tiling(d, g)
        assert np.array_equal(rl.lefts, lefts) and np.array_equal(rl.lengths, lengths)
    with pytest.raises(pb.BudgetExceededError):
        pb.uniform_split(8, 20)
    with pytest.raises(pb.UnsupportedDimensionError):
        pb.uniform_split(13, 2)
    for key, want in golden["rng"]["derive_seed"].items():
        s, l = map(int, key.split(","))
        assert pb.derive_seed(s, l) == want


def test_domain_validation():
    with pytest.raises(ValueError):
        pb.RegionList(np.zeros((2, 3)), np.zeros((2, 3)))
    with pytest.raises(ValueError):
        pb.IntegrationBounds([0, 1], [1, 1])
    with pytest.raises(ValueError):
        pb.PaganiConfig(rel_tol=0)
    with pytest.raises(ValueError):
        pb.PaganiConfig(err_mode="nope")
    with pytest.raises(KeyError):
        pb.get_integrand("f9", 3)
    f = pb.scale_to_bounds(pb.get_integrand("f4", 2), pb.IntegrationBounds([-1, 0], [1, 2]))
    spec = f.device_spec()
    assert spec.bounded and spec.jac == 4.0 and list(spec.width) == [2.0, 2.0]
    with pytest.raises(TypeError):
        pb.FunctionIntegrand(lambda x: 1.0, 3).device_spec()
    assert pb.reference_value("sum", 6).value == 3.0
    assert abs(pb.reference_value("f4", 5).value - 1.7918e-06) < 1e-9


def test_no_cpu_fallback_and_no_oracle_in_product():
    try:
        import torch
        have_gpu = torch.cuda.is_available()
    except Exception:  # noqa: BLE001
        have_gpu = False
    if not have_gpu:
        with pytest.raises(_native.NativeError):
            pb.pagani_kernel(pb.get_integrand("f4", 3), pb.uniform_split(3, 2), pb.build_rule(3))
        with pytest.raises(_native.NativeError):
            pb.mcubes_run(pb.get_integrand("f4", 3), 1000, 3, 2)
    pkg = os.path.join(ROOT, "paper_2302_05730_b200")
    for dirpath, _, files in os.walk(pkg):
        for name in files:
            if name.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, name)).read()
                assert "parcube_oracle" not in text and "from oracle" not in text and "import oracle" not in text, name
                for line in text.splitlines():  # citations are fine, reading the tree at run time is not
                    if "/root/reference" in line:
                        assert not any(tok in line for tok in ("sys.path", "open(", "import ", "PYTHONPATH")), (name, line)


def test_cli_argument_handling_matches_reference(capsys):
    from paper_2302_05730_b200 import harness

    assert harness.COMPARE_HEADER == "id,mean_a_ms,mean_b_ms,std_a,std_b,ratio"          # cli.py:33
    assert harness.main(["integrate", "--integrator", "pagani", "--integrand", "f9", "-d", "5"]) == 2
    assert harness.main(["integrate", "--integrator", "nope", "--integrand", "f1", "-d", "5"]) == 2
    assert harness.main(["compare", "--config-a", "workers=1", "--config-b", "workers=8"]) == 2
    assert harness.main(["bench-invoke", "--integrand", "f1", "-d", "3", "--points", "0"]) == 2
    sc = harness.parse_scenario("pagani:f4:d=8:g=4:reps=5")
    assert (sc["integrator"], sc["integrand"], sc["d"], sc["g"], sc["reps"]) == ("pagani", "f4", 8, 4, 5)
    assert harness.parse_scenario("mcubes:f5:d=5:n=1e5:reps=5")["n"] == 100000
    for bad in ("pagani:f4", "vegas:f4:d=3", "pagani:f9:d=3", "pagani:f4:g=3", "pagani:f4:d=3:zz=1", "pagani:f4:d=3:reps=0"):
        with pytest.raises(harness.CliError):
            harness.parse_scenario(bad)
    cfg = harness.parse_config("workers=8,deterministic=false")
    assert cfg.workers == 8 and cfg.deterministic is False
    with pytest.raises(harness.CliError):
        harness.parse_config("threads=8")
    capsys.readouterr()


def test_abs_tol_is_an_extension_with_reference_default():
    """epsabs (BASELINE.json north_star): accepted everywhere, 0 by default = the reference's rel_tol-only rule."""
    import paper_2302_05730_b200 as pb
    assert pb.PaganiConfig().abs_tol == 0.0
    assert pb.PaganiConfig(abs_tol=1e-7).abs_tol == 1e-7
    with pytest.raises(ValueError):
        pb.PaganiConfig(abs_tol=-1.0)
    c = _native.pagani_config_to_c(pb.PaganiConfig(rel_tol=1e-4, abs_tol=2e-9))
    assert (c.rel_tol, c.abs_tol) == (1e-4, 2e-9)


def test_bench_refuses_to_claim_gpus_it_does_not_have():
    """`bench.py --gpus N` launched without torchrun spawns N ranks itself -- and says so instead of printing n_gpus = N
    from one process when the node has fewer devices (missing #2)."""
    import json
    import subprocess
    import sys
    proc = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"], capture_output=True,
                          text=True, timeout=300, env={k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK")})
    assert proc.returncode == 2, (proc.stdout, proc.stderr[-500:])
    line = json.loads(proc.stdout.strip().splitlines()[-1])
    assert "error" in line and "n_gpus" not in line
    # under a launcher whose world size disagrees with --gpus it refuses as well
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    proc = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4", "--steps", "1"], capture_output=True,
                          text=True, timeout=300, env=env)
    assert proc.returncode != 0 and "refusing to report n_gpus=4" in proc.stderr


def test_run_time_family_image_builds_and_carries_every_kernel():
    """userfn.build_image cross-compiles here (no GPU needed): the cubin must hold the eight kernels whose mangled
    names userfn._kernel_names predicts, and a source error must surface as ValueError with the compiler's log."""
    from paper_2302_05730_b200 import userfn

    image = userfn.build_image(9, 4, "double u = x - 0.3; return u * u;", "return exp(-param[0] * acc);", "numpy_sum")
    for key, name in userfn._kernel_names(9, 4).items():
        assert name.encode() in image, key
    with pytest.raises(ValueError, match="does not compile"):
        userfn.build_image(9, 4, "return no_such_symbol;", "return acc;", "sum")
    assert userfn.USER_FAMILY_BASE == 8 and userfn.MAX_USER_FAMILIES == 8      # include/parcube_b200.h
