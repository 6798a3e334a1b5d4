"""The independent QMC oracle on the device (reference: integrands.py:223-260)."""

import numpy as np
import pytest

import paper_2302_05730_b200 as pb
from oracle import parcube_oracle as po
from paper_2302_05730_b200 import _native

pytestmark = pytest.mark.gpu


def test_sobol_points_are_scipys():
    """One shift of zero and the coordinate-sum integrand turn the per-shift sum into the sum of all coordinates of
    the point set: compared with scipy's generator for every dimension the library supports."""
    from scipy.stats import qmc
    for d in (1, 2, 5, 8, 12):
        got = _native.qmc_shift_sums(pb.get_integrand("sum", d).device_spec(), 12, np.zeros((1, d)))[0]
        want = qmc.Sobol(d=d, scramble=False).random(2**12).sum()
        assert abs(got - want) <= 1e-12 * want, d
    # a nonlinear probe distinguishes permuted coordinates or wrong direction numbers per axis
    f = pb.get_integrand("f3", 12)
    got = _native.qmc_shift_sums(f.device_spec(), 14, np.zeros((1, 12)))[0]
    want = po.genz_eval("f3", 12, qmc.Sobol(d=12, scramble=False).random(2**14)).sum()
    assert abs(got - want) <= 1e-12 * abs(want)


@pytest.mark.parametrize("fam,d", [("f3", 8), ("f2", 6), ("f4", 5), ("f1", 7), ("f6", 5)])
def test_oracle_integral_matches_reference_restatement(fam, d):
    value, bound = pb.oracle_integral(pb.get_integrand(fam, d), d, 2**16 + 1, n_shifts=4)   # rounds up to 2^17 points
    want_v, want_b, _ = po.oracle_integral(fam, d, 2**16 + 1, n_shifts=4)
    assert abs(value - want_v) <= 1e-11 * abs(want_v)
    assert abs(bound - want_b) <= 1e-7 * abs(want_b) + 1e-13 * abs(want_v)


def test_oracle_integral_agrees_with_the_integrators():
    d = 5
    f = pb.get_integrand("f3", d)
    value, bound = pb.oracle_integral(f, d, 2**20)
    truth = pb.reference_value("f3", d).value
    assert abs(value - truth) <= max(bound, 1e-6 * abs(truth))
    res = pb.refine(f, pb.PaganiConfig(rel_tol=1e-6))
    assert abs(res.estimate - value) <= bound + res.errorest
    # bounded domain (core.py:134-148) goes through the same wrapper as everywhere else
    b = pb.IntegrationBounds([0.0] * d, [0.5] * d)
    vb, bb = pb.oracle_integral(pb.scale_to_bounds(f, b), d, 2**18)
    rb = pb.refine(pb.scale_to_bounds(f, b), pb.PaganiConfig(rel_tol=1e-7))
    assert abs(vb - rb.estimate) <= bb + rb.errorest


def test_oracle_integral_argument_errors():
    f = pb.get_integrand("f1", 3)
    with pytest.raises(ValueError):
        pb.oracle_integral(f, 3, 1000)
    with pytest.raises(ValueError):
        pb.oracle_integral(f, 3, 2**16, n_shifts=1)
    with pytest.raises(ValueError):
        pb.oracle_integral(f, 4, 2**16)
