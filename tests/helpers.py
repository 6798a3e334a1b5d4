"""Shared helpers for parity tests."""

import numpy as np


def random_boxes(d, n, seed):
    """Same generator as oracle/make_golden.py:random_boxes."""
    rng = np.random.default_rng(seed)
    lengths = rng.uniform(0.01, 0.5, size=(n, d))
    lefts = rng.uniform(0.0, 1.0, size=(n, d)) * (1.0 - lengths)
    return lefts, lengths


def same_numpy_build(golden):
    return golden["numpy"] == np.__version__


def ulp_diff(a, b):
    """Distance in units-in-the-last-place between float64 arrays (same sign assumed)."""
    a = np.ascontiguousarray(a, dtype=np.float64).view(np.int64)
    b = np.ascontiguousarray(b, dtype=np.float64).view(np.int64)
    return np.abs(a - b)
