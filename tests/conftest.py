"""pytest configuration: the `gpu` marker and shared fixture loaders."""

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")


def pytest_collection_modifyitems(config, items):
    try:
        import torch

        have = torch.cuda.is_available()
    except Exception:  # noqa: BLE001
        have = False
    if have:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN, "golden.json")) as fh:
        meta = json.load(fh)
    meta["_rules"] = np.load(os.path.join(GOLDEN, "rules.npz"))
    meta["_pagani_eval"] = np.load(os.path.join(GOLDEN, "pagani_eval.npz"))
    meta["_mcubes"] = np.load(os.path.join(GOLDEN, "mcubes.npz"))
    return meta


def golden_rule(golden, d):
    """Reference rule table for d <= 8 as the dict the oracle takes."""
    z, m = golden["_rules"], golden["rules"][str(d)]
    return dict(generators=z[f"gen{d}"], weights=z[f"w{d}"], axial_indices=z[f"ax{d}"],
                split_weights=np.array([float.fromhex(v) for v in m["split"]]),
                null_degrees=tuple(m["null_degrees"]), null_scales=tuple(m["null_scales"]))


def fromhex(x):
    return float.fromhex(x)
