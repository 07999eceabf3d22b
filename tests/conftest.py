"""Test configuration: the `gpu` marker and shared helpers.

CPU tests (`-m "not gpu"`) exercise the parity oracle against the reference's
known answers, the host-side RNG and model code, the C-ABI library's exports,
and the multi-process sharding logic (gloo).  GPU tests (`-m gpu`) call the
B200 path through the C ABI and compare with the oracle on identical inputs.
"""
import os
import pathlib
import sys

import numpy as np
import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) device")


def gpu_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if gpu_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def oracle():
    from oracle import pyoracle
    pyoracle.build()
    return pyoracle


def assert_close(got, want, rtol=1e-9, what=""):
    """|got - want| <= rtol * max(1, |want|) elementwise (FP64 contract, BASELINE.json)."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    assert got.shape == want.shape, f"{what}: shape {got.shape} vs {want.shape}"
    err = np.abs(got - want) / np.maximum(1.0, np.abs(want))
    worst = float(np.nanmax(err)) if err.size else 0.0
    assert np.all(np.isfinite(got) == np.isfinite(want)), f"{what}: finiteness differs"
    assert worst <= rtol, f"{what}: max rel err {worst:.3e} > {rtol:.1e}"
    return worst
