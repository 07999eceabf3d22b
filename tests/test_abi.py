"""C-ABI checks that need no GPU: the shared library loads, exports every
entry point include/auxmc_gpu.h declares, and refuses compute without a
device (no CPU fallback)."""
import ctypes
import pathlib
import re

import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]


def declared_functions():
    text = (ROOT / "include" / "auxmc_gpu.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(auxmc_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2303_00301_b200 import _lib
    return _lib.load()


def test_library_exports_every_declared_symbol(lib):
    names = declared_functions()
    assert len(names) > 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, f"missing exports: {missing}"


def test_version_and_status_strings(lib):
    assert lib.auxmc_version().decode() == "0.1.0"
    assert b"jitter" in lib.auxmc_status_string(2)


def test_compute_refused_without_device(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    assert lib.auxmc_device_ok() == 0
    rc = lib.auxmc_rng_normals(None, 0, 1, 0, 0, 0, None, None)
    assert rc == 6  # AUXMC_E_CUDA: no silent CPU path


def test_sizes_are_host_computable(lib):
    from paper_2303_00301_b200 import _lib
    m = _lib.Lgssm()
    m.T, m.dx, m.dy = 65536, 4, 1
    m.nF = m.nb = m.nQ = m.nH = m.nc = m.nR = 1
    for sampler in (0, 1, 2):
        n = lib.auxmc_sample_paths_workspace(ctypes.byref(m), 1, 1024, sampler)
        assert n > 0
    assert lib.auxmc_dnc_bridge_count(65536) == 65536
    assert lib.auxmc_dnc_bridge_count(5) == 8
