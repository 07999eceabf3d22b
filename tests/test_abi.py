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


@pytest.mark.parametrize("T", [1, 7, 300, 3000, 4095, 65536, 1 << 20, (1 << 20) + 5])
def test_time_shard_geometry_nests_sampler_blocks(lib, T):
    """The scan filter's super-blocks hold whole prefix-sampler blocks (a time-sharded
    rank's range is a run of super-blocks, tshard.ShardedPrefixSampler), and the
    block tree covers the horizon.  Host-computable, no device."""
    LB, nblk, nsup, SB, ed = (ctypes.c_int() for _ in range(5))
    assert lib.auxmc_tshard_geometry(T, 16, *(ctypes.byref(x) for x in (LB, nblk, nsup, SB, ed))) == 0
    Lb, P = ctypes.c_int(), ctypes.c_int()
    assert lib.auxmc_tshard_prefix_geometry(T, ctypes.byref(Lb), ctypes.byref(P)) == 0
    assert SB.value % Lb.value == 0, (SB.value, Lb.value)
    assert nblk.value * LB.value >= T + 1 > (nblk.value - 1) * LB.value
    assert nsup.value * SB.value >= T + 1
    assert P.value * Lb.value >= T
