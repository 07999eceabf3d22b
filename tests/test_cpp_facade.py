"""The C++ host facade (include/auxmc_b200.hpp: the reference's lgssm / pit /
auxk / fkpg / bench API over the C ABI) checked by the compiled test program
tests/cpp/test_facade.cpp against the CPU oracle.

CPU: the facade's host-side checks and its refusal to compute without a device.
GPU: filters, the three pathwise samplers (stream and pre-drawn NoiseSource),
path_logpdf, the auxiliary Kalman kernel (all backends, both filters), the
reference cSMC sweep, batched chains and the run driver, against the oracle.
"""
import subprocess

import pytest

from conftest import ROOT


@pytest.fixture(scope="module")
def binary():
    from oracle import pyoracle
    from paper_2303_00301_b200 import build as b
    if not b.LIB.exists():
        pytest.skip("libauxmc_b200.so not built (run __graft_entry__.build())")
    pyoracle.build()
    return b.build_tests()


def _run(binary, *args, timeout=600):
    r = subprocess.run([str(binary), *args], capture_output=True, text=True, timeout=timeout,
                       cwd=ROOT)
    return r.returncode, r.stdout + r.stderr


def test_facade_host_checks_and_no_cpu_path(binary):
    rc, out = _run(binary, "--no-device")
    assert rc == 0, out
    assert "0 failures" in out


@pytest.mark.gpu
def test_facade_parity_on_device(binary):
    rc, out = _run(binary)
    print(out)
    assert rc == 0, out
    assert "0 failures" in out
