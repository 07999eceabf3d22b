"""The facade's run driver (bench::run, host/chains.cpp) against the reference's own
(oracle/_ref: bench/runner.cpp:112-244) on the same JSON-equivalent config, including
the diffusion-coefficient move (sample_param: runner.cpp:61-85, :159-167) that swaps
the target whenever γ moves.  Trace rows (chain 0's probe coordinates at every kept
iteration) and the summary's γ moments must agree."""
import csv
import json
import subprocess

import numpy as np
import pytest

from conftest import ROOT, assert_close

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def binary():
    from paper_2303_00301_b200 import build as b
    if not b.LIB.exists():
        pytest.skip("libauxmc_b200.so not built")
    return b.build_tests()


@pytest.fixture(scope="module")
def ref():
    from oracle import refbridge as R
    if not R.available():
        pytest.skip("oracle/_ref not built")
    return R


def _trace(path):
    rows = list(csv.reader(open(path)))
    return rows[0], np.array([[float(v) for v in r] for r in rows[1:]])


@pytest.mark.parametrize("sampler,sample_param", [("aux-kalman-seq", 1), ("aux-kalman-seq", 0),
                                                  ("pgibbs-gradient", 1)])
def test_run_matches_reference(binary, ref, tmp_path, sampler, sample_param):
    T, length, burn, seed, step, delta = 30, 24, 8, 3, 0.2, 1.0
    cfg = {"sampler": sampler, "chain_length": length, "burn_in": burn, "seed": seed,
           "sample_param": bool(sample_param), "param_step": step, "delta_init": delta,
           "particles": 16, "output_dir": str(tmp_path / "ref"),
           "model": {"kind": "diffusion-smoothing", "T": T}}
    ref.run_json(json.dumps(cfg))
    out = tmp_path / "b200"
    r = subprocess.run([str(binary), "--run", sampler, "diffusion-smoothing", str(T), str(length),
                        str(burn), str(seed), str(sample_param), str(step), str(delta), str(out)],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout + r.stderr
    h0, t0 = _trace(tmp_path / "ref" / "trace.csv")
    h1, t1 = _trace(out / "trace.csv")
    assert h0 == h1
    assert t0.shape == t1.shape == (length - burn, len(h0))
    assert np.array_equal(t0[:, 0], t1[:, 0])
    assert_close(t1[:, 1:], t0[:, 1:], 1e-8, f"{sampler} trace")
    s0 = json.load(open(tmp_path / "ref" / "summary.json"))
    s1 = json.load(open(out / "summary.json"))
    assert_close(s1["rate"], s0["rate"], 1e-12, "rate")
    if sample_param:
        assert_close(s1["param_mean"], s0["param_mean"], 1e-10, "param mean")
        assert_close(s1["param_sd"], s0["param_sd"], 1e-8, "param sd")
        assert s0["param_sd"] > 0  # γ moved at least once in the kept phase
