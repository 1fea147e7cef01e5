"""CPU: bench.py's formulas and the reference arm's JSON contract.

The reference arm (--impl reference) runs the compiled reference on the host,
so it is exercised here at a tiny scale; the GPU arm is run by the driver.
"""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_algorithmic_bytes_match_survey():
    # S=24, nnz_f = 261,074,939
    n, m, nnz = 1 << 24, 1 << 28, 261074939
    k1, k2, k3, k3_iter = bench.alg_bytes(n, m, nnz, 20)
    assert round(k1 / 1e9, 2) == 8.59
    assert round(k2 / 1e9, 2) == 7.49 or round(k2 / 1e9, 2) == 7.50
    assert round(k3 / 1e9, 1) == 69.5
    assert k3 == 20 * k3_iter + 8 * n


def test_peaks_source():
    peak, src = bench.peaks()
    assert peak > 1000 and isinstance(src, str)


def test_clock_sampler_summary():
    s = bench.ClockSampler(0)
    s.rows = [["0", "1965", "1965", "500", "0x0", "Not Active", "Not Active", "Not Active", "Active"],
              ["0", "1900", "1965", "510", "0x4", "Not Active", "Not Active", "Not Active", "Not Active"]]
    out = s.summary()
    assert out["sm_max_mhz"] == 1965 and out["reasons"] == ["sw_power_cap"] and out["samples"] == 2


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libprpipe_ref.so")),
                    reason="reference library not built")
def test_reference_arm_json_contract():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--scale", "10",
                        "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    j = json.loads(r.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "config", "cpu_baseline", "e2e"):
        assert key in j
    assert j["impl"] == "reference" and j["value"] > 0
    assert j["e2e"]["h2d_bytes_per_step"] == 0 and j["e2e"]["d2h_bytes_per_step"] == 0
    assert j["cpu_baseline"]["kind"] == "reference"
