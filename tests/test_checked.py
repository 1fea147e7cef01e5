"""Checked-build runs (compute-sanitizer is closed on this GPU pool).

build/libprg_checked.so is the library compiled with -DPRG_CHECKED=1: device-side
bounds and invariant checks (PRG_DCHECK) on the sort engine's scatters and
local-stage slots, K2's output slots and in-degree runs, the K3 key build and
SpMV gathers. tools/sanitize_driver.py drives every device path (K0, K1 all
levels, K2 passes and fix-ups, CSC build, K3 timed / parity / Neumaier modes,
the host-buffer e2e path) against the CPU oracle through that library, on a
Kronecker and a uniform graph, and requires prg_debug_check_failures() == 0.
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "build", "libprg_checked.so")


def test_checked_library_exports_the_header():
    """The checked variant is the same C-ABI (it only adds device checks)."""
    if not os.path.exists(CHECKED):
        pytest.skip("checked library not built (paper_1603_01876_b200.build)")
    out = subprocess.run(["nm", "-D", "--defined-only", CHECKED], capture_output=True, text=True).stdout
    sys.path.insert(0, ROOT)
    from paper_1603_01876_b200 import capi

    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    missing = [s for s in capi.HEADER_SYMBOLS if s not in exported]
    assert not missing, missing


def _ensure_checked_library():
    if not os.path.exists(CHECKED):  # a checkout without build/: compile it (nvcc, ~1 min)
        sys.path.insert(0, ROOT)
        from paper_1603_01876_b200 import build

        build.build_libprg(checked=True)
    assert os.path.exists(CHECKED)


@pytest.mark.gpu
@pytest.mark.parametrize("scale", [10, 14])
def test_every_device_path_passes_its_checks(scale):
    _ensure_checked_library()
    env = dict(os.environ, PRG_LIB=CHECKED)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_driver.py"), str(scale)],
                       capture_output=True, text=True, env=env, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "checked library: True" in r.stdout
