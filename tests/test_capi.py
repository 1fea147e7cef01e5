"""CPU: the C-ABI library loads and exports every symbol include/prg.h declares.

No compute calls here (no GPU); prg_device_count / prg_version are safe.
"""
import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "prg.h")
LIB = os.path.join(ROOT, "paper_1603_01876_b200", "lib", "libprg.so")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(prg_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        from paper_1603_01876_b200 import build

        build.build_libprg()
    return ctypes.CDLL(LIB)


def test_header_declares_the_hot_path():
    syms = declared_symbols()
    for s in ("prg_k1_sort_device", "prg_k1_sort_host", "prg_k2_filter_device", "prg_k2_filter_host",
              "prg_k3_pagerank_device", "prg_k3_pagerank_host", "prg_init_rank_device",
              "prg_pagerank_step_device", "prg_matrix_download", "prg_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol(lib):
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_exported_symbols_via_nm():
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (prg_[a-z0-9_]+)", out))
    assert set(declared_symbols()) <= exported


def test_version_and_device_count_without_gpu(lib):
    lib.prg_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.prg_version()
    lib.prg_device_count.restype = ctypes.c_int32
    assert lib.prg_device_count() >= 0


def test_library_is_built_for_sm_100a():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_capi_binding_covers_header():
    from paper_1603_01876_b200 import capi

    assert set(declared_symbols()) == set(capi.HEADER_SYMBOLS)


def test_no_cpu_fallback_in_product_code():
    # The product path must not route through the oracle or any CPU compute.
    pkg = os.path.join(ROOT, "paper_1603_01876_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".hpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "from oracle" not in txt and "import oracle" not in txt, f
