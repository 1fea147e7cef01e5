"""ctypes bindings for the CPU checkers — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this module, and only as the checker or the CPU
baseline; the product path (paper_1603_01876_b200/) never does.

Two checkers live behind it:
  * ``liboracle.so``   — oracle/prg_oracle.c, a C restatement of the reference's
    K0/K1/K2/K3 (each function cites the reference file:line it follows);
  * ``libprpipe_ref.so`` — the reference itself, compiled from
    /root/reference/proj/src by oracle/build_ref.sh (absent on hosts where the
    reference was never built; ``have_reference()`` tells).
Parity of the restatement is pinned by tests/test_oracle_pins.py against the
reference's own known-answer tests and the reference-generated golden vectors
in tests/golden/.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_REF_DIR = os.path.join(_HERE, "_ref")
GRAPH500 = (0.57, 0.19, 0.19, 0.05)
UNIFORM = (0.25, 0.25, 0.25, 0.25)

_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")


def _load(name: str):
    path = os.path.join(_REF_DIR, name)
    if not os.path.exists(path) and name == "liboracle.so":
        subprocess.run(["bash", os.path.join(_HERE, "build_ref.sh")], check=True,
                       stdout=subprocess.DEVNULL)
    return C.CDLL(path) if os.path.exists(path) else None


_lib = _load("liboracle.so")
_ref = _load("libprpipe_ref.so")


def have_reference() -> bool:
    return _ref is not None


def _sig(lib, name, res, args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = args
    return f


_mix_seed = _sig(_lib, "oracle_mix_seed", C.c_uint64, [C.c_uint64, C.c_uint64])
_perm = _sig(_lib, "oracle_permutation", None, [C.c_int64, C.c_uint64, _i64p])
_make = _sig(_lib, "oracle_make_edges", None,
             [C.c_int, C.c_uint64, _f64p, C.c_void_p, C.c_int64, C.c_int64, _i64p])
_k1 = _sig(_lib, "oracle_k1_sort", C.c_int, [_i64p, C.c_int64, C.c_int, _i64p])
_k2 = _sig(_lib, "oracle_k2", C.c_int64,
           [_i64p, C.c_int64, C.c_int64, _i64p, _i64p, _f64p, _i64p, C.POINTER(C.c_int64)])
_init = _sig(_lib, "oracle_init_rank", C.c_double, [C.c_int64, C.c_uint64, _f64p, C.c_int])
_step = _sig(_lib, "oracle_pagerank_step", C.c_double,
             [C.c_int64, _i64p, _i64p, _f64p, _f64p, C.c_double, _f64p, C.c_int])
_k3 = _sig(_lib, "oracle_run_kernel3", C.c_double,
           [C.c_int64, _i64p, _i64p, _f64p, C.c_double, C.c_int, C.c_uint64, _f64p, C.c_int])


def mix_seed(seed: int, stream: int) -> int:
    return int(_mix_seed(seed, stream))


def permutation(n: int, seed: int) -> np.ndarray:
    out = np.empty(n, dtype=np.int64)
    _perm(n, seed, out)
    return out


def generate(scale: int, seed: int, initiator=GRAPH500, permute: bool = True,
             edge_factor: int = 16) -> np.ndarray:
    """K0 restatement (graph_gen.cpp:60-111): (M, 2) int64 edge list."""
    n = 1 << scale
    m = edge_factor * n
    init = np.asarray(initiator, dtype=np.float64)
    labels = permutation(n, seed) if permute else None
    uv = np.empty((m, 2), dtype=np.int64)
    _make(scale, seed, init, labels.ctypes.data if labels is not None else None, 0, m, uv)
    return uv


def k1_sort(uv: np.ndarray, scale: int) -> np.ndarray:
    """K1 with canonical tie order (u, then v) — tests/helpers.hpp:29-34."""
    uv = np.ascontiguousarray(uv, dtype=np.int64)
    out = np.empty_like(uv)
    rc = _k1(uv, len(uv), scale, out)
    if rc:
        raise ValueError(f"oracle_k1_sort failed ({rc})")
    return out


class K2Result:
    def __init__(self, n, row_offsets, cols, values, d_in, nnz_raw):
        self.n, self.row_offsets, self.cols, self.values = n, row_offsets, cols, values
        self.d_in, self.nnz_raw = d_in, nnz_raw

    @property
    def nnz(self) -> int:
        return len(self.cols)


def k2(uv: np.ndarray, n: int) -> K2Result:
    """K2 core restatement (kernel2_filter.cpp:12-152)."""
    uv = np.ascontiguousarray(uv, dtype=np.int64).reshape(-1, 2)
    m = len(uv)
    ro = np.empty(n + 1, dtype=np.int64)
    cols = np.empty(max(m, 1), dtype=np.int64)
    vals = np.empty(max(m, 1), dtype=np.float64)
    din = np.empty(n, dtype=np.int64)
    raw = C.c_int64(0)
    nf = _k2(uv, m, n, ro, cols, vals, din, C.byref(raw))
    if nf < 0:
        raise ValueError({-1: "label outside [1, n]", -2: "input not sorted by start vertex",
                          -3: "vertex count must be positive"}[int(nf)])
    return K2Result(n, ro, cols[:nf].copy(), vals[:nf].copy(), din, int(raw.value))


def init_rank(n: int, seed: int, accurate: bool = False):
    r = np.empty(n, dtype=np.float64)
    norm = _init(n, seed, r, int(accurate))
    return r, norm


def pagerank_step(r, row_offsets, cols, values, n: int, damping=0.85, accurate=False):
    out = np.empty(n, dtype=np.float64)
    norm = _step(n, _c64(row_offsets), _c64(cols), _cf(values), _cf(r), damping, out,
                 int(accurate))
    return out, norm


def run_kernel3(row_offsets, cols, values, n: int, damping=0.85, iterations=20, seed=0,
                accurate=False):
    """run_kernel3 restatement (kernel3_pagerank.cpp:67-79); accurate=True is the
    Neumaier-Σr variant used to attribute drift."""
    r = np.empty(n, dtype=np.float64)
    norm = _k3(n, _c64(row_offsets), _c64(cols), _cf(values), damping, iterations, seed, r,
               int(accurate))
    return r, norm


def _c64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _cf(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# ---- the reference itself (oracle/_ref/libprpipe_ref.so) -------------------
if _ref is not None:
    _ref.ref_last_error.restype = C.c_char_p
    _rgen = _sig(_ref, "ref_generate", C.c_int,
                 [C.c_int, C.c_uint64, _f64p, C.c_int, C.c_int, _i64p])
    _rk1 = _sig(_ref, "ref_k1_sort_core", C.c_double, [_i64p, C.c_int64])
    _rk2 = _sig(_ref, "ref_k2_core", C.c_int64,
                [_i64p, C.c_int64, C.c_int64, _i64p, _i64p, _f64p, _i64p,
                 C.POINTER(C.c_int64), C.POINTER(C.c_double)])
    _rk3 = _sig(_ref, "ref_k3", C.c_double,
                [C.c_int64, C.c_int64, _i64p, _i64p, _f64p, C.c_double, C.c_int, C.c_uint64,
                 C.c_int64, _f64p, C.POINTER(C.c_double)])
    _rinit = _sig(_ref, "ref_init_rank", C.c_double, [C.c_int64, C.c_uint64, _f64p])
    _rstep = _sig(_ref, "ref_pagerank_step", C.c_double,
                  [C.c_int64, C.c_int64, _i64p, _i64p, _f64p, _f64p, C.c_double, _f64p])


def _need_ref():
    if _ref is None:
        raise RuntimeError("oracle/_ref/libprpipe_ref.so not built (no /root/reference here)")


def ref_generate(scale: int, seed: int, initiator=GRAPH500, permute=True, threads=None):
    _need_ref()
    m = 16 << scale
    uv = np.empty((m, 2), dtype=np.int64)
    if _rgen(scale, seed, np.asarray(initiator, dtype=np.float64), int(permute),
             threads or os.cpu_count() or 1, uv):
        raise RuntimeError(_ref.ref_last_error().decode())
    return uv


def ref_k1_sort_core(uv: np.ndarray):
    """std::sort by u (kernel1_sort.cpp:66), in place on a copy; (sorted, seconds)."""
    _need_ref()
    out = np.ascontiguousarray(uv, dtype=np.int64).copy()
    t = _rk1(out, len(out))
    return out, t


def ref_k2(uv: np.ndarray, n: int):
    """The reference's K2 core; returns (K2Result, seconds)."""
    _need_ref()
    uv = np.ascontiguousarray(uv, dtype=np.int64).reshape(-1, 2)
    m = len(uv)
    ro = np.empty(n + 1, dtype=np.int64)
    cols = np.empty(max(m, 1), dtype=np.int64)
    vals = np.empty(max(m, 1), dtype=np.float64)
    din = np.empty(n, dtype=np.int64)
    raw, el = C.c_int64(0), C.c_double(0)
    nf = _rk2(uv, m, n, ro, cols, vals, din, C.byref(raw), C.byref(el))
    if nf < 0:
        raise RuntimeError(_ref.ref_last_error().decode())
    return K2Result(n, ro, cols[:nf].copy(), vals[:nf].copy(), din, int(raw.value)), el.value


def ref_run_kernel3(row_offsets, cols, values, n, damping=0.85, iterations=20, seed=0,
                    total_edges=0):
    """The reference's run_kernel3; returns (ranks, norm1, seconds)."""
    _need_ref()
    r = np.empty(n, dtype=np.float64)
    el = C.c_double(0)
    norm = _rk3(n, len(cols), _c64(row_offsets), _c64(cols), _cf(values), damping, iterations,
                seed, total_edges, r, C.byref(el))
    return r, norm, el.value


def ref_init_rank(n: int, seed: int):
    _need_ref()
    r = np.empty(n, dtype=np.float64)
    return r, _rinit(n, seed, r)


def ref_pagerank_step(r, row_offsets, cols, values, n, damping=0.85):
    _need_ref()
    out = np.empty(n, dtype=np.float64)
    norm = _rstep(n, len(cols), _c64(row_offsets), _c64(cols), _cf(values), _cf(r), damping, out)
    return out, norm


# ---- K2 step-level restatements (kernel2_filter.cpp:12-152) -------------
_bld = _sig(_lib, "oracle_build_adjacency", C.c_int64, [_i64p, C.c_int64, C.c_int64, _i64p, _i64p, _i64p])
_ind = _sig(_lib, "oracle_in_degree", None, [C.c_int64, C.c_int64, _i64p, _i64p, _i64p])
_zc = _sig(_lib, "oracle_zero_columns", C.c_int64, [C.c_int64, _i64p, _i64p, _i64p, _i64p, _i64p, _i64p, _i64p])
_rn = _sig(_lib, "oracle_row_normalize", None, [C.c_int64, _i64p, _i64p, _f64p])


def build_adjacency(uv, n: int):
    """CountMatrix as (row_offsets, cols, counts); raises ValueError like build_from."""
    uv = np.ascontiguousarray(uv, dtype=np.int64).reshape(-1, 2)
    m = len(uv)
    ro = np.empty(n + 1, dtype=np.int64)
    cols = np.empty(max(m, 1), dtype=np.int64)
    cnt = np.empty(max(m, 1), dtype=np.int64)
    nnz = _bld(uv, m, n, ro, cols, cnt)
    if nnz < 0:
        raise ValueError({-1: "label outside [1, n]", -2: "input not sorted by start vertex",
                          -3: "vertex count must be positive"}[int(nnz)])
    return ro, cols[:nnz].copy(), cnt[:nnz].copy()


def in_degree(n, cols, counts):
    d = np.empty(n, dtype=np.int64)
    _ind(n, len(cols), _c64(cols), _c64(counts), d)
    return d


def zero_columns(n, row_offsets, cols, counts, d_in):
    ro = np.empty(n + 1, dtype=np.int64)
    oc = np.empty(max(len(cols), 1), dtype=np.int64)
    ocnt = np.empty(max(len(cols), 1), dtype=np.int64)
    nz = _zc(n, _c64(row_offsets), _c64(cols), _c64(counts), _c64(d_in), ro, oc, ocnt)
    return ro, oc[:nz].copy(), ocnt[:nz].copy()


def row_normalize(n, row_offsets, counts):
    v = np.zeros(max(len(counts), 1), dtype=np.float64)
    _rn(n, _c64(row_offsets), _c64(counts), v)
    return v[: len(counts)]


def ref_write_edges(uv, directory: str, num_files: int, scale: int, sorted_by_start=False):
    """The reference's write_edges (edge_io.cpp:191-196)."""
    _need_ref()
    f = _sig(_ref, "ref_write_edges", C.c_int, [_i64p, C.c_int64, C.c_char_p, C.c_int, C.c_int, C.c_int])
    uv = np.ascontiguousarray(uv, dtype=np.int64).reshape(-1, 2)
    if f(uv, len(uv), directory.encode(), num_files, scale, int(sorted_by_start)):
        raise RuntimeError(_ref.ref_last_error().decode())
