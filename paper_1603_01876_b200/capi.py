"""ctypes binding of lib/libprg.so (the C-ABI in include/prg.h).

Product-side Python access to the device path: functions take torch CUDA
tensors (device entry points) or numpy arrays (host entry points). There is no
fallback: if the native library is missing or no GPU is present, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# PRG_LIB: an alternative build of the same library (A/B measurements)
LIB_PATH = os.environ.get("PRG_LIB") or os.path.join(_HERE, "lib", "libprg.so")

PRG_OK = 0
PRG_ERRORS = {
    -1: "invalid argument",
    -2: "label out of range",
    -3: "unsorted input",
    -4: "CUDA error",
    -5: "internal error",
}

HEADER_SYMBOLS = (
    "prg_last_error", "prg_version", "prg_device_count", "prg_k0_permutation",
    "prg_k0_generate_device", "prg_k1_sort_device", "prg_k1_sort_host", "prg_k2_filter_device",
    "prg_k2_filter_host", "prg_matrix_info", "prg_matrix_download", "prg_matrix_device_arrays",
    "prg_matrix_build_csc", "prg_matrix_drop_csc", "prg_matrix_has_csc",
    "prg_matrix_from_host", "prg_matrix_destroy", "prg_k3_pagerank_device", "prg_k3_pagerank_host",
    "prg_init_rank_device", "prg_pagerank_step_device", "prg_launch_count", "prg_debug_check_failures",
    "prg_last_h2d_bytes", "prg_profile_enable",
    "prg_profile_report", "prg_build_adjacency_host", "prg_in_degree_host", "prg_zero_columns_host",
    "prg_row_normalize_host", "prg_init_rank_host", "prg_pagerank_step_host", "prg_k3_pagerank_matrix_host",
    "prg_run_to_convergence_host", "prg_trim_memory", "prg_k1_sort_streamed", "prg_k3_pagerank_sharded",
    "prg_k3_shard_bounds", "prg_shard_bounds_host",
)


class PrgError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{PRG_ERRORS.get(code, code)}: {msg}")
        self.code = code


_lib: Optional[C.CDLL] = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"native library {LIB_PATH} is not built; run paper_1603_01876_b200.build")
        L = C.CDLL(LIB_PATH)
        vp, i64, i32, u64, f64 = C.c_void_p, C.c_int64, C.c_int32, C.c_uint64, C.c_double
        pp = C.POINTER(C.c_void_p)
        sig = {
            "prg_last_error": (C.c_char_p, []),
            "prg_version": (C.c_char_p, []),
            "prg_device_count": (i32, []),
            "prg_k0_permutation": (i32, [i32, u64, vp]),
            "prg_k0_generate_device": (i32, [i32, i64, u64, vp, vp, i64, i64, vp, vp]),
            "prg_k1_sort_device": (i32, [vp, i64, i32, vp, vp]),
            "prg_k1_sort_host": (i32, [vp, i64, i32, vp]),
            "prg_k2_filter_device": (i32, [vp, i64, i64, pp, vp]),
            "prg_k2_filter_host": (i32, [vp, i64, i64, pp]),
            "prg_matrix_info": (i32, [vp, vp, vp, vp, vp]),
            "prg_matrix_download": (i32, [vp, vp, vp, vp, vp]),
            "prg_matrix_device_arrays": (i32, [vp, vp, vp, vp, vp]),
            "prg_matrix_from_host": (i32, [i64, i64, vp, vp, vp, pp]),
            "prg_matrix_destroy": (None, [vp]),
            "prg_matrix_build_csc": (i32, [vp, vp]),
            "prg_matrix_drop_csc": (i32, [vp]),
            "prg_matrix_has_csc": (i32, [vp]),
            "prg_k3_pagerank_device": (i32, [vp, f64, i32, u64, i32, vp, vp, vp]),
            "prg_k3_pagerank_host": (i32, [i64, i64, vp, vp, vp, f64, i32, u64, i32, vp, vp]),
            "prg_init_rank_device": (i32, [i64, u64, i32, vp, vp, vp]),
            "prg_pagerank_step_device": (i32, [vp, vp, f64, i32, vp, vp, vp]),
            "prg_launch_count": (i64, []),
            "prg_debug_check_failures": (i64, []),
            "prg_last_h2d_bytes": (i64, []),
            "prg_profile_enable": (None, [i32]),
            "prg_profile_report": (i64, [vp, i64, i32]),
            "prg_build_adjacency_host": (i32, [vp, i64, i64, vp, vp, vp, vp]),
            "prg_in_degree_host": (i32, [i64, i64, vp, vp, vp]),
            "prg_zero_columns_host": (i32, [i64, i64, vp, vp, vp, vp, vp, vp, vp, vp]),
            "prg_row_normalize_host": (i32, [i64, i64, vp, vp, vp]),
            "prg_init_rank_host": (i32, [i64, u64, i32, vp, vp]),
            "prg_pagerank_step_host": (i32, [i64, i64, vp, vp, vp, vp, f64, i32, vp, vp]),
            "prg_k3_pagerank_matrix_host": (i32, [vp, f64, i32, u64, i32, vp, vp]),
            "prg_run_to_convergence_host": (i32, [i64, i64, vp, vp, vp, f64, f64, i32, vp, vp, vp, vp]),
            "prg_trim_memory": (i32, []),
            "prg_k1_sort_streamed": (i32, [vp, vp, vp, i64, i32, i64]),
            "prg_k3_pagerank_sharded": (i32, [vp, f64, i32, u64, i32, i32, vp, vp, vp, vp, vp]),
            "prg_k3_shard_bounds": (i32, [vp, i32, vp, vp]),
            "prg_shard_bounds_host": (i32, [vp, C.c_uint32, i32, vp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(rc: int) -> None:
    if rc != PRG_OK:
        raise PrgError(rc, lib().prg_last_error().decode())


def _ptr(a) -> int:
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data


def _stream(stream) -> int:
    if stream is None:
        import torch

        return torch.cuda.current_stream().cuda_stream
    return getattr(stream, "cuda_stream", stream)


def trim_memory() -> None:
    """Return the library pool's unused device memory to the driver (prg_trim_memory)."""
    _check(lib().prg_trim_memory())


# ---- K0 -------------------------------------------------------------------
def k0_permutation(scale: int, seed: int) -> np.ndarray:
    out = np.empty(1 << scale, dtype=np.int64)
    _check(lib().prg_k0_permutation(scale, seed, _ptr(out)))
    return out


def k0_generate(scale: int, seed: int, initiator=(0.57, 0.19, 0.19, 0.05), permute: bool = True,
                edge_factor: int = 16, device="cuda", stream=None):
    """The reference's K0 edge list (graph_gen.cpp:60-111) as an (M, 2) int64 CUDA tensor."""
    import torch

    m = edge_factor << scale
    init = np.asarray(initiator, dtype=np.float64)
    labels = None
    if permute:
        labels = torch.from_numpy(k0_permutation(scale, seed)).to(device)
    uv = torch.empty((m, 2), dtype=torch.int64, device=device)
    _check(lib().prg_k0_generate_device(scale, edge_factor, seed, _ptr(init), _ptr(labels), 0, m, _ptr(uv),
                                        _stream(stream)))
    torch.cuda.current_stream().synchronize() if stream is None else None
    return uv


# ---- K1 -------------------------------------------------------------------
def k1_sort(uv, scale: int, out=None, stream=None):
    """Device K1: (M,2) int64 CUDA tensor sorted by (u, v)."""
    import torch

    if out is None:
        out = torch.empty_like(uv)
    _check(lib().prg_k1_sort_device(_ptr(uv), uv.shape[0], scale, _ptr(out), _stream(stream)))
    return out


def k1_sort_host(uv: np.ndarray, scale: int) -> np.ndarray:
    uv = np.ascontiguousarray(uv, dtype=np.int64).reshape(-1, 2)
    out = np.empty_like(uv)
    _check(lib().prg_k1_sort_host(_ptr(uv), len(uv), scale, _ptr(out)))
    return out


# ---- K2 / matrix ------------------------------------------------------------
class DeviceMatrix:
    """Owning wrapper of a prg_matrix handle (device CSR)."""

    def __init__(self, handle: int):
        self.handle = handle
        n, nnz, raw, mx = (C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64())
        _check(lib().prg_matrix_info(handle, C.byref(n), C.byref(nnz), C.byref(raw), C.byref(mx)))
        self.n, self.nnz, self.nnz_raw, self.max_in = n.value, nnz.value, raw.value, mx.value

    def download(self):
        ro = np.empty(self.n + 1, dtype=np.int64)
        cols = np.empty(max(self.nnz, 1), dtype=np.int64)
        vals = np.empty(max(self.nnz, 1), dtype=np.float64)
        din = np.empty(self.n, dtype=np.int64)
        _check(lib().prg_matrix_download(self.handle, _ptr(ro), _ptr(cols), _ptr(vals), _ptr(din)))
        return ro, cols[: self.nnz], vals[: self.nnz], din

    def device_views(self):
        """Zero-copy torch views of the device arrays (prg_matrix_device_arrays):
        (row_offsets u32[n+1], cols u32[nnz], values f64[nnz], d_in u32[n] or None),
        the u32 arrays viewed as int32 (every value is < 2^31 up to S=30)."""
        import torch

        ro, cols, vals, din = (C.c_void_p(), C.c_void_p(), C.c_void_p(), C.c_void_p())
        _check(lib().prg_matrix_device_arrays(self.handle, C.byref(ro), C.byref(cols), C.byref(vals), C.byref(din)))

        class _View:
            def __init__(self, ptr, count, typestr):
                self.__cuda_array_interface__ = {"shape": (count,), "typestr": typestr, "data": (ptr or 0, False),
                                                 "version": 3, "strides": None}

        def view(p, count, typestr):
            if count == 0 or not p.value:
                return torch.empty(0, dtype=torch.float64 if typestr == "<f8" else torch.int32, device="cuda")
            return torch.as_tensor(_View(p.value, count, typestr), device="cuda")

        return (view(ro, self.n + 1, "<i4"), view(cols, self.nnz, "<i4"), view(vals, self.nnz, "<f8"),
                view(din, self.n, "<i4") if din.value else None)

    def build_csc(self, stream=None) -> "DeviceMatrix":
        """K2's CSC build: keep K3's column layout on the handle (prg_matrix_build_csc)."""
        _check(lib().prg_matrix_build_csc(self.handle, _stream(stream)))
        return self

    def drop_csc(self) -> None:
        _check(lib().prg_matrix_drop_csc(self.handle))

    @property
    def has_csc(self) -> bool:
        return bool(lib().prg_matrix_has_csc(self.handle))

    def close(self):
        if self.handle:
            lib().prg_matrix_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def from_host(n: int, row_offsets, cols, values) -> "DeviceMatrix":
        ro = np.ascontiguousarray(row_offsets, dtype=np.int64)
        c = np.ascontiguousarray(cols, dtype=np.int64)
        v = np.ascontiguousarray(values, dtype=np.float64)
        h = C.c_void_p()
        _check(lib().prg_matrix_from_host(n, len(c), _ptr(ro), _ptr(c), _ptr(v), C.byref(h)))
        return DeviceMatrix(h.value)


def k2_filter(uv_sorted, n: int, stream=None, csc: bool = False) -> DeviceMatrix:
    """Device K2. csc=True also runs K2's CSC build (the layout K3 iterates over)."""
    h = C.c_void_p()
    _check(lib().prg_k2_filter_device(_ptr(uv_sorted), uv_sorted.shape[0], n, C.byref(h), _stream(stream)))
    m = DeviceMatrix(h.value)
    if csc:
        m.build_csc(stream)
    return m


def k2_filter_host(uv_sorted: np.ndarray, n: int) -> DeviceMatrix:
    uv = np.ascontiguousarray(uv_sorted, dtype=np.int64).reshape(-1, 2)
    h = C.c_void_p()
    _check(lib().prg_k2_filter_host(_ptr(uv), len(uv), n, C.byref(h)))
    return DeviceMatrix(h.value)


# ---- K3 -------------------------------------------------------------------
def k3_pagerank(mat: DeviceMatrix, damping=0.85, iterations=20, seed=0, mode=0, out=None, stream=None):
    """Device K3 (run_kernel3): returns (ranks CUDA tensor, norm1)."""
    import torch

    if out is None:
        out = torch.empty(mat.n, dtype=torch.float64, device="cuda")
    norm = C.c_double()
    _check(lib().prg_k3_pagerank_device(mat.handle, damping, iterations, seed, mode, _ptr(out), C.byref(norm),
                                        _stream(stream)))
    return out, norm.value


def k3_pagerank_host(n, row_offsets, cols, values, damping=0.85, iterations=20, seed=0, mode=0):
    ro = np.ascontiguousarray(row_offsets, dtype=np.int64)
    c = np.ascontiguousarray(cols, dtype=np.int64)
    v = np.ascontiguousarray(values, dtype=np.float64)
    r = np.empty(n, dtype=np.float64)
    norm = C.c_double()
    _check(lib().prg_k3_pagerank_host(n, len(c), _ptr(ro), _ptr(c), _ptr(v), damping, iterations, seed, mode,
                                      _ptr(r), C.byref(norm)))
    return r, norm.value


# ---- multi-GPU K3 -------------------------------------------------------------
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p)


def device_f64_view(ptr: int, count: int):
    """Zero-copy torch view of `count` device doubles at `ptr`."""
    import torch

    class _View:
        __cuda_array_interface__ = {"shape": (count,), "typestr": "<f8", "data": (ptr, False), "version": 3,
                                    "strides": None}

    return torch.as_tensor(_View(), device="cuda")


def torch_allreduce(group=None):
    """The exchange prg_k3_pagerank_sharded needs, as torch.distributed does it:
    an in-place all_reduce(SUM) of the buffer (NCCL on GPUs, gloo on CPU
    tensors), ordered after the library's kernels on the caller's stream."""
    import torch.distributed as dist

    def allreduce(buf, stream=None):
        if buf.is_cuda and stream:
            import torch

            with torch.cuda.stream(torch.cuda.ExternalStream(stream)):  # ordered after the SpMV
                dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
        else:
            dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)

    return allreduce


def shard_bounds_host(slice_ptr, world: int) -> np.ndarray:
    """The sharded K3's partition rule (prg_shard_bounds_host) on host slice offsets."""
    sp = np.ascontiguousarray(slice_ptr, dtype=np.uint32)
    out = np.empty(world + 1, dtype=np.uint32)
    _check(lib().prg_shard_bounds_host(_ptr(sp), len(sp) - 1, world, _ptr(out)))
    return out


def k3_shard_bounds(mat: "DeviceMatrix", world: int, stream=None) -> np.ndarray:
    out = np.empty(world + 1, dtype=np.uint32)
    _check(lib().prg_k3_shard_bounds(mat.handle, world, _ptr(out), _stream(stream)))
    return out


def k3_pagerank_sharded(mat: "DeviceMatrix", rank: int, world: int, allreduce, damping=0.85, iterations=20, seed=0,
                        out=None, stream=None):
    """Column-sharded K3 (prg_k3_pagerank_sharded): this process's share of a
    world-GPU run_kernel3; `allreduce(tensor, stream)` sums a CUDA tensor over
    the ranks in place. Returns (ranks CUDA tensor — complete on every rank,
    norm1); bit-identical to k3_pagerank(mode=0)."""
    import torch

    if out is None:
        out = torch.empty(mat.n, dtype=torch.float64, device="cuda")
    failure = []

    def cb(_user, buf, count, strm):
        try:
            allreduce(device_f64_view(buf, count), strm)
            return 0
        except BaseException as e:  # noqa: BLE001 - reported after the call
            failure.append(e)
            return 1

    fn = ALLREDUCE_FN(cb)
    norm = C.c_double()
    rc = lib().prg_k3_pagerank_sharded(mat.handle, damping, iterations, seed, rank, world, fn, None, _ptr(out),
                                       C.byref(norm), _stream(stream))
    if failure:
        raise failure[0]
    _check(rc)
    return out, norm.value


def init_rank(n: int, seed: int, mode=0, stream=None):
    import torch

    out = torch.empty(n, dtype=torch.float64, device="cuda")
    norm = C.c_double()
    _check(lib().prg_init_rank_device(n, seed, mode, _ptr(out), C.byref(norm), _stream(stream)))
    return out, norm.value


def pagerank_step(mat: DeviceMatrix, r, damping=0.85, mode=0, stream=None):
    import torch

    out = torch.empty_like(r)
    norm = C.c_double()
    _check(lib().prg_pagerank_step_device(mat.handle, _ptr(r), damping, mode, _ptr(out), C.byref(norm),
                                          _stream(stream)))
    return out, norm.value
