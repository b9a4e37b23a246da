"""Loader of the in-tree C-ABI library ``libisf_lossy.so`` (include/isf_lossy.h).

The product path has no fallback: if the CUDA library is missing or fails to
load, every entry point raises.  Build it with ``python -c "import
__graft_entry__ as g; g.build()"`` (nvcc, sm_100a).
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# ISF_LOSSY_LIB: development knob to load an alternative in-tree build (variant timing)
LIB_PATH = os.environ.get("ISF_LOSSY_LIB") or os.path.join(_HERE, "libisf_lossy.so")

# every symbol declared in include/isf_lossy.h
EXPORTS = (
    "isf_lossy_plan_create", "isf_lossy_plan_destroy", "isf_lossy_stream_capacity",
    "isf_lossy_stream_header_bytes", "isf_lossy_compress_async", "isf_lossy_compress",
    "isf_lossy_decompress_async", "isf_lossy_decompress", "isf_lossy_compress_host",
    "isf_lossy_decompress_host", "isf_lossy_allreduce", "isf_lossy_allreduce_n", "isf_lossy_compression_ratio",
    "isf_lossy_last_error", "isf_lossy_error_code_name", "isf_lossy_plan_operators",
    "isf_lossy_plan_last_launches", "isf_lossy_plan_set_compress_mode", "isf_lossy_generate_tgv", "isf_lossy_generate_spectral",
    "isf_lossy_solver_standin", "isf_lossy_crc32", "isf_lossy_frame_async", "isf_lossy_frame_capacity",
)
FRAME_OVERHEAD = 62  # ISF_FRAME_OVERHEAD: 48-B header + codec trailer (10 B) + CRC (4 B); + 4 n_el + 12 K payload


class Stats(ctypes.Structure):
    """isf_lossy_stats (include/isf_lossy.h)."""
    _fields_ = [
        ("err2", ctypes.c_double), ("nrm2", ctypes.c_double),
        ("err_inf", ctypes.c_double), ("u_inf", ctypes.c_double),
        ("disc2", ctypes.c_double), ("tot2", ctypes.c_double),
        ("kept", ctypes.c_uint64), ("blocks", ctypes.c_uint64),
        ("stream_bytes", ctypes.c_uint64), ("field_bytes", ctypes.c_uint64),
        ("status", ctypes.c_uint64), ("reserved", ctypes.c_uint64),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None


def lib() -> ctypes.CDLL:
    """Load the CUDA library (raises OSError if it is absent: no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise OSError(f"{LIB_PATH} not built; run __graft_entry__.build() (no CPU fallback exists)")
    L = ctypes.CDLL(LIB_PATH)
    P, u64, u32, i32, f64 = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int, ctypes.c_double
    Sp = ctypes.POINTER(Stats)
    sig = {
        "isf_lossy_plan_create": ([ctypes.POINTER(P), u32, u32, i32], i32),
        "isf_lossy_plan_destroy": ([P], i32),
        "isf_lossy_stream_capacity": ([u32, u32, u64], u64),
        "isf_lossy_stream_header_bytes": ([u32, u32, u64], u64),
        "isf_lossy_compress_async": ([P, P, u64, f64, i32, P, u64, P, P], i32),
        "isf_lossy_compress": ([P, P, u64, f64, i32, P, u64, ctypes.POINTER(u64), Sp, P], i32),
        "isf_lossy_decompress_async": ([P, P, u64, u64, P, P, P, P], i32),
        "isf_lossy_decompress": ([P, P, u64, u64, P, P, Sp, P], i32),
        "isf_lossy_compress_host": ([P, P, u64, f64, i32, P, u64, ctypes.POINTER(u64), Sp], i32),
        "isf_lossy_decompress_host": ([P, P, u64, u64, P, P, Sp], i32),
        "isf_lossy_allreduce": ([P, P, P], i32),
        "isf_lossy_allreduce_n": ([P, u32, P, P], i32),
        "isf_lossy_compression_ratio": ([u64, u64], f64),
        "isf_lossy_last_error": ([], ctypes.c_char_p),
        "isf_lossy_error_code_name": ([i32], ctypes.c_char_p),
        "isf_lossy_plan_operators": ([P, P, P, P, P], i32),
        "isf_lossy_plan_last_launches": ([P], i32),
        "isf_lossy_plan_set_compress_mode": ([P, i32], i32),
        "isf_lossy_generate_tgv": ([P, P, u32, u32, u32, i32, f64, P], i32),
        "isf_lossy_generate_spectral": ([P, P, u64, u64, u64, P, P], i32),
        "isf_lossy_solver_standin": ([P, P, P, u64, f64, P], i32),
        "isf_lossy_crc32": ([P, P, u64, P, P], i32),
        "isf_lossy_frame_async": ([P, P, u64, P, u64, P, u32, u64, f64, P], i32),
        "isf_lossy_frame_capacity": ([u32, u32, u64], u64),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


def last_error() -> str:
    return lib().isf_lossy_last_error().decode()
