"""ctypes binding of libmns_b200.so (include/mns_b200.h).

PyTorch is used only for device memory and streams; every computation on the
hot path is one of the library's sm_100a kernels.  There is deliberately no
CPU fallback: if the library or a CUDA device is missing, calls raise.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MNS_B200_LIB") or os.path.join(_HERE, "libmns_b200.so")  # env: debug builds only
CSRC = os.path.join(_HERE, "csrc")
INCLUDE = os.path.join(os.path.dirname(_HERE), "include")

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-Xcompiler",
              "-fPIC", "-shared"]

_lib = None
_lock = threading.Lock()


class NativeError(RuntimeError):
    """A CUDA / argument error reported by libmns_b200 (mns_last_error)."""


class EncCfg(ctypes.Structure):
    _fields_ = [("e", ctypes.c_double * 3), ("mean_tol", ctypes.c_double), ("mns", ctypes.c_int32),
                ("root_level", ctypes.c_int32), ("n_iso", ctypes.c_int32), ("map_form", ctypes.c_int32)]


def sources() -> list[str]:
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def build(verbose: bool = False) -> str:
    """Compile every CUDA source for sm_100a into the in-tree shared library."""
    cmd = ["nvcc", *NVCC_FLAGS, "-o", LIB_PATH, *sources()]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    return LIB_PATH


def _declare(L):
    P, I32, I64, D, F = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_float
    sig = {
        "mns_encode_workspace_bytes": [I32, I32, I32, I32, P],
        "mns_encode_quadtree": [P, I32, I32, I64, I64, I32, I32, I32, ctypes.POINTER(EncCfg), P, I64, P, P, P, P,
                                I64, P],
        "mns_encode_quadtree_split": [P, I32, I32, I64, I64, I32, I32, I32, ctypes.POINTER(EncCfg), P, I64, P, P,
                                      P, P, I64, P, P],
        "mns_build_unit_map": [P, P, I32, I32, I32, P, P],
        "mns_build_block_map": [P, P, I32, I32, I32, P, P],
        "mns_try_node": [P, I32, I32, I64, I32, I32, I32, I32, ctypes.POINTER(EncCfg), P, P, P],
        "mns_decode_workspace_bytes": [I32, I32, P],
        "mns_decode_quadtree": [P, P, I32, I32, I32, D, F, P, P, P, P, P, I64, P],
        "mns_decode_unit_map": [P, I32, I32, I32, D, F, P, P, P, P, P, I64, P],
        "mns_decode_sweep": [P, I32, I32, I32, I32, P, F, P, P, P, D, P],
        "mns_decode_sweep2": [P, I32, I32, I32, I32, I32, P, F, P, P, P],
        "mns_decode_pass_lattice": [P, I32, I32, I32, I32, I32, P, F, P, P, P, P],
        "mns_decode_flat_lattice": [P, I32, I32, I32, I32, I32, F, P, P, P],
        "mns_decode_quadtree_lattice": [P, P, I32, I32, I32, F, P, P, P, P, P, I64, P],
        "mns_decode_unit_map_lattice": [P, I32, I32, I32, F, P, P, P, P, P, I64, P],
        "mns_decode_units": [P, P, P, P, P, P, P, I64, I32, I32, I32, D, F, P, P, P, P, P, I64, P],
        "mns_decode_step_f64": [P, P, P, P, P, P, P, I64, I32, I32, P, P, P],
        "mns_decode_f64": [P, P, P, P, P, P, P, I64, I32, I32, I32, D, D, P, P, P, P, P, I64, P],
        "mns_records_to_units": [P, I64, I32, I32, P, P, P, P, P, P, P, P],
        "mns_decode_f64_sweep": [P, P, P, P, P, P, P, I64, I32, P, P, P, P],
        "mns_decode_f64_decide": [P, D, P],
        "mns_decode_f64_finalize": [P, P, P, I32, I32, I32, P, P, P],
        "mns_search_workspace_bytes": [I32, I32, I32, I32, I32, P],
        "mns_full_search": [P, I32, I32, I32, I32, I32, I32, I32, P, P, P, P, P, I64, P],
        "mns_local_search": [P, I32, I32, I32, I32, P, P, P, P, P, P],
        "mns_local_search_workspace_bytes": [I32, I32, I32, I32, P],
        "mns_local_search_tc": [P, I32, I32, I32, I32, P, P, P, P, P, P, I64, P],
        "mns_stream_workspace_bytes": [I64, P],
        "mns_write_stream": [P, I64, I32, I32, I32, I32, I32, I32, P, I64, P, P, I64, P],
        "mns_read_stream_workspace_bytes": [I64, P],
        "mns_read_stream": [P, I64, I32, I32, I32, I32, P, I64, P, P, P, P, I64, P],
        "mns_image_sse": [P, I64, P, I64, I32, I32, P, P],
        "mns_code_stats": [P, I64, P, P],
        "mns_offset_histogram": [P, I64, I32, I32, I32, I32, P, P, P, P],
        "mns_version": [],
    }
    for name, args in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = ctypes.c_int
    L.mns_last_error.argtypes = []
    L.mns_last_error.restype = ctypes.c_char_p
    return L


EXPORTS = ("mns_encode_workspace_bytes", "mns_encode_quadtree", "mns_encode_quadtree_split", "mns_try_node", "mns_build_unit_map", "mns_build_block_map", "mns_decode_workspace_bytes", "mns_decode_quadtree", "mns_decode_unit_map",
           "mns_decode_sweep", "mns_decode_sweep2", "mns_decode_pass_lattice",
           "mns_decode_flat_lattice", "mns_decode_quadtree_lattice", "mns_decode_unit_map_lattice", "mns_decode_units", "mns_decode_step_f64",
           "mns_decode_f64", "mns_records_to_units", "mns_decode_f64_sweep", "mns_decode_f64_decide",
           "mns_decode_f64_finalize", "mns_search_workspace_bytes", "mns_full_search",
           "mns_local_search", "mns_local_search_workspace_bytes", "mns_local_search_tc", "mns_stream_workspace_bytes", "mns_write_stream", "mns_read_stream_workspace_bytes", "mns_read_stream",
           "mns_image_sse", "mns_code_stats", "mns_offset_histogram",
           "mns_last_error",
           "mns_version")


def load_library():
    """Load (no GPU needed) the in-tree library; raises if it has not been built."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
            _lib = _declare(ctypes.CDLL(LIB_PATH))
    return _lib


def lib():
    """The library, after checking that a CUDA device is present (the product path is GPU-only)."""
    import torch

    if not torch.cuda.is_available():
        raise NativeError("libmns_b200 needs a CUDA device (B200, sm_100a); no CPU fallback exists")
    return load_library()


def check(rc: int) -> None:
    if rc != 0:
        msg = load_library().mns_last_error().decode(errors="replace")
        raise NativeError(f"libmns_b200 error {rc}: {msg}")


def ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def stream_ptr(stream=None) -> ctypes.c_void_p:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def out_i64(L, fn, *args) -> int:
    v = ctypes.c_int64(0)
    check(fn(*args, ctypes.byref(v)))
    return int(v.value)
