"""CPU ORACLE wrapper -- test infrastructure only.

Loads ``oracle/libmns_oracle.so`` (a literal fp64 restatement of the reference
``mnscodec`` hot path, see ``mns_oracle.c``) and exposes it with numpy arrays.
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and the ``--impl reference`` arm) may import this module,
and only as the checker / the timed CPU baseline.  The product package
``paper_1501_02894_b200`` never imports it.

Reference functions restated (file:line in /root/reference/pkg/src/mnscodec):
  encode_quadtree_records  <- encoder.py:215-246 (+ try_phase1 :145-166, try_phase2 :169-212)
  decode_units             <- decoder.py:37-77 (+ transform.py:63-66 apply_map)
  full_search              <- encoder.py:249-309
  local_search             <- encoder.py:312-347
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libmns_oracle.so")
_lib = None


class EncCfg(ctypes.Structure):
    _fields_ = [
        ("e", ctypes.c_double * 3),
        ("mean_tol", ctypes.c_double),
        ("mns", ctypes.c_int),
        ("root_level", ctypes.c_int),
        ("n_iso", ctypes.c_int),
    ]


UNIT_DTYPE = np.dtype(
    [("x", "<i4"), ("y", "<i4"), ("size", "<i4"), ("dx", "<i4"), ("dy", "<i4"), ("s", "<f8"), ("o", "<f8")],
    align=True,
)
assert UNIT_DTYPE.itemsize == 40


def build() -> str:
    """Compile the oracle with its Makefile (gcc only; no reference sources are used)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        L.orc_encode_quadtree.restype = ctypes.c_int64
        L.orc_encode_quadtree.argtypes = [P, ctypes.c_int, ctypes.c_int, ctypes.POINTER(EncCfg), P,
                                          ctypes.c_int64, P, ctypes.c_int]
        for name in ("orc_try_phase1", "orc_try_phase2"):
            f = getattr(L, name)
            f.restype = ctypes.c_int
            f.argtypes = [P, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                          ctypes.POINTER(EncCfg), P, P]
        L.orc_records_to_units.restype = ctypes.c_int64
        L.orc_records_to_units.argtypes = [P, ctypes.c_int64, ctypes.c_int, ctypes.c_int, P]
        L.orc_decode.restype = ctypes.c_int
        L.orc_decode.argtypes = [P, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                 ctypes.c_double, P, P, ctypes.c_int]
        L.orc_decode_step.restype = None
        L.orc_decode_step.argtypes = [P, ctypes.c_int64, ctypes.c_int, ctypes.c_int, P, P, ctypes.c_int]
        L.orc_full_search.restype = ctypes.c_int
        L.orc_full_search.argtypes = [P, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, P,
                                      ctypes.c_int64, P, P, P, P, ctypes.c_int]
        L.orc_local_search.restype = ctypes.c_int
        L.orc_local_search.argtypes = [P, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, P, P, P, P, P,
                                       ctypes.c_int]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def default_threads() -> int:
    return max(1, len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1))


def pad(pixels: np.ndarray, m: int) -> np.ndarray:
    """image.py:123-132 pad_to_multiple (edge replication)."""
    h, w = pixels.shape
    nh, nw = -(-h // m) * m, -(-w // m) * m
    if (nh, nw) == (h, w):
        return np.ascontiguousarray(pixels, dtype=np.uint8)
    return np.ascontiguousarray(np.pad(pixels, ((0, nh - h), (0, nw - w)), mode="edge"), dtype=np.uint8)


def _cfg(e, mean_tol, mns, root_level, n_iso=1) -> EncCfg:
    c = EncCfg()
    c.n_iso = int(n_iso)
    for i in range(3):
        c.e[i] = float(e[i])
    c.mean_tol = float(mean_tol)
    c.mns = 1 if mns else 0
    c.root_level = int(root_level)
    return c


def encode_quadtree_records(pixels: np.ndarray, e=(8.0, 8.0, 8.0), mean_tol=16.0, mns=True, root_level=1,
                            nthreads=None, n_iso=1):
    """Packed leaf records (include/mns_record.h) of the reference quadtree encode of the
    16-padded image, plus per-root leaf counts."""
    img = pad(np.asarray(pixels, dtype=np.uint8), 16)
    h, w = img.shape
    nroots = (w // 16) * (h // 16)
    cap = nroots * 64
    out = np.empty(cap, dtype=np.uint64)
    counts = np.empty(nroots, dtype=np.int32)
    cfg = _cfg(e, mean_tol, mns, root_level, n_iso)
    n = lib().orc_encode_quadtree(_ptr(img), w, h, ctypes.byref(cfg), _ptr(out), cap, _ptr(counts),
                                  nthreads or default_threads())
    if n < 0:
        raise RuntimeError("oracle record buffer too small")
    return out[:n].copy(), counts


def try_phase(phase: int, pixels: np.ndarray, x: int, y: int, size: int, level: int, e=(8.0, 8.0, 8.0),
              mean_tol=16.0):
    img = np.ascontiguousarray(pixels, dtype=np.uint8)
    h, w = img.shape
    cfg = _cfg(e, mean_tol, True, 1)
    rec = np.zeros(1, dtype=np.uint64)
    rms = np.zeros(1, dtype=np.float64)
    fn = lib().orc_try_phase1 if phase == 1 else lib().orc_try_phase2
    ok = fn(_ptr(img), w, h, x, y, size, level, ctypes.byref(cfg), _ptr(rec), _ptr(rms))
    return (int(rec[0]) if ok else None), float(rms[0])


def records_to_units(records: np.ndarray, w: int, h: int) -> np.ndarray:
    rec = np.ascontiguousarray(records, dtype=np.uint64)
    units = np.empty(len(rec) * 4, dtype=UNIT_DTYPE)
    n = lib().orc_records_to_units(_ptr(rec), len(rec), w, h, _ptr(units))
    return units[:n].copy()


def decode_units(units: np.ndarray, w: int, h: int, max_iters=10, stop_delta=0.5, initial_value=128.0,
                 nthreads=None):
    """decoder.py:66-77 over the padded raster. Returns (uint8 padded image, fp64 raster, sweeps)."""
    u = np.ascontiguousarray(units, dtype=UNIT_DTYPE)
    out = np.empty((h, w), dtype=np.uint8)
    raster = np.empty((h, w), dtype=np.float64)
    it = lib().orc_decode(_ptr(u), len(u), w, h, int(max_iters), float(stop_delta), float(initial_value),
                          _ptr(out), _ptr(raster), nthreads or default_threads())
    return out, raster, it


def decode_step_units(units: np.ndarray, current: np.ndarray, nthreads=None) -> np.ndarray:
    cur = np.ascontiguousarray(current, dtype=np.float64)
    h, w = cur.shape
    out = np.empty_like(cur)
    u = np.ascontiguousarray(units, dtype=UNIT_DTYPE)
    lib().orc_decode_step(_ptr(u), len(u), w, h, _ptr(cur), _ptr(out), nthreads or default_threads())
    return out


def decode_records(records: np.ndarray, w: int, h: int, **kw):
    return decode_units(records_to_units(records, w, h), w, h, **kw)


def full_search(pixels: np.ndarray, B: int = 8, step: int = 1, n_iso: int = 1, range_ids=None, nthreads=None):
    """encoder.py:249-309 over the B-padded image.  Returns dict of per-range arrays
    (range ids in raster order): dom (domain index on the stride lattice), iso, o, code."""
    img = pad(np.asarray(pixels, dtype=np.uint8), B)
    h, w = img.shape
    nranges = (w // B) * (h // B)
    ids = np.arange(nranges, dtype=np.int32) if range_ids is None else np.ascontiguousarray(range_ids, np.int32)
    n = len(ids)
    dom = np.empty(n, np.int32)
    iso = np.empty(n, np.int8)
    o = np.empty(n, np.uint8)
    code = np.empty(n, np.uint8)
    lib().orc_full_search(_ptr(img), w, h, B, step, n_iso, _ptr(ids), n, _ptr(dom), _ptr(iso), _ptr(o),
                          _ptr(code), nthreads or default_threads())
    ndx = (w - 2 * B) // step + 1
    return {"range_ids": ids, "dom": dom, "dom_x": (dom % ndx) * step, "dom_y": (dom // ndx) * step,
            "iso": iso, "o": o, "code": code, "padded_w": w, "padded_h": h}


def local_search(pixels: np.ndarray, radius: int = 4, nthreads=None, n_iso: int = 1):
    """encoder.py:312-347 over the 8-padded image (radius 4, n_iso 1 = the reference)."""
    img = pad(np.asarray(pixels, dtype=np.uint8), 8)
    h, w = img.shape
    n = (w // 8) * (h // 8)
    dx = np.empty(n, np.int32)
    dy = np.empty(n, np.int32)
    iso = np.empty(n, np.int8)
    o = np.empty(n, np.uint8)
    code = np.empty(n, np.uint8)
    lib().orc_local_search(_ptr(img), w, h, int(radius), int(n_iso), _ptr(dx), _ptr(dy), _ptr(iso), _ptr(o),
                           _ptr(code), nthreads or default_threads())
    return {"dom_x": dx, "dom_y": dy, "iso": iso, "o": o, "code": code, "padded_w": w, "padded_h": h}


# ---------------------------------------------------------------- records

def unpack_records(records: np.ndarray) -> dict:
    r = np.asarray(records, dtype=np.uint64)
    f = lambda s, m: ((r >> np.uint64(s)) & np.uint64(m)).astype(np.int64)  # noqa: E731
    d = [f(41 + 6 * j, 63) for j in range(3)]
    d = [np.where(v >= 32, v - 64, v) for v in d]
    return {
        "x": f(0, 0x7FFF) * 2, "y": f(15, 0x7FFF) * 2, "level": f(30, 3) + 1, "phase2": f(32, 1),
        "o": f(33, 0xFF), "s_code": f(41, 7), "d0": d[0], "d1": d[1], "d2": d[2], "s_bits": f(59, 15),
    }
