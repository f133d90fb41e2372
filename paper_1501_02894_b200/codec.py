"""Reference-API mirror of the MNS hot path on B200 (drop-in for mnscodec's encoder/decoder).

Same function names, arguments, return types and ValueError messages as the
reference (file:line citations per function); every computation runs in the
sm_100a kernels of libmns_b200.so through ``_native``.  Two layers:

* device layer (``encode_device`` / ``decode_device`` / ``full_search_device`` /
  ``local_search_device``): torch CUDA tensors in, torch CUDA tensors out,
  stream-ordered, no host synchronisation unless asked -- used by bench.py,
  the multi-GPU sharding and the host layer;
* host layer (``encode_quadtree``, ``decode``, ``decode_step``,
  ``encode_full_search``, ``encode_local_search``, ``write_stream`` ...):
  the reference's signatures over numpy / GrayImage, with H2D/D2H copies.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, replace
from typing import Optional

import numpy as np

from . import _native as N
from .types import (
    CONTRAST_SETS,
    LEVEL_SIZES,
    ROOT_SIZE,
    SIZE_LEVELS,
    BaselinePayload,
    BlockRect,
    DecodeConfig,
    EncoderConfig,
    GrayImage,
    Phase1Payload,
    Phase2Payload,
    QuadtreeCode,
    dequantize_contrast,
    unpack_leaves,
)


def _torch():
    import torch

    return torch


# ------------------------------------------------------------------ geometry (host)

def pad_to_multiple(image, m: int) -> GrayImage:
    """image.py:123-132: grow each axis to the next multiple of m by edge replication."""
    if m < 1:
        raise ValueError("padding multiple must be >= 1")
    px = _pixels(image)
    new_h = -(-px.shape[0] // m) * m
    new_w = -(-px.shape[1] // m) * m
    if (new_h, new_w) == px.shape:
        return image if isinstance(image, GrayImage) else GrayImage(px)
    return GrayImage(np.pad(px, ((0, new_h - px.shape[0]), (0, new_w - px.shape[1])), mode="edge"))


def co_domain_rect(range_rect: BlockRect, img_w: int, img_h: int) -> BlockRect:
    """image.py:174-187."""
    if range_rect.size % 2:
        raise ValueError("range size must be even")
    d = range_rect.size * 2
    if d > img_w or d > img_h:
        raise ValueError(f"no {d}x{d} domain fits a {img_w}x{img_h} image")
    x = min(max(range_rect.x - range_rect.size // 2, 0), img_w - d)
    y = min(max(range_rect.y - range_rect.size // 2, 0), img_h - d)
    return BlockRect(x, y, d)


def _pixels(image) -> np.ndarray:
    px = image.pixels if hasattr(image, "pixels") else np.asarray(image)
    if px.ndim != 2:
        raise ValueError(f"expected a 2-D pixel array, got shape {px.shape}")
    if px.dtype != np.uint8:
        px = GrayImage(px).pixels
    return px


def _padded_np(px: np.ndarray, m: int) -> np.ndarray:
    h, w = px.shape
    nh, nw = -(-h // m) * m, -(-w // m) * m
    if (nh, nw) != (h, w):
        px = np.pad(px, ((0, nh - h), (0, nw - w)), mode="edge")
    return np.ascontiguousarray(px)


# ------------------------------------------------------------------ device layer

@dataclass
class DeviceCode:
    """Packed transform code resident on the GPU (records in DFS order, grouped by root)."""

    records: "object"       # torch.int64 [capacity] (bit pattern of include/mns_record.h)
    root_offsets: "object"  # torch.int32 [n_roots + 1]
    count: "object"         # torch.int64 [1] (device) -- records[:count] are valid
    padded_w: int
    padded_h: int
    n_images: int = 1
    root_row_begin: int = 0
    root_row_end: int = 0
    mode: str = "mns"
    technique2: bool = True
    unit_map: "object" = None  # torch.int32: decoder map (mns_record.h) in map_form, optional
    min_leaf: int = 0          # smallest painted unit side if known (4: no 2x2 units -> lattice-state decode), 0 unknown
    unit_map_valid: bool = False  # unit_map holds this code's map (emitted by the encoder / build_unit_map)
    compact_event: "object" = None  # set by encode_device(compact_stream=...): records/count valid after it
    decode_error: "object" = None   # set by decode_device on the lattice path (device int32 flag)
    n_iso: int = 1                  # 8: the isometry extension (phase-1 records carry an isometry)
    map_form: int = 0               # unit_map holds 0: the unit map (32 words per root), 1: the block map (8)

    def join(self, stream=None) -> None:
        """Make `stream` (default: current) wait until records / root_offsets / count are complete
        (they are produced on the compaction stream when encode_device got one)."""
        if self.compact_event is not None:
            torch = _torch()
            (stream if stream is not None else torch.cuda.current_stream()).wait_event(self.compact_event)

    def n_records(self) -> int:
        self.join()
        return int(self.count.item())


class _Workspace:
    """Per-device cache of scratch buffers (the caching allocator would also do; this keeps the
    timed loops free of allocator calls)."""

    def __init__(self):
        self.buf = {}

    def get(self, key, nbytes, device):
        torch = _torch()
        t = self.buf.get((key, device))
        if t is None or t.numel() < nbytes:
            t = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
            self.buf[(key, device)] = t
        return t


_WS = _Workspace()


MAP_WORDS = (32, 8)  # int32 words per root of the unit map / the block map


def enc_cfg(config: EncoderConfig, root_level: int = 1, n_iso: int = 1, map_form: int = 0) -> N.EncCfg:
    c = N.EncCfg()
    c.n_iso = int(n_iso)
    c.map_form = int(map_form)
    c.e[0], c.e[1], c.e[2] = float(config.e1), float(config.e2), float(config.e3)
    c.mean_tol = float(config.mean_tol)
    c.mns = 1 if config.mode == "mns" else 0
    c.root_level = int(root_level)
    return c


def encode_device(img, config: EncoderConfig, *, root_level: int = 1, root_rows: Optional[tuple] = None,
                  height: Optional[int] = None, out: Optional[DeviceCode] = None, with_unit_map: bool = True,
                  stream=None, compact_stream=None, n_iso: int = 1, map_form: Optional[int] = None) -> DeviceCode:
    """MNS quadtree encode of a padded uint8 CUDA tensor [H, W] or a batch [B, H, W].

    root_rows=(r0, r1) restricts the work to root rows [r0, r1) (strip sharding); then ``img``
    may be a halo'd slice and ``height`` gives the full image height (global clamping).
    n_iso=8 is the isometry extension (BASELINE configs[1]): phase 1 also tries the 8 isometries of
    the co-centred domain; such codes carry no decoder unit map and decode on the exact unit path.
    map_form: the decoder map emitted beside the records -- 1, the block map of the lattice decoders
    (default for e3 = inf, whose codes have no 2x2 units), or 0, the unit map (default otherwise);
    with ``out`` given, its ``map_form``.
    """
    if n_iso not in (1, 8):
        raise ValueError("n_iso must be 1 or 8")
    torch = _torch()
    L = N.lib()
    if config.mode not in ("no_search", "mns"):
        raise ValueError(f"encode_quadtree handles no_search/mns, not {config.mode!r}")
    if img.dim() == 2:
        img = img.unsqueeze(0)
    nb, h, w = img.shape
    H = int(height) if height is not None else h
    r0, r1 = root_rows if root_rows is not None else (0, H // 16)
    n_roots = nb * (r1 - r0) * (w // 16)
    dev = img.device
    if map_form is None:
        map_form = out.map_form if out is not None else (1 if math.isinf(config.e3) and n_iso == 1 else 0)
    if map_form not in (0, 1):
        raise ValueError("map_form must be 0 (unit map) or 1 (block map)")
    if out is None:
        out = DeviceCode(torch.empty(64 * n_roots, dtype=torch.int64, device=dev),
                         torch.empty(n_roots + 1, dtype=torch.int32, device=dev),
                         torch.zeros(1, dtype=torch.int64, device=dev), w, H, nb, r0, r1, config.mode,
                         config.technique2,
                         torch.empty(MAP_WORDS[map_form] * n_roots, dtype=torch.int32, device=dev)
                         if with_unit_map else None)
    if out.unit_map is not None and out.unit_map.numel() < MAP_WORDS[map_form] * n_roots:
        raise ValueError("unit_map is too small for the requested map_form")
    out.map_form = map_form
    wsb = N.out_i64(L, L.mns_encode_workspace_bytes, w, nb, r0, r1)
    ws = _WS.get("enc", wsb, dev)
    # `img` points at global row 0 even for halo'd strips: offset the base pointer back
    base = img.data_ptr()
    if root_rows is not None and h != H:
        base -= max(0, 16 * r0 - 16) * img.stride(1)
    # e3 = inf: every visited level-3 node passes phase 1 (encoder.py:160-165, before phase 2), so no
    # leaf is 2x2 and no level-3 phase-2 leaf has 2x2 quadrants
    out.min_leaf = 4 if math.isinf(config.e3) else 0
    out.unit_map_valid = out.unit_map is not None and n_iso == 1
    out.n_iso = n_iso
    cfg = enc_cfg(config, root_level, n_iso, map_form)
    if compact_stream is None:
        N.check(L.mns_encode_quadtree(ctypes.c_void_p(base), w, H, img.stride(1), img.stride(0), nb, r0, r1,
                                      ctypes.byref(cfg), N.ptr(out.records), out.records.numel(),
                                      N.ptr(out.root_offsets), N.ptr(out.count), N.ptr(out.unit_map), N.ptr(ws),
                                      ws.numel(), N.stream_ptr(stream)))
        out.compact_event = None
    else:  # records / root_offsets / count become valid on compact_stream (the unit map on stream)
        N.check(L.mns_encode_quadtree_split(ctypes.c_void_p(base), w, H, img.stride(1), img.stride(0), nb, r0, r1,
                                            ctypes.byref(cfg), N.ptr(out.records), out.records.numel(),
                                            N.ptr(out.root_offsets), N.ptr(out.count), N.ptr(out.unit_map),
                                            N.ptr(ws), ws.numel(), N.stream_ptr(stream),
                                            N.stream_ptr(compact_stream)))
        if out.compact_event is None:
            out.compact_event = torch.cuda.Event()
        out.compact_event.record(compact_stream)
    return out


def build_unit_map(code: DeviceCode, stream=None, map_form: int = 0):
    """Decoder map of a device code from its records (map_form 0: the unit map, 1: the block map)."""
    torch = _torch()
    L = N.lib()
    r0, r1 = code.root_row_begin, code.root_row_end or code.padded_h // 16
    n_roots = (code.padded_w // 16) * (r1 - r0)
    code.unit_map = torch.empty(MAP_WORDS[map_form] * n_roots, dtype=torch.int32, device=code.records.device)
    code.map_form = map_form
    code.join(stream)
    build = L.mns_build_block_map if map_form == 1 else L.mns_build_unit_map
    N.check(build(N.ptr(code.records), N.ptr(code.root_offsets), code.padded_w, r0, r1, N.ptr(code.unit_map),
                  N.stream_ptr(stream)))
    code.unit_map_valid = True
    return code.unit_map


def min_leaf_side(code: DeviceCode) -> int:
    """Smallest unit side the decoder paints for a device code: 2 if any leaf is 2x2 or is a level-3
    phase-2 leaf (2x2 quadrants), else 4 (from the encoder's guarantee, else counted on the GPU)."""
    if not code.min_leaf:
        from .rd import unit2_leaves

        code.min_leaf = 2 if unit2_leaves(code.records, code.n_records()) else 4
    return code.min_leaf


def decode_device(code: DeviceCode, iters: int = 10, stop_delta: float = 0.0, initial_value: float = 128.0,
                  out=None, rasters=None, want_u8: bool = True, stream=None, lattice=None):
    """Jacobi decode of a device quadtree code (single image); returns (uint8 [H, W] padded, iters_done tensor).

    Codes without 2x2 units decoded to uint8 with stop_delta == 0 run on lattice state
    (mns_decode_quadtree_lattice: a quarter of the raster traffic, identical output); the rest on
    fp32 rasters (mns_decode_quadtree).  ``code.decode_error`` (device int32) is set to 1 by a lattice
    decode that met a 2x2 unit (a wrong ``min_leaf``); callers that sync check it and rerun with
    ``lattice=False`` (``decode`` does).
    """
    torch = _torch()
    L = N.lib()
    W, H = code.padded_w, code.padded_h
    dev = code.records.device
    if rasters is None:
        rasters = (torch.empty((H, W), dtype=torch.float32, device=dev),
                   torch.empty((H, W), dtype=torch.float32, device=dev))
    if out is None and want_u8:
        out = torch.empty((H, W), dtype=torch.uint8, device=dev)
    if (stop_delta > 0.0 or code.n_iso > 1) and want_u8:
        # the reference's early stop (decoder.py:70-75) decided exactly: bit-exact fp64 sweeps (also the
        # isometry extension's codes, which the unit-map decoders cannot express)
        code.decode_error = None
        return decode_device_f64(code, iters, stop_delta, initial_value, out=out, stream=stream) + (None,)
    wsb = N.out_i64(L, L.mns_decode_workspace_bytes, W, H)
    ws = _WS.get("dec", wsb, dev)
    if want_u8 and stop_delta == 0.0 and lattice is not False and min_leaf_side(code) >= 4:
        it = torch.full((1,), int(iters), dtype=torch.int32, device=dev)
        err = torch.empty(1, dtype=torch.int32, device=dev)  # zeroed by the library
        n_lat = (H // 2) * (W // 2)
        lat = (rasters[0].view(-1)[:n_lat], rasters[1].view(-1)[:n_lat])
        whole = code.n_images == 1 and code.root_row_begin == 0 and code.root_row_end in (0, H // 16)
        code.decode_error = err  # 1 if a 2x2 unit was met (min_leaf wrong): rerun with lattice=False
        if code.unit_map is not None and code.unit_map_valid and code.map_form == 1 and whole:
            # the encoder's own block map: no rebuild from the records
            N.check(L.mns_decode_unit_map_lattice(N.ptr(code.unit_map), W, H, int(iters), float(initial_value),
                                                  N.ptr(lat[0]), N.ptr(lat[1]), N.ptr(out), N.ptr(err), N.ptr(ws),
                                                  ws.numel(), N.stream_ptr(stream)))
        else:
            code.join(stream)
            N.check(L.mns_decode_quadtree_lattice(N.ptr(code.records), N.ptr(code.root_offsets), W, H, int(iters),
                                                  float(initial_value), N.ptr(lat[0]), N.ptr(lat[1]), N.ptr(out),
                                                  N.ptr(err), N.ptr(ws), ws.numel(), N.stream_ptr(stream)))
        return out, it, rasters
    it = torch.zeros(1, dtype=torch.int32, device=dev)
    code.decode_error = None
    whole = code.n_images == 1 and code.root_row_begin == 0 and code.root_row_end in (0, H // 16)
    if code.unit_map is not None and code.unit_map_valid and code.map_form == 0 and whole:
        # the encoder's own unit map: no rebuild from the records
        N.check(L.mns_decode_unit_map(N.ptr(code.unit_map), W, H, int(iters), float(stop_delta),
                                      float(initial_value), N.ptr(rasters[0]), N.ptr(rasters[1]), N.ptr(out),
                                      N.ptr(it), N.ptr(ws), ws.numel(), N.stream_ptr(stream)))
        return out, it, rasters
    code.join(stream)
    N.check(L.mns_decode_quadtree(N.ptr(code.records), N.ptr(code.root_offsets), W, H, int(iters), float(stop_delta),
                                  float(initial_value), N.ptr(rasters[0]), N.ptr(rasters[1]), N.ptr(out), N.ptr(it),
                                  N.ptr(ws), ws.numel(), N.stream_ptr(stream)))
    return out, it, rasters


def records_to_units_device(records, n: int, W: int, H: int, stream=None) -> dict:
    """Packed records -> 4n painted-unit slots (decoder.py:48-59) on the device (mns_records_to_units):
    slot i = record i's first unit, slots n + 3i .. n + 3i + 2 = quadrants 1..3 of a phase-2 record."""
    torch = _torch()
    L = N.lib()
    dev = records.device
    u = {k: torch.empty(max(4 * n, 1), dtype=torch.int32, device=dev) for k in ("x", "y", "size", "dx", "dy")}
    u["s"] = torch.empty(max(4 * n, 1), dtype=torch.float64, device=dev)
    u["o"] = torch.empty(max(4 * n, 1), dtype=torch.float64, device=dev)
    N.check(L.mns_records_to_units(N.ptr(records), int(n), W, H, N.ptr(u["x"]), N.ptr(u["y"]), N.ptr(u["size"]),
                                   N.ptr(u["dx"]), N.ptr(u["dy"]), N.ptr(u["s"]), N.ptr(u["o"]),
                                   N.stream_ptr(stream)))
    u["n"] = 4 * n
    return u


def decode_units_f64(units: dict, W: int, H: int, iters: int, stop_delta: float, initial_value: float, out=None,
                     stream=None):
    """decoder.py:66-77 bit for bit (mns_decode_f64): fp64 sweeps, exact early stop, exact rounding.
    Returns (uint8 [H, W] padded, sweeps-done int32 tensor)."""
    torch = _torch()
    L = N.lib()
    if iters < 1:
        raise ValueError("max_iters must be >= 1")
    dev = units["x"].device
    ping = torch.empty((H, W), dtype=torch.float64, device=dev)
    pong = torch.empty((H, W), dtype=torch.float64, device=dev)
    if out is None:
        out = torch.empty((H, W), dtype=torch.uint8, device=dev)
    it = torch.zeros(1, dtype=torch.int32, device=dev)
    ws = _WS.get("decf64", 64, dev)
    n = int(units.get("n", units["x"].numel()))
    N.check(L.mns_decode_f64(N.ptr(units["x"]), N.ptr(units["y"]), N.ptr(units["size"]), N.ptr(units["dx"]),
                             N.ptr(units["dy"]), N.ptr(units["s"]), N.ptr(units["o"]), n, W, H, int(iters),
                             float(stop_delta), float(initial_value), N.ptr(ping), N.ptr(pong), N.ptr(out),
                             N.ptr(it), N.ptr(ws), ws.numel(), N.stream_ptr(stream)))
    return out, it


def decode_device_f64(code: "DeviceCode", iters: int, stop_delta: float, initial_value: float, out=None,
                      stream=None):
    """Exact fp64 decode of a device quadtree code (records expanded to units on the device)."""
    code.join(stream)
    n = code.n_records()
    u = records_to_units_device(code.records, n, code.padded_w, code.padded_h, stream)
    return decode_units_f64(u, code.padded_w, code.padded_h, iters, stop_delta, initial_value, out, stream)


def decode_units_device(units: dict, W: int, H: int, iters: int, stop_delta: float, initial_value: float,
                        stream=None):
    torch = _torch()
    L = N.lib()
    dev = units["x"].device
    ping = torch.empty((H, W), dtype=torch.float32, device=dev)
    pong = torch.empty((H, W), dtype=torch.float32, device=dev)
    out = torch.empty((H, W), dtype=torch.uint8, device=dev)
    it = torch.zeros(1, dtype=torch.int32, device=dev)
    ws = _WS.get("decu", 64, dev)
    N.check(L.mns_decode_units(N.ptr(units["x"]), N.ptr(units["y"]), N.ptr(units["size"]), N.ptr(units["dx"]),
                               N.ptr(units["dy"]), N.ptr(units["s"]), N.ptr(units["o"]), units["x"].numel(), W, H,
                               int(iters), float(stop_delta), float(initial_value), N.ptr(ping), N.ptr(pong),
                               N.ptr(out), N.ptr(it), N.ptr(ws), ws.numel(), N.stream_ptr(stream)))
    return out, it


def full_search_device(img, B: int, step: int = 1, n_iso: int = 1, ranges: Optional[tuple] = None, stream=None):
    """Exhaustive search over a B-padded uint8 CUDA image; returns per-range (dom, iso, o, code) tensors."""
    torch = _torch()
    L = N.lib()
    h, w = img.shape
    nr = (w // B) * (h // B)
    r0, r1 = ranges if ranges is not None else (0, nr)
    dev = img.device
    out = {"dom": torch.empty(r1 - r0, dtype=torch.int32, device=dev),
           "iso": torch.empty(r1 - r0, dtype=torch.int8, device=dev),
           "o": torch.empty(r1 - r0, dtype=torch.uint8, device=dev),
           "code": torch.empty(r1 - r0, dtype=torch.uint8, device=dev)}
    wsb = N.out_i64(L, L.mns_search_workspace_bytes, w, h, B, step, n_iso)
    ws = _WS.get("search", wsb, dev)
    N.check(L.mns_full_search(N.ptr(img), w, h, B, step, n_iso, r0, r1, N.ptr(out["dom"]), N.ptr(out["iso"]),
                              N.ptr(out["o"]), N.ptr(out["code"]), N.ptr(ws), ws.numel(), N.stream_ptr(stream)))
    return out


def local_search_device(img, radius: int = 4, stream=None, n_iso: int = 1, tensor_cores=None):
    """Local search (encoder.py:312-347; radius 4 / n_iso 1 = the reference) over an 8-padded uint8 CUDA
    image; per-range (dx, dy, iso, o, code) tensors.  tensor_cores: the windowed tcgen05 GEMM
    (mns_local_search_tc) or the CUDA-core kernel (mns_local_search), bit-identical; None picks the
    faster one measured on B200 (tcgen05 for wide windows with isometries, +-16 and up x 8)."""
    if tensor_cores is None:
        tensor_cores = n_iso == 8 and radius >= 16
    torch = _torch()
    L = N.lib()
    h, w = img.shape
    nr = (w // 8) * (h // 8)
    dev = img.device
    out = {k: torch.empty(nr, dtype=dt, device=dev) for k, dt in
           (("dx", torch.int32), ("dy", torch.int32), ("iso", torch.int8), ("o", torch.uint8),
            ("code", torch.uint8))}
    if tensor_cores:  # the windowed tcgen05 GEMM (mns_local_search_tc)
        wsb = N.out_i64(L, L.mns_local_search_workspace_bytes, w, h, int(radius), int(n_iso))
        ws = _WS.get("local", wsb, dev)
        N.check(L.mns_local_search_tc(N.ptr(img), w, h, int(radius), int(n_iso), N.ptr(out["dx"]), N.ptr(out["dy"]),
                                      N.ptr(out["iso"]), N.ptr(out["o"]), N.ptr(out["code"]), N.ptr(ws), ws.numel(),
                                      N.stream_ptr(stream)))
    else:  # the CUDA-core kernel
        N.check(L.mns_local_search(N.ptr(img), w, h, int(radius), int(n_iso), N.ptr(out["dx"]), N.ptr(out["dy"]),
                                   N.ptr(out["iso"]), N.ptr(out["o"]), N.ptr(out["code"]), N.stream_ptr(stream)))
    return out


def write_stream_device(records, n: int, orig_w: int, orig_h: int, padded_w: int, padded_h: int, mns: bool,
                        technique2: bool, stream=None):
    """GPU .mns packer; returns (uint8 byte tensor with >= ceil(bits/8) valid bytes, bits tensor)."""
    torch = _torch()
    L = N.lib()
    dev = records.device
    cap = 4 * ((104 + 33 * n + 31) // 32)
    out = torch.zeros(cap, dtype=torch.uint8, device=dev)
    bits = torch.zeros(1, dtype=torch.int64, device=dev)
    wsb = N.out_i64(L, L.mns_stream_workspace_bytes, n)
    ws = _WS.get("stream", wsb, dev)
    N.check(L.mns_write_stream(N.ptr(records), n, orig_w, orig_h, padded_w, padded_h, 1 if mns else 0,
                               1 if technique2 else 0, N.ptr(out), cap, N.ptr(bits), N.ptr(ws), ws.numel(),
                               N.stream_ptr(stream)))
    return out, bits


def read_stream_device(data, mns: bool, technique2: bool, padded_w: int, padded_h: int, stream=None):
    """GPU .mns body parser (csrc/mns_stream_read.cu).  ``data`` is the whole container as a uint8
    CUDA tensor (header validated by the caller).  Returns (DeviceCode, status int64[2]): status[0]
    the first format-error key (-1 none), status[1] the bit position after the final leaf."""
    torch = _torch()
    L = N.lib()
    dev = data.device
    n_roots = (padded_w // 16) * (padded_h // 16)
    code = DeviceCode(torch.empty(64 * n_roots, dtype=torch.int64, device=dev),
                      torch.zeros(n_roots + 1, dtype=torch.int32, device=dev),
                      torch.zeros(1, dtype=torch.int64, device=dev), padded_w, padded_h, 1, 0, padded_h // 16,
                      "mns" if mns else "no_search", bool(technique2))
    status = torch.empty(2, dtype=torch.int64, device=dev)
    wsb = N.out_i64(L, L.mns_read_stream_workspace_bytes, data.numel())
    ws = _WS.get("read", wsb, dev)
    N.check(L.mns_read_stream(N.ptr(data), data.numel(), 1 if mns else 0, 1 if technique2 else 0, padded_w, padded_h,
                              N.ptr(code.records), code.records.numel(), N.ptr(code.root_offsets), N.ptr(code.count),
                              N.ptr(status), N.ptr(ws), ws.numel(), N.stream_ptr(stream)))
    return code, status


# ------------------------------------------------------------------ host layer (reference API)

def _device():
    torch = _torch()
    N.lib()
    return torch.device("cuda", torch.cuda.current_device())


def _to_device_u8(px: np.ndarray):
    torch = _torch()
    px = np.ascontiguousarray(px)
    if not px.flags.writeable:  # torch.from_numpy wants a writable buffer
        px = px.copy()
    return torch.from_numpy(px).to(_device(), non_blocking=False)


def encode_quadtree(image, config: EncoderConfig, *, root_level: int = 1, n_iso: int = 1) -> QuadtreeCode:
    """encoder.py:215-246.  root_level=2 is the '8->4' extension (every root split once); n_iso=8 the
    isometry extension (records carry each phase-1 leaf's isometry; see encode_device)."""
    if config.mode not in ("no_search", "mns"):
        raise ValueError(f"encode_quadtree handles no_search/mns, not {config.mode!r}")
    px = _pixels(image)
    padded = _padded_np(px, ROOT_SIZE)
    code = encode_device(_to_device_u8(padded), config, root_level=root_level, n_iso=n_iso)
    n = code.n_records()
    rec = code.records[:n].cpu().numpy().view(np.uint64)
    offs = code.root_offsets.cpu().numpy()
    return QuadtreeCode.from_records(rec, padded.shape[1], padded.shape[0], px.shape[1], px.shape[0], config.mode,
                                     config.technique2, root_offsets=offs)


def _check_rect(w: int, h: int, rect: BlockRect) -> None:
    """image.py:140-143."""
    if rect.size < 1 or rect.x < 0 or rect.y < 0 or rect.x + rect.size > w or rect.y + rect.size > h:
        raise ValueError(f"{rect} out of bounds for {w}x{h} raster")


def _try_node(image, rect: BlockRect, level: int, config: EncoderConfig, phase: int):
    torch = _torch()
    L = N.lib()
    px = _pixels(image)
    h, w = px.shape
    img = _to_device_u8(px)
    rec = torch.zeros(1, dtype=torch.int64, device=img.device)
    rms = torch.zeros(1, dtype=torch.float64, device=img.device)
    cfg = enc_cfg(config)
    N.check(L.mns_try_node(N.ptr(img), w, h, w, rect.x, rect.y, level, phase, ctypes.byref(cfg), N.ptr(rec),
                           N.ptr(rms), N.stream_ptr(None)))
    packed = rec.cpu().numpy().view(np.uint64)
    r = float(rms.cpu().item())
    if not packed[0]:
        return None, r
    (leaf,) = unpack_leaves(packed)
    return replace(leaf, rect=rect), r  # packed records hold even corners; keep the caller's rect


def try_phase1(image, rect: BlockRect, level: int, config: EncoderConfig):
    """encoder.py:145-166: fit the co-centred domain onto rect; (LeafRecord | None, rms).

    One ``try_node_kernel`` launch: exact integer moments decide, and the rms is replayed in the
    reference's fp64 order, so both match the reference bit for bit (tests/golden/nodes.npz).
    """
    if LEVEL_SIZES[level] != rect.size:
        raise ValueError(f"level {level} expects block size {LEVEL_SIZES[level]}, got {rect.size}")
    px = _pixels(image)
    co_domain_rect(rect, px.shape[1], px.shape[0])  # raises like the reference when no domain fits
    _check_rect(px.shape[1], px.shape[0], rect)
    return _try_node(px, rect, level, config, 1)


def try_phase2(image, rect: BlockRect, level: int, config: EncoderConfig):
    """encoder.py:169-212: quadrant-mean coding with 1-bit contrast picks; (LeafRecord, worst
    quadrant rms) or (None, inf)."""
    if level not in CONTRAST_SETS:
        raise ValueError("phase 2 exists only at levels 1..3")
    px = _pixels(image)
    _check_rect(px.shape[1], px.shape[0], rect)
    if rect.size != LEVEL_SIZES[level]:  # the reference codes any even square; the kernel codes level sizes
        raise ValueError(f"level {level} expects block size {LEVEL_SIZES[level]}, got {rect.size}")
    return _try_node(px, rect, level, config, 2)


def _records_grouped(code) -> tuple[np.ndarray, np.ndarray]:
    """Records grouped by root (stable, so DFS order is kept) and root offsets."""
    rec = np.ascontiguousarray(code.records, dtype=np.uint64)
    W, H = code.padded_w, code.padded_h
    rw = W // 16
    if getattr(code, "root_offsets", None) is not None and len(code.root_offsets) == rw * (H // 16) + 1:
        return rec, np.ascontiguousarray(code.root_offsets, dtype=np.int32)
    x = ((rec >> np.uint64(0)) & np.uint64(0x7FFF)).astype(np.int64) * 2
    y = ((rec >> np.uint64(15)) & np.uint64(0x7FFF)).astype(np.int64) * 2
    root = (y // 16) * rw + x // 16
    order = np.argsort(root, kind="stable")
    counts = np.bincount(root, minlength=rw * (H // 16))
    offs = np.zeros(len(counts) + 1, dtype=np.int32)
    np.cumsum(counts, out=offs[1:])
    return rec[order], offs


def _baseline_units(code) -> dict:
    leaves = code.leaves
    cols = {k: np.empty(len(leaves), dtype=np.int32) for k in ("x", "y", "size", "dx", "dy")}
    s = np.empty(len(leaves), dtype=np.float64)
    o = np.empty(len(leaves), dtype=np.float64)
    for i, lf in enumerate(leaves):
        p = lf.payload
        cols["x"][i], cols["y"][i], cols["size"][i] = lf.rect.x, lf.rect.y, lf.rect.size
        cols["dx"][i], cols["dy"][i] = p.domain.x, p.domain.y
        s[i] = dequantize_contrast(p.s_code)
        o[i] = float(p.o_byte)
    cols["s"], cols["o"] = s, o
    return cols


def _quadtree_units(code) -> dict:
    """Painted units of a no_search/mns code (decoder.py:48-59): 1 per phase-1 leaf, 4 per phase-2 leaf."""
    from .types import unpack_fields

    f = unpack_fields(code.records)
    W, H = code.padded_w, code.padded_h
    xs, ys, ss, ss_, os_ = [], [], [], [], []
    size = np.array([LEVEL_SIZES[int(v)] for v in range(1, 5)])[f["level"] - 1]
    p1 = ~f["phase2"]
    iso = ((np.asarray(code.records, dtype=np.uint64) >> np.uint64(44)) & np.uint64(7)).astype(np.int64)
    xs.append(f["x"][p1]); ys.append(f["y"][p1]); ss.append(size[p1] | (iso[p1] << 8))  # side | isometry << 8
    ss_.append(-0.875 + 0.25 * f["s_code"][p1]); os_.append(f["o"][p1].astype(np.float64))
    p2 = f["phase2"]
    if p2.any():
        lv, h = f["level"][p2], size[p2] // 2
        d0, d1, d2, ob, sb = f["d0"][p2], f["d1"][p2], f["d2"][p2], f["o"][p2], f["s_bits"][p2]
        targets = [ob + d0, ob + d1, ob + d2, ob - (d0 + d1 + d2)]
        sets = np.array([[0, 0], list(CONTRAST_SETS[1]), list(CONTRAST_SETS[2]), list(CONTRAST_SETS[3])])
        for q in range(4):
            xs.append(f["x"][p2] + (q & 1) * h); ys.append(f["y"][p2] + (q >> 1) * h); ss.append(h)
            ss_.append(sets[lv, (sb >> q) & 1]); os_.append(targets[q].astype(np.float64))
    x = np.concatenate(xs).astype(np.int32)
    y = np.concatenate(ys).astype(np.int32)
    sz = np.concatenate(ss).astype(np.int32)
    side = sz & 255
    dx = np.clip(x - side // 2, 0, W - 2 * side).astype(np.int32)
    dy = np.clip(y - side // 2, 0, H - 2 * side).astype(np.int32)
    return {"x": x, "y": y, "size": sz, "dx": dx, "dy": dy, "s": np.concatenate(ss_), "o": np.concatenate(os_)}


def _units_to_device(u: dict, float_dtype):
    torch = _torch()
    dev = _device()
    out = {k: torch.from_numpy(np.ascontiguousarray(u[k])).to(dev) for k in ("x", "y", "size", "dx", "dy")}
    out["s"] = torch.from_numpy(np.ascontiguousarray(u["s"], dtype=float_dtype)).to(dev)
    out["o"] = torch.from_numpy(np.ascontiguousarray(u["o"], dtype=float_dtype)).to(dev)
    return out


def decode(code, config: Optional[DecodeConfig] = None) -> GrayImage:
    """decoder.py:66-77.  stop_delta > 0 (the default DecodeConfig): bit-exact with the reference
    (fp64 sweeps, the early stop decided exactly; mns_decode_f64).  stop_delta == 0: the fp32
    raster / lattice decoders (parity bar <= 1 LSB and 0.01 dB)."""
    torch = _torch()
    cfg = config if config is not None else DecodeConfig()
    W, H = code.padded_w, code.padded_h
    if cfg.max_iters < 1:
        raise ValueError("max_iters must be >= 1")
    from .bitstream import has_isometries

    iso = code.mode in ("no_search", "mns") and isinstance(code, QuadtreeCode) and code.has_records and \
        has_isometries(code.records)
    if cfg.stop_delta > 0.0 or iso:  # exact fp64 path (the isometry extension always decodes here)
        if code.mode in ("no_search", "mns"):
            u = _quadtree_units(code if isinstance(code, QuadtreeCode) else _wrap_reference(code))
        else:
            u = _baseline_units(code)
        out, _ = decode_units_f64(_units_to_device(u, np.float64), W, H, cfg.max_iters, cfg.stop_delta,
                                  cfg.initial_value)
        return GrayImage(out.cpu().numpy()[: code.orig_h, : code.orig_w])
    if code.mode in ("no_search", "mns") and (not hasattr(code, "has_records") or code.has_records):
        rec, offs = _records_grouped(code if isinstance(code, QuadtreeCode) else _wrap_reference(code))
        dev = _device()
        lv = (rec >> np.uint64(30)) & np.uint64(3)  # level - 1 (include/mns_record.h)
        p2 = (rec >> np.uint64(32)) & np.uint64(1)
        unit2 = bool(((lv == 3) | ((lv == 2) & (p2 == 1))).any())  # 2x2 leaves or level-3 phase-2 quadrants
        dcode = DeviceCode(torch.from_numpy(rec.view(np.int64)).to(dev), torch.from_numpy(offs).to(dev),
                           torch.tensor([len(rec)], dtype=torch.int64, device=dev), W, H,
                           min_leaf=2 if unit2 else 4)
        out, _, _ = decode_device(dcode, cfg.max_iters, cfg.stop_delta, cfg.initial_value)
        if dcode.decode_error is not None and int(dcode.decode_error.item()):
            out, _, _ = decode_device(dcode, cfg.max_iters, cfg.stop_delta, cfg.initial_value, lattice=False)
    else:
        u = _units_to_device(_baseline_units(code), np.float32)
        out, _ = decode_units_device(u, W, H, cfg.max_iters, cfg.stop_delta, cfg.initial_value)
    px = out.cpu().numpy()
    return GrayImage(px[: code.orig_h, : code.orig_w])


def _wrap_reference(code) -> QuadtreeCode:
    """Accept a reference mnscodec.QuadtreeCode (same fields) by repacking its leaves."""
    return QuadtreeCode(code.leaves, code.padded_w, code.padded_h, code.orig_w, code.orig_h, code.mode,
                        code.technique2)


def decode_step(code, current) -> np.ndarray:
    """decoder.py:37-63: one fp64 Jacobi sweep, bit-identical to the reference (numpy order emulated)."""
    torch = _torch()
    cur = np.asarray(current, dtype=np.float64)
    if cur.shape != (code.padded_h, code.padded_w):
        raise ValueError(f"raster shape {cur.shape} does not match padded {code.padded_h}x{code.padded_w}")
    L = N.lib()
    if code.mode in ("no_search", "mns"):
        q = code if isinstance(code, QuadtreeCode) else _wrap_reference(code)
        u = _quadtree_units(q)
    else:
        u = _baseline_units(code)
    du = _units_to_device(u, np.float64)
    dev = _device()
    dcur = torch.from_numpy(np.ascontiguousarray(cur)).to(dev)
    dout = torch.empty_like(dcur)
    N.check(L.mns_decode_step_f64(N.ptr(du["x"]), N.ptr(du["y"]), N.ptr(du["size"]), N.ptr(du["dx"]),
                                  N.ptr(du["dy"]), N.ptr(du["s"]), N.ptr(du["o"]), du["x"].numel(), code.padded_w,
                                  code.padded_h, N.ptr(dcur), N.ptr(dout), N.stream_ptr()))
    return dout.cpu().numpy()


def encode_full_search(image, range_size: int, config: EncoderConfig, *, n_iso: int = 1):
    """encoder.py:249-309.  n_iso=8 adds the isometry extension (parity vs the restated oracle)."""
    if range_size not in SIZE_LEVELS:
        raise ValueError(f"range size must be one of {sorted(SIZE_LEVELS)}")
    px = _pixels(image)
    dsize = 2 * range_size
    if px.shape[1] < dsize or px.shape[0] < dsize:
        raise ValueError(f"image too small for any {dsize}x{dsize} domain")
    padded = _padded_np(px, range_size)
    h, w = padded.shape
    res = full_search_device(_to_device_u8(padded), range_size, config.full_search_step, n_iso)
    step = config.full_search_step
    ndx = (w - dsize) // step + 1
    dom = res["dom"].cpu().numpy().astype(np.int64)
    B = range_size
    rpr = w // B
    ids = np.arange(len(dom))
    cols = {"range_size": B, "rx": (ids % rpr) * B, "ry": (ids // rpr) * B, "dom_x": (dom % ndx) * step,
            "dom_y": (dom // ndx) * step, "o": res["o"].cpu().numpy(), "code": res["code"].cpu().numpy(),
            "iso": res["iso"].cpu().numpy()}
    half = B // 2
    samples = list(zip(((cols["dom_x"] + B) - (cols["rx"] + half)).tolist(),
                       ((cols["dom_y"] + B) - (cols["ry"] + half)).tolist()))
    code = QuadtreeCode(None, w, h, px.shape[1], px.shape[0], "full_search", False, columns=cols)
    return code, samples


def encode_local_search(image, config: EncoderConfig, *, radius: int = 4, n_iso: int = 1) -> QuadtreeCode:
    """encoder.py:312-347 (radius 4, n_iso 1 = the reference's 81 candidates; other radii and 8
    isometries are the extension)."""
    px = _pixels(image)
    if px.shape[1] < 16 or px.shape[0] < 16:
        raise ValueError("local search needs at least a 16x16 image")
    padded = _padded_np(px, 8)
    h, w = padded.shape
    res = local_search_device(_to_device_u8(padded), radius, n_iso=n_iso)
    ids = np.arange(res["dx"].numel())
    rpr = w // 8
    cols = {"range_size": 8, "rx": (ids % rpr) * 8, "ry": (ids // rpr) * 8, "dom_x": res["dx"].cpu().numpy(),
            "dom_y": res["dy"].cpu().numpy(), "o": res["o"].cpu().numpy(), "code": res["code"].cpu().numpy(),
            "iso": res["iso"].cpu().numpy()}
    return QuadtreeCode(None, w, h, px.shape[1], px.shape[0], "local_search", False, columns=cols)
