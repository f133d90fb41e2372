"""Host-side mirror of the reference's data model (same names, fields, defaults,
validation messages and equality), so code written against ``mnscodec`` reads
the same against this package.

Reference: /root/reference/pkg/src/mnscodec
  BlockRect            image.py:17-33
  GrayImage            image.py:36-66
  EncoderConfig        encoder.py:52-76
  Phase1Payload        encoder.py:79-84
  Phase2Payload        encoder.py:87-98
  BaselinePayload      encoder.py:101-107
  LeafRecord           encoder.py:113-117
  QuadtreeCode         encoder.py:120-142
  DecodeConfig         decoder.py:21-29

``QuadtreeCode`` additionally carries the packed device records
(``include/mns_record.h``) so that codes of 10^7+ leaves never have to be
materialised as Python objects; ``leaves`` is built lazily on first access.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional, Union

import numpy as np

MODES = ("no_search", "mns", "local_search", "full_search")
ROOT_SIZE = 16
LEVEL_SIZES = {1: 16, 2: 8, 3: 4, 4: 2}
SIZE_LEVELS = {size: level for level, size in LEVEL_SIZES.items()}
CONTRAST_SETS = {1: (0.2, 0.5), 2: (0.4, 0.65), 3: (0.5, 0.9)}
DELTA_MAGNITUDE_BITS = {1: 4, 2: 5, 3: 5}
CONTRAST_CODES = 8
CONTRAST_VALUES = tuple(-0.875 + 0.25 * k for k in range(CONTRAST_CODES))


def delta_limit(level: int) -> int:
    """Largest phase-2 quadrant-mean offset encodable at ``level`` (encoder.py:42-44)."""
    return (1 << DELTA_MAGNITUDE_BITS[level]) - 1


def round_to_int(value: float) -> int:
    """floor(v + 0.5): halves toward +infinity (encoder.py:47-49)."""
    return int(math.floor(value + 0.5))


def dequantize_contrast(code: int) -> float:
    """Centre of contrast bin ``code`` (transform.py:56-60)."""
    if not 0 <= code < CONTRAST_CODES:
        raise ValueError(f"contrast code {code} outside [0, {CONTRAST_CODES - 1}]")
    return -0.875 + 0.25 * code


@dataclass(frozen=True)
class BlockRect:
    """Axis-aligned square; (x, y) is the top-left corner (image.py:17-33)."""

    x: int
    y: int
    size: int

    def quadrants(self) -> tuple["BlockRect", "BlockRect", "BlockRect", "BlockRect"]:
        h = self.size // 2
        return (BlockRect(self.x, self.y, h), BlockRect(self.x + h, self.y, h),
                BlockRect(self.x, self.y + h, h), BlockRect(self.x + h, self.y + h, h))


class GrayImage:
    """8-bit single-channel raster, immutable after construction (image.py:36-66)."""

    def __init__(self, pixels) -> None:
        arr = np.array(pixels)
        if arr.ndim != 2:
            raise ValueError(f"expected a 2-D pixel array, got shape {arr.shape}")
        if arr.size == 0:
            raise ValueError("image must contain at least one pixel")
        if arr.dtype != np.uint8:
            if not np.issubdtype(arr.dtype, np.integer):
                raise ValueError("pixel values must be integers in [0, 255]")
            if arr.min() < 0 or arr.max() > 255:
                raise ValueError("pixel values must lie in [0, 255]")
            arr = arr.astype(np.uint8)
        arr.setflags(write=False)
        self.pixels = arr

    @property
    def width(self) -> int:
        return self.pixels.shape[1]

    @property
    def height(self) -> int:
        return self.pixels.shape[0]

    def __eq__(self, other) -> bool:
        return hasattr(other, "pixels") and np.array_equal(self.pixels, np.asarray(other.pixels))

    def __repr__(self) -> str:
        return f"GrayImage({self.width}x{self.height})"


@dataclass(frozen=True)
class EncoderConfig:
    """Encoder knobs (encoder.py:52-76); e1..e3 are per-level RMS tolerances."""

    e1: float = 8.0
    e2: float = 8.0
    e3: float = 8.0
    mean_tol: float = 16.0
    mode: str = "mns"
    technique2: bool = True
    full_search_step: int = 1

    def __post_init__(self) -> None:
        if self.mode not in MODES:
            raise ValueError(f"unknown mode {self.mode!r}")
        if min(self.e1, self.e2, self.e3) <= 0:
            raise ValueError("error thresholds must be positive")
        if self.mean_tol < 0:
            raise ValueError("mean_tol must be non-negative")
        if self.full_search_step < 1:
            raise ValueError("full_search_step must be >= 1")

    def threshold(self, level: int) -> float:
        return (self.e1, self.e2, self.e3)[level - 1]


@dataclass(frozen=True)
class DecodeConfig:
    """decoder.py:21-29."""

    max_iters: int = 10
    stop_delta: float = 0.5
    initial_value: float = 128.0

    def __post_init__(self) -> None:
        if self.max_iters < 1:
            raise ValueError("max_iters must be >= 1")


@dataclass(frozen=True)
class Phase1Payload:
    o_byte: int
    s_code: int


@dataclass(frozen=True)
class Phase2Payload:
    o_byte: int
    deltas: tuple[int, int, int]
    s_bits: tuple[int, int, int, int]


@dataclass(frozen=True)
class BaselinePayload:
    domain: BlockRect
    o_byte: int
    s_code: int


Payload = Union[Phase1Payload, Phase2Payload, BaselinePayload]


@dataclass(frozen=True)
class LeafRecord:
    rect: BlockRect
    level: int
    payload: Payload


# --------------------------------------------------------------- packed records

def pack_leaf(leaf) -> int:
    """One no_search/mns LeafRecord -> packed u64 (include/mns_record.h)."""
    r, p = leaf.rect, leaf.payload
    base = (r.x >> 1) | ((r.y >> 1) << 15) | ((leaf.level - 1) << 30) | ((p.o_byte & 0xFF) << 33)
    if hasattr(p, "deltas"):
        d = [v & 63 for v in p.deltas]
        bits = sum((b & 1) << k for k, b in enumerate(p.s_bits))
        return base | (1 << 32) | (d[0] << 41) | (d[1] << 47) | (d[2] << 53) | (bits << 59)
    return base | ((p.s_code & 7) << 41)


def unpack_fields(records: np.ndarray) -> dict:
    """Vectorised field extraction from packed records."""
    r = np.asarray(records, dtype=np.uint64)

    def f(shift, mask):
        return ((r >> np.uint64(shift)) & np.uint64(mask)).astype(np.int64)

    ds = []
    for j in range(3):
        v = f(41 + 6 * j, 63)
        ds.append(np.where(v >= 32, v - 64, v))
    return {"x": f(0, 0x7FFF) * 2, "y": f(15, 0x7FFF) * 2, "level": f(30, 3) + 1, "phase2": f(32, 1).astype(bool),
            "o": f(33, 0xFF), "s_code": f(41, 7), "d0": ds[0], "d1": ds[1], "d2": ds[2], "s_bits": f(59, 15)}


def unpack_leaves(records: np.ndarray) -> tuple:
    fl = unpack_fields(records)
    cols = [fl[k].tolist() for k in ("x", "y", "level", "phase2", "o", "s_code", "d0", "d1", "d2", "s_bits")]
    out = []
    for x, y, lv, p2, o, sc, d0, d1, d2, sb in zip(*cols):
        rect = BlockRect(x, y, LEVEL_SIZES[lv])
        if p2:
            payload = Phase2Payload(o, (d0, d1, d2), (sb & 1, (sb >> 1) & 1, (sb >> 2) & 1, (sb >> 3) & 1))
        else:
            payload = Phase1Payload(o, sc)
        out.append(LeafRecord(rect, lv, payload))
    return tuple(out)


class QuadtreeCode:
    """DFS-ordered leaf records plus header metadata (encoder.py:120-142).

    Constructed either like the reference (a ``leaves`` tuple) or from packed
    records (``QuadtreeCode.from_records``); the other representation is built
    on demand.  Search-baseline codes (``BaselinePayload`` leaves) have no packed
    form and keep their leaves / column arrays.
    """

    def __init__(self, leaves, padded_w: int, padded_h: int, orig_w: int, orig_h: int, mode: str,
                 technique2: bool, *, records: Optional[np.ndarray] = None, root_offsets=None, columns=None):
        self._leaves = tuple(leaves) if leaves is not None else None
        self._records = records
        self.root_offsets = root_offsets
        self.columns = columns  # baseline codes: dict of per-range arrays
        self.padded_w = int(padded_w)
        self.padded_h = int(padded_h)
        self.orig_w = int(orig_w)
        self.orig_h = int(orig_h)
        self.mode = mode
        self.technique2 = bool(technique2)

    @classmethod
    def from_records(cls, records, padded_w, padded_h, orig_w, orig_h, mode, technique2, root_offsets=None):
        return cls(None, padded_w, padded_h, orig_w, orig_h, mode, technique2,
                   records=np.ascontiguousarray(records, dtype=np.uint64), root_offsets=root_offsets)

    @property
    def leaves(self) -> tuple:
        if self._leaves is None:
            if self._records is not None:
                self._leaves = unpack_leaves(self._records)
            else:
                self._leaves = _baseline_leaves(self.columns, self.mode)
        return self._leaves

    @property
    def has_records(self) -> bool:
        return self._records is not None or (self.mode in ("no_search", "mns") and self._leaves is not None)

    @property
    def records(self) -> np.ndarray:
        if self._records is None:
            if self.mode not in ("no_search", "mns"):
                raise ValueError("search-baseline codes have no packed record form")
            self._records = np.fromiter((pack_leaf(lf) for lf in self._leaves), dtype=np.uint64,
                                        count=len(self._leaves))
        return self._records

    def __len__(self) -> int:
        if self._records is not None:
            return len(self._records)
        return len(self.leaves)

    def level_counts(self) -> tuple[int, int, int, int]:
        if self.has_records:
            lv = ((self.records >> np.uint64(30)) & np.uint64(3)).astype(np.int64)
            c = np.bincount(lv, minlength=4)
            return (int(c[0]), int(c[1]), int(c[2]), int(c[3]))
        counts = [0, 0, 0, 0]
        for leaf in self.leaves:
            counts[leaf.level - 1] += 1
        return tuple(counts)

    def phase2_count(self) -> int:
        if self.has_records:
            return int(((self.records >> np.uint64(32)) & np.uint64(1)).sum())
        return sum(1 for leaf in self.leaves if isinstance(leaf.payload, Phase2Payload))

    def _meta(self):
        return (self.padded_w, self.padded_h, self.orig_w, self.orig_h, self.mode, self.technique2)

    def __eq__(self, other) -> bool:
        if not hasattr(other, "leaves") or not hasattr(other, "padded_w"):
            return NotImplemented
        meta_o = (other.padded_w, other.padded_h, other.orig_w, other.orig_h, other.mode, other.technique2)
        if self._meta() != meta_o:
            return False
        if isinstance(other, QuadtreeCode) and self.has_records and other.has_records:
            return np.array_equal(self.records, other.records)
        return tuple(_as_plain(lf) for lf in self.leaves) == tuple(_as_plain(lf) for lf in other.leaves)

    def __repr__(self) -> str:
        return (f"QuadtreeCode({len(self)} leaves, {self.padded_w}x{self.padded_h} padded, "
                f"{self.orig_w}x{self.orig_h} orig, mode={self.mode!r}, technique2={self.technique2})")


def _as_plain(leaf):
    """Structural tuple of any leaf (ours or the reference's) for equality."""
    p = leaf.payload
    rect = (leaf.rect.x, leaf.rect.y, leaf.rect.size)
    if hasattr(p, "deltas"):
        body = ("p2", p.o_byte, tuple(p.deltas), tuple(p.s_bits))
    elif hasattr(p, "domain"):
        body = ("bl", (p.domain.x, p.domain.y, p.domain.size), p.o_byte, p.s_code)
    else:
        body = ("p1", p.o_byte, p.s_code)
    return (rect, leaf.level, body)


def _baseline_leaves(cols, mode) -> tuple:
    if cols is None:
        return ()
    B = int(cols["range_size"])
    level = SIZE_LEVELS[B]
    out = []
    for rx, ry, dx, dy, o, c in zip(cols["rx"].tolist(), cols["ry"].tolist(), cols["dom_x"].tolist(),
                                    cols["dom_y"].tolist(), cols["o"].tolist(), cols["code"].tolist()):
        out.append(LeafRecord(BlockRect(rx, ry, B), level, BaselinePayload(BlockRect(dx, dy, 2 * B), o, c)))
    return tuple(out)
