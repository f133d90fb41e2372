""".mns container (reference: bitstream.py) over packed records.

write_stream packs on the GPU (csrc/mns_stream.cu: widths -> look-back scan ->
MSB-first word gather) and read_stream parses on the GPU (csrc/mns_stream_read.cu:
speculative token walks + scans); stream_bit_count / level_id_bit_count are
vectorised numpy accounting over the packed records; read_stream_host is the
sequential host parser used as the checker (the reference's format, byte for byte).  Error messages follow the reference
(bitstream.py:107-200, :208-279).
"""

from __future__ import annotations

import struct

import numpy as np

from .types import (
    DELTA_MAGNITUDE_BITS,
    ROOT_SIZE,
    BlockRect,
    LeafRecord,
    Phase1Payload,
    Phase2Payload,
    QuadtreeCode,
    delta_limit,
    unpack_fields,
)

MAGIC = b"MNS1"
HEADER_BYTES = 13
FLAG_MNS = 0x01
FLAG_TECHNIQUE2 = 0x02


class StreamFormatError(ValueError):
    """Byte stream that does not parse as a valid .mns container."""


def payload_bit_width(level: int, phase2: bool) -> int:
    """bitstream.py:87-92."""
    if phase2:
        return 8 + 3 * (1 + DELTA_MAGNITUDE_BITS[level]) + 4
    return 11


def leaf_bit_width(level: int, phase2: bool, mode: str, id_elided: bool = False) -> int:
    """bitstream.py:95-100."""
    bits = 0 if id_elided else 2
    if mode == "mns" and level <= 3:
        bits += 1
    return bits + payload_bit_width(level, phase2)


def _widths(code: QuadtreeCode) -> np.ndarray:
    f = unpack_fields(code.records)
    lv, p2 = f["level"], f["phase2"]
    w = np.where(p2, 8 + 3 * (1 + np.where(lv == 1, 4, 5)) + 4, 11)
    if code.mode == "mns":
        w = w + (lv <= 3)
    elided = (lv == 4) & (((f["x"] // 2) | (f["y"] // 2)) & 1).astype(bool) & code.technique2
    return w + np.where(elided, 0, 2)


def stream_bit_count(code: QuadtreeCode) -> int:
    """bitstream.py:282-300: exact serialized size in bits, header included."""
    return HEADER_BYTES * 8 + int(_widths(code).sum())


def level_id_bit_count(code: QuadtreeCode, technique2: bool) -> int:
    """bitstream.py:303-314."""
    lv = unpack_fields(code.records)["level"]
    count4 = int((lv == 4).sum())
    others = len(lv) - count4
    if not technique2:
        return 2 * (others + count4)
    if count4 % 4:
        raise ValueError("level-4 leaves must form complete quartets")
    return 2 * (others + count4 // 4)


def _validate_leaf(leaf, mode: str) -> None:
    """bitstream.py:107-127 (messages kept)."""
    p = leaf.payload
    if hasattr(p, "domain"):
        raise ValueError("search-baseline records have no stream encoding")
    if leaf.level not in (1, 2, 3, 4):
        raise ValueError(f"bad leaf level {leaf.level}")
    if not 0 <= p.o_byte <= 255:
        raise ValueError(f"luminance byte {p.o_byte} out of range")
    if not hasattr(p, "deltas"):
        if not 0 <= p.s_code <= 7:
            raise ValueError(f"contrast code {p.s_code} out of range")
        return
    if mode != "mns":
        raise ValueError("phase-2 record in a no_search code")
    if leaf.level == 4:
        raise ValueError("phase-2 record at level 4")
    limit = delta_limit(leaf.level)
    if len(p.deltas) != 3 or any(abs(d) > limit for d in p.deltas):
        raise ValueError(f"delta exceeds level-{leaf.level} width: {p.deltas}")
    if len(p.s_bits) != 4 or any(b not in (0, 1) for b in p.s_bits):
        raise ValueError(f"bad contrast selection bits {p.s_bits}")


def _validate_tiling(leaves, w: int, h: int, mode: str) -> None:
    """DFS tiling check of user-built leaf lists (codes from the GPU encoder tile by construction)."""
    pos = 0

    def emit(rect, level):
        nonlocal pos
        if pos >= len(leaves):
            raise ValueError("leaf list under-fills the padded raster")
        nxt = leaves[pos].level
        if nxt == level:
            leaf = leaves[pos]
            if leaf.rect.x != rect.x or leaf.rect.y != rect.y or leaf.rect.size != rect.size:
                raise ValueError(f"leaf {pos} ({leaf.level}, {leaf.rect}) does not tile at level {level}, {rect}")
            _validate_leaf(leaf, mode)
            pos += 1
            return
        if nxt < level or level >= 4:
            raise ValueError(f"leaf level {nxt} cannot tile a level-{level} node")
        for q in rect.quadrants():
            emit(q, level + 1)

    for y in range(0, h, ROOT_SIZE):
        for x in range(0, w, ROOT_SIZE):
            emit(BlockRect(x, y, ROOT_SIZE), 1)
    if pos != len(leaves):
        raise ValueError("excess leaf records beyond the padded raster")


def _check_header(code) -> None:
    if code.mode not in ("no_search", "mns"):
        raise ValueError(f"only no_search/mns codes serialize, not {code.mode!r}")
    if code.padded_w % ROOT_SIZE or code.padded_h % ROOT_SIZE:
        raise ValueError("padded dimensions must be multiples of 16")
    if not (0 < code.orig_w <= code.padded_w and 0 < code.orig_h <= code.padded_h):
        raise ValueError("original dimensions must fit inside the padded raster")
    if code.padded_w > 0xFFFF or code.padded_h > 0xFFFF:
        raise ValueError("dimensions exceed the 16-bit header fields")


def has_isometries(records) -> bool:
    """True for records of the n_iso = 8 extension: a phase-1 leaf with a non-identity isometry
    (bits 44..46, mns_record.h MNS_REC_ISO_SHIFT; phase-2 records use those bits for deltas)."""
    r = np.asarray(records, dtype=np.uint64)
    p1 = ((r >> np.uint64(32)) & np.uint64(1)) == 0
    return bool((((r >> np.uint64(44)) & np.uint64(7)) != 0)[p1].any())


def write_stream(code) -> bytes:
    """bitstream.py:203-205 on the GPU packer."""
    from . import codec

    if not isinstance(code, QuadtreeCode):
        code = QuadtreeCode(code.leaves, code.padded_w, code.padded_h, code.orig_w, code.orig_h, code.mode,
                            code.technique2)
    _check_header(code)
    if code._records is None:  # user-built leaf list: validate like the reference before packing
        _validate_tiling(code.leaves, code.padded_w, code.padded_h, code.mode)
    elif code.mode in ("no_search", "mns") and has_isometries(code.records):
        raise ValueError("isometry codes (the n_iso=8 extension) have no .mns representation (SPEC.md:16)")
    import torch

    rec = torch.from_numpy(np.ascontiguousarray(code.records).view(np.int64)).to(codec._device())
    out, bits = codec.write_stream_device(rec, len(code.records), code.orig_w, code.orig_h, code.padded_w,
                                          code.padded_h, code.mode == "mns", code.technique2)
    nbits = int(bits.item())
    return bytes(out[: (nbits + 7) // 8].cpu().numpy())


class _Bits:
    def __init__(self, data: bytes, offset: int) -> None:
        self.data = data
        self.pos = offset * 8
        self.end = len(data) * 8

    def read(self, n: int) -> int:
        if self.pos + n > self.end:
            raise StreamFormatError("truncated stream")
        v = 0
        for _ in range(n):
            v = (v << 1) | ((self.data[self.pos >> 3] >> (7 - (self.pos & 7))) & 1)
            self.pos += 1
        return v


def _header(data: bytes):
    """bitstream.py:210-222: magic, flags and dimensions, with the reference's errors."""
    if len(data) < HEADER_BYTES:
        raise StreamFormatError("truncated header")
    if data[:4] != MAGIC:
        raise StreamFormatError(f"bad magic {bytes(data[:4])!r}")
    flags = data[4]
    if flags & ~(FLAG_MNS | FLAG_TECHNIQUE2):
        raise StreamFormatError(f"unknown flag bits 0x{flags:02x}")
    mode = "mns" if flags & FLAG_MNS else "no_search"
    t2 = bool(flags & FLAG_TECHNIQUE2)
    ow, oh, pw, ph = struct.unpack(">4H", data[5:HEADER_BYTES])
    if min(ow, oh) < 1:
        raise StreamFormatError("zero image dimension in header")
    if pw % ROOT_SIZE or ph % ROOT_SIZE or pw < ow or ph < oh:
        raise StreamFormatError("padded dimensions inconsistent with original dimensions")
    return mode, t2, ow, oh, pw, ph


def read_stream(data: bytes) -> QuadtreeCode:
    """bitstream.py:208-279: exact inverse of write_stream, parsed on the GPU
    (csrc/mns_stream_read.cu: speculative token walks + scans); the first format error raises
    the same StreamFormatError as the reference's sequential parser."""
    from . import codec

    data = bytes(data)
    mode, t2, ow, oh, pw, ph = _header(data)
    import torch

    buf = torch.frombuffer(bytearray(data), dtype=torch.uint8).to(codec._device())
    code, status = codec.read_stream_device(buf, mode == "mns", t2, pw, ph)
    key, end = (int(v) for v in status.cpu().tolist())
    if key != -1:
        err, a, b = (key >> 8) & 0xFF, (key >> 4) & 0xF, key & 0xF
        if err == 1:
            raise StreamFormatError(f"level-{a} leaf cannot appear inside a level-{b} node")
        if err == 2:
            raise StreamFormatError(f"level-4 quartet interrupted by level-{a} id")
        if err == 3:
            raise StreamFormatError("non-canonical negative-zero delta")
        raise StreamFormatError("truncated stream")
    if end < 0:
        raise StreamFormatError("truncated stream")
    left = len(data) * 8 - end
    if left >= 8:
        raise StreamFormatError(f"{left} trailing bits after the final leaf")
    if left and data[-1] & ((1 << left) - 1):
        raise StreamFormatError("nonzero padding bits")
    n = code.n_records()
    rec = code.records[:n].cpu().numpy().view(np.uint64)
    return QuadtreeCode.from_records(rec, pw, ph, ow, oh, mode, t2, root_offsets=code.root_offsets.cpu().numpy())


def read_stream_host(data: bytes) -> QuadtreeCode:
    """bitstream.py:208-279 as a sequential host parser (the checker for read_stream's errors)."""
    mode, t2, ow, oh, pw, ph = _header(data)
    rd = _Bits(data, HEADER_BYTES)
    leaves = []

    def leaf(rect, level):
        p2 = bool(rd.read(1)) if (mode == "mns" and level <= 3) else False
        o = rd.read(8)
        if p2:
            nb = DELTA_MAGNITUDE_BITS[level]
            ds = []
            for _ in range(3):
                sign, mag = rd.read(1), rd.read(nb)
                if sign and mag == 0:
                    raise StreamFormatError("non-canonical negative-zero delta")
                ds.append(-mag if sign else mag)
            payload = Phase2Payload(o, (ds[0], ds[1], ds[2]), (rd.read(1), rd.read(1), rd.read(1), rd.read(1)))
        else:
            payload = Phase1Payload(o, rd.read(3))
        leaves.append(LeafRecord(rect, level, payload))

    def walk(rect, level, pending):
        lid = rd.read(2) if pending is None else pending
        depth = lid + 1
        if depth < level:
            raise StreamFormatError(f"level-{depth} leaf cannot appear inside a level-{level} node")
        if depth == level:
            leaf(rect, level)
            return
        quads = rect.quadrants()
        if level == 3:
            leaf(quads[0], 4)
            for q in quads[1:]:
                if not t2:
                    sib = rd.read(2)
                    if sib != 3:
                        raise StreamFormatError(f"level-4 quartet interrupted by level-{sib + 1} id")
                leaf(q, 4)
            return
        walk(quads[0], level + 1, lid)
        for q in quads[1:]:
            walk(q, level + 1, None)

    for y in range(0, ph, ROOT_SIZE):
        for x in range(0, pw, ROOT_SIZE):
            walk(BlockRect(x, y, ROOT_SIZE), 1, None)
    left = rd.end - rd.pos
    if left >= 8:
        raise StreamFormatError(f"{left} trailing bits after the final leaf")
    if left and rd.read(left) != 0:
        raise StreamFormatError("nonzero padding bits")
    return QuadtreeCode(tuple(leaves), pw, ph, ow, oh, mode, t2)
