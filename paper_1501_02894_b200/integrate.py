"""Drop-in installation into the reference package ``mnscodec``.

``install()`` rebinds the hot-path names of an importable ``mnscodec`` to this package's B200
path, converting at the boundary so callers get the reference's OWN types back:

  encode_quadtree      encoder.py:215-246  -> mnscodec.encoder.QuadtreeCode of mnscodec LeafRecords
  try_phase1/2         encoder.py:145-212  -> (mnscodec LeafRecord | None, rms)
  encode_full_search   encoder.py:249-309  -> (QuadtreeCode of BaselinePayload leaves, offsets)
  encode_local_search  encoder.py:312-347  -> QuadtreeCode
  decode               decoder.py:66-77    -> mnscodec.image.GrayImage
  decode_step          decoder.py:37-63    -> float64 ndarray (bit-identical)

The reference binds these names at import time in several modules (``mnscodec/__init__.py:19-33``,
``cli.py:18-19``, ``bench.py:13-14``), so every binding site is patched.  The returned leaves
are ``mnscodec.encoder`` dataclasses holding Python ints, so ``bitstream._validate_leaf`` and
``decode_step``'s ``isinstance`` dispatch (``bitstream.py:107-121``, ``decoder.py:50-62``) and
``BitWriter.write`` (``bitstream.py:45-54``) see exactly what the reference encoder produces.
Configs are duck-typed: the reference's ``EncoderConfig`` / ``DecodeConfig`` pass straight through.

Usage::

    import mnscodec
    from paper_1501_02894_b200 import integrate
    handle = integrate.install(mnscodec)   # mnscodec.encode_quadtree now runs on the GPU
    ...
    handle.uninstall()
"""

from __future__ import annotations

import importlib

from . import codec as _codec
from .types import LEVEL_SIZES, unpack_fields

ENCODER_NAMES = ("encode_quadtree", "encode_full_search", "encode_local_search", "try_phase1", "try_phase2")
DECODER_NAMES = ("decode", "decode_step")
SITES = ("mnscodec", "mnscodec.encoder", "mnscodec.decoder", "mnscodec.cli", "mnscodec.bench")


def to_reference_leaves(code, ref) -> tuple:
    """This package's QuadtreeCode -> tuple of ``ref.encoder.LeafRecord`` (Python ints)."""
    E, I = ref.encoder, ref.image
    if code.mode in ("no_search", "mns") and code.has_records:
        f = unpack_fields(code.records)
        cols = [f[k].tolist() for k in ("x", "y", "level", "phase2", "o", "s_code", "d0", "d1", "d2", "s_bits")]
        rect, leaf, p1, p2 = I.BlockRect, E.LeafRecord, E.Phase1Payload, E.Phase2Payload
        out = []
        for x, y, lv, ph2, o, sc, d0, d1, d2, sb in zip(*cols):
            pay = (p2(o, (d0, d1, d2), (sb & 1, (sb >> 1) & 1, (sb >> 2) & 1, (sb >> 3) & 1)) if ph2
                   else p1(o, sc))
            out.append(leaf(rect(x, y, LEVEL_SIZES[lv]), lv, pay))
        return tuple(out)
    out = []
    for lf in code.leaves:  # baseline (search) codes: per-range columns
        p = lf.payload
        pay = E.BaselinePayload(I.BlockRect(p.domain.x, p.domain.y, p.domain.size), int(p.o_byte), int(p.s_code))
        out.append(E.LeafRecord(I.BlockRect(lf.rect.x, lf.rect.y, lf.rect.size), int(lf.level), pay))
    return tuple(out)


def to_reference_code(code, ref):
    """This package's QuadtreeCode -> ``ref.encoder.QuadtreeCode`` (encoder.py:120-142)."""
    return ref.encoder.QuadtreeCode(to_reference_leaves(code, ref), code.padded_w, code.padded_h, code.orig_w,
                                    code.orig_h, code.mode, code.technique2)


def _leaf_to_reference(leaf, rect, ref):
    E = ref.encoder
    p = leaf.payload
    if hasattr(p, "deltas"):
        pay = E.Phase2Payload(int(p.o_byte), tuple(int(v) for v in p.deltas), tuple(int(v) for v in p.s_bits))
    else:
        pay = E.Phase1Payload(int(p.o_byte), int(p.s_code))
    return E.LeafRecord(rect, int(leaf.level), pay)


class Installed:
    """Handle returned by install(): the rebound functions and the originals they replaced."""

    def __init__(self, ref, functions: dict, saved: list):
        self.ref = ref
        self.functions = functions
        self._saved = saved

    def uninstall(self) -> None:
        for mod, name, fn in reversed(self._saved):
            setattr(mod, name, fn)
        self._saved = []


def make_functions(ref) -> dict:
    """The reference-signature wrappers over this package for reference package ``ref``."""
    I = ref.image

    def encode_quadtree(image, config):
        return to_reference_code(_codec.encode_quadtree(image, config), ref)

    def encode_full_search(image, range_size, config):
        code, samples = _codec.encode_full_search(image, range_size, config)
        return to_reference_code(code, ref), samples

    def encode_local_search(image, config):
        return to_reference_code(_codec.encode_local_search(image, config), ref)

    def _try(fn):
        def call(image, rect, level, config):
            leaf, rms = fn(image, rect, level, config)
            return (None if leaf is None else _leaf_to_reference(leaf, rect, ref)), rms

        call.__name__ = fn.__name__
        call.__doc__ = fn.__doc__
        return call

    def decode(code, config=None):
        return I.GrayImage(_codec.decode(code, config).pixels)

    def decode_step(code, current):
        return _codec.decode_step(code, current)

    for f, src in ((encode_quadtree, _codec.encode_quadtree), (encode_full_search, _codec.encode_full_search),
                   (encode_local_search, _codec.encode_local_search), (decode, _codec.decode),
                   (decode_step, _codec.decode_step)):
        f.__doc__ = src.__doc__
    return {"encode_quadtree": encode_quadtree, "encode_full_search": encode_full_search,
            "encode_local_search": encode_local_search, "try_phase1": _try(_codec.try_phase1),
            "try_phase2": _try(_codec.try_phase2), "decode": decode, "decode_step": decode_step}


def install(ref=None) -> Installed:
    """Rebind every binding site of the reference's hot-path names to the B200 path."""
    if ref is None:
        ref = importlib.import_module("mnscodec")
    for sub in SITES[1:]:
        importlib.import_module(sub)
    functions = make_functions(ref)
    saved = []
    for site in SITES:
        mod = importlib.import_module(site)
        for name, fn in functions.items():
            if hasattr(mod, name):
                saved.append((mod, name, getattr(mod, name)))
                setattr(mod, name, fn)
    return Installed(ref, functions, saved)


def codes_equal(a, b) -> bool:
    """Field-wise equality of two codes of either package (encoder.py:120-142 semantics)."""
    meta = lambda c: (c.padded_w, c.padded_h, c.orig_w, c.orig_h, c.mode, c.technique2)  # noqa: E731
    if meta(a) != meta(b) or len(a.leaves) != len(b.leaves):
        return False
    from .types import _as_plain

    return all(_as_plain(x) == _as_plain(y) for x, y in zip(a.leaves, b.leaves))


__all__ = ["install", "Installed", "to_reference_code", "to_reference_leaves", "make_functions", "codes_equal"]
