"""Generate tests/golden/*.npz by running the REFERENCE implementation itself.

Runs only in the build container, where the read-only reference lives at
/root/reference (pure Python: PYTHONPATH=/root/reference/pkg/src).  Fixture
images come from the reference's own test generators (imported, not copied:
/root/reference/pkg/tests/util.py) and from this repo's pinned synthetic
generator; outputs are the reference's encode / decode / search results,
packed into this repo's record layout.  The GPU box never needs the reference.

    python oracle/gen_golden.py            # rewrites tests/golden/*.npz
"""

from __future__ import annotations

import json
import math
import os
import sys
from fractions import Fraction

import numpy as np

REF = "/root/reference/pkg"
sys.path.insert(0, os.path.join(REF, "src"))
sys.path.insert(0, os.path.join(REF, "tests"))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import mnscodec.encoder as enc  # noqa: E402
from mnscodec.bench import histogram_csv, offset_histogram, rd_sweep  # noqa: E402
from mnscodec.bitstream import stream_bit_count, write_stream  # noqa: E402
from mnscodec.decoder import DecodeConfig, decode, decode_step  # noqa: E402
from mnscodec.encoder import EncoderConfig, encode_full_search, encode_local_search, encode_quadtree  # noqa: E402
from mnscodec.image import BlockRect, GrayImage, pad_to_multiple  # noqa: E402
from util import gradient_image, natural_image, noise_image, scene_image  # noqa: E402

from paper_1501_02894_b200.synth import synth_image  # noqa: E402
from paper_1501_02894_b200.types import pack_leaf  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def quadrant_image(values, size=16):
    h = size // 2
    arr = np.zeros((size, size), dtype=np.uint8)
    arr[:h, :h], arr[:h, h:], arr[h:, :h], arr[h:, h:] = values
    return arr


def fixture_images():
    imgs = {
        "natural_256": natural_image(256, 256, seed=7).pixels,
        "natural_128": natural_image(128, 128, seed=3).pixels,
        "scene_crop_64": np.ascontiguousarray(scene_image(256, 256, seed=7).pixels[96:160, 64:128]),
        "noise_64": noise_image(64, 64, seed=11).pixels,
        "gradient_64": gradient_image(64, 64).pixels,
        "constant_64": np.full((64, 64), 42, dtype=np.uint8),
        "odd_50x34": np.random.default_rng(17).integers(0, 256, (34, 50), dtype=np.uint8),
        "tiny_16": noise_image(16, 16, seed=5).pixels,
        "strip_16x48": np.random.default_rng(23).integers(0, 256, (16, 48), dtype=np.uint8),
        "checker_64": (np.indices((64, 64)).sum(axis=0) % 2 * 255).astype(np.uint8),
        "synth_c1_256": synth_image(256, 1),
    }
    return imgs


def _tie_patches(seed=7, batches=16, per_batch=1_000_000):
    """6x6 patches around a level-3 node (node = patch[1:5, 1:5]) in which at least one phase-2
    quadrant has an EXACT real-arithmetic tie between its two contrast candidates
    (7*Dn == 40*Nn, Dn != 0: SSE(0.5) == SSE(0.9)), so the reference's pick is decided by
    fp64 rounding in numpy's evaluation order.  Kept only if phase 2 beats phase 1 on the node;
    returns (patches, phase-2 rms, phase-1 rms) from the reference itself."""
    rng = np.random.default_rng(seed)
    quads = ((1, 1), (1, 3), (3, 1), (3, 3))
    keep, rms = [], []
    for _ in range(batches):
        n = per_batch
        k, step = int(rng.integers(2, 4)), int(rng.integers(1, 3))
        P = rng.integers(0, k, (n, 6, 6)) * step
        off = rng.integers(-3, 4, (n, 4)) * int(rng.integers(1, 4))
        P[:, :3, :3] += off[:, 0, None, None]
        P[:, :3, 3:] += off[:, 1, None, None]
        P[:, 3:, :3] += off[:, 2, None, None]
        P[:, 3:, 3:] += off[:, 3, None, None]
        P += 100
        hit = np.zeros(n, bool)
        for qy, qx in quads:
            r = P[:, qy:qy + 2, qx:qx + 2].reshape(n, 4)
            d = P[:, qy - 1:qy + 3, qx - 1:qx + 3]
            q = (d[:, 0::2, 0::2] + d[:, 0::2, 1::2] + d[:, 1::2, 0::2] + d[:, 1::2, 1::2]).reshape(n, 4)
            sr, sq, srq, sqq = r.sum(1), q.sum(1), (r * q).sum(1), (q * q).sum(1)
            dn = 4 * sqq - sq * sq
            hit |= (7 * dn == 40 * (4 * srq - sr * sq)) & (dn != 0)
        for i in np.nonzero(hit)[0]:
            canvas = np.full((16, 16), 100, np.uint8)
            canvas[3:9, 3:9] = P[i]
            img = GrayImage(canvas)
            _, rms1 = enc.try_phase1(img, BlockRect(4, 4, 4), 3, EncoderConfig(e3=1e9))
            _, rms2 = enc.try_phase2(img, BlockRect(4, 4, 4), 3, EncoderConfig(e3=1e9))
            if rms2 < rms1:
                keep.append(P[i].astype(np.uint8))
                rms.append((rms2, rms1))
    return np.array(keep), np.array(rms)


def tie_rich_images():
    """80x80 images with up to 64 planted tie nodes each (level-3 nodes at offsets 4 and 12 inside every
    root); e1 = e2 = 0.01 forces levels 1-2 to split, e3 = E accepts the planted nodes through
    phase 2 (rms2 <= E < rms1).  Returns {name: (pixels, config dict)}."""
    patches, rms = _tie_patches()
    out = {}
    used = np.zeros(len(patches), bool)
    for img_i, E in enumerate((0.9, 1.5, 2.2, 3.0, 4.5)):
        ok = np.nonzero((rms[:, 0] <= E) & (E < rms[:, 1]) & ~used)[0][:64]
        if len(ok) < 16:
            continue
        used[ok] = True
        canvas = np.full((80, 80), 100, np.uint8)  # 5x5 roots; plants in the first 4x4
        for j, pi in enumerate(ok):
            root, sub = divmod(j, 4)
            x0 = (root % 4) * 16 + 4 + 8 * (sub % 2)
            y0 = (root // 4) * 16 + 4 + 8 * (sub // 2)
            canvas[y0 - 1:y0 + 5, x0 - 1:x0 + 5] = patches[pi]
        out[f"ties_{img_i}"] = (canvas, dict(e1=0.01, e2=0.01, e3=E, mean_tol=16.0, mode="mns"))
    return out


def records_of(code) -> np.ndarray:
    return np.array([pack_leaf(lf) for lf in code.leaves], dtype=np.uint64)


def redrive_level2(image: GrayImage, config: EncoderConfig):
    """The '8->4' mapping: every 16x16 root forced to split once,
    the reference's own try_phase1/try_phase2 driving levels 2..4."""
    padded = pad_to_multiple(image, 16)
    min_dim = min(padded.width, padded.height)
    leaves = []

    def visit(rect, level):
        record = None
        if 2 * rect.size <= min_dim:
            record, _ = enc.try_phase1(padded, rect, level, config)
            if record is None and config.mode == "mns":
                record, _ = enc.try_phase2(padded, rect, level, config)
        if record is not None:
            leaves.append(record)
            return
        for q in rect.quadrants():
            visit(q, level + 1)

    for y in range(0, padded.height, 16):
        for x in range(0, padded.width, 16):
            for q in BlockRect(x, y, 16).quadrants():
                visit(q, 2)
    return enc.QuadtreeCode(tuple(leaves), padded.width, padded.height, image.width, image.height, config.mode,
                            config.technique2)


def count_exact_phase2_ties(image: GrayImage, config: EncoderConfig):
    """Count phase-2 quadrant evaluations whose two candidate errors are equal in exact
    arithmetic for the DECIMAL contrast values (0.5 vs 0.9 etc.; their binary doubles differ from
    the decimals by ~1e-17, far below fp64 rounding of the error sums), and how many of those the
    reference resolved to bit 1.  These picks are decided by fp64 rounding alone."""
    calls = []
    real = enc.rms_error

    def spy(r, d, s, o):
        v = real(r, d, s, o)
        calls.append((np.asarray(r, float).ravel(), np.asarray(d, float).ravel(), s, o, v))
        return v

    enc.rms_error = spy
    try:
        encode_quadtree(image, config)
    finally:
        enc.rms_error = real
    ties = ones = 0
    # phase-2 evaluations come in (lo, hi) pairs with non-dyadic s from CONTRAST_SETS
    sets = {s for pair in enc.CONTRAST_SETS.values() for s in pair}
    i = 0
    while i + 1 < len(calls):
        a, b = calls[i], calls[i + 1]
        if a[2] in sets and b[2] in sets and a[3] == b[3] and a[0].size == b[0].size and a[2] < b[2] \
                and np.array_equal(a[0], b[0]):
            def exact(c):
                r, d, s, o = c[0], c[1], Fraction(repr(c[2])), Fraction(c[3])  # decimal set value
                dm = sum(Fraction(v) for v in d) / len(d)
                return sum((Fraction(rv) - (s * (Fraction(dv) - dm) + o)) ** 2 for rv, dv in zip(r, d))
            if exact(a) == exact(b) and len(set(a[1].tolist())) > 1:
                ties += 1
                ones += int(not (a[4] <= b[4]))
            i += 2
        else:
            i += 1
    return ties, ones


ENC_CONFIGS = [
    dict(e1=8.0, e2=8.0, e3=8.0, mean_tol=16.0, mode="mns"),
    dict(e1=8.0, e2=8.0, e3=8.0, mean_tol=16.0, mode="no_search"),
    dict(e1=5.0, e2=5.0, e3=5.0, mean_tol=16.0, mode="mns"),
    dict(e1=4.0, e2=5.0, e3=6.0, mean_tol=16.0, mode="mns"),
    dict(e1=2.2, e2=3.0, e3=6.3, mean_tol=8.0, mode="mns"),
    dict(e1=8.0, e2=8.0, e3=math.inf, mean_tol=16.0, mode="mns"),
    dict(e1=0.5, e2=0.5, e3=0.5, mean_tol=16.0, mode="mns"),
]


def gen_encode(store, manifest):
    tie_imgs = tie_rich_images()
    imgs = {**fixture_images(), **{k: v[0] for k, v in tie_imgs.items()}}
    k = 0
    tie_total = tie_ones = 0
    for name, px in imgs.items():
        image = GrayImage(px)
        cfgs = ENC_CONFIGS if not name.startswith("ties") else [tie_imgs[name][1]]
        if name == "checker_64":
            cfgs = cfgs + [dict(e1=1.0, e2=1.0, e3=1.0, mean_tol=16.0, mode="mns")]
        for cfg in cfgs:
            for root_level in (1, 2):
                if root_level == 2 and name not in ("synth_c1_256", "natural_128", "noise_64", "odd_50x34"):
                    continue
                config = EncoderConfig(**cfg)
                code = encode_quadtree(image, config) if root_level == 1 else redrive_level2(image, config)
                key = f"enc{k}"
                store[f"{key}/img"] = px
                store[f"{key}/records"] = records_of(code)
                dec8 = decode(code, DecodeConfig(max_iters=8, stop_delta=0.0)).pixels
                dec_def = decode(code, DecodeConfig()).pixels
                store[f"{key}/decode8"] = dec8
                store[f"{key}/decode_default"] = dec_def
                store[f"{key}/stream"] = np.frombuffer(write_stream(code), dtype=np.uint8)
                store[f"{key}/stream_bits"] = np.array(stream_bit_count(code), dtype=np.int64)
                ties = ones = 0
                if name.startswith("ties") and root_level == 1:
                    ties, ones = count_exact_phase2_ties(image, config)
                    tie_total += ties
                    tie_ones += ones
                manifest.append(dict(key=key, image=name, cfg={k2: (None if v == math.inf else v) for k2, v in
                                                               cfg.items()},
                                     root_level=root_level, padded_w=code.padded_w, padded_h=code.padded_h,
                                     leaves=len(code.leaves), phase2=code.phase2_count(), exact_ties=ties,
                                     ties_bit1=ones))
                k += 1
    print(f"encode cases: {k}; exact phase-2 ties {tie_total} (reference picked bit 1 in {tie_ones})")


def gen_decode_step(store, manifest):
    rng = np.random.default_rng(0)
    for k, (name, px, cfg) in enumerate([
        ("natural_128", natural_image(128, 128, seed=3).pixels, EncoderConfig(e1=5, e2=5, e3=5, mode="mns")),
        ("odd_50x34", np.random.default_rng(17).integers(0, 256, (34, 50), dtype=np.uint8), EncoderConfig()),
    ]):
        code = encode_quadtree(GrayImage(px), cfg)
        raster = rng.uniform(0, 255, (code.padded_h, code.padded_w))
        out = decode_step(code, raster)
        store[f"step{k}/img"] = px
        store[f"step{k}/records"] = records_of(code)
        store[f"step{k}/raster_in"] = raster
        store[f"step{k}/raster_out"] = out
        manifest.append(dict(key=f"step{k}", image=name, padded_w=code.padded_w, padded_h=code.padded_h))


def gen_search(store, manifest):
    rng = np.random.default_rng(9)
    arr = rng.integers(0, 256, (48, 48), dtype=np.uint8)
    pattern = np.where(np.indices((8, 8)).sum(axis=0) % 2 == 0, 136, 120)
    arr[8:24, 24:40] = np.kron(pattern, np.ones((2, 2), dtype=int)).astype(np.uint8)
    arr[0:8, 0:8] = (0.875 * (pattern - 128) + 128).astype(np.uint8)
    imgs = {
        "noise_64": noise_image(64, 64, seed=11).pixels,
        "natural_128": natural_image(128, 128, seed=3).pixels,
        "constant_64": np.full((64, 64), 42, dtype=np.uint8),
        "constructed_48": arr,
        "odd_52x40": np.random.default_rng(3).integers(0, 256, (40, 52), dtype=np.uint8),
        "synth_c4_crop_96": np.ascontiguousarray(synth_image(512, 4)[200:296, 64:160]),
    }
    k = 0
    for name, px in imgs.items():
        for B in (2, 4, 8, 16):
            for step in (1, 2):
                if min(px.shape) < 2 * B or (B == 2 and px.shape[0] > 64):
                    continue
                code, samples = encode_full_search(GrayImage(px), B, EncoderConfig(mode="full_search",
                                                                                   full_search_step=step))
                key = f"full{k}"
                store[f"{key}/img"] = px
                store[f"{key}/dom"] = np.array([[lf.payload.domain.x, lf.payload.domain.y] for lf in code.leaves],
                                               dtype=np.int32)
                store[f"{key}/o"] = np.array([lf.payload.o_byte for lf in code.leaves], dtype=np.uint8)
                store[f"{key}/code"] = np.array([lf.payload.s_code for lf in code.leaves], dtype=np.uint8)
                store[f"{key}/samples"] = np.array(samples, dtype=np.int32)
                store[f"{key}/decode"] = decode(code, DecodeConfig(max_iters=6, stop_delta=0.0)).pixels
                manifest.append(dict(key=key, image=name, B=B, step=step, padded_w=code.padded_w,
                                     padded_h=code.padded_h))
                k += 1
    j = 0
    for name, px in {**imgs, "noise_32": noise_image(32, 32, seed=8).pixels}.items():
        if min(px.shape) < 16:
            continue
        code = encode_local_search(GrayImage(px), EncoderConfig(mode="local_search"))
        key = f"local{j}"
        store[f"{key}/img"] = px
        store[f"{key}/dom"] = np.array([[lf.payload.domain.x, lf.payload.domain.y] for lf in code.leaves],
                                       dtype=np.int32)
        store[f"{key}/o"] = np.array([lf.payload.o_byte for lf in code.leaves], dtype=np.uint8)
        store[f"{key}/code"] = np.array([lf.payload.s_code for lf in code.leaves], dtype=np.uint8)
        manifest.append(dict(key=key, image=name, padded_w=code.padded_w, padded_h=code.padded_h))
        j += 1
    print(f"search cases: full {k}, local {j}")


def gen_nodes(store, manifest):
    """Single-node try_phase1 / try_phase2 known answers (reference test_encoder.py:45-107 cases
    plus random nodes)."""
    cases = []
    for vals in [(100, 104, 96, 100), (178, 100, 100, 100), (116, 100, 100, 84), (3, 3, 3, 0), (42, 42, 42, 42),
                 (10, 20, 30, 40), (250, 255, 255, 248)]:
        cases.append((quadrant_image(vals), 0, 0, 16, 1, EncoderConfig()))
    rng = np.random.default_rng(5)
    nat = natural_image(128, 128, seed=3).pixels
    for _ in range(60):
        level = int(rng.integers(1, 4))
        size = 32 >> level
        x = int(rng.integers(0, 128 // size)) * size
        y = int(rng.integers(0, 128 // size)) * size
        e = float(rng.choice([1.0, 2.5, 4.0, 8.0]))
        cases.append((nat, x, y, size, level, EncoderConfig(e1=e, e2=e, e3=e)))
    # rects at arbitrary (odd, unaligned) positions, level 4, and domains clamped at the borders
    rng2 = np.random.default_rng(55)
    small = scene_image(40, 24, seed=9).pixels
    for _ in range(40):
        level = int(rng2.integers(1, 5))
        size = 32 >> level
        px = nat if rng2.random() < 0.7 else small
        x = int(rng2.integers(0, px.shape[1] - size + 1))
        y = int(rng2.integers(0, px.shape[0] - size + 1))
        e = float(rng2.choice([1.0, 2.5, 4.0, 8.0]))
        cases.append((px, x, y, size, level, EncoderConfig(e1=e, e2=e, e3=e, mean_tol=float(rng2.choice([4.0, 8.0, 30.0])))))
    for k, (px, x, y, size, level, cfg) in enumerate(cases):
        image = GrayImage(px)
        if 2 * size <= min(px.shape):
            r1, rms1 = enc.try_phase1(image, BlockRect(x, y, size), level, cfg)
        else:  # no room for the domain: the quadtree driver never calls phase 1 here
            r1, rms1 = None, math.nan
        r2, rms2 = enc.try_phase2(image, BlockRect(x, y, size), level, cfg) if level <= 3 else (None, math.inf)
        key = f"node{k}"
        store[f"{key}/img"] = px
        store[f"{key}/rec"] = np.array([pack_leaf(r1) if r1 else 0, pack_leaf(r2) if r2 else 0], dtype=np.uint64)
        store[f"{key}/rms"] = np.array([rms1, rms2], dtype=np.float64)
        manifest.append(dict(key=key, x=x, y=y, size=size, level=level, e=cfg.e1, mean_tol=cfg.mean_tol,
                             ok1=r1 is not None, ok2=r2 is not None))
    print(f"node cases: {len(cases)}")


def gen_rd(store, manifest):
    """Reference rd_sweep rows (bench.py:39-79) and offset-histogram CSVs (bench.py:119-142)."""
    imgs = {
        "constant_64": np.full((64, 64), 42, dtype=np.uint8),
        "natural_128": natural_image(128, 128, seed=3).pixels,
        "synth_c2_crop_96x80": np.ascontiguousarray(synth_image(512, 2)[100:180, 300:396]),
        "scene_72x56": np.ascontiguousarray(scene_image(256, 256, seed=7).pixels[40:96, 20:92]),
    }
    grid = [4.0, 8.0, (6.0, 8.0, 10.0)]
    k = 0
    for name, px in imgs.items():
        for dec in (None, DecodeConfig(max_iters=6, stop_delta=0.0)):
            pts = rd_sweep(GrayImage(px), ["no_search", "mns"], grid, (True, False), decode_config=dec)
            key = f"rd{k}"
            store[f"{key}/img"] = px
            store[f"{key}/bits"] = np.array([p.bits for p in pts], dtype=np.int64)
            store[f"{key}/psnr"] = np.array([p.psnr for p in pts], dtype=np.float64)
            store[f"{key}/leaves"] = np.array([p.leaf_counts for p in pts], dtype=np.int64)
            store[f"{key}/phase2"] = np.array([p.phase2_count for p in pts], dtype=np.int64)
            manifest.append(dict(key=key, image=name, grid=[list(g) if isinstance(g, tuple) else g for g in grid],
                                 decode=None if dec is None else [dec.max_iters, dec.stop_delta, dec.initial_value],
                                 rows=[[p.mode, list(p.thresholds), p.technique2] for p in pts]))
            k += 1
    j = 0
    for name in ("natural_128", "scene_72x56"):
        px = imgs[name]
        for B in (4, 8):
            _, samples = encode_full_search(GrayImage(px), B, EncoderConfig(mode="full_search"))
            key = f"hist{j}"
            store[f"{key}/img"] = px
            store[f"{key}/csv"] = np.array(histogram_csv(offset_histogram(samples)))
            manifest.append(dict(key=key, image=name, B=B))
            j += 1
    print(f"rd cases: {k} sweeps, {j} histograms")


def stress_images():
    """Adversarial structures for the exact decisions: saturated blocks, hard edges, checkerboards at
    several node sizes, gradients (contrast-bin edges), flat patches (D = 0), small-amplitude noise."""
    rng = np.random.default_rng(99)
    n = 192
    y, x = np.mgrid[0:n, 0:n]
    imgs = {
        "checker2": np.where(((x // 2) + (y // 2)) % 2 == 0, 255, 0),
        "checker4x8": np.where(((x // 4) + (y // 8)) % 2 == 0, 250, 3),
        "ramp": np.clip(x * 1.33 + y * 0.01, 0, 255),
        "sincos": np.clip(128 + 127 * np.sin(x / 3.0) * np.cos(y / 5.0), 0, 255),
        "edge": np.where(x < n // 2, 0, 255) + 0 * y,
        "binary_noise": rng.integers(0, 2, (n, n)) * 255,
        "low_noise": rng.integers(120, 137, (n, n)),
        "gauss_noise": np.clip(rng.normal(128, 40, (n, n)), 0, 255),
        "flat": np.full((n, n), 77),
        "tiles": np.clip((x % 16) * 16 + (y % 16), 0, 255),
    }
    return {k: np.ascontiguousarray(np.rint(v).astype(np.uint8)) for k, v in imgs.items()}


STRESS_CONFIGS = [dict(e1=8.0, e2=8.0, e3=8.0, mean_tol=16.0, mode="mns"),
                  dict(e1=2.0, e2=3.0, e3=math.inf, mean_tol=16.0, mode="mns"),
                  dict(e1=0.5, e2=1.0, e3=1.5, mean_tol=4.0, mode="mns"),
                  dict(e1=20.0, e2=12.0, e3=6.0, mean_tol=40.0, mode="mns"),
                  dict(e1=5.0, e2=5.0, e3=5.0, mean_tol=16.0, mode="no_search")]


def gen_stress(store, manifest):
    """Reference encode_quadtree records (and an 8-sweep decode) of adversarial images."""
    k = 0
    for name, px in stress_images().items():
        store[f"img/{name}"] = px
        for ci, cfg in enumerate(STRESS_CONFIGS):
            code = encode_quadtree(GrayImage(px), EncoderConfig(**cfg))
            key = f"s{k}"
            store[f"{key}/records"] = records_of(code)
            store[f"{key}/decode8"] = decode(code, DecodeConfig(max_iters=8, stop_delta=0.0)).pixels
            manifest.append(dict(key=key, image=name, cfg={k2: (None if v == math.inf else v) for k2, v in
                                                          cfg.items()}))
            k += 1
    print(f"stress cases: {k}")


def main(argv=None):
    """Regenerate every golden set, or only the named ones (e.g. ``gen_golden.py rd``)."""
    os.makedirs(OUT, exist_ok=True)
    table = (("encode", gen_encode), ("decode_step", gen_decode_step), ("search", gen_search),
             ("nodes", gen_nodes), ("rd", gen_rd), ("stress", gen_stress))
    want = set(argv or []) or {n for n, _ in table}
    for name, fn in table:
        if name not in want:
            continue
        store, manifest = {}, []
        fn(store, manifest)
        store["manifest"] = np.array(json.dumps(manifest))
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **store)
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main(sys.argv[1:])
