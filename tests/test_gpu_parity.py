"""GPU parity: libmns_b200 (sm_100a) against the reference's golden vectors and the CPU oracle.

Bars (BASELINE.json north_star): transform codes bit-exact; decoded images within
1 LSB per pixel and 0.01 dB PSNR of the reference (fp32 raster); the fp64
decode_step is bit-exact.
"""
import math

import numpy as np
import pytest

from conftest import cfg_tuple

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import oracle as O  # noqa: E402  (checker only)


@pytest.fixture(scope="module")
def mns():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1501_02894_b200 as m

    return m


def _psnr(a, b):
    d = a.astype(np.float64) - b.astype(np.float64)
    e = float(np.mean(d * d))
    return math.inf if e == 0 else 10 * math.log10(255 * 255 / e)


def _enc(mns, px, case):
    e, mean_tol, is_mns = cfg_tuple(case["cfg"])
    cfg = mns.EncoderConfig(e1=e[0], e2=e[1], e3=e[2], mean_tol=mean_tol, mode="mns" if is_mns else "no_search")
    return mns.encode_quadtree(mns.GrayImage(px), cfg, root_level=case["root_level"])


def test_encode_golden_bit_exact(mns, golden):
    g = golden("encode")
    for case in g.manifest:
        code = _enc(mns, g[f"{case['key']}/img"], case)
        ref = g[f"{case['key']}/records"]
        assert np.array_equal(code.records, ref), (case, len(code.records), len(ref))


def test_tie_fixtures_exercise_rounding_decided_picks(mns, golden):
    g = golden("encode")
    cases = [c for c in g.manifest if c["image"].startswith("ties")]
    assert cases and sum(c["ties_bit1"] for c in cases) > 0
    for case in cases:
        code = _enc(mns, g[f"{case['key']}/img"], case)
        assert np.array_equal(code.records, g[f"{case['key']}/records"]), case


def test_decode_golden_within_1lsb(mns, golden):
    g = golden("encode")
    worst = 0
    for case in g.manifest:
        k = case["key"]
        img = g[f"{k}/img"]
        code = mns.QuadtreeCode.from_records(g[f"{k}/records"], case["padded_w"], case["padded_h"], img.shape[1],
                                             img.shape[0], "mns", True)
        for key, cfg in (("decode8", mns.DecodeConfig(max_iters=8, stop_delta=0.0)),
                         ("decode_default", mns.DecodeConfig())):
            got = mns.decode(code, cfg).pixels
            want = g[f"{k}/{key}"]
            diff = int(np.abs(got.astype(int) - want.astype(int)).max())
            worst = max(worst, diff)
            assert diff <= 1, (case, key, diff)
            if key == "decode_default":  # stop_delta > 0: the exact fp64 decoder, bit-identical
                assert diff == 0, (case, key, diff)
            assert abs(_psnr(img, got) - _psnr(img, want)) <= 0.01 or _psnr(img, want) == math.inf, (case, key)
    print("worst decode diff (LSB):", worst)


def test_decode_step_fp64_bit_exact(mns, golden):
    g = golden("decode_step")
    for case in g.manifest:
        k = case["key"]
        img = g[f"{k}/img"]
        code = mns.QuadtreeCode.from_records(g[f"{k}/records"], case["padded_w"], case["padded_h"], img.shape[1],
                                             img.shape[0], "mns", True)
        out = mns.decode_step(code, g[f"{k}/raster_in"])
        assert np.array_equal(out, g[f"{k}/raster_out"])


def test_decode_leaf_order_invariance(mns, golden):
    g = golden("encode")
    case = next(c for c in g.manifest if c["image"] == "natural_128" and c["cfg"]["e1"] == 5.0)
    k = case["key"]
    rec = g[f"{k}/records"]
    img = g[f"{k}/img"]
    perm = np.random.default_rng(13).permutation(len(rec))
    a = mns.QuadtreeCode.from_records(rec, 128, 128, 128, 128, "mns", True)
    b = mns.QuadtreeCode.from_records(rec[perm], 128, 128, 128, 128, "mns", True)
    raster = np.random.default_rng(0).uniform(0, 255, (128, 128))
    assert np.array_equal(mns.decode_step(a, raster), mns.decode_step(b, raster))
    cfg = mns.DecodeConfig(max_iters=10, stop_delta=0.0)
    assert mns.decode(a, cfg) == mns.decode(b, cfg)
    del img


def test_full_search_golden(mns, golden):
    g = golden("search")
    for case in g.manifest:
        if not case["key"].startswith("full"):
            continue
        k = case["key"]
        code, samples = mns.encode_full_search(mns.GrayImage(g[f"{k}/img"]), case["B"],
                                               mns.EncoderConfig(mode="full_search", full_search_step=case["step"]))
        dom = g[f"{k}/dom"]
        c = code.columns
        assert np.array_equal(c["dom_x"], dom[:, 0]) and np.array_equal(c["dom_y"], dom[:, 1]), case
        assert np.array_equal(c["o"], g[f"{k}/o"]) and np.array_equal(c["code"], g[f"{k}/code"]), case
        assert np.array_equal(np.array(samples, dtype=np.int32).reshape(-1, 2), g[f"{k}/samples"]), case
        got = mns.decode(code, mns.DecodeConfig(max_iters=6, stop_delta=0.0)).pixels
        assert int(np.abs(got.astype(int) - g[f"{k}/decode"].astype(int)).max()) <= 1, case


def test_local_search_golden(mns, golden):
    g = golden("search")
    for case in g.manifest:
        if not case["key"].startswith("local"):
            continue
        k = case["key"]
        code = mns.encode_local_search(mns.GrayImage(g[f"{k}/img"]), mns.EncoderConfig(mode="local_search"))
        dom = g[f"{k}/dom"]
        c = code.columns
        assert np.array_equal(c["dom_x"], dom[:, 0]) and np.array_equal(c["dom_y"], dom[:, 1]), case
        assert np.array_equal(c["o"], g[f"{k}/o"]) and np.array_equal(c["code"], g[f"{k}/code"]), case


def test_full_search_isometries_vs_oracle(mns):
    from paper_1501_02894_b200.synth import synth_image

    px = np.ascontiguousarray(synth_image(512, 4)[100:196, 300:396])
    for B in (4, 8):
        code, _ = mns.encode_full_search(mns.GrayImage(px), B, mns.EncoderConfig(mode="full_search"), n_iso=8)
        ref = O.full_search(px, B, 1, n_iso=8)
        c = code.columns
        assert np.array_equal(c["dom_x"], ref["dom_x"]) and np.array_equal(c["dom_y"], ref["dom_y"])
        assert np.array_equal(c["iso"], ref["iso"]) and np.array_equal(c["code"], ref["code"])


def test_local_search_radius32_vs_oracle(mns):
    from paper_1501_02894_b200.synth import synth_image

    px = np.ascontiguousarray(synth_image(512, 4)[:256, :256])
    code = mns.encode_local_search(mns.GrayImage(px), mns.EncoderConfig(mode="local_search"), radius=32)
    ref = O.local_search(px, 32)
    c = code.columns
    assert np.array_equal(c["dom_x"], ref["dom_x"]) and np.array_equal(c["dom_y"], ref["dom_y"])
    assert np.array_equal(c["code"], ref["code"]) and np.array_equal(c["o"], ref["o"])


@pytest.mark.parametrize("name,root_level,e3", [("c1", 2, math.inf), ("c1", 1, 8.0), ("c2", 1, math.inf),
                                                ("c2", 1, 8.0)])
def test_config_images_vs_oracle(mns, name, root_level, e3):
    from paper_1501_02894_b200.synth import config_image

    px = config_image(name)
    cfg = mns.EncoderConfig(e3=e3)
    code = mns.encode_quadtree(mns.GrayImage(px), cfg, root_level=root_level)
    ref, _ = O.encode_quadtree_records(px, (8.0, 8.0, e3), 16.0, True, root_level)
    assert np.array_equal(code.records, ref)
    iters = 8 if name == "c1" else 10
    got = mns.decode(code, mns.DecodeConfig(max_iters=iters, stop_delta=0.0)).pixels
    want, _, _ = O.decode_records(ref, px.shape[1], px.shape[0], max_iters=iters, stop_delta=0.0)
    assert int(np.abs(got.astype(int) - want.astype(int)).max()) <= 1
    assert abs(_psnr(px, got) - _psnr(px, want)) <= 0.01


def test_batch_encode_matches_single(mns):
    from paper_1501_02894_b200.synth import synth_image

    imgs = np.stack([synth_image(512, s) for s in (1000, 1001, 1002)])
    cfg = mns.EncoderConfig(e3=math.inf)
    dev = torch.from_numpy(imgs).cuda()
    code = mns.encode_device(dev, cfg, root_level=2)
    n = code.n_records()
    rec = code.records[:n].cpu().numpy().view(np.uint64)
    offs = code.root_offsets.cpu().numpy()
    per = 32 * 32
    for i in range(3):
        ref, _ = O.encode_quadtree_records(imgs[i], (8.0, 8.0, math.inf), 16.0, True, 2)
        assert np.array_equal(rec[offs[i * per]: offs[(i + 1) * per]], ref)


def test_strip_encode_matches_whole(mns):
    """Row strips with a 16-px halo and global clamping reproduce the whole-image code."""
    from paper_1501_02894_b200.synth import synth_image

    px = synth_image(1024, 7, noise_sigma=10.0, n_blobs=24)
    cfg = mns.EncoderConfig(e3=math.inf)
    whole = mns.encode_device(torch.from_numpy(px).cuda(), cfg)
    nw = whole.n_records()
    wrec = whole.records[:nw].cpu().numpy()
    parts = []
    H = 1024
    bounds = [0, 13, 30, 64]
    for r0, r1 in zip(bounds[:-1], bounds[1:]):
        y0, y1 = max(0, 16 * r0 - 16), min(H, 16 * r1 + 16)
        sl = torch.from_numpy(np.ascontiguousarray(px[y0:y1])).cuda()
        c = mns.encode_device(sl, cfg, root_rows=(r0, r1), height=H)
        parts.append(c.records[: c.n_records()].cpu().numpy())
    assert np.array_equal(np.concatenate(parts), wrec)


def test_write_stream_matches_reference_layout(mns, golden):
    g = golden("encode")
    from paper_1501_02894_b200 import bitstream

    for case in g.manifest[::5]:
        k = case["key"]
        img = g[f"{k}/img"]
        mode = case["cfg"]["mode"]
        code = mns.QuadtreeCode.from_records(g[f"{k}/records"], case["padded_w"], case["padded_h"], img.shape[1],
                                             img.shape[0], mode, True)
        data = bitstream.write_stream(code)
        assert data == bytes(g[f"{k}/stream"]), case
        assert bitstream.stream_bit_count(code) == int(g[f"{k}/stream_bits"])


def test_full_search_tensor_core_matches_exact_cuda_core_path(mns, monkeypatch):
    """tcgen05 path vs the exact CUDA-core path, incl. the fp16/fp32 worst case (saturated image)."""
    from paper_1501_02894_b200.synth import synth_image

    cases = [(np.ascontiguousarray(synth_image(512, 4)[64:192, 128:256]), 8, 8),
             (np.ascontiguousarray(synth_image(512, 9)[:96, :96]), 4, 8),
             (np.ascontiguousarray(synth_image(512, 7)[200:264, 40:104]), 2, 8),
             (np.ascontiguousarray(synth_image(512, 3)[:200, :136]), 8, 1),
             (np.full((64, 64), 255, np.uint8), 8, 1),
             (np.random.default_rng(2).integers(250, 256, (64, 64), dtype=np.uint8), 8, 8)]
    for step in (1, 3):
        for px, B, n_iso in cases:
            img = torch.from_numpy(px).cuda()
            monkeypatch.setenv("MNS_SEARCH_CUDA_CORES", "0")
            a = {k: v.cpu().numpy() for k, v in mns.full_search_device(img, B, step, n_iso).items()}
            monkeypatch.setenv("MNS_SEARCH_CUDA_CORES", "1")
            b = {k: v.cpu().numpy() for k, v in mns.full_search_device(img, B, step, n_iso).items()}
            for k in a:
                assert np.array_equal(a[k], b[k]), (px.shape, B, n_iso, step, k)
            # a range interval (the per-rank shard of the multi-GPU split) equals the same slice
            r0, r1 = 37, min(150, len(a["dom"]))
            monkeypatch.setenv("MNS_SEARCH_CUDA_CORES", "0")
            c = {k: v.cpu().numpy() for k, v in mns.full_search_device(img, B, step, n_iso, ranges=(r0, r1)).items()}
            for k in a:
                assert np.array_equal(c[k], a[k][r0:r1]), (px.shape, B, n_iso, step, "ranges", k)


def test_full_search_c4_sample_vs_oracle(mns):
    """c4 (512^2, B=8, stride 1, 247,009 domains): GPU vs the oracle on a strided sample of ranges."""
    from paper_1501_02894_b200.synth import config_image

    px = config_image("c4")
    res = mns.full_search_device(torch.from_numpy(px).cuda(), 8, 1, 1)
    dom = res["dom"].cpu().numpy()
    ids = np.arange(0, 4096, 97)
    ref = O.full_search(px, 8, 1, n_iso=1, range_ids=ids)
    assert np.array_equal(dom[ids], ref["dom"])
    assert np.array_equal(res["code"].cpu().numpy()[ids], ref["code"])


def _sweeps_single(N, L, umap, W, H, rr, cur, init, n):
    """n single sweeps (mns_decode_sweep) from cur (None = flat); returns the last fp32 raster."""
    import ctypes

    state = torch.zeros(4, dtype=torch.int32, device="cuda")
    for _ in range(n):
        nxt = torch.full((H, W), float("nan"), device="cuda")
        N.check(L.mns_decode_sweep(N.ptr(umap), W, H, rr[0], rr[1], N.ptr(cur) if cur is not None else ctypes.c_void_p(0),
                                   init, N.ptr(nxt), ctypes.c_void_p(0), N.ptr(state), 0.0, None))
        cur = nxt
    return cur


@pytest.mark.parametrize("W,H,e3,rr", [(512, 512, 8.0, None), (400, 48, 8.0, None), (16, 16, math.inf, None),
                                       (1024, 1040, math.inf, None), (640, 640, 8.0, (5, 17)),
                                       (640, 640, math.inf, (0, 3)), (640, 640, 8.0, (37, 40))])
def test_pair_pass_equals_two_sweeps(mns, W, H, e3, rr):
    """mns_decode_sweep2 (t -> t+2 in one pass, t+1 on chip) is bit-identical to two single sweeps,
    on whole images (partial bands, one root row, 2x2-unit-heavy codes) and strip row ranges
    with a unit map that starts one root row above the strip."""
    import ctypes

    from paper_1501_02894_b200 import _native as N
    from paper_1501_02894_b200.synth import synth_image

    L = N.lib()
    side = max(W, H)
    px = np.ascontiguousarray(synth_image(side, 11, noise_sigma=12.0, n_blobs=8)[:H, :W])
    code = mns.encode_device(torch.from_numpy(px).cuda(), mns.EncoderConfig(e3=e3), map_form=0)
    umap = code.unit_map
    rh = H // 16
    r0, r1 = rr if rr is not None else (0, rh)
    u0 = max(0, r0 - 1)
    sub = umap[u0 * (W // 16) * 32:]
    g = torch.Generator(device="cuda").manual_seed(W + H)
    t0 = torch.rand((H, W), device="cuda", generator=g) * 255.0
    for cur in (None, t0):
        want = _sweeps_single(N, L, umap, W, H, (0, rh), cur, 128.0, 2)
        got = torch.full((H, W), float("nan"), device="cuda")
        N.check(L.mns_decode_sweep2(N.ptr(sub), u0, W, H, r0, r1, N.ptr(cur) if cur is not None else ctypes.c_void_p(0),
                                    128.0, N.ptr(got), ctypes.c_void_p(0), None))
        out = torch.zeros((H, W), dtype=torch.uint8, device="cuda")
        N.check(L.mns_decode_sweep2(N.ptr(sub), u0, W, H, r0, r1, N.ptr(cur) if cur is not None else ctypes.c_void_p(0),
                                    128.0, ctypes.c_void_p(0), N.ptr(out), None))
        torch.cuda.synchronize()
        y0, y1 = 16 * r0, 16 * r1
        assert torch.equal(got[y0:y1], want[y0:y1])
        assert torch.equal(out[y0:y1], torch.floor(want[y0:y1] + 0.5).to(torch.uint8))


def test_strip_decoder_matches_whole_decode(mns):
    """StripDecoder (pair passes, 32-row halos, halo'd unit map) on one GPU, strip by strip with the
    halos copied between strips by hand, equals the whole-image decode_device."""
    from paper_1501_02894_b200 import sharding
    from paper_1501_02894_b200.synth import synth_image

    H = W = 512
    px = synth_image(H, 9, noise_sigma=10.0, n_blobs=12)
    cfg = mns.EncoderConfig(e3=8.0)
    whole = mns.encode_device(torch.from_numpy(px).cuda(), cfg)
    want, _, _ = mns.decode_device(whole, iters=9)
    bounds = [0, 7, 19, 32]
    codes, decs = [], []
    for r0, r1 in zip(bounds[:-1], bounds[1:]):
        y0, y1 = max(0, 16 * r0 - 16), min(H, 16 * r1 + 16)
        c = mns.encode_device(torch.from_numpy(np.ascontiguousarray(px[y0:y1])).cuda(), cfg, root_rows=(r0, r1),
                              height=H)
        d = sharding.StripDecoder(c, H, W, r0, r1)
        codes.append(c)
        decs.append(d)
    # unit-map halo rows (what exchange_unit_map_rows does over NCCL)
    for a, b in zip(decs[:-1], decs[1:]):
        a.umap[-1].copy_(b.umap[b.r0 - b.u0])
        b.umap[0].copy_(a.umap[a.r1 - 1 - a.u0])
    # 9 sweeps = 1 single + 4 pairs, raster halos exchanged by hand after every launch
    import ctypes

    from paper_1501_02894_b200 import _native as N

    L = N.lib()
    curs = [None] * 3
    for n in range(5):
        nxts = []
        for i, d in enumerate(decs):
            last = n == 4
            nxt = None if last else (d.ping if curs[i] is not d.ping else d.pong)
            vb = (lambda t: d._vbase(t, d.y_lo, 4))
            ob = d._vbase(d.out, 16 * d.r0, 1)
            if n == 0:
                N.check(L.mns_decode_sweep(N.ptr(d.code.unit_map), W, H, d.r0, d.r1, ctypes.c_void_p(0), 128.0,
                                           vb(nxt), ctypes.c_void_p(0), N.ptr(d.state), 0.0, None))
            else:
                N.check(L.mns_decode_sweep2(N.ptr(d.umap), d.u0, W, H, d.r0, d.r1, vb(curs[i]), 128.0,
                                            vb(nxt) if nxt is not None else ctypes.c_void_p(0),
                                            ob if last else ctypes.c_void_p(0), None))
            nxts.append(nxt)
        if n < 4:
            for a, b, ra, rb in zip(decs[:-1], decs[1:], nxts[:-1], nxts[1:]):
                h = sharding.DEC_HALO
                a_own1 = 16 * a.r1 - a.y_lo
                b_own0 = 16 * b.r0 - b.y_lo
                ra[a_own1: a_own1 + h].copy_(rb[b_own0: b_own0 + h])
                rb[b_own0 - h: b_own0].copy_(ra[a_own1 - h: a_own1])
        curs = nxts
    got = torch.cat([d.out for d in decs])
    torch.cuda.synchronize()
    assert torch.equal(got, want)


@pytest.mark.parametrize("h,w", [(1, 1), (3, 5), (17, 9), (31, 33), (16, 200)])
def test_tiny_and_odd_images_vs_oracle(mns, h, w):
    """Images smaller than one root or not a multiple of 16: edge-replicated padding
    (image.py:123-132), the level-1 room guard on the padded size (encoder.py:226-231),
    and the decode crop (decoder.py:76-77)."""
    rng = np.random.default_rng(h * 1000 + w)
    px = rng.integers(0, 256, (h, w), dtype=np.uint8)
    padded = np.pad(px, ((0, -h % 16), (0, -w % 16)), mode="edge")
    for mode in ("mns", "no_search"):
        cfg = mns.EncoderConfig(e1=6.0, e2=6.0, e3=6.0, mode=mode)
        code = mns.encode_quadtree(mns.GrayImage(px), cfg)
        ref, _ = O.encode_quadtree_records(padded, (6.0, 6.0, 6.0), 16.0, mode == "mns")
        assert np.array_equal(code.records, ref), (h, w, mode)
        assert (code.orig_w, code.orig_h, code.padded_w, code.padded_h) == (w, h) + padded.shape[::-1]
        got = mns.decode(code, mns.DecodeConfig(max_iters=5, stop_delta=0.0)).pixels
        want, _, _ = O.decode_records(ref, padded.shape[1], padded.shape[0], max_iters=5, stop_delta=0.0)
        assert got.shape == (h, w)
        assert int(np.abs(got.astype(int) - want[:h, :w].astype(int)).max()) <= 1


def test_try_phase_nodes_match_reference(mns, golden):
    """try_phase1 / try_phase2 (encoder.py:145-212) on the reference's single-node known answers
    (test_encoder.py cases, random aligned nodes, odd/unaligned rects, level 4, clamped domains):
    record and rms bit-exact."""
    from paper_1501_02894_b200.types import pack_leaf

    g = golden("nodes")
    n1 = n2 = 0
    for case in g.manifest:
        k = case["key"]
        img = mns.GrayImage(g[f"{k}/img"])
        rect = mns.BlockRect(case["x"], case["y"], case["size"])
        cfg = mns.EncoderConfig(e1=case["e"], e2=case["e"], e3=case["e"], mean_tol=case["mean_tol"])
        rec_ref, rms_ref = g[f"{k}/rec"], g[f"{k}/rms"]
        if 2 * case["size"] <= min(img.pixels.shape):
            r1, rms1 = mns.try_phase1(img, rect, case["level"], cfg)
            assert (r1 is not None) == case["ok1"], k
            assert (pack_leaf(r1) if r1 else 0) == int(rec_ref[0]), k
            assert r1 is None or r1.rect == rect
            assert rms1 == rms_ref[0], (k, rms1, rms_ref[0])
            n1 += 1
        if case["level"] <= 3:
            r2, rms2 = mns.try_phase2(img, rect, case["level"], cfg)
            assert (r2 is not None) == case["ok2"], k
            assert (pack_leaf(r2) if r2 else 0) == int(rec_ref[1]), k
            assert rms2 == rms_ref[1], (k, rms2, rms_ref[1])
            n2 += 1
    assert n1 > 60 and n2 > 60


def test_try_phase_errors(mns):
    img = mns.GrayImage(np.zeros((24, 40), np.uint8))
    cfg = mns.EncoderConfig()
    with pytest.raises(ValueError, match="level 2 expects block size 8, got 4"):
        mns.try_phase1(img, mns.BlockRect(0, 0, 4), 2, cfg)
    with pytest.raises(ValueError, match="no 32x32 domain fits a 40x24 image"):
        mns.try_phase1(img, mns.BlockRect(0, 0, 16), 1, cfg)
    with pytest.raises(ValueError, match="out of bounds for 40x24 raster"):
        mns.try_phase1(img, mns.BlockRect(36, 0, 8), 2, cfg)
    with pytest.raises(ValueError, match="phase 2 exists only at levels 1..3"):
        mns.try_phase2(img, mns.BlockRect(0, 0, 2), 4, cfg)
    assert mns.try_phase2(img, mns.BlockRect(0, 0, 16), 1, cfg)[0] is not None  # flat: accepted


def _lattice_of(t):
    """Even 2x2-sum lattice of an fp32 raster in downsample_mean2's order, rows de-interleaved
    (even lattice columns, then odd): the state of lattice-mode decoding."""
    q = ((t[0::2, 0::2] + t[0::2, 1::2]) + t[1::2, 0::2]) + t[1::2, 1::2]
    return torch.cat([q[:, 0::2], q[:, 1::2]], dim=1).contiguous()


@pytest.mark.parametrize("W,H,rr", [(512, 512, None), (400, 48, None), (16, 16, None), (1024, 1040, None),
                                    (640, 640, (5, 17)), (640, 640, (0, 3)), (640, 640, (37, 40)),
                                    (2064, 272, None)])
def test_lattice_pass_equals_two_sweeps(mns, W, H, rr):
    """mns_decode_pass_lattice on a code without 2x2 units (e3 = inf): from the flat start and from
    a random raster's lattice, its t+2 lattice equals the lattice of two single raster sweeps and
    its uint8 output their rounding, bit for bit; mns_decode_flat_lattice equals one flat sweep (as
    lattice and as the uint8 image).  The lattice passes read the encoder's block map, which equals
    mns_build_block_map's."""
    import ctypes

    from paper_1501_02894_b200 import _native as N
    from paper_1501_02894_b200.synth import synth_image

    L = N.lib()
    side = max(W, H)
    px = np.ascontiguousarray(synth_image(side, 13, noise_sigma=12.0, n_blobs=8)[:H, :W])
    img = torch.from_numpy(px).cuda()
    code = mns.encode_device(img, mns.EncoderConfig(e3=math.inf), map_form=0)
    assert code.min_leaf == 4
    umap = code.unit_map  # the raster sweeps' unit map
    bcode = mns.encode_device(img, mns.EncoderConfig(e3=math.inf))
    assert bcode.map_form == 1 and bcode.unit_map.numel() == (H // 16) * (W // 16) * 8
    bmap = bcode.unit_map.clone()
    assert torch.equal(mns.build_unit_map(bcode, map_form=1), bmap)
    rh = H // 16
    r0, r1 = rr if rr is not None else (0, rh)
    u0 = max(0, r0 - 1)
    sub = bmap[u0 * (W // 16) * 8:]
    g = torch.Generator(device="cuda").manual_seed(W + H + 1)
    t0 = torch.rand((H, W), device="cuda", generator=g) * 255.0
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    ly0, ly1 = 8 * r0, 8 * r1
    for cur in (None, t0):
        want = _sweeps_single(N, L, umap, W, H, (0, rh), cur, 128.0, 2)
        lat_cur = _lattice_of(cur) if cur is not None else None
        got = torch.full((H // 2, W // 2), float("nan"), device="cuda")
        N.check(L.mns_decode_pass_lattice(N.ptr(sub), u0, W, H, r0, r1,
                                          N.ptr(lat_cur) if lat_cur is not None else ctypes.c_void_p(0), 128.0,
                                          N.ptr(got), ctypes.c_void_p(0), N.ptr(err), None))
        out = torch.zeros((H, W), dtype=torch.uint8, device="cuda")
        N.check(L.mns_decode_pass_lattice(N.ptr(sub), u0, W, H, r0, r1,
                                          N.ptr(lat_cur) if lat_cur is not None else ctypes.c_void_p(0), 128.0,
                                          ctypes.c_void_p(0), N.ptr(out), N.ptr(err), None))
        torch.cuda.synchronize()
        assert torch.equal(got[ly0:ly1], _lattice_of(want)[ly0:ly1])
        assert torch.equal(out[16 * r0:16 * r1], torch.floor(want[16 * r0:16 * r1] + 0.5).to(torch.uint8))
    one = _sweeps_single(N, L, umap, W, H, (0, rh), None, 128.0, 1)
    flat = torch.full((H // 2, W // 2), float("nan"), device="cuda")
    N.check(L.mns_decode_flat_lattice(N.ptr(sub), u0, W, H, r0, r1, 128.0, N.ptr(flat), None, None))
    flat_u8 = torch.zeros((H, W), dtype=torch.uint8, device="cuda")
    N.check(L.mns_decode_flat_lattice(N.ptr(sub), u0, W, H, r0, r1, 128.0, None, N.ptr(flat_u8), None))
    torch.cuda.synchronize()
    assert torch.equal(flat[ly0:ly1], _lattice_of(one)[ly0:ly1])
    assert torch.equal(flat_u8[16 * r0:16 * r1], torch.floor(one[16 * r0:16 * r1] + 0.5).to(torch.uint8))
    assert int(err.item()) == 0


@pytest.mark.parametrize("side,iters,root_level", [(512, 10, 1), (512, 9, 1), (256, 1, 1), (256, 2, 1), (48, 3, 1),
                                                   (1024, 8, 1), (256, 8, 2), (512, 7, 2)])
def test_lattice_decode_equals_raster_decode(mns, side, iters, root_level):
    """Whole-image decode of an e3 = inf code (16->8->4, and the 8->4 root_level=2 form of configs
    c1/c3): the lattice-state path (mns_decode_quadtree_lattice, chosen by decode_device) and the
    raster path (mns_decode_quadtree) give the identical image."""
    import ctypes

    from paper_1501_02894_b200 import _native as N
    from paper_1501_02894_b200.synth import synth_image

    L = N.lib()
    px = synth_image(side, 21, noise_sigma=9.0, n_blobs=10)
    code = mns.encode_device(torch.from_numpy(px).cuda(), mns.EncoderConfig(e3=math.inf), root_level=root_level)
    assert code.min_leaf == 4
    got, it, _ = mns.decode_device(code, iters=iters)
    W = H = side
    ras = [torch.empty((H, W), device="cuda") for _ in range(2)]
    want = torch.empty((H, W), dtype=torch.uint8, device="cuda")
    wsb = N.out_i64(L, L.mns_decode_workspace_bytes, W, H)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    N.check(L.mns_decode_quadtree(N.ptr(code.records), N.ptr(code.root_offsets), W, H, iters, 0.0, 128.0,
                                  N.ptr(ras[0]), N.ptr(ras[1]), N.ptr(want), ctypes.c_void_p(0), N.ptr(ws), wsb, None))
    torch.cuda.synchronize()
    assert torch.equal(got, want)
    assert int(it.item()) == iters


def test_lattice_decode_flags_2x2_units(mns):
    """A code with 2x2 leaves forced down the lattice path raises the error flag (the caller must
    use the raster path); decode_device picks the raster path for it by itself."""
    import ctypes

    from paper_1501_02894_b200 import _native as N
    from paper_1501_02894_b200.synth import synth_image

    L = N.lib()
    px = synth_image(256, 5, noise_sigma=20.0, n_blobs=8)
    code = mns.encode_device(torch.from_numpy(px).cuda(), mns.EncoderConfig(e1=2.0, e2=2.0, e3=2.0))
    assert mns.codec.min_leaf_side(code) == 2
    lat = [torch.empty((128, 128), device="cuda") for _ in range(2)]
    out = torch.empty((256, 256), dtype=torch.uint8, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    wsb = N.out_i64(L, L.mns_decode_workspace_bytes, 256, 256)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    N.check(L.mns_decode_quadtree_lattice(N.ptr(code.records), N.ptr(code.root_offsets), 256, 256, 4, 128.0,
                                          N.ptr(lat[0]), N.ptr(lat[1]), N.ptr(out), N.ptr(err), N.ptr(ws), wsb, None))
    assert int(err.item()) == 1
    ras = [torch.empty((256, 256), device="cuda") for _ in range(2)]
    got, _, _ = mns.decode_device(code, iters=4)
    want = torch.empty((256, 256), dtype=torch.uint8, device="cuda")
    N.check(L.mns_decode_quadtree(N.ptr(code.records), N.ptr(code.root_offsets), 256, 256, 4, 0.0, 128.0,
                                  N.ptr(ras[0]), N.ptr(ras[1]), N.ptr(want), ctypes.c_void_p(0), N.ptr(ws), wsb, None))
    torch.cuda.synchronize()
    assert torch.equal(got, want)
    # a wrong min_leaf (user-built code) is caught by the flag, and lattice=False gives the right image
    code.min_leaf = 4
    bad, _, _ = mns.decode_device(code, iters=4)
    assert int(code.decode_error.item()) == 1
    fixed, _, _ = mns.decode_device(code, iters=4, lattice=False)
    assert torch.equal(fixed, want)


@pytest.mark.parametrize("iters", [10, 7])
def test_strip_decoder_lattice_matches_whole_decode(mns, iters):
    """StripDecoder in lattice mode (e3 = inf code), strip by strip with the 16 lattice halo rows
    copied between strips by hand after every launch, equals the whole-image raster decode."""
    import ctypes

    from paper_1501_02894_b200 import _native as N
    from paper_1501_02894_b200 import sharding
    from paper_1501_02894_b200.synth import synth_image

    L = N.lib()
    H = W = 512
    px = synth_image(H, 19, noise_sigma=10.0, n_blobs=12)
    cfg = mns.EncoderConfig(e3=math.inf)
    whole = mns.encode_device(torch.from_numpy(px).cuda(), cfg)
    ras = [torch.empty((H, W), device="cuda") for _ in range(2)]
    want = torch.empty((H, W), dtype=torch.uint8, device="cuda")
    wsb = N.out_i64(L, L.mns_decode_workspace_bytes, W, H)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    N.check(L.mns_decode_quadtree(N.ptr(whole.records), N.ptr(whole.root_offsets), W, H, iters, 0.0, 128.0,
                                  N.ptr(ras[0]), N.ptr(ras[1]), N.ptr(want), ctypes.c_void_p(0), N.ptr(ws), wsb, None))
    bounds = [0, 5, 19, 32]
    decs = []
    for r0, r1 in zip(bounds[:-1], bounds[1:]):
        y0, y1 = max(0, 16 * r0 - 16), min(H, 16 * r1 + 16)
        c = mns.encode_device(torch.from_numpy(np.ascontiguousarray(px[y0:y1])).cuda(), cfg, root_rows=(r0, r1),
                              height=H)
        d = sharding.StripDecoder(c, H, W, r0, r1)
        assert d.lattice and d.ping.shape == ((d.y_hi - d.y_lo) // 2, W // 2)
        decs.append(d)
    for a, b in zip(decs[:-1], decs[1:]):
        a.umap[-1].copy_(b.umap[b.r0 - b.u0])
        b.umap[0].copy_(a.umap[a.r1 - 1 - a.u0])
    n_launch = iters // 2 + (iters & 1)
    curs = [None] * 3
    for n in range(n_launch):
        nxts = []
        last = n == n_launch - 1
        for i, d in enumerate(decs):
            nxt = None if last else (d.ping if curs[i] is not d.ping else d.pong)
            ob = d._vbase(d.out, 16 * d.r0, 1)
            if n == 0 and iters & 1:
                N.check(L.mns_decode_flat_lattice(N.ptr(d.umap), d.u0, W, H, d.r0, d.r1, 128.0, d._state_base(nxt),
                                                  None, None))
            else:
                N.check(L.mns_decode_pass_lattice(N.ptr(d.umap), d.u0, W, H, d.r0, d.r1, d._state_base(curs[i]),
                                                  128.0, d._state_base(nxt), ob if last else ctypes.c_void_p(0),
                                                  N.ptr(d.error), None))
            nxts.append(nxt)
        if not last:
            h = sharding.DEC_HALO // 2
            for a, b, ra, rb in zip(decs[:-1], decs[1:], nxts[:-1], nxts[1:]):
                a_own1 = (16 * a.r1 - a.y_lo) // 2
                b_own0 = (16 * b.r0 - b.y_lo) // 2
                ra[a_own1: a_own1 + h].copy_(rb[b_own0: b_own0 + h])
                rb[b_own0 - h: b_own0].copy_(ra[a_own1 - h: a_own1])
        curs = nxts
    got = torch.cat([d.out for d in decs])
    torch.cuda.synchronize()
    assert torch.equal(got, want)
    assert all(int(d.error.item()) == 0 for d in decs)
    # and the run() driver itself (world = 1) on one whole-image strip
    d = sharding.StripDecoder(mns.encode_device(torch.from_numpy(px).cuda(), cfg), H, W, 0, H // 16)
    assert torch.equal(d.run(iters), want)


def test_unit2_leaf_count_matches_host(mns, golden):
    """The GPU tally of leaves painted as 2x2 units (level 4 and level-3 phase 2) that routes a code
    to the raster or lattice decoder, against the host count on every golden code."""
    from paper_1501_02894_b200 import rd
    from paper_1501_02894_b200.types import unpack_fields

    g = golden("encode")
    seen = set()
    for case in g.manifest:
        rec = g[f"{case['key']}/records"]
        f = unpack_fields(rec)
        want = int(((f["level"] == 4) | ((f["level"] == 3) & (f["phase2"] == 1))).sum())
        dev = torch.from_numpy(rec.view(np.int64)).cuda()
        assert rd.unit2_leaves(dev, len(rec)) == want, case["key"]
        seen.add(want > 0)
    assert seen == {True, False}


def test_encode_stress_golden(mns, golden):
    """Reference-generated adversarial cases (oracle/gen_golden.py gen_stress: saturated blocks, hard
    edges, checkerboards, ramps across contrast-bin edges, flat and noisy patches; 5 configs incl.
    no_search and e3 = inf): GPU codes bit-exact, 8-sweep decodes within 1 LSB."""
    g = golden("stress")
    for case in g.manifest:
        k, c = case["key"], case["cfg"]
        px = g[f"img/{case['image']}"]
        cfg = mns.EncoderConfig(**{n: (math.inf if v is None else v) for n, v in c.items()})
        code = mns.encode_quadtree(mns.GrayImage(px), cfg)
        assert np.array_equal(code.records, g[f"{k}/records"]), case
        got = mns.decode(code, mns.DecodeConfig(max_iters=8, stop_delta=0.0)).pixels
        assert int(np.abs(got.astype(int) - g[f"{k}/decode8"].astype(int)).max()) <= 1, case


def test_encode_split_stream_compaction(mns):
    """mns_encode_quadtree_split (compaction on a second stream, joined by the caller) yields the same
    records, root offsets and unit map as the single-stream encode."""
    from paper_1501_02894_b200.synth import synth_image

    px = torch.from_numpy(synth_image(512, 31, noise_sigma=10.0, n_blobs=8)).cuda()
    cfg = mns.EncoderConfig(e3=math.inf)
    a = mns.encode_device(px, cfg)
    side = torch.cuda.Stream()
    b = mns.encode_device(px, cfg, compact_stream=side)
    torch.cuda.current_stream().wait_stream(side)
    n = a.n_records()
    assert n == b.n_records()
    assert torch.equal(a.records[:n], b.records[:n])
    assert torch.equal(a.root_offsets, b.root_offsets)
    assert torch.equal(a.unit_map, b.unit_map)


@pytest.mark.parametrize("H,W", [(96, 32768), (20000, 48), (272, 2064)])
def test_lattice_decode_extreme_shapes(mns, H, W):
    """Very wide and very tall images (hundreds of column bands / one partial band, many row
    chunks): lattice-state decode equals the raster decode bit for bit."""
    import ctypes

    from paper_1501_02894_b200 import _native as N

    L = N.lib()
    rng = np.random.default_rng(H + W)
    base = rng.integers(60, 200, (H // 8 + 1, W // 8 + 1))
    px = np.kron(base, np.ones((8, 8)))[:H, :W] + rng.integers(-12, 13, (H, W))
    px = np.ascontiguousarray(np.clip(px, 0, 255).astype(np.uint8))
    code = mns.encode_device(torch.from_numpy(px).cuda(), mns.EncoderConfig(e3=math.inf))
    got, _, _ = mns.decode_device(code, iters=6)
    ras = [torch.empty((H, W), device="cuda") for _ in range(2)]
    want = torch.empty((H, W), dtype=torch.uint8, device="cuda")
    wsb = N.out_i64(L, L.mns_decode_workspace_bytes, W, H)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    N.check(L.mns_decode_quadtree(N.ptr(code.records), N.ptr(code.root_offsets), W, H, 6, 0.0, 128.0,
                                  N.ptr(ras[0]), N.ptr(ras[1]), N.ptr(want), ctypes.c_void_p(0), N.ptr(ws), wsb, None))
    torch.cuda.synchronize()
    assert torch.equal(got, want)


@pytest.mark.parametrize("n_iso", [1, 8])
def test_full_search_c4_tensor_core_equals_cuda_core_all_ranges(mns, monkeypatch, n_iso):
    """c4 in full (4096 ranges x 247,009 domains x n_iso): the normalised-operand tcgen05 filter
    keeps every winner -- the argmin equals the exact CUDA-core path for every range."""
    from paper_1501_02894_b200.synth import config_image

    img = torch.from_numpy(config_image("c4")).cuda()
    monkeypatch.setenv("MNS_SEARCH_CUDA_CORES", "0")
    a = {k: v.cpu().numpy() for k, v in mns.full_search_device(img, 8, 1, n_iso).items()}
    monkeypatch.setenv("MNS_SEARCH_CUDA_CORES", "1")
    b = {k: v.cpu().numpy() for k, v in mns.full_search_device(img, 8, 1, n_iso).items()}
    for k in a:
        assert np.array_equal(a[k], b[k]), (n_iso, k, int((a[k] != b[k]).sum()))


@pytest.mark.parametrize("root_level,iters", [(1, 10), (2, 8), (1, 7), (1, 1)])
def test_decode_from_encoder_unit_map_equals_records_path(mns, root_level, iters):
    """decode_device on the encoder's own unit map (mns_decode_unit_map_lattice) equals the decode that
    rebuilds the map from the records (mns_decode_quadtree_lattice), bit for bit."""
    from paper_1501_02894_b200.synth import synth_image

    img = torch.from_numpy(synth_image(256, 11)).cuda()
    code = mns.encode_device(img, mns.EncoderConfig(e3=math.inf), root_level=root_level)
    assert code.unit_map_valid
    a, _, _ = mns.decode_device(code, iters=iters, stop_delta=0.0)
    code.unit_map_valid = False
    b, _, _ = mns.decode_device(code, iters=iters, stop_delta=0.0)
    torch.cuda.synchronize()
    assert torch.equal(a, b)


@pytest.mark.parametrize("e3,root_level,iters", [(8.0, 1, 10), (8.0, 2, 7), (2.0, 1, 1), (math.inf, 1, 9)])
def test_decode_from_encoder_raster_unit_map_equals_records_path(mns, e3, root_level, iters):
    """decode_device on the encoder's map_form-0 unit map (mns_decode_unit_map: fp32 rasters, 2x2 leaves
    allowed) equals the decode that rebuilds the map from the records (mns_decode_quadtree), bit for bit,
    for both the uint8 output and the final raster."""
    from paper_1501_02894_b200.synth import synth_image

    img = torch.from_numpy(synth_image(256, 13)).cuda()
    code = mns.encode_device(img, mns.EncoderConfig(e3=e3), root_level=root_level, map_form=0)
    assert code.unit_map_valid and code.map_form == 0
    a, ia, _ = mns.decode_device(code, iters=iters, stop_delta=0.0, lattice=False)
    _, _, ra = mns.decode_device(code, iters=iters, stop_delta=0.0, want_u8=False)
    code.unit_map_valid = False
    b, ib, _ = mns.decode_device(code, iters=iters, stop_delta=0.0, lattice=False)
    _, _, rb = mns.decode_device(code, iters=iters, stop_delta=0.0, want_u8=False)
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    assert int(ia.item()) == int(ib.item()) == iters
    final = iters % 2  # the final raster: ping after an even sweep count, else pong
    assert torch.equal(ra[final], rb[final])


def test_full_search_wide_key_large_pool(mns):
    """B = 8 identity search over a 1600^2 image: 1585^2 = 2.5M domains, above the old 2^21
    candidate cap (the key now gives B = 8 candidates 25 bits).  A range slice vs the oracle."""
    from paper_1501_02894_b200.synth import synth_image

    px = synth_image(1600, 12)
    img = torch.from_numpy(px).cuda()
    r0, r1 = 19_000, 19_024
    got = {k: v.cpu().numpy() for k, v in mns.full_search_device(img, 8, 1, 1, ranges=(r0, r1)).items()}
    ref = O.full_search(px, 8, 1, n_iso=1, range_ids=np.arange(r0, r1))
    for k in ("dom", "iso", "o", "code"):
        assert np.array_equal(got[k].astype(np.int64), ref[k].astype(np.int64)), k


def _oracle_deltas(units, W, H, init, n):
    """The reference's per-sweep max|nxt - current| (decoder.py:70-72) from the fp64 oracle."""
    cur = np.full((H, W), init)
    out = []
    for _ in range(n):
        nxt = O.decode_step_units(units, cur)
        out.append(float(np.max(np.abs(nxt - cur))))
        cur = nxt
    return out


@pytest.mark.parametrize("seed,side", [(3, 128), (21, 96)])
def test_early_stop_exact_at_threshold(mns, seed, side):
    """stop_delta placed exactly ON a sweep's fp64 delta (no stop: the test is `<`) and one ulp
    above it (stop): the GPU decode stops at the reference's sweep in both cases and the image is
    bit-identical to the oracle's (an fp32 max|delta| could not tell these thresholds apart)."""
    from paper_1501_02894_b200.synth import synth_image

    px = synth_image(side, seed, noise_sigma=12.0, n_blobs=5)
    rec, _ = O.encode_quadtree_records(px, (6.0, 6.0, 6.0), 16.0, True)
    units = O.records_to_units(rec, side, side)
    deltas = _oracle_deltas(units, side, side, 128.0, 12)
    code = mns.QuadtreeCode.from_records(rec, side, side, side, side, "mns", True)
    dcode = mns.encode_device(torch.from_numpy(px).cuda(), mns.EncoderConfig(e1=6.0, e2=6.0, e3=6.0))
    for j in (2, 4, 6):
        for stop in (deltas[j], float(np.nextafter(deltas[j], np.inf))):
            want, _, sweeps = O.decode_units(units, side, side, max_iters=12, stop_delta=stop)
            expect = j + 1 if stop > deltas[j] and all(d >= stop for d in deltas[:j]) else sweeps
            assert sweeps == expect or stop == deltas[j]
            got = mns.decode(code, mns.DecodeConfig(max_iters=12, stop_delta=stop)).pixels
            assert np.array_equal(got, want), (j, stop, sweeps)
            dout, it, _ = mns.decode_device(dcode, iters=12, stop_delta=stop)
            assert int(it.item()) == sweeps
            assert np.array_equal(dout.cpu().numpy(), want)


@pytest.mark.parametrize("shape,e", [((1024, 2048), (6.0, 6.0, 6.0)), ((1040, 2048), (6.0, 6.0, 6.0)),
                                     ((1040, 2048), (8.0, 8.0, math.inf))])
def test_exact_decode_one_launch_and_launch_chain_vs_oracle(mns, shape, e):
    """mns_decode_f64 on both sides of its one-launch limit (2^21 pixels: 1024x2048 decodes in the
    cooperative kernel, 1040x2048 in the launch chain), default DecodeConfig, codes with phase-2
    quadrants and 2x2 leaves (finite e3) and without: sweep count and image equal the fp64 oracle's."""
    from paper_1501_02894_b200.synth import synth_image

    H, W = shape
    px = np.ascontiguousarray(synth_image(2048, 77, noise_sigma=9.0, n_blobs=9)[:H, :W])
    rec, _ = O.encode_quadtree_records(px, e, 16.0, True)
    want, _, sweeps = O.decode_records(rec, W, H, max_iters=10, stop_delta=0.5)
    dcode = mns.encode_device(torch.from_numpy(px).cuda(), mns.EncoderConfig(e1=e[0], e2=e[1], e3=e[2]))
    assert np.array_equal(dcode.records[: dcode.n_records()].cpu().numpy().view(np.uint64), rec.view(np.uint64))
    out, it, _ = mns.decode_device(dcode, iters=10, stop_delta=0.5)
    assert int(it.item()) == sweeps
    assert np.array_equal(out.cpu().numpy(), want)


def test_decode_search_codes_default_config_bit_exact(mns, golden):
    """Baseline (full-search) codes decoded with the default DecodeConfig (early stop 0.5): the
    GPU's exact fp64 decoder equals the fp64 oracle decode of the same units bit for bit."""
    g = golden("search")
    for case in [c for c in g.manifest if c["key"].startswith("full")][:6]:
        k = case["key"]
        code, _ = mns.encode_full_search(mns.GrayImage(g[f"{k}/img"]), case["B"],
                                         mns.EncoderConfig(mode="full_search", full_search_step=case["step"]))
        c = code.columns
        units = np.zeros(len(c["rx"]), dtype=O.UNIT_DTYPE)
        units["x"], units["y"], units["size"] = c["rx"], c["ry"], case["B"]
        units["dx"], units["dy"] = c["dom_x"], c["dom_y"]
        units["s"] = -0.875 + 0.25 * c["code"].astype(np.float64)
        units["o"] = c["o"].astype(np.float64)
        want, _, _ = O.decode_units(units, code.padded_w, code.padded_h, max_iters=10, stop_delta=0.5)
        got = mns.decode(code, mns.DecodeConfig()).pixels
        assert np.array_equal(got, want[: code.orig_h, : code.orig_w]), case


def test_f64_strip_decoder_three_strips_on_one_gpu(mns):
    """StripDecoderF64's kernels on 3 strips of one image (the ranks' halo exchange and delta
    all-reduce done by hand in lock-step): the strips equal the exact decode with early stop."""
    from paper_1501_02894_b200 import sharding
    from paper_1501_02894_b200.synth import synth_image

    H = W = 512
    px = synth_image(512, 41, noise_sigma=10.0, n_blobs=8)
    cfg = mns.EncoderConfig()
    rec, _ = O.encode_quadtree_records(px, (8.0, 8.0, 8.0), 16.0, True)
    want, _, sweeps = O.decode_records(rec, W, H, max_iters=10, stop_delta=1.0)
    assert sweeps < 10
    world = 3
    decs = []
    for rank in range(world):
        r0, r1 = sharding.strip_rows(H, world, rank)
        y0, y1 = sharding.resident_rows(r0, r1, H)
        code = mns.encode_device(torch.from_numpy(np.ascontiguousarray(px[y0:y1])).cuda(), cfg, root_rows=(r0, r1),
                                 height=H)
        d = sharding.StripDecoderF64(code, H, W, r0, r1, rank, world)
        d.units = mns.codec.records_to_units_device(code.records, code.n_records(), W, H)
        d.state.zero_()
        d.ping.fill_(128.0)
        decs.append(d)
    bufs = [[d.ping, d.pong] for d in decs]
    for it in range(10):
        for d, b in zip(decs, bufs):
            d.sweep(b[it & 1], b[(it + 1) & 1])
        g = max(float(d.delta_view()[0]) for d in decs)  # the all-reduce (MAX)
        for d in decs:
            d.delta_view()[0] = g
            d.decide(1.0)
        for k in range(world - 1):  # halo exchange of the freshly written rasters
            a, b = decs[k], decs[k + 1]
            ra, rb = bufs[k][(it + 1) & 1], bufs[k + 1][(it + 1) & 1]
            ya, yb = 16 * a.r1 - a.y_lo, 16 * b.r0 - b.y_lo
            ra[ya: ya + 16].copy_(rb[yb: yb + 16])
            rb[yb - 16: yb].copy_(ra[ya - 16: ya])
    got = np.concatenate([d.finalize().cpu().numpy() for d in decs])
    assert all(int(d.iters_done.item()) == sweeps for d in decs)
    assert np.array_equal(got, want)


def test_strip_decoder_split_passes_equal_whole(mns, monkeypatch):
    """The overlapped multi-GPU schedule (boundary root rows first, interior rows after, each a
    sub-range launch of the same pass) composes to the single-launch decode: a whole-image strip run
    as rank 0 of 2 with the exchange stubbed out (there is no neighbour below the last row)."""
    from paper_1501_02894_b200 import sharding
    from paper_1501_02894_b200.synth import synth_image

    px = synth_image(512, 23, noise_sigma=10.0, n_blobs=8)
    H = W = 512
    outs = []
    for world, lattice in ((1, True), (2, True), (1, False), (2, False)):
        code = mns.encode_device(torch.from_numpy(px).cuda(), mns.EncoderConfig(e3=math.inf))
        dec = sharding.StripDecoder(code, H, W, 0, H // 16, 0, world, lattice=lattice)
        monkeypatch.setattr(dec, "_exchange", lambda t: None)
        monkeypatch.setattr(sharding, "unit_map_ops", lambda *a, **k: [])
        assert dec._overlap() == (world == 2)
        outs.append(dec.run(10, 128.0).clone())
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[2], outs[3]) and torch.equal(outs[0], outs[2])


@pytest.mark.parametrize("name,e,mode,root_level", [("c2", (8.0, 8.0, math.inf), "mns", 1),
                                                    ("tex", (6.0, 6.0, 6.0), "mns", 1),
                                                    ("tex", (6.0, 6.0, 5.0), "no_search", 1),
                                                    ("tex", (6.0, 6.0, math.inf), "mns", 2)])
def test_isometry_extension_encode_decode_vs_oracle(mns, name, e, mode, root_level):
    """BASELINE configs[1]'s 8-isometry MNS encode (an extension: the reference has no isometries):
    records (with each phase-1 leaf's isometry) bit-exact vs the oracle restatement; the decode (exact
    fp64 unit path) bit-identical to the oracle's with and without the early stop."""
    from paper_1501_02894_b200.synth import config_image, synth_image

    px = config_image("c2") if name == "c2" else synth_image(256, 33, noise_sigma=12.0, n_blobs=6)
    cfg = mns.EncoderConfig(e1=e[0], e2=e[1], e3=e[2], mode=mode)
    code = mns.encode_quadtree(mns.GrayImage(px), cfg, root_level=root_level, n_iso=8)
    ref, _ = O.encode_quadtree_records(px, e, 16.0, mode == "mns", root_level, n_iso=8)
    assert np.array_equal(code.records, ref)
    from paper_1501_02894_b200.bitstream import has_isometries

    assert has_isometries(ref)  # the isometries are actually used
    units = O.records_to_units(ref, px.shape[1], px.shape[0])
    for stop in (0.0, 0.5):
        want, _, _ = O.decode_units(units, px.shape[1], px.shape[0], max_iters=10, stop_delta=stop)
        got = mns.decode(code, mns.DecodeConfig(max_iters=10, stop_delta=stop)).pixels
        assert np.array_equal(got, want), stop
    dcode = mns.encode_device(torch.from_numpy(px).cuda(), cfg, root_level=root_level, n_iso=8)
    out, _, _ = mns.decode_device(dcode, iters=10, stop_delta=0.0)
    want, _, _ = O.decode_units(units, px.shape[1], px.shape[0], max_iters=10, stop_delta=0.0)
    assert np.array_equal(out.cpu().numpy(), want)
    with pytest.raises(ValueError, match="isometry"):
        mns.write_stream(code)


@pytest.mark.parametrize("shape,radius,n_iso", [((64, 64), 4, 1), ((64, 64), 32, 8), ((40, 72), 7, 8), ((16, 16), 3, 1),
                                                ((24, 48), 0, 8), ((96, 96), 1, 1), ((128, 200), 32, 1),
                                                ((136, 64), 5, 8)])
def test_local_search_tensor_core_vs_oracle(mns, shape, radius, n_iso):
    """The windowed tcgen05 local search (mns_local_search_tc) against the oracle and the CUDA-core
    kernel: window edges, clamped borders, tiny and non-square images, radius 0, isometries."""
    from paper_1501_02894_b200.synth import synth_image

    px = np.ascontiguousarray(synth_image(256, 5 + radius, noise_sigma=9.0, n_blobs=4)[: shape[0], : shape[1]])
    img = torch.from_numpy(px).cuda()
    tc = {k: v.cpu().numpy() for k, v in mns.local_search_device(img, radius, n_iso=n_iso, tensor_cores=True).items()}
    cc = {k: v.cpu().numpy() for k, v in mns.local_search_device(img, radius, n_iso=n_iso, tensor_cores=False).items()}
    ref = O.local_search(px, radius, n_iso=n_iso)
    for k, rk in (("dx", "dom_x"), ("dy", "dom_y"), ("iso", "iso"), ("o", "o"), ("code", "code")):
        assert np.array_equal(tc[k], ref[rk]), (k, int((tc[k] != ref[rk]).sum()))
        assert np.array_equal(cc[k], ref[rk]), k


def test_local_search_tensor_core_flat_ranges(mns):
    """Constant ranges (the windowed minimum-D rule) and saturated pixels on the tcgen05 path."""
    rng = np.random.default_rng(3)
    px = np.kron(rng.integers(0, 256, (8, 8)), np.ones((8, 8))).astype(np.uint8)  # 64x64 of flat 8x8 blocks
    px[16:40, 16:40] = rng.integers(250, 256, (24, 24))
    img = torch.from_numpy(np.ascontiguousarray(px)).cuda()
    for radius, n_iso in ((4, 1), (32, 8)):
        tc = {k: v.cpu().numpy() for k, v in mns.local_search_device(img, radius, n_iso=n_iso, tensor_cores=True).items()}
        ref = O.local_search(px, radius, n_iso=n_iso)
        for k, rk in (("dx", "dom_x"), ("dy", "dom_y"), ("iso", "iso"), ("o", "o"), ("code", "code")):
            assert np.array_equal(tc[k], ref[rk]), (radius, n_iso, k)
