"""Full-size parity at the benchmarked configurations (BASELINE.json configs[2..4]).

Every check compares the CUDA path with the CPU oracle (oracle/, pinned to the reference's
own goldens by tests/test_oracle_golden.py) on the very inputs bench.py times:

* c5  -- one 16384^2 image (seed 5, sigma 10, 24 blobs), 16->8->4 (e3 = inf): the records and
         root offsets of the whole image bit-exact; the 10-sweep decode through bench.py's own
         path (StripDecoder, lattice state) and through decode_device within 1 LSB per pixel
         and 0.01 dB PSNR of the fp64 oracle decode (north_star's bar); row-strip encodes
         (4 strips, 16-row halo) concatenate to the same code;
* c3  -- all 256 images of the batch (seeds 1000..1255), 8->4, bit-exact per image;
* c4  -- all 4096 ranges x 247,009 domains at 1 and 8 isometries, and the +-4 / +-32 local
         search, bit-exact (domain, isometry, offset, contrast) per range.
Reference: encoder.py:215-246 (quadtree), :249-309 (full search), :312-347 (local search),
decoder.py:66-77 (decode).
"""
import math

import numpy as np
import pytest

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


@pytest.fixture(scope="module")
def c5():
    """The c5 image and its oracle code + 10-sweep fp64 decode (computed once per module)."""
    from paper_1501_02894_b200.synth import config_image

    px = config_image("c5")
    rec, counts = O.encode_quadtree_records(px, (8.0, 8.0, math.inf), 16.0, True, 1)
    want, _, sweeps = O.decode_records(rec, px.shape[1], px.shape[0], max_iters=10, stop_delta=0.0)
    assert sweeps == 10
    offs = np.zeros(len(counts) + 1, np.int64)
    np.cumsum(counts, out=offs[1:])
    return {"px": px, "rec": rec, "offs": offs, "want": want}


def test_c5_encode_bit_exact(mns, c5):
    px = c5["px"]
    code = mns.encode_device(torch.from_numpy(px).cuda(), mns.EncoderConfig(e3=math.inf))
    n = code.n_records()
    assert n == len(c5["rec"]) == 16_555_747
    got = code.records[:n].cpu().numpy().view(np.uint64)
    bad = np.flatnonzero(got != c5["rec"])
    assert bad.size == 0, f"{bad.size} records differ, first at {bad[:5]}"
    assert np.array_equal(code.root_offsets.cpu().numpy().astype(np.int64), c5["offs"])


def test_c5_bench_path_decode_within_1lsb(mns, c5):
    """bench.py's step at N=1: encode (compaction on a second stream) + StripDecoder lattice decode."""
    from paper_1501_02894_b200 import sharding

    px = c5["px"]
    H, W = px.shape
    img = torch.from_numpy(px).cuda()
    n_roots = (H // 16) * (W // 16)
    code = mns.DeviceCode(torch.empty(64 * n_roots, dtype=torch.int64, device="cuda"),
                          torch.empty(n_roots + 1, dtype=torch.int32, device="cuda"),
                          torch.zeros(1, dtype=torch.int64, device="cuda"), W, H, 1, 0, H // 16,
                          unit_map=torch.empty(8 * n_roots, dtype=torch.int32, device="cuda"), map_form=1)
    dec = sharding.StripDecoder(code, H, W, 0, H // 16, 0, 1, lattice=True)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    mns.encode_device(img, mns.EncoderConfig(e3=math.inf), root_rows=(0, H // 16), height=H, out=code,
                      compact_stream=side)
    out = dec.run(10, 128.0)
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    assert int(dec.error.item()) == 0
    n = code.n_records()
    assert np.array_equal(code.records[:n].cpu().numpy().view(np.uint64), c5["rec"])
    got = out.cpu().numpy()
    want = c5["want"]
    diff = np.abs(got.astype(np.int16) - want.astype(np.int16))
    assert int(diff.max()) <= 1, int(diff.max())
    assert abs(_psnr(px, got) - _psnr(px, want)) <= 0.01


def test_c5_decode_device_within_1lsb(mns, c5):
    """The public device API (decode_device on the encoder's unit map) at c5."""
    px = c5["px"]
    code = mns.encode_device(torch.from_numpy(px).cuda(), mns.EncoderConfig(e3=math.inf))
    out, _, _ = mns.decode_device(code, iters=10, stop_delta=0.0)
    got = out.cpu().numpy()
    diff = np.abs(got.astype(np.int16) - c5["want"].astype(np.int16))
    assert int(diff.max()) <= 1
    assert abs(_psnr(px, got) - _psnr(px, c5["want"])) <= 0.01


def test_c5_strip_encode_bit_exact(mns, c5):
    """4 row strips (bench.py --gpus 4 layout: strip rows + 16-row read-only halo, global clamping)."""
    from paper_1501_02894_b200 import sharding

    px = c5["px"]
    H = px.shape[0]
    parts = []
    for rank in range(4):
        r0, r1 = sharding.strip_rows(H, 4, rank)
        y0, y1 = sharding.resident_rows(r0, r1, H)
        sl = torch.from_numpy(np.ascontiguousarray(px[y0:y1])).cuda()
        c = mns.encode_device(sl, mns.EncoderConfig(e3=math.inf), root_rows=(r0, r1), height=H)
        parts.append(c.records[: c.n_records()].cpu().numpy().view(np.uint64))
        del sl, c
    assert np.array_equal(np.concatenate(parts), c5["rec"])


def test_c3_all_256_images_bit_exact(mns):
    """The whole c3 batch (bench.py's images) in one batched launch vs the oracle image by image."""
    from paper_1501_02894_b200.synth import batch_seeds, synth_image

    seeds = batch_seeds()
    imgs = np.stack([synth_image(512, s, noise_sigma=6.0, n_blobs=6) for s in seeds])
    code = mns.encode_device(torch.from_numpy(imgs).cuda(), mns.EncoderConfig(e3=math.inf), root_level=2)
    n = code.n_records()
    rec = code.records[:n].cpu().numpy().view(np.uint64)
    offs = code.root_offsets.cpu().numpy()
    per = 32 * 32
    for i in range(len(seeds)):
        ref, _ = O.encode_quadtree_records(imgs[i], (8.0, 8.0, math.inf), 16.0, True, 2)
        assert np.array_equal(rec[offs[i * per]: offs[(i + 1) * per]], ref), seeds[i]


@pytest.mark.parametrize("n_iso", [1, 8])
def test_c4_full_search_all_ranges_vs_oracle(mns, n_iso):
    """All 4096 ranges x 247,009 stride-1 domains (x 8 isometries): the oracle's exact fp64 argmin."""
    from paper_1501_02894_b200.synth import config_image

    px = config_image("c4")
    res = {k: v.cpu().numpy() for k, v in mns.full_search_device(torch.from_numpy(px).cuda(), 8, 1, n_iso).items()}
    ref = O.full_search(px, 8, 1, n_iso=n_iso)
    for k in ("dom", "iso", "o", "code"):
        bad = np.flatnonzero(res[k].astype(np.int64) != ref[k].astype(np.int64))
        assert bad.size == 0, (n_iso, k, bad[:5])


@pytest.mark.parametrize("radius,n_iso", [(4, 1), (32, 1), (4, 8), (32, 8)])
@pytest.mark.parametrize("tensor_cores", [True, False])
def test_c4_local_search_all_ranges_vs_oracle(mns, radius, n_iso, tensor_cores):
    """All 4096 ranges, on the windowed tcgen05 GEMM and on the CUDA-core kernel; (32, 8) is config
    c4's +-32 x 8-isometry variant (1.38e8 pairs)."""
    from paper_1501_02894_b200.synth import config_image

    px = config_image("c4")
    res = {k: v.cpu().numpy() for k, v in
           mns.local_search_device(torch.from_numpy(px).cuda(), radius, n_iso=n_iso, tensor_cores=tensor_cores).items()}
    ref = O.local_search(px, radius, n_iso=n_iso)
    assert np.array_equal(res["dx"], ref["dom_x"]) and np.array_equal(res["dy"], ref["dom_y"])
    assert np.array_equal(res["iso"], ref["iso"])
    assert np.array_equal(res["o"], ref["o"]) and np.array_equal(res["code"], ref["code"])
