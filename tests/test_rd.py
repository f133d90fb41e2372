"""Rate-distortion sweep and offset histograms against the reference harness.

Golden rows come from the reference's own ``mnscodec.bench.rd_sweep`` / ``histogram_csv``
(oracle/gen_golden.py ``gen_rd``).  Bars: stream bits, leaf tallies and phase-2 counts
exact; PSNR within 0.01 dB (the decoder's bar); histogram CSV text identical.
"""
import math

import numpy as np
import pytest

from paper_1501_02894_b200 import rd
from paper_1501_02894_b200.types import DecodeConfig


# ---------------------------------------------------------------- host (no GPU)

def test_rd_csv_format():
    pts = [rd.RdPoint("no_search", (8.0, 8.0, 8.0), True, 1234, 1234 / 4096, math.inf, 0.01234, (16, 0, 0, 0), 0),
           rd.RdPoint("mns", (6.0, 8.0, 10.0), False, 99, 99 / 4096, 31.123456, 1.5, (1, 2, 3, 4), 5)]
    lines = rd.rd_csv(pts).strip().split("\n")
    assert lines[0] == ",".join(rd.RD_CSV_COLUMNS)
    assert lines[1] == "no_search,8,8,8,1,1234,0.301270,inf,0.0123,16,0,0,0,0"
    assert lines[2] == "mns,6,8,10,0,99,0.024170,31.1235,1.5000,1,2,3,4,5"


def test_rd_sweep_rejects_empty_grid():
    with pytest.raises(ValueError, match="at least one mode"):
        rd.rd_sweep(np.zeros((64, 64), np.uint8), [], [8.0])
    with pytest.raises(ValueError, match="at least one mode"):
        rd.rd_sweep(np.zeros((64, 64), np.uint8), ["mns"], [])


def test_offset_histogram_host():
    rng = np.random.default_rng(0)
    samples = [tuple(map(int, rng.integers(-20, 21, 2))) for _ in range(500)]
    h = rd.offset_histogram(samples)
    assert h.total == 500 and sum(h.joint.values()) == 500
    assert sum(h.marginal_x.values()) == 500 and sum(h.marginal_y.values()) == 500
    text = rd.histogram_csv(rd.offset_histogram([(1, -2), (1, -2), (0, 3)]))
    lines = text.strip().split("\n")
    assert lines[0] == "section,dx,dy,count"
    assert "x,0,,1" in lines and "x,1,,2" in lines and "joint,1,-2,2" in lines
    with pytest.raises(ValueError):
        rd.offset_histogram([])


# ---------------------------------------------------------------- device vs reference

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    return True


def _grid(g):
    return [tuple(e) if isinstance(e, list) else e for e in g]


@pytest.mark.gpu
def test_rd_sweep_matches_reference(cuda, golden):
    G = golden("rd")
    for case in G.manifest:
        if not case["key"].startswith("rd"):
            continue
        k = case["key"]
        dec = None if case["decode"] is None else DecodeConfig(*case["decode"])
        pts = rd.rd_sweep(G[f"{k}/img"], ["no_search", "mns"], _grid(case["grid"]), (True, False), decode_config=dec)
        assert [[p.mode, list(p.thresholds), p.technique2] for p in pts] == case["rows"]
        np.testing.assert_array_equal([p.bits for p in pts], G[f"{k}/bits"], err_msg=k)
        np.testing.assert_array_equal([p.leaf_counts for p in pts], G[f"{k}/leaves"], err_msg=k)
        np.testing.assert_array_equal([p.phase2_count for p in pts], G[f"{k}/phase2"], err_msg=k)
        for got, want in zip([p.psnr for p in pts], G[f"{k}/psnr"]):
            assert (math.isinf(got) and math.isinf(want)) or abs(got - want) <= 0.01, (k, got, want)
        assert all(p.bpp == p.bits / G[f"{k}/img"].size for p in pts)


@pytest.mark.gpu
def test_rd_sweep_wraps_point_failures(cuda):
    with pytest.raises(RuntimeError, match="sweep point failed"):
        rd.rd_sweep(np.full((64, 64), 42, np.uint8), ["full_search"], [8.0])


@pytest.mark.gpu
def test_offset_histogram_device_matches_reference_csv(cuda, golden):
    G = golden("rd")
    for case in G.manifest:
        if not case["key"].startswith("hist"):
            continue
        k = case["key"]
        h = rd.offset_histogram_device(G[f"{k}/img"], case["B"])
        assert rd.histogram_csv(h) == str(G[f"{k}/csv"]), k
        B, (ih, iw) = case["B"], G[f"{k}/img"].shape
        assert h.total == (-(-ih // B)) * (-(-iw // B))  # one sample per range of the B-padded image


@pytest.mark.gpu
def test_mse_psnr_match_float64_mean(cuda):
    """metrics.py:16-31: the GPU's exact SSE / n equals numpy's float64 mean of the squares."""
    import paper_1501_02894_b200 as mns

    rng = np.random.default_rng(3)
    for h, w in [(1, 1), (7, 13), (64, 64), (333, 517), (1024, 2048)]:
        a = rng.integers(0, 256, (h, w), dtype=np.uint8)
        b = np.clip(a.astype(int) + rng.integers(-9, 10, (h, w)), 0, 255).astype(np.uint8)
        d = a.astype(np.float64) - b.astype(np.float64)
        want = float(np.mean(d * d))
        assert mns.mse(mns.GrayImage(a), mns.GrayImage(b)) == want
        assert mns.psnr(a, b) == (math.inf if want == 0 else 10.0 * math.log10(255.0 * 255.0 / want))
    assert mns.psnr(a, a) == math.inf
    with pytest.raises(ValueError, match="image dimensions differ"):
        mns.mse(np.zeros((4, 4), np.uint8), np.zeros((4, 5), np.uint8))


def test_csv_writers_byte_identical_to_reference():
    """rd_csv / histogram_csv against the reference's own writers (baseline/_ref, when installed)."""
    import math
    import os
    import sys

    ref_dir = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "mnscodec")):
        pytest.skip("reference not installed (tools/install_reference.py)")
    sys.path.insert(0, ref_dir)
    try:
        import mnscodec.bench as RB
    finally:
        sys.path.remove(ref_dir)
    rng = np.random.default_rng(4)
    pts = [rd.RdPoint(mode=m, thresholds=(float(a), float(b), math.inf if i % 3 == 0 else 2.5), technique2=bool(i % 2),
                      bits=int(rng.integers(0, 10**7)), bpp=float(rng.random()), psnr=math.inf if i == 4 else 30 + rng.random(),
                      encode_seconds=float(rng.random()), leaf_counts=tuple(int(v) for v in rng.integers(0, 999, 4)),
                      phase2_count=int(rng.integers(0, 99)))
           for i, (m, a, b) in enumerate([("mns", 4, 8), ("no_search", 0.5, 12), ("mns", 1e-3, 7.25)] * 3)]
    assert rd.rd_csv(pts) == RB.rd_csv(pts)
    samples = [tuple(int(v) for v in rng.integers(-9, 10, 2)) for _ in range(500)]
    mine, theirs = rd.offset_histogram(samples), RB.offset_histogram(samples)
    assert rd.histogram_csv(mine) == RB.histogram_csv(theirs)
    assert (mine.mode_x(), mine.mode_y()) == (theirs.mode_x(), theirs.mode_y())
