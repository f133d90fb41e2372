"""GPU .mns reader (bitstream.py:208-279 read_stream).

* the reference-written golden streams parse to the golden records;
* write -> read round trips for Technique 2 on/off and no_search codes, up to a 4096^2 image
  (thousands of speculative chunks, resync rounds);
* a mutation fuzz (bit flips, truncations, appended bytes, byte rewrites) against the sequential
  host parser (the reference's algorithm): both accept with identical records, or both raise
  StreamFormatError with the identical message (the GPU reports the first error in stream order).
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mns():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1501_02894_b200 as m

    return m


def _outcome(fn, blob):
    from paper_1501_02894_b200 import bitstream

    try:
        code = fn(blob)
    except bitstream.StreamFormatError as e:
        return ("error", str(e))
    return ("ok", code.mode, code.technique2, code.orig_w, code.orig_h, code.padded_w, code.padded_h,
            np.asarray(code.records).tobytes())


def test_golden_streams_parse_to_golden_records(mns, golden):
    from paper_1501_02894_b200 import bitstream

    g = golden("encode")
    for case in g.manifest:
        k = case["key"]
        back = bitstream.read_stream(bytes(g[f"{k}/stream"]))
        assert np.array_equal(back.records, g[f"{k}/records"]), k
        img = g[f"{k}/img"]
        assert (back.orig_w, back.orig_h, back.padded_w, back.padded_h) == (img.shape[1], img.shape[0],
                                                                            case["padded_w"], case["padded_h"])


@pytest.mark.parametrize("side,mode,t2", [(64, "mns", True), (64, "mns", False), (256, "no_search", True),
                                          (512, "mns", False), (4096, "mns", True)])
def test_round_trip(mns, side, mode, t2):
    from paper_1501_02894_b200 import bitstream
    from paper_1501_02894_b200.synth import synth_image

    px = synth_image(side, 40 + side, noise_sigma=10.0, n_blobs=8)
    code = mns.encode_quadtree(mns.GrayImage(px), mns.EncoderConfig(e1=6.0, e2=7.0, e3=8.0, mode=mode,
                                                                    technique2=t2))
    blob = bitstream.write_stream(code)
    back = bitstream.read_stream(blob)
    assert np.array_equal(back.records, code.records)
    assert (back.mode, back.technique2) == (mode, t2)
    if side <= 512:
        assert _outcome(bitstream.read_stream, blob) == _outcome(bitstream.read_stream_host, blob)


def test_mutation_fuzz_matches_sequential_parser(mns, golden):
    from paper_1501_02894_b200 import bitstream

    g = golden("encode")
    rng = np.random.default_rng(17)
    keys = [c["key"] for c in g.manifest][::7]
    n_err = n_ok = 0
    for k in keys:
        base = bytearray(bytes(g[f"{k}/stream"]))
        for trial in range(12):
            blob = bytearray(base)
            kind = trial % 4
            if kind == 0:  # flip 1..3 body bits
                for _ in range(int(rng.integers(1, 4))):
                    pos = int(rng.integers(13 * 8, len(blob) * 8))
                    blob[pos >> 3] ^= 0x80 >> (pos & 7)
            elif kind == 1:  # truncate
                blob = blob[: int(rng.integers(13, len(blob)))]
            elif kind == 2:  # append bytes
                blob += bytes(rng.integers(0, 256, int(rng.integers(1, 4)), dtype=np.uint8))
            else:  # rewrite one body byte
                blob[int(rng.integers(13, len(blob)))] = int(rng.integers(0, 256))
            got, want = _outcome(bitstream.read_stream, bytes(blob)), _outcome(bitstream.read_stream_host, bytes(blob))
            assert got == want, (k, trial, got[:2], want[:2])
            n_err += got[0] == "error"
            n_ok += got[0] == "ok"
    assert n_err > 50  # the fuzz exercises the error paths


def test_error_messages(mns):
    from paper_1501_02894_b200 import bitstream

    code = mns.encode_quadtree(mns.GrayImage(np.full((32, 32), 9, np.uint8)), mns.EncoderConfig())
    blob = bytearray(bitstream.write_stream(code))
    with pytest.raises(bitstream.StreamFormatError, match="trailing bits"):
        bitstream.read_stream(bytes(blob) + b"\x00\x00")
    with pytest.raises(bitstream.StreamFormatError, match="truncated stream"):
        bitstream.read_stream(bytes(blob[:-1]))
