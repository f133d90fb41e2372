"""CPU-only checks: the C-ABI library loads and exports every declared symbol, the
host-side mirror (types, geometry, bitstream accounting/parser) matches the
reference's goldens, and the product path refuses to run without a GPU."""
import math
import os
import re

import numpy as np
import pytest

from conftest import ROOT

import paper_1501_02894_b200 as mns
from paper_1501_02894_b200 import _native, bitstream


def test_library_exports_every_declared_symbol():
    lib = _native.load_library()
    header = open(os.path.join(ROOT, "include", "mns_b200.h")).read()
    declared = set(re.findall(r"\b(mns_[a-z0-9_]+)\s*\(", header))
    assert declared == set(_native.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name


def test_library_built_for_sm100a():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(_native.NativeError):
        mns.encode_quadtree(mns.GrayImage(np.zeros((32, 32), np.uint8)), mns.EncoderConfig())


def test_config_validation_messages():
    with pytest.raises(ValueError, match="unknown mode"):
        mns.EncoderConfig(mode="turbo")
    with pytest.raises(ValueError, match="thresholds"):
        mns.EncoderConfig(e2=0.0)
    with pytest.raises(ValueError, match="full_search_step"):
        mns.EncoderConfig(full_search_step=0)
    with pytest.raises(ValueError, match="max_iters"):
        mns.DecodeConfig(max_iters=0)
    with pytest.raises(ValueError, match="no_search/mns"):
        mns.encode_quadtree(np.zeros((16, 16), np.uint8), mns.EncoderConfig(mode="full_search"))
    with pytest.raises(ValueError, match="range size must be one of"):
        mns.encode_full_search(np.zeros((64, 64), np.uint8), 3, mns.EncoderConfig())
    with pytest.raises(ValueError, match="too small"):
        mns.encode_full_search(np.zeros((12, 12), np.uint8), 8, mns.EncoderConfig())
    with pytest.raises(ValueError, match="16x16"):
        mns.encode_local_search(np.zeros((8, 20), np.uint8), mns.EncoderConfig())


def test_geometry_helpers():
    assert mns.co_domain_rect(mns.BlockRect(0, 0, 16), 64, 64) == mns.BlockRect(0, 0, 32)
    assert mns.co_domain_rect(mns.BlockRect(48, 16, 16), 64, 64) == mns.BlockRect(32, 8, 32)
    assert mns.co_domain_rect(mns.BlockRect(6, 6, 2), 64, 64) == mns.BlockRect(5, 5, 4)
    p = mns.pad_to_multiple(mns.GrayImage(np.arange(10 * 10, dtype=np.uint8).reshape(10, 10)), 16)
    assert (p.width, p.height) == (16, 16) and np.array_equal(p.pixels[15], p.pixels[9])


def test_record_roundtrip_and_counts(golden):
    g = golden("encode")
    for case in g.manifest[:20]:
        rec = g[f"{case['key']}/records"]
        code = mns.QuadtreeCode.from_records(rec, case["padded_w"], case["padded_h"], 1, 1, case["cfg"]["mode"], True)
        again = mns.QuadtreeCode(code.leaves, case["padded_w"], case["padded_h"], 1, 1, case["cfg"]["mode"], True)
        assert np.array_equal(again.records, rec)
        assert sum(code.level_counts()) == len(rec) == case["leaves"]
        assert code.phase2_count() == case["phase2"]


def test_stream_accounting_and_parser_match_reference(golden):
    g = golden("encode")
    for case in g.manifest:
        k = case["key"]
        img = g[f"{k}/img"]
        code = mns.QuadtreeCode.from_records(g[f"{k}/records"], case["padded_w"], case["padded_h"], img.shape[1],
                                             img.shape[0], case["cfg"]["mode"], True)
        assert bitstream.stream_bit_count(code) == int(g[f"{k}/stream_bits"])
        back = bitstream.read_stream_host(bytes(g[f"{k}/stream"]))
        assert np.array_equal(back.records, g[f"{k}/records"])
        assert (back.orig_w, back.orig_h, back.padded_w, back.padded_h) == (img.shape[1], img.shape[0],
                                                                            case["padded_w"], case["padded_h"])


def test_stream_errors():
    with pytest.raises(bitstream.StreamFormatError, match="truncated header"):
        bitstream.read_stream(b"MNS1")
    with pytest.raises(bitstream.StreamFormatError, match="bad magic"):
        bitstream.read_stream(b"XXXX" + bytes(9))
    bad = mns.QuadtreeCode((mns.LeafRecord(mns.BlockRect(0, 0, 16), 1, mns.Phase1Payload(300, 1)),), 16, 16, 16, 16,
                           "mns", True)
    with pytest.raises(ValueError, match="luminance byte 300"):
        bitstream._validate_tiling(bad.leaves, 16, 16, "mns")
    with pytest.raises(ValueError, match="only no_search/mns"):
        bitstream._check_header(mns.QuadtreeCode((), 16, 16, 16, 16, "full_search", False))


def test_sqrt_bound_semantics():
    # the phase-1 integer acceptance rule depends on bound(E) = max{x : sqrt(x) <= E}
    for E in (8.0, 6.3, 2.2, 0.5, 1e-3, 1.7976931348623157e154):
        x = E * E
        while math.sqrt(x) > E:
            x = math.nextafter(x, 0.0)
        while math.sqrt(math.nextafter(x, math.inf)) <= E:
            x = math.nextafter(x, math.inf)
        assert math.sqrt(x) <= E < math.sqrt(math.nextafter(x, math.inf))


def test_integration_listing_matches_binding():
    """INTEGRATION.md's ctypes listing (what a maintainer would paste into mnscodec) declares every
    exported entry point with the same argument types as paper_1501_02894_b200/_native.py."""
    import os
    import re

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    integ = open(os.path.join(root, "INTEGRATION.md")).read()
    nat = open(os.path.join(root, "paper_1501_02894_b200", "_native.py")).read()
    sig = dict(re.findall(r'"(mns_\w+)": (\[.*?\]),', nat, re.S))
    doc = dict(re.findall(r"L\.(mns_\w+)\.argtypes = (\[.*?\])", integ, re.S))

    def norm(x):
        return re.sub(r"\s+", "", x)

    assert sig, "no signatures parsed from _native.py"
    assert not [k for k, v in doc.items() if k not in sig or norm(v) != norm(sig[k])]
    assert not [k for k in sig if k not in doc and k != "mns_version"]
