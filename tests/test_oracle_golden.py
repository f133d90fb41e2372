"""Pin the CPU oracle (oracle/, test infrastructure) to the reference's own outputs.

Every fixture in tests/golden/ was produced by running the reference implementation
(/root/reference, pure Python) in the build container: oracle/gen_golden.py.
"""
import numpy as np
import pytest

from conftest import cfg_tuple
from oracle import oracle as O


def test_encode_records_match_reference(golden):
    g = golden("encode")
    for case in g.manifest:
        e, mean_tol, mns = cfg_tuple(case["cfg"])
        rec, counts = O.encode_quadtree_records(g[f"{case['key']}/img"], e, mean_tol, mns, case["root_level"])
        ref = g[f"{case['key']}/records"]
        assert np.array_equal(rec, ref), case
        assert counts.sum() == len(ref)


def test_decode_matches_reference(golden):
    g = golden("encode")
    for case in g.manifest[::3]:
        k = case["key"]
        img = g[f"{k}/img"]
        w, h = case["padded_w"], case["padded_h"]
        out8, _, it = O.decode_records(g[f"{k}/records"], w, h, max_iters=8, stop_delta=0.0)
        assert it == 8
        assert np.array_equal(out8[: img.shape[0], : img.shape[1]], g[f"{k}/decode8"]), case
        outd, _, _ = O.decode_records(g[f"{k}/records"], w, h)
        assert np.array_equal(outd[: img.shape[0], : img.shape[1]], g[f"{k}/decode_default"]), case


def test_decode_step_bit_exact(golden):
    g = golden("decode_step")
    for case in g.manifest:
        k = case["key"]
        units = O.records_to_units(g[f"{k}/records"], case["padded_w"], case["padded_h"])
        out = O.decode_step_units(units, g[f"{k}/raster_in"])
        assert np.array_equal(out, g[f"{k}/raster_out"])


def test_full_search_matches_reference(golden):
    g = golden("search")
    for case in g.manifest:
        if not case["key"].startswith("full"):
            continue
        k = case["key"]
        res = O.full_search(g[f"{k}/img"], case["B"], case["step"])
        dom = g[f"{k}/dom"]
        assert np.array_equal(res["dom_x"], dom[:, 0]) and np.array_equal(res["dom_y"], dom[:, 1]), case
        assert np.array_equal(res["o"], g[f"{k}/o"]) and np.array_equal(res["code"], g[f"{k}/code"]), case


def test_local_search_matches_reference(golden):
    g = golden("search")
    for case in g.manifest:
        if not case["key"].startswith("local"):
            continue
        k = case["key"]
        res = O.local_search(g[f"{k}/img"], 4)
        dom = g[f"{k}/dom"]
        assert np.array_equal(res["dom_x"], dom[:, 0]) and np.array_equal(res["dom_y"], dom[:, 1]), case
        assert np.array_equal(res["o"], g[f"{k}/o"]) and np.array_equal(res["code"], g[f"{k}/code"]), case


def test_single_node_phases(golden):
    g = golden("nodes")
    for case in g.manifest:
        k = case["key"]
        img = g[f"{k}/img"]
        e = (case["e"],) * 3
        rec_ref = g[f"{k}/rec"]
        rms_ref = g[f"{k}/rms"]
        if 2 * case["size"] <= min(img.shape):
            r1, rms1 = O.try_phase(1, img, case["x"], case["y"], case["size"], case["level"], e, case["mean_tol"])
            assert (r1 is not None) == case["ok1"] and (r1 or 0) == int(rec_ref[0])
            assert rms1 == rms_ref[0]
        if case["level"] <= 3:
            r2, rms2 = O.try_phase(2, img, case["x"], case["y"], case["size"], case["level"], e, case["mean_tol"])
            assert (r2 is not None) == case["ok2"] and (r2 or 0) == int(rec_ref[1])
            if r2 is not None:
                assert rms2 == rms_ref[1]


def test_tie_fixtures_contain_rounding_decided_picks(golden):
    g = golden("encode")
    ties = [c for c in g.manifest if c["image"].startswith("ties")]
    assert sum(c["exact_ties"] for c in ties) > 100
    assert sum(c["ties_bit1"] for c in ties) > 0


def test_oracle_stress_golden(golden):
    """The oracle restatement against the reference on adversarial images (gen_stress)."""
    import math

    g = golden("stress")
    for case in g.manifest:
        c = case["cfg"]
        e = tuple(math.inf if c[n] is None else c[n] for n in ("e1", "e2", "e3"))
        rec, _ = O.encode_quadtree_records(g[f"img/{case['image']}"], e, c["mean_tol"], c["mode"] == "mns")
        assert np.array_equal(rec, g[f"{case['key']}/records"]), case
