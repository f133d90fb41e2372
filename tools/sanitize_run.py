"""Small invocations of every libmns_b200 kernel family, for compute-sanitizer (memcheck, racecheck,
synccheck): encode (+ split-stream compaction, batch, strips), try_node, every decoder (raster pair
/ single sweep / lattice / flat / units / fp64 exact + early stop / strip fp64), full search
(tcgen05 + CUDA-core paths, 1 and 8 isometries), local search, stream writer / reader, metrics.
Prints one line per family; exits non-zero on a mismatch with the oracle."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1501_02894_b200 as mns  # noqa: E402
from oracle import oracle as O  # noqa: E402  (checker)
from paper_1501_02894_b200 import bitstream, rd, sharding  # noqa: E402
from paper_1501_02894_b200.synth import synth_image  # noqa: E402

only = sys.argv[1] if len(sys.argv) > 1 else "all"
px = synth_image(96, 3, noise_sigma=10.0, n_blobs=4)
img = torch.from_numpy(px).cuda()


def done(name):
    torch.cuda.synchronize()
    print("ok", name, flush=True)


if only in ("all", "encode"):
    for e3, rl in ((math.inf, 1), (4.0, 1), (math.inf, 2)):
        code = mns.encode_quadtree(mns.GrayImage(px), mns.EncoderConfig(e1=6.0, e2=6.0, e3=e3), root_level=rl)
        ref, _ = O.encode_quadtree_records(px, (6.0, 6.0, e3), 16.0, True, rl)
        assert np.array_equal(code.records, ref)
    side = torch.cuda.Stream()
    c = mns.encode_device(img, mns.EncoderConfig(e3=math.inf), compact_stream=side)
    c.n_records()
    batch = torch.from_numpy(np.stack([px, px[::-1].copy()])).cuda()
    mns.encode_device(batch, mns.EncoderConfig(), root_level=2).n_records()
    mns.encode_device(torch.from_numpy(np.ascontiguousarray(px[16:80])).cuda(), mns.EncoderConfig(),
                      root_rows=(2, 4), height=96).n_records()
    mns.try_phase1(mns.GrayImage(px), mns.BlockRect(16, 16, 8), 2, mns.EncoderConfig())
    mns.try_phase2(mns.GrayImage(px), mns.BlockRect(16, 16, 8), 2, mns.EncoderConfig())
    done("encode")
if only in ("all", "decode"):
    rec, _ = O.encode_quadtree_records(px, (6.0, 6.0, 6.0), 16.0, True)
    code = mns.QuadtreeCode.from_records(rec, 96, 96, 96, 96, "mns", True)
    for cfg in (mns.DecodeConfig(max_iters=5, stop_delta=0.0), mns.DecodeConfig(max_iters=4, stop_delta=0.0),
                mns.DecodeConfig()):
        want, _, _ = O.decode_records(rec, 96, 96, max_iters=cfg.max_iters, stop_delta=cfg.stop_delta)
        got = mns.decode(code, cfg).pixels
        assert int(np.abs(got.astype(int) - want.astype(int)).max()) <= 1
    mns.decode_step(code, np.full((96, 96), 128.0))
    dc = mns.encode_device(img, mns.EncoderConfig(e3=math.inf))
    for it in (1, 2, 5, 6):
        mns.decode_device(dc, iters=it)
    dec = sharding.StripDecoder(dc, 96, 96, 0, 6, 0, 1, lattice=True)
    dec.run(6)
    dec = sharding.StripDecoder(mns.encode_device(img, mns.EncoderConfig()), 96, 96, 0, 6, 0, 1, lattice=False)
    dec.run(5)
    f64 = sharding.StripDecoderF64(mns.encode_device(img, mns.EncoderConfig()), 96, 96, 0, 6)
    f64.run(6, 1.0)
    done("decode")
if only in ("all", "search"):
    small = np.ascontiguousarray(px[:64, :64])
    for n_iso in (1, 8):
        res = mns.full_search_device(torch.from_numpy(small).cuda(), 8, 1, n_iso)
        ref = O.full_search(small, 8, 1, n_iso=n_iso)
        assert np.array_equal(res["dom"].cpu().numpy(), ref["dom"])
    os.environ["MNS_SEARCH_CUDA_CORES"] = "1"
    mns.full_search_device(torch.from_numpy(small).cuda(), 4, 2, 8)
    os.environ["MNS_SEARCH_CUDA_CORES"] = "0"
    mns.full_search_device(torch.from_numpy(small).cuda(), 4, 1, 1)
    for radius in (4, 32):
        mns.local_search_device(torch.from_numpy(small).cuda(), radius)
    done("search")
if only in ("all", "stream"):
    code = mns.encode_quadtree(mns.GrayImage(px), mns.EncoderConfig())
    data = bitstream.write_stream(code)
    back = bitstream.read_stream(data)
    assert np.array_equal(back.records, code.records)
    rd.mse(mns.GrayImage(px), mns.GrayImage(px[::-1].copy()))
    done("stream")
