"""Multi-GPU decomposition logic on CPU: world-size-2 gloo process groups.

* exchange_halos moves the right 16-row halos between neighbouring strips;
* a strip-wise Jacobi decode (each rank paints only its own units from a raster
  that holds ONLY its resident rows -- everything else is NaN-poisoned -- and
  exchanges halos after every sweep) reproduces the whole-image decode exactly,
  proving the 16-row halo suffices for every clamped domain (the GPU path runs
  the same split with NCCL).
"""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1501_02894_b200 import sharding


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _run(world, fn, *args):
    port = _free_port()
    mp.spawn(_entry, args=(world, port, fn, args), nprocs=world, join=True)


def _entry(rank, world, port, fn, args):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fn(rank, world, *args)
    finally:
        dist.destroy_process_group()


def test_split_covers_rows():
    for H in (16, 64, 512, 16384):
        for world in (1, 2, 3, 4, 8):
            rows = [sharding.strip_rows(H, world, r) for r in range(world)]
            assert rows[0][0] == 0 and rows[-1][1] == H // 16
            assert all(a[1] == b[0] for a, b in zip(rows, rows[1:]))
            for r0, r1 in rows:
                y_lo, y_hi = sharding.resident_rows(r0, r1, H)
                assert y_lo == max(0, 16 * r0 - 16) and y_hi == min(H, 16 * r1 + 16)


def _halo_worker(rank, world, H, W, halo):
    r0, r1 = sharding.strip_rows(H, world, rank)
    y_lo, y_hi = sharding.resident_rows(r0, r1, H, halo)
    rows = torch.arange(y_lo, y_hi, dtype=torch.float32)[:, None].repeat(1, W)
    raster = rows.clone()
    own0, own1 = 16 * r0 - y_lo, 16 * r1 - y_lo
    raster[:own0] = -1.0
    raster[own1:] = -1.0
    sharding.exchange_halos(raster, r0, r1, H, rank, world, halo=halo)
    assert torch.equal(raster, rows), f"rank {rank}: halo rows not exchanged"


@pytest.mark.parametrize("world,halo", [(2, 16), (3, 16), (2, 32), (3, 32)])
def test_exchange_halos_gloo(world, halo):
    _run(world, _halo_worker, 128, 48, halo)


def _lattice_halo_worker(rank, world, H, W):
    # lattice-state decoding: one lattice row per two raster rows, DEC_HALO / 2 rows exchanged
    r0, r1 = sharding.strip_rows(H, world, rank)
    y_lo, y_hi = sharding.resident_rows(r0, r1, H, sharding.DEC_HALO)
    rows = torch.arange(y_lo // 2, y_hi // 2, dtype=torch.float32)[:, None].repeat(1, W // 2)
    lat = rows.clone()
    own0, own1 = (16 * r0 - y_lo) // 2, (16 * r1 - y_lo) // 2
    lat[:own0] = -1.0
    lat[own1:] = -1.0
    sharding.exchange_halos(lat, r0, r1, H, rank, world, halo=sharding.DEC_HALO, row_div=2)
    assert torch.equal(lat, rows), f"rank {rank}: lattice halo rows not exchanged"


@pytest.mark.parametrize("world", [2, 3])
def test_exchange_lattice_halos_gloo(world):
    _run(world, _lattice_halo_worker, 160, 48)


def _umap_worker(rank, world, H, rw32):
    r0, r1 = sharding.strip_rows(H, world, rank)
    u0, u1 = sharding.unit_map_rows(r0, r1, H)
    want = torch.arange(u0, u1, dtype=torch.int32)[:, None].repeat(1, rw32)
    umap = want.clone()
    umap[: r0 - u0] = -1
    umap[r1 - u0:] = -1
    sharding.exchange_unit_map_rows(umap, r0, r1, H, rank, world)
    assert torch.equal(umap, want), f"rank {rank}: unit-map halo rows not exchanged"


@pytest.mark.parametrize("world", [2, 3])
def test_exchange_unit_map_rows_gloo(world):
    _run(world, _umap_worker, 160, 64)


def _strip_decode_worker(rank, world, px, records, iters, out_dir):
    from oracle import oracle as O

    H, W = px.shape
    r0, r1 = sharding.strip_rows(H, world, rank)
    y_lo, y_hi = sharding.resident_rows(r0, r1, H)
    units = O.records_to_units(records, W, H)
    mine = units[(units["y"] >= 16 * r0) & (units["y"] < 16 * r1)]
    local = torch.full((y_hi - y_lo, W), 128.0, dtype=torch.float64)
    for it in range(iters):
        full = np.full((H, W), np.nan)  # anything outside the resident rows is poison
        full[y_lo:y_hi] = local.numpy()
        nxt = O.decode_step_units(mine, full, nthreads=1)
        local[16 * r0 - y_lo: 16 * r1 - y_lo] = torch.from_numpy(nxt[16 * r0: 16 * r1])
        sharding.exchange_halos(local, r0, r1, H, rank, world)
    own = local[16 * r0 - y_lo: 16 * r1 - y_lo].numpy()
    assert np.isfinite(own).all()
    np.save(os.path.join(out_dir, f"strip{rank}.npy"), own)


@pytest.mark.parametrize("world", [2, 4])
def test_strip_decode_matches_whole_image(world, tmp_path):
    from oracle import oracle as O
    from paper_1501_02894_b200.synth import synth_image

    px = synth_image(128, 21, noise_sigma=10.0, n_blobs=6)
    records, _ = O.encode_quadtree_records(px, (8.0, 8.0, 8.0), 16.0, True)
    iters = 6
    _run(world, _strip_decode_worker, px, records, iters, str(tmp_path))
    _, whole, _ = O.decode_records(records, 128, 128, max_iters=iters, stop_delta=0.0)
    strips = np.concatenate([np.load(tmp_path / f"strip{r}.npy") for r in range(world)])
    assert np.array_equal(strips, whole)


def _pair_decode_worker(rank, world, px, records, iters, out_dir):
    """Two sweeps per pass like mns_decode_sweep2: sweep A over the strip +- one root row (units
    of the neighbour rows come from the unit-map halo), sweep B over the strip, then the 32-row
    raster halo exchange.  Everything outside the resident rows is NaN poison."""
    from oracle import oracle as O

    H, W = px.shape
    r0, r1 = sharding.strip_rows(H, world, rank)
    y_lo, y_hi = sharding.resident_rows(r0, r1, H, sharding.DEC_HALO)
    u0, u1 = sharding.unit_map_rows(r0, r1, H)
    units = O.records_to_units(records, W, H)
    wide = units[(units["y"] >= 16 * u0) & (units["y"] < 16 * u1)]
    mine = units[(units["y"] >= 16 * r0) & (units["y"] < 16 * r1)]
    local = torch.full((y_hi - y_lo, W), 128.0, dtype=torch.float64)
    for _ in range(iters // 2):
        full = np.full((H, W), np.nan)
        full[y_lo:y_hi] = local.numpy()
        mid = O.decode_step_units(wide, full, nthreads=1)
        keep = np.full((H, W), np.nan)
        keep[16 * u0: 16 * u1] = mid[16 * u0: 16 * u1]
        nxt = O.decode_step_units(mine, keep, nthreads=1)
        local[16 * r0 - y_lo: 16 * r1 - y_lo] = torch.from_numpy(nxt[16 * r0: 16 * r1])
        sharding.exchange_halos(local, r0, r1, H, rank, world, halo=sharding.DEC_HALO)
    own = local[16 * r0 - y_lo: 16 * r1 - y_lo].numpy()
    assert np.isfinite(own).all()
    np.save(os.path.join(out_dir, f"strip{rank}.npy"), own)


@pytest.mark.parametrize("world", [2, 3])
def test_pair_pass_strip_decode_matches_whole_image(world, tmp_path):
    from oracle import oracle as O
    from paper_1501_02894_b200.synth import synth_image

    px = synth_image(128, 23, noise_sigma=10.0, n_blobs=6)
    records, _ = O.encode_quadtree_records(px, (8.0, 8.0, 8.0), 16.0, True)
    iters = 6
    _run(world, _pair_decode_worker, px, records, iters, str(tmp_path))
    _, whole, _ = O.decode_records(records, 128, 128, max_iters=iters, stop_delta=0.0)
    strips = np.concatenate([np.load(tmp_path / f"strip{r}.npy") for r in range(world)])
    assert np.array_equal(strips, whole)


def _lattice_decode_worker(rank, world, px, records, iters, out_dir):
    """Lattice-state strip decode (StripDecoder with min_leaf 4): the carried state is the 2x2-sum
    lattice of the resident rows; each pass expands it to a raster whose lattice it is (in fp64,
    l/4 in each of the four pixels sums back to l exactly), runs the two oracle sweeps, keeps the
    lattice of the own rows and exchanges 16 lattice halo rows.  NaN poison outside the halo."""
    from oracle import oracle as O

    H, W = px.shape
    r0, r1 = sharding.strip_rows(H, world, rank)
    y_lo, y_hi = sharding.resident_rows(r0, r1, H, sharding.DEC_HALO)
    u0, u1 = sharding.unit_map_rows(r0, r1, H)
    units = O.records_to_units(records, W, H)
    wide = units[(units["y"] >= 16 * u0) & (units["y"] < 16 * u1)]
    mine = units[(units["y"] >= 16 * r0) & (units["y"] < 16 * r1)]
    lat = torch.full(((y_hi - y_lo) // 2, W // 2), 4 * 128.0, dtype=torch.float64)
    own = None
    for p in range(iters // 2):
        full = np.full((H, W), np.nan)
        full[y_lo:y_hi] = np.repeat(np.repeat(lat.numpy() / 4, 2, axis=0), 2, axis=1)
        mid = O.decode_step_units(wide, full, nthreads=1)
        keep = np.full((H, W), np.nan)
        keep[16 * u0: 16 * u1] = mid[16 * u0: 16 * u1]
        nxt = O.decode_step_units(mine, keep, nthreads=1)
        own = nxt[16 * r0: 16 * r1]
        q = ((own[0::2, 0::2] + own[0::2, 1::2]) + own[1::2, 0::2]) + own[1::2, 1::2]
        lat[(16 * r0 - y_lo) // 2: (16 * r1 - y_lo) // 2] = torch.from_numpy(q)
        if p + 1 < iters // 2:
            sharding.exchange_halos(lat, r0, r1, H, rank, world, halo=sharding.DEC_HALO, row_div=2)
    assert np.isfinite(own).all()
    np.save(os.path.join(out_dir, f"strip{rank}.npy"), own)


@pytest.mark.parametrize("world", [2, 3])
def test_lattice_strip_decode_matches_whole_image(world, tmp_path):
    from oracle import oracle as O
    from paper_1501_02894_b200.synth import synth_image

    px = synth_image(128, 29, noise_sigma=10.0, n_blobs=6)
    records, _ = O.encode_quadtree_records(px, (8.0, 8.0, float("inf")), 16.0, True)
    iters = 6
    _run(world, _lattice_decode_worker, px, records, iters, str(tmp_path))
    _, whole, _ = O.decode_records(records, 128, 128, max_iters=iters, stop_delta=0.0)
    strips = np.concatenate([np.load(tmp_path / f"strip{r}.npy") for r in range(world)])
    assert np.array_equal(strips, whole)


def _gather_worker(rank, world, out_dir):  # noqa: ARG001
    counts = [5, 0, 9, 3][:world]
    n_roots = [2, 1, 3, 2][:world]
    base = 1000 * rank
    rec = torch.arange(base, base + counts[rank] + 4, dtype=torch.int64)  # 4 junk slots past count
    offs = torch.tensor(sorted(np.random.default_rng(rank).integers(0, counts[rank] + 1, n_roots[rank]).tolist())
                        + [counts[rank]], dtype=torch.int32)
    offs[0] = 0
    got = sharding.gather_codes(rec, counts[rank], offs, rank, world)
    if rank != 0:
        assert got is None
        return
    out, o = got
    want = np.concatenate([np.arange(1000 * r, 1000 * r + counts[r]) for r in range(world)])
    assert np.array_equal(out.numpy(), want)
    want_o = []
    for r in range(world):  # each rank's strip-local offsets, rebased by the records before it
        lo = sorted(np.random.default_rng(r).integers(0, counts[r] + 1, n_roots[r]).tolist())
        lo[0] = 0
        want_o += [v + sum(counts[:r]) for v in lo]
    assert o.numpy().tolist() == want_o + [sum(counts)]


@pytest.mark.parametrize("world", [2, 3])
def test_gather_codes_gloo(world, tmp_path):
    _run(world, _gather_worker, str(tmp_path))


def test_batch_and_range_splits():
    for n, world in ((256, 1), (256, 8), (4096, 3), (7, 4)):
        parts = [sharding.split(n, world, r) for r in range(world)]
        assert sum(b - a for a, b in parts) == n
        assert max(b - a for a, b in parts) - min(b - a for a, b in parts) <= 1
    assert math.isclose(sum(b - a for a, b in [sharding.split(4096, 8, r) for r in range(8)]) / 8, 512)


class _OracleStripF64(sharding.StripDecoderF64):
    """StripDecoderF64 with its two device kernels replaced by the fp64 oracle (same contract:
    the sweep paints this rank's units and folds its max|delta| into state[2]; decide applies the
    reference's test), so the rank-level control -- delta all-reduce, device-side stop, halo
    exchange, final rows -- runs here on gloo.  Rows outside the resident strip are NaN poison."""

    def __init__(self, px, records, rank, world):
        from oracle import oracle as O

        H, W = px.shape
        r0, r1 = sharding.strip_rows(H, world, rank)
        super().__init__(None, H, W, r0, r1, rank, world)
        units = O.records_to_units(records, W, H)
        self.mine = units[(units["y"] >= 16 * r0) & (units["y"] < 16 * r1)]
        self.units = {"n": len(self.mine)}
        self.swept = 0

    def sweep(self, cur, nxt, stream=None):
        from oracle import oracle as O

        if self.state[0]:
            return
        full = np.full((self.H, self.W), np.nan)
        full[self.y_lo:self.y_hi] = cur.numpy()
        res = O.decode_step_units(self.mine, full, nthreads=1)
        a, b = 16 * self.r0, 16 * self.r1
        nxt[a - self.y_lo: b - self.y_lo] = torch.from_numpy(res[a:b])
        d = float(np.max(np.abs(res[a:b] - full[a:b])))
        self.delta_view()[0] = max(float(self.delta_view()[0]), d)
        self.swept += 1

    def decide(self, stop_delta, stream=None):
        if self.state[0]:
            return
        self.state[1] += 1
        if float(self.delta_view()[0]) < stop_delta:
            self.state[0] = 1
        self.state[2] = 0

    def finalize(self, stream=None):
        src = self.pong if int(self.state[1]) & 1 else self.ping
        own = src[16 * self.r0 - self.y_lo: 16 * self.r1 - self.y_lo].numpy()
        return np.clip(np.floor(own + 0.5), 0, 255).astype(np.uint8)


def _f64_strip_worker(rank, world, px, records, iters, stop, out_dir):
    dec = _OracleStripF64(px, records, rank, world)
    out = dec.run(iters, stop, 128.0)
    np.save(os.path.join(out_dir, f"strip{rank}.npy"), out)
    np.save(os.path.join(out_dir, f"iters{rank}.npy"), np.array([int(dec.state[1]), dec.swept]))


@pytest.mark.parametrize("world,stop", [(2, 0.5), (3, 0.5), (2, 2.0), (3, 0.0)])
def test_f64_strip_decode_early_stop_matches_whole_image(world, stop, tmp_path):
    """Early stop across strips (decoder.py:70-75): the all-reduced max|delta| makes every rank stop
    after the reference's sweep, and the strips equal the whole-image decode bit for bit."""
    from oracle import oracle as O
    from paper_1501_02894_b200.synth import synth_image

    px = synth_image(96, 31, noise_sigma=10.0, n_blobs=5)
    records, _ = O.encode_quadtree_records(px, (8.0, 8.0, 8.0), 16.0, True)
    _run(world, _f64_strip_worker, px, records, 12, stop, str(tmp_path))
    want, _, sweeps = O.decode_records(records, 96, 96, max_iters=12, stop_delta=stop)
    strips = np.concatenate([np.load(tmp_path / f"strip{r}.npy") for r in range(world)])
    assert np.array_equal(strips, want)
    for r in range(world):
        done, swept = np.load(tmp_path / f"iters{r}.npy")
        assert done == sweeps and swept == sweeps
    assert stop == 0.0 or sweeps < 12  # the stop actually triggered


def _search_worker(rank, world, px, kind, out_dir):
    """Config c4's range split: every rank searches its share of the ranges (the oracle stands in
    for the GPU search on CPU) and search_sharded all-gathers the packed per-range results."""
    from oracle import oracle as O

    B = 8
    n_ranges = (px.shape[0] // B) * (px.shape[1] // B)

    def search_fn(r0, r1):
        if kind == "full":
            res = O.full_search(px, B, 1, n_iso=8, range_ids=np.arange(r0, r1), nthreads=1)
            return {k: torch.from_numpy(np.ascontiguousarray(res[k])) for k in ("dom", "iso", "o", "code")}
        res = O.local_search(px, 4, nthreads=1, n_iso=8)
        ndx = px.shape[1] - 16 + 1
        dom = (res["dom_y"] * ndx + res["dom_x"]).astype(np.int32)
        return {"dom": torch.from_numpy(dom[r0:r1]), "iso": torch.from_numpy(res["iso"][r0:r1]),
                "o": torch.from_numpy(res["o"][r0:r1]), "code": torch.from_numpy(res["code"][r0:r1])}

    got = sharding.search_sharded(search_fn, n_ranges, rank, world)
    np.save(os.path.join(out_dir, f"search{rank}.npy"),
            np.stack([got[k].numpy().astype(np.int64) for k in ("dom", "iso", "o", "code")]))


@pytest.mark.parametrize("world,kind", [(2, "full"), (3, "full"), (3, "local")])
def test_search_range_split_gloo(world, kind, tmp_path):
    from oracle import oracle as O
    from paper_1501_02894_b200.synth import synth_image

    px = synth_image(64, 17, noise_sigma=8.0, n_blobs=3)
    _run(world, _search_worker, px, kind, str(tmp_path))
    if kind == "full":
        ref = O.full_search(px, 8, 1, n_iso=8)
        want = np.stack([ref[k].astype(np.int64) for k in ("dom", "iso", "o", "code")])
    else:
        ref = O.local_search(px, 4, n_iso=8)
        want = np.stack([(ref["dom_y"] * 49 + ref["dom_x"]).astype(np.int64), ref["iso"].astype(np.int64),
                         ref["o"].astype(np.int64), ref["code"].astype(np.int64)])
    for r in range(world):  # every rank holds the whole result
        assert np.array_equal(np.load(tmp_path / f"search{r}.npy"), want)


def _gather_tensor_count_worker(rank, world, out_dir):  # noqa: ARG001
    counts = [7, 3, 0][:world]
    rec = torch.arange(100 * rank, 100 * rank + counts[rank] + 5, dtype=torch.int64)
    offs = torch.tensor([0, counts[rank]], dtype=torch.int32)
    got = sharding.gather_codes(rec, torch.tensor([counts[rank]], dtype=torch.int64), offs, rank, world)
    if rank == 0:
        out, o = got
        want = np.concatenate([np.arange(100 * r, 100 * r + counts[r]) for r in range(world)])
        assert np.array_equal(out.numpy(), want)
        assert o.numpy().tolist()[-1] == sum(counts)


@pytest.mark.parametrize("world", [2, 3])
def test_gather_codes_device_count_gloo(world, tmp_path):
    _run(world, _gather_tensor_count_worker, str(tmp_path))
