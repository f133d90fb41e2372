"""Multi-GPU decomposition of the MNS hot path (one process per GPU, torch.distributed).

SURVEY 8(e):
* batches of images (config c3)  -- images split across ranks, no data-path collective;
* one huge image (config c5)     -- row strips of whole root rows; every strip reads a
  16-row read-only halo of the input (all clamped domains of a root lie within 16 rows
  of it) and uses GLOBAL coordinates for clamping, so encode needs no exchange;
  the Jacobi decode runs two sweeps per pass, so it keeps a 32-row raster halo and
  exchanges the 32 boundary rows with the up/down neighbours after every pass (NCCL
  send/recv over NVLink; gloo in the CPU tests), plus one unit-map root row per side
  once per code;
* full / local search (config c4) -- ranges split across ranks, pool replicated.
Codes stay on the rank that produced them (root_offsets are strip-local);
gather_codes concatenates them on rank 0 in strip (= root raster) order: one
all_gather of the sizes, then point-to-point sends of each rank's records and
root offsets straight into their slices of rank 0's buffers.
"""

from __future__ import annotations

import ctypes

HALO = 16      # rows: every co-centred domain of a 16x16 root lies within 16 rows of it
DEC_HALO = 32  # decode rasters: two sweeps per pass need the halo of the halo


def split(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous near-equal split of n items: [begin, end) of `rank`."""
    return n * rank // world, n * (rank + 1) // world


def strip_rows(height: int, world: int, rank: int) -> tuple[int, int]:
    """Root rows [r0, r1) of this rank's strip of a height-pixel image."""
    return split(height // 16, world, rank)


def resident_rows(r0: int, r1: int, height: int, halo: int = HALO) -> tuple[int, int]:
    """Pixel rows [y_lo, y_hi) a strip needs resident (its rows plus the halo, clipped)."""
    return max(0, 16 * r0 - halo), min(height, 16 * r1 + halo)


def halo_ops(raster, r0: int, r1: int, height: int, rank: int, world: int, group=None, halo: int = HALO,
             row_div: int = 1) -> list:
    """The point-to-point operations of one halo exchange (see exchange_halos); reusable as long as
    ``raster`` is the same tensor."""
    import torch.distributed as dist

    if world == 1:
        return []
    if 16 * (r1 - r0) < halo:
        raise ValueError(f"strip of {16 * (r1 - r0)} rows is thinner than the {halo}-row halo")
    y_lo, y_hi = resident_rows(r0, r1, height, halo)
    own0, own1, hl = (16 * r0 - y_lo) // row_div, (16 * r1 - y_lo) // row_div, halo // row_div
    ops = []
    if rank > 0:
        ops.append(dist.P2POp(dist.isend, raster[own0: own0 + hl], rank - 1, group))
        ops.append(dist.P2POp(dist.irecv, raster[own0 - hl: own0], rank - 1, group))
    if rank < world - 1:
        ops.append(dist.P2POp(dist.isend, raster[own1 - hl: own1], rank + 1, group))
        ops.append(dist.P2POp(dist.irecv, raster[own1: own1 + hl], rank + 1, group))
    return ops


def run_ops(ops) -> None:
    """Issue a batch of point-to-point operations and wait for them (stream-ordered on NCCL)."""
    import torch.distributed as dist

    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()


def exchange_halos(raster, r0: int, r1: int, height: int, rank: int, world: int, group=None,
                   halo: int = HALO, row_div: int = 1) -> None:
    """After a sweep: send my first/last `halo` own rows to the neighbours, receive theirs into my halos.

    ``raster`` holds rows [y_lo, y_hi) (resident_rows with the same halo) of the full image, or with
    row_div = 2 the lattice rows [y_lo/2, y_hi/2) of lattice-state decoding (one lattice row per two
    raster rows; halo/2 rows exchanged).  Works for any torch.distributed backend (NCCL on GPUs,
    gloo on CPU).
    """
    run_ops(halo_ops(raster, r0, r1, height, rank, world, group, halo, row_div))


def unit_map_rows(r0: int, r1: int, height: int) -> tuple[int, int]:
    """Root rows [u0, u1) of a strip's decoder unit map: its own rows plus one on each side."""
    return max(0, r0 - 1), min(height // 16, r1 + 1)


def unit_map_ops(umap, r0: int, r1: int, height: int, rank: int, world: int, group=None) -> list:
    """The point-to-point operations of exchange_unit_map_rows (reusable for the same tensor)."""
    import torch.distributed as dist

    if world == 1:
        return []
    u0, _ = unit_map_rows(r0, r1, height)
    own0, own1 = r0 - u0, r1 - u0
    ops = []
    if rank > 0:
        ops.append(dist.P2POp(dist.isend, umap[own0], rank - 1, group))
        ops.append(dist.P2POp(dist.irecv, umap[own0 - 1], rank - 1, group))
    if rank < world - 1:
        ops.append(dist.P2POp(dist.isend, umap[own1 - 1], rank + 1, group))
        ops.append(dist.P2POp(dist.irecv, umap[own1], rank + 1, group))
    return ops


def exchange_unit_map_rows(umap, r0: int, r1: int, height: int, rank: int, world: int, group=None) -> None:
    """Swap the boundary root rows of the decoder unit map with the neighbours (once per code).

    ``umap`` is [u1 - u0, W/16 * words] int32 (unit_map_rows; 32 words per root for the unit map, 8 for
    the block map); own rows are [r0 - u0, r1 - u0).
    """
    run_ops(unit_map_ops(umap, r0, r1, height, rank, world, group))


def gather_codes(records, count, root_offsets, rank: int, world: int, dst: int = 0, group=None):
    """Concatenate per-rank codes on rank ``dst`` (the final code gather).

    ``records[:count]`` (int64, mns_record.h; ``count`` an int or the encoder's device count tensor)
    and ``root_offsets`` (int32, n_local_roots + 1, strip-local) of each rank's contiguous share of roots (strip rows of one image, or images of a
    batch).  Returns (records, root_offsets) of the whole job on ``dst`` -- records in rank order,
    root offsets rebased -- and None on the other ranks.  Any torch.distributed backend.
    """
    import torch
    import torch.distributed as dist

    n_roots = root_offsets.numel() - 1
    if torch.is_tensor(count):  # the encoder's device count: no separate host read
        sizes = torch.cat([count.reshape(1).to(torch.int64),
                           torch.full((1,), n_roots, dtype=torch.int64, device=count.device)])
    else:
        sizes = torch.tensor([count, n_roots], dtype=torch.int64, device=records.device)
    if world == 1:
        return records[: int(sizes[0])], root_offsets
    all_sizes = torch.empty(2 * world, dtype=torch.int64, device=sizes.device)
    dist.all_gather_into_tensor(all_sizes, sizes, group=group)
    table = all_sizes.view(world, 2).tolist()  # the one host read: transfer sizes
    counts = [int(t[0]) for t in table]
    roots = [int(t[1]) for t in table]
    count = counts[rank]
    if rank != dst:
        ops = [dist.P2POp(dist.isend, records[:count].contiguous(), dst, group),
               dist.P2POp(dist.isend, root_offsets[:n_roots].contiguous(), dst, group)]
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        return None
    total, total_roots = sum(counts), sum(roots)
    out = torch.empty(total, dtype=records.dtype, device=records.device)
    offs = torch.empty(total_roots + 1, dtype=root_offsets.dtype, device=root_offsets.device)
    rb = [sum(counts[:r]) for r in range(world)]
    ob = [sum(roots[:r]) for r in range(world)]
    ops = []
    for r in range(world):
        if r == dst:
            out[rb[r]: rb[r] + counts[r]].copy_(records[:count])
            offs[ob[r]: ob[r] + roots[r]].copy_(root_offsets[:n_roots])
        else:
            ops.append(dist.P2POp(dist.irecv, out[rb[r]: rb[r] + counts[r]], r, group))
            ops.append(dist.P2POp(dist.irecv, offs[ob[r]: ob[r] + roots[r]], r, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    for r in range(world):  # strip-local offsets -> global
        if rb[r]:
            offs[ob[r]: ob[r] + roots[r]] += rb[r]
    offs[total_roots] = total
    return out, offs


class StripDecoder:
    """Jacobi decode of one rank's strip: strip-local code + fp32 halo'd ping/pong state.

    Sweeps run two per pass on state with DEC_HALO resident raster rows; the boundary rows are
    exchanged once per pass, and the decoder map carries one neighbour root row on each side.
    ``code.unit_map`` is rebound to a view of that halo'd map, so an encoder writing into ``code``
    fills it in place.  Codes without 2x2 units (``code.min_leaf == 4``, e.g. e3 = inf) run on
    lattice state (mns_decode_pass_lattice: the even 2x2-sum lattice, a quarter of the raster's
    bytes, identical output) from the block map (``code.map_form == 1``); the raster passes read
    the unit map.  ``lattice`` forces the choice.
    """

    def __init__(self, code, height: int, width: int, r0: int, r1: int, rank: int = 0, world: int = 1,
                 lattice=None):
        import torch

        self.code, self.H, self.W, self.r0, self.r1 = code, height, width, r0, r1
        self.rank, self.world = rank, world
        self.lattice = (getattr(code, "min_leaf", 0) == 4) if lattice is None else bool(lattice)
        self.y_lo, self.y_hi = resident_rows(r0, r1, height, DEC_HALO)
        dev = code.records.device
        rows = self.y_hi - self.y_lo
        shape = (rows // 2, width // 2) if self.lattice else (rows, width)
        self.ping = torch.empty(shape, dtype=torch.float32, device=dev)
        self.pong = torch.empty(shape, dtype=torch.float32, device=dev)
        self.out = torch.empty((16 * (r1 - r0), width), dtype=torch.uint8, device=dev)
        self.state = torch.zeros(4, dtype=torch.int32, device=dev)
        self.error = torch.zeros(1, dtype=torch.int32, device=dev)  # lattice mode: 1 if a 2x2 unit was met
        from .codec import MAP_WORDS, build_unit_map

        form = 1 if self.lattice else 0
        if code.unit_map is None or (code.map_form != form and code.unit_map_valid):
            build_unit_map(code, map_form=form)
        elif code.map_form != form:
            raise ValueError(f"code.map_form {code.map_form} does not match the {'lattice' if form else 'raster'} "
                             "decoder (set it before encoding into the code)")
        self.u0, self.u1 = unit_map_rows(r0, r1, height)
        row_words = (width // 16) * MAP_WORDS[form]
        self.umap = torch.zeros((self.u1 - self.u0, row_words), dtype=torch.int32, device=dev)
        own = self.umap[r0 - self.u0: r1 - self.u0]
        own.copy_(code.unit_map[: (r1 - r0) * row_words].view(r1 - r0, row_words))
        code.unit_map = own.view(-1)
        self._ops = {}
        self.overlap = True  # world > 1: boundary rows first, halo exchange beside the interior rows
        self._comm = None

    def _vbase(self, t, row0: int, elem: int):
        return ctypes.c_void_p(t.data_ptr() - row0 * self.W * elem)

    def _state_base(self, t):
        """Virtual-global base (row 0) of a resident state tensor."""
        if t is None:
            return ctypes.c_void_p(0)
        if self.lattice:
            return ctypes.c_void_p(t.data_ptr() - (self.y_lo // 2) * (self.W // 2) * 4)
        return self._vbase(t, self.y_lo, 4)

    def launches(self, iters: int) -> int:
        """Kernel launches of run(iters): an odd first sweep alone, then two sweeps per pass."""
        return iters // 2 + (iters & 1)

    def _exchange(self, t):
        key = id(t)
        if key not in self._ops:  # the P2P descriptors of each resident state tensor are built once
            self._ops[key] = halo_ops(t, self.r0, self.r1, self.H, self.rank, self.world, halo=DEC_HALO,
                                      row_div=2 if self.lattice else 1)
        run_ops(self._ops[key])

    def run(self, iters: int = 10, initial_value: float = 128.0, stream=None, sweep_events=None, out=None):
        """iters sweeps (stop_delta = 0); the last pass writes the rounded uint8 strip into `out` (default self.out).

        sweep_events[i] = (start, end) CUDA events recorded around launch i (see launches()).
        """
        out = self.out if out is None else out
        from . import _native as N

        if iters < 1:
            raise ValueError("max_iters must be >= 1")
        L = N.lib()
        s = N.stream_ptr(stream)
        if "umap" not in self._ops:
            self._ops["umap"] = unit_map_ops(self.umap, self.r0, self.r1, self.H, self.rank, self.world)
        run_ops(self._ops["umap"])
        ob = self._vbase(out, 16 * self.r0, 1)
        cur, it, n = None, 0, 0
        if iters & 1:  # odd count: the flat first sweep alone
            last = iters == 1
            if sweep_events is not None:
                sweep_events[n][0].record()
            if self.lattice:
                N.check(L.mns_decode_flat_lattice(N.ptr(self.umap), self.u0, self.W, self.H, self.r0, self.r1,
                                                  float(initial_value),
                                                  ctypes.c_void_p(0) if last else self._state_base(self.pong),
                                                  ob if last else ctypes.c_void_p(0), s))
            else:
                N.check(L.mns_decode_sweep(N.ptr(self.code.unit_map), self.W, self.H, self.r0, self.r1,
                                           ctypes.c_void_p(0), float(initial_value),
                                           ctypes.c_void_p(0) if last else self._state_base(self.pong),
                                           ob if last else ctypes.c_void_p(0), N.ptr(self.state), 0.0, s))
            if sweep_events is not None:
                sweep_events[n][1].record()
            n += 1
            it = 1
            if not last:
                cur = self.pong
                self._exchange(cur)
        while it < iters:
            last = it + 2 == iters
            nxt = None if last else (self.ping if cur is not self.ping else self.pong)
            if sweep_events is not None:
                sweep_events[n][0].record()
            if last or not self._overlap():
                self._pass(L, cur, nxt, ob, last, initial_value, self.r0, self.r1, s)
                if not last:
                    self._exchange(nxt)
            else:
                # the rows the neighbours need first, their halo exchange on the side stream while the
                # interior rows compute; the next pass waits for both
                import torch

                main = torch.cuda.current_stream() if stream is None else stream
                b0, b1 = self._boundary()
                for a, b in ((self.r0, b0), (b1, self.r1)):
                    if a < b:
                        self._pass(L, cur, nxt, ob, False, initial_value, a, b, s)
                self._comm.wait_stream(main)
                with torch.cuda.stream(self._comm):
                    self._exchange(nxt)
                if b0 < b1:
                    self._pass(L, cur, nxt, ob, False, initial_value, b0, b1, s)
                main.wait_stream(self._comm)
            if sweep_events is not None:
                sweep_events[n][1].record()
            n += 1
            it += 2
            if not last:
                cur = nxt
        return out

    def _overlap(self) -> bool:
        """Split passes into boundary + interior (halo exchange overlapped) for strips of >= 6 root rows."""
        if self.world == 1 or not self.overlap or self.r1 - self.r0 < 6:
            return False
        if self._comm is None:
            import torch

            self._comm = torch.cuda.Stream(device=self.code.records.device)
        return True

    def _boundary(self):
        """Root rows [b0, b1) not sent to a neighbour: the 32 halo rows are the first / last two root rows."""
        return self.r0 + (2 if self.rank > 0 else 0), self.r1 - (2 if self.rank < self.world - 1 else 0)

    def _pass(self, L, cur, nxt, ob, last, initial_value, a, b, s):
        from . import _native as N

        if self.lattice:
            N.check(L.mns_decode_pass_lattice(N.ptr(self.umap), self.u0, self.W, self.H, a, b, self._state_base(cur),
                                              float(initial_value), self._state_base(nxt),
                                              ob if last else ctypes.c_void_p(0), N.ptr(self.error), s))
        else:
            N.check(L.mns_decode_sweep2(N.ptr(self.umap), self.u0, self.W, self.H, a, b, self._state_base(cur),
                                        float(initial_value), self._state_base(nxt),
                                        ob if last else ctypes.c_void_p(0), s))


class StripDecoderF64:
    """Strip decode with the reference's early stop (decoder.py:66-77) across ranks, bit-exact.

    Every sweep is the exact fp64 step (mns_decode_f64_sweep) of this rank's units on its strip
    plus a 16-row halo (one sweep per exchange; every clamped domain of a root lies within 16 rows
    of it).  The sweep's local max|delta| lands in ``state[2]`` (fp64 bits); ranks all-reduce it
    (MAX) -- the whole image's delta, exactly as the reference computes it -- before
    mns_decode_f64_decide applies ``delta < stop_delta`` on the device, so every rank stops after
    the same sweep with no host synchronisation (later sweeps are no-ops).  ``code`` is a
    strip-local DeviceCode (global coordinates, encode_device(root_rows=...)).
    """

    def __init__(self, code, height: int, width: int, r0: int, r1: int, rank: int = 0, world: int = 1,
                 group=None, units=None):
        import torch

        self.code, self.H, self.W, self.r0, self.r1 = code, height, width, r0, r1
        self.rank, self.world, self.group = rank, world, group
        self.y_lo, self.y_hi = resident_rows(r0, r1, height, HALO)
        dev = code.records.device if code is not None else torch.device("cpu")
        rows = self.y_hi - self.y_lo
        self.ping = torch.empty((rows, width), dtype=torch.float64, device=dev)
        self.pong = torch.empty((rows, width), dtype=torch.float64, device=dev)
        self.out = torch.empty((16 * (r1 - r0), width), dtype=torch.uint8, device=dev)
        self.state = torch.zeros(4, dtype=torch.int64, device=dev)
        self.iters_done = torch.zeros(1, dtype=torch.int32, device=dev)
        self.units = units
        self._ops = {}

    def _base(self, t):
        return ctypes.c_void_p(t.data_ptr() - self.y_lo * self.W * 8)

    def delta_view(self):
        """state[2] as a float64 tensor (the all-reduced word)."""
        import torch

        return self.state[2:3].view(torch.float64)

    def sweep(self, cur, nxt, stream=None) -> None:
        from . import _native as N

        L = N.lib()
        u = self.units
        N.check(L.mns_decode_f64_sweep(N.ptr(u["x"]), N.ptr(u["y"]), N.ptr(u["size"]), N.ptr(u["dx"]),
                                       N.ptr(u["dy"]), N.ptr(u["s"]), N.ptr(u["o"]), int(u["n"]), self.W,
                                       self._base(cur), self._base(nxt), N.ptr(self.state), N.stream_ptr(stream)))

    def decide(self, stop_delta: float, stream=None) -> None:
        from . import _native as N

        N.check(N.lib().mns_decode_f64_decide(N.ptr(self.state), float(stop_delta), N.stream_ptr(stream)))

    def finalize(self, stream=None):
        from . import _native as N

        N.check(N.lib().mns_decode_f64_finalize(self._base(self.ping), self._base(self.pong), N.ptr(self.state),
                                                self.W, 16 * self.r0, 16 * self.r1, N.ptr(self.out),
                                                N.ptr(self.iters_done), N.stream_ptr(stream)))
        return self.out

    def _exchange(self, t):
        key = id(t)
        if key not in self._ops:
            self._ops[key] = halo_ops(t, self.r0, self.r1, self.H, self.rank, self.world, self.group, HALO)
        run_ops(self._ops[key])

    def run(self, max_iters: int = 10, stop_delta: float = 0.5, initial_value: float = 128.0, stream=None):
        """max_iters sweeps at most; returns the uint8 strip (own rows).  ``iters_done`` holds the
        sweep count after the stream reaches the end (the same on every rank)."""
        import torch.distributed as dist

        if max_iters < 1:
            raise ValueError("max_iters must be >= 1")
        if self.units is None:
            from .codec import records_to_units_device

            self.code.join(stream)
            self.units = records_to_units_device(self.code.records, self.code.n_records(), self.W, self.H, stream)
        self.state.zero_()
        self.ping.fill_(float(initial_value))
        cur, nxt = self.ping, self.pong
        delta = self.delta_view()
        for _ in range(max_iters):
            self.sweep(cur, nxt, stream)
            if self.world > 1:
                dist.all_reduce(delta, op=dist.ReduceOp.MAX, group=self.group)
            self.decide(stop_delta, stream)
            self._exchange(nxt)
            cur, nxt = nxt, cur
        return self.finalize(stream)


def pack_search(res: dict):
    """Per-range search result (dom int32, iso int8, o uint8, code uint8) -> one int64 per range."""
    import torch

    return (res["dom"].to(torch.int64) | (res["iso"].to(torch.int64) & 0xFF) << 32 |
            res["o"].to(torch.int64) << 40 | res["code"].to(torch.int64) << 48)


def unpack_search(packed) -> dict:
    import torch

    return {"dom": (packed & 0xFFFFFFFF).to(torch.int32), "iso": ((packed >> 32) & 0xFF).to(torch.int8),
            "o": ((packed >> 40) & 0xFF).to(torch.uint8), "code": ((packed >> 48) & 0xFF).to(torch.uint8)}


def search_sharded(search_fn, n_ranges: int, rank: int, world: int, group=None):
    """Full / local search with the ranges split across ranks: this rank runs
    ``search_fn(r0, r1)`` on its contiguous share [r0, r1) (image and domain pool replicated, no
    data-path collective) and the per-range results (8 B each: domain, isometry, offset, contrast)
    are all-gathered, so every rank ends with the whole image's result in range order.  Shares are
    near-equal (split), so the gather pads to the largest share."""
    import torch
    import torch.distributed as dist

    r0, r1 = split(n_ranges, world, rank)
    mine = pack_search(search_fn(r0, r1))
    if world == 1:
        return unpack_search(mine)
    width = -(-n_ranges // world)
    buf = torch.zeros(width, dtype=torch.int64, device=mine.device)
    buf[: r1 - r0] = mine
    allb = torch.empty(world * width, dtype=torch.int64, device=mine.device)
    dist.all_gather_into_tensor(allb, buf, group=group)
    parts = [allb[r * width: r * width + (split(n_ranges, world, r)[1] - split(n_ranges, world, r)[0])]
             for r in range(world)]
    return unpack_search(torch.cat(parts))
