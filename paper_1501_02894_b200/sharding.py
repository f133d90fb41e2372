"""Multi-GPU decomposition of the MNS hot path (one process per GPU, torch.distributed).

SURVEY 8(e):
* batches of images (config c3)  -- images split across ranks, no data-path collective;
* one huge image (config c5)     -- row strips of whole root rows; every strip reads a
  16-row read-only halo of the input (all clamped domains of a root lie within 16 rows
  of it) and uses GLOBAL coordinates for clamping, so encode needs no exchange;
  the Jacobi decode exchanges the 16 boundary rows of the raster with the up/down
  neighbours after every sweep (NCCL send/recv over NVLink; gloo in the CPU tests);
* full / local search (config c4) -- ranges split across ranks, pool replicated.
Codes stay on the rank that produced them (root_offsets are strip-local); a
gather to rank 0 is a plain all_gather of sizes + records when the caller needs it.
"""

from __future__ import annotations

import ctypes

HALO = 16  # rows: every co-centred domain of a 16x16 root lies within 16 rows of it


def split(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous near-equal split of n items: [begin, end) of `rank`."""
    return n * rank // world, n * (rank + 1) // world


def strip_rows(height: int, world: int, rank: int) -> tuple[int, int]:
    """Root rows [r0, r1) of this rank's strip of a height-pixel image."""
    return split(height // 16, world, rank)


def resident_rows(r0: int, r1: int, height: int) -> tuple[int, int]:
    """Pixel rows [y_lo, y_hi) a strip needs resident (its rows plus the halo, clipped)."""
    return max(0, 16 * r0 - HALO), min(height, 16 * r1 + HALO)


def exchange_halos(raster, r0: int, r1: int, height: int, rank: int, world: int, group=None) -> None:
    """After a sweep: send my first/last HALO own rows to the neighbours, receive theirs into my halos.

    ``raster`` holds rows [y_lo, y_hi) (resident_rows) of the full image.  Works for any
    torch.distributed backend (NCCL on GPUs, gloo on CPU).
    """
    import torch.distributed as dist

    if world == 1:
        return
    y_lo, y_hi = resident_rows(r0, r1, height)
    own0, own1 = 16 * r0 - y_lo, 16 * r1 - y_lo
    ops = []
    if rank > 0:
        ops.append(dist.P2POp(dist.isend, raster[own0: own0 + HALO], rank - 1, group))
        ops.append(dist.P2POp(dist.irecv, raster[own0 - HALO: own0], rank - 1, group))
    if rank < world - 1:
        ops.append(dist.P2POp(dist.isend, raster[own1 - HALO: own1], rank + 1, group))
        ops.append(dist.P2POp(dist.irecv, raster[own1: own1 + HALO], rank + 1, group))
    for req in dist.batch_isend_irecv(ops):
        req.wait()


class StripDecoder:
    """Jacobi decode of one rank's strip: strip-local code + fp32 halo'd ping/pong rasters."""

    def __init__(self, code, height: int, width: int, r0: int, r1: int, rank: int = 0, world: int = 1):
        import torch

        self.code, self.H, self.W, self.r0, self.r1 = code, height, width, r0, r1
        self.rank, self.world = rank, world
        self.y_lo, self.y_hi = resident_rows(r0, r1, height)
        dev = code.records.device
        rows = self.y_hi - self.y_lo
        self.ping = torch.empty((rows, width), dtype=torch.float32, device=dev)
        self.pong = torch.empty((rows, width), dtype=torch.float32, device=dev)
        self.out = torch.empty((16 * (r1 - r0), width), dtype=torch.uint8, device=dev)
        self.state = torch.zeros(4, dtype=torch.int32, device=dev)
        if code.unit_map is None:
            from .codec import build_unit_map

            build_unit_map(code)

    def _vbase(self, t, row0: int, elem: int):
        return ctypes.c_void_p(t.data_ptr() - row0 * self.W * elem)

    def run(self, iters: int = 10, initial_value: float = 128.0, stream=None, sweep_events=None, out=None):
        """iters sweeps (stop_delta = 0); the last writes the rounded uint8 strip into `out` (default self.out)."""
        out = self.out if out is None else out
        from . import _native as N

        L = N.lib()
        s = N.stream_ptr(stream)
        bufs = (self.ping, self.pong)
        for it in range(iters):
            cur = None if it == 0 else bufs[(it - 1) & 1]
            last = it == iters - 1
            nxt = None if last else bufs[it & 1]
            if sweep_events is not None:
                sweep_events[it][0].record()
            N.check(L.mns_decode_sweep(N.ptr(self.code.unit_map), self.W, self.H, self.r0, self.r1,
                                       self._vbase(cur, self.y_lo, 4) if cur is not None else ctypes.c_void_p(0),
                                       float(initial_value),
                                       self._vbase(nxt, self.y_lo, 4) if nxt is not None else ctypes.c_void_p(0),
                                       self._vbase(out, 16 * self.r0, 1) if last else ctypes.c_void_p(0),
                                       N.ptr(self.state), 0.0, s))
            if sweep_events is not None:
                sweep_events[it][1].record()
            if not last and self.world > 1:
                exchange_halos(nxt, self.r0, self.r1, self.H, self.rank, self.world)
        return out
