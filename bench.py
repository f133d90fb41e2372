#!/usr/bin/env python
"""Benchmark of the MNS hot path on B200 (contract: one JSON line on rank 0).

Workload (BASELINE.json configs[4], the largest single-GPU config; configs[1] is a
512^2 image that is launch-latency bound): one 16384 x 16384 uint8 image from the
pinned synthetic generator (noise sigma 10, 24 blobs, seed 5), MNS encode with the
16->8->4 quadtree (EncoderConfig(e3=inf)) and a 10-sweep Jacobi decode from flat 128
(DecodeConfig(max_iters=10, stop_delta=0)).  A step = encode + decode of the whole
image; with N GPUs the image is split into N row strips (16-row read-only input
halo; the decode runs two Jacobi sweeps per kernel pass on lattice state with a 32-row
halo, exchanged over NCCL on a side stream beside the interior rows after every pass)
-- fixed total work, "scaling": "strong".

  value   8x8-range blocks (W*H/64 = 4,194,304 per image) per second of the whole
          encode+decode step, inputs resident in HBM, max over ranks; at N = 1 two steps
          are in flight (two streams, each with its own code and decoder buffers), the
          one-step latency is components.latency_ms_per_step;
  e2e     the same through the public device API with the image copied from pinned
          host memory and the decoded image copied back inside the timed region;
  roofline  the dominant kernel (decode_pair_lat_kernel: two sweeps per pass on the fp32 2x2-sum
          lattice, lattice t read + lattice t+2 written, 2 B/px per launch);
  cpu_baseline  the CPU oracle (oracle/, literal fp64 port of the reference) on a
          bounded sample on this host.

--impl reference runs the reference's CPU implementation of the path (the oracle
port -- the reference is pure Python/numpy and has no build) on the same metric, plus
the unmodified Python reference itself (baseline/_ref) on c1, c2 and a c5 window.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

MEASURED = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM_GBS = 6650.0
FALLBACK_TENSOR_TFLOPS = 1590.0  # dense bf16, B200_PROFILING.md fallback
IMG = 16384
ITERS = 10
METRIC = "range blocks encoded/sec (MNS) and Mpixel/s decoded; full-search pair-evals/s"


def measured_traffic(kernel):
    """DRAM bytes per launch of `kernel` from the committed ncu --set full capture (profiles/traffic.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return int(json.load(f)[kernel]["per_launch_bytes"])
    except Exception:
        return None


def peaks():
    try:
        with open(MEASURED) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


def tensor_peak():
    """Dense bf16 TF/s (FP16 runs at the same tensor rate on B200): the full-search denominator.  The
    search is timed in isolation (a few ms), so the burst figure applies; the sustained one (a matmul
    loop of 4 s, clocks dropping under power) is reported beside it."""
    try:
        with open(MEASURED) as f:
            d = json.load(f)
        return float(d["bf16_tflops"]), "measured (bf16 burst)", float(d.get("bf16_tflops_sustained", 0.0)) or None
    except Exception:
        return FALLBACK_TENSOR_TFLOPS, "fallback", None


class ClockSampler:
    """SM clock and throttle reasons sampled during the timed region: NVML every 2 ms from a thread
    (a timed region is often well under 100 ms), nvidia-smi -lms 50 when NVML is unavailable."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    BITS = [0x8, 0x40, 0x20, 0x4]  # nvmlClocksEventReason{HwSlowdown, HwThermalSlowdown, SwThermalSlowdown, SwPowerCap}

    def __init__(self, index: int):
        self.index = index
        self.rows = []  # (sm_mhz, max_mhz, reason names)
        self.proc = None
        self.nvml = None
        self.stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self.nvml = pynvml

            def poll():
                while not self.stop.is_set():
                    try:
                        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        bits = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.rows.append((float(sm), float(mx), [n for n, b in zip(self.NAMES, self.BITS) if bits & b]))
                    except Exception:
                        pass
                    time.sleep(0.002)

            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            r = [v.strip() for v in line.split(",")]
            if len(r) >= 6 and r[0].replace(".", "").isdigit() and r[1].replace(".", "").isdigit():
                self.rows.append((float(r[0]), float(r[1]), [self.NAMES[k] for k in range(4) if r[2 + k] == "Active"]))

    def __exit__(self, *a):
        self.stop.set()
        if self.nvml:
            self.t.join(timeout=1)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm = [r[0] for r in self.rows]
        mx = [r[1] for r in self.rows]
        reasons = sorted({n for r in self.rows for n in r[2]})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm), "source": "nvml" if self.nvml else "nvidia-smi"}


# ------------------------------------------------------------------------- CPU legs

def cpu_sample(img: np.ndarray, rows: int = 2048, threads: int | None = None, keep: bool = False):
    """Oracle encode + 10-sweep decode of the top `rows` rows of the c5 image (own image).
    keep=True also returns the oracle's records, per-root counts and decoded image (the parity check)."""
    from oracle import oracle as O

    s = np.ascontiguousarray(img[:rows])
    t0 = time.perf_counter()
    rec, counts = O.encode_quadtree_records(s, (8.0, 8.0, math.inf), 16.0, True, 1, nthreads=threads)
    out, _, _ = O.decode_records(rec, s.shape[1], s.shape[0], max_iters=ITERS, stop_delta=0.0, nthreads=threads)
    dt = time.perf_counter() - t0
    if keep:
        return s.size / 64 / dt, dt, (rec, counts, out)
    return s.size / 64 / dt, dt


def parity_check(img_np, got_rec, got_offs, got_out, r0, r1, oracle_result=None):
    """The benchmarked output against the CPU oracle (north_star's bar): this rank's strip of the c5
    code bit-exact (records and root offsets) and its decoded rows within 1 LSB and 0.01 dB."""
    from oracle import oracle as O

    if oracle_result is None:
        rec, counts = O.encode_quadtree_records(img_np, (8.0, 8.0, math.inf), 16.0, True, 1)
        out, _, _ = O.decode_records(rec, img_np.shape[1], img_np.shape[0], max_iters=ITERS, stop_delta=0.0)
    else:
        rec, counts, out = oracle_result
    rw = img_np.shape[1] // 16
    offs = np.zeros(len(counts) + 1, np.int64)
    np.cumsum(counts, out=offs[1:])
    a, b = offs[r0 * rw], offs[r1 * rw]
    want_rec = rec[a:b]
    want_offs = offs[r0 * rw: r1 * rw + 1] - a
    rec_ok = len(got_rec) == len(want_rec) and bool(np.array_equal(got_rec, want_rec))
    offs_ok = bool(np.array_equal(got_offs.astype(np.int64), want_offs))
    rows = slice(16 * r0, 16 * r1)
    src = img_np[rows].astype(np.float64)
    want = out[rows]
    d = np.abs(got_out.astype(np.int16) - want.astype(np.int16))

    def psnr(x):
        e = float(np.mean((src - x.astype(np.float64)) ** 2))
        return math.inf if e == 0 else 10 * math.log10(255 * 255 / e)

    dpsnr = abs(psnr(got_out) - psnr(want))
    return {"codes": "bit-exact" if rec_ok and offs_ok else "MISMATCH", "records": int(len(got_rec)),
            "oracle_records": int(len(want_rec)), "decode_max_lsb": int(d.max()),
            "pixels_off_by_1": int((d == 1).sum()), "psnr_delta_db": dpsnr,
            "pass": bool(rec_ok and offs_ok and int(d.max()) <= 1 and dpsnr <= 0.01),
            "scope": f"root rows {r0}..{r1 - 1} of 1024 (rank 0's strip) vs the fp64 CPU oracle "
                     "(oracle/mns_oracle.c, pinned to reference goldens)"}


def python_reference_timings():
    """The unmodified pure-Python reference (baseline/_ref/mnscodec, installed by build()) timed on this
    host, one process, best of 3 (BASELINE.md's CPU-baseline plan): c1 and c2 as the configs name them,
    and a 512^2 window of the c5 image (e3 = inf, 10 sweeps) as the c5 per-block rate.  Informational:
    the arm's value is the oracle port over the c5 sample."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "mnscodec")):
        return {"unavailable": "baseline/_ref/mnscodec not installed (build() installs it where /root/reference exists)"}
    if ref not in sys.path:
        sys.path.insert(0, ref)
    try:
        import mnscodec as M
    except Exception as e:  # pragma: no cover - depends on the box
        return {"unavailable": f"import failed: {e}"}
    from paper_1501_02894_b200.synth import config_image

    out = {"package": os.path.relpath(os.path.dirname(M.__file__), ROOT), "processes": 1,
           "host_cpus": os.cpu_count(), "timing": "best of 3, time.perf_counter"}
    cases = (("c1", config_image("c1"), M.EncoderConfig(), 8),
             ("c1_e3_inf", config_image("c1"), M.EncoderConfig(e3=math.inf), 8),
             ("c2", config_image("c2"), M.EncoderConfig(), 10),
             ("c5_window_512", config_image("c5")[:512, :512].copy(), M.EncoderConfig(e3=math.inf), 10))
    from paper_1501_02894_b200.synth import batch_seeds, synth_image

    # c3: encode only (the reference has no 8->4 root level: its 16->8->4 with e3 = inf), a 4-image
    # subset, extrapolated per block
    t_c3 = []
    for _ in range(3):
        t0 = time.perf_counter()
        for sd in batch_seeds(4):
            M.encode_quadtree(M.GrayImage(synth_image(512, sd)), M.EncoderConfig(e3=math.inf))
        t_c3.append(time.perf_counter() - t0)
    out["c3_subset_4_images"] = {"encode_s": min(t_c3), "blocks_per_s": 4 * 4096 / min(t_c3),
                                 "extrapolated_256_images_s": 64 * min(t_c3)}
    # c4 searches on a 128^2 crop of the c4 image (the full 512^2 full search takes about a minute
    # on one core): full search B = 8 stride 1 (256 ranges x 113^2 domains) and the +-4 local search
    c4 = M.GrayImage(config_image("c4")[:128, :128].copy())
    t_fs, t_ls = [], []
    for _ in range(2):
        t0 = time.perf_counter()
        M.encode_full_search(c4, 8, M.EncoderConfig(mode="full_search"))
        t_fs.append(time.perf_counter() - t0)
        t0 = time.perf_counter()
        M.encode_local_search(c4, M.EncoderConfig())
        t_ls.append(time.perf_counter() - t0)
    out["c4_full_search_crop_128"] = {"s": min(t_fs), "pair_evals": 256 * 113 * 113,
                                      "pair_evals_per_s": 256 * 113 * 113 / min(t_fs)}
    out["c4_local_search_crop_128"] = {"s": min(t_ls), "candidate_fits": 256 * 81,
                                       "candidate_fits_per_s": 256 * 81 / min(t_ls)}
    for name, px, cfg, iters in cases:
        img = M.GrayImage(px)
        enc, dec = [], []
        for _ in range(3):
            t0 = time.perf_counter()
            code = M.encode_quadtree(img, cfg)
            t1 = time.perf_counter()
            M.decode(code, M.DecodeConfig(max_iters=iters, stop_delta=0.0))
            t2 = time.perf_counter()
            enc.append(t1 - t0)
            dec.append(t2 - t1)
        blocks = px.shape[0] * px.shape[1] / 64
        e, d = min(enc), min(dec)
        out[name] = {"image": f"{px.shape[1]}x{px.shape[0]}", "encode_s": e, "decode_s": d, "decode_sweeps": iters,
                     "blocks_per_s": blocks / (e + d)}
    return out


def run_reference(args, img):
    from oracle import oracle as O

    threads = O.default_threads()
    rows = args.cpu_rows
    for _ in range(args.warmup):
        cpu_sample(img, rows, threads)
    times = []
    for _ in range(args.steps):
        _, dt = cpu_sample(img, rows, threads)
        times.append(dt)
    per_step = float(np.mean(times))
    value = (rows * IMG / 64) / per_step
    sample = f"c5 rows 0..{rows - 1} ({rows}x{IMG}, {rows // 16} of 1024 root rows) encoded + {ITERS}-sweep decoded"
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "blocks/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_step * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "c5: MNS encode (16->8->4, e3=inf) + 10-sweep decode, 16384^2 uint8, sigma 10, "
                                   "24 blobs, seed 5", "image": f"{IMG}x{IMG}", "sample_rows": rows},
            "cpu_baseline": {"value": value, "unit": "blocks/s", "cores": threads, "kind": "port",
                             "sample": sample},
            "e2e": {"value": value, "unit": "blocks/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if not args.no_python_ref:
        line["python_reference"] = python_reference_timings()
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------- GPU leg

def _med_ms(fn, reps=5, warm=2):
    """Median device time (CUDA events on the current stream) of fn() over reps calls."""
    import torch

    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def next_rows_components(dev, code, W, H, r0, r1, whole=False):
    """SURVEY 8(f), measured beside the path (rank 0, informational): the GPU .mns packer and the GPU
    stream reader on rank 0's c5 code (round trip checked bit-exact), the device RD sweep on c2 and
    the offset histogram on c4 (full search + counting)."""
    import torch

    import paper_1501_02894_b200 as mns
    from paper_1501_02894_b200 import rd
    from paper_1501_02894_b200.synth import config_image

    out = {}
    n = code.n_records()
    h = 16 * (r1 - r0)
    rec = code.records[:n]
    packed, bits_t = mns.write_stream_device(rec, n, W, h, W, h, True, True)
    nbytes = (int(bits_t.item()) + 7) // 8
    w_ms = _med_ms(lambda: mns.write_stream_device(rec, n, W, h, W, h, True, True))
    buf = packed[:nbytes].clone()
    from paper_1501_02894_b200.codec import read_stream_device

    back, status = read_stream_device(buf, True, True, W, h)
    ok = int(status[0].item()) == -1 and back.n_records() == n and bool(torch.equal(back.records[:n], rec))
    r_ms = _med_ms(lambda: read_stream_device(buf, True, True, W, h))
    out["mns_stream"] = {"code": f"c5 rank-0 strip ({W}x{h}), {n} leaves, {nbytes} bytes .mns",
                         "write_ms": w_ms, "write_leaves_per_s": n / (w_ms / 1e3),
                         "write_gbs": (8 * n + nbytes) / (w_ms / 1e3) / 1e9,
                         "read_ms": r_ms, "read_leaves_per_s": n / (r_ms / 1e3),
                         "read_gbs": (nbytes + 8 * n) / (r_ms / 1e3) / 1e9,
                         "roundtrip": "bit-exact" if ok else "MISMATCH",
                         "note": "write: records (8 B/leaf) in, .mns out; read: .mns in, records out"}
    if whole:  # the reference's default DecodeConfig (max_iters 10, stop_delta 0.5): the exact fp64 path
        _, it, _ = mns.decode_device(code, iters=10, stop_delta=0.5)
        torch.cuda.synchronize()
        x_ms = _med_ms(lambda: mns.decode_device(code, iters=10, stop_delta=0.5))
        sweeps = int(it.item())
        out["exact_decode"] = {"config": f"c5 code ({n} leaves), DecodeConfig() defaults: max_iters 10, stop_delta 0.5",
                               "ms": x_ms, "sweeps": sweeps, "mpix_per_s": W * h / (x_ms / 1e3) / 1e6,
                               "gbs": sweeps * 16.0 * W * h / (x_ms / 1e3) / 1e9,
                               "note": "bit-exact fp64 decode_step sweeps with the reference's early stop decided on the "
                                       "device (records -> units, fill, sweeps + decisions, uint8 finalize); gbs = 16 B "
                                       "per pixel per executed sweep over the whole call"}
    c2 = config_image("c2")
    grid = (2.0, 4.0, 8.0, 16.0, 32.0)
    rd.rd_sweep(c2, ["mns"], grid[:1])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pts = rd.rd_sweep(c2, ["mns", "no_search"], grid)
    dt = time.perf_counter() - t0
    out["rd_sweep"] = {"config": "c2 512^2, modes mns + no_search x E in {2, 4, 8, 16, 32}, default decode",
                       "points": len(pts), "s": dt, "ms_per_point": 1e3 * dt / len(pts),
                       "note": "host wall clock per point (encode, .mns bit count, decode, SSE on the device)"}
    c4 = config_image("c4")
    rd.offset_histogram_device(c4)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        rd.offset_histogram_device(c4)
    torch.cuda.synchronize()
    out["offset_histogram"] = {"config": "c4 512^2, B = 8 stride 1, identity", "ms": 1e3 * (time.perf_counter() - t0) / 3,
                               "note": "host wall clock: H2D of the image, full search, histogram, D2H"}
    return out


def small_configs(dev, rank, world):
    """BASELINE configs 1-3: c1/c2 are latency-bound single images -- one encode +
    decode step captured in a CUDA graph and replayed 1000 times back to back (rank 0); c3 is the
    batched 8->4 encode of 256 512^2 images (seeds 1000..1255), split across ranks, no collective."""
    import torch
    import torch.distributed as dist

    import paper_1501_02894_b200 as mns
    from paper_1501_02894_b200 import sharding
    from paper_1501_02894_b200.synth import batch_seeds, config_image, synth_image

    def dev_code(nb, H, W):
        n_roots = nb * (H // 16) * (W // 16)
        return mns.DeviceCode(torch.empty(64 * n_roots, dtype=torch.int64, device=dev),
                              torch.empty(n_roots + 1, dtype=torch.int32, device=dev),
                              torch.zeros(1, dtype=torch.int64, device=dev), W, H, nb,
                              unit_map=torch.empty(8 * n_roots, dtype=torch.int32, device=dev), map_form=1)

    def ev():
        return torch.cuda.Event(enable_timing=True)

    out = {}
    cfg = mns.EncoderConfig(e3=math.inf)
    if rank == 0:
        for name, root_level, iters, desc in (("c1", 2, 8, "256^2, 8->4 quadtree, 8 decode sweeps"),
                                              ("c2", 1, 10, "512^2, 16->8->4 quadtree, 10 decode sweeps")):
            px = config_image(name)
            H, W = px.shape
            img = torch.from_numpy(px).to(dev)
            code = dev_code(1, H, W)
            u8 = torch.empty((H, W), dtype=torch.uint8, device=dev)
            rasters = (torch.empty((H, W), dtype=torch.float32, device=dev),
                       torch.empty((H, W), dtype=torch.float32, device=dev))

            s_cmp = torch.cuda.Stream()

            def step():
                # as in the c5 step: the record compaction runs on its own stream beside the decode
                # (which reads the encoder's unit map) and is joined before the step ends
                cur = torch.cuda.current_stream()
                s_cmp.wait_stream(cur)
                mns.encode_device(img, cfg, root_level=root_level, out=code, compact_stream=s_cmp)
                mns.decode_device(code, iters=iters, stop_delta=0.0, initial_value=128.0, out=u8, rasters=rasters)
                cur.wait_stream(s_cmp)

            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                for _ in range(3):
                    step()
            torch.cuda.current_stream().wait_stream(side)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                step()
            for _ in range(10):
                g.replay()
            torch.cuda.synchronize()
            reps = 1000
            a, b = ev(), ev()
            a.record()
            for _ in range(reps):
                g.replay()
            b.record()
            torch.cuda.synchronize()
            us = a.elapsed_time(b) * 1e3 / reps
            out[name] = {"config": desc, "latency_us": us, "blocks_per_s": W * H / 64 / (us * 1e-6),
                         "graph_replays": reps}
    if rank == 0:  # c2 with the 8-isometry extension (BASELINE configs[1]): encode + exact fp64 decode
        px = config_image("c2")
        img = torch.from_numpy(px).to(dev)
        for _ in range(3):
            c = mns.encode_device(img, cfg, n_iso=8)
            mns.decode_device(c, iters=10, stop_delta=0.0)
        torch.cuda.synchronize()
        reps, a, b = 20, ev(), ev()
        a.record()
        for _ in range(reps):
            c = mns.encode_device(img, cfg, n_iso=8)
            mns.decode_device(c, iters=10, stop_delta=0.0)
        b.record()
        torch.cuda.synchronize()
        us = a.elapsed_time(b) * 1e3 / reps
        out["c2_iso8"] = {"config": "512^2, 16->8->4 quadtree, 8 isometries (extension), 10 exact fp64 decode sweeps",
                          "latency_us": us, "blocks_per_s": 4096 / (us * 1e-6), "note": "not graph-captured"}
    # c3: batched encode, images split across ranks
    i0, i1 = sharding.split(256, world, rank)
    seeds = batch_seeds()[i0:i1]
    batch = torch.from_numpy(np.stack([synth_image(512, s, noise_sigma=6.0, n_blobs=6) for s in seeds])).to(dev)
    code = dev_code(len(seeds), 512, 512)
    for _ in range(3):
        mns.encode_device(batch, cfg, root_level=2, out=code)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    reps = 20
    a, b = ev(), ev()
    a.record()
    for _ in range(reps):
        mns.encode_device(batch, cfg, root_level=2, out=code)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    if world > 1:
        m = torch.tensor([ms], device=dev)
        dist.all_reduce(m, op=dist.ReduceOp.MAX)
        ms = float(m.item())
    out["c3"] = {"config": "256 x 512^2 (seeds 1000..1255), 8->4 quadtree, encode only, images split across "
                           f"{world} rank(s)", "ms_per_batch": ms, "images_per_s": 256 / (ms / 1e3),
                 "blocks_per_s": 256 * 4096 / (ms / 1e3)}
    return out


def run_ours(args, img_np, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_1501_02894_b200 as mns
    from paper_1501_02894_b200 import sharding

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    H = W = IMG
    r0, r1 = sharding.strip_rows(H, world, rank)
    y_lo, y_hi = sharding.resident_rows(r0, r1, H)
    cfg = mns.EncoderConfig(e3=math.inf)
    host = torch.from_numpy(np.ascontiguousarray(img_np[y_lo:y_hi])).pin_memory()
    img = host.to(dev)
    n_roots = (r1 - r0) * (W // 16)
    code = mns.DeviceCode(torch.empty(64 * n_roots, dtype=torch.int64, device=dev),
                          torch.empty(n_roots + 1, dtype=torch.int32, device=dev),
                          torch.zeros(1, dtype=torch.int64, device=dev), W, H, 1, r0, r1,
                          unit_map=torch.empty(8 * n_roots, dtype=torch.int32, device=dev), map_form=1)
    # e3 = inf: the code has no 2x2 leaves, so the decoder carries the 2x2-sum lattice between passes
    dec = sharding.StripDecoder(code, H, W, r0, r1, rank, world, lattice=True)
    out_host = torch.empty((16 * (r1 - r0), W), dtype=torch.uint8).pin_memory()
    if os.environ.get("MNS_BENCH_PRIORITY", "1") != "0":
        # the step's kernels on a high-priority stream: the compaction's CTAs (low priority) fill the
        # decode passes' tails instead of taking SMs from their waves
        torch.cuda.set_stream(torch.cuda.Stream(priority=torch.cuda.Stream.priority_range()[1]))
    stream = torch.cuda.current_stream()
    # the record compaction (second encode kernel) runs on its own stream, overlapping the decode,
    # which only needs the unit map; every step joins it before the step ends
    s_cmp = torch.cuda.Stream()

    def step(e2e=False, ev=None):
        if e2e:
            img.copy_(host, non_blocking=True)
        if ev:
            ev[0].record()
        mns.encode_device(img, cfg, root_rows=(r0, r1), height=H, out=code, compact_stream=s_cmp)
        if ev:
            ev[1].record()
        dec.run(ITERS, 128.0, sweep_events=ev[2] if ev else None)
        stream.wait_stream(s_cmp)  # the code (records, root offsets) is complete inside the step
        if ev:
            ev[3].record()
        if e2e:
            out_host.copy_(dec.out, non_blocking=True)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local_rank])
        torch.cuda.synchronize()

    def timed(k, e2e, record=False):
        evs = []
        for _ in range(k):
            evs.append([torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
                        [[torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)]
                         for _ in range(dec.launches(ITERS))],
                        torch.cuda.Event(enable_timing=True)] if record else None)
        barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record()
        for i in range(k):
            step(e2e, evs[i])
        t1.record()
        barrier()
        ms = t0.elapsed_time(t1)
        if world > 1:
            m = torch.tensor([ms], device=dev)
            dist.all_reduce(m, op=dist.ReduceOp.MAX)
            ms = float(m.item())
        return ms, evs

    img2 = [img, torch.empty_like(img)]
    out2 = [dec.out, torch.empty_like(dec.out)]
    out_host2 = [out_host, torch.empty_like(out_host).pin_memory()]
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()

    def timed_e2e(k):
        ev = lambda: torch.cuda.Event()  # noqa: E731
        h2d = [ev() for _ in range(k)]
        enc_done = [ev() for _ in range(k)]
        comp = [ev() for _ in range(k)]
        d2h = [ev() for _ in range(k)]
        barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(s_in)
        for i in range(k):
            b = i & 1
            with torch.cuda.stream(s_in):  # H2D of step i (its buffer was last read by step i-2's encode)
                if i >= 2:
                    s_in.wait_event(enc_done[i - 2])
                img2[b].copy_(host, non_blocking=True)
                h2d[i].record(s_in)
            stream.wait_event(h2d[i])
            if i >= 2:
                stream.wait_event(d2h[i - 2])  # output buffer b drained
            mns.encode_device(img2[b], cfg, root_rows=(r0, r1), height=H, out=code, compact_stream=s_cmp)
            enc_done[i].record(stream)
            dec.run(ITERS, 128.0, out=out2[b])
            stream.wait_stream(s_cmp)
            # the transform code as the reference serialises it (.mns, bitstream.py:130-205), packed on
            # the GPU; its size is fixed for this image (deterministic encode), measured in the warm-up
            packed, _ = mns.write_stream_device(code.records, n_rec, W, H, W, H, True, True)
            keep[b] = packed
            comp[i].record(stream)
            with torch.cuda.stream(s_out):  # D2H of step i: the decoded image and the code
                s_out.wait_event(comp[i])
                out_host2[b].copy_(out2[b], non_blocking=True)
                mns_host2[b].copy_(packed[:n_mns], non_blocking=True)
                d2h[i].record(s_out)
        stream.wait_event(d2h[k - 1])
        t1.record(stream)
        barrier()
        ms = t0.elapsed_time(t1)
        if world > 1:
            m = torch.tensor([ms], device=dev)
            dist.all_reduce(m, op=dist.ReduceOp.MAX)
            ms = float(m.item())
        return ms

    for _ in range(args.warmup):
        step()
    stream.wait_stream(s_cmp)
    n_rec = code.n_records()
    _, bits_t = mns.write_stream_device(code.records, n_rec, W, H, W, H, True, True)
    n_mns = (int(bits_t.item()) + 7) // 8  # .mns bytes of this strip's code
    mns_host2 = [torch.empty(n_mns, dtype=torch.uint8).pin_memory() for _ in range(2)]
    keep = [None, None]
    timed_e2e(2)
    barrier()
    # two steps in flight (N = 1): a second code / decoder state on a second high-priority stream, so
    # one step's kernels fill the SMs the other's pass tails leave idle (every step still encodes,
    # compacts and decodes the whole image into its own buffers; both streams join inside the timed
    # region).  N > 1 keeps one step in flight (its NCCL halo exchanges stay in one order).
    pipe = None
    if world == 1 and not args.no_pipeline:
        code_b = mns.DeviceCode(torch.empty(64 * n_roots, dtype=torch.int64, device=dev),
                                torch.empty(n_roots + 1, dtype=torch.int32, device=dev),
                                torch.zeros(1, dtype=torch.int64, device=dev), W, H, 1, r0, r1,
                                unit_map=torch.empty(8 * n_roots, dtype=torch.int32, device=dev), map_form=1)
        dec_b = sharding.StripDecoder(code_b, H, W, r0, r1, rank, world, lattice=True)
        hp = torch.cuda.Stream.priority_range()[1]
        pipe = [(code, dec, stream, s_cmp), (code_b, dec_b, torch.cuda.Stream(priority=hp), torch.cuda.Stream())]

        def pstep(j):
            c_, d_, s_, sc_ = pipe[j]
            with torch.cuda.stream(s_):
                sc_.wait_stream(s_)
                mns.encode_device(img, cfg, root_rows=(r0, r1), height=H, out=c_, compact_stream=sc_)
                d_.run(ITERS, 128.0)
                s_.wait_stream(sc_)

        def timed_pipe(k):
            for j in range(2):
                pstep(j)  # warm the second set
            barrier()
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record(stream)
            pipe[1][2].wait_event(t0)
            for i in range(k):
                pstep(i % 2)
            stream.wait_stream(pipe[1][2])
            t1.record(stream)
            barrier()
            return t0.elapsed_time(t1)

    with ClockSampler(local_rank) as clk:
        ms = timed_pipe(args.steps) if pipe else timed(args.steps, False)[0]
    # the per-kernel breakdown (and the one-step-in-flight latency) from a serial run with events
    ms_serial, evs = timed(args.steps, False, record=True)
    ms_step = ms / args.steps
    blocks = H * W / 64
    value = blocks / (ms_step / 1e3)
    # component times (device events; per step averages over the timed steps)
    enc_ms = float(np.mean([e[0].elapsed_time(e[1]) for e in evs]))
    dec_ms = float(np.mean([e[1].elapsed_time(e[3]) for e in evs]))
    n_launch = dec.launches(ITERS)
    # steady-state passes: not the first (flat start, reads nothing) nor the last (uint8 output)
    # (the median: the low-priority record compaction shares the SMs with one of them)
    mid = [e[2][i][0].elapsed_time(e[2][i][1]) for e in evs for i in range(1, n_launch - 1)]
    pass_ms = float(np.median(mid))
    pass_ms_each = [float(np.mean([e[2][i][0].elapsed_time(e[2][i][1]) for e in evs])) for i in range(n_launch)]
    own_px = 16 * (r1 - r0) * W
    n_leaves = int(code.count.item())

    # multi-GPU: the same step with the final code gather to rank 0
    gather = None
    if world > 1:
        def step_gather():
            step()
            code.join()
            sharding.gather_codes(code.records, code.count, code.root_offsets, rank, world)

        for _ in range(2):
            step_gather()
        barrier()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record()
        for _ in range(args.steps):
            step_gather()
        g1.record()
        barrier()
        gms = g0.elapsed_time(g1) / args.steps
        m = torch.tensor([gms], device=dev)
        dist.all_reduce(m, op=dist.ReduceOp.MAX)
        gms = float(m.item())
        gather = {"ms_per_step": gms, "blocks_per_s": H * W / 64 / (gms / 1e3),
                  "note": "step + gather of every strip's records and root offsets to rank 0 (size all_gather, "
                          "then point-to-point sends over NCCL)"}

    # e2e through the public device API with host buffers: every step copies its image from pinned host
    # memory and its decoded image back; copies of steps k+1 / k-1 overlap step k's kernels on two copy
    # streams (double-buffered device image and output), all inside the timed region
    ms_e2e = timed_e2e(args.steps)
    e2e_value = blocks / (ms_e2e / args.steps / 1e3)

    # full-search component (config c4 identity + isometries) on rank 0 only, informational
    fs = None
    if rank == 0 and not args.no_search:
        from paper_1501_02894_b200.synth import config_image

        c4 = torch.from_numpy(config_image("c4")).to(dev)
        fs = {}
        for n_iso in (1, 8):
            for _ in range(2):
                mns.full_search_device(c4, 8, 1, n_iso)
            torch.cuda.synchronize()
            runs = []
            for _ in range(5):  # median of 5 device-timed calls
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                mns.full_search_device(c4, 8, 1, n_iso)
                b.record()
                torch.cuda.synchronize()
                runs.append(a.elapsed_time(b))
            pairs = 4096 * 497 * 497 * n_iso
            ms = float(np.median(runs))
            tf = 2 * 64 * pairs / (ms / 1e3) / 1e12
            tpk, tsrc, tsus = tensor_peak()
            fs[f"iso{n_iso}"] = {"config": f"c4 512^2 B=8 stride 1, {n_iso} isometr{'y' if n_iso == 1 else 'ies'}",
                                 "pair_evals": pairs, "ms": ms, "pair_evals_per_s": pairs / (ms / 1e3),
                                 "effective_tflops": tf, "tensor_peak_tflops": tpk, "tensor_peak_source": tsrc,
                                 "frac_of_tensor_peak": tf / tpk,
                                 "frac_of_sustained_peak": tf / tsus if tsus else None}
        for radius, n_iso in ((4, 1), (32, 1), (32, 8)):  # encoder.py:312-347 local search (+-4 identity =
            # the reference, CUDA cores; +-32 x 8 isometries is the config-c4 extension, windowed tcgen05 GEMM)
            for _ in range(2):
                mns.local_search_device(c4, radius, n_iso=n_iso)
            torch.cuda.synchronize()
            runs = []
            for _ in range(5):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                mns.local_search_device(c4, radius, n_iso=n_iso)
                b.record()
                torch.cuda.synchronize()
                runs.append(a.elapsed_time(b))
            ms = float(np.median(runs))
            pairs = 4096 * (2 * radius + 1) ** 2 * n_iso
            fs[f"local{radius}" + ("" if n_iso == 1 else f"_iso{n_iso}")] = {
                "config": f"c4 512^2 B=8 local search +-{radius}, {n_iso} isometr{'y' if n_iso == 1 else 'ies'}",
                "pair_evals": pairs, "ms": ms, "pair_evals_per_s": pairs / (ms / 1e3)}

    small = None if args.no_small else small_configs(dev, rank, world)
    next_rows = None
    if not args.no_small and rank == 0:
        next_rows = next_rows_components(dev, code, W, H, r0, r1, whole=world == 1)

    # config c4 as SURVEY 8(e) shards it: ranges split across ranks (pool replicated, no data-path
    # collective), then the all-gather of the 8-byte per-range results; max over ranks
    c4_split = None
    if not args.no_search:
        from paper_1501_02894_b200.synth import config_image

        c4 = torch.from_numpy(config_image("c4")).to(dev)
        c4_split = {}
        for n_iso in (1, 8):
            fn = lambda a, b, n_iso=n_iso: mns.full_search_device(c4, 8, 1, n_iso, ranges=(a, b))  # noqa: E731
            for _ in range(2):
                sharding.search_sharded(fn, 4096, rank, world)
            barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            reps = 5
            for _ in range(reps):
                sharding.search_sharded(fn, 4096, rank, world)
            b.record()
            barrier()
            ms = a.elapsed_time(b) / reps
            if world > 1:
                m = torch.tensor([ms], device=dev)
                dist.all_reduce(m, op=dist.ReduceOp.MAX)
                ms = float(m.item())
            pairs = 4096 * 497 * 497 * n_iso
            c4_split[f"iso{n_iso}"] = {"ms": ms, "pair_evals_per_s": pairs / (ms / 1e3), "ranks": world,
                                       "note": "ranges split across ranks + all_gather of (domain, isometry, o, code)"}

    # the benchmarked output, read back after timing for the parity check (one more untimed step)
    final = None
    if not args.no_parity:  # every rank steps (the decode exchanges halos); rank 0 checks its strip
        step()
        stream.wait_stream(s_cmp)
        torch.cuda.synchronize()
    if rank == 0 and not args.no_parity:
        n_rec = int(code.count.item())
        final = {"rec": code.records[:n_rec].cpu().numpy().view(np.uint64),
                 "offs": code.root_offsets.cpu().numpy(), "out": dec.out.cpu().numpy()}

    if rank != 0:
        return
    hbm, which = peaks()
    # state read + written per steady-state pass: the fp32 lattice (W/2 x H/2) of t and of t+2 in lattice
    # mode, else the fp32 raster of t and of t+2
    algo = (2.0 if dec.lattice else 8.0) * own_px
    kname = "decode_pair_lat_kernel" if dec.lattice else "decode_pair_kernel"
    achieved = algo / (pass_ms / 1e3) / 1e9
    cpu_v, cpu_dt, oracle_result = (None, None, None)
    if world == 1 and not args.no_cpu:
        from oracle import oracle as O

        cpu_v, cpu_dt, oracle_result = cpu_sample(img_np, args.cpu_baseline_rows, O.default_threads(), keep=True)
        if args.cpu_baseline_rows != IMG:
            oracle_result = None
    parity = None
    if not args.no_parity:
        parity = parity_check(img_np, final["rec"], final["offs"], final["out"], r0, r1, oracle_result)
    launches_per_step = 2 + n_launch  # encode + compaction kernels + decode passes (+ memsets, not kernels)
    line = {
        "metric": METRIC, "value": value, "unit": "blocks/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u8/int32 encode, fp32 decode", "data": "synthetic",
        "config": {"workload": "c5: MNS encode (16->8->4, e3=inf) + 10-sweep decode, 16384^2 uint8, sigma 10, "
                               "24 blobs, seed 5", "image": f"{IMG}x{IMG}", "parallelism": f"strips{world}",
                   "l2": "inputs (256 MiB image, 1 GiB fp32 rasters) exceed the 126 MB L2",
                   "steps_in_flight": (2 if pipe else 1)},
        "components": {"steps_in_flight": 2 if pipe else 1, "latency_ms_per_step": ms_serial / args.steps,
                       "encode_ms": enc_ms, "encode_blocks_per_s": blocks / world / (enc_ms / 1e3),
                       "encode_note": "encoder kernel; the record compaction runs on a second stream, "
                                      "overlapping the decode, and is joined before the step ends",
                       "decode_ms": dec_ms, "decode_mpix_per_s": own_px / (dec_ms / 1e3) / 1e6,
                       "pass_ms": pass_ms, "pass_ms_each": pass_ms_each, "sweeps_per_pass": 2,
                       "sweep_ms_effective": pass_ms / 2,
                       "leaves_rank0": n_leaves, "full_search": fs, "c4_range_split": c4_split,
                       "small_configs": small,
                       "with_code_gather": gather,
                       "next_rows": next_rows},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                     "traffic": measured_traffic(kname) if world == 1 else None,
                     "algorithmic_bytes": algo, "kernel": f"{kname} (steady-state pass = 2 sweeps)",
                     "peak_source": which,
                     "limiter": ("instruction issue (ncu: ~77% issue slots busy, DRAM ~1.02x the algorithmic "
                                 "bytes; profiles/r2/ncu_dec_r2_blockmap.txt)") if dec.lattice else "latency",
                     # informational, NOT a roofline fraction: the bytes SURVEY 8(d)'s raster-state formula
                     # (8 B/px per sweep) would move at this speed; the lattice state moves 2 B/px per pass
                     "raster_equivalent_gbs": 2 * 8 * own_px / (pass_ms / 1e3) / 1e9},
        "cpu_baseline": ({"value": cpu_v, "unit": "blocks/s", "cores": O.default_threads(), "kind": "port",
                          "sample": f"c5 rows 0..{args.cpu_baseline_rows - 1} encoded + {ITERS}-sweep decoded as its own "
                                    f"image by the fp64 oracle ({cpu_dt:.2f} s)"} if cpu_v else None),
        "e2e": {"value": e2e_value, "unit": "blocks/s", "h2d_bytes_per_step": int(host.numel()) * world,
                "d2h_bytes_per_step": (int(out_host.numel()) + n_mns) * world,
                "note": "per step: image H2D (pinned), encode, the code packed to .mns on the GPU and copied "
                        "back, decode, decoded image D2H; copies of neighbouring steps overlap on two copy "
                        "streams (double-buffered)"},
        "parity": parity,
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-rows", type=int, default=2048, help="rows per --impl reference step (bounded sample)")
    ap.add_argument("--no-pipeline", action="store_true",
                    help="N = 1: one step in flight (default: two, on two streams with their own buffers)")
    ap.add_argument("--no-python-ref", action="store_true",
                    help="--impl reference: skip the pure-Python reference timings (baseline/_ref)")
    ap.add_argument("--cpu-baseline-rows", type=int, default=IMG,
                    help="rows of the c5 image the cpu_baseline leg encodes + decodes (default: all of it)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-parity", action="store_true", help="skip the post-timing oracle check of the output")
    ap.add_argument("--no-search", action="store_true")
    ap.add_argument("--no-small", action="store_true", help="skip the c1/c2 graph-replay latency and c3 batch legs")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    from paper_1501_02894_b200.synth import config_image

    if args.impl == "reference":
        if rank != 0:
            return
        run_reference(args, config_image("c5"))
        return
    import torch.distributed as dist

    if world > 1:
        import torch

        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, config_image("c5"), rank, world, local_rank)
    finally:
        if world > 1:
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
