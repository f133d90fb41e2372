"""c5 step throughput: steps one after another on one stream vs two steps in flight on two streams
(each with its own code and decoder state), CUDA events around K steps."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1501_02894_b200 as mns  # noqa: E402
from paper_1501_02894_b200 import sharding  # noqa: E402
from paper_1501_02894_b200.synth import config_image  # noqa: E402

img = torch.from_numpy(config_image("c5")).cuda()
H, W = img.shape
n_roots = (H // 16) * (W // 16)
hp = torch.cuda.Stream.priority_range()[1]
NS = int(os.environ.get("NSETS", "2"))
sets = []
for _ in range(NS):
    code = mns.DeviceCode(torch.empty(64 * n_roots, dtype=torch.int64, device="cuda"),
                          torch.empty(n_roots + 1, dtype=torch.int32, device="cuda"),
                          torch.zeros(1, dtype=torch.int64, device="cuda"), W, H, 1, 0, H // 16,
                          unit_map=torch.empty(8 * n_roots, dtype=torch.int32, device="cuda"), map_form=1)
    dec = sharding.StripDecoder(code, H, W, 0, H // 16, 0, 1, lattice=True)
    sets.append((code, dec, torch.cuda.Stream(priority=hp), torch.cuda.Stream()))
cfg = mns.EncoderConfig(e3=math.inf)


def step(j):
    code, dec, s, c = sets[j]
    with torch.cuda.stream(s):
        c.wait_stream(s)
        mns.encode_device(img, cfg, root_rows=(0, H // 16), height=H, out=code, compact_stream=c)
        dec.run(10, 128.0)
        s.wait_stream(c)


def run(k, pipelined):
    main = torch.cuda.current_stream()
    for _, _, s, _ in sets:
        s.wait_stream(main)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _, _, s, _ in sets:
        s.wait_event(a)
    for i in range(k):
        j = i % NS if pipelined else 0
        if not pipelined and i:
            pass
        step(j)
    for _, _, s, _ in sets:
        main.wait_stream(s)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / k


for _ in range(3):
    for j in range(NS):
        step(j)
torch.cuda.synchronize()
for rep in range(2):
    print(f"serial {run(20, False):.4f} ms/step  pipelined {run(20, True):.4f} ms/step", flush=True)
