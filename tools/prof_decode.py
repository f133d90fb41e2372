"""c5 decode (bench.py's lattice StripDecoder path, 10 sweeps = 5 passes) after warm-up: the ncu
target for the decoder (ncu -k regex:decode_pair_lat --launch-skip 11 -c 1: a steady pass)."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1501_02894_b200 as mns  # noqa: E402
from paper_1501_02894_b200 import sharding  # noqa: E402
from paper_1501_02894_b200.synth import config_image  # noqa: E402

img = torch.from_numpy(config_image(os.environ.get("CFG", "c5"))).cuda()
H, W = img.shape
n_roots = (H // 16) * (W // 16)
code = mns.DeviceCode(torch.empty(64 * n_roots, dtype=torch.int64, device="cuda"),
                      torch.empty(n_roots + 1, dtype=torch.int32, device="cuda"),
                      torch.zeros(1, dtype=torch.int64, device="cuda"), W, H, 1, 0, H // 16,
                      unit_map=torch.empty(8 * n_roots, dtype=torch.int32, device="cuda"), map_form=1)
dec = sharding.StripDecoder(code, H, W, 0, H // 16, 0, 1, lattice=True)
mns.encode_device(img, mns.EncoderConfig(e3=math.inf), root_rows=(0, H // 16), height=H, out=code)
for _ in range(3):
    dec.run(10, 128.0)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
for _ in range(10):
    dec.run(10, 128.0)
ev[1].record()
torch.cuda.synchronize()
print(f"decode (10 sweeps) {ev[0].elapsed_time(ev[1]) / 10:.4f} ms")
