"""Exact fp64 decode (stop_delta > 0 path) timing on c2 and c5 codes."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1501_02894_b200 as mns  # noqa: E402
from paper_1501_02894_b200.synth import config_image  # noqa: E402

for name in ("c2", "c5"):
    img = torch.from_numpy(config_image(name)).cuda()
    code = mns.encode_device(img, mns.EncoderConfig(e3=math.inf))
    for stop in (0.5, 0.0):
        out, it, _ = mns.decode_device(code, iters=10, stop_delta=stop if stop else 1e-300)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            out, it, _ = mns.decode_device(code, iters=10, stop_delta=stop if stop else 1e-300)
        e1.record()
        torch.cuda.synchronize()
        print(name, "stop", stop, "sweeps", int(it.item()), f"{e0.elapsed_time(e1) / 3:.3f} ms", flush=True)
