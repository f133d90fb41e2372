"""One c5 encode (16384^2, 16->8->4, e3=inf) after warm-up: the ncu target for the encoder kernel
(ncu -k regex:mns_encode_kernel --launch-skip 2 -c 1 ...)."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1501_02894_b200 as mns  # noqa: E402
from paper_1501_02894_b200.synth import config_image  # noqa: E402

img = torch.from_numpy(config_image(os.environ.get("CFG", "c5"))).cuda()
cfg = mns.EncoderConfig(e3=math.inf)
for _ in range(3):
    code = mns.encode_device(img, cfg)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
for _ in range(20):
    mns.encode_device(img, cfg, out=code)
ev[1].record()
torch.cuda.synchronize()
print(f"encode {ev[0].elapsed_time(ev[1]) / 20:.4f} ms")
