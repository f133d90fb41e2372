"""c2 with 8 isometries (BASELINE configs[1]): one encode + 10-sweep decode after warm-up, for the launch list
(ncu --metrics gpu__time_duration.sum ...) and a CUDA-event time."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1501_02894_b200 as mns  # noqa: E402
from paper_1501_02894_b200.synth import config_image  # noqa: E402

img = torch.from_numpy(config_image("c2")).cuda()
cfg = mns.EncoderConfig(e3=math.inf)
for _ in range(3):
    c = mns.encode_device(img, cfg, n_iso=8)
    mns.decode_device(c, iters=10, stop_delta=0.0)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
ev[0].record()
c = mns.encode_device(img, cfg, n_iso=8)
ev[1].record()
mns.decode_device(c, iters=10, stop_delta=0.0)
ev[2].record()
torch.cuda.synchronize()
print(f"c2 iso8: encode {ev[0].elapsed_time(ev[1]) * 1e3:.1f} us, decode {ev[1].elapsed_time(ev[2]) * 1e3:.1f} us, "
      f"{c.n_records()} leaves")
