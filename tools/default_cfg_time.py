"""c5 with the reference's default EncoderConfig (E = 8 at every level, 16->8->4->2: 2x2 leaves, so the
decoder runs on fp32 rasters): encode and 10-sweep decode device times."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1501_02894_b200 as mns  # noqa: E402
from paper_1501_02894_b200.synth import config_image  # noqa: E402

img = torch.from_numpy(config_image("c5")).cuda()
cfg = mns.EncoderConfig()
for _ in range(2):
    code = mns.encode_device(img, cfg)
    out, it, _ = mns.decode_device(code, iters=10, stop_delta=0.0)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
ev[0].record()
code = mns.encode_device(img, cfg)
ev[1].record()
out, it, _ = mns.decode_device(code, iters=10, stop_delta=0.0)
ev[2].record()
torch.cuda.synchronize()
print(f"default config c5: {code.n_records()} leaves, min leaf {code.min_leaf}; encode {ev[0].elapsed_time(ev[1]):.3f} ms, "
      f"decode (10 sweeps) {ev[1].elapsed_time(ev[2]):.3f} ms")
