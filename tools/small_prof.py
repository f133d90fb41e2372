"""One c1 (256^2, 8->4, 8 sweeps) and one c2 (512^2, 16->8->4, 10 sweeps) encode + decode step after warm-up,
for an ncu launch list of the latency-bound small configs."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1501_02894_b200 as mns
from paper_1501_02894_b200.synth import config_image

cfg = mns.EncoderConfig(e3=math.inf)
for name, rl, iters in (("c1", 2, 8), ("c2", 1, 10)):
    img = torch.from_numpy(config_image(name)).cuda()
    for _ in range(3):
        code = mns.encode_device(img, cfg, root_level=rl)
        mns.decode_device(code, iters=iters, stop_delta=0.0, initial_value=128.0)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push(name)
    code = mns.encode_device(img, cfg, root_level=rl)
    mns.decode_device(code, iters=iters, stop_delta=0.0, initial_value=128.0)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
