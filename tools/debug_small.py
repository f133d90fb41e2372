import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
def log(*a):
    print(f"[{time.time()-T0:7.2f}]", *a, flush=True)
T0 = time.time()
import numpy as np
log("numpy")
import torch
log("torch", torch.cuda.is_available())
import paper_1501_02894_b200 as mns
from paper_1501_02894_b200.synth import synth_image
log("pkg")
for n in (int(a) for a in sys.argv[1:]):
    px = synth_image(n, 1)
    img = torch.from_numpy(px).cuda()
    torch.cuda.synchronize(); log("h2d", n)
    code = mns.encode_device(img, mns.EncoderConfig())
    log("launched enc")
    torch.cuda.synchronize(); log("enc done", code.n_records())
    out, it, _ = mns.decode_device(code, 8, 0.0)
    torch.cuda.synchronize(); log("dec done", int(out.float().mean().item()))
from oracle import oracle as O
log("oracle imported")
rec, _ = O.encode_quadtree_records(px, (8, 8, 8), 16.0, True)
log("oracle enc", len(rec))
