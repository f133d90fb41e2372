import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1501_02894_b200 as mns
from paper_1501_02894_b200.synth import synth_image
px = synth_image(512, 4); img = torch.from_numpy(px).cuda()
for n_iso in (1, 8):
    for _ in range(2): mns.full_search_device(img, 8, 1, n_iso)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); mns.full_search_device(img, 8, 1, n_iso); e1.record(); torch.cuda.synchronize()
    print(os.environ.get("MNS_B200_LIB", "prod").split("/")[-1], n_iso, f"{e0.elapsed_time(e1):.3f} ms", flush=True)
