"""Median-of-5 device time of the c4 full search (identity and 8 isometries) for the loaded library."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1501_02894_b200 as mns
from paper_1501_02894_b200.synth import config_image
img = torch.from_numpy(config_image("c4")).cuda()
for n_iso in (1, 8):
    for _ in range(2): mns.full_search_device(img, 8, 1, n_iso)
    torch.cuda.synchronize()
    runs = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); mns.full_search_device(img, 8, 1, n_iso); e1.record(); torch.cuda.synchronize()
        runs.append(e0.elapsed_time(e1))
    print(os.environ.get("MNS_B200_LIB", "prod").split("/")[-1], n_iso, f"{np.median(runs):.3f} ms", [f"{r:.3f}" for r in runs], flush=True)
