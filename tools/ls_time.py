"""Median-of-5 device time of the c4 local search (+-4 / +-32, 1 and 8 isometries)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1501_02894_b200 as mns  # noqa: E402
from paper_1501_02894_b200.synth import config_image  # noqa: E402

img = torch.from_numpy(config_image("c4")).cuda()
for radius, n_iso in ((4, 1), (32, 1), (4, 8), (32, 8)):
    for _ in range(2):
        mns.local_search_device(img, radius, n_iso=n_iso)
    torch.cuda.synchronize()
    runs = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        mns.local_search_device(img, radius, n_iso=n_iso)
        e1.record()
        torch.cuda.synchronize()
        runs.append(e0.elapsed_time(e1))
    pairs = 4096 * (2 * radius + 1) ** 2 * n_iso
    ms = float(np.median(runs))
    print(f"local +-{radius} iso{n_iso}: {ms:.3f} ms  {pairs / ms * 1e3:.3e} pairs/s", flush=True)
