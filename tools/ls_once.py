"""c4 local search, tensor-core path, +-R x n_iso (argv), after warm-up: ncu target."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1501_02894_b200 as mns  # noqa: E402
from paper_1501_02894_b200.synth import config_image  # noqa: E402

R, n_iso = int(sys.argv[1]), int(sys.argv[2])
img = torch.from_numpy(config_image("c4")).cuda()
for _ in range(3):
    mns.local_search_device(img, R, n_iso=n_iso)
torch.cuda.synchronize()
mns.local_search_device(img, R, n_iso=n_iso)
torch.cuda.synchronize()
