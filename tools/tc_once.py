import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1501_02894_b200 as mns
from paper_1501_02894_b200.synth import synth_image
px = synth_image(512, 4); img = torch.from_numpy(px).cuda()
n_iso = int(sys.argv[1]) if len(sys.argv) > 1 else 1
for _ in range(2): mns.full_search_device(img, 8, 1, n_iso)
torch.cuda.synchronize(); print("ok")
