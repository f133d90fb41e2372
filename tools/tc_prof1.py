"""Three identity-only c4 full searches (for an ncu launch list)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1501_02894_b200 as mns
from paper_1501_02894_b200.synth import config_image
c4 = torch.from_numpy(config_image("c4")).cuda()
for _ in range(3):
    mns.full_search_device(c4, 8, 1, int(os.environ.get("N_ISO", "1")))
torch.cuda.synchronize()
