import sys, torch
sys.path.insert(0, '.')
import paper_1501_02894_b200 as mns
from paper_1501_02894_b200.synth import config_image
c4 = torch.from_numpy(config_image("c4")).cuda()
for _ in range(3):
    mns.full_search_device(c4, 8, 1, 8)
torch.cuda.synchronize()
