import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1501_02894_b200 as mns
from paper_1501_02894_b200 import _native as N
from paper_1501_02894_b200.synth import config_image
img = torch.from_numpy(config_image("c4")).cuda()
L = N.load_library()
st = (ctypes.c_ulonglong * 4)()
for R, n_iso in ((4, 1), (32, 1), (4, 8), (32, 8)):
    mns.local_search_device(img, R, n_iso=n_iso); torch.cuda.synchronize(); L.mns_tc_stats(st)
    mns.local_search_device(img, R, n_iso=n_iso); torch.cuda.synchronize(); L.mns_tc_stats(st)
    print(f"R={R} iso={n_iso}: groups={st[0]} l1pass={st[1]} l2={st[2]} exact={st[3]} (per range {st[2]/4096:.1f} l2, {st[3]/4096:.1f} exact)")
