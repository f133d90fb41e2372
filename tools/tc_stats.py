import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1501_02894_b200 as mns
from paper_1501_02894_b200 import _native as N
from paper_1501_02894_b200.synth import synth_image
px = synth_image(512, 4); img = torch.from_numpy(px).cuda()
L = N.load_library()
st = (ctypes.c_ulonglong * 4)()
for n_iso in (1, 8):
    mns.full_search_device(img, 8, 1, n_iso); torch.cuda.synchronize()
    L.mns_tc_stats(st)
    mns.full_search_device(img, 8, 1, n_iso); torch.cuda.synchronize()
    L.mns_tc_stats(st)
    el = 4096 * n_iso * 247009
    print(f"n_iso={n_iso}: warp-chunks={st[0]} l1pass={st[1]} ({st[1]/max(1,st[0])*100:.2f}%) l2 pairs={st[2]} ({st[2]/el*1e6:.1f} ppm) exact={st[3]} ({st[3]/el*1e6:.2f} ppm)")
