import sys, os, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
CASE = r'''
import sys, math, numpy as np, torch
sys.path.insert(0, "{root}")
import paper_1501_02894_b200 as mns
from paper_1501_02894_b200.synth import synth_image
n, mode, e, rl = {n}, "{mode}", {e}, {rl}
px = synth_image(n, 1)
img = torch.from_numpy(px).cuda()
code = mns.encode_device(img, mns.EncoderConfig(e1=e, e2=e, e3=e, mode=mode), root_level=rl)
torch.cuda.synchronize()
print("ok", n, mode, e, rl, code.n_records(), flush=True)
'''
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for n, mode, e, rl in [(128, "no_search", 8.0, 1), (128, "mns", "math.inf", 1), (128, "mns", 8.0, 2),
                       (128, "mns", 8.0, 1), (256, "mns", 8.0, 1), (64, "mns", 8.0, 1), (128, "mns", 1.0, 1),
                       (256, "no_search", 1.0, 1), (256, "mns", 30.0, 1)]:
    code = CASE.format(root=root, n=n, mode=mode, e=e, rl=rl)
    try:
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=25)
        print(n, mode, e, rl, "->", (r.stdout.strip() or r.stderr.strip()[-300:]), flush=True)
    except subprocess.TimeoutExpired:
        print(n, mode, e, rl, "-> HANG", flush=True)
