import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1501_02894_b200 as mns
from paper_1501_02894_b200.synth import synth_image
def run(px, B, n_iso, step=1):
    img = torch.from_numpy(np.ascontiguousarray(px)).cuda()
    torch.cuda.synchronize(); t = time.time()
    out = mns.full_search_device(img, B, step, n_iso)
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in out.items()}, time.time() - t
cases = [(synth_image(512, 4)[:64, :64], 8, 1), (synth_image(512, 4)[:128, :128], 8, 8), (synth_image(512, 4)[:96, :96], 4, 1),
         (synth_image(512, 4)[:64, :64], 2, 8), (np.full((64, 64), 42, np.uint8), 8, 1), (np.full((64, 64), 255, np.uint8), 8, 1)]
for px, B, n_iso in cases:
    os.environ["MNS_SEARCH_CUDA_CORES"] = "0"
    a, ta = run(px, B, n_iso)
    os.environ["MNS_SEARCH_CUDA_CORES"] = "1"
    b, tb = run(px, B, n_iso)
    same = all(np.array_equal(a[k], b[k]) for k in a)
    print(px.shape, B, n_iso, "tc==cc", same, f"tc {ta*1e3:.1f} ms cc {tb*1e3:.1f} ms", flush=True)
    if not same:
        bad = np.nonzero(a["dom"] != b["dom"])[0][:5]
        print("  first diffs", bad, a["dom"][bad], b["dom"][bad], a["iso"][bad], b["iso"][bad])
os.environ["MNS_SEARCH_CUDA_CORES"] = "0"
px = synth_image(512, 4)
for n_iso in (1, 8):
    run(px, 8, n_iso)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    img = torch.from_numpy(px).cuda()
    e0.record(); mns.full_search_device(img, 8, 1, n_iso); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1); pairs = 4096 * 497 * 497 * n_iso
    print(f"c4 512^2 B=8 n_iso={n_iso}: {ms:.3f} ms  {pairs/ms/1e9:.3f} Gpair/s  {2*64*pairs/ms/1e9:.1f} TFLOP/s", flush=True)
