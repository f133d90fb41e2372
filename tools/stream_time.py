"""Device time of the .mns writer and reader on the c5 code (16384^2, 16->8->4)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import math
import numpy as np, torch
import paper_1501_02894_b200 as mns
from paper_1501_02894_b200 import codec
from paper_1501_02894_b200.synth import config_image
img = torch.from_numpy(config_image("c5")).cuda()
code = mns.encode_device(img, mns.EncoderConfig(e3=math.inf))
n = code.n_records()
out, bits = codec.write_stream_device(code.records, n, 16384, 16384, 16384, 16384, True, True)
nb = (int(bits.item()) + 7) // 8
blob = out[:nb].clone()
for _ in range(2):
    c2, st = codec.read_stream_device(blob, True, True, 16384, 16384)
torch.cuda.synchronize()
assert torch.equal(c2.records[:n], code.records[:n]) and int(st[0]) == -1
ts = []
for _ in range(5):
    t0 = time.perf_counter(); codec.read_stream_device(blob, True, True, 16384, 16384); torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
tw = []
for _ in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); codec.write_stream_device(code.records, n, 16384, 16384, 16384, 16384, True, True); b.record()
    torch.cuda.synchronize(); tw.append(a.elapsed_time(b))
print(f"c5 stream {nb/1e6:.1f} MB, {n} leaves: read {np.median(ts)*1e3:.3f} ms (wall, incl. resync round trips) "
      f"= {nb/np.median(ts)/1e9:.1f} GB/s; write {np.median(tw):.3f} ms")
