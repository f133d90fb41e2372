for lib in tools/dbg/*.so; do
  MNS_B200_LIB=$PWD/$lib timeout 30 python -c "
import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_1501_02894_b200 as mns
from paper_1501_02894_b200.synth import synth_image
px = synth_image(128, 1)
code = mns.encode_device(torch.from_numpy(px).cuda(), mns.EncoderConfig())
torch.cuda.synchronize(); print('ok', code.n_records())
" > /tmp/o.txt 2>&1; echo "$lib rc=$? $(tail -1 /tmp/o.txt)"
done
