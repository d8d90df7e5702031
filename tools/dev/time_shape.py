"""Dev: device time of one matching shape on a config's image (CUDA events, L2 flushed)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2103_10765_b200 as g
from synth import CONFIGS, config_images
name, P, S, r, K = sys.argv[1].split(":")
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1
z = torch.from_numpy(config_images(CONFIGS[name])[:B].copy()).cuda()
z = z[0].contiguous() if B == 1 else z
flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
for _ in range(3):
    g.block_match(z, int(P), int(S), int(r), int(K), None, check=False)
ts = []
for _ in range(10):
    flush.zero_()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); g.block_match(z, int(P), int(S), int(r), int(K), None, check=False); e.record()
    torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
print(sys.argv[1], B, "median %.3f ms" % np.median(ts))
