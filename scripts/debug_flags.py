import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench as B
import paper_2406_09904_b200 as Q
from paper_2406_09904_b200 import _lib
dev = torch.device("cuda", 0)
qw, fused, prep = B.make_weights(4096, 4096, "per-group", 0, dev)
print("mode", prep.mode)
s = fused.s_star.float().cpu().numpy()
print("s* min/max", s.min(), s.max())
sv = s.astype(np.float64)
r_lo = (-8 * sv + 1152).astype(np.float16).astype(np.float64)
r_hi = (7 * sv + 1152).astype(np.float16).astype(np.float64)
print("np inadmissible", int(((r_lo < 1025) | (r_hi > 1279)).sum()), "tiny", int((sv < 2**-10).sum()))
lib = _lib.load()
sc = torch.empty(lib.qqq_repacked_scale_bytes(4096, 4096, 128) // 2, dtype=torch.float16, device=dev)
flags = torch.zeros(1, dtype=torch.int32, device=dev)
rc = lib.qqq_repack_scales(_lib.ptr(fused.s_star.contiguous()), 4096, 4096, 128, _lib.ptr(sc), _lib.ptr(flags), _lib.stream_of(dev))
torch.cuda.synchronize()
print("rc", rc, "flags", int(flags.item()))
