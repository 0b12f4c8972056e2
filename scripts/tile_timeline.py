"""One launch's per-CTA timeline, printing a CTA's per-k-block converter /
MMA stamps and its tiles' accumulator / epilogue stamps (developer tool)."""
import argparse, json, os, sys
os.environ["QQQ_TIMELINE_LIB"] = "1"
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench as B
import paper_2406_09904_b200 as Q
from paper_2406_09904_b200 import gemm as G
ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="4096x11008")
ap.add_argument("--m", type=int, default=1024)
ap.add_argument("--cfg", default="{}")
ap.add_argument("--cta", type=int, default=0)
a = ap.parse_args()
k, n = map(int, a.shape.split("x"))
dev = torch.device("cuda", 0)
qw, fused, prep = B.make_weights(k, n, "per-group", 0, dev)
x = torch.randn((a.m, k), dtype=torch.float16, device=dev)
aq = Q.quant_act_per_token(x)
y = torch.empty((a.m, n), dtype=torch.float16, device=dev)
dbg = torch.zeros((1024, 192), dtype=torch.int64, device=dev)
cfg = json.loads(a.cfg)
for _ in range(3):
    dbg.zero_()
    G.run_gemm(aq, prep, n, False, y_out=y, cfg=dict(cfg, dbg=dbg))
    torch.cuda.synchronize()
d = dbg.cpu().numpy().astype(np.int64)
ok = d[:, 0] > 0
t0 = d[ok, 0].min()
print(a.shape, a.m, G.plan_info(prep.mode, a.m, n, k, cfg or None), "ctas", int(ok.sum()))
ends = (d[ok, 42] - t0) / 1e3
print("CTA exit min/med/max us: %.2f %.2f %.2f" % (ends.min(), np.median(ends), ends.max()))
c = d[a.cta]
f = lambda v: "%.2f" % ((v - t0) / 1e3) if v > 0 else "-"
print("cta", a.cta, "start", f(c[0]), "exit", f(c[42]))
print(" kb: w_issue full(w) | x_issue | conv_done mma_xfull mma_issued")
for it in range(16):
    print("  %2d: %s %s | %s | %s %s %s" % (it, f(c[155 + it]), f(c[4 + it]), f(c[112 + it]), f(c[80 + it]), f(c[96 + it]), f(c[20 + it])))
for sg in range(4):
    print(" seg %d: accfull %s epi_done %s" % (sg, f(c[36 + 2 * sg]), f(c[37 + 2 * sg])))
print(" epi chunk tmem-ld done (lead warp, seg 0):", " ".join(f(c[44 + li]) for li in range(16)))
print(" epi loop end %s  stores read %s" % (f(c[154]), f(c[63])))
for li in range(4):
    print("  chunk %d: tmem-ld %s dequant %s wait-read %s sts+fence %s store %s" % (li, f(c[44 + li]), f(c[128 + li]), f(c[132 + li]), f(c[136 + li]), f(c[140 + li])))
