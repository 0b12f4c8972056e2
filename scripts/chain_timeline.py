"""Per-CTA timeline of a PDL chain of back-to-back W4A8 GEMMs (rotated cold
weight replicas, replayed from one CUDA graph, as bench.py times a point).

For every launch of the chain: CTA start / PDL-release / first weight stage /
first MMA / epilogue end (min, median, max over CTAs, us relative to the first
CTA of the chain), and the steady-state period between consecutive launches.
Needs the developer build with timeline stamps (build.py --timeline).

    python scripts/chain_timeline.py --shape 4096x4096 --m 1 [--len 6] [--cfg '{}']
"""
import argparse
import json
import os
import sys

os.environ["QQQ_TIMELINE_LIB"] = "1"
import numpy as np  # noqa: E402
import torch  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench as B  # noqa: E402
import paper_2406_09904_b200 as Q  # noqa: E402
from paper_2406_09904_b200 import gemm as G  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="4096x4096")
ap.add_argument("--m", type=int, default=1)
ap.add_argument("--scheme", default="per-group")
ap.add_argument("--cfg", default="{}")
ap.add_argument("--len", type=int, default=6)
ap.add_argument("--fused", action="store_true", help="the fused smooth-quant launch (quant_linear_smoothed)")
a = ap.parse_args()
k, n = map(int, a.shape.split("x"))
dev = torch.device("cuda", 0)
qw, fused, prep = B.make_weights(k, n, a.scheme, 0, dev)
L = a.len
preps = [prep] + [B.clone_prep(prep) for _ in range(L - 1)]
x = torch.randn((a.m, k), dtype=torch.float16, device=dev)
aq = Q.quant_act_per_token(x)
y = torch.empty((a.m, n), dtype=torch.float16, device=dev)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
dbgs = [torch.zeros((1024, 192), dtype=torch.int64, device=dev) for _ in range(L)]
cfg = json.loads(a.cfg)


from paper_2406_09904_b200 import pipeline as P  # noqa: E402
from paper_2406_09904_b200 import _lib  # noqa: E402
sm = torch.ones(k, dtype=torch.float64, device=dev)
sm[::8] = 1.5
rc = Q.smoothing_reciprocal(sm)


def launch():
    for i in range(L):
        if a.fused:
            # (the dbg timeline buffer rides in the plan config)
            P.quant_linear_smoothed(x, sm, rc, preps[i], n, check=False, y_out=y, cfg=dict(cfg, dbg=dbgs[i]))
        else:
            G.run_gemm(aq, preps[i], n, False, y_out=y, cfg=dict(cfg, dbg=dbgs[i]))


launch()
torch.cuda.synchronize()
graph = torch.cuda.CUDAGraph()
with torch.cuda.graph(graph):
    launch()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for rep in range(3):
    for d in dbgs:
        d.zero_()
    flush.zero_()
    torch.cuda.synchronize()
    s.record()
    graph.replay()
    e.record()
    torch.cuda.synchronize()
info = G.plan_info(prep.mode, a.m, n, k, cfg or None)
print(f"{a.shape} M={a.m} {a.scheme} plan={info} chain={L} graph {s.elapsed_time(e) * 1e3:.2f} us "
      f"({s.elapsed_time(e) * 1e3 / L:.2f} us/GEMM incl. first-launch latency)")
ds = [d.cpu().numpy().astype(np.int64) for d in dbgs]
t0 = min(d[d[:, 0] > 0, 0].min() for d in ds)
SLOTS = [("start", 0), ("dep_wait", 3), ("x_issued", 181), ("full0", 4), ("conv0", 80), ("mma_xfull0", 96), ("mma0", 20), ("mma3", 23), ("conv3", 83),
         ("accfull0", 36), ("cs_own", 150), ("cs_recv", 151), ("cs_add", 152), ("cs_done", 153), ("loop_end", 154), ("epi_end", 63), ("exit", 42)]
if a.fused:
    SLOTS = [("start", 0), ("q_start", 176), ("q_phaseA", 177), ("q_phaseB", 178), ("q_all", 179), ("x_wait", 180),
             ("full0", 4), ("conv0", 80), ("mma_xfull0", 96), ("mma0", 20), ("accfull0", 36), ("epi_end", 63), ("exit", 42)]


def stat(d, sl):
    v = d[:, sl]
    v = v[v > 0]
    if v.size == 0:
        return "      -         "
    r = (v - t0) / 1e3
    return f"{r.min():6.2f}/{np.median(r):6.2f}/{r.max():6.2f}"


print("launch  ctas  " + "  ".join(f"{nm:>20s}" for nm, _ in SLOTS) + "   (min/med/max us)")
ends = []
for i, d in enumerate(ds):
    d = d[d[:, 0] > 0]
    print(f"{i:6d}  {len(d):4d}  " + "  ".join(f"{stat(d, sl):>20s}" for _, sl in SLOTS))
    ends.append((d[:, 42][d[:, 42] > 0].max() - t0) / 1e3)
print("last-CTA-exit deltas (us):", " ".join(f"{ends[i] - ends[i - 1]:.2f}" for i in range(1, L)))
# the 6 latest-exiting CTAs of the middle launch: every stamp, and the SM they ran on
mid = ds[L // 2]
mid = mid[mid[:, 0] > 0]
order = np.argsort(-mid[:, 42])
print(f"launch {L // 2}: latest-exiting CTAs (sm, then us per stamp)")
for r in order[:6]:
    print(f"  sm={int(mid[r, 191]):3d} " + " ".join(f"{nm}={(mid[r, sl] - t0) / 1e3:.2f}" for nm, sl in SLOTS if mid[r, sl] > 0))
# SM sharing: how many CTAs of launches L//2-1 and L//2+1 ran on the same SMs as the latest CTAs
for j in (L // 2 - 1, L // 2 + 1):
    o = ds[j][ds[j][:, 0] > 0]
    sms = set(int(v) for v in o[:, 191])
    print(f"  launch {j}: {len(o)} CTAs on {len(sms)} SMs; latest-6 SMs shared: "
          f"{sum(int(mid[r, 191]) in sms for r in order[:6])}/6")
