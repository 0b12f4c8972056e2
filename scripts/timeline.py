"""Per-CTA in-kernel timeline (%globaltimer stamps) of one W4A8 GEMM launch."""
import argparse, json, os, sys
os.environ["QQQ_TIMELINE_LIB"] = "1"  # the instrumented developer build (build.py --timeline)
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench as B
import paper_2406_09904_b200 as Q
from paper_2406_09904_b200 import gemm as G

NAMES = {0: "start", 1: "setup", 2: "w_issued", 3: "dep_wait", 60: "own_cnt", 61: "contrib_done", 62: "part_ready",
         63: "epi_end"}
for i in range(16):
    NAMES[4 + i] = f"full{i}"
    NAMES[20 + i] = f"mma{i}"
    NAMES[96 + i] = f"mma_xfull{i}"
    NAMES[112 + i] = f"ctl_xissued{i}"
    NAMES[128 + i] = f"mma_issued{i}"
for c in range(16):
    NAMES[44 + c] = f"epi0_c{c}"
    NAMES[64 + c] = f"conv_ae{c}"
    NAMES[80 + c] = f"conv_done{c}"
for sg in range(4):
    NAMES[36 + 2 * sg] = f"accfull{sg}"
    NAMES[37 + 2 * sg] = f"epi_done{sg}"

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="4096x11008")
ap.add_argument("--m", type=int, default=16)
ap.add_argument("--scheme", default="per-group")
ap.add_argument("--cfg", default="{}")
ap.add_argument("--pair", action="store_true", help="two back-to-back launches (PDL overlap); report both")
a = ap.parse_args()
k, n = map(int, a.shape.split("x"))
dev = torch.device("cuda", 0)
qw, fused, prep = B.make_weights(k, n, a.scheme, 0, dev)
x = torch.randn((a.m, k), dtype=torch.float16, device=dev)
aq = Q.quant_act_per_token(x)
y = torch.empty((a.m, n), dtype=torch.float16, device=dev)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
prep2 = G.PreparedWeights(prep.mode, prep.w.clone(), None if prep.sc is None else prep.sc.clone(), prep.group,
                           prep.s_col.clone())
dbg = torch.zeros((1024, 192), dtype=torch.int64, device=dev)
dbg2 = torch.zeros((1024, 192), dtype=torch.int64, device=dev)
def launch():
    G.run_gemm(aq, prep, n, False, y_out=y, cfg=dict(json.loads(a.cfg), dbg=dbg))
    if a.pair:
        G.run_gemm(aq, prep2, n, False, y_out=y, cfg=dict(json.loads(a.cfg), dbg=dbg2))
launch()
torch.cuda.synchronize()
graph = torch.cuda.CUDAGraph()  # the pair is replayed from a graph: no host gap, PDL edges kept
with torch.cuda.graph(graph):
    launch()
for rep in range(3):
    dbg.zero_()
    dbg2.zero_()
    flush.zero_()
    torch.cuda.synchronize()
    graph.replay()
    torch.cuda.synchronize()
if a.pair:
    d1 = dbg.cpu().numpy().astype(np.int64)
    d2 = dbg2.cpu().numpy().astype(np.int64)
    t0 = d1[d1[:, 0] > 0, 0].min()
    for name, d in (("first", d1), ("second", d2)):
        d = d[d[:, 0] > 0]
        st = (d[:, 0] - t0) / 1e3
        en = (d[:, 63] - t0) / 1e3
        print(f"{name}: ctas={len(d)} start min/med/max {st.min():.2f}/{np.median(st):.2f}/{st.max():.2f}  "
              f"end min/med/max {en.min():.2f}/{np.median(en):.2f}/{en.max():.2f}  "
              f"dep_wait med {np.median((d[:, 3] - t0) / 1e3):.2f}")
        for sl, nm in ((4, "full0"), (96, "mma_xfull0"), (20, "mma0")):
            v = d[:, sl]
            v = v[v > 0]
            if v.size:
                print(f"   {nm}: min/med/max {((v - t0) / 1e3).min():.2f}/{np.median((v - t0) / 1e3):.2f}/{((v - t0) / 1e3).max():.2f}")
    sys.exit(0)
dall = dbg.cpu().numpy().astype(np.int64)
t0 = dall[dall[:, 0] > 0, 0].min()
# pair plans (split=3): even and odd CTAs of each cluster reported separately
views = [("", dall)] if json.loads(a.cfg).get("split") != 3 else [("even CTAs ", dall[0::2]), ("odd CTAs ", dall[1::2])]
for tag, d in views:
    ctas = d[:, 0] > 0
    d = d[ctas]
    print(f"{tag}{a.shape} M={a.m} {a.scheme} cfg={a.cfg} ctas={int(ctas.sum())}  (us relative to first CTA start)")
    for slot in sorted(NAMES, key=lambda sl: ({20: 1}.get(sl // 16 * 16, 0), sl)):
        col = d[:, slot]
        v = col[col > 0]
        if v.size == 0:
            continue
        r = (v - t0) / 1e3
        print(f"  {NAMES[slot]:>10s}: n={v.size:4d} min={r.min():8.2f} med={np.median(r):8.2f} max={r.max():8.2f}")
