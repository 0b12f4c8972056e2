"""C4 stack decomposition: GEMMs only / act quant only / both (graph-timed)."""
import json, math, os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench as B
import paper_2406_09904_b200 as Q
from paper_2406_09904_b200 import gemm as G

dev = torch.device("cuda", 0)
lin = []
for li, (name, k, n) in enumerate(B.C4_LINEARS):
    qw, fused, prep = B.make_weights(k, n, "per-group", seed=li, device=dev)
    sm = torch.ones(k, dtype=torch.float64, device=dev)
    sm[torch.randperm(k, device=dev)[: k // 8]] = 1.7
    lin.append((k, n, prep, sm, Q.smoothing_reciprocal(sm)))
for m in (1, 16, 64, 256):
    xs = [torch.randn((m, k), dtype=torch.float16, device=dev) for _, k, _n in B.C4_LINEARS]
    ys = [torch.empty((m, n), dtype=torch.float16, device=dev) for _, _k, n in B.C4_LINEARS]
    aqs = [Q.quant_act_smoothed(xs[i], lin[i][3]) for i in range(4)]
    G.workspace(dev, max(Q._lib.load().qqq_gemm_workspace_bytes(m, n, k) for _, k, n in B.C4_LINEARS))
    def gemms():
        for i, (k, n, prep, sm, rc) in enumerate(lin):
            G.run_gemm(aqs[i], prep, n, False, y_out=ys[i])
    def quants():
        for i, (k, n, prep, sm, rc) in enumerate(lin):
            Q.quant_act_smoothed(xs[i], sm, check=False)
    def quants_rcp():
        for i, (k, n, prep, sm, rc) in enumerate(lin):
            Q.quant_act_smoothed(xs[i], sm, check=False, recip=rc)
    def both_rcp():
        for i, (k, n, prep, sm, rc) in enumerate(lin):
            aq = Q.quant_act_smoothed(xs[i], sm, check=False, recip=rc)
            G.run_gemm(aq, prep, n, False, y_out=ys[i])
    def quants_plain():
        for i, (k, n, prep, sm, rc) in enumerate(lin):
            Q.quant_act_per_token(xs[i], check=False)
    def both():
        for i, (k, n, prep, sm, rc) in enumerate(lin):
            aq = Q.quant_act_smoothed(xs[i], sm, check=False)
            G.run_gemm(aq, prep, n, False, y_out=ys[i])
    r = {f.__name__: round(B.graph_time_us([f], reps=20), 2) for f in (gemms, quants, quants_rcp, quants_plain, both, both_rcp)}
    print(json.dumps(dict(M=m, **r)), flush=True)
