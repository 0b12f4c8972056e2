"""Does PDL overlap consecutive GEMMs? Time R back-to-back launches (distinct
weight replicas) on one stream, eagerly and in a CUDA graph, per grid size."""
import json, math, os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench as B
import paper_2406_09904_b200 as Q
from paper_2406_09904_b200 import gemm as G

dev = torch.device("cuda", 0)
for shp in sys.argv[1].split(","):
    k, n = map(int, shp.split("x"))
    qw, fused, prep = B.make_weights(k, n, "per-group", 0, dev)
    R = max(2, math.ceil(2.5 * B.L2_BYTES / (k * n / 2)))
    reps = [prep] + [G.PreparedWeights(prep.mode, prep.w.clone(), None if prep.sc is None else prep.sc.clone(), prep.group, prep.s_col.clone())
                     for _ in range(R - 1)]
    for m in map(int, sys.argv[2].split(",")):
        x = torch.randn((m, k), dtype=torch.float16, device=dev)
        aq = Q.quant_act_per_token(x)
        y = torch.empty((m, n), dtype=torch.float16, device=dev)
        G.workspace(dev, Q._lib.load().qqq_gemm_workspace_bytes(m, n, k))
        for cfg in [None] + [json.loads(c) for c in sys.argv[3:]]:
            fns = [(lambda p: (lambda: G.run_gemm(aq, p, n, False, y_out=y, cfg=cfg)))(p) for p in reps]
            tg = B.graph_time_us(fns, reps=max(2, 60 // R))
            # eager
            for f in fns: f()
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(max(2, 60 // R)):
                for f in fns: f()
            e.record(); torch.cuda.synchronize()
            te = s.elapsed_time(e) * 1e3 / (max(2, 60 // R) * R)
            print(json.dumps(dict(shape=shp, M=m, cfg=cfg, graph_us=round(tg, 2), eager_us=round(te, 2),
                                  pdl=os.environ.get("QQQ_NO_PDL") is None)), flush=True)
