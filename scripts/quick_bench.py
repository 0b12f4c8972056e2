"""Developer sweep: device time per (shape, M, tile plan) via CUDA graphs over
rotated cold weight replicas. bench.py is the contract benchmark."""
import argparse
import json
import math
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench as B  # noqa: E402
import paper_2406_09904_b200 as Q  # noqa: E402
from paper_2406_09904_b200 import gemm as G  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="4096x4096,4096x11008,11008x4096")
    ap.add_argument("--ms", default="1,16,64,128,256,512,1024")
    ap.add_argument("--schemes", default="per-group")
    ap.add_argument("--cfgs", default="auto", help="';'-separated JSON tile plans or 'auto'")
    ap.add_argument("--fp16", action="store_true")
    ap.add_argument("--profile", action="store_true", help="few plain launches (for ncu), no timing")
    ap.add_argument("--reps", type=int, default=0, help="cold replicas per point (default: > 2.5x L2)")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    cfgs = [None if c == "auto" else json.loads(c) for c in a.cfgs.split(";")]
    peaks = B.load_peaks()
    for shp in a.shapes.split(","):
        k, n = map(int, shp.split("x"))
        for scheme in a.schemes.split(","):
            qw, fused, prep = B.make_weights(k, n, scheme, 0, dev)
            R = a.reps or max(2, math.ceil(2.5 * B.L2_BYTES / (k * n / 2)))
            if a.profile:
                R = 2
            reps = [prep] + [G.PreparedWeights(prep.mode, prep.w.clone(), None if prep.sc is None else prep.sc.clone(),
                                               prep.group, prep.s_col.clone()) for _ in range(R - 1)]
            r16 = max(2, math.ceil(2.5 * B.L2_BYTES / (k * n * 2)))
            w16 = [torch.randn((k, n), dtype=torch.float16, device=dev) for _ in range(r16)] if a.fp16 else None
            for m in map(int, a.ms.split(",")):
                x = torch.randn((m, k), dtype=torch.float16, device=dev)
                aq = Q.quant_act_per_token(x)
                y = torch.empty((m, n), dtype=torch.float16, device=dev)
                G.workspace(dev, Q._lib.load().qqq_gemm_workspace_bytes(m, n, k))
                for cfg in cfgs:
                    fns = [(lambda p: (lambda: G.run_gemm(aq, p, n, False, y_out=y, cfg=cfg)))(p) for p in reps]
                    if a.profile:
                        for f in fns * 2:
                            f()
                        torch.cuda.synchronize()
                        continue
                    t = B.graph_time_us(fns, reps=max(2, 60 // R))
                    ops = 2.0 * m * n * k
                    byt = B.alg_bytes(m, k, n, scheme)
                    roof = max(byt / (peaks["hbm_gbs"] * 1e3), ops / (2 * peaks["bf16_tflops"] * 1e6))
                    rec = dict(shape=shp, scheme=scheme, M=m, cfg=cfg, us=round(t, 2), TOPS=round(ops / t / 1e6, 1),
                               GBps=round(byt / t / 1e3, 1), roof_frac=round(roof / t, 3))
                    if w16:
                        t16 = B.graph_time_us([(lambda wi: (lambda: torch.matmul(x, wi)))(wi) for wi in w16],
                                              reps=max(2, 40 // len(w16)))
                        rec["fp16_us"] = round(t16, 2)
                        rec["speedup"] = round(t16 / t, 2)
                    print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
