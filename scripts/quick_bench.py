"""Quick device-time sweep of the W4A8 GEMM (CUDA events, L2 flushed between
iterations by rotating weight replicas). Developer tool; bench.py is the
contract benchmark."""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_09904_b200 as Q  # noqa: E402
from paper_2406_09904_b200 import gemm as G  # noqa: E402


def make(k, n, scheme, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    q4 = torch.randint(-8, 8, (k, n), dtype=torch.int8, device="cuda", generator=g)
    if scheme == "per-channel":
        s_w = (0.02 * (0.5 + torch.rand(n, dtype=torch.float64, device="cuda", generator=g)))
        qw = Q.QuantizedWeights(Q.pack_i4(q4), k, n, "per-channel", s_w=s_w)
    else:
        s_wg = 0.02 * (0.5 + torch.rand((k // 128, n), dtype=torch.float64, device="cuda", generator=g))
        qw = Q.QuantizedWeights(Q.pack_i4(q4), k, n, "per-group", 128, s_wg=s_wg, s_wc=Q.requant_scale(q4, s_wg))
    fused = Q.FusedScales.from_quantized(qw)
    return G.prepare(qw, fused)


def time_fn(fn, iters, flush):
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(iters)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(iters)]
    for i in range(iters):
        flush()
        starts[i].record()
        fn(i)
        ends[i].record()
    torch.cuda.synchronize()
    ts = sorted(s.elapsed_time(e) for s, e in zip(starts, ends))
    return ts[len(ts) // 2] * 1e3  # us median


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="4096x4096,4096x11008,11008x4096")
    ap.add_argument("--ms", default="1,16,64,128,256,512,1024")
    ap.add_argument("--schemes", default="per-group,per-channel")
    ap.add_argument("--iters", type=int, default=30)
    ap.add_argument("--cfg", default="")
    a = ap.parse_args()
    flushbuf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    flush = lambda: flushbuf.zero_()
    cfg = json.loads(a.cfg) if a.cfg else None
    for shp in a.shapes.split(","):
        k, n = map(int, shp.split("x"))
        for scheme in a.schemes.split(","):
            prep = make(k, n, scheme)
            wf16 = torch.randn((k, n), dtype=torch.float16, device="cuda")
            for m in map(int, a.ms.split(",")):
                x = torch.randn((m, k), dtype=torch.float16, device="cuda")
                aq = Q.quant_act_per_token(x)
                y = torch.empty((m, n), dtype=torch.float16, device="cuda")
                t_g = time_fn(lambda i: G.run_gemm(aq, prep, n, False, y_out=y, cfg=cfg), a.iters, flush)
                t_q = time_fn(lambda i: Q.quant_act_per_token(x, check=False), a.iters, flush)
                t_h = time_fn(lambda i: torch.matmul(x, wf16), a.iters, flush)
                ops = 2.0 * m * n * k
                byt = m * k + 8 * m + k * n / 2 + 2 * m * n + (8 * n if scheme == "per-channel" else 2 * (k // 128) * n + 8 * n)
                print(json.dumps(dict(shape=shp, scheme=scheme, M=m, gemm_us=round(t_g, 2), actq_us=round(t_q, 2),
                                      fp16_us=round(t_h, 2), TOPS=round(ops / t_g / 1e6, 1),
                                      GBps=round(byt / t_g / 1e3, 1), speedup_vs_fp16=round(t_h / t_g, 2))), flush=True)


if __name__ == "__main__":
    main()
