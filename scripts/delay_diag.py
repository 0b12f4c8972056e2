import sys, json, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2406_09904_b200 as Q
from paper_2406_09904_b200 import gemm as G
from oracle import qqq_oracle as O
k, n, m = 4096, 4096, 256
rng = np.random.default_rng(5)
w = rng.standard_normal((k, n)); x16 = rng.standard_normal((m, k)).astype(np.float16)
for scheme in ("per-channel", "per-group"):
    if scheme == "per-channel":
        qw, qo = Q.quant_weight_per_channel(w), O.quant_weight_per_channel(w)
    else:
        qw, qo = Q.quant_weight_per_group(w, Q.QuantSpec("per-group", 128)), O.quant_weight_per_group(w, 128)
    ao = O.quant_act_per_token(x16.astype(np.float64))
    run_o = O.w4a8_gemm_per_channel if scheme == "per-channel" else O.w4a8_gemm_per_group
    want = torch.from_numpy(run_o(ao, qo, O.FusedScales.from_quantized(qo), fast=True).acc).cuda()
    prep = G.prepare(qw, Q.FusedScales.from_quantized(qw))
    aq = Q.quant_act_per_token(torch.from_numpy(x16).cuda())
    for cfg in ({"ntok": 256, "split": 1}, {"ntok": 128, "split": 0}, {"ntok": 128, "split": 1}, None):
        bad = 0
        for rep in range(10):
            out = G.run_gemm(aq, prep, n, True, cfg=cfg)
            torch.cuda.synchronize()
            bad += int(not torch.equal(out.acc, want))
        print(scheme, cfg, G.plan_info(prep.mode, m, n, k, cfg), "bad", bad, "/10", flush=True)
