"""Repeat GEMM launches of given tile plans many times against one reference
result (the first launch of the auto plan, itself checked against the oracle),
to expose intermittent races. Prints mismatch counts per plan.

    python scripts/stress_plans.py --shape 4096x4096 --m 64 --reps 200 \
        --cfgs '{"ntok":32,"split":4,"csplit":4};auto'
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2406_09904_b200 as Q  # noqa: E402
from paper_2406_09904_b200 import gemm as G  # noqa: E402
from oracle import qqq_oracle as O  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="4096x4096")
ap.add_argument("--m", type=int, default=64)
ap.add_argument("--reps", type=int, default=200)
ap.add_argument("--scheme", default="per-group")
ap.add_argument("--cfgs", default="auto")
ap.add_argument("--interleave", action="store_true", help="alternate the plans launch by launch (PDL overlap)")
ap.add_argument("--requant", action="store_true", help="re-run the activation quantizer before every GEMM")
a = ap.parse_args()
k, n = map(int, a.shape.split("x"))
rng = np.random.default_rng(7)
w = rng.standard_normal((k, n))
x16 = rng.standard_normal((a.m, k)).astype(np.float16)
if a.scheme == "per-channel":
    qw = Q.quant_weight_per_channel(w)
    qo = O.quant_weight_per_channel(w)
else:
    qw = Q.quant_weight_per_group(w, Q.QuantSpec("per-group", 128))
    qo = O.quant_weight_per_group(w, 128)
fused = Q.FusedScales.from_quantized(qw)
x = torch.from_numpy(x16).cuda()
aq = Q.quant_act_per_token(x)
prep = G.prepare(qw, fused)
ao = O.quant_act_per_token(x16.astype(np.float64))
run_o = O.w4a8_gemm_per_channel if a.scheme == "per-channel" else O.w4a8_gemm_per_group
want = run_o(ao, qo, O.FusedScales.from_quantized(qo), fast=True)
want_acc = torch.from_numpy(want.acc).cuda()
want_y = torch.from_numpy(want.y.view(np.int16)).cuda()
cfgs = [None if c == "auto" else json.loads(c) for c in a.cfgs.split(";")]
bad = {i: 0 for i in range(len(cfgs))}
outs = []
order = [(r, i) for r in range(a.reps) for i in range(len(cfgs))] if a.interleave else \
    [(r, i) for i in range(len(cfgs)) for r in range(a.reps)]
pending = []
for r, i in order:
    if a.requant:
        aq = Q.quant_act_per_token(x)
    out = G.run_gemm(aq, prep, n, True, cfg=cfgs[i])
    pending.append((i, out))
    if len(pending) >= 16:
        torch.cuda.synchronize()
        for j, o in pending:
            if not (torch.equal(o.acc, want_acc) and torch.equal(o.y.view(torch.int16), want_y)):
                bad[j] += 1
                if bad[j] <= 3:
                    d = (o.acc.long() - want_acc.long()).cpu().numpy()
                    cols = np.nonzero(d.any(0))[0]
                    tiles = sorted(set((cols // 128).tolist()))
                    rows = sorted(set((cols % 128).tolist()))
                    print(f"  mismatch cfg={cfgs[j]}: {cols.size} cols, tiles {tiles[:12]}, rows-in-tile "
                          f"{rows[:40]}{'...' if len(rows) > 40 else ''}; diff sample {d[0, cols[:6]].tolist()}",
                          flush=True)
        pending = []
torch.cuda.synchronize()
for j, o in pending:
    if not (torch.equal(o.acc, want_acc) and torch.equal(o.y.view(torch.int16), want_y)):
        bad[j] += 1
for i, c in enumerate(cfgs):
    info = G.plan_info(prep.mode, a.m, n, k, c)
    print(f"{a.shape} M={a.m} {a.scheme} cfg={c} plan={info}: {bad[i]} / {a.reps} mismatches", flush=True)
