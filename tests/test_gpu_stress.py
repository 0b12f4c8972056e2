"""Repeated launches (activation quantizer + GEMM, PDL-chained as in serving)
of the plans with co-resident cluster CTAs, each checked bit-exactly against
the oracle: intermittent races show up here, not in single-launch parity.

Covers the two-CTA-per-SM 16- and 32-token cluster split-K decode plans the
planner picks on the 7B shapes and the 128-token whole-SM clusters
(scripts/stress_plans.py is the long version).
"""

import numpy as np
import pytest
import torch

import paper_2406_09904_b200 as Q
from paper_2406_09904_b200 import gemm as G
from oracle import qqq_oracle as O

pytestmark = pytest.mark.gpu

CASES = [
    # (K, N, M, scheme, cfg)
    (11008, 4096, 1, "per-group", {"ntok": 16, "split": 4, "csplit": 6}),   # 192 CTAs, 2 per SM
    (4096, 11008, 16, "per-channel", {"ntok": 16, "split": 4, "csplit": 2}),  # 172 CTAs
    (8192, 8192, 1, "per-channel", {"ntok": 32, "split": 4, "csplit": 4}),  # two CTAs per SM
    (4096, 11008, 24, "per-group", {"ntok": 32, "split": 4, "csplit": 2}),  # (the planner's pick there)
    (4096, 4096, 128, "per-group", {"ntok": 128, "split": 4, "csplit": 4}),  # whole-SM clusters
]


@pytest.mark.parametrize("k,n,m,scheme,cfg", CASES)
def test_repeated_launches_bit_exact(k, n, m, scheme, cfg):
    rng = np.random.default_rng(k + n + m)
    w = rng.standard_normal((k, n))
    x16 = rng.standard_normal((m, k)).astype(np.float16)
    if scheme == "per-channel":
        qw, qo = Q.quant_weight_per_channel(w), O.quant_weight_per_channel(w)
    else:
        qw, qo = Q.quant_weight_per_group(w, Q.QuantSpec("per-group", 128)), O.quant_weight_per_group(w, 128)
    ao = O.quant_act_per_token(x16.astype(np.float64))
    run_o = O.w4a8_gemm_per_channel if scheme == "per-channel" else O.w4a8_gemm_per_group
    want = run_o(ao, qo, O.FusedScales.from_quantized(qo), fast=True)
    want_acc = torch.from_numpy(want.acc).cuda()
    want_y = torch.from_numpy(want.y.view(np.int16)).cuda()
    prep = G.prepare(qw, Q.FusedScales.from_quantized(qw))
    x = torch.from_numpy(x16).cuda()
    info = G.plan_info(prep.mode, m, n, k, cfg)
    bad, outs = 0, []
    for rep in range(120):
        aq = Q.quant_act_per_token(x)
        outs.append(G.run_gemm(aq, prep, n, True, cfg=cfg))
        if len(outs) == 12:
            torch.cuda.synchronize()
            bad += sum(not (torch.equal(o.acc, want_acc) and torch.equal(o.y.view(torch.int16), want_y)) for o in outs)
            outs = []
    assert bad == 0, (k, n, m, scheme, info, bad)
