"""The sm_100a pieces of the K-split / N-split TP path, ranks simulated on one
GPU: per-shard absmax -> MAX -> quantize with the global max -> int32 partial
GEMM -> SUM -> dequant epilogue must equal the unsplit GEMM bit for bit."""

import numpy as np
import pytest
import torch

import paper_2406_09904_b200 as Q
from paper_2406_09904_b200 import tp
from oracle import qqq_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("scheme", ["per-channel", "per-group"])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_ksplit_simulated(scheme, world):
    m, k, n = 7, 4096, 512
    x16, w = O.recipe_r1(m, n, k, seed=world)
    x = torch.from_numpy(x16).cuda()
    qw = Q.quant_weight_per_channel(w) if scheme == "per-channel" else Q.quant_weight_per_group(w, Q.QuantSpec("per-group", 128))
    fused = Q.FusedScales.from_quantized(qw)
    run = Q.w4a8_gemm_per_channel if scheme == "per-channel" else Q.w4a8_gemm_per_group
    ref = run(Q.quant_act_per_token(x), qw, fused)
    ops = tp.TPOps()
    shards = [tp.shard_ksplit(qw, r, world) for r in range(world)]
    ks = k // world
    row_max = torch.stack([ops.row_absmax(x[:, r * ks:(r + 1) * ks]) for r in range(world)]).max(0).values
    acc = None
    s_a = None
    for r, sh in enumerate(shards):
        aq = ops.quant_with_max(x[:, r * ks:(r + 1) * ks], row_max)
        part = ops.gemm_acc(aq, sh, Q.FusedScales.from_quantized(sh))
        acc = part if acc is None else acc + part
        s_a = aq.s_a
    s_col = fused.s_w_folded if scheme == "per-channel" else fused.s_wc
    y = ops.epilogue(acc, s_a, s_col)
    assert torch.equal(acc, ref.acc)
    assert torch.equal(s_a, Q.quant_act_per_token(x).s_a)
    assert torch.equal(y.view(torch.int16), ref.y.view(torch.int16))


@pytest.mark.parametrize("world", [2, 8])
def test_nsplit_simulated(world):
    m, k, n = 9, 1024, 2048
    x16, w = O.recipe_r1(m, n, k, seed=11)
    x = torch.from_numpy(x16).cuda()
    qw = Q.quant_weight_per_group(w, Q.QuantSpec("per-group", 128))
    ref = Q.w4a8_gemm_per_group(Q.quant_act_per_token(x), qw, Q.FusedScales.from_quantized(qw))
    ops = tp.TPOps()
    parts = []
    for r in range(world):
        sh = tp.shard_nsplit(qw, r, world)
        parts.append(ops.gemm(ops.quant(x), sh, Q.FusedScales.from_quantized(sh)))
    assert torch.equal(torch.cat(parts, 1).view(torch.int16), ref.y.view(torch.int16))
