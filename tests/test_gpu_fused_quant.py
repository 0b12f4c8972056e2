"""apply_quant_linear's activation step fused into the GEMM launch
(qqq_w4a8_gemm_smooth_fused; reference pipeline.py:144-152).

The fused launch must produce exactly what the two-kernel form produces:
quant_act_smoothed (pinned to the oracle and the reference pipeline goldens
in tests/test_pipeline.py) followed by the W4A8 GEMM (pinned in
tests/test_gpu_parity.py): the same codes, per-token scales, code sums and
y bits, under the planner's choice and under every CTA shape / plan the
fused prologue runs in (half-SM cluster CTAs, whole-SM tiles, 128-token
clusters, pair tiles, stream-K), with and without the reciprocal table, and
across repeated PDL-chained launches (the row counter re-arms itself).
"""

import numpy as np
import pytest
import torch

import paper_2406_09904_b200 as Q
from paper_2406_09904_b200 import gemm as G
from paper_2406_09904_b200 import pipeline as P
from oracle import qqq_oracle as O

pytestmark = pytest.mark.gpu


def _weights(k, n, scheme, seed):
    rng = np.random.default_rng(seed)
    w = rng.standard_normal((k, n))
    qw = Q.quant_weight_per_channel(w) if scheme == "per-channel" else \
        Q.quant_weight_per_group(w, Q.QuantSpec("per-group", 128))
    fused = Q.FusedScales.from_quantized(qw)
    return qw, fused, G.prepare(qw, fused)


def _smoothing(k, seed, frac=8):
    g = torch.Generator().manual_seed(seed)
    s = torch.ones(k, dtype=torch.float64)
    idx = torch.randperm(k, generator=g)[: max(1, k // frac)]
    s[idx] = 0.25 + 3.0 * torch.rand(idx.numel(), dtype=torch.float64, generator=g)
    return s.cuda()


def _two_kernel(x, s, recip, prep, n, cfg=None):
    aq = Q.quant_act_smoothed(x, s, recip=recip)
    y = G.run_gemm(aq, prep, n, False, cfg=cfg).y
    return y, aq


def _check(x, s, recip, prep, n, cfg, tag):
    y0, a0 = _two_kernel(x, s, recip, prep, n, cfg)
    y1, a1 = P.quant_linear_smoothed(x, s, recip, prep, n, cfg=cfg)
    torch.cuda.synchronize()
    assert torch.equal(a1.q, a0.q), tag
    assert torch.equal(a1.s_a.view(torch.int64), a0.s_a.view(torch.int64)), tag
    assert torch.equal(Q.quantize.rowsum_of(a1), Q.quantize.rowsum_of(a0)), tag
    assert torch.equal(y1.view(torch.int16), y0.view(torch.int16)), tag


@pytest.mark.parametrize("scheme", ["per-channel", "per-group"])
@pytest.mark.parametrize("k,n", [(4096, 12288), (4096, 4096), (4096, 22016), (11008, 4096)])
def test_fused_equals_two_kernel_c4_linears(k, n, scheme):
    """The C4 decoder-layer linears (BASELINE configs[3]) at batch 1..256 under the planner."""
    qw, fused, prep = _weights(k, n, scheme, k + n)
    s = _smoothing(k, k)
    recip = Q.smoothing_reciprocal(s)
    for m in (1, 16, 64, 256):
        x = (torch.randn((m, k), generator=torch.Generator().manual_seed(m)) * 3).to(torch.float16).cuda()
        _check(x, s, recip, prep, n, None, (k, n, scheme, m, G.plan_info(prep.mode, m, n, k)))


def test_fused_every_plan():
    """Every CTA shape / plan family the fused prologue runs in, forced."""
    k, n = 2048, 1280
    cfgs = [{"ntok": 16, "split": 4, "csplit": 4}, {"ntok": 32, "split": 4, "csplit": 2}, {"ntok": 16, "split": 1},
            {"ntok": 64, "split": 0}, {"ntok": 128, "split": 0}, {"ntok": 128, "split": 1}, {"ntok": 128, "split": 2},
            {"ntok": 128, "split": 4, "csplit": 2}, {"ntok": 128, "split": 4, "csplit": 4}, {"ntok": 256, "split": 3},
            {"ntok": 256, "split": 5}, {"ntok": 256, "split": 6}, {"ntok": 192, "split": 3}, {"ntok": 384, "split": 3},
            {"ntok": 128, "split": 3}, {"ntok": 256, "split": 0}]
    for scheme in ("per-channel", "per-group"):
        qw, fused, prep = _weights(k, n, scheme, 5)
        s = _smoothing(k, 3, frac=1)  # every channel smoothed
        recip = Q.smoothing_reciprocal(s)
        for m in (7, 100, 333, 1100):
            x = (torch.randn((m, k), generator=torch.Generator().manual_seed(m)) * 2).to(torch.float16).cuda()
            for cfg in (cfgs if m < 1000 else [None, {"ntok": 384, "split": 3}, {"ntok": 256, "split": 3},
                                               {"ntok": 128, "split": 0}]):
                _check(x, s, recip, prep, n, cfg, (scheme, m, cfg, G.plan_info(prep.mode, m, n, k, cfg)))


def test_fused_without_table_and_odd_shapes():
    """IEEE division (no reciprocal table), K not a multiple of 128, a strided x, M not a multiple of 16."""
    for (k, n, m) in ((1000, 640, 37), (2056, 384, 5), (4096, 256, 130)):
        qw, fused, prep = _weights(k, n, "per-group" if k % 128 == 0 else "per-channel", k)
        s = _smoothing(k, 11, frac=2)
        base = (torch.randn((m, k + 24), generator=torch.Generator().manual_seed(k)) * 4).to(torch.float16).cuda()
        x = base[:, 8: 8 + k]  # row pitch k + 24, 16-byte aligned start
        assert P._fused_ok(x, prep)
        _check(x, s, None, prep, n, None, (k, n, m))


def test_fused_matches_oracle_small():
    """Anchor: the fused launch against the oracle's apply_quant_linear arithmetic."""
    k, n, m = 512, 256, 9
    rng = np.random.default_rng(1)
    w = rng.standard_normal((k, n))
    x16 = (rng.standard_normal((m, k)) * 2).astype(np.float16)
    s = np.ones(k)
    s[rng.choice(k, 64, replace=False)] = 0.5 + rng.random(64) * 2
    for scheme in ("per-channel", "per-group"):
        if scheme == "per-channel":
            qw, qo = Q.quant_weight_per_channel(w), O.quant_weight_per_channel(w)
        else:
            qw, qo = Q.quant_weight_per_group(w, Q.QuantSpec("per-group", 128)), O.quant_weight_per_group(w, 128)
        want = O.apply_quant_linear(x16.astype(np.float64), s, qo)
        prep = G.prepare(qw, Q.FusedScales.from_quantized(qw))
        st = torch.from_numpy(s).cuda()
        y, aq = P.quant_linear_smoothed(torch.from_numpy(x16).cuda(), st, Q.smoothing_reciprocal(st), prep, n)
        got = y.double().cpu().numpy()
        assert np.array_equal(got.view(np.uint64), np.asarray(want).view(np.uint64)), scheme


def test_fused_repeated_chain_rearms():
    """120 back-to-back fused launches on one stream (PDL-chained), alternating
    plans and batch sizes: the in-workspace row counter must re-arm every time."""
    k, n = 4096, 4096
    qw, fused, prep = _weights(k, n, "per-group", 9)
    s = _smoothing(k, 2)
    recip = Q.smoothing_reciprocal(s)
    xs = {m: (torch.randn((m, k), generator=torch.Generator().manual_seed(m))).to(torch.float16).cuda()
          for m in (1, 16, 64, 256)}
    want = {m: _two_kernel(xs[m], s, recip, prep, n)[0] for m in xs}
    outs = []
    for rep in range(120):
        m = (1, 16, 64, 256)[rep % 4]
        y, _ = P.quant_linear_smoothed(xs[m], s, recip, prep, n, check=False)
        outs.append((m, y))
    torch.cuda.synchronize()
    bad = sum(not torch.equal(y.view(torch.int16), want[m].view(torch.int16)) for m, y in outs)
    assert bad == 0


def test_fused_nonfinite_raises():
    k, n = 1024, 256
    qw, fused, prep = _weights(k, n, "per-channel", 4)
    s = _smoothing(k, 4)
    x = torch.randn((3, k)).to(torch.float16).cuda()
    x[1, 17] = float("inf")
    with pytest.raises(Q.DataError):
        P.quant_linear_smoothed(x, s, Q.smoothing_reciprocal(s), prep, n)
    # the launch after an error is clean again
    x[1, 17] = 0.5
    _check(x, s, Q.smoothing_reciprocal(s), prep, n, None, "after error")


def test_apply_quant_linear_takes_fused_path():
    """apply_quant_linear(fused=True) on fp16 CUDA activations runs the fused launch (same y as the two-kernel form)."""
    k, n, m = 4096, 1024, 33
    rng = np.random.default_rng(3)
    w = rng.standard_normal((k, n))
    qw = Q.quant_weight_per_group(w, Q.QuantSpec("per-group", 128))
    s = np.ones(k)
    s[:100] = 1.5
    layer = Q.QuantizedLayer(name="l", qweights=qw, plan=Q.SmoothingPlan(sigma=1.0, selected=(), s=s, objective=0.0))
    x = torch.from_numpy((rng.standard_normal((m, k)) * 2).astype(np.float16)).cuda()
    called = []
    orig = P.quant_linear_smoothed

    def spy(*a, **kw):
        called.append(1)
        return orig(*a, **kw)

    P.quant_linear_smoothed = spy
    try:
        y = Q.apply_quant_linear(x, layer, fused=True)
    finally:
        P.quant_linear_smoothed = orig
    assert called
    fused = Q.FusedScales.from_quantized(qw)
    y0 = Q.w4a8_gemm_per_group(Q.quant_act_smoothed(x, s), qw, fused, with_acc=False).y_wide()
    assert torch.equal(y.view(torch.int64), y0.view(torch.int64))
