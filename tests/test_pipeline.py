"""apply_quant_linear (pipeline.py:144-152): the CPU oracle against golden
vectors made by the reference itself (tests/golden/make_golden_pipeline.py),
and (GPU) the fused smooth+quantize kernel and the B200 linear against the
same vectors — bit-exact (codes, f64 scales, y widened to f64)."""

import os

import numpy as np
import pytest

from oracle import qqq_oracle as O

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "pipeline_cases.npz")


def _cases():
    g = np.load(GOLD)
    for i in range(int(g["n_cases"])):
        p = f"c{i}_"
        t, k, n, gs, pg, f16 = (int(v) for v in g[p + "meta"])
        yield dict(i=i, t=t, k=k, n=n, gs=gs, pg=bool(pg), f16=bool(f16), x=g[p + "x"], s=g[p + "s"],
                   packed=g[p + "packed"], s_w=g.get(p + "s_w"), s_wg=g.get(p + "s_wg"), s_wc=g.get(p + "s_wc"),
                   q=g[p + "q"], s_a=g[p + "s_a"], y=g[p + "y"])


def _oracle_qw(c):
    if c["pg"]:
        return O.QuantizedWeights(c["packed"], c["k"], c["n"], O.PER_GROUP, c["gs"], s_wg=c["s_wg"], s_wc=c["s_wc"])
    return O.QuantizedWeights(c["packed"], c["k"], c["n"], O.PER_CHANNEL, s_w=c["s_w"])


def test_oracle_apply_quant_linear_matches_reference_goldens():
    for c in _cases():
        qa = O.quant_act_per_token(c["x"] / c["s"][None, :])
        assert np.array_equal(qa.q, c["q"]) and np.array_equal(qa.s_a.view(np.uint64), c["s_a"].view(np.uint64))
        y = O.apply_quant_linear(c["x"], c["s"], _oracle_qw(c))
        assert np.array_equal(y.view(np.uint64), c["y"].view(np.uint64)), c["i"]


@pytest.mark.gpu
def test_gpu_apply_quant_linear_bit_exact():
    import torch

    import paper_2406_09904_b200 as Q

    dev = torch.device("cuda")
    f = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    for c in _cases():
        qw = (Q.QuantizedWeights(f(c["packed"]), c["k"], c["n"], Q.PER_GROUP, c["gs"], s_wg=f(c["s_wg"]),
                                 s_wc=f(c["s_wc"])) if c["pg"]
              else Q.QuantizedWeights(f(c["packed"]), c["k"], c["n"], Q.PER_CHANNEL, s_w=f(c["s_w"])))
        plan = Q.SmoothingPlan(sigma=1.0, selected=(), s=c["s"], objective=0.0)
        layer = Q.QuantizedLayer(name=f"case{c['i']}", qweights=qw, plan=plan)
        # fp16 activations arrive as fp16 tensors when they are fp16-exact, else as f64
        x = torch.from_numpy(c["x"]).to(dev)
        if c["f16"]:
            x = x.to(torch.float16)
        qa = Q.quant_act_smoothed(x, c["s"])
        assert np.array_equal(qa.q.cpu().numpy(), c["q"]), c["i"]
        assert np.array_equal(qa.s_a.cpu().numpy().view(np.uint64), c["s_a"].view(np.uint64)), c["i"]
        y = Q.apply_quant_linear(x, layer)
        assert y.dtype == torch.float64
        assert np.array_equal(y.cpu().numpy().view(np.uint64), c["y"].view(np.uint64)), c["i"]
        # the one-launch form (quantization inside the GEMM launch) where the inputs allow it
        yf = Q.apply_quant_linear(x, layer, fused=True)
        assert np.array_equal(yf.cpu().numpy().view(np.uint64), c["y"].view(np.uint64)), c["i"]


@pytest.mark.gpu
def test_gpu_apply_quant_linear_errors():
    import torch

    import paper_2406_09904_b200 as Q

    dev = torch.device("cuda")
    x = torch.randn(4, 128, device=dev, dtype=torch.float16)
    with pytest.raises(Q.ShapeError):
        Q.quant_act_smoothed(x, np.ones(64))
    x[1, 3] = float("inf")
    with pytest.raises(Q.DataError):
        Q.quant_act_smoothed(x, np.ones(128))


@pytest.mark.gpu
@pytest.mark.parametrize("k", [4096, 11008, 13000])
def test_gpu_quant_act_smoothed_random_vs_oracle(k):
    """The register-resident smoothed quantizer (one IEEE f64 division per
    element) against the oracle's quant_act_per_token(x / s) on random rows,
    ~1/8 of the channels smoothed (pipeline.py:146)."""
    import torch

    import paper_2406_09904_b200 as Q

    rng = np.random.default_rng(k)
    for m in (1, 3, 64):
        x16 = (rng.standard_normal((m, k)) * rng.uniform(0.1, 8.0, (m, 1))).astype(np.float16)
        s = np.ones(k)
        sel = rng.choice(k, k // 8, replace=False)
        s[sel] = rng.uniform(0.05, 20.0, k // 8)
        want = O.quant_act_per_token(x16.astype(np.float64) / s)
        got = Q.quant_act_smoothed(torch.from_numpy(x16).cuda(), s)
        assert np.array_equal(got.q.cpu().numpy(), want.q), (k, m)
        assert np.array_equal(got.s_a.cpu().numpy().view(np.uint64), want.s_a.view(np.uint64)), (k, m)


def _markstein(a: float, b: float) -> float:
    """The kernel's division (act_quant.cu div_markstein) in exact rational
    arithmetic (float(Fraction) rounds to nearest even, like each FMA):
    y = RN(1/b), q0 = RN(a*y), q1 = fma(fma(-q0, b, a), y, q0),
    result = fma(fma(-q1, b, a), y, q1)."""
    from fractions import Fraction as F

    y = 1.0 / b
    q0 = a * y
    q1 = float(F(q0) + F(float(F(a) - F(q0) * F(b))) * F(y))
    r_exact = F(a) - F(q1) * F(b)
    r = float(r_exact)
    assert F(r) == r_exact  # q1 is within one ulp: the residual is exact (Markstein)
    return float(F(q1) + F(r) * F(y))


def test_markstein_division_is_ieee():
    """x / s_k and x / s as Markstein FMA sequences equal numpy's IEEE division:
    fp16 numerators against smoothing factors, and f64 numerators against
    per-token scales, at the magnitudes the quantizer admits."""
    rng = np.random.default_rng(7)
    f16 = np.arange(0, 0x7C00, dtype=np.uint16).view(np.float16).astype(np.float64)
    a = np.concatenate([f16[rng.integers(0, f16.size, 6000)], -f16[rng.integers(0, f16.size, 2000)],
                        rng.standard_normal(4000) * 10.0 ** rng.uniform(-30, 30, 4000)])
    b = np.concatenate([rng.uniform(0.05, 20.0, 4000), 10.0 ** rng.uniform(-100, 100, 4000),
                        rng.uniform(1e-3, 1.0, 4000) / 127.0])
    b[:50] = 1.0
    b[50:100] = np.nextafter(1.0, 2.0) * np.arange(1, 51)
    for ai, bi in zip(a.tolist(), b.tolist()):
        assert _markstein(ai, bi) == ai / bi, (ai, bi)


@pytest.mark.gpu
@pytest.mark.parametrize("k", [4096, 11008])
def test_gpu_quant_act_smoothed_recip_vs_oracle(k):
    """The reciprocal-table (Markstein) quantizer: cluster rows (M <= 256) and
    register rows (M > 256), every finite fp16 value present, unsafe smoothing
    factors (NaN table entries) mixed in."""
    import torch

    import paper_2406_09904_b200 as Q

    rng = np.random.default_rng(k + 1)
    all16 = np.arange(0, 0x7C00, dtype=np.uint16).view(np.float16)
    for m in (1, 16, 256, 300):
        x16 = (rng.standard_normal((m, k)) * rng.uniform(0.1, 8.0, (m, 1))).astype(np.float16)
        flat = x16.reshape(-1)
        n = min(flat.size, all16.size)
        flat[:n] = all16[rng.permutation(all16.size)[:n]] * np.where(rng.random(n) < 0.5, -1, 1).astype(np.float16)
        s = np.ones(k)
        sel = rng.choice(k, k // 8, replace=False)
        s[sel] = rng.uniform(0.05, 20.0, k // 8)
        s[sel[:4]] = [1e-130, 3e200, 2.0 ** -400, 2.0 ** 400]
        want = O.quant_act_per_token(x16.astype(np.float64) / s)
        st = torch.from_numpy(s).cuda()
        recip = Q.smoothing_reciprocal(st)
        r = recip.cpu().numpy()
        ok = (np.abs(s) >= 2.0 ** -400) & (np.abs(s) <= 2.0 ** 400)
        assert np.array_equal(r[ok].view(np.uint64), (1.0 / s[ok]).view(np.uint64)) and np.isnan(r[~ok]).all()
        got = Q.quant_act_smoothed(torch.from_numpy(x16).cuda(), st, recip=recip)
        assert np.array_equal(got.q.cpu().numpy(), want.q), (k, m)
        assert np.array_equal(got.s_a.cpu().numpy().view(np.uint64), want.s_a.view(np.uint64)), (k, m)
        assert np.array_equal(got._rowsum[1].cpu().numpy(), want.q.sum(1, dtype=np.int64)), (k, m)
