"""Bit-exact parity at every point bench.py reports, under the planner's own
choice AND every tile plan the planner can pick at that shape.

Configs (BASELINE.json / SURVEY.md §8):
  * C2  per-group g=128, M in {1, 2, 4, ..., 1024} on the Llama-2-7B shapes
        4096x4096, 4096x11008, 11008x4096;
  * C3  per-channel and per-group on the Llama-2-70B shapes 8192x8192,
        8192x28672, 28672x8192 at M in {1, 16, 1024};
  * C4  the decoder-layer linears (QKV 4096->12288, gate-up 4096->22016)
        through apply_quant_linear at batch {1, 16, 64, 256};
  * C5  the 70B tensor-parallel shards at P = 2, 4, 8 (N-split gate_up,
        K-split down and o_proj), ranks simulated on one GPU.

The checker is the oracle (oracle/qqq_oracle.py, pinned to the reference's
goldens and to its C1/C2 digests): FusedDequantQuant of gemm.py:130-142 and
the exact integer matmul of gemm.py:145-154 (evaluated as f64 BLAS, exact
below 2^53), then the f64 epilogue of gemm.py:182-184 / 200-202.
int8 codes, s_a, int32 acc and fp16 y must be identical (tolerance 0).

The per-token quantizer and the GEMM are row-independent, so the oracle runs
once per weight at the largest M and smaller M compare against its leading rows.
Reference: /root/reference/pkg/src/qqq/gemm.py:173-203.
"""

import functools

import numpy as np
import pytest
import torch

import paper_2406_09904_b200 as Q
from paper_2406_09904_b200 import _lib
from paper_2406_09904_b200 import gemm as G
from paper_2406_09904_b200 import tp
from oracle import qqq_oracle as O

pytestmark = pytest.mark.gpu

GS = 128
MS_C2 = [1, 2, 4, 8, 16, 32, 64, 128, 256, 512, 1024]
SHAPES_C2 = [(4096, 4096), (4096, 11008), (11008, 4096)]
SHAPES_C3 = [(8192, 8192), (8192, 28672), (28672, 8192)]


# --------------------------------------------------------------------- oracle


def _oracle_gemm(q, q4, scheme, s_star, chunk=2048):
    """acc = q . w8 (gemm.py:145-154) column block by column block, w8 from the
    codes by the reference's per-channel x16 (gemm.py:180) or FusedDequantQuant
    (gemm.py:130-142)."""
    m, n = q.shape[0], q4.shape[1]
    acc = np.empty((m, n), dtype=np.int32)
    for c0 in range(0, n, chunk):
        c1 = min(n, c0 + chunk)
        if scheme == O.PER_CHANNEL:
            w8 = q4[:, c0:c1].astype(np.int16) * 16
        else:
            w8 = O.fused_dequant_quant_cols(q4[:, c0:c1], s_star[:, c0:c1], GS)
        acc[:, c0:c1] = O.gemm_i8_i32_fast(q, w8)
    return acc


def _requant_chunked(q4, s_wg, chunk=2048):
    return np.concatenate([O.requant_scale(q4[:, c0:c0 + chunk], s_wg[:, c0:c0 + chunk])
                           for c0 in range(0, q4.shape[1], chunk)])


@functools.lru_cache(maxsize=6)
def case(k, n, scheme, m_max=1024):
    """Synthetic weights (SURVEY §8d recipe R2: uniform int4 codes, 0.02*U(0.5,1.5)
    scales, s_wc via requant_scale), fp16 activations, and the oracle's result at
    m_max tokens; GPU copies of the operands."""
    rng = np.random.default_rng(k * 100003 + n * 7 + (1 if scheme == O.PER_GROUP else 0))
    q4 = rng.integers(-8, 8, (k, n), dtype=np.int8)
    if scheme == O.PER_CHANNEL:
        qw_o = O.QuantizedWeights(O.pack_i4(q4), k, n, O.PER_CHANNEL, s_w=0.02 * rng.uniform(0.5, 1.5, n))
    else:
        s_wg = 0.02 * rng.uniform(0.5, 1.5, (k // GS, n))
        qw_o = O.QuantizedWeights(O.pack_i4(q4), k, n, O.PER_GROUP, GS, s_wg=s_wg, s_wc=_requant_chunked(q4, s_wg))
    fo = O.FusedScales.from_quantized(qw_o)
    x16 = rng.standard_normal((m_max, k)).astype(np.float16)
    aq_o = O.quant_act_per_token(x16.astype(np.float64))
    acc = _oracle_gemm(aq_o.q, q4, scheme, fo.s_star)
    y = O._epilogue(acc, aq_o.s_a, fo.s_w_folded if scheme == O.PER_CHANNEL else fo.s_wc)
    dev = torch.device("cuda")
    g = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    qw = Q.QuantizedWeights(g(qw_o.packed), k, n, scheme, GS if scheme == O.PER_GROUP else 0, s_w=g(qw_o.s_w),
                            s_wg=g(qw_o.s_wg), s_wc=g(qw_o.s_wc))
    fused = Q.FusedScales.from_quantized(qw)
    if scheme == O.PER_GROUP:
        assert torch.equal(fused.s_star.view(torch.int16).cpu(), torch.from_numpy(fo.s_star.view(np.int16)))
    return dict(qw=qw, fused=fused, x=g(x16), q=g(aq_o.q), s_a=g(aq_o.s_a), acc=g(acc),
                y=g(y.view(np.int16)), qw_o=qw_o, fo=fo)


# ---------------------------------------------------------------- plan lists


def candidate_plans(mode, m, n, k):
    """Every (ntok, split, csplit) the planner evaluates at this shape (the
    candidate loop of make_plan in csrc/w4a8_gemm.cu), resolved the way a launch
    resolves it, deduplicated; plus the planner's own choice first."""
    auto = G.plan_info(mode, m, n, k)
    seen, out = set(), []

    def add(cfg):
        info = G.plan_info(mode, m, n, k, cfg)
        key = (info["ntok"], info["split"], info["csplit"], info["grid"])
        if key not in seen:
            seen.add(key)
            out.append((cfg, info))

    add(None)
    for nt in (16, 32, 128, 192, 256):
        if nt > 32 and nt // 4 >= m:
            break
        if nt == 192:  # pair tiles only (whole tiles, stream-K, waves + stream-K)
            for sk in (3, 5, 6):
                add({"ntok": 192, "split": sk})
            continue
        for sk in (0, 1, 3, 4):
            if (sk == 3 and nt not in (128, 256)) or (sk == 4 and nt > 32 and nt != 128):
                continue
            if sk == 4:
                for s in (range(2, 9) if nt <= 32 else (2, 4)):
                    add({"ntok": nt, "split": 4, "csplit": s})
            else:
                add({"ntok": nt, "split": sk})
        if nt == 256:
            for sk in (5, 6):  # pair stream-K / pair waves + stream-K (forced-plan options)
                add({"ntok": 256, "split": sk})
    if m > 96:  # 384-token pair tiles (whole tiles only)
        add({"ntok": 384, "split": 3})
    return auto, out


def _run_and_check(c, m, mode, cfg, tag, with_acc=True):
    aq = Q.quant_act_per_token(c["x"][:m])
    assert torch.equal(aq.q, c["q"][:m]) and torch.equal(aq.s_a, c["s_a"][:m]), tag
    prep = G.prepare(c["qw"], c["fused"])
    assert prep.mode == mode
    out = G.run_gemm(aq, prep, c["qw"].cols, with_acc, cfg=cfg)
    if with_acc:
        assert torch.equal(out.acc, c["acc"][:m]), ("acc", tag)
    assert torch.equal(out.y.view(torch.int16), c["y"][:m]), ("y", tag)


def _sweep(k, n, scheme, ms):
    c = case(k, n, scheme)
    mode = _lib.MODE_PC if scheme == O.PER_CHANNEL else _lib.MODE_PG
    picked = []
    for m in ms:
        auto, plans = candidate_plans(mode, m, n, k)
        # the production call (public API, no acc) under the planner's choice
        aq = Q.quant_act_per_token(c["x"][:m])
        run = Q.w4a8_gemm_per_channel if scheme == O.PER_CHANNEL else Q.w4a8_gemm_per_group
        out = run(aq, c["qw"], c["fused"], with_acc=False)
        assert torch.equal(out.y.view(torch.int16), c["y"][:m]), (k, n, scheme, m, "auto/no-acc")
        for cfg, info in plans:
            _run_and_check(c, m, mode, cfg, (k, n, scheme, m, info))
        picked.append((m, auto))
        # a second launch of the planner's plan: split plans leave the workspace clean
        _run_and_check(c, m, mode, None, (k, n, scheme, m, "auto again"))
    return picked


@pytest.mark.parametrize("k,n", SHAPES_C2)
def test_c2_sweep_every_plan(k, n):
    picked = _sweep(k, n, O.PER_GROUP, MS_C2)
    assert len(picked) == len(MS_C2)


@pytest.mark.parametrize("scheme", [O.PER_CHANNEL, O.PER_GROUP])
@pytest.mark.parametrize("k,n", SHAPES_C3)
def test_c3_70b_every_plan(k, n, scheme):
    _sweep(k, n, scheme, [1, 16, 1024])


@pytest.mark.parametrize("scheme", [O.PER_CHANNEL, O.PER_GROUP])
def test_c1_per_channel_point(scheme):
    # BASELINE configs[0] (M=16, 4096^2) through every plan, both schemes
    _sweep(4096, 4096, scheme, [16])


# ------------------------------------------------------------------------ C4

C4_LINEARS = [("qkv", 4096, 12288), ("o", 4096, 4096), ("gate_up", 4096, 22016), ("down", 11008, 4096)]


@pytest.mark.parametrize("name,k,n", C4_LINEARS)
def test_c4_linears_apply_quant_linear(name, k, n):
    """apply_quant_linear (pipeline.py:144-152: x / s in f64, per-token quantize,
    per-group GEMM, y widened) at the C4 batches, against the oracle's restatement."""
    rng = np.random.default_rng(k * 7 + n)
    q4 = rng.integers(-8, 8, (k, n), dtype=np.int8)
    s_wg = 0.02 * rng.uniform(0.5, 1.5, (k // GS, n))
    qw_o = O.QuantizedWeights(O.pack_i4(q4), k, n, O.PER_GROUP, GS, s_wg=s_wg, s_wc=_requant_chunked(q4, s_wg))
    s = np.ones(k)
    idx = rng.permutation(k)[: k // 8]
    s[idx] = rng.uniform(0.5, 2.0, idx.size)
    x16 = rng.standard_normal((256, k)).astype(np.float16)
    # oracle: same steps as O.apply_quant_linear, with the chunked GEMM
    aq_o = O.quant_act_per_token(x16.astype(np.float64) / s[None, :])
    fo = O.FusedScales.from_quantized(qw_o)
    want = O._epilogue(_oracle_gemm(aq_o.q, q4, O.PER_GROUP, fo.s_star), aq_o.s_a, fo.s_wc).astype(np.float64)
    dev = torch.device("cuda")
    g = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    qw = Q.QuantizedWeights(g(qw_o.packed), k, n, "per-group", GS, s_wg=g(qw_o.s_wg), s_wc=g(qw_o.s_wc))
    layer = Q.QuantizedLayer(name, qw, Q.SmoothingPlan(1.0, tuple(int(i) for i in idx), s, 0.0))
    want_t = g(want)
    for b in (1, 16, 64, 256):
        y = Q.apply_quant_linear(g(x16[:b]), layer)
        assert y.dtype == torch.float64
        assert torch.equal(y.view(torch.int64), want_t[:b].view(torch.int64)), (name, b)


# ------------------------------------------------------------------------ C5


@pytest.mark.parametrize("scheme", [O.PER_CHANNEL, O.PER_GROUP])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_c5_nsplit_gate_up_shards(scheme, world):
    """Column-parallel 8192x28672: each rank's shard GEMM equals the oracle's
    columns of the unsplit GEMM; concatenated, the whole output."""
    k, n = 8192, 28672
    c = case(k, n, scheme)
    ops = tp.TPOps()
    ns = n // world
    for m in (1, 16, 1024):
        aq = ops.quant(c["x"][:m])
        for r in range(world):
            sh = tp.shard_nsplit(c["qw"], r, world)
            y = ops.gemm(aq, sh, Q.FusedScales.from_quantized(sh))
            assert torch.equal(y.view(torch.int16), c["y"][:m, r * ns:(r + 1) * ns]), (scheme, world, m, r)


@pytest.mark.parametrize("scheme", [O.PER_CHANNEL, O.PER_GROUP])
@pytest.mark.parametrize("k,n", [(28672, 8192), (8192, 8192)])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_c5_ksplit_shards(k, n, scheme, world):
    """Row-parallel down (28672x8192) and o_proj (8192x8192): per-rank absmax ->
    MAX -> quantize with the global max -> int32 partial GEMM -> SUM -> f64
    epilogue equals the oracle's unsplit GEMM (the NCCL collectives replaced by
    the same exact reductions on one GPU)."""
    c = case(k, n, scheme)
    ops = tp.TPOps()
    ks = k // world
    shards = [tp.shard_ksplit(c["qw"], r, world) for r in range(world)]
    fused = [Q.FusedScales.from_quantized(sh) for sh in shards]
    for m in (1, 16, 1024):
        x = c["x"][:m]
        row_max = torch.stack([ops.row_absmax(x[:, r * ks:(r + 1) * ks]) for r in range(world)]).max(0).values
        acc, s_a = None, None
        for r in range(world):
            aq = ops.quant_with_max(x[:, r * ks:(r + 1) * ks], row_max)
            assert torch.equal(aq.q, c["q"][:m, r * ks:(r + 1) * ks])
            part = ops.gemm_acc(aq, shards[r], fused[r])
            acc = part if acc is None else acc + part
            s_a = aq.s_a
        assert torch.equal(s_a, c["s_a"][:m])
        assert torch.equal(acc, c["acc"][:m]), (k, n, scheme, world, m)
        s_col = c["fused"].s_w_folded if scheme == O.PER_CHANNEL else c["fused"].s_wc
        y = ops.epilogue(acc, s_a, s_col)
        assert torch.equal(y.view(torch.int16), c["y"][:m]), (k, n, scheme, world, m)
