"""GPU parity: the sm_100a path vs the CPU oracle (pinned to the reference).

Integer outputs (codes, packed bytes, int32 accumulators) and the fp16 output
are required to be BIT-EXACT (tolerance 0): the kernel's epilogue is the
reference's f64 (acc*s_a)*s_col with one RN rounding to binary16, so the
BASELINE ≤1e-3 relative tolerance is met with margin 0.
"""

import numpy as np
import pytest
import torch

import paper_2406_09904_b200 as Q
from oracle import qqq_oracle as O

pytestmark = pytest.mark.gpu


def np_(t):
    return t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


def same_bits(a, b):
    a, b = np_(a), np_(b)
    if a.dtype == np.float16:
        return a.shape == b.shape and np.array_equal(a.view(np.uint16), b.astype(np.float16).view(np.uint16))
    if a.dtype == np.float64:
        return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.astype(np.float64).view(np.uint64))
    return a.shape == b.shape and np.array_equal(a, b)


def gpu_weights_from_case(c):
    t, k, n, gs, f16, pg = (int(v) for v in c["meta"])
    dev = torch.device("cuda")
    packed = torch.from_numpy(c["packed"]).to(dev)
    if pg:
        qw = Q.QuantizedWeights(packed, k, n, Q.PER_GROUP, gs, s_wg=torch.from_numpy(c["s_wg"]).to(dev),
                                s_wc=torch.from_numpy(c["s_wc"]).to(dev))
    else:
        qw = Q.QuantizedWeights(packed, k, n, Q.PER_CHANNEL, s_w=torch.from_numpy(c["s_w"]).to(dev))
    return qw


# ---------------------------------------------------------------- quantizers


def test_act_quant_golden(golden):
    for c in golden:
        x = c["x"]
        f16 = bool(c["meta"][4])
        xt = torch.from_numpy(x.astype(np.float16) if f16 else x).cuda()
        aq = Q.quant_act_per_token(xt)
        assert same_bits(aq.q, c["q"]), c["meta"]
        assert same_bits(aq.s_a, c["s_a"]), c["meta"]
        # f64 and f32 entry points agree with the reference as well
        aq64 = Q.quant_act_per_token(torch.from_numpy(x).cuda())
        assert same_bits(aq64.q, c["q"]) and same_bits(aq64.s_a, c["s_a"])


def test_act_quant_ties_and_edges():
    # rows whose absmax m is fixed and whose entries are every fp16 value in
    # [-m, m]: covers all exact ties x*127/m = n + 1/2 for those m
    rng = np.random.default_rng(11)
    bits = np.arange(0x0000, 0x7C00, dtype=np.uint16)
    vals = bits.view(np.float16)
    ms = np.concatenate([vals[rng.integers(1, vals.size, 48)], np.array([1.0, 127.0, 0.5, 65504.0, 6e-8],
                                                                          dtype=np.float16)])
    for m in ms:
        sel = vals[(vals.astype(np.float64) <= float(m))]
        row = np.concatenate([sel, -sel, np.array([m], dtype=np.float16)])
        x = row[None, :]
        want = O.quant_act_per_token(x.astype(np.float64))
        got = Q.quant_act_per_token(torch.from_numpy(x).cuda())
        assert same_bits(got.q, want.q), float(m)
        assert same_bits(got.s_a, want.s_a)


def test_act_quant_kat_and_errors():
    out = Q.quant_act_per_token(np.array([[0.0, 63.5, -127.0]]))  # test_quantize.py:23-27
    assert np_(out.s_a).tolist() == [1.0] and np_(out.q).tolist() == [[0, 64, -127]]
    out = Q.quant_act_per_token(np.zeros((1, 3)))
    assert np_(out.s_a).tolist() == [1.0] and np_(out.q).tolist() == [[0, 0, 0]]
    with pytest.raises(Q.DataError):
        Q.quant_act_per_token(np.array([[1.0, np.inf]]))
    with pytest.raises(Q.DataError):
        Q.quant_act_per_token(torch.tensor([[1.0, float("nan")]], dtype=torch.float16).cuda())
    with pytest.raises(Q.ShapeError):
        Q.quant_act_per_token(np.zeros(4))


def test_weight_quantizers_golden(golden):
    for c in golden:
        t, k, n, gs, f16, pg = (int(v) for v in c["meta"])
        if pg:
            qw = Q.quant_weight_per_group(c["w"], Q.QuantSpec("per-group", gs))
            assert same_bits(qw.s_wg, c["s_wg"]) and same_bits(qw.s_wc, c["s_wc"])
            fused = Q.FusedScales.from_quantized(qw)
            assert same_bits(fused.s_star, c["s_star"])
        else:
            qw = Q.quant_weight_per_channel(c["w"])
            assert same_bits(qw.s_w, c["s_w"])
            fused = Q.FusedScales.from_quantized(qw)
            assert same_bits(fused.s_w_folded, c["s_w_folded"])
        assert same_bits(qw.packed, c["packed"]), c["meta"]
        assert same_bits(qw.codes(), O.unpack_i4(c["packed"], k))


def test_packing_kats_and_errors():
    assert np_(Q.pack_i4(np.array([[-8], [7]], dtype=np.int8))).tolist() == [[0xF0]]
    assert np_(Q.pack_i4(np.array([[0], [0]], dtype=np.int8))).tolist() == [[0x88]]
    rng = np.random.default_rng(0)
    for k, n in ((1, 1), (7, 3), (33, 9), (256, 130)):
        qq = rng.integers(-8, 8, (k, n)).astype(np.int8)
        assert same_bits(Q.pack_i4(qq), O.pack_i4(qq))
        assert same_bits(Q.unpack_i4(Q.pack_i4(qq), k), qq)
    with pytest.raises(Q.DataError):
        Q.pack_i4(np.array([[8]], dtype=np.int16))
    with pytest.raises(Q.CorruptionError):
        Q.unpack_i4(Q.pack_i4(np.zeros((4, 2), dtype=np.int8)), 7)
    bad = O.pack_i4(np.zeros((3, 1), dtype=np.int8)).copy()
    bad[1, 0] = 0x08 | (0x3 << 4)
    with pytest.raises(Q.CorruptionError):
        Q.unpack_i4(bad, 3)
    assert np_(Q.requant_scale(np.array([[3], [1]], dtype=np.int8), np.array([[0.5]]))).tolist() == [1.5 / 127]


# --------------------------------------------------------------- conversions


def test_fused_dequant_quant_exhaustive():
    bits = np.arange(65536, dtype=np.uint16)
    vals = bits.view(np.float16).astype(np.float64)
    s_bits = bits[np.isfinite(vals) & (vals > 0)]
    S = s_bits.size
    q = np.tile(np.arange(-8, 8, dtype=np.int8), S)  # 16 codes per scale
    s_rep = np.repeat(s_bits, 16)
    want = O.fused_dequant_quant_cols(q.reshape(1, -1), s_rep.view(np.float16).reshape(1, -1), 1).ravel()
    got = Q.gemm.fused_dequant_quant_array(q, s_rep, word_path=False)
    assert np.array_equal(got, want)
    # the GEMM's HFMA2 word path: exact wherever the repack admits the fast path
    s_word = np.repeat(s_bits, 2)  # two words (16 codes) per scale
    got_w = Q.gemm.fused_dequant_quant_array(q, s_word, word_path=True)
    sv = s_bits.view(np.float16).astype(np.float64)
    with np.errstate(over="ignore"):  # huge s*: the f16 cast overflows to inf (not admissible)
        r_lo = (-8 * sv + 1152).astype(np.float16).astype(np.float64)
        r_hi = (7 * sv + 1152).astype(np.float16).astype(np.float64)
    admissible = (r_lo >= 1025) & (r_hi <= 1279)  # tiny s* included: both paths give 1152
    adm = np.repeat(admissible, 16)
    assert admissible.sum() > 14000
    assert np.array_equal(got_w[adm], want[adm])


def test_fast_conversions_exhaustive():
    bits = np.arange(65536, dtype=np.uint16)
    vals = bits.view(np.float16).astype(np.float64)
    inr = np.isfinite(vals) & (vals >= -128.0) & (vals < 127.5)
    assert np.array_equal(Q.gemm.fast_f16_to_i8_bits(bits[inr]), O.fast_f16_to_i8_bits(bits[inr]))
    codes = np.arange(-8, 8, dtype=np.int8)
    assert np.array_equal(Q.gemm.fast_i4_to_i8_array(codes).astype(np.int32), 16 * codes.astype(np.int32))
    assert Q.fast_i4_to_i8(7) == 112 and Q.fast_i4_to_i8(-8) == -128
    for u in range(16):
        assert Q.fast_i4_to_f16(u).to_float() == u - 8
    assert Q.fused_dequant_quant(8 + 3, Q.encode_f16(42.34375)) == 127
    with pytest.raises(Q.ConfigError):
        Q.fused_dequant_quant(3, Q.Binary16(0x7C00))


# ---------------------------------------------------------------------- GEMM


def _gemm_case(c, aq=None):
    t, k, n, gs, f16, pg = (int(v) for v in c["meta"])
    qw = gpu_weights_from_case(c)
    fused = Q.FusedScales.from_quantized(qw)
    if aq is None:
        aq = Q.QuantizedActivations(torch.from_numpy(c["q"]).cuda(), torch.from_numpy(c["s_a"]).cuda())
    run = Q.w4a8_gemm_per_group if pg else Q.w4a8_gemm_per_channel
    return run(aq, qw, fused)


def test_gemm_golden_bit_exact(golden):
    for c in golden:
        out = _gemm_case(c)
        assert same_bits(out.acc, c["acc"]), c["meta"]
        assert same_bits(out.y, c["y"]), c["meta"]


def test_gemm_hand_traces():
    # test_gemm.py:162-175 per-channel
    aq = Q.QuantizedActivations(torch.tensor([[2]], dtype=torch.int8).cuda(), torch.tensor([0.1]).double().cuda())
    qw = Q.QuantizedWeights(Q.pack_i4(np.array([[3]], dtype=np.int8)), 1, 1, "per-channel",
                            s_w=torch.tensor([0.2], dtype=torch.float64).cuda())
    out = Q.w4a8_gemm_per_channel(aq, qw, Q.FusedScales.from_quantized(qw))
    assert np_(out.acc).tolist() == [[96]]
    assert float(np_(out.y)[0, 0]) == float(np.float16(96 * 0.1 * (0.2 / 16)))
    # test_gemm.py:234-256 per-group (g = 2 -> exact int8 layout)
    aq = Q.QuantizedActivations(torch.tensor([[10, 20]], dtype=torch.int8).cuda(),
                                torch.tensor([0.05], dtype=torch.float64).cuda())
    q4 = np.array([[3], [-2]], dtype=np.int8)
    s_wg = torch.tensor([[0.5]], dtype=torch.float64).cuda()
    s_wc = Q.requant_scale(q4, s_wg)
    qw = Q.QuantizedWeights(Q.pack_i4(q4), 2, 1, "per-group", 2, s_wg=s_wg, s_wc=s_wc)
    fused = Q.FusedScales.from_quantized(qw)
    assert float(np_(fused.s_star)[0, 0]) == 42.34375
    out = Q.w4a8_gemm_per_group(aq, qw, fused)
    assert np_(out.acc).tolist() == [[-430]]


def test_gemm_validation_errors(golden):
    c = golden[6]  # per-group case
    qw = gpu_weights_from_case(c)
    fused = Q.FusedScales.from_quantized(qw)
    aq = Q.QuantizedActivations(torch.from_numpy(c["q"]).cuda(), torch.from_numpy(c["s_a"]).cuda())
    with pytest.raises(Q.ConfigError):
        Q.w4a8_gemm_per_channel(aq, qw, fused)
    bad = Q.QuantizedActivations(aq.q[:, :-1], aq.s_a)
    with pytest.raises(Q.ShapeError):
        Q.w4a8_gemm_per_group(bad, qw, fused)
    with pytest.raises(Q.ShapeError):
        Q.w4a8_gemm_per_group(Q.QuantizedActivations(aq.q, aq.s_a[:-1]), qw, fused)


def _rand_problem(m, k, n, scheme, gs, seed):
    rng = np.random.default_rng(seed)
    x16 = rng.standard_normal((m, k)).astype(np.float16)
    q4 = rng.integers(-8, 8, (k, n)).astype(np.int8)
    if scheme == "per-channel":
        s_w = 0.02 * rng.uniform(0.5, 1.5, n)
        qw_o = O.QuantizedWeights(O.pack_i4(q4), k, n, O.PER_CHANNEL, s_w=s_w)
    else:
        s_wg = 0.02 * rng.uniform(0.5, 1.5, (k // gs, n))
        qw_o = O.QuantizedWeights(O.pack_i4(q4), k, n, O.PER_GROUP, gs, s_wg=s_wg, s_wc=O.requant_scale(q4, s_wg))
    return x16, qw_o


def _to_gpu_qw(qw_o):
    dev = torch.device("cuda")
    f = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    return Q.QuantizedWeights(f(qw_o.packed), qw_o.rows, qw_o.cols, qw_o.scheme, qw_o.group_size, s_w=f(qw_o.s_w),
                              s_wg=f(qw_o.s_wg), s_wc=f(qw_o.s_wc))


@pytest.mark.parametrize("scheme,gs", [("per-channel", 0), ("per-group", 128), ("per-group", 32),
                                       ("per-group", 512)])
def test_gemm_m_sweep_vs_oracle(scheme, gs):
    k, n = 1024, 384
    for m in (1, 2, 5, 16, 17, 31, 48, 64, 65, 100, 128, 129, 200, 256, 300, 513):
        x16, qw_o = _rand_problem(m, k, n, scheme, gs or 128, seed=m)
        aq_o = O.quant_act_per_token(x16.astype(np.float64))
        fused_o = O.FusedScales.from_quantized(qw_o)
        run_o = O.w4a8_gemm_per_channel if scheme == "per-channel" else O.w4a8_gemm_per_group
        want = run_o(aq_o, qw_o, fused_o, fast=True)
        qw = _to_gpu_qw(qw_o)
        fused = Q.FusedScales.from_quantized(qw)
        aq = Q.quant_act_per_token(torch.from_numpy(x16).cuda())
        run = Q.w4a8_gemm_per_channel if scheme == "per-channel" else Q.w4a8_gemm_per_group
        out = run(aq, qw, fused)
        assert same_bits(aq.q, aq_o.q)
        assert same_bits(out.acc, want.acc), (scheme, gs, m)
        assert same_bits(out.y, want.y), (scheme, gs, m)


@pytest.mark.parametrize("ntok", [16, 32, 64, 128, 256])
@pytest.mark.parametrize("split", [0, 1, 2])
def test_gemm_all_tile_plans(ntok, split):
    m, k, n = 77, 2304, 640
    for scheme in ("per-channel", "per-group"):
        x16, qw_o = _rand_problem(m, k, n, scheme, 128, seed=ntok + split)
        aq_o = O.quant_act_per_token(x16.astype(np.float64))
        run_o = O.w4a8_gemm_per_channel if scheme == "per-channel" else O.w4a8_gemm_per_group
        want = run_o(aq_o, qw_o, O.FusedScales.from_quantized(qw_o), fast=True)
        qw = _to_gpu_qw(qw_o)
        fused = Q.FusedScales.from_quantized(qw)
        aq = Q.quant_act_per_token(torch.from_numpy(x16).cuda())
        prep = Q.gemm.prepare(qw, fused)
        for grid in (0, 7, 148, 1000):
            out = Q.gemm.run_gemm(aq, prep, n, True, cfg={"ntok": ntok, "split": split, "grid": grid})
            assert same_bits(out.acc, want.acc), (scheme, ntok, split, grid)
            assert same_bits(out.y, want.y), (scheme, ntok, split, grid)
            if split == 0:
                break


@pytest.mark.parametrize("scheme,gs", [("per-channel", 0), ("per-group", 128), ("per-group", 32)])
@pytest.mark.parametrize("ntok", [256, 192, 384, 128])
def test_gemm_pair_tiles(scheme, gs, ntok):
    """2-CTA pair plans (tcgen05.mma.cta_group::2, 256-channel x 256-, 192- or
    384-token tiles; the 192-token tile double-buffers its accumulators, the
    384-token tile issues two N=192 MMAs per K step; whole tiles only): whole
    tiles, stream-K and hybrid; odd channel-tile counts, ragged tokens, partial
    last k-block, few pairs, several tiles per pair."""
    for (m, k, n, grid) in ((77, 2304, 640, 0), (256, 1024, 384, 0), (300, 896, 1024, 0), (600, 1152, 1000, 7),
                            (1, 256, 128, 0), (513, 4096, 256, 4), (1024, 1024, 1280, 4)):
        x16, qw_o = _rand_problem(m, k, n, scheme, gs or 128, seed=m + n)
        aq_o = O.quant_act_per_token(x16.astype(np.float64))
        run_o = O.w4a8_gemm_per_channel if scheme == "per-channel" else O.w4a8_gemm_per_group
        want = run_o(aq_o, qw_o, O.FusedScales.from_quantized(qw_o), fast=True)
        qw = _to_gpu_qw(qw_o)
        prep = Q.gemm.prepare(qw, Q.FusedScales.from_quantized(qw))
        aq = Q.quant_act_per_token(torch.from_numpy(x16).cuda())
        # 3 = whole pair tiles, 5 = stream-K over pair units, 6 = whole-tile waves + stream-K remainder
        for split in (3, 5, 6):
            for _ in range(2):  # the split plans must leave the workspace zeroed for the next launch
                out = Q.gemm.run_gemm(aq, prep, n, True, cfg={"ntok": ntok, "split": split, "grid": grid})
                assert same_bits(out.acc, want.acc), (scheme, gs, ntok, m, k, n, grid, split)
                assert same_bits(out.y, want.y), (scheme, gs, ntok, m, k, n, grid, split)


@pytest.mark.parametrize("scheme,gs", [("per-channel", 0), ("per-group", 128), ("per-group", 32)])
@pytest.mark.parametrize("ntok", [16, 32])
def test_gemm_cluster_splitk(scheme, gs, ntok):
    """Cluster split-K plan (split=4): one tile per cluster of S in {8, 4, 2} decode
    CTAs, int32 partials reduce-scattered over DSMEM; ragged M, partial last k-block."""
    for (m, k, n) in ((1, 4096, 4096), (16, 2048, 11008), (5, 1024, 640), (31, 2304, 384), (13, 4352, 256),
                      (100, 4096, 4096), (128, 1024, 1280), (3, 4096, 11008), (2, 1792, 5376), (4, 2560, 7552)):
        x16, qw_o = _rand_problem(m, k, n, scheme, gs or 128, seed=m * 7 + n)
        aq_o = O.quant_act_per_token(x16.astype(np.float64))
        run_o = O.w4a8_gemm_per_channel if scheme == "per-channel" else O.w4a8_gemm_per_group
        want = run_o(aq_o, qw_o, O.FusedScales.from_quantized(qw_o), fast=True)
        qw = _to_gpu_qw(qw_o)
        prep = Q.gemm.prepare(qw, Q.FusedScales.from_quantized(qw))
        aq = Q.quant_act_per_token(torch.from_numpy(x16).cuda())
        for _ in range(2):  # second launch: the plan leaves no state behind
            out = Q.gemm.run_gemm(aq, prep, n, True, cfg={"ntok": ntok, "split": 4})
            assert same_bits(out.acc, want.acc), (scheme, gs, ntok, m, k, n)
            assert same_bits(out.y, want.y), (scheme, gs, ntok, m, k, n)


@pytest.mark.parametrize("scheme,gs", [("per-channel", 0), ("per-group", 128), ("per-group", 32)])
@pytest.mark.parametrize("cs", [2, 4])
def test_gemm_cluster_splitk_128_token_tiles(scheme, gs, cs):
    """Big-CTA cluster split-K (128-token tiles, S in {2, 4} whole-SM CTAs, int32
    partials reduce-scattered over DSMEM by token range): ragged M (token ranges
    with no valid token, partial 16-token chunks), several token tiles, partial
    last k-block, both schemes; a second launch leaves no state behind."""
    for (m, k, n) in ((1, 4096, 4096), (16, 2048, 1280), (33, 2304, 384), (64, 4096, 4096), (100, 1024, 640),
                      (128, 4352, 256), (129, 2048, 512), (300, 1792, 1280), (512, 4096, 4096)):
        x16, qw_o = _rand_problem(m, k, n, scheme, gs or 128, seed=m * 3 + k + n)
        aq_o = O.quant_act_per_token(x16.astype(np.float64))
        run_o = O.w4a8_gemm_per_channel if scheme == "per-channel" else O.w4a8_gemm_per_group
        want = run_o(aq_o, qw_o, O.FusedScales.from_quantized(qw_o), fast=True)
        qw = _to_gpu_qw(qw_o)
        prep = Q.gemm.prepare(qw, Q.FusedScales.from_quantized(qw))
        aq = Q.quant_act_per_token(torch.from_numpy(x16).cuda())
        cfg = {"ntok": 128, "split": 4, "csplit": cs}
        info = Q.gemm.plan_info(prep.mode, m, n, k, cfg)
        for _ in range(2):
            out = Q.gemm.run_gemm(aq, prep, n, True, cfg=cfg)
            assert same_bits(out.acc, want.acc), (scheme, gs, cs, m, k, n, info)
            assert same_bits(out.y, want.y), (scheme, gs, cs, m, k, n, info)
        y_only = Q.gemm.run_gemm(aq, prep, n, False, cfg=cfg)  # the serving path (TMA y stores, no acc)
        assert same_bits(y_only.y, want.y), (scheme, gs, cs, m, k, n, info, "no-acc")


def test_gemm_plans_share_a_zeroed_workspace():
    """Every plan leaves the shared split-K workspace zeroed (counters re-armed,
    slots returned to zero): a chain of GEMMs of different shapes and plans —
    stream-K, hybrid, pair stream-K, cluster split-K — on ONE workspace stays
    bit-exact, twice over."""
    cases = [((128, 4096, 512), {"ntok": 128, "split": 1}), ((77, 2304, 640), {"ntok": 128, "split": 2}),
             ((300, 1024, 1024), {"ntok": 256, "split": 5}), ((16, 4096, 4096), {"ntok": 16, "split": 1}),
             ((5, 2048, 1280), {"ntok": 16, "split": 4}), ((600, 1152, 1000), {"ntok": 256, "split": 6})]
    import paper_2406_09904_b200._lib as L
    need = max(L.load().qqq_gemm_workspace_bytes(m, n, k) for (m, k, n), _ in cases)
    ws = torch.zeros(need, dtype=torch.uint8, device="cuda")
    for rep in range(2):
        for (m, k, n), cfg in cases:
            x16, qw_o = _rand_problem(m, k, n, "per-group", 128, seed=m + k + n + rep)
            aq_o = O.quant_act_per_token(x16.astype(np.float64))
            want = O.w4a8_gemm_per_group(aq_o, qw_o, O.FusedScales.from_quantized(qw_o), fast=True)
            qw = _to_gpu_qw(qw_o)
            prep = Q.gemm.prepare(qw, Q.FusedScales.from_quantized(qw))
            aq = Q.quant_act_per_token(torch.from_numpy(x16).cuda())
            out = Q.gemm.run_gemm(aq, prep, n, True, cfg=cfg, ws=ws)
            assert same_bits(out.acc, want.acc), (m, k, n, cfg, rep)
            assert same_bits(out.y, want.y), (m, k, n, cfg, rep)
    torch.cuda.synchronize()
    assert int(ws.count_nonzero()) == 0  # counters re-armed, every slot returned to zero


def test_gemm_ragged_shapes():
    for (m, k, n, scheme, gs) in ((3, 33, 5, "per-channel", 0), (9, 100, 130, "per-channel", 0),
                                  (4, 96, 129, "per-group", 32), (2, 300, 1, "per-group", 100)):
        rng = np.random.default_rng(m * 1000 + k)
        x = rng.standard_normal((m, k)) * 3
        w = rng.standard_normal((k, n))
        aq_o = O.quant_act_per_token(x)
        qw_o = O.quant_weight_per_channel(w) if scheme == "per-channel" else O.quant_weight_per_group(w, gs)
        fo = O.FusedScales.from_quantized(qw_o)
        want = (O.w4a8_gemm_per_channel if scheme == "per-channel" else O.w4a8_gemm_per_group)(aq_o, qw_o, fo)
        aq = Q.quant_act_per_token(x)
        qw = (Q.quant_weight_per_channel(w) if scheme == "per-channel"
              else Q.quant_weight_per_group(w, Q.QuantSpec("per-group", gs)))
        fused = Q.FusedScales.from_quantized(qw)
        out = (Q.w4a8_gemm_per_channel if scheme == "per-channel" else Q.w4a8_gemm_per_group)(aq, qw, fused)
        assert same_bits(out.acc, want.acc), (m, k, n, scheme)
        assert same_bits(out.y, want.y), (m, k, n, scheme)


def test_gemm_per_group_clamp_fallback():
    # s* large enough that FusedDequantQuant saturates: the repack must route
    # through the exact (clamping) int8 layout and still match the reference.
    rng = np.random.default_rng(5)
    m, k, n, gs = 8, 256, 128, 128
    q4 = rng.integers(-8, 8, (k, n)).astype(np.int8)
    s_star = np.full((k // gs, n), 30.0, dtype=np.float16)  # 8*30 > 127 -> clamps
    s_star[0, :5] = np.float16(1e-5)  # tiny scales too
    s_wc = rng.uniform(0.01, 0.02, n)
    x16 = rng.standard_normal((m, k)).astype(np.float16)
    aq_o = O.quant_act_per_token(x16.astype(np.float64))
    qw_o = O.QuantizedWeights(O.pack_i4(q4), k, n, O.PER_GROUP, gs, s_wg=None, s_wc=s_wc)
    fo = O.FusedScales(O.PER_GROUP, s_star=s_star, s_wc=s_wc)
    want = O.w4a8_gemm_per_group(aq_o, qw_o, fo)
    qw = Q.QuantizedWeights(torch.from_numpy(qw_o.packed).cuda(), k, n, "per-group", gs,
                            s_wc=torch.from_numpy(s_wc).cuda())
    fused = Q.FusedScales("per-group", s_star=torch.from_numpy(s_star).cuda(), s_wc=torch.from_numpy(s_wc).cuda())
    assert Q.gemm.prepare(qw, fused).mode == 2
    out = Q.w4a8_gemm_per_group(Q.quant_act_per_token(torch.from_numpy(x16).cuda()), qw, fused)
    assert same_bits(out.acc, want.acc) and same_bits(out.y, want.y)


def test_gemm_i8_i32():
    rng = np.random.default_rng(2)
    for m, k, n in ((1, 2, 1), (8, 8, 8), (33, 520, 200), (256, 1024, 256)):
        a = rng.integers(-127, 128, (m, k)).astype(np.int8)
        b = rng.integers(-128, 128, (k, n)).astype(np.int8)
        assert same_bits(Q.gemm_i8_i32(a, b), O.gemm_i8_i32(a, b))
    with pytest.raises(Q.ShapeError):
        Q.gemm_i8_i32(np.zeros((1, 3), np.int8), np.zeros((2, 1), np.int8))


def test_gemm_overflow_to_inf():
    # y overflows binary16 -> +-inf, silently, like the reference (gemm.py:183)
    aq = Q.QuantizedActivations(torch.full((1, 256), 127, dtype=torch.int8).cuda(),
                                torch.tensor([1e3], dtype=torch.float64).cuda())
    qw = Q.QuantizedWeights(Q.pack_i4(np.full((256, 1), 7, np.int8)), 256, 1, "per-channel",
                            s_w=torch.tensor([1e3], dtype=torch.float64).cuda())
    out = Q.w4a8_gemm_per_channel(aq, qw, Q.FusedScales.from_quantized(qw))
    assert np.isinf(np_(out.y)[0, 0]) and np_(out.y)[0, 0] > 0


@pytest.mark.parametrize("scheme", ["per-channel", "per-group"])
def test_c1_golden_digests(digests, scheme):
    d = digests[f"C1/{scheme}"]
    x16, w = O.recipe_r1(16, 4096, 4096, seed=0)
    aq = Q.quant_act_per_token(torch.from_numpy(x16).cuda())
    assert O.digest(np_(aq.q)) == d["q"] and O.digest(np_(aq.s_a)) == d["s_a"]
    if scheme == "per-channel":
        qw = Q.quant_weight_per_channel(w)
    else:
        qw = Q.quant_weight_per_group(w, Q.QuantSpec("per-group", 128))
    assert O.digest(np_(qw.packed)) == d["packed"]
    fused = Q.FusedScales.from_quantized(qw)
    run = Q.w4a8_gemm_per_channel if scheme == "per-channel" else Q.w4a8_gemm_per_group
    out = run(aq, qw, fused)
    assert O.digest(np_(out.acc)) == d["acc"]
    assert O.digest(np_(out.y)) == d["y"]


def test_c2_golden_digests(digests):
    for (k, n) in ((4096, 4096), (4096, 11008), (11008, 4096)):
        d = digests[f"C2/{k}x{n}/M4"]
        rng = np.random.default_rng(1000 * 2 + 4)
        x = rng.standard_normal((4, k))
        w = rng.standard_normal((k, n))
        aq = Q.quant_act_per_token(torch.from_numpy(x.astype(np.float16)).cuda())
        qw = Q.quant_weight_per_group(w, Q.QuantSpec("per-group", 128))
        fused = Q.FusedScales.from_quantized(qw)
        out = Q.w4a8_gemm_per_group(aq, qw, fused)
        assert O.digest(np_(aq.q)) == d["q"]
        assert O.digest(np_(qw.packed)) == d["packed"] and O.digest(np_(fused.s_star)) == d["s_star"]
        assert O.digest(np_(out.acc)) == d["acc"] and O.digest(np_(out.y)) == d["y"]


@pytest.mark.parametrize("m,n,ntok,split", [(64, 256, 0, -1), (1024, 512, 0, -1), (200, 384, 128, 1),
                                            (16, 512, 16, 4)])
def test_gemm_epilogue_exact_f16_ties(m, n, ntok, split):
    """Outputs on exact f16 rounding midpoints: integer activations with s_a = 1
    and weights q * 2^-8 (s_w = 2^-8) make y = a * 2^-8 (a = sum x q), a tie
    whenever a is odd in [2048, 4096) (or 2 mod 4 in [4096, 8192), ...). The epilogue's fp32
    fast path must hand every tie (and every value near one) to the f64 path:
    y bit-identical to the reference's f16((acc * s_a) * s_w/16), ties to even."""
    rng = np.random.default_rng(m + n)
    k = 256
    x = rng.integers(-127, 128, (m, k)).astype(np.float64)
    x[:, 0] = 127.0  # s_a = 127 / 127 = 1
    q = rng.integers(-7, 8, (k, n))
    q[0, :] = 7  # column max 7 * 2^-8 -> s_w = 2^-8, codes = q
    w = q * 2.0 ** -8
    qw_o = O.quant_weight_per_channel(w)
    assert np.all(qw_o.s_w == 2.0 ** -8)
    x16 = x.astype(np.float16)
    aq_o = O.quant_act_per_token(x16.astype(np.float64))
    want = O.w4a8_gemm_per_channel(aq_o, qw_o, O.FusedScales.from_quantized(qw_o), fast=True)
    a = want.acc.astype(np.int64) // 16  # acc carries the x16 of w8 = 16 q (gemm.py:180)
    assert np.sum((np.abs(a) >= 2048) & (np.abs(a) < 4096) & (a % 2 == 1)) > 0  # ties present
    qw = _to_gpu_qw(qw_o)
    fused = Q.FusedScales.from_quantized(qw)
    aq = Q.quant_act_per_token(torch.from_numpy(x16).cuda())
    from paper_2406_09904_b200 import gemm as G

    cfg = None if ntok == 0 else {"ntok": ntok, "split": split}
    out = G.run_gemm(aq, G.prepare(qw, fused), n, True, cfg=cfg)
    assert same_bits(out.acc, want.acc)
    assert same_bits(out.y, want.y), (m, n, ntok, split)
