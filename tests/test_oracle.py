"""Pin the CPU oracle against the reference (CPU-only, no GPU needed).

The oracle (oracle/qqq_oracle.py) is the checker for every GPU parity test,
so before trusting it we check it against:
  * golden vectors produced by the reference itself (tests/golden/*),
  * the reference's own known-answer tests (pkg/tests/test_gemm.py,
    test_quantize.py), restated here with the same inputs and answers.
"""

import numpy as np
import pytest

from oracle import qqq_oracle as O


def _run(c):
    t, k, n, gs, f16, pg = (int(v) for v in c["meta"])
    aq = O.quant_act_per_token(c["x"])
    if pg:
        qw = O.quant_weight_per_group(c["w"], gs)
    else:
        qw = O.quant_weight_per_channel(c["w"])
    fused = O.FusedScales.from_quantized(qw)
    run = O.w4a8_gemm_per_group if pg else O.w4a8_gemm_per_channel
    return aq, qw, fused, run(aq, qw, fused), run(aq, qw, fused, fast=True)


def test_small_cases_bit_exact(golden):
    assert len(golden) >= 10
    for c in golden:
        aq, qw, fused, out, fast = _run(c)
        assert np.array_equal(aq.q, c["q"])
        assert np.array_equal(aq.s_a.view(np.uint64), c["s_a"].view(np.uint64))
        assert np.array_equal(qw.packed, c["packed"])
        if "s_star" in c:
            assert np.array_equal(fused.s_star.view(np.uint16), c["s_star"].view(np.uint16))
            assert np.array_equal(fused.s_wc, c["s_wc"])
        else:
            assert np.array_equal(fused.s_w_folded, c["s_w_folded"])
        for o in (out, fast):
            assert np.array_equal(o.acc, c["acc"])
            assert np.array_equal(o.y.view(np.uint16), c["y"].view(np.uint16))


@pytest.mark.parametrize("scheme", ["per-channel", "per-group"])
def test_c1_digests(digests, scheme):
    d = digests[f"C1/{scheme}"]
    x16, w = O.recipe_r1(16, 4096, 4096, seed=0)
    assert O.digest(x16) == d["x16"]
    aq = O.quant_act_per_token(x16.astype(np.float64))
    assert O.digest(aq.q) == d["q"] and O.digest(aq.s_a) == d["s_a"]
    if scheme == "per-channel":
        qw = O.quant_weight_per_channel(w)
    else:
        qw = O.quant_weight_per_group(w, 128)
    fused = O.FusedScales.from_quantized(qw)
    assert O.digest(qw.packed) == d["packed"]
    run = O.w4a8_gemm_per_channel if scheme == "per-channel" else O.w4a8_gemm_per_group
    out = run(aq, qw, fused, fast=True)
    assert O.digest(out.acc) == d["acc"]
    assert O.digest(out.y) == d["y"]
    assert out.y[0, :4].astype(float).tolist() == d["y_row0"]


def test_fused_dequant_quant_table_digest(digests):
    bits = np.arange(65536, dtype=np.uint16)
    vals = bits.view(np.float16).astype(np.float64)
    s_all = bits[np.isfinite(vals) & (vals > 0)].view(np.float16)
    q4 = np.repeat(np.arange(-8, 8, dtype=np.int8)[:, None], s_all.size, axis=1)
    table = O.fused_dequant_quant_cols(q4, s_all[None, :], 16)
    d = digests["fused_dequant_quant_table"]
    assert s_all.size == d["n_scales"]
    assert O.digest(table) == d["digest"]


def test_fast_f16_to_i8_digest(digests):
    bits = np.arange(65536, dtype=np.uint16)
    vals = bits.view(np.float16).astype(np.float64)
    inr = np.isfinite(vals) & (vals >= -128.0) & (vals < 127.5)
    got = O.fast_f16_to_i8_bits(bits[inr])
    assert O.digest(got) == digests["fast_f16_to_i8_inrange"]["digest"]
    assert np.array_equal(got.astype(np.int64), np.rint(vals[inr]).astype(np.int64))


# ---- the reference's own known-answer tests, restated on the oracle --------


def test_kat_act_quant():  # test_quantize.py:23-32
    out = O.quant_act_per_token(np.array([[0.0, 63.5, -127.0]]))
    assert out.s_a.tolist() == [1.0] and out.q.tolist() == [[0, 64, -127]]
    out = O.quant_act_per_token(np.zeros((1, 3)))
    assert out.s_a.tolist() == [1.0] and out.q.tolist() == [[0, 0, 0]]


def test_kat_packing():  # test_quantize.py:133-135
    assert O.pack_i4(np.array([[-8], [7]], dtype=np.int8)).tolist() == [[0xF0]]
    assert O.pack_i4(np.array([[0], [0]], dtype=np.int8)).tolist() == [[0x88]]


def test_kat_requant():  # test_quantize.py:113-117
    assert O.requant_scale(np.array([[3], [1]], dtype=np.int8), np.array([[0.5]])).tolist() == [1.5 / 127]


def test_kat_per_channel_hand_trace():  # test_gemm.py:162-175
    aq = O.QuantizedActivations(np.array([[2]], dtype=np.int8), np.array([0.1]))
    qw = O.QuantizedWeights(O.pack_i4(np.array([[3]], dtype=np.int8)), 1, 1, O.PER_CHANNEL, s_w=np.array([0.2]))
    out = O.w4a8_gemm_per_channel(aq, qw, O.FusedScales.from_quantized(qw))
    assert out.acc.tolist() == [[96]]
    assert float(out.y[0, 0]) == float(np.float16(96 * 0.1 * (0.2 / 16)))


def test_kat_per_group_hand_example():  # test_gemm.py:234-256
    aq = O.QuantizedActivations(np.array([[10, 20]], dtype=np.int8), np.array([0.05]))
    q4 = np.array([[3], [-2]], dtype=np.int8)
    s_wg = np.array([[0.5]])
    s_wc = O.requant_scale(q4, s_wg)
    qw = O.QuantizedWeights(O.pack_i4(q4), 2, 1, O.PER_GROUP, 2, s_wg=s_wg, s_wc=s_wc)
    fused = O.FusedScales.from_quantized(qw)
    assert float(fused.s_star[0, 0]) == 42.34375
    out = O.w4a8_gemm_per_group(aq, qw, fused)
    assert out.acc.tolist() == [[-430]]


def test_kat_fused_dequant_quant():  # test_gemm.py:89-113
    f = lambda u, s: int(O.fused_dequant_quant_cols(np.array([[u - 8]]), np.array([[s]], np.float16), 1)[0, 0])
    assert f(12, 2.0) == 8
    assert f(8 + 3, 42.34375) == 127
    assert f(15, 1000.0) == 127 and f(0, 1000.0) == -127 and f(0, 16.0) == -127
    rng = np.random.default_rng(0)
    for _ in range(500):
        u = int(rng.integers(0, 16))
        s = float(np.float16(float(np.abs(rng.standard_normal()) * 10 + 1e-3)))
        assert f(u, s) == int(np.clip(np.rint((u - 8) * s), -127, 127))


def test_faithful_and_fast_gemm_agree():
    rng = np.random.default_rng(3)
    a = rng.integers(-127, 128, (8, 2048)).astype(np.int8)
    b = rng.integers(-128, 128, (2048, 24)).astype(np.int8)
    assert np.array_equal(O.gemm_i8_i32(a, b), O.gemm_i8_i32_fast(a, b))


def test_oracle_calibration_vs_reference_goldens():
    """The calibration restatements reproduce the reference's own outputs
    (tests/golden/make_golden_{smoothing,gptq}.py): search_sigma's plan and
    candidate objectives exactly, the GPTQ sweep's codes and scales exactly."""
    import os

    here = os.path.join(os.path.dirname(__file__), "golden")
    d = np.load(os.path.join(here, "smoothing_cases.npz"))
    for i in range(int(d["n_cases"])):
        m, k, n, g = (int(v) for v in d[f"c{i}_meta"])
        x, w = d[f"c{i}_x"], d[f"c{i}_w"]
        assert np.array_equal(O.matmul_ref(x, w).view(np.uint64), d[f"c{i}_exact"].view(np.uint64))
        sigma, sel, s, obj = O.search_sigma(x, w, g if bool(d[f"c{i}_pg"]) else 0, int(d[f"c{i}_grid"]))
        assert sigma == float(d[f"c{i}_sigma"]) and obj == float(d[f"c{i}_obj"])
        assert sel == tuple(int(t) for t in np.flatnonzero(d[f"c{i}_sel"]))
        assert np.array_equal(s.view(np.uint64), d[f"c{i}_s"].view(np.uint64))
    d = np.load(os.path.join(here, "gptq_cases.npz"))
    for i in range(int(d["n_cases"])):
        m, k, n, g, bs = (int(v) for v in d[f"c{i}_meta"])
        codes, scales, col_err = O.gptq_sweep(d[f"c{i}_w"], d[f"c{i}_u"], d[f"c{i}_dead"], g, bs)
        assert np.array_equal(codes, d[f"c{i}_codes"]), i
        assert np.array_equal(scales.view(np.uint64), d[f"c{i}_scales"].view(np.uint64)), i
        assert np.array_equal(col_err.view(np.uint64), d[f"c{i}_col_errors"].view(np.uint64)), i
