"""One small W4A8 GEMM per tile plan and mode, checked bit-exactly against the
oracle: the workload compute-sanitizer (racecheck / synccheck / memcheck)
runs over (scripts/sanitize.sh -> profiles/r02_sanitizer_*.txt).

Plans (csrc/w4a8_gemm.cu plan_for): split 0 whole tiles, 1 stream-K, 2 hybrid,
3 pair tiles (cta_group::2), 4 cluster split-K (DSMEM), 5 pair stream-K,
6 pair waves + stream-K; modes PC / PG / I8 (clamp fallback layout).
Also the activation quantizers (plain, smoothed, with the reciprocal table).
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2406_09904_b200 as Q  # noqa: E402
from paper_2406_09904_b200 import _lib  # noqa: E402
from paper_2406_09904_b200 import gemm as G  # noqa: E402
from paper_2406_09904_b200 import pipeline as P  # noqa: E402
from oracle import qqq_oracle as O  # noqa: E402

QUICK = "--quick" in sys.argv


def case(m, k, n, scheme, seed):
    rng = np.random.default_rng(seed)
    w = rng.standard_normal((k, n))
    x16 = rng.standard_normal((m, k)).astype(np.float16)
    if scheme == "per-channel":
        qw, qo = Q.quant_weight_per_channel(w), O.quant_weight_per_channel(w)
    else:
        qw, qo = Q.quant_weight_per_group(w, Q.QuantSpec("per-group", 128)), O.quant_weight_per_group(w, 128)
    ao = O.quant_act_per_token(x16.astype(np.float64))
    run_o = O.w4a8_gemm_per_channel if scheme == "per-channel" else O.w4a8_gemm_per_group
    want = run_o(ao, qo, O.FusedScales.from_quantized(qo), fast=True)
    return torch.from_numpy(x16).cuda(), qw, want


def check(tag, x, qw, want, cfg):
    aq = Q.quant_act_per_token(x)
    prep = G.prepare(qw, Q.FusedScales.from_quantized(qw))
    out = G.run_gemm(aq, prep, qw.cols, True, cfg=cfg)
    torch.cuda.synchronize()
    ok = np.array_equal(out.acc.cpu().numpy(), want.acc) and np.array_equal(
        out.y.cpu().numpy().view(np.uint16), want.y.view(np.uint16))
    info = G.plan_info(prep.mode, x.shape[0], qw.cols, qw.rows, cfg)
    print(f"{tag:34s} mode={prep.mode} plan={info} {'OK' if ok else 'MISMATCH'}", flush=True)
    return ok


def main():
    torch.cuda.set_device(0)
    ok = True
    plans = [
        ("whole tiles ntok16", 16, {"ntok": 16, "split": 0}),
        ("stream-K ntok32", 24, {"ntok": 32, "split": 1, "grid": 5}),
        ("hybrid ntok128", 130, {"ntok": 128, "split": 2, "grid": 3}),
        ("pair tiles ntok256", 200, {"ntok": 256, "split": 3}),
        ("cluster split-K S=4", 9, {"ntok": 16, "split": 4, "csplit": 4}),
        ("cluster split-K S=3 ntok32", 20, {"ntok": 32, "split": 4, "csplit": 2}),
        ("pair stream-K", 256, {"ntok": 256, "split": 5, "grid": 6}),
        ("pair waves + stream-K", 256, {"ntok": 256, "split": 6, "grid": 4}),
        ("ntok64 stream-K", 64, {"ntok": 64, "split": 1, "grid": 7}),
        ("whole tiles ntok128 (4 x-stages)", 200, {"ntok": 128, "split": 0}),
        ("cluster split-K ntok128 S=2", 100, {"ntok": 128, "split": 4, "csplit": 2}),
        ("pair tiles ntok384", 400, {"ntok": 384, "split": 3}),
    ]
    if QUICK:
        plans = plans[:1] + plans[3:5]
    for scheme in ("per-channel", "per-group"):
        for i, (tag, m, cfg) in enumerate(plans):
            x, qw, want = case(m, 1024, 512, scheme, seed=100 + i)
            ok &= check(f"{scheme[:5]} {tag}", x, qw, want, cfg)
    # I8 layout (clamp fallback of the per-group conversion; test_gemm_per_group_clamp_fallback's construction)
    for tag, m, cfg in (("I8 whole tiles", 16, {"ntok": 16, "split": 0}),
                        ("I8 stream-K", 40, {"ntok": 32, "split": 1, "grid": 5})):
        rng = np.random.default_rng(5)
        k, n, gs = 1024, 256, 128
        q4 = rng.integers(-8, 8, (k, n)).astype(np.int8)
        s_star = np.full((k // gs, n), 30.0, dtype=np.float16)
        s_star[0, :5] = np.float16(1e-5)
        s_wc = rng.uniform(0.01, 0.02, n)
        x16 = rng.standard_normal((m, k)).astype(np.float16)
        aq_o = O.quant_act_per_token(x16.astype(np.float64))
        qw_o = O.QuantizedWeights(O.pack_i4(q4), k, n, O.PER_GROUP, gs, s_wg=None, s_wc=s_wc)
        want = O.w4a8_gemm_per_group(aq_o, qw_o, O.FusedScales(O.PER_GROUP, s_star=s_star, s_wc=s_wc))
        qw = Q.QuantizedWeights(torch.from_numpy(qw_o.packed).cuda(), k, n, "per-group", gs,
                                s_wc=torch.from_numpy(s_wc).cuda())
        fused = Q.FusedScales("per-group", s_star=torch.from_numpy(s_star).cuda(), s_wc=torch.from_numpy(s_wc).cuda())
        x = torch.from_numpy(x16).cuda()
        aq = Q.quant_act_per_token(x)
        prep = G.prepare(qw, fused)
        out = G.run_gemm(aq, prep, n, True, cfg=cfg)
        torch.cuda.synchronize()
        good = prep.mode == _lib.MODE_I8 and np.array_equal(out.acc.cpu().numpy(), want.acc) and np.array_equal(
            out.y.cpu().numpy().view(np.uint16), want.y.view(np.uint16))
        print(f"{tag:34s} mode={prep.mode} plan={G.plan_info(prep.mode, m, n, k, cfg)} {'OK' if good else 'MISMATCH'}",
              flush=True)
        ok &= good
    # quantizers: plain (fp16, f64 rows) and the smoothed one (with and without the reciprocal table)
    rng = np.random.default_rng(3)
    for m, k in ((3, 4096), (40, 11008)):
        x16 = rng.standard_normal((m, k)).astype(np.float16)
        aq = Q.quant_act_per_token(torch.from_numpy(x16).cuda())
        ao = O.quant_act_per_token(x16.astype(np.float64))
        good = np.array_equal(aq.q.cpu().numpy(), ao.q) and np.array_equal(aq.s_a.cpu().numpy(), ao.s_a)
        print(f"act quant M={m} K={k} {'OK' if good else 'MISMATCH'}", flush=True)
        ok &= good
        # the smoothed quantizer of apply_quant_linear (pipeline.py:146): x / s then quantize
        s = np.ones(k)
        s[rng.permutation(k)[: k // 8]] = rng.uniform(0.5, 2.0, k // 8)
        ao = O.quant_act_per_token(x16.astype(np.float64) / s[None, :])
        aq = P.quant_act_smoothed(torch.from_numpy(x16).cuda(), torch.from_numpy(s).cuda())
        good = np.array_equal(aq.q.cpu().numpy(), ao.q) and np.array_equal(aq.s_a.cpu().numpy(), ao.s_a)
        print(f"smoothed act quant M={m} K={k} {'OK' if good else 'MISMATCH'}", flush=True)
        ok &= good
    # the one-launch smoothed quantization + GEMM (qqq_w4a8_gemm_smooth_fused) against the two-kernel form
    for tag, m, cfg in (("fused quant cluster split-K", 5, {"ntok": 16, "split": 4, "csplit": 4}),
                        ("fused quant whole tiles", 150, {"ntok": 128, "split": 0})):
        k, n = 2048, 512
        rng = np.random.default_rng(9)
        qw = Q.quant_weight_per_group(rng.standard_normal((k, n)), Q.QuantSpec("per-group", 128))
        prep = G.prepare(qw, Q.FusedScales.from_quantized(qw))
        s = torch.from_numpy(rng.uniform(0.5, 2.0, k)).cuda()
        rc = Q.smoothing_reciprocal(s)
        x = torch.from_numpy(rng.standard_normal((m, k)).astype(np.float16)).cuda()
        aq = P.quant_act_smoothed(x, s, recip=rc)
        y0 = G.run_gemm(aq, prep, n, False, cfg=cfg).y
        y1, a1 = P.quant_linear_smoothed(x, s, rc, prep, n, cfg=cfg)
        torch.cuda.synchronize()
        good = torch.equal(y0.view(torch.int16), y1.view(torch.int16)) and torch.equal(aq.q, a1.q)
        print(f"{tag:34s} plan={G.plan_info(prep.mode, m, n, k, cfg)} {'OK' if good else 'MISMATCH'}", flush=True)
        ok &= good
    print("ALL OK" if ok else "FAILURES", flush=True)
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
