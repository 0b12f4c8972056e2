"""Generate golden vectors for the W4A8 hot path FROM THE REFERENCE ITSELF.

Run in the build container (the only place /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports the reference package read-only from /root/reference/pkg/src and
writes, next to this script:
  * small_cases.npz   — full input/output vectors for small shapes (both
                        schemes, several group sizes, ragged/odd shapes,
                        zero rows/columns), consumed by the CPU oracle tests
                        and the GPU parity tests;
  * digests.json      — sha256/16 digests of reference outputs at the
                        BASELINE config shapes (C1 = per-channel and
                        per-group M=16 N=K=4096, recipe R1; C2 shapes at M=4)
                        plus exhaustive conversion tables.
Nothing at GPU-test or bench time reads /root/reference.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import qqq  # noqa: E402  (reference, read-only)
from qqq import gemm as rgemm  # noqa: E402


def digest(a) -> str:
    import hashlib

    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def run_case(x, w, scheme, gs):
    aq = qqq.quant_act_per_token(x)
    if scheme == "per-channel":
        qw = qqq.quant_weight_per_channel(w)
        fused = qqq.FusedScales.from_quantized(qw)
        out = qqq.w4a8_gemm_per_channel(aq, qw, fused)
    else:
        qw = qqq.quant_weight_per_group(w, qqq.QuantSpec("per-group", gs))
        fused = qqq.FusedScales.from_quantized(qw)
        out = qqq.w4a8_gemm_per_group(aq, qw, fused)
    return aq, qw, fused, out


def small_cases():
    rng = np.random.default_rng(2406_09904)
    cases = []
    # (t, k, n, scheme, gs, fp16_acts, scale)
    spec = [
        (1, 32, 8, "per-channel", 0, True, 1.0),
        (3, 64, 16, "per-channel", 0, True, 3.0),
        (5, 96, 40, "per-channel", 0, True, 0.01),
        (16, 256, 128, "per-channel", 0, True, 1.0),
        (7, 33, 5, "per-channel", 0, False, 4.0),  # odd K, f64 acts
        (17, 384, 136, "per-channel", 0, True, 100.0),
        (2, 64, 16, "per-group", 32, True, 1.0),
        (4, 256, 64, "per-group", 128, True, 3.0),
        (9, 384, 200, "per-group", 128, True, 1.0),
        (3, 16, 3, "per-group", 4, False, 3.0),
        (3, 16, 3, "per-group", 8, False, 3.0),
        (33, 512, 256, "per-group", 64, True, 0.5),
        (1, 256, 130, "per-group", 256, True, 1.0),
        (20, 128, 24, "per-group", 32, True, 20.0),
    ]
    for i, (t, k, n, scheme, gs, f16, sc) in enumerate(spec):
        x = rng.standard_normal((t, k)) * sc
        if f16:
            x = x.astype(np.float16).astype(np.float64)
        w = rng.standard_normal((k, n))
        if i % 4 == 1:  # a zero activation row and a zero weight column
            x[0, :] = 0.0
            w[:, 0] = 0.0
        aq, qw, fused, out = run_case(x, w, scheme, gs)
        c = dict(
            x=x, w=w, q=aq.q, s_a=aq.s_a, packed=qw.packed, acc=out.acc, y=out.y,
            meta=np.array([t, k, n, gs, int(f16), 1 if scheme == "per-group" else 0]),
        )
        if scheme == "per-channel":
            c["s_w"] = qw.s_w
            c["s_w_folded"] = fused.s_w_folded
        else:
            c["s_wg"] = qw.s_wg
            c["s_wc"] = qw.s_wc
            c["s_star"] = fused.s_star
        cases.append(c)
    flat = {}
    for i, c in enumerate(cases):
        for key, v in c.items():
            flat[f"c{i}_{key}"] = v
    flat["n_cases"] = np.array(len(cases))
    return flat


def config_digests():
    out = {}
    # C1: recipe R1 (cli.py:167-169 draw order), activations via fp16
    for scheme in ("per-channel", "per-group"):
        rng = np.random.default_rng(0)
        x = rng.standard_normal((16, 4096))
        w = rng.standard_normal((4096, 4096))
        x16 = x.astype(np.float16)
        aq, qw, fused, o = run_case(x16.astype(np.float64), w, scheme, 128)
        d = dict(x16=digest(x16), q=digest(aq.q), s_a=digest(aq.s_a), packed=digest(qw.packed),
                 acc=digest(o.acc), y=digest(o.y), y_row0=o.y[0, :4].astype(float).tolist(),
                 acc_row0=o.acc[0, :4].tolist())
        if scheme == "per-channel":
            d["s_w_folded"] = digest(fused.s_w_folded)
        else:
            d["s_star"] = digest(fused.s_star)
            d["s_wc"] = digest(fused.s_wc)
        out[f"C1/{scheme}"] = d
    # C2 shapes, per-group g=128, M=4, seed = 1000*2 + M (SURVEY.md §8d R2 seeding)
    for (k, n) in ((4096, 4096), (4096, 11008), (11008, 4096)):
        m = 4
        rng = np.random.default_rng(1000 * 2 + m)
        x = rng.standard_normal((m, k))
        w = rng.standard_normal((k, n))
        x16 = x.astype(np.float16)
        aq, qw, fused, o = run_case(x16.astype(np.float64), w, "per-group", 128)
        out[f"C2/{k}x{n}/M{m}"] = dict(
            q=digest(aq.q), s_a=digest(aq.s_a), packed=digest(qw.packed), s_star=digest(fused.s_star),
            s_wc=digest(fused.s_wc), acc=digest(o.acc), y=digest(o.y))
    # exhaustive conversion tables
    bits = np.arange(65536, dtype=np.uint16)
    vals = bits.view(np.float16).astype(np.float64)
    pos = np.isfinite(vals) & (vals > 0)
    s_all = bits[pos].view(np.float16)  # every positive finite binary16 s*
    codes = np.arange(-8, 8, dtype=np.int8)
    q4 = np.repeat(codes[:, None], s_all.size, axis=1)  # 16 x S
    table = rgemm._fused_dequant_quant_cols(q4, s_all[None, :], 16)
    out["fused_dequant_quant_table"] = dict(n_scales=int(s_all.size), digest=digest(table))
    inr = np.isfinite(vals) & (vals >= -128.0) & (vals < 127.5)
    f2i = np.array([rgemm.fast_f16_to_i8(qqq.Binary16(int(b))) for b in bits[inr]], dtype=np.int8)
    out["fast_f16_to_i8_inrange"] = dict(n=int(inr.sum()), digest=digest(f2i))
    return out


def main():
    np.savez_compressed(os.path.join(HERE, "small_cases.npz"), **small_cases())
    with open(os.path.join(HERE, "digests.json"), "w") as f:
        json.dump(config_digests(), f, indent=1, sort_keys=True)
    print("wrote", HERE)


if __name__ == "__main__":
    main()
