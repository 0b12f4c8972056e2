"""Golden vectors for apply_quant_linear (pipeline.py:144-152) FROM THE
REFERENCE ITSELF. Run in the build container (the only place /root/reference
exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_pipeline.py

Writes pipeline_cases.npz next to this script: per case the activations x,
the smoothing vector s (1.0 outside a random selected channel set, as
smoothing.py builds it), the quantized weights (packed codes + scales) and the
reference's outputs (the smoothed activation codes/scales and y widened to
f64). Nothing at GPU-test or bench time reads /root/reference.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import qqq  # noqa: E402  (reference, read-only)
from qqq import pipeline as rpipe  # noqa: E402
from qqq import smoothing as rsmooth  # noqa: E402


def main():
    rng = np.random.default_rng(144_152)
    out = {}
    spec = [  # (tokens, K, N, scheme, group, fp16 activations)
        (1, 128, 16, "per-group", 128, True),
        (5, 256, 40, "per-group", 128, True),
        (16, 256, 128, "per-channel", 0, True),
        (9, 384, 24, "per-group", 64, False),
        (33, 128, 130, "per-channel", 0, False),
        (2, 512, 8, "per-group", 32, True),
    ]
    for i, (t, k, n, scheme, gs, f16) in enumerate(spec):
        x = rng.standard_normal((t, k)) * 2.0
        x[:, rng.choice(k, size=max(1, k // 16), replace=False)] *= 25.0  # outlier channels
        if f16:
            x = x.astype(np.float16).astype(np.float64)
        sel = tuple(sorted(rng.choice(k, size=max(1, k // 8), replace=False).tolist()))
        s = np.ones(k, dtype=np.float64)
        s[list(sel)] = rng.uniform(0.3, 6.0, size=len(sel))
        plan = rsmooth.SmoothingPlan(sigma=1.0, selected=sel, s=s, objective=0.0)
        w = rng.standard_normal((k, n)) * s[:, None]  # smoothed weights, as the pipeline would hold them
        qw = (qqq.quant_weight_per_channel(w) if scheme == "per-channel"
              else qqq.quant_weight_per_group(w, qqq.QuantSpec("per-group", gs)))
        layer = rpipe.QuantizedLayer(name=f"case{i}", qweights=qw, plan=plan)
        y = rpipe.apply_quant_linear(x, layer)
        qa = qqq.quant_act_per_token(np.asarray(x, dtype=np.float64) / s[None, :])
        p = f"c{i}_"
        out[p + "x"] = x
        out[p + "s"] = s
        out[p + "packed"] = qw.packed
        out[p + "meta"] = np.array([t, k, n, gs, 1 if scheme == "per-group" else 0, 1 if f16 else 0])
        if scheme == "per-channel":
            out[p + "s_w"] = qw.s_w
        else:
            out[p + "s_wg"] = qw.s_wg
            out[p + "s_wc"] = qw.s_wc
        out[p + "q"] = qa.q
        out[p + "s_a"] = qa.s_a
        out[p + "y"] = y
    out["n_cases"] = np.array(len(spec))
    np.savez_compressed(os.path.join(HERE, "pipeline_cases.npz"), **out)
    print("wrote", len(spec), "cases")


if __name__ == "__main__":
    main()
