"""Golden QQQ1 checkpoint FROM THE REFERENCE ITSELF (pkg/src/qqq/checkpoint.py,
pipeline.py:230-251 _store_layer). Run in the build container (the only
place /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_checkpoint.py

Writes layers.qqq (two quantized layers: per-channel and per-group g=128, each
with a smoothing plan) and layers_expected.npz: per layer the activations x
and the reference's apply_quant_linear output on the layer it loads back
(_load_layer), y widened to f64. Nothing at test or bench time reads
/root/reference.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from qqq import checkpoint as rckpt  # noqa: E402  (reference, read-only)
from qqq import pipeline as rpipe  # noqa: E402
from qqq import quantize as rq  # noqa: E402
from qqq import smoothing as rsmooth  # noqa: E402


def main():
    rng = np.random.default_rng(121_168)
    ck = rckpt.Checkpoint(metadata={"layers": {}, "model": "golden"})
    exp = {}
    for name, (k, n, scheme, gs) in {"blk0.qkv": (256, 128, "per-channel", 0),
                                     "blk0.down": (384, 96, "per-group", 128)}.items():
        w = rng.standard_normal((k, n))
        qw = rq.quant_weight_per_channel(w) if scheme == "per-channel" else rq.quant_weight_per_group(
            w, rq.QuantSpec("per-group", gs))
        s = np.ones(k)
        sel = np.sort(rng.choice(k, k // 8, replace=False))
        s[sel] = rng.uniform(0.3, 3.0, sel.size)
        plan = rsmooth.SmoothingPlan(sigma=0.5, selected=tuple(int(i) for i in sel), s=s, objective=0.25)
        rpipe._store_layer(ck, rpipe.QuantizedLayer(name=name, qweights=qw, plan=plan))
        x = rng.standard_normal((7, k)).astype(np.float16).astype(np.float64)
        exp[f"{name}.x"] = x
    path = os.path.join(HERE, "layers.qqq")
    rckpt.write_checkpoint(ck, path)
    back = rckpt.read_checkpoint(path)
    for name in back.metadata["layers"]:
        layer = rpipe._load_layer(back, name)
        exp[f"{name}.y"] = rpipe.apply_quant_linear(exp[f"{name}.x"], layer)
    np.savez_compressed(os.path.join(HERE, "layers_expected.npz"), **exp)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
