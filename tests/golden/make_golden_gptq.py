"""Golden vectors for the GPTQ sweep (gptq.py:63-206) FROM THE REFERENCE
ITSELF. Run in the build container (the only place /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_gptq.py

Writes gptq_cases.npz next to this script: per case the calibration
activations x (one dead channel), the weights w, the reference's HessianState
(damping, chol_inv, dead), the block size, and its result: codes,
scales, layer_error and col_errors. Nothing at GPU-test time reads
/root/reference.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from qqq import gptq as rg  # noqa: E402  (reference, read-only)
from qqq import quantize as rq  # noqa: E402


def main():
    rng = np.random.default_rng(161_183)
    out = {}
    cases = [(48, 128, 48, "per-channel", 0, 128), (48, 128, 48, "per-channel", 0, 32),
             (64, 192, 40, "per-group", 64, 192), (64, 256, 32, "per-group", 128, 128)]
    for ci, (m, k, n, scheme, g, bs) in enumerate(cases):
        x = rng.standard_normal((m, k))
        x[:, rng.integers(0, k)] = 0.0  # a dead input dimension
        w = rng.standard_normal((k, n)) * 0.05
        spec = rq.QuantSpec(scheme) if scheme == "per-channel" else rq.QuantSpec(scheme, g)
        hs = rg.build_hessian(x)
        res = rg.gptq_sweep(w, hs, spec, block_size=bs)
        qw = res.qweights
        pre = f"c{ci}_"
        out.update({pre + "x": x, pre + "w": w, pre + "lam": np.float64(hs.damping),
                    pre + "u": hs.chol_inv, pre + "dead": hs.dead, pre + "codes": qw.codes(),
                    pre + "scales": qw.s_w if scheme == "per-channel" else qw.s_wg,
                    pre + "s_wc": qw.s_wc if scheme == "per-group" else np.zeros(0),
                    pre + "layer_error": np.float64(res.layer_error), pre + "col_errors": res.col_errors,
                    pre + "meta": np.array([m, k, n, g, bs], dtype=np.int64)})
    out["n_cases"] = np.int64(len(cases))
    np.savez_compressed(os.path.join(HERE, "gptq_cases.npz"), **out)
    print("wrote", len(cases), "cases")


if __name__ == "__main__":
    main()
