"""Golden vectors for the smoothing-threshold search (smoothing.py:88-155) and
matmul_ref (numerics.py:94-109) FROM THE REFERENCE ITSELF. Run in the build
container (the only place /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_smoothing.py

Writes smoothing_cases.npz next to this script: per case the calibration
activations x and weights w (a few outlier channels in x), the scheme, the
reference's exact product matmul_ref(x, w), every candidate's objective (the
no-smoothing plan, then sigma = i/grid * max|x| for i = grid..1) and the plan
search_sigma returns. Nothing at GPU-test or bench time reads /root/reference.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from qqq import numerics as rnum  # noqa: E402  (reference, read-only)
from qqq import quantize as rq  # noqa: E402
from qqq import smoothing as rs  # noqa: E402


def main():
    rng = np.random.default_rng(146_155)
    out = {}
    cases = [(16, 256, 64, "per-channel", 0), (24, 256, 96, "per-group", 128), (8, 384, 32, "per-group", 64),
             (32, 128, 48, "per-channel", 0)]
    for ci, (m, k, n, scheme, g) in enumerate(cases):
        x = rng.standard_normal((m, k))
        out_ch = rng.choice(k, max(2, k // 32), replace=False)
        x[:, out_ch] *= rng.uniform(5.0, 40.0, out_ch.size)
        w = rng.standard_normal((k, n)) * 0.05
        spec = rq.QuantSpec(scheme) if scheme == "per-channel" else rq.QuantSpec(scheme, g)
        grid = 12
        exact = rnum.matmul_ref(x, w)
        mx = rs.channel_maxima(x)
        xmax = float(mx.max())
        cand = [rs.smoothing_objective(x, w, np.ones(k), spec)]
        for i in range(grid, 0, -1):
            sigma = (i / grid) * xmax
            cand.append(rs.smoothing_objective(x, w, rs.smoothing_vector(mx, rs.select_outlier_channels(mx, sigma),
                                                                            sigma), spec))
        plan = rs.search_sigma(x, w, spec, grid_points=grid)
        sel = np.zeros(k, dtype=bool)
        sel[list(plan.selected)] = True
        out.update({f"c{ci}_x": x, f"c{ci}_w": w, f"c{ci}_exact": exact, f"c{ci}_cand": np.array(cand),
                    f"c{ci}_sigma": np.float64(plan.sigma), f"c{ci}_sel": sel, f"c{ci}_s": plan.s,
                    f"c{ci}_obj": np.float64(plan.objective), f"c{ci}_grid": np.int64(grid),
                    f"c{ci}_meta": np.array([m, k, n, g], dtype=np.int64),
                    f"c{ci}_pg": np.bool_(scheme == "per-group")})
    out["n_cases"] = np.int64(len(cases))
    np.savez_compressed(os.path.join(HERE, "smoothing_cases.npz"), **out)
    print("wrote", len(cases), "cases")


if __name__ == "__main__":
    main()
