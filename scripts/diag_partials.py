"""Debug (QQQ_DBG_PARTIALS build): per-CTA int32 partials of the small-CTA
cluster split-K plan checked against the exact per-rank partial, to tell an
operand/MMA fault from an exchange fault when the final acc mismatches.

    QQQ_LIB_PATH=.../xdbg.so python scripts/diag_partials.py --shape 11008x4096 --ntok 32 --cs 8
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2406_09904_b200 as Q  # noqa: E402
from paper_2406_09904_b200 import gemm as G  # noqa: E402
from oracle import qqq_oracle as O  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="11008x4096")
ap.add_argument("--m", type=int, default=1)
ap.add_argument("--ntok", type=int, default=32)
ap.add_argument("--cs", type=int, default=8)
ap.add_argument("--reps", type=int, default=400)
ap.add_argument("--stop", type=int, default=6)
a = ap.parse_args()
k, n = map(int, a.shape.split("x"))
rng = np.random.default_rng(7)
w = rng.standard_normal((k, n))
x16 = rng.standard_normal((a.m, k)).astype(np.float16)
qw = Q.quant_weight_per_group(w, Q.QuantSpec("per-group", 128))
qo = O.quant_weight_per_group(w, 128)
fused = Q.FusedScales.from_quantized(qw)
x = torch.from_numpy(x16).cuda()
prep = G.prepare(qw, fused)
cfg = {"ntok": a.ntok, "split": 4, "csplit": a.cs}
info = G.plan_info(prep.mode, a.m, n, k, cfg)
S, grid, bk = info["csplit"], info["grid"], 256
ao = O.quant_act_per_token(x16.astype(np.float64))
fo = O.FusedScales.from_quantized(qo)
q4 = O.unpack_i4(qo.packed, k)
w8 = O.fused_dequant_quant_cols(q4, fo.s_star, 128).astype(np.int64)  # [k, n]
kb = (k + bk - 1) // bk
# exact partial of CTA b: tile c = b // S, rank r = b % S, k-blocks [r*kb//S, (r+1)*kb//S), u8 (+128) weights
qa = ao.q.astype(np.int64)
want_part = np.zeros((grid, 128, a.ntok), dtype=np.int64)
for b in range(grid):
    c, r = b // S, b % S
    k0, k1 = (r * kb // S) * bk, min(k, ((r + 1) * kb // S) * bk)
    cols = slice(c * 128, min(n, c * 128 + 128))
    p = qa[:, k0:k1] @ (w8[k0:k1, cols] + 128)  # [m, ncols]
    want_part[b, : p.shape[1], : a.m] = p.T
want_part = want_part.astype(np.int32)
dbg = torch.zeros(2 * grid * 128 * a.ntok, dtype=torch.int32, device="cuda")
nbad_final = nbad_part = 0
for rep in range(a.reps):
    aq = Q.quant_act_per_token(x)
    dbg.zero_()
    out = G.run_gemm(aq, prep, n, True, cfg=dict(cfg, dbg=dbg))
    torch.cuda.synchronize()
    both = dbg.view(2, grid, 128, a.ntok).cpu().numpy()
    got, got2 = both[0], both[1]
    bad_ctas = [b for b in range(grid) if not np.array_equal(got[b, :, : a.m], want_part[b, :, : a.m])]
    acc = out.acc.cpu().numpy()
    final_ok = np.array_equal(acc, (qa @ w8.astype(np.int64)).astype(np.int32))
    if bad_ctas or not final_ok:
        nbad_part += bool(bad_ctas)
        nbad_final += (not final_ok)
        if nbad_part + nbad_final > 2 * a.stop:
            break
        if nbad_part + nbad_final <= 2 * a.stop:
            desc = []
            for b in bad_ctas[:4]:
                rows = np.nonzero((got[b, :, : a.m] != want_part[b, :, : a.m]).any(1))[0]
                ok2 = np.array_equal(got2[b, :, : a.m], want_part[b, :, : a.m])
                desc.append(f"cta {b} (tile {b // S} rank {b % S}) rows {rows.min()}..{rows.max()} n={rows.size} "
                            f"re-read-4us-later-ok={ok2}")
            print(f"rep {rep}: final_ok={final_ok} bad partial CTAs={len(bad_ctas)}: {'; '.join(desc)}", flush=True)
print(f"{a.shape} M={a.m} plan={info}: {nbad_final} bad finals, {nbad_part} launches with a bad partial, "
      f"of {a.reps}", flush=True)
