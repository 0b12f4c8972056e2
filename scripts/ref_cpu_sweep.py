"""The reference's CPU path timed per BASELINE.md §2 on the GPU box's host.

The reference's own harness is `qqq.cli gemm-bench` (cli.py:166-190): draw
x, w ~ N(0,1) with default_rng(0), quantize them, then time w4a8_gemm_* after
one warm-up, repeating until 0.5 s, and report gemm/s and 2*M*N*K op/s. The
reference package does not travel to the GPU box, so this runs the oracle's
restatement of the same functions (oracle/qqq_oracle.py: unpack_i4,
FusedDequantQuant, the int64 numpy matmul of gemm.py:153, the f64 epilogue)
with the same semantics: single-threaded (numpy's integer matmul does not use
BLAS), "cores used: 1 of nproc".

Points: M in {1, 16, 64} on every C2 shape, M in {256, 1024}
on 4096x4096; per-group g=128, plus per-channel at the C1 point. Output: one
JSON document (host facts + per-point seconds, gemm/s and Mop/s).

    python scripts/ref_cpu_sweep.py > profiles/r02_ref_cpu_sweep.json
"""
import json
import os
import platform
import subprocess
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import qqq_oracle as O  # noqa: E402


def lscpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        for line in out.splitlines():
            if line.startswith("Model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor()


def bench_point(m, n, k, scheme, budget=0.5):
    rng = np.random.default_rng(0)  # cli.py:167-169 draw order
    x = rng.standard_normal((m, k))
    w = rng.standard_normal((k, n))
    aq = O.quant_act_per_token(x.astype(np.float16).astype(np.float64))
    qw = O.quant_weight_per_channel(w) if scheme == "per-channel" else O.quant_weight_per_group(w, 128)
    fused = O.FusedScales.from_quantized(qw)
    run = O.w4a8_gemm_per_channel if scheme == "per-channel" else O.w4a8_gemm_per_group
    run(aq, qw, fused)  # warm-up (cli.py:180)
    reps, t0 = 0, time.perf_counter()
    while True:
        run(aq, qw, fused)
        reps += 1
        el = time.perf_counter() - t0
        if el >= budget:
            break
    per = el / reps
    return dict(scheme=scheme, M=m, K=k, N=n, s_per_gemm=round(per, 4), gemm_per_s=round(1 / per, 4),
                Mops=round(2.0 * m * n * k / per / 1e6, 2), reps=reps)


def main():
    pts = [(1, 4096, 4096, "per-channel"), (16, 4096, 4096, "per-channel")]
    for (k, n) in ((4096, 4096), (4096, 11008), (11008, 4096)):
        for m in (1, 16, 64):
            pts.append((m, n, k, "per-group"))
    pts += [(256, 4096, 4096, "per-group"), (1024, 4096, 4096, "per-group")]
    out = dict(host=dict(nproc=os.cpu_count(), cpu=lscpu_model(), python=platform.python_version(),
                         numpy=np.__version__, cores_used="1 of %d (numpy integer matmul is single-threaded)" %
                         (os.cpu_count() or 1)),
               harness="oracle restatement of qqq.cli gemm-bench (cli.py:166-190), same draw order and timing loop",
               points=[])
    for (m, n, k, scheme) in pts:
        r = bench_point(m, n, k, scheme)
        out["points"].append(r)
        print(json.dumps(r), file=sys.stderr, flush=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
