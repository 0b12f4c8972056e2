"""GPTQ (build_hessian + gptq_sweep) timing: GPU (this package) on
the box, or the reference CPU implementation with --reference (build container
only: it imports /root/reference). Same synthetic calibration data for both."""
import json, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ref = "--reference" in sys.argv
    sizes = [(256, 1024, 1024), (512, 4096, 4096)]
    if ref:
        sys.path.insert(0, "/root/reference/pkg/src")
        from qqq import gptq as G, quantize as QZ
        sizes = sizes[:1]
    else:
        import torch
        import paper_2406_09904_b200 as G
        QZ = G
    for (m, k, n) in sizes:
        rng = np.random.default_rng(0)
        x, w = rng.standard_normal((m, k)), rng.standard_normal((k, n)) * 0.05
        for scheme in ("per-channel", "per-group"):
            spec = QZ.QuantSpec(scheme) if scheme == "per-channel" else QZ.QuantSpec(scheme, 128)
            if not ref:
                xd, wd = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
                G.gptq_sweep(wd, G.build_hessian(xd), spec); torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = G.gptq_sweep(w if ref else wd, G.build_hessian(x if ref else xd), spec)
            if not ref:
                torch.cuda.synchronize()
            t = time.perf_counter() - t0
            print(json.dumps(dict(impl="reference-cpu" if ref else "b200", M=m, K=k, N=n, scheme=scheme,
                                  seconds=round(t, 4), layer_error=res.layer_error)), flush=True)


if __name__ == "__main__":
    main()
