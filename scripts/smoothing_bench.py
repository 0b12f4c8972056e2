"""search_sigma timing: GPU (this package) on the box, or the
reference CPU implementation with --reference (build container only: it
imports /root/reference). Same synthetic calibration data for both."""
import json, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def data(m, k, n, seed=0):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((m, k))
    ch = rng.choice(k, k // 32, replace=False)
    x[:, ch] *= rng.uniform(5.0, 40.0, ch.size)
    return x, rng.standard_normal((k, n)) * 0.05


def main():
    ref = "--reference" in sys.argv
    sizes = [(64, 512, 512), (128, 1024, 1024), (256, 4096, 4096)]
    if ref:
        sys.path.insert(0, "/root/reference/pkg/src")
        from qqq import quantize as rq, smoothing as rs
        sizes = sizes[:2]
    else:
        import torch
        import paper_2406_09904_b200 as Q
    for (m, k, n) in sizes:
        x, w = data(m, k, n)
        for scheme in ("per-channel", "per-group"):
            if ref:
                spec = rq.QuantSpec(scheme) if scheme == "per-channel" else rq.QuantSpec(scheme, 128)
                t0 = time.perf_counter(); p = rs.search_sigma(x, w, spec); t = time.perf_counter() - t0
            else:
                spec = Q.QuantSpec(scheme) if scheme == "per-channel" else Q.QuantSpec(scheme, 128)
                xd, wd = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
                Q.search_sigma(xd, wd, spec); torch.cuda.synchronize()
                t0 = time.perf_counter(); p = Q.search_sigma(xd, wd, spec); torch.cuda.synchronize()
                t = time.perf_counter() - t0
            print(json.dumps(dict(impl="reference-cpu" if ref else "b200", M=m, K=k, N=n, scheme=scheme,
                                  seconds=round(t, 4), sigma=p.sigma, n_smoothed=len(p.selected),
                                  objective=p.objective)), flush=True)


if __name__ == "__main__":
    main()
