#!/usr/bin/env python
"""bench.py — contract benchmark of the B200 W4A8 GEMM (QQQ, arXiv 2406.09904).

Metric (BASELINE.json): "W4A8 GEMM TOPS & HBM GB/s vs M (1–1024), speedup over
FP16 GEMM".

* N = 1 (default): workload = BASELINE.json configs[1] (C2): per-group (g=128)
  W4A8 GEMM, M sweep {1,2,4,...,1024} on the Llama-2-7B linear shapes
  4096x4096, 4096x11008, 11008x4096. One "step" = the 33 GEMMs with
  activations already quantized and resident in HBM; weights are read cold
  (rotated replicas whose total exceeds 2x the 126 MB L2).
* N > 1 (torchrun, one rank per GPU): workload = BASELINE.json configs[4]
  (C5): the Llama-2-70B linears tensor-parallel over NCCL — gate_up
  8192x28672 column-parallel (N-split, no collective), o_proj 8192x8192 and
  down 28672x8192 row-parallel (K-split: all-reduce MAX of the per-token
  absmax, int32 partial GEMM, exact all-reduce SUM, f64 epilogue) at
  M in {1, 16, 1024}; strong scaling (total work fixed). `--replicas` runs N
  independent copies of the C2 sweep instead (weak scaling).

`value` = aggregate TOPS of the step (2*M*N*K summed / device time), max over
ranks. `e2e` = the same step through the public API from pinned host fp16
activations (H2D + quantize + GEMM + D2H of y, every step).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

L2_BYTES = 126 * 1024 * 1024
SHAPES_C2 = [(4096, 4096), (4096, 11008), (11008, 4096)]
MS_C2 = [1, 2, 4, 8, 16, 32, 64, 128, 256, 512, 1024]
MS_C5 = [1, 16, 1024]
# Llama-2-70B linears of BASELINE configs[2]/[4]: (name, K, N, split)
C5_LAYERS = [("o_proj", 8192, 8192, "k"), ("gate_up", 8192, 28672, "n"), ("down", 28672, 8192, "k")]
GROUP = 128
METRIC = "W4A8 GEMM TOPS & HBM GB/s vs M (1-1024), speedup over FP16 GEMM"
PLAN_NAMES = {0: "whole tiles", 1: "stream-K", 2: "waves+stream-K", 3: "pair tiles", 4: "cluster split-K",
              5: "pair stream-K", 6: "pair waves+stream-K"}


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            pk = json.load(f)
        return dict(hbm_gbs=float(pk["hbm_gbs"]), bf16_tflops=float(pk["bf16_tflops"]), source="measured")
    except Exception:
        return dict(hbm_gbs=6650.0, bf16_tflops=1590.0, source="fallback")


def alg_bytes(m, k, n, scheme="per-group", g=GROUP):
    """Algorithmic bytes per GEMM: int8 A + f64 s_A + int4 W + fp16 Y + scales."""
    sc = 8 * n if scheme == "per-channel" else 2 * (k // g) * n + 8 * n
    return m * k + 8 * m + k * n / 2 + 2 * m * n + sc


TRAFFIC_FILE = "profiles/r02_traffic.json"


def load_traffic(shapes, ms):
    """DRAM bytes per step measured by ncu (scripts/traffic_summary.py), only when
    the committed capture covers exactly this step's GEMMs."""
    for name in (TRAFFIC_FILE, "profiles/r01_traffic.json"):
        try:
            with open(os.path.join(ROOT, name)) as f:
                t = json.load(f)
        except Exception:
            continue
        want = sorted("%dx%d/%d" % (k, n, m) for (k, n) in shapes for m in ms)
        have = sorted("%s/%d" % (p["shape"], p["M"]) for p in t["points"])
        if want == have:
            t["file"] = name
            return t
    return None


def c2_config(world: int, replicas: bool):
    """The C2 workload description (identical for both arms, see run_reference_arm)."""
    set_bytes = sum(k * n / 2 for k, n in SHAPES_C2)
    R = max(2, math.ceil(2.5 * L2_BYTES / set_bytes))
    return dict(workload="C2 (BASELINE.json configs[1]): per-group g=128 W4A8 GEMM, M sweep "
                         f"{MS_C2} x shapes {['%dx%d' % s for s in SHAPES_C2]} (K x N)",
                scheme="per-group", group_size=GROUP, gemms_per_step=len(MS_C2) * len(SHAPES_C2),
                l2="weights read cold: %d rotated replicas per shape (%.0f MB > 2x L2)" % (R, R * set_bytes / 2**20),
                parallelism=f"replicas x{world}" if (world > 1 and replicas) else "single GPU")


def c5_config(world: int):
    return dict(workload="C5 (BASELINE.json configs[4]): Llama-2-70B linears tensor-parallel over NCCL, per-group "
                         "g=128: gate_up 8192x28672 N-split, o_proj 8192x8192 and down 28672x8192 K-split "
                         f"(all-reduce MAX absmax + int32 all-reduce SUM), M in {MS_C5}",
                scheme="per-group", group_size=GROUP, gemms_per_step=len(MS_C5) * len(C5_LAYERS),
                l2="weights read cold: rotated shard replicas (> 2x L2 per rank)",
                parallelism=f"tp{world}")


# ---------------------------------------------------------------------------
# clocks sampler (NVML during the timed region)
# ---------------------------------------------------------------------------
class ClockSampler:
    """Polls NVML (SM clock + clock-event reasons) every ~2 ms during the timed
    region."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.reasons = set()
        self.sm_max = None
        self._stop = threading.Event()
        self._nvml = None

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.sm_max = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._t = threading.Thread(target=self._poll, daemon=True)
            self._t.start()
        except Exception:
            self._nvml = None
        return self

    def _poll(self):
        nv = self._nvml
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for name, bit in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __exit__(self, *a):
        self._stop.set()
        if self._nvml is not None:
            self._t.join(timeout=1)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.sm_max, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.sm_max,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# distributed plumbing
# ---------------------------------------------------------------------------
def dist_setup(args):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        # --dist-backend gloo: developer check of the TP plumbing with every rank on one GPU
        dev_index = local if args.dist_backend == "nccl" else 0
        torch.cuda.set_device(dev_index)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_index))
        else:
            dist.init_process_group("gloo")
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return world, rank, local


def barrier(world):
    import torch

    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        torch.cuda.synchronize()


def _reduce(v, world, op):
    if world == 1:
        return v
    import torch
    import torch.distributed as dist

    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=op)
    return float(t.item())


def max_over_ranks(v, world):
    import torch.distributed as dist

    return _reduce(v, world, dist.ReduceOp.MAX if world > 1 else None)


def sum_over_ranks(v, world):
    import torch.distributed as dist

    return _reduce(v, world, dist.ReduceOp.SUM if world > 1 else None)


def min_over_ranks(v, world):
    import torch.distributed as dist

    return _reduce(v, world, dist.ReduceOp.MIN if world > 1 else None)


# ---------------------------------------------------------------------------
# CPU legs (oracle = the reference algorithm restated; only here and in tests)
# ---------------------------------------------------------------------------
def cpu_reference_sample(shapes=SHAPES_C2, ms=(1, 16), threads=0):
    """Time the reference's CPU path (restated in oracle/: unpack, FusedDequantQuant,
    exact int64 matmul split over `threads` host threads, f64 epilogue —
    gemm.py:188-203) at M in `ms` on each shape. Returns per-shape fits
    t(M) = a + b*M (the weight conversion is M-independent, the matmul linear in
    M) and the timed points."""
    import numpy as np

    from oracle import qqq_oracle as O

    threads = threads or (os.cpu_count() or 1)
    fits, pts = {}, []
    for (k, n) in shapes:
        rng = np.random.default_rng(7 + k + n)
        q4 = rng.integers(-8, 8, (k, n)).astype(np.int8)
        s_wg = 0.02 * rng.uniform(0.5, 1.5, (k // GROUP, n))
        qw = O.QuantizedWeights(O.pack_i4(q4), k, n, O.PER_GROUP, GROUP, s_wg=s_wg, s_wc=O.requant_scale(q4, s_wg))
        fused = O.FusedScales.from_quantized(qw)
        ts = []
        for m in ms:
            x = rng.standard_normal((m, k)).astype(np.float16).astype(np.float64)
            aq = O.quant_act_per_token(x)
            t0 = time.perf_counter()
            O.w4a8_gemm_per_group(aq, qw, fused, fast="threads" if threads > 1 else False)
            dt = time.perf_counter() - t0
            ts.append(dt)
            pts.append(dict(shape=f"{k}x{n}", M=m, s=round(dt, 4), TOPS=2.0 * m * n * k / dt / 1e12))
        b = (ts[-1] - ts[0]) / (ms[-1] - ms[0]) if len(ms) > 1 else ts[0] / ms[0]
        b = max(b, 1e-12)
        fits[(k, n)] = (max(ts[0] - b * ms[0], 0.0), b)
    return fits, pts, threads


def extrapolated_sweep_tops(fits):
    """Whole C2 sweep on the CPU path: per point t = a + b*M from the per-shape fit."""
    ops = sum(2.0 * m * n * k for (k, n) in SHAPES_C2 for m in MS_C2)
    t = sum(fits[(k, n)][0] + fits[(k, n)][1] * m for (k, n) in SHAPES_C2 for m in MS_C2)
    return ops / t / 1e12, t


def cpu_baseline_block(fits, pts, threads):
    v, t_sweep = extrapolated_sweep_tops(fits)
    return dict(value=v, unit="TOPS", cores=threads, kind="port",
                sample=("per-group g=128 W4A8 GEMM, the oracle's restatement of gemm.py:188-203 (exact int64 matmul "
                        f"over {threads} host threads): timed at " +
                        "; ".join(f"{p['shape']} M={p['M']}: {p['s'] * 1e3:.0f} ms" for p in pts) +
                        f"; the 33-point C2 sweep extrapolated linearly in M from those (BASELINE.md §2): "
                        f"{t_sweep:.1f} s per step (extrapolated)"),
                timed_points=pts)


def run_reference_arm(args, world, rank):
    """The reference's own CPU implementation of the path (restated in oracle/,
    which is what travels to the GPU box; the reference itself is pure Python
    and absent there), on the host cores, on OUR arm's workload: each step is a
    bounded sample (one C2 shape at M=1 and M=16, rotating over the shapes),
    the whole sweep extrapolated linearly in M from the latest sample of each
    shape."""
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    fits = {}
    for i in range(max(0, args.warmup)):
        f, _, _ = cpu_reference_sample([SHAPES_C2[i % 3]], (1, 16), threads)
        fits.update(f)
    vals, all_pts = [], []
    t0 = time.perf_counter()
    for i in range(args.steps):
        f, pts, _ = cpu_reference_sample([SHAPES_C2[i % 3]], (1, 16), threads)
        fits.update(f)
        all_pts = [p for p in all_pts if p["shape"] != pts[0]["shape"]] + pts
        if len(fits) == len(SHAPES_C2):
            vals.append(extrapolated_sweep_tops(fits)[0])
    wall = time.perf_counter() - t0
    if len(fits) < len(SHAPES_C2):  # fewer steps than shapes: complete the fit once
        f, pts, _ = cpu_reference_sample([s for s in SHAPES_C2 if s not in fits], (1, 16), threads)
        fits.update(f)
        all_pts += pts
        vals.append(extrapolated_sweep_tops(fits)[0])
    v = statistics.median(vals)
    cb = cpu_baseline_block(fits, all_pts, threads)
    cb["value"] = v
    gpus = max(args.gpus, world)
    cfg = c5_config(gpus) if (gpus > 1 and not args.replicas) else c2_config(gpus, args.replicas)
    line = dict(metric=METRIC, value=v, unit="TOPS", n_gpus=gpus, steps=args.steps, warmup=args.warmup,
                ms_per_step=wall / max(1, args.steps) * 1e3, higher_is_better=True,
                scaling="strong" if (gpus > 1 and not args.replicas) else "weak",
                vs_baseline=None, dtype="int8", data="synthetic", config=cfg, impl="reference", cpu_baseline=cb,
                e2e=dict(value=v, unit="TOPS", h2d_bytes_per_step=0, d2h_bytes_per_step=0),
                note=("CPU path of the reference on the host cores; the sweep value is extrapolated linearly in M "
                      "from timed M=1/16 points per shape (the matmul cost is linear in M, the weight "
                      "conversion constant). For N>1 the same single-host number is reported (the reference has "
                      "no multi-device path)."))
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm helpers
# ---------------------------------------------------------------------------
def make_weights(k, n, scheme, seed, device):
    import torch

    import paper_2406_09904_b200 as Q
    from paper_2406_09904_b200 import gemm as G

    gen = torch.Generator(device=device).manual_seed(seed)
    q4 = torch.randint(-8, 8, (k, n), dtype=torch.int8, device=device, generator=gen)
    if scheme == "per-channel":
        s_w = 0.02 * (0.5 + torch.rand(n, dtype=torch.float64, device=device, generator=gen))
        qw = Q.QuantizedWeights(Q.pack_i4(q4), k, n, "per-channel", s_w=s_w)
    else:
        s_wg = 0.02 * (0.5 + torch.rand((k // GROUP, n), dtype=torch.float64, device=device, generator=gen))
        qw = Q.QuantizedWeights(Q.pack_i4(q4), k, n, "per-group", GROUP, s_wg=s_wg, s_wc=Q.requant_scale(q4, s_wg))
    fused = Q.FusedScales.from_quantized(qw)
    return qw, fused, G.prepare(qw, fused)


def clone_prep(prep):
    from paper_2406_09904_b200 import gemm as G

    return G.PreparedWeights(prep.mode, prep.w.clone(), None if prep.sc is None else prep.sc.clone(), prep.group,
                             prep.s_col.clone())


_CAPTURE_STREAM = {}


def capture_stream(dev):
    """One side stream for every CUDA-graph capture of this process, so the
    split-K workspace (per device and stream) is sized once, outside capture."""
    import torch

    s = _CAPTURE_STREAM.get(dev.index)
    if s is None:
        s = _CAPTURE_STREAM[dev.index] = torch.cuda.Stream(dev)
    return s


def presize_workspace(dev, nbytes):
    from paper_2406_09904_b200 import gemm as G

    G.workspace(dev, nbytes)
    G.workspace(dev, nbytes, stream=capture_stream(dev))


def graph_time_us(fns, reps, warm=2, dev=None):
    """Device time per launch of `fns` (captured once in a CUDA graph)."""
    import torch

    dev = dev or torch.device("cuda", torch.cuda.current_device())
    for f in fns:
        f()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=capture_stream(dev)):
        for f in fns:
            f()
    for _ in range(warm):
        g.replay()
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) * 1e3 / (reps * len(fns))


def measure_int8_peak(dev):
    """Dense INT8 tensor-core peak measured on this GPU: the library's probe
    (every SM issuing back-to-back tcgen05 kind::i8 M=128 N=256 K=32, no
    memory traffic), best of 5, beside cuBLASLt's int8 GEMM (torch._int_mm at
    8192^3) for reference. The probe is the roofline denominator."""
    import ctypes

    import torch

    from paper_2406_09904_b200 import _lib

    lib = _lib.lib_for_device(dev)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    ops = ctypes.c_double(0.0)
    best = 0.0
    st = _lib.stream_of(dev)
    for i in range(6):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        _lib.check(lib.qqq_probe_int8_peak(sms, 1 << 16, ctypes.byref(ops), st), "probe_int8_peak")
        e.record()
        torch.cuda.synchronize()
        if i:
            best = max(best, ops.value / (s.elapsed_time(e) * 1e-3) / 1e12)
    cublas = None
    try:
        a = torch.randint(-127, 128, (8192, 8192), dtype=torch.int8, device=dev)
        b = torch.randint(-127, 128, (8192, 8192), dtype=torch.int8, device=dev)
        for _ in range(2):
            torch._int_mm(a, b)
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            torch._int_mm(a, b)
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
        cublas = 2.0 * 8192 ** 3 / (min(ts) * 1e-3) / 1e12
        del a, b
    except Exception:
        cublas = None
    return dict(tops=round(best, 1), source="measured: tcgen05 kind::i8 M=128 N=256 K=32 issue loop on every SM "
                                            "(qqq_probe_int8_peak), best of 5",
                cublaslt_int8_8192cubed_tops=None if cublas is None else round(cublas, 1))


def point_record(shape_k, shape_n, m, scheme, t_us, t16_us, peaks, plan=None):
    ops = 2.0 * m * shape_n * shape_k
    byts = alg_bytes(m, shape_k, shape_n, scheme)
    t_hbm = byts / (peaks["hbm_gbs"] * 1e3)  # us
    t_ten = ops / (peaks["int8_tops"] * 1e6)
    r = dict(shape=f"{shape_k}x{shape_n}", M=m, us=round(t_us, 3), TOPS=round(ops / t_us / 1e6, 2),
             GBps=round(byts / t_us / 1e3, 1), bound="hbm" if t_hbm >= t_ten else "tensor",
             frac=round(max(t_hbm, t_ten) / t_us, 4), roof_us=round(max(t_hbm, t_ten), 3))
    if t16_us is not None:
        r.update(fp16_us=round(t16_us, 3), speedup_vs_fp16=round(t16_us / t_us, 3))
    if plan is not None:
        r["plan"] = f"ntok={plan['ntok']} {PLAN_NAMES.get(plan['split'], plan['split'])}" + (
            f" S={plan['csplit']}" if plan["split"] == 4 else "") + f" grid={plan['grid']}"
    return r


def regime_summary(points):
    def stats(vals):
        return None if not vals else dict(min=round(min(vals), 4), median=round(statistics.median(vals), 4),
                                          max=round(max(vals), 4), n=len(vals))

    hb = [p["frac"] for p in points if p["M"] <= 16]
    tn = [p["frac"] for p in points if p["M"] >= 512]
    return dict(hbm_frac_m_le_16=stats(hb), int8_frac_m_ge_512=stats(tn),
                targets="north_star: >=0.70 of the HBM roofline at M<=16, >=0.60 of dense INT8 peak at M>=512")


def extra_points(peaks, dev, specs):
    """Supplementary device-time points outside the contract workload: BASELINE
    configs[0] (C1, per-channel M=16, N=K=4096) and configs[2] (C3, Llama-2-70B
    shapes, per-channel vs per-group). Same method as roofline_points: CUDA
    graph over rotated cold weight replicas, fp16 cuBLAS with cold weights."""
    import torch

    import paper_2406_09904_b200 as Q
    from paper_2406_09904_b200 import _lib
    from paper_2406_09904_b200 import gemm as G

    out = []
    for (k, n, scheme, ms) in specs:
        qw, fused, prep = make_weights(k, n, scheme, seed=77, device=dev)
        R = max(2, math.ceil(2.5 * L2_BYTES / (k * n / 2)))
        reps = [prep] + [clone_prep(prep) for _ in range(R - 1)]
        r16 = max(2, math.ceil(2.5 * L2_BYTES / (k * n * 2)))
        w16 = [torch.randn((k, n), dtype=torch.float16, device=dev) for _ in range(r16)]
        mode = _lib.MODE_PC if scheme == "per-channel" else _lib.MODE_PG
        for m in ms:
            x = torch.randn((m, k), dtype=torch.float16, device=dev)
            aq = Q.quant_act_per_token(x)
            y = torch.empty((m, n), dtype=torch.float16, device=dev)
            presize_workspace(dev, _lib.load().qqq_gemm_workspace_bytes(m, n, k))
            fns = [(lambda p_: (lambda: G.run_gemm(aq, p_, n, False, y_out=y)))(p_) for p_ in reps]
            t_us = graph_time_us(fns, reps=max(2, 40 // R), dev=dev)
            t16 = graph_time_us([(lambda wi: (lambda: torch.matmul(x, wi)))(wi) for wi in w16],
                                reps=max(2, 40 // len(w16)), dev=dev)
            rec = point_record(k, n, m, scheme, t_us, t16, peaks, G.plan_info(mode, m, n, k))
            rec["scheme"] = scheme
            out.append(rec)
        del reps, w16
        torch.cuda.empty_cache()
    return out


C4_LINEARS = [("qkv", 4096, 12288), ("o", 4096, 4096), ("gate_up", 4096, 22016), ("down", 11008, 4096)]


def c4_stack_points(peaks, dev, batches=(1, 16, 64, 256)):
    """BASELINE configs[3] (C4): the Llama-2-7B decoder-layer linear stack
    (QKV 4096->12288, O 4096->4096, gate-up 4096->22016, down 11008->4096),
    each linear = apply_quant_linear's path (pipeline.py:144-152): fused
    smooth-divide + per-token act quant kernel, then the per-group g=128 W4A8
    GEMM, the 8 launches of a stack chained with PDL in one CUDA graph; weights
    cold (rotated layer replicas). Also timed: the one-launch form
    (apply_quant_linear(fused=True): quantization inside the GEMM launch).
    Compared with the fp16 torch.matmul stack."""
    import torch

    import paper_2406_09904_b200 as Q
    from paper_2406_09904_b200 import _lib
    from paper_2406_09904_b200 import gemm as G
    from paper_2406_09904_b200 import pipeline as P

    layer_bytes = sum(k * n / 2 for _, k, n in C4_LINEARS)
    R = max(2, math.ceil(2.5 * L2_BYTES / layer_bytes))
    layers = []
    for r in range(R):
        lin = []
        for li, (name, k, n) in enumerate(C4_LINEARS):
            qw, fused, prep = make_weights(k, n, "per-group", seed=500 + 10 * r + li, device=dev)
            sm = torch.ones(k, dtype=torch.float64, device=dev)
            idx = torch.randperm(k, device=dev)[: k // 8]
            sm[idx] = 0.5 + 1.5 * torch.rand(k // 8, dtype=torch.float64, device=dev)
            lin.append((k, n, prep, sm, Q.smoothing_reciprocal(sm)))  # (the layer's cached table)
        layers.append(lin)
    r16 = max(2, math.ceil(2.5 * L2_BYTES / (4 * layer_bytes)))
    w16 = [[torch.randn((k, n), dtype=torch.float16, device=dev) for _, k, n in C4_LINEARS] for _ in range(r16)]
    ops_stack = lambda m: sum(2.0 * m * k * n for _, k, n in C4_LINEARS)
    out = []
    for m in batches:
        xs = [torch.randn((m, k), dtype=torch.float16, device=dev) for _, k, _n in C4_LINEARS]
        ys = [torch.empty((m, n), dtype=torch.float16, device=dev) for _, _k, n in C4_LINEARS]
        presize_workspace(dev, max(_lib.load().qqq_gemm_workspace_bytes(m, n, k) for _, k, n in C4_LINEARS))

        def stack_fn(lin):
            def f():
                for i, (k, n, prep, sm, rc) in enumerate(lin):
                    P.quant_linear_smoothed(xs[i], sm, rc, prep, n, check=False, y_out=ys[i])
            return f

        def stack_fn_2k(lin):
            def f():
                for i, (k, n, prep, sm, rc) in enumerate(lin):
                    aq = Q.quant_act_smoothed(xs[i], sm, check=False, recip=rc)
                    G.run_gemm(aq, prep, n, False, y_out=ys[i])
            return f

        t_fu = graph_time_us([stack_fn(lin) for lin in layers], reps=max(2, 20 // R), dev=dev)
        t_us = graph_time_us([stack_fn_2k(lin) for lin in layers], reps=max(2, 20 // R), dev=dev)
        t16 = graph_time_us([(lambda ws: (lambda: [torch.matmul(xs[i], ws[i]) for i in range(4)]))(ws) for ws in w16],
                            reps=max(2, 20 // r16), dev=dev)
        out.append(dict(batch=m, us_per_stack=round(t_us, 2), us_per_stack_fused_launch=round(t_fu, 2),
                        TOPS=round(ops_stack(m) / t_us / 1e6, 2),
                        fp16_us=round(t16, 2), speedup_vs_fp16=round(t16 / t_us, 3)))
    del layers, w16
    torch.cuda.empty_cache()
    return out


# ---------------------------------------------------------------------------
# C2: the contract sweep (N = 1, or N replicas with --replicas)
# ---------------------------------------------------------------------------
def run_c2_arm(args, world, rank, local):
    import torch

    import paper_2406_09904_b200 as Q
    from paper_2406_09904_b200 import _lib
    from paper_2406_09904_b200 import gemm as G

    dev = torch.device("cuda", torch.cuda.current_device())
    peaks = load_peaks()
    i8 = measure_int8_peak(dev)
    peaks["int8_tops"] = i8["tops"]
    hbm_peak = peaks["hbm_gbs"]
    shapes = SHAPES_C2
    ms = MS_C2 if not args.quick else [1, 16, 128, 1024]
    scheme = "per-group"

    # ---- weights: one logical matrix per shape, R cold replicas ----------------
    preps, w16 = {}, {}
    set_bytes = sum(k * n / 2 for k, n in shapes)
    R = max(2, math.ceil(2.5 * L2_BYTES / set_bytes))
    for si, (k, n) in enumerate(shapes):
        qw, fused, prep = make_weights(k, n, scheme, seed=1000 + si + 17 * rank, device=dev)
        preps[(k, n)] = [prep] + [clone_prep(prep) for _ in range(R - 1)]
        r16 = max(2, math.ceil(2.5 * L2_BYTES / (k * n * 2)))  # fp16 baseline weights also read cold
        w16[(k, n)] = [torch.randn((k, n), dtype=torch.float16, device=dev) for _ in range(r16)]
    acts, outs = {}, {}
    for (k, n) in shapes:
        for m in ms:
            x = torch.randn((m, k), dtype=torch.float16, device=dev)
            acts[(k, n, m)] = (x, Q.quant_act_per_token(x))
            outs[(k, n, m)] = torch.empty((m, n), dtype=torch.float16, device=dev)
    # pre-size the split-K workspaces (eager and capture streams) outside any capture
    presize_workspace(dev, max(_lib.load().qqq_gemm_workspace_bytes(max(ms), n, k) for k, n in shapes))

    order = [(k, n, m) for m in ms for (k, n) in shapes]
    counters = {s: 0 for s in shapes}

    def gemm_fn(k, n, m, rep):
        aq = acts[(k, n, m)][1]
        y = outs[(k, n, m)]
        p = preps[(k, n)][rep]
        return lambda: G.run_gemm(aq, p, n, False, y_out=y)

    step_fns = []
    for (k, n, m) in order:
        step_fns.append(gemm_fn(k, n, m, counters[(k, n)] % R))
        counters[(k, n)] += 1

    # ---- per-point device times (explanatory; not the contract number) ----------
    points = []
    for (k, n, m) in order:
        fns = [gemm_fn(k, n, m, r) for r in range(R)]
        t_us = graph_time_us(fns, reps=max(2, 40 // R), dev=dev)
        x = acts[(k, n, m)][0]
        f16_fns = [(lambda wi: (lambda: torch.matmul(x, wi)))(wi) for wi in w16[(k, n)]]
        t16 = graph_time_us(f16_fns, reps=max(2, 40 // len(f16_fns)), dev=dev)
        points.append(point_record(k, n, m, scheme, t_us, t16, peaks, G.plan_info(_lib.MODE_PG, m, n, k)))

    # ---- supplementary configs (not part of the contract number) ---------------
    c1_points = c3_points = c4_points = c5_points = None
    if not args.quick and rank == 0:
        c4_points = c4_stack_points(peaks, dev)
        c1_points = extra_points(peaks, dev, [(4096, 4096, "per-channel", [16])])
        c3_points = extra_points(peaks, dev, [(k, n, sch, [1, 16, 1024]) for (k, n) in
                                             [(8192, 8192), (8192, 28672), (28672, 8192)]
                                             for sch in ("per-channel", "per-group")])
        if world == 1:
            c5_points = run_c5(args, 1, 0, dev, peaks, summary_only=True)

    # ---- the contract timed region: K steps of the 33-GEMM sweep ---------------
    g = torch.cuda.CUDAGraph()
    for f in step_fns:
        f()
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=capture_stream(dev)):
        for f in step_fns:
            f()
    for _ in range(args.warmup):
        g.replay()
    barrier(world)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index) as clk:
        barrier(world)
        start.record()
        for _ in range(args.steps):
            g.replay()
        end.record()
        torch.cuda.synchronize()
        barrier(world)
    elapsed_ms = max_over_ranks(start.elapsed_time(end), world)
    ops_step = sum(2.0 * m * n * k for (k, n, m) in order)
    value = sum_over_ranks(ops_step * args.steps, world) / (elapsed_ms * 1e-3) / 1e12
    ms_per_step = elapsed_ms / args.steps

    # ---- e2e through the public API from pinned host memory ---------------------
    e2e = None
    if not args.no_e2e:
        e2e = c2_e2e(args, world, rank, dev, shapes, order, acts, outs, scheme, ops_step)

    # ---- roofline: every launch of the step is the W4A8 GEMM kernel ------------
    step_us = ms_per_step * 1e3
    tops = ops_step / (step_us * 1e-6) / 1e12
    roof_us = sum(p["roof_us"] for p in points)
    traffic = load_traffic(shapes, ms)
    ceiling_tops = ops_step / (roof_us * 1e-6) / 1e12
    roofline = dict(bound="tensor", achieved=round(tops, 2), peak=round(ceiling_tops, 1), unit="TFLOP/s",
                    frac=round(tops / ceiling_tops, 4),
                    traffic=traffic and traffic["step_dram_bytes"],
                    traffic_note=traffic and ("bytes per step (the 33 GEMM launches) from ncu dram__bytes_read.sum "
                                              "+ dram__bytes_write.sum, %s; %.3f x the algorithmic bytes" % (
                                                  traffic["file"], traffic["step_ratio"])),
                    peak_note=("mixed per-launch roofline of the step: peak = sum(2MNK) / sum_i max(bytes_i / HBM, "
                               "ops_i / INT8) over the 33 launches (%.1f us), so frac = sum_i t_roof_i / step time; "
                               "HBM = %.1f GB/s (MEASURED_PEAKS.json, %s), INT8 = %.1f TOPS (%s). The tensor-bound "
                               "launches carry %.0f%% of the roofline time." % (
                                   roof_us, hbm_peak, peaks["source"], i8["tops"], i8["source"],
                                   100.0 * sum(p["roof_us"] for p in points if p["bound"] == "tensor") / roof_us)),
                    hbm_peak_gbs=hbm_peak, int8_peak_tops=i8["tops"],
                    int8_peak_cublaslt_8192cubed=i8["cublaslt_int8_8192cubed_tops"],
                    device_sum_of_points_us=round(sum(p["us"] for p in points), 2))
    roofline.update(regime_summary(points))
    f16_total = sum(p["fp16_us"] for p in points)
    ours_total = sum(p["us"] for p in points)
    line = dict(metric=METRIC, value=round(value, 3), unit="TOPS", n_gpus=world, steps=args.steps,
                warmup=args.warmup, ms_per_step=round(ms_per_step, 4), higher_is_better=True, scaling="weak",
                vs_baseline=None, dtype="int8", data="synthetic", config=c2_config(world, args.replicas),
                roofline=roofline,
                fp16_baseline=dict(impl="torch.matmul fp16 (cuBLAS), same shapes, cold weights",
                                   total_us=round(f16_total, 2), ours_total_us=round(ours_total, 2),
                                   sweep_speedup=round(f16_total / ours_total, 3),
                                   min_point_speedup=min(p["speedup_vs_fp16"] for p in points),
                                   points_slower_than_fp16=[f"{p['shape']}/M={p['M']}" for p in points
                                                            if p["speedup_vs_fp16"] < 1.0]),
                roofline_points=points,
                c1_points=c1_points,
                c3_points=c3_points,
                c4_points=c4_points,
                c5_points=c5_points,
                gpu_launches=len(order) * args.steps,
                clocks=clk.summary())
    if e2e:
        line["e2e"] = e2e
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        fits, pts, threads = cpu_reference_sample()
        cb = cpu_baseline_block(fits, pts, threads)
        sel = [p for p in points if (p["shape"], p["M"]) in {(q["shape"], q["M"]) for q in pts}]
        g_ops = sum(2.0 * p["M"] * int(p["shape"].split("x")[0]) * int(p["shape"].split("x")[1]) for p in sel)
        cb["gpu_matched"] = dict(value=round(g_ops / (sum(p["us"] for p in sel) * 1e-6) / 1e12, 3), unit="TOPS",
                                 points=[f"{p['shape']}/M={p['M']}" for p in sel],
                                 note="this GPU on exactly the CPU-timed points (device time, cold weights)")
        cpu_pts_tops = sum(2.0 * q["M"] * int(q["shape"].split("x")[0]) * int(q["shape"].split("x")[1])
                           for q in pts) / sum(q["s"] for q in pts) / 1e12
        cb["matched_points_cpu_tops"] = cpu_pts_tops
        line["cpu_baseline"] = cb
    if rank == 0:
        print(json.dumps(line), flush=True)


def c2_e2e(args, world, rank, dev, shapes, order, acts, outs, scheme, ops_step):
    import torch

    import paper_2406_09904_b200 as Q

    host_x = {key: acts[key][0].cpu().pin_memory() for key in order}
    host_y = {key: torch.empty(outs[key].shape, dtype=torch.float16).pin_memory() for key in order}
    dev_x = {key: torch.empty_like(acts[key][0]) for key in order}
    qws = {}
    for si, (k, n) in enumerate(shapes):
        qws[(k, n)] = make_weights(k, n, scheme, seed=1000 + si + 17 * rank, device=dev)[:2]

    # H2D, compute and D2H on three streams (PCIe is full duplex): input i+1
    # uploads and output i-1 downloads while GEMM i runs; every byte still
    # crosses the bus inside the timed region
    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def e2e_step():
        comp = torch.cuda.current_stream(dev)  # (the capture stream while a graph is captured)
        s_in.wait_stream(comp)  # the previous step is done with dev_x
        for (k, n, m) in order:
            dx = dev_x[(k, n, m)]
            with torch.cuda.stream(s_in):
                dx.copy_(host_x[(k, n, m)], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(s_in)
            comp.wait_event(ev)
            aq = Q.quant_act_per_token(dx, check=False)
            qw, fused = qws[(k, n)]
            out = Q.w4a8_gemm_per_group(aq, qw, fused, with_acc=False)
            s_out.wait_stream(comp)
            out.y.record_stream(s_out)
            with torch.cuda.stream(s_out):
                host_y[(k, n, m)].copy_(out.y, non_blocking=True)
        comp.wait_stream(s_out)

    def timed(step):
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        barrier(world)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            step()
        torch.cuda.synchronize()
        return max_over_ranks(time.perf_counter() - t0, world)

    t_eager = timed(e2e_step)
    # The same public-API calls captured once in a CUDA graph (as a serving
    # loop would): each replay still uploads every input from pinned host
    # memory and downloads every y; only the Python dispatch is gone.
    t_graph, mode = None, "eager"
    try:
        cap = capture_stream(dev)
        with torch.cuda.stream(cap):
            e2e_step()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=cap):
            e2e_step()
        # the replays really move the bytes: a fresh input pattern must come back as its y
        key = order[-1]
        host_x[key].copy_(torch.randn(host_x[key].shape, dtype=torch.float16))
        g.replay()
        torch.cuda.synchronize()
        want = Q.w4a8_gemm_per_group(Q.quant_act_per_token(host_x[key].to(dev)), *qws[key[:2]], with_acc=False).y
        if not torch.equal(host_y[key], want.cpu()):
            raise RuntimeError("graph replay did not round-trip the host buffers")
        t_graph, mode = timed(g.replay), "cuda graph of the API calls"
    except Exception as exc:  # capture unsupported here: report the eager loop
        mode = f"eager (graph capture failed: {type(exc).__name__}: {exc})"
    t_e2e = t_graph if t_graph is not None else t_eager
    bi = sum(m * k * 2 for (k, n, m) in order)
    bo = sum(m * n * 2 for (k, n, m) in order)
    tops = lambda t: sum_over_ranks(ops_step * args.steps, world) / t / 1e12
    return dict(value=tops(t_e2e), unit="TOPS", h2d_bytes_per_step=bi, d2h_bytes_per_step=bo,
                ms_per_step=t_e2e / args.steps * 1e3, mode=mode, eager_value=tops(t_eager),
                eager_ms_per_step=t_eager / args.steps * 1e3)


# ---------------------------------------------------------------------------
# C5: tensor-parallel 70B linears over NCCL (N > 1; also N = 1 as a reference)
# ---------------------------------------------------------------------------
def run_c5(args, world, rank, dev, peaks, summary_only=False):
    """The C5 step on `world` ranks through paper_2406_09904_b200.tp
    (ColumnParallelW4A8 / RowParallelW4A8, NCCL collectives), weights cold
    (rotated shard replicas). Returns the per-layer / per-M breakdown and the
    step time (max over ranks); checks every layer output bit-exact against
    the unsplit single-GPU GEMM on this rank."""
    import torch
    import torch.distributed as dist

    import paper_2406_09904_b200 as Q
    from paper_2406_09904_b200 import _lib
    from paper_2406_09904_b200 import tp

    ops = tp.TPOps(check=False)
    layers = []
    per_rank_bytes = 0
    for li, (name, k, n, split) in enumerate(C5_LAYERS):
        qw, fused, _ = make_weights(k, n, "per-group", seed=3000 + li, device=dev)  # same on every rank
        shard = tp.shard_nsplit(qw, rank, world) if split == "n" else tp.shard_ksplit(qw, rank, world)
        per_rank_bytes += shard.rows * shard.cols / 2
        layers.append(dict(name=name, k=k, n=n, split=split, full=(qw, fused), shard=shard))
    R = max(2, math.ceil(2.5 * L2_BYTES / per_rank_bytes))
    for L in layers:
        reps = []
        for r in range(R):
            sh = L["shard"]
            if r:  # an independent copy of the shard (cold replica)
                sh = Q.QuantizedWeights(sh.packed.clone(), sh.rows, sh.cols, sh.scheme, sh.group_size,
                                        s_wg=sh.s_wg.clone(), s_wc=sh.s_wc.clone())
            cls = tp.ColumnParallelW4A8 if L["split"] == "n" else tp.RowParallelW4A8
            reps.append(cls(sh, Q.FusedScales.from_quantized(sh), None, ops))
        L["reps"] = reps
    xs = {}
    for L in layers:
        for m in MS_C5:
            x = torch.randn((m, L["k"]), dtype=torch.float16, device=dev,
                            generator=torch.Generator(device=dev).manual_seed(m * 7 + L["k"]))
            if L["split"] == "k":
                k0, k1 = L["reps"][0].k_bounds()
                xs[(L["name"], m)] = (x, x[:, k0:k1].contiguous())
            else:
                xs[(L["name"], m)] = (x, x)
    presize_workspace(dev, max(_lib.load().qqq_gemm_workspace_bytes(m, L["shard"].cols, L["shard"].rows)
                               for L in layers for m in MS_C5))

    order = [(L, m) for m in MS_C5 for L in layers]

    def call(L, m, r):
        return L["reps"][r % R](xs[(L["name"], m)][1])

    # parity: the TP output equals the unsplit single-GPU GEMM, bit for bit
    ok = True
    for (L, m) in order:
        y = call(L, m, 0)
        qw, fused = L["full"]
        ref = Q.w4a8_gemm_per_group(Q.quant_act_per_token(xs[(L["name"], m)][0]), qw, fused, with_acc=False).y
        if L["split"] == "n":
            n0 = rank * (L["n"] // world)
            ref = ref[:, n0:n0 + L["n"] // world]
        ok = ok and torch.equal(y.view(torch.int16), ref.view(torch.int16))
    ok = bool(min_over_ranks(1.0 if ok else 0.0, world))

    # per-layer timing (eager, events on the compute stream), GEMM vs collectives
    def timed_eager(fn, reps):
        for _ in range(2):
            fn(0)
        barrier(world)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for i in range(reps):
            fn(i)
        e.record()
        torch.cuda.synchronize()
        return max_over_ranks(s.elapsed_time(e) * 1e3 / reps, world)

    # Device time per call: the rank's launches (and NCCL collectives) captured in
    # one CUDA graph over the R cold replicas; eager (host-launch-bound for these
    # microsecond kernels) only where capture is unavailable (gloo).
    def timed(fn, reps):
        if args.dist_backend != "gloo":
            try:
                t = graph_time_us([(lambda i: (lambda: fn(i)))(i) for i in range(R)], reps=max(2, reps // R), dev=dev)
                return max_over_ranks(t, world), "cuda graph"
            except Exception:  # (capture unsupported here: fall back to eager launches)
                torch.cuda.synchronize()
        return timed_eager(fn, reps), "eager"

    breakdown = []
    for (L, m) in order:
        t_layer, how = timed(lambda i: call(L, m, i), 4 * R)
        t_comm = 0.0
        if world > 1 and L["split"] == "k":
            nb = torch.empty((m, L["n"]), dtype=torch.int32, device=dev)
            mx = torch.empty((m,), dtype=torch.float64, device=dev)

            def comm(i):
                dist.all_reduce(mx, op=dist.ReduceOp.MAX)
                dist.all_reduce(nb, op=dist.ReduceOp.SUM)

            t_comm, _ = timed(comm, 10)
        ops_full = 2.0 * m * L["k"] * L["n"]
        breakdown.append(dict(layer=L["name"], split=L["split"], M=m, us=round(t_layer, 2), timing=how,
                              comm_us=round(t_comm, 2), gemm_us=round(max(t_layer - t_comm, 0.0), 2),
                              TOPS=round(ops_full / (t_layer * 1e-6) / 1e12, 2),
                              allreduce_bytes=(4 * m * L["n"] + 8 * m) if L["split"] == "k" else 0))
    ops_step = sum(2.0 * m * L["k"] * L["n"] for (L, m) in order)

    def step(i):
        for (L, m) in order:
            call(L, m, i)

    # the step (every layer at every M, NCCL collectives between our launches),
    # captured once as a CUDA graph (eager where capture is unavailable); K timed steps
    for i in range(max(args.warmup, 3)):
        step(i)
    torch.cuda.synchronize()
    run_step, step_mode = step, "eager"
    if args.dist_backend != "gloo":
        try:
            graphs = []
            for r in range(R):  # one graph per cold replica: step i replays graph i % R
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=capture_stream(dev)):
                    step(r)
                graphs.append(g)
            graphs[0].replay()
            torch.cuda.synchronize()
            run_step, step_mode = (lambda i: graphs[i % R].replay()), "cuda graph"
        except Exception:
            torch.cuda.synchronize()
    for i in range(max(args.warmup, 3)):
        run_step(i)
    barrier(world)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk_summary = None
    with ClockSampler(dev.index) as clk:
        barrier(world)
        s.record()
        for i in range(args.steps):
            run_step(i)
        e.record()
        torch.cuda.synchronize()
        barrier(world)
        clk_summary = clk.summary()
    elapsed_ms = max_over_ranks(s.elapsed_time(e), world)
    value = ops_step * args.steps / (elapsed_ms * 1e-3) / 1e12
    out = dict(value=round(value, 3), unit="TOPS", n_gpus=world, ms_per_step=round(elapsed_ms / args.steps, 4),
               tp_parity_vs_1gpu=ok, layers=breakdown, clocks=clk_summary, ops_step=ops_step, step_mode=step_mode,
               l2=f"{R} rotated shard replicas per rank ({R * per_rank_bytes / 2**20:.0f} MB)")
    if summary_only:
        return out
    # e2e: host fp16 activations (pinned) -> H2D -> TP layer -> D2H y, every step
    hx = {(L["name"], m): xs[(L["name"], m)][1].cpu().pin_memory() for (L, m) in order}
    dx = {key: torch.empty_like(xs[key][1]) for key in hx}
    hy = {}

    def e2e_step(i):
        for (L, m) in order:
            key = (L["name"], m)
            dx[key].copy_(hx[key], non_blocking=True)
            y = L["reps"][i % R](dx[key])
            if key not in hy:
                hy[key] = torch.empty(y.shape, dtype=y.dtype).pin_memory()
            hy[key].copy_(y, non_blocking=True)

    for i in range(max(args.warmup, 3)):
        e2e_step(i)
    torch.cuda.synchronize()
    barrier(world)
    t0 = time.perf_counter()
    for i in range(args.steps):
        e2e_step(i)
    torch.cuda.synchronize()
    t_e2e = max_over_ranks(time.perf_counter() - t0, world)
    bi = sum(hx[k].numel() * 2 for k in hx)
    bo = sum(hy[k].numel() * 2 for k in hy)
    out["e2e"] = dict(value=ops_step * args.steps / t_e2e / 1e12, unit="TOPS", h2d_bytes_per_step=bi,
                      d2h_bytes_per_step=bo, ms_per_step=t_e2e / args.steps * 1e3,
                      mode="eager public API (tp layers) from pinned host memory, per rank")
    return out


def run_c5_arm(args, world, rank, local):
    import torch

    dev = torch.device("cuda", torch.cuda.current_device())
    peaks = load_peaks()
    res = run_c5(args, world, rank, dev, peaks)
    if rank != 0:
        return
    line = dict(metric=METRIC, value=res["value"], unit="TOPS", n_gpus=world, steps=args.steps, warmup=args.warmup,
                ms_per_step=res["ms_per_step"], higher_is_better=True, scaling="strong", vs_baseline=None,
                dtype="int8", data="synthetic", config=c5_config(world),
                tp=dict(parity_vs_1gpu=res["tp_parity_vs_1gpu"], layers=res["layers"], l2=res["l2"],
                        backend=args.dist_backend),
                gpu_launches=None, clocks=res["clocks"], e2e=res["e2e"])
    # launches per step: N-split = quant + GEMM; K-split = absmax + quant + GEMM + epilogue
    per = {"n": 2, "k": 4}
    line["gpu_launches"] = args.steps * sum(per[s] for (_, _, _, s) in C5_LAYERS) * len(MS_C5)
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--replicas", action="store_true", help="N>1: N independent C2 sweeps instead of C5 TP")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: every rank on cuda:0 (developer check of the TP plumbing on one GPU)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        run_reference_arm(args, int(os.environ.get("WORLD_SIZE", "1")), rank)
        return
    world, rank, local = dist_setup(args)
    try:
        if world > 1 and not args.replicas:
            run_c5_arm(args, world, rank, local)
        else:
            run_c2_arm(args, world, rank, local)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
