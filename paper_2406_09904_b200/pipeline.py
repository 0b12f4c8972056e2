"""Drop-in for the reference's quantized linear (pkg/src/qqq/pipeline.py:144-152).

`apply_quant_linear(x, layer)` is the caller of the W4A8 GEMM in the reference
pipeline: divide the activations by the layer's smoothing vector, quantize per
token, run the per-channel or per-group W4A8 GEMM and return y widened to f64.
Here the divide is fused into the activation quantizer (`qqq_act_quant_smooth`),
and the GEMM is the tcgen05 kernel; both launch with programmatic dependent
launch, so a chain of linears (the C4 decoder-layer stack) overlaps each GEMM's
weight prefetch with its predecessor. `apply_quant_linear(..., fused=True)`
runs the one-launch form instead (`qqq_w4a8_gemm_smooth_fused`: the GEMM's
epilogue warps quantize the token rows while its weights stream in;
bit-identical results). It measured slower on the C4 stack (its
activation loads and cross-CTA reductions queue behind the weight stream), so
the two-kernel form is the default.

The containers mirror the reference's field names: `SmoothingPlan`
(smoothing.py:36-48) and `QuantizedLayer` (pipeline.py:86-90).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from . import gemm as _gemm
from .errors import ConfigError, ShapeError
from .gemm import FusedScales, GemmOutput, _version_key, w4a8_gemm_per_channel, w4a8_gemm_per_group
from .quantize import (PER_CHANNEL, QuantizedActivations, QuantizedWeights, as_cuda, attach_rowsum, deferred_status,
                       raise_if_bad)

__all__ = ["SmoothingPlan", "QuantizedLayer", "identity_plan", "smoothing_reciprocal", "quant_act_smoothed",
           "quant_linear_smoothed", "apply_quant_linear"]


@dataclass(frozen=True)
class SmoothingPlan:  # smoothing.py:36-48
    sigma: float
    selected: tuple
    s: object  # f64 [K], 1.0 outside `selected` (numpy or torch)
    objective: float

    @property
    def n_smoothed(self) -> int:
        return len(self.selected)


def identity_plan(n_channels: int, sigma: float = 0.0, objective: float = 0.0) -> SmoothingPlan:  # smoothing.py:52-58
    return SmoothingPlan(sigma=sigma, selected=(), s=np.ones(n_channels, dtype=np.float64), objective=objective)


@dataclass
class QuantizedLayer:  # pipeline.py:86-90
    name: str
    qweights: QuantizedWeights
    plan: SmoothingPlan
    _cache: dict = field(default_factory=dict, repr=False, compare=False)


def smoothing_reciprocal(s) -> torch.Tensor:
    """Device table RN(1/s_k) (NaN where |s_k| is outside [2^-400, 2^400]) for
    quant_act_smoothed(..., recip=): computed once per smoothing vector."""
    st = as_cuda(s if isinstance(s, torch.Tensor) else np.asarray(s, dtype=np.float64), torch.float64).contiguous()
    if st.ndim != 1:
        raise ShapeError("smoothing vector must be 1-D")
    out = torch.empty_like(st)
    if st.numel():
        _lib.check(_lib.lib_for_device(st.device).qqq_smooth_reciprocal(_lib.ptr(st), st.numel(), _lib.ptr(out),
                                                                        _lib.stream_of(st.device)),
                   "smoothing_reciprocal")
    return out


def quant_act_smoothed(x, s, check: bool = True, recip: torch.Tensor = None) -> QuantizedActivations:
    """quant_act_per_token(x / s) with the f64 divide fused into the quantizer
    (pipeline.py:146): bit-identical codes and scales to the reference. With
    `recip` (smoothing_reciprocal(s)) the divisions run as Markstein FMA
    sequences — the same IEEE quotients at a fraction of the instructions."""
    xt = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float64)))
    if xt.ndim != 2:
        raise ShapeError("activations must be 2-D (tokens x K)")
    if xt.dtype not in (torch.float16, torch.float32, torch.float64):
        xt = xt.to(torch.float64)
    xt = as_cuda(xt)
    m, k = xt.shape
    if xt.stride(1) != 1 or (m > 1 and xt.stride(0) < k):
        xt = xt.contiguous()
    st = as_cuda(s if isinstance(s, torch.Tensor) else np.asarray(s, dtype=np.float64), torch.float64).contiguous()
    if st.ndim != 1 or st.shape[0] != k:
        raise ShapeError(f"smoothing vector has {tuple(st.shape)} entries, activations have K={k}")
    dev = xt.device
    lib = _lib.lib_for_device(dev)
    kp = (k + 127) // 128 * 128
    qbuf = torch.empty((m, kp), dtype=torch.int8, device=dev)
    s_a = torch.empty((m,), dtype=torch.float64, device=dev)
    rowsum = torch.empty((m,), dtype=torch.int32, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev) if check else deferred_status(dev)
    if m > 0:
        dt = {torch.float16: 0, torch.float32: 1, torch.float64: 2}[xt.dtype]
        ldx = xt.stride(0) if m > 1 else k
        # (no channel mask: with ~1/8 smoothed channels every warp diverges into the
        # division anyway, and the mask loads measured slower)
        if recip is not None:
            if tuple(recip.shape) != (k,) or recip.dtype != torch.float64 or recip.device != dev:
                raise ShapeError("recip must be smoothing_reciprocal(s) on the activations' device")
            recip = recip.contiguous()
            rc = lib.qqq_act_quant_smooth_rcp(_lib.ptr(xt), dt, m, k, ldx, _lib.ptr(st), _lib.ptr(recip),
                                              _lib.ptr(qbuf), kp, _lib.ptr(s_a), _lib.ptr(rowsum), _lib.ptr(status),
                                              _lib.stream_of(dev))
        else:
            rc = lib.qqq_act_quant_smooth(_lib.ptr(xt), dt, m, k, ldx, _lib.ptr(st), None, _lib.ptr(qbuf), kp,
                                          _lib.ptr(s_a), _lib.ptr(rowsum), _lib.ptr(status), _lib.stream_of(dev))
        _lib.check(rc, "quant_act_smoothed")
    out = QuantizedActivations(q=qbuf[:, :k], s_a=s_a)
    attach_rowsum(out, rowsum)
    if check:
        raise_if_bad(status, "activations")
    else:
        out._status = status  # type: ignore[attr-defined]
    return out


def _fused_ok(x: torch.Tensor, prep) -> bool:
    """Inputs qqq_w4a8_gemm_smooth_fused takes (else the two-kernel form)."""
    if x.dtype != torch.float16 or not x.is_cuda or x.ndim != 2 or prep.mode == _lib.MODE_I8:
        return False
    m, k = x.shape
    ldx = x.stride(0) if m > 1 else k
    # (m <= 4096: the launch keeps per-row counters in the workspace head)
    return (0 < m <= 4096 and k % 8 == 0 and x.stride(1) == 1 and ldx % 8 == 0 and ldx >= k
            and x.data_ptr() % 16 == 0)


def quant_linear_smoothed(x: torch.Tensor, s: torch.Tensor, recip, prep, n: int, check: bool = True,
                          y_out=None, cfg=None):
    """One launch: quant_act_per_token(x / s) (pipeline.py:146, bit-identical
    to quant_act_smoothed) fused into the W4A8 GEMM on the prepared weights.
    x: fp16 CUDA [M, K] (see _fused_ok); s: f64 [K] on the same device; recip:
    smoothing_reciprocal(s) or None. Returns (y fp16 [M, n], the quantized
    activations)."""
    m, k = x.shape
    dev = x.device
    lib = _lib.lib_for_device(dev)
    kp = (k + 127) // 128 * 128
    qbuf = torch.empty((m, kp), dtype=torch.int8, device=dev)
    s_a = torch.empty((m,), dtype=torch.float64, device=dev)
    rowsum = torch.empty((m,), dtype=torch.int32, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev) if check else deferred_status(dev)
    y = y_out if y_out is not None else torch.empty((m, n), dtype=torch.float16, device=dev)
    if m > 0:
        wsb = lib.qqq_gemm_workspace_bytes(m, n, k)
        ws = _gemm.workspace(dev, wsb)
        c = None
        if cfg:
            dbg = cfg.get("dbg")
            c = _lib.GemmConfig(int(cfg.get("ntok", 0)), int(cfg.get("grid", 0)), int(cfg.get("split", -1)),
                                int(cfg.get("csplit", 0)), None if dbg is None else dbg.data_ptr())
        rc = lib.qqq_w4a8_gemm_smooth_fused(prep.mode, _lib.ptr(x), x.stride(0) if m > 1 else k, _lib.ptr(s),
                                            None if recip is None else _lib.ptr(recip), _lib.ptr(qbuf), kp,
                                            _lib.ptr(s_a), _lib.ptr(rowsum), _lib.ptr(status), _lib.ptr(prep.w),
                                            prep.group, _lib.ptr(prep.s_col), m, n, k, _lib.ptr(y), y.stride(0),
                                            None, n, _lib.ptr(ws), ws.numel(), c, _lib.stream_of(dev))
        _lib.check(rc, "quant_linear_smoothed")
    aq = QuantizedActivations(q=qbuf[:, :k], s_a=s_a)
    attach_rowsum(aq, rowsum)
    if check:
        raise_if_bad(status, "activations")
    else:
        aq._status = status  # type: ignore[attr-defined]
    return y, aq


def layer_fused_scales(layer: QuantizedLayer) -> FusedScales:
    """FusedScales of the layer's weights, cached on the layer and keyed on the
    identity and version of qweights and its scales (the reference rebuilds
    them per call: they are a pure function of the weights, gemm.py:61-69)."""
    qw = layer.qweights
    fkey = (id(qw), qw.scheme, qw.group_size, qw.rows, qw.cols,
            *(None if a is None else _version_key(a) for a in (qw.s_w, qw.s_wg, qw.s_wc)))
    hit = layer._cache.get("fused")
    if hit is None or hit[0] != fkey:
        hit = layer._cache["fused"] = (fkey, FusedScales.from_quantized(qw))
    return hit[1]


def apply_quant_linear(x, layer: QuantizedLayer, check: bool = True, fused: bool = False) -> torch.Tensor:
    """Quantized forward of one linear (pipeline.py:144-152): divide by s,
    quantize, W4A8 GEMM; returns y widened to f64 (GemmOutput.y_wide).
    fused=True: one launch (quant_linear_smoothed) where the inputs allow it."""
    # Per-layer caches, keyed on the identity and version of what they were
    # built from: a reassigned plan / qweights (or an in-place edit of s or of
    # the weight scales) rebuilds them instead of reusing stale values.
    s = layer.plan.s
    rkey = (id(layer.plan), _version_key(s))
    hit = layer._cache.get("recip")
    if hit is None or hit[0] != rkey:  # the plan's s on the device and its reciprocal table, once per plan
        st = as_cuda(s if isinstance(s, torch.Tensor) else np.asarray(s, dtype=np.float64), torch.float64).contiguous()
        hit = layer._cache["recip"] = (rkey, smoothing_reciprocal(st), st)
    qw = layer.qweights
    fused = layer_fused_scales(layer)
    xt = x if isinstance(x, torch.Tensor) else None
    if fused and xt is not None and xt.is_cuda and xt.dtype == torch.float16 and xt.ndim == 2:
        if xt.shape[1] != qw.rows:
            raise ShapeError(f"activation K={xt.shape[1]} does not match weight K={qw.rows}")
        if qw.scheme != fused.scheme:
            raise ConfigError(f"engine expects {qw.scheme} operands, got scales={fused.scheme!r}")
        _gemm._check_padding(qw)
        if qw.scheme != PER_CHANNEL and (qw.rows % qw.group_size != 0 or tuple(fused.s_star.shape)
                                         != (qw.rows // qw.group_size, qw.cols)):
            raise ConfigError("fused group scales do not match the group structure")
        prep = _gemm.prepare(qw, fused)
        st = hit[2]
        if _fused_ok(xt, prep) and st.ndim == 1 and st.shape[0] == xt.shape[1] and st.device == xt.device:
            y, _ = quant_linear_smoothed(xt, st, hit[1], prep, qw.cols, check=check)
            return GemmOutput(y=y, acc=None).y_wide()
    qa = quant_act_smoothed(x, s, check=check, recip=hit[1])
    run = w4a8_gemm_per_channel if qw.scheme == PER_CHANNEL else w4a8_gemm_per_group
    return run(qa, qw, fused, with_acc=False).y_wide()
