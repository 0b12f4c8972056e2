"""Drop-in for the reference's quantized linear (pkg/src/qqq/pipeline.py:144-152).

`apply_quant_linear(x, layer)` is the caller of the W4A8 GEMM in the reference
pipeline: divide the activations by the layer's smoothing vector, quantize per
token, run the per-channel or per-group W4A8 GEMM and return y widened to f64.
Here the divide is fused into the activation quantizer (one kernel,
`qqq_act_quant_smooth`), and the GEMM is the tcgen05 kernel; both launch with
programmatic dependent launch, so a chain of linears (the C4 decoder-layer
stack) overlaps each GEMM's weight prefetch with its predecessor.

The containers mirror the reference's field names: `SmoothingPlan`
(smoothing.py:36-48) and `QuantizedLayer` (pipeline.py:86-90).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .errors import ShapeError
from .gemm import FusedScales, _version_key, w4a8_gemm_per_channel, w4a8_gemm_per_group
from .quantize import (PER_CHANNEL, QuantizedActivations, QuantizedWeights, as_cuda, attach_rowsum, deferred_status,
                       raise_if_bad)

__all__ = ["SmoothingPlan", "QuantizedLayer", "identity_plan", "smoothing_reciprocal", "quant_act_smoothed",
           "apply_quant_linear"]


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


def apply_quant_linear(x, layer: QuantizedLayer, check: bool = True) -> torch.Tensor:
    """Quantized forward of one linear (pipeline.py:144-152): divide by s,
    quantize, W4A8 GEMM; returns y widened to f64 (GemmOutput.y_wide)."""
    # Per-layer caches, keyed on the identity and version of what they were
    # built from: a reassigned plan / qweights (or an in-place edit of s or of
    # the weight scales) rebuilds them instead of reusing stale values.
    s = layer.plan.s
    rkey = (id(layer.plan), _version_key(s))
    hit = layer._cache.get("recip")
    if hit is None or hit[0] != rkey:  # the plan's reciprocal table, once per plan
        hit = layer._cache["recip"] = (rkey, smoothing_reciprocal(s))
    qa = quant_act_smoothed(x, s, check=check, recip=hit[1])
    qw = layer.qweights
    fused = layer_fused_scales(layer)
    run = w4a8_gemm_per_channel if qw.scheme == PER_CHANNEL else w4a8_gemm_per_group
    return run(qa, qw, fused, with_acc=False).y_wide()
