"""Adaptive smoothing threshold search on the GPU (reference
pkg/src/qqq/smoothing.py).

Same functions, arguments and error behaviour as the reference module. Every
step runs on the device: the per-token quantizer of x / s (csrc/act_quant.cu),
the weight quantizers of w * s (csrc/weight_prep.cu), the dequantization
(`dequantize_ref`) and the two f64 products through `matmul_ref`, the
sequential-k product of numerics.py:94-109 reproduced rounding for rounding
(csrc/smoothing.cu). The error matrices are therefore bit-identical to the
reference's; only the final sum of squares is a device reduction whose order
differs from numpy's pairwise sum (relative difference ~1e-16), so the
objectives agree to that tolerance and the chosen plan is the reference's
unless two candidates tie to within it.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .errors import DataError, ShapeError
from .pipeline import SmoothingPlan, identity_plan
from .quantize import (PER_CHANNEL, QuantSpec, as_cuda, dequantize_ref, quant_act_per_token,
                       quant_weight_per_channel, quant_weight_per_group)

__all__ = ["matmul_ref", "channel_maxima", "select_outlier_channels", "smoothing_vector", "smoothing_objective",
           "search_sigma"]


def _f64(a, what: str) -> torch.Tensor:
    t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64)))
    return as_cuda(t, torch.float64).contiguous()


def matmul_ref(a, b) -> torch.Tensor:
    """f64 product with the reference's sequential-k rounding (numerics.py:94-109)."""
    a, b = _f64(a, "a"), _f64(b, "b")
    if a.ndim != 2 or b.ndim != 2:
        raise ShapeError("matmul_ref expects 2-D operands")
    if a.shape[1] != b.shape[0]:
        raise ShapeError(f"inner dimensions differ: {tuple(a.shape)} x {tuple(b.shape)}")
    out = torch.empty((a.shape[0], b.shape[1]), dtype=torch.float64, device=a.device)
    lib = _lib.lib_for_device(a.device)
    _lib.check(lib.qqq_matmul_ref_f64(_lib.ptr(a), _lib.ptr(b), _lib.ptr(out), a.shape[0], a.shape[1], b.shape[1],
                                      _lib.stream_of(a.device)), "matmul_ref")
    return out


def channel_maxima(x) -> torch.Tensor:
    """Per-channel absolute maxima over tokens (smoothing.py:60-65)."""
    x = _f64(x, "x")
    if x.ndim != 2 or x.shape[0] < 1:
        raise ShapeError("activations must be 2-D with at least one token")
    return x.abs().amax(dim=0)


def select_outlier_channels(m, sigma: float) -> tuple:
    """Channels whose maximum reaches the threshold (smoothing.py:68-72)."""
    if sigma <= 0:
        raise DataError("sigma must be positive")
    m = _f64(m, "m")
    return tuple(int(t) for t in torch.nonzero(m >= sigma).flatten().tolist())


def smoothing_vector(m, selected: tuple, sigma: float) -> torch.Tensor:
    """s[t] = m[t]/sigma on selected channels, else 1 (smoothing.py:75-85)."""
    if sigma <= 0:
        raise DataError("sigma must be positive")
    m = _f64(m, "m")
    s = torch.ones(m.shape[0], dtype=torch.float64, device=m.device)
    if selected:
        idx = torch.tensor(list(selected), dtype=torch.int64, device=m.device)
        sel = m[idx]
        # IEEE f64 division, as numpy (a Python-scalar divisor would make torch
        # multiply by its reciprocal)
        s[idx] = sel / torch.full_like(sel, sigma)
    return s


def _quant_weights(w: torch.Tensor, spec: QuantSpec):
    if spec.scheme == PER_CHANNEL:
        return quant_weight_per_channel(w)
    return quant_weight_per_group(w, spec)


def _objective_given_exact(x: torch.Tensor, w: torch.Tensor, s: torch.Tensor, spec: QuantSpec,
                           exact: torch.Tensor) -> float:
    """smoothing.py:108-113: both operands quantized round-to-nearest and
    dequantized, their product compared with the exact one."""
    qa = quant_act_per_token(x / s[None, :])
    qw = _quant_weights(w * s[:, None], spec)
    a_deq = qa.q.to(torch.float64) * qa.s_a[:, None]  # QuantizedActivations.dequantize (quantize.py:60-61)
    diff = matmul_ref(a_deq, dequantize_ref(qw)) - exact
    return float((diff * diff).sum())


def smoothing_objective(x, w, s, spec: QuantSpec) -> float:
    """Squared Frobenius error of the quantized product (smoothing.py:88-105)."""
    x, w, s = _f64(x, "x"), _f64(w, "w"), _f64(s, "s")
    if x.ndim != 2 or w.ndim != 2 or x.shape[1] != w.shape[0] or tuple(s.shape) != (x.shape[1],):
        raise ShapeError(f"inconsistent shapes: X {tuple(x.shape)}, W {tuple(w.shape)}, s {tuple(s.shape)}")
    return _objective_given_exact(x, w, s, spec, matmul_ref(x, w))


def search_sigma(x, w, spec: QuantSpec, grid_points: int = 20) -> SmoothingPlan:
    """Exhaustive threshold search over sigma_i = (i/grid)*max|X| (smoothing.py:116-155):
    the no-smoothing plan first, then sigma from high to low, replaced only on a
    strict improvement. The plan's `s` is returned as a numpy f64 vector."""
    if grid_points < 2:
        raise DataError("grid_points must be >= 2")
    x, w = _f64(x, "x"), _f64(w, "w")
    m = channel_maxima(x)
    xmax = float(m.max())
    k = x.shape[1]
    exact = matmul_ref(x, w)
    base_obj = _objective_given_exact(x, w, torch.ones(k, dtype=torch.float64, device=x.device), spec, exact)
    if xmax == 0.0:
        return identity_plan(k, sigma=1.0, objective=base_obj)
    best = identity_plan(k, sigma=xmax, objective=base_obj)
    for i in range(grid_points, 0, -1):
        sigma = (i / grid_points) * xmax
        selected = select_outlier_channels(m, sigma)
        s = smoothing_vector(m, selected, sigma)
        obj = _objective_given_exact(x, w, s, spec, exact)
        if obj < best.objective:
            best = SmoothingPlan(sigma=sigma, selected=selected, s=s.cpu().numpy(), objective=obj)
    return best
