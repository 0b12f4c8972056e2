"""Drop-in for the reference quantizer module (pkg/src/qqq/quantize.py), on B200.

Same names, dataclasses, argument meaning and exceptions as the reference;
tensors are torch CUDA tensors (numpy inputs are accepted and moved to the
GPU). Every numeric step runs in the sm_100a library (libqqq_b200.so): there
is no CPU fallback.

Reference conventions (quantize.py:1-9): activations per-token scale
max|row|/127, codes in [-127, 127]; weights scale max|col|/7 per channel or
per group, codes in [-8, 7]; half-even rounding; all-zero rows/columns get
scale 1.0.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch

from . import _lib
from .errors import ConfigError, CorruptionError, DataError, ShapeError

__all__ = [
    "PER_CHANNEL",
    "PER_GROUP",
    "QuantSpec",
    "QuantizedActivations",
    "QuantizedWeights",
    "quant_act_per_token",
    "quant_weight_per_channel",
    "quant_weight_per_group",
    "requant_scale",
    "pack_i4",
    "unpack_i4",
    "dequantize_ref",
]

PER_CHANNEL = "per-channel"
PER_GROUP = "per-group"


def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise _lib.KernelError("no CUDA device: the B200 path has no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def as_cuda(x, dtype: Optional[torch.dtype] = None) -> torch.Tensor:
    """Host arrays/tensors -> CUDA tensor (plumbing only; no compute on host)."""
    if isinstance(x, torch.Tensor):
        t = x
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(x)))
    if not t.is_cuda:
        t = t.to(_device(), non_blocking=False)
    if dtype is not None and t.dtype != dtype:
        t = t.to(dtype)
    return t


def _status(device) -> torch.Tensor:
    return torch.zeros(1, dtype=torch.int32, device=device)


_deferred: dict = {}


def deferred_status(device) -> torch.Tensor:
    """Per-device status word for asynchronous (check=False) calls: kernels only
    OR error bits into it, so no per-call zero-fill launch breaks a PDL chain;
    `raise_if_bad` on it raises and re-arms it."""
    key = torch.device(device).index
    st = _deferred.get(key)
    if st is None:
        st = torch.zeros(1, dtype=torch.int32, device=device)
        _deferred[key] = st
    return st


@dataclass(frozen=True)
class QuantSpec:
    """Weight/activation bit widths and weight quantization granularity (quantize.py:38-52)."""

    scheme: str = PER_CHANNEL
    group_size: int = 128

    weight_bits = 4
    act_bits = 8

    def __post_init__(self) -> None:
        if self.scheme not in (PER_CHANNEL, PER_GROUP):
            raise ConfigError(f"unknown scheme {self.scheme!r}")
        if self.group_size <= 0:
            raise ConfigError("group_size must be positive")


@dataclass
class QuantizedActivations:  # quantize.py:55-61
    q: torch.Tensor  # int8, tokens x K (CUDA)
    s_a: torch.Tensor  # float64, per-token scales (CUDA)

    def dequantize(self) -> torch.Tensor:
        return self.q.to(torch.float64) * self.s_a[:, None]


@dataclass
class QuantizedWeights:  # quantize.py:64-82
    """Packed INT4 weight tensor with its scale hierarchy (reference byte layout)."""

    packed: torch.Tensor  # uint8, ceil(K/2) x N (CUDA)
    rows: int
    cols: int
    scheme: str
    group_size: int = 0
    s_w: Optional[torch.Tensor] = None
    s_wg: Optional[torch.Tensor] = None
    s_wc: Optional[torch.Tensor] = None
    _cache: dict = field(default_factory=dict, repr=False, compare=False)

    def codes(self) -> torch.Tensor:
        return unpack_i4(self.packed, self.rows)


def quant_act_per_token(x, check: bool = True) -> QuantizedActivations:
    """Symmetric per-token INT8 quantization (quantize.py:92-100), one CUDA launch.

    x: 2-D fp16 / fp32 / fp64 tensor (tokens x K). Non-finite input raises
    DataError (quantize.py:85-89); with check=False the test is deferred to
    `raise_if_bad(status)` so the call stays asynchronous.
    """
    if isinstance(x, torch.Tensor):
        xt = x
    else:
        xt = torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float64)))
    if xt.ndim != 2:
        raise ShapeError("activations must be 2-D (tokens x K)")
    if xt.dtype not in (torch.float16, torch.float32, torch.float64):
        xt = xt.to(torch.float64)
    xt = as_cuda(xt)
    m, k = xt.shape
    if xt.stride(1) != 1 or (m > 1 and xt.stride(0) < k):
        xt = xt.contiguous()
    ldx = xt.stride(0) if m > 1 else k
    dev = xt.device
    lib = _lib.lib_for_device(dev)
    kp = (k + 127) // 128 * 128  # row pitch = whole 128-byte atoms for the GEMM's TMA; view is M x K
    qbuf = torch.empty((m, kp), dtype=torch.int8, device=dev)
    s_a = torch.empty((m,), dtype=torch.float64, device=dev)
    rowsum = torch.empty((m,), dtype=torch.int32, device=dev)
    status = _status(dev) if check else deferred_status(dev)
    if m > 0 and k > 0:
        dt = {torch.float16: 0, torch.float32: 1, torch.float64: 2}[xt.dtype]
        _lib.check(lib.qqq_act_quant_ex(_lib.ptr(xt), dt, m, k, ldx, _lib.ptr(qbuf), kp, _lib.ptr(s_a),
                                        _lib.ptr(rowsum), _lib.ptr(status), _lib.stream_of(dev)),
                   "quant_act_per_token")
    elif k == 0:
        raise ShapeError("activations must have K >= 1")
    out = QuantizedActivations(q=qbuf[:, :k], s_a=s_a)
    attach_rowsum(out, rowsum)
    if check:
        raise_if_bad(status, "activations")
    else:
        out._status = status  # type: ignore[attr-defined]
    return out


def _q_key(q: torch.Tensor):
    return (q.data_ptr(), q._version, tuple(q.shape))


def attach_rowsum(aq: QuantizedActivations, rowsum: torch.Tensor) -> None:
    """Cache sum_k q[t, k] on the activations (valid while aq.q is unmodified)."""
    aq._rowsum = (_q_key(aq.q), rowsum)  # type: ignore[attr-defined]


def rowsum_of(aq: QuantizedActivations) -> torch.Tensor:
    """int32 per-token code sums, cached or recomputed on the GPU if aq.q changed."""
    hit = getattr(aq, "_rowsum", None)
    q = as_cuda(aq.q, torch.int8)
    if hit is not None and hit[0] == _q_key(aq.q):
        return hit[1]
    m, k = q.shape
    out = torch.empty((m,), dtype=torch.int32, device=q.device)
    if m:
        if q.stride(1) != 1:
            q = q.contiguous()
        lib = _lib.lib_for_device(q.device)
        _lib.check(lib.qqq_act_rowsum(_lib.ptr(q), m, k, q.stride(0) if m > 1 else k, _lib.ptr(out),
                                      _lib.stream_of(q.device)), "act_rowsum")
    if isinstance(aq.q, torch.Tensor) and aq.q.is_cuda:
        attach_rowsum(aq, out)
    return out


def raise_if_bad(status: torch.Tensor, what: str) -> None:
    v = int(status.item())
    if v:
        status.zero_()  # re-arm (matters for the shared deferred status word)
    if v & _lib.STAT_NONFINITE:
        raise DataError(f"{what} contains non-finite values")
    if v & _lib.STAT_CODE_RANGE:
        raise DataError("INT4 codes out of [-8, 7]")
    if v & _lib.STAT_PAD_NIBBLE:
        raise CorruptionError("nonzero padding nibble for odd K")
    if v & _lib.STAT_SCALE_INF:
        raise ConfigError("fused per-group scale overflows binary16")


def _weights_f64(w) -> torch.Tensor:
    if isinstance(w, torch.Tensor):
        wt = w
    else:
        wt = torch.from_numpy(np.ascontiguousarray(np.asarray(w, dtype=np.float64)))
    if wt.ndim != 2:
        raise ShapeError("weights must be 2-D (K x N)")
    return as_cuda(wt, torch.float64).contiguous()


def _quant_weight(w: torch.Tensor, group: int):
    k, n = w.shape
    dev = w.device
    lib = _lib.lib_for_device(dev)
    codes = torch.empty((k, n), dtype=torch.int8, device=dev)
    g = k if group <= 0 else group
    scales = torch.empty((k // g, n), dtype=torch.float64, device=dev)
    status = _status(dev)
    _lib.check(lib.qqq_quant_weight(_lib.ptr(w), k, n, group, _lib.ptr(codes), _lib.ptr(scales), _lib.ptr(status),
                                    _lib.stream_of(dev)), "quant_weight")
    raise_if_bad(status, "weights")
    return codes, scales


def quant_weight_per_channel(w) -> QuantizedWeights:
    """Symmetric per-output-channel INT4 quantization of a K x N weight matrix (quantize.py:111-123)."""
    w = _weights_f64(w)
    if w.shape[0] == 0 or w.shape[1] == 0:
        raise ShapeError("weights must be non-empty")
    codes, s = _quant_weight(w, 0)
    return QuantizedWeights(packed=pack_i4(codes), rows=w.shape[0], cols=w.shape[1], scheme=PER_CHANNEL, s_w=s[0])


def quant_weight_per_group(w, spec: QuantSpec) -> QuantizedWeights:
    """Per-group INT4 quantization plus the derived requant scale (quantize.py:126-149)."""
    w = _weights_f64(w)
    k, n = w.shape
    gs = spec.group_size
    if k % gs != 0:
        raise ConfigError(f"group_size {gs} does not divide K={k}")
    codes, s_wg = _quant_weight(w, gs)
    s_wc = requant_scale(codes, s_wg)
    return QuantizedWeights(packed=pack_i4(codes), rows=k, cols=n, scheme=PER_GROUP, group_size=gs, s_wg=s_wg,
                            s_wc=s_wc)


def requant_scale(q4, s_wg) -> torch.Tensor:
    """Per-channel requant scale over binary16-dequantized group weights (quantize.py:152-168)."""
    q4 = as_cuda(q4 if isinstance(q4, torch.Tensor) else np.asarray(q4), torch.int8).contiguous()
    s_wg = as_cuda(s_wg if isinstance(s_wg, torch.Tensor) else np.asarray(s_wg, dtype=np.float64),
                   torch.float64).contiguous()
    k, n = q4.shape
    groups = s_wg.shape[0]
    if groups == 0 or k % groups != 0:
        raise ShapeError("group scale rows do not divide code rows")
    dev = q4.device
    lib = _lib.lib_for_device(dev)
    out = torch.empty((n,), dtype=torch.float64, device=dev)
    _lib.check(lib.qqq_requant_scale(_lib.ptr(q4), _lib.ptr(s_wg), k, n, groups, _lib.ptr(out),
                                     _lib.stream_of(dev)), "requant_scale")
    return out


def pack_i4(q4) -> torch.Tensor:
    """Pack INT4 codes two-per-byte, row 2k low nibble, 2k+1 high (quantize.py:171-189)."""
    if isinstance(q4, torch.Tensor):
        t = q4
    else:
        arr = np.asarray(q4)
        if arr.ndim != 2:
            raise ShapeError("codes must be 2-D (K x N)")
        if arr.size and (arr.min() < -128 or arr.max() > 127):
            raise DataError("INT4 codes out of [-8, 7]")
        t = torch.from_numpy(np.ascontiguousarray(arr.astype(np.int8)))
    if t.ndim != 2:
        raise ShapeError("codes must be 2-D (K x N)")
    if t.dtype != torch.int8:
        t = as_cuda(t)
        if t.numel() and (int(t.min()) < -8 or int(t.max()) > 7):
            raise DataError("INT4 codes out of [-8, 7]")
        t = t.to(torch.int8)
    t = as_cuda(t).contiguous()
    k, n = t.shape
    dev = t.device
    lib = _lib.lib_for_device(dev)
    packed = torch.empty(((k + 1) // 2, n), dtype=torch.uint8, device=dev)
    if k and n:
        status = _status(dev)
        _lib.check(lib.qqq_pack_i4(_lib.ptr(t), k, n, _lib.ptr(packed), _lib.ptr(status), _lib.stream_of(dev)),
                   "pack_i4")
        raise_if_bad(status, "codes")
    return packed


def unpack_i4(packed, rows: int) -> torch.Tensor:
    """Inverse of pack_i4; validates the padding nibble against the true K (quantize.py:192-208)."""
    p = as_cuda(packed if isinstance(packed, torch.Tensor) else np.asarray(packed, dtype=np.uint8))
    if p.ndim != 2:
        raise ShapeError("packed tensor must be 2-D")
    p = p.to(torch.uint8).contiguous()
    if p.shape[0] != (rows + 1) // 2:
        raise CorruptionError(f"packed rows {p.shape[0]} inconsistent with true K={rows}")
    n = p.shape[1]
    dev = p.device
    out = torch.empty((rows, n), dtype=torch.int8, device=dev)
    if rows and n:
        lib = _lib.lib_for_device(dev)
        status = _status(dev)
        _lib.check(lib.qqq_unpack_i4(_lib.ptr(p), rows, n, _lib.ptr(out), _lib.ptr(status), _lib.stream_of(dev)),
                   "unpack_i4")
        raise_if_bad(status, "packed")
    return out


def dequantize_ref(qw: QuantizedWeights) -> torch.Tensor:
    """Wide-precision dequantization, f64 K x N (quantize.py:211-217)."""
    codes = qw.codes()
    k, n = codes.shape
    dev = codes.device
    lib = _lib.lib_for_device(dev)
    out = torch.empty((k, n), dtype=torch.float64, device=dev)
    if qw.scheme == PER_CHANNEL:
        scales, g = as_cuda(qw.s_w, torch.float64).contiguous(), 0
    else:
        scales, g = as_cuda(qw.s_wg, torch.float64).contiguous(), qw.group_size
    _lib.check(lib.qqq_dequantize(_lib.ptr(codes), k, n, g, _lib.ptr(scales), _lib.ptr(out), _lib.stream_of(dev)),
               "dequantize_ref")
    return out
