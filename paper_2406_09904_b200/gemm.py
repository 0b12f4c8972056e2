"""Drop-in for the reference GEMM module (pkg/src/qqq/gemm.py) on B200.

`w4a8_gemm_per_channel` / `w4a8_gemm_per_group` keep the reference's
signature, validation (`_check_gemm_operands`, gemm.py:157-170) and outputs
(`GemmOutput(y, acc)`), and run one sm_100a kernel: INT4->INT8 conversion in
shared memory, tcgen05 INT8 MMA with int32 accumulators in TMEM, and the f64
dequant epilogue — bit-identical to the reference (y and acc).

The one-time weight repack into the kernel layout is cached on the
QuantizedWeights / FusedScales objects (the reference re-unpacks per call).
"""

from __future__ import annotations

import threading
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch

from . import _lib
from .errors import ConfigError, CorruptionError, ShapeError
from .quantize import (
    PER_CHANNEL,
    PER_GROUP,
    QuantizedActivations,
    QuantizedWeights,
    as_cuda,
    raise_if_bad,
    rowsum_of,
)

__all__ = [
    "MAGIC_ADDEND",
    "FusedScales",
    "GemmOutput",
    "fast_i4_to_i8",
    "fast_i4_to_f16",
    "fast_f16_to_i8",
    "fused_dequant_quant",
    "gemm_i8_i32",
    "w4a8_gemm_per_channel",
    "w4a8_gemm_per_group",
]

MAGIC_ADDEND = 1152.0  # gemm.py:44
_MAX_GEMM_K = 1 << 16  # gemm.py:49


@dataclass(frozen=True)
class FusedScales:
    """Offline-prepared epilogue scales for one GEMM dataflow (gemm.py:52-69)."""

    scheme: str
    s_w_folded: Optional[torch.Tensor] = None  # per-channel: s_W / 16, length N (f64)
    s_star: Optional[torch.Tensor] = None  # per-group: float16 s_Wg / s_Wc, G x N
    s_wc: Optional[torch.Tensor] = None  # per-group: requant scales, length N (f64)
    _cache: dict = field(default_factory=dict, repr=False, compare=False, hash=False)

    @classmethod
    def from_quantized(cls, qw: QuantizedWeights) -> "FusedScales":
        if qw.scheme == PER_CHANNEL:
            return cls(scheme=PER_CHANNEL, s_w_folded=as_cuda(qw.s_w, torch.float64) / 16.0)
        s_wg = as_cuda(qw.s_wg, torch.float64).contiguous()
        s_wc = as_cuda(qw.s_wc, torch.float64).contiguous()
        g, n = s_wg.shape
        dev = s_wg.device
        lib = _lib.lib_for_device(dev)
        s_star = torch.empty((g, n), dtype=torch.float16, device=dev)
        status = torch.zeros(1, dtype=torch.int32, device=dev)
        _lib.check(lib.qqq_fused_scales_pg(_lib.ptr(s_wg), _lib.ptr(s_wc), g, n, _lib.ptr(s_star), _lib.ptr(status),
                                           _lib.stream_of(dev)), "FusedScales.from_quantized")
        raise_if_bad(status, "fused scales")
        return cls(scheme=PER_GROUP, s_star=s_star, s_wc=s_wc.clone())


@dataclass
class GemmOutput:  # gemm.py:72-78
    y: torch.Tensor  # float16, tokens x N
    acc: Optional[torch.Tensor]  # int32, tokens x N (None when with_acc=False)

    def y_wide(self) -> torch.Tensor:
        return self.y.to(torch.float64)


# ---------------------------------------------------------------------------
# kernel-layout caches and workspace
# ---------------------------------------------------------------------------

_ws_lock = threading.Lock()
_workspaces: dict = {}
_retired: list = []  # outgrown workspaces stay allocated: captured CUDA graphs may still address them


def workspace(device: torch.device, nbytes: int, stream=None) -> torch.Tensor:
    """Zeroed split-K workspace (tile counters + partial slots) per (device,
    stream); every launch leaves it zeroed again.

    GEMMs on one stream run in order, so they share one workspace; GEMMs on
    different streams (which may overlap) get different ones. A workspace that
    is outgrown is replaced but never freed, because a CUDA graph captured
    earlier may still launch into it.
    """
    dev = torch.device(device)
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    st = torch.cuda.current_stream(dev) if stream is None else stream
    key = (dev.index, st.cuda_stream)
    with _ws_lock:
        ws = _workspaces.get(key)
        if ws is None or ws.numel() < nbytes:
            with torch.cuda.stream(st):
                new = torch.zeros(max(nbytes, 1 << 20), dtype=torch.uint8, device=dev)
            if ws is not None:
                _retired.append(ws)
            ws = _workspaces[key] = new
    return ws


def _version_key(t):
    """Cache key of a weight/scale operand: identity + in-place version for torch
    tensors; identity + data pointer + a CRC of the bytes for host arrays (numpy
    has no version counter, so in-place edits are caught by the checksum)."""
    if isinstance(t, torch.Tensor):
        return ("t", t.data_ptr(), t._version, tuple(t.shape), t.dtype)
    import zlib

    a = np.ascontiguousarray(np.asarray(t))
    return ("np", id(t), a.__array_interface__["data"][0], a.shape, a.dtype.str, zlib.crc32(a.view(np.uint8).ravel()))


def _pg_fast_ok(g: int) -> bool:
    """Per-group group sizes the nibble kernel layout supports (qqq_layout.cuh)."""
    return g > 0 and ((g % 32 == 0 and 128 % g == 0) or g % 128 == 0)


def _check_padding(qw: QuantizedWeights) -> None:
    # unpack_i4's odd-K padding check (quantize.py:206-207) is part of codes()
    if qw.rows % 2:
        last = as_cuda(qw.packed, torch.uint8)[-1]
        if bool(((last >> 4) != 8).any()):
            raise CorruptionError("nonzero padding nibble for odd K")


@dataclass
class PreparedWeights:
    """Kernel-ready weights: mode, repacked bytes, optional per-tile scales."""

    mode: int
    w: torch.Tensor
    sc: Optional[torch.Tensor]
    group: int
    s_col: torch.Tensor


def prepare(qw: QuantizedWeights, fused: FusedScales) -> PreparedWeights:
    """One-time repack (cached) of the reference packing into the tcgen05 blob.

    Cache key: the identity and in-place version of qw.packed (and fused.s_star,
    fused.s_wc), so a mutated or replaced operand is repacked again; host
    (numpy) operands are keyed by identity and a checksum of their bytes.
    """
    k, n = qw.rows, qw.cols
    if tuple(qw.packed.shape) != ((k + 1) // 2, n):
        raise CorruptionError(f"packed shape {tuple(qw.packed.shape)} inconsistent with K={k}, N={n}")
    if qw.scheme == PER_CHANNEL:
        key = ("pc", _version_key(qw.packed))
        hit = qw._cache.get("pc")
        if hit is None or hit[0] != key:
            packed = as_cuda(qw.packed, torch.uint8).contiguous()
            dev = packed.device
            lib = _lib.lib_for_device(dev)
            w = torch.empty(lib.qqq_repacked_weight_bytes(_lib.MODE_PC, k, n, 0), dtype=torch.uint8, device=dev)
            _lib.check(lib.qqq_repack_weights(_lib.ptr(packed), None, k, n, _lib.MODE_PC, 0, _lib.ptr(w), None,
                                              _lib.stream_of(dev)), "repack_weights")
            hit = (key, w)
            qw._cache["pc"] = hit
        return PreparedWeights(_lib.MODE_PC, hit[1], None, 0, as_cuda(fused.s_w_folded, torch.float64).contiguous())
    g = qw.group_size
    key = ("pg", _version_key(qw.packed), _version_key(fused.s_star), _version_key(fused.s_wc), g)
    hit = fused._cache.get("pg")
    if hit is not None and hit[0] == key:
        return hit[1]
    packed = as_cuda(qw.packed, torch.uint8).contiguous()
    dev = packed.device
    lib = _lib.lib_for_device(dev)
    s_star = as_cuda(fused.s_star, torch.float16).contiguous()
    s_wc = as_cuda(fused.s_wc, torch.float64).contiguous()
    prep = None
    if _pg_fast_ok(g):
        w = torch.empty(lib.qqq_repacked_weight_bytes(_lib.MODE_PG, k, n, g), dtype=torch.uint8, device=dev)
        flags = torch.zeros(1, dtype=torch.int32, device=dev)
        _lib.check(lib.qqq_repack_weights(_lib.ptr(packed), _lib.ptr(s_star), k, n, _lib.MODE_PG, g, _lib.ptr(w),
                                          _lib.ptr(flags), _lib.stream_of(dev)), "repack_weights")
        if (int(flags.item()) & _lib.STAT_NEED_CLAMP) == 0:
            prep = PreparedWeights(_lib.MODE_PG, w, None, g, s_wc)
    if prep is None:
        # exact scalar FusedDequantQuant (with the reference clamp) into int8 once
        w8 = torch.empty(lib.qqq_repacked_weight_bytes(_lib.MODE_I8, k, n, 0), dtype=torch.uint8, device=dev)
        _lib.check(lib.qqq_repack_weights_i8(None, _lib.ptr(packed), _lib.ptr(s_star), g, k, n, _lib.ptr(w8),
                                             _lib.stream_of(dev)), "repack_weights_i8")
        prep = PreparedWeights(_lib.MODE_I8, w8, None, 0, s_wc)
    fused._cache["pg"] = (key, prep)
    return prep


def _aligned_q(aq: QuantizedActivations) -> torch.Tensor:
    """The kernel reads rows as 128-byte atoms: row pitch % 16 == 0 and >= round_up(K, 128)."""
    q = as_cuda(aq.q, torch.int8)
    m, k = q.shape
    kp = (k + 127) // 128 * 128
    if m == 0:
        return q
    pitch = q.stride(0) if m > 1 else kp
    if (q.stride(1) == 1 and q.data_ptr() % 16 == 0 and pitch % 16 == 0 and pitch >= kp
            and q.untyped_storage().nbytes() - q.storage_offset() >= (m - 1) * pitch + kp):
        return q
    buf = torch.zeros((m, kp), dtype=torch.int8, device=q.device)
    buf[:, :k] = q
    return buf[:, :k]


def run_gemm(aq: QuantizedActivations, prep: PreparedWeights, n: int, with_acc: bool = True,
             y_out: Optional[torch.Tensor] = None, cfg: Optional[dict] = None,
             ws: Optional[torch.Tensor] = None) -> GemmOutput:
    """Launch the W4A8 kernel on the current stream (no host sync)."""
    q = _aligned_q(aq)
    m, k = q.shape
    if k > _MAX_GEMM_K:
        raise ShapeError(f"K={k} risks INT32 accumulator overflow")
    dev = q.device
    lib = _lib.lib_for_device(dev)
    s_a = as_cuda(aq.s_a, torch.float64).contiguous()
    y = y_out if y_out is not None else torch.empty((m, n), dtype=torch.float16, device=dev)
    acc = torch.empty((m, n), dtype=torch.int32, device=dev) if with_acc else None
    if m == 0:
        return GemmOutput(y=y, acc=acc)
    wsb = lib.qqq_gemm_workspace_bytes(m, n, k)
    if ws is None or ws.numel() < wsb:
        ws = workspace(dev, wsb)
    c = None
    if cfg:
        dbg = cfg.get("dbg")
        c = _lib.GemmConfig(int(cfg.get("ntok", 0)), int(cfg.get("grid", 0)), int(cfg.get("split", -1)),
                            int(cfg.get("csplit", 0)), None if dbg is None else dbg.data_ptr())
    ldq = q.stride(0) if m > 1 else (k + 127) // 128 * 128
    rs = rowsum_of(aq) if prep.mode == _lib.MODE_PG else None
    rc = lib.qqq_w4a8_gemm_ex(prep.mode, _lib.ptr(q), ldq, _lib.ptr(s_a), _lib.ptr(rs), _lib.ptr(prep.w),
                              prep.group, _lib.ptr(prep.s_col), m, n, k, _lib.ptr(y), y.stride(0),
                              _lib.ptr(acc), n, _lib.ptr(ws), ws.numel(),
                              None if c is None else c, _lib.stream_of(dev))
    _lib.check(rc, "w4a8_gemm")
    return GemmOutput(y=y, acc=acc)


def plan_info(mode: int, m: int, n: int, k: int, cfg: Optional[dict] = None) -> dict:
    """The tile plan a GEMM launch would use (no device work): ntok, split,
    grid, csplit. Split codes as in qqq_gemm_config (include/qqq_b200.h)."""
    lib = _lib.load()
    c = None
    if cfg:
        c = _lib.GemmConfig(int(cfg.get("ntok", 0)), int(cfg.get("grid", 0)), int(cfg.get("split", -1)),
                            int(cfg.get("csplit", 0)), None)
    out = _lib.GemmConfig()
    _lib.check(lib.qqq_gemm_plan_info(mode, m, n, k, c, out), "gemm_plan_info")
    return {"ntok": out.ntok, "split": out.split, "grid": out.grid, "csplit": out.csplit}


def _check_gemm_operands(aq: QuantizedActivations, qw: QuantizedWeights, fused: FusedScales, scheme: str) -> None:
    """gemm.py:157-170."""
    if qw.scheme != scheme or fused.scheme != scheme:
        raise ConfigError(
            f"engine expects {scheme} operands, got weights={qw.scheme!r} scales={fused.scheme!r}")
    if aq.q.shape[1] != qw.rows:
        raise ShapeError(f"activation K={aq.q.shape[1]} does not match weight K={qw.rows}")
    if tuple(aq.s_a.shape) != (aq.q.shape[0],):
        raise ShapeError("per-token scale length does not match token count")


def w4a8_gemm_per_channel(aq: QuantizedActivations, qw: QuantizedWeights, fused: FusedScales,
                          with_acc: bool = True) -> GemmOutput:
    """Per-channel dataflow: x16 shift, INT8 GEMM, dequant with s_W/16 (gemm.py:173-185)."""
    _check_gemm_operands(aq, qw, fused, PER_CHANNEL)
    if tuple(fused.s_w_folded.shape) != (qw.cols,):
        raise ShapeError("folded scale length does not match N")
    _check_padding(qw)
    return run_gemm(aq, prepare(qw, fused), qw.cols, with_acc)


def w4a8_gemm_per_group(aq: QuantizedActivations, qw: QuantizedWeights, fused: FusedScales,
                        with_acc: bool = True) -> GemmOutput:
    """Per-group dataflow: FusedDequantQuant to INT8, INT8 GEMM, dequant with s_Wc (gemm.py:188-203)."""
    _check_gemm_operands(aq, qw, fused, PER_GROUP)
    if qw.rows % qw.group_size != 0 or tuple(fused.s_star.shape) != (qw.rows // qw.group_size, qw.cols):
        raise ConfigError("fused group scales do not match the group structure")
    _check_padding(qw)
    return run_gemm(aq, prepare(qw, fused), qw.cols, with_acc)


def gemm_i8_i32(aq, w8) -> torch.Tensor:
    """Exact INT8 x INT8 -> INT32 matrix multiply (gemm.py:145-154) on tcgen05 (I8 mode)."""
    a = as_cuda(aq if isinstance(aq, torch.Tensor) else np.asarray(aq), torch.int8)
    b = as_cuda(w8 if isinstance(w8, torch.Tensor) else np.asarray(w8), torch.int8)
    if a.ndim != 2 or b.ndim != 2 or a.shape[1] != b.shape[0]:
        raise ShapeError(f"inner dimensions differ: {tuple(a.shape)} x {tuple(b.shape)}")
    if a.shape[1] > _MAX_GEMM_K:
        raise ShapeError(f"K={a.shape[1]} risks INT32 accumulator overflow")
    m, k = a.shape
    n = b.shape[1]
    dev = a.device
    lib = _lib.lib_for_device(dev)
    b = b.contiguous()
    wb = torch.empty(lib.qqq_repacked_weight_bytes(_lib.MODE_I8, k, n, 0), dtype=torch.uint8, device=dev)
    _lib.check(lib.qqq_repack_weights_i8(_lib.ptr(b), None, None, 0, k, n, _lib.ptr(wb), _lib.stream_of(dev)),
               "repack_weights_i8")
    ones = torch.ones(max(m, 1), dtype=torch.float64, device=dev)
    aqq = QuantizedActivations(q=a, s_a=ones[:m])
    prep = PreparedWeights(_lib.MODE_I8, wb, None, 0, None)
    q = _aligned_q(aqq)
    acc = torch.empty((m, n), dtype=torch.int32, device=dev)
    if m == 0:
        return acc
    ws = workspace(dev, lib.qqq_gemm_workspace_bytes(m, n, k))
    ldq = q.stride(0) if m > 1 else (k + 127) // 128 * 128
    _lib.check(lib.qqq_w4a8_gemm_ex(_lib.MODE_I8, _lib.ptr(q), ldq, _lib.ptr(aqq.s_a), None, _lib.ptr(prep.w),
                                    0, None, m, n, k, None, n, _lib.ptr(acc), n, _lib.ptr(ws), ws.numel(), None,
                                    _lib.stream_of(dev)), "gemm_i8_i32")
    return acc


# ---------------------------------------------------------------------------
# The paper's bit-trick conversions (gemm.py:81-127). Scalar reference API,
# evaluated by the exact device functions the GEMM kernel uses.
# ---------------------------------------------------------------------------


def fast_i4_to_i8(q: int) -> int:
    """q * 16 via the kernel's (u << 4) ^ 0x80 converter (gemm.py:81-85)."""
    if not -8 <= int(q) <= 7:
        raise CorruptionError(f"INT4 code out of range: {q}")
    return int(fast_i4_to_i8_array(np.full(8, q, dtype=np.int8))[0])


def fast_i4_to_i8_array(codes) -> np.ndarray:
    c = as_cuda(np.asarray(codes, dtype=np.int8)).contiguous()
    n = c.numel()
    pad = (-n) % 8
    if pad:
        c = torch.cat([c, torch.zeros(pad, dtype=torch.int8, device=c.device)])
    out = torch.empty_like(c)
    lib = _lib.lib_for_device(c.device)
    _lib.check(lib.qqq_test_pc_convert(_lib.ptr(c), _lib.ptr(out), c.numel(), _lib.stream_of(c.device)),
               "fast_i4_to_i8")
    return out[:n].cpu().numpy()


def fast_i4_to_f16(u: int):
    """Magic-number nibble-to-FP16 (gemm.py:88-96): f16(0x6400 | u) - 1032 == u - 8."""
    from .numerics import Binary16, encode_f16

    if not 0 <= int(u) <= 15:
        raise CorruptionError(f"nibble out of range: {u}")
    h = torch.tensor([0x6400 | int(u)], dtype=torch.int16).view(torch.float16)
    h = as_cuda(h) - torch.tensor(1032.0, dtype=torch.float16, device=_lib_device())
    return Binary16(int(h.view(torch.int16).cpu().item()) & 0xFFFF)


def _lib_device():
    return torch.device("cuda", torch.cuda.current_device())


def fast_f16_to_i8(x) -> int:
    """Magic-number FP16 -> INT8 (gemm.py:99-107), device FastFP16toINT8."""
    bits = np.array([x.bits], dtype=np.uint16)
    return int(fast_f16_to_i8_bits(bits)[0])


def fast_f16_to_i8_bits(bits) -> np.ndarray:
    b = as_cuda(torch.from_numpy(np.ascontiguousarray(np.asarray(bits, dtype=np.uint16)).view(np.int16))).contiguous()
    out = torch.empty(b.shape, dtype=torch.int8, device=b.device)
    lib = _lib.lib_for_device(b.device)
    _lib.check(lib.qqq_test_fast_f16_to_i8(_lib.ptr(b), _lib.ptr(out), b.numel(), _lib.stream_of(b.device)),
               "fast_f16_to_i8")
    return out.cpu().numpy()


def fused_dequant_quant(u: int, s_star) -> int:
    """FusedDequantQuant of one nibble with a binary16 scale (gemm.py:110-127)."""
    if not 0 <= int(u) <= 15:
        raise CorruptionError(f"nibble out of range: {u}")
    sval = s_star.to_float()
    if not np.isfinite(sval) or sval <= 0.0:
        raise ConfigError(f"fused scale must be positive and finite: {sval}")
    return int(fused_dequant_quant_array(np.array([int(u) - 8]), np.array([s_star.bits], dtype=np.uint16))[0])


def fused_dequant_quant_array(q, s_bits, word_path: bool = False) -> np.ndarray:
    """Vectorized FusedDequantQuant on the device (scalar branch or the GEMM's HFMA2 word path)."""
    qq = as_cuda(np.ascontiguousarray(np.asarray(q, dtype=np.int8))).contiguous()
    ss = as_cuda(torch.from_numpy(np.ascontiguousarray(np.asarray(s_bits, dtype=np.uint16)).view(np.int16)))
    out = torch.empty_like(qq)
    lib = _lib.lib_for_device(qq.device)
    _lib.check(lib.qqq_test_fused_dequant_quant(_lib.ptr(qq), _lib.ptr(ss.contiguous()), _lib.ptr(out), qq.numel(),
                                                1 if word_path else 0, _lib.stream_of(qq.device)),
               "fused_dequant_quant")
    return out.cpu().numpy()
