"""ctypes binding of the C ABI in include/qqq_b200.h (libqqq_b200.so).

There is no fallback: if the library is missing or the current device is not
an sm_100 B200, every entry point raises KernelError.
"""

from __future__ import annotations

import ctypes
import os
import threading
from ctypes import c_char_p, c_int, c_int64, c_size_t, c_void_p

from .errors import ConfigError, CorruptionError, DataError, KernelError, ShapeError

# QQQ_TIMELINE_LIB=1 selects the developer build with in-kernel timeline stamps
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib",
                        "libqqq_b200_tl.so" if os.environ.get("QQQ_TIMELINE_LIB") == "1" else "libqqq_b200.so")
LIB_PATH = os.environ.get("QQQ_LIB_PATH", LIB_PATH)  # developer A/B builds (scripts/)

QQQ_OK, QQQ_ERR_SHAPE, QQQ_ERR_DATA, QQQ_ERR_CONFIG, QQQ_ERR_CORRUPTION, QQQ_ERR_CUDA, QQQ_ERR_UNSUPPORTED = range(7)
STAT_NONFINITE, STAT_CODE_RANGE, STAT_PAD_NIBBLE, STAT_SCALE_INF, STAT_NEED_CLAMP, STAT_TINY_SCALE = 1, 2, 4, 8, 16, 32
MODE_PC, MODE_PG, MODE_I8 = 0, 1, 2


class GemmConfig(ctypes.Structure):
    _fields_ = [("ntok", c_int), ("grid", c_int), ("split", c_int), ("csplit", c_int), ("dbg", c_void_p)]


P = c_void_p
I64 = c_int64
S = c_void_p  # cudaStream_t

# name -> (restype, argtypes); mirrors include/qqq_b200.h exactly
SIGNATURES = {
    "qqq_act_quant": (c_int, [P, c_int, I64, I64, I64, P, I64, P, P, S]),
    "qqq_act_quant_ex": (c_int, [P, c_int, I64, I64, I64, P, I64, P, P, P, S]),
    "qqq_act_rowsum": (c_int, [P, I64, I64, I64, P, S]),
    "qqq_act_quant_smooth": (c_int, [P, c_int, I64, I64, I64, P, P, P, I64, P, P, P, S]),
    "qqq_smooth_reciprocal": (c_int, [P, I64, P, S]),
    "qqq_matmul_ref_f64": (c_int, [P, P, P, I64, I64, I64, S]),
    "qqq_gptq_block": (c_int, [P, I64, I64, P, I64, I64, I64, P, P, P, P, S]),
    "qqq_act_quant_smooth_rcp": (c_int, [P, c_int, I64, I64, I64, P, P, P, I64, P, P, P, S]),
    "qqq_act_absmax": (c_int, [P, c_int, I64, I64, I64, P, P, S]),
    "qqq_act_quant_with_max": (c_int, [P, c_int, I64, I64, I64, P, P, I64, P, P, P, S]),
    "qqq_dequant_epilogue": (c_int, [P, I64, I64, I64, P, P, P, I64, S]),
    "qqq_quant_weight": (c_int, [P, I64, I64, I64, P, P, P, S]),
    "qqq_requant_scale": (c_int, [P, P, I64, I64, I64, P, S]),
    "qqq_pack_i4": (c_int, [P, I64, I64, P, P, S]),
    "qqq_unpack_i4": (c_int, [P, I64, I64, P, P, S]),
    "qqq_fused_scales_pg": (c_int, [P, P, I64, I64, P, P, S]),
    "qqq_dequantize": (c_int, [P, I64, I64, I64, P, P, S]),
    "qqq_repacked_weight_bytes": (c_size_t, [c_int, I64, I64, I64]),
    "qqq_repack_weights": (c_int, [P, P, I64, I64, c_int, I64, P, P, S]),
    "qqq_repack_weights_i8": (c_int, [P, P, P, I64, I64, I64, P, S]),
    "qqq_gemm_workspace_bytes": (c_size_t, [I64, I64, I64]),
    "qqq_w4a8_gemm_pc": (c_int, [P, I64, P, P, P, I64, I64, I64, P, I64, P, I64, P, c_size_t, S]),
    "qqq_w4a8_gemm_pg": (c_int, [P, I64, P, P, P, I64, P, I64, I64, I64, P, I64, P, I64, P, c_size_t, S]),
    "qqq_w4a8_gemm_ex": (c_int, [c_int, P, I64, P, P, P, I64, P, I64, I64, I64, P, I64, P, I64, P, c_size_t,
                                  ctypes.POINTER(GemmConfig), S]),
    "qqq_w4a8_gemm_smooth_fused": (c_int, [c_int, P, I64, P, P, P, I64, P, P, P, P, I64, P, I64, I64, I64, P, I64,
                                            P, I64, P, c_size_t, ctypes.POINTER(GemmConfig), S]),
    "qqq_gemm_plan_info": (c_int, [c_int, I64, I64, I64, ctypes.POINTER(GemmConfig), ctypes.POINTER(GemmConfig)]),
    "qqq_test_fused_dequant_quant": (c_int, [P, P, P, I64, c_int, S]),
    "qqq_test_pc_convert": (c_int, [P, P, I64, S]),
    "qqq_test_fast_f16_to_i8": (c_int, [P, P, I64, S]),
    "qqq_probe_int8_peak": (c_int, [c_int, c_int, P, S]),
    "qqq_device_ok": (c_int, []),
    "qqq_version": (c_char_p, []),
}

_lib = None
_lock = threading.Lock()
_device_checked = set()


def load() -> ctypes.CDLL:
    """Load the in-tree CUDA library (no JIT, no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise KernelError(
                    f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                    "(nvcc, sm_100a). There is no CPU fallback.")
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


class _OnDevice:
    """The library with every entry point called under `torch.cuda.device(idx)`:
    the C ABI launches on the calling thread's current device, so a call for a
    tensor on another GPU of the process switches to it for the call."""

    def __init__(self, lib, idx: int):
        self._lib = lib
        self._idx = idx

    def __getattr__(self, name):
        import torch

        fn = getattr(self._lib, name)
        idx = self._idx

        def call(*args):
            with torch.cuda.device(idx):
                return fn(*args)

        return call


def lib_for_device(device):
    """The library, after checking that `device` is an sm_100 GPU. When `device`
    is not the current device, the returned handle switches to it per call."""
    import torch

    lib = load()
    idx = torch.device(device).index
    cur = torch.cuda.current_device()
    idx = cur if idx is None else idx
    if idx not in _device_checked:
        major, minor = torch.cuda.get_device_capability(idx)
        if (major, minor) != (10, 0):
            raise KernelError(f"device {idx} is sm_{major}{minor}; the kernels are built for sm_100a only")
        _device_checked.add(idx)
    return lib if idx == cur else _OnDevice(lib, idx)


_RC = {
    QQQ_ERR_SHAPE: ShapeError,
    QQQ_ERR_DATA: DataError,
    QQQ_ERR_CONFIG: ConfigError,
    QQQ_ERR_CORRUPTION: CorruptionError,
    QQQ_ERR_CUDA: KernelError,
    QQQ_ERR_UNSUPPORTED: ConfigError,
}


def check(rc: int, what: str) -> None:
    if rc != QQQ_OK:
        raise _RC.get(rc, KernelError)(f"{what} failed (status {rc})")


def ptr(t) -> int:
    return 0 if t is None else t.data_ptr()


def stream_of(device) -> int:
    import torch

    return torch.cuda.current_stream(device).cuda_stream
