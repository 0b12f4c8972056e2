"""QQQ1 checkpoint container and the `i4p` -> GPU loader.

File format (the reference's, pkg/src/qqq/checkpoint.py:1-15): 4-byte magic
"QQQ1", little-endian u64 header length, UTF-8 JSON header
{"tensors": {name: {dtype, shape, offset, nbytes[, rows]}}, "metadata": ...},
then tensor data starting at the first 64-byte boundary; offsets are
relative to it, 64-byte aligned and non-overlapping. dtypes f32 / f16 / i8 /
i4p ("i4p" = pack_i4 bytes, "rows" = the true K).

`read_checkpoint` / `write_checkpoint` keep the reference's validation,
error messages (CheckpointFormatError) and byte-exact output. The loader
side is B200-specific: the file is memory-mapped (only the tensors a layer
needs are touched), the packed int4 bytes and scales go to the GPU as
QuantizedWeights, and the one-time repack into the GEMM's tile layout runs on
the GPU at load time (`gemm.prepare`) instead of at the first GEMM.
"""

from __future__ import annotations

import json
import mmap
import struct
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch

from .errors import CheckpointFormatError

__all__ = ["MAGIC", "ALIGN", "TensorRecord", "Checkpoint", "write_checkpoint", "read_checkpoint",
           "store_layer", "load_layer", "load_layers"]

MAGIC = b"QQQ1"  # checkpoint.py:30
ALIGN = 64       # checkpoint.py:31

_DTYPES = {"f32": np.dtype("<f4"), "f16": np.dtype("<f2"), "i8": np.dtype("i1"), "i4p": np.dtype("u1")}


def _aligned(n: int) -> int:
    return -(-n // ALIGN) * ALIGN


@dataclass
class TensorRecord:  # checkpoint.py:41-64
    dtype: str
    array: np.ndarray
    rows: Optional[int] = None  # true K of an i4p tensor

    def __post_init__(self) -> None:
        if self.dtype not in _DTYPES:
            raise CheckpointFormatError(f"unknown dtype {self.dtype!r}")
        self.array = np.ascontiguousarray(self.array, dtype=_DTYPES[self.dtype])
        if self.dtype == "i4p" and self.rows is None:
            raise CheckpointFormatError("i4p tensor requires a true row count")

    def __eq__(self, other: object) -> bool:
        if not isinstance(other, TensorRecord):
            return NotImplemented
        return (self.dtype, self.rows, self.array.shape) == (other.dtype, other.rows, other.array.shape) and bool(
            np.array_equal(self.array, other.array))


@dataclass
class Checkpoint:  # checkpoint.py:67-79
    tensors: dict = field(default_factory=dict)
    metadata: dict = field(default_factory=dict)

    def add(self, name: str, dtype: str, array, rows: Optional[int] = None) -> None:
        if isinstance(array, torch.Tensor):
            array = array.detach().cpu().numpy()
        self.tensors[name] = TensorRecord(dtype=dtype, array=array, rows=rows)

    def __eq__(self, other: object) -> bool:
        if not isinstance(other, Checkpoint):
            return NotImplemented
        return self.tensors == other.tensors and self.metadata == other.metadata


def write_checkpoint(ckpt: Checkpoint, path: str) -> None:
    """checkpoint.py:86-118: tensors in name order at 64-byte aligned offsets,
    sorted-key JSON header — the bytes are a pure function of the content."""
    index, pos = {}, 0
    names = sorted(ckpt.tensors)
    for name in names:
        rec = ckpt.tensors[name]
        e = {"dtype": rec.dtype, "shape": list(rec.array.shape), "offset": pos, "nbytes": int(rec.array.nbytes)}
        if rec.rows is not None:
            e["rows"] = rec.rows
        index[name] = e
        pos = _aligned(pos + rec.array.nbytes)
    header = json.dumps({"tensors": index, "metadata": ckpt.metadata}, sort_keys=True).encode("utf-8")
    head = MAGIC + struct.pack("<Q", len(header)) + header
    with open(path, "wb") as f:
        f.write(head + bytes(_aligned(len(head)) - len(head)))
        at = 0
        for name in names:
            arr = ckpt.tensors[name].array
            f.write(bytes(index[name]["offset"] - at))
            f.write(arr.tobytes())
            at = index[name]["offset"] + arr.nbytes


class _Mapped:
    """Read-only memory map of a checkpoint file (empty files map to b"")."""

    def __init__(self, path: str):
        self._f = open(path, "rb")
        try:
            self.buf = mmap.mmap(self._f.fileno(), 0, access=mmap.ACCESS_READ)
        except ValueError:  # zero-length file
            self.buf = b""

    def close(self) -> None:
        if isinstance(self.buf, mmap.mmap):
            self.buf.close()
        self._f.close()


def _parse(buf) -> tuple[dict, int]:
    """Header checks of checkpoint.py:125-139; returns (header, data start)."""
    if bytes(buf[:4]) != MAGIC:
        raise CheckpointFormatError(f"bad magic: {bytes(buf[:4])!r}")
    if len(buf) < 12:
        raise CheckpointFormatError("file truncated before header length")
    (hlen,) = struct.unpack("<Q", bytes(buf[4:12]))
    if 12 + hlen > len(buf):
        raise CheckpointFormatError("file truncated inside header")
    try:
        header = json.loads(bytes(buf[12:12 + hlen]).decode("utf-8"))
    except (UnicodeDecodeError, json.JSONDecodeError) as exc:
        raise CheckpointFormatError(f"header is not valid JSON: {exc}") from exc
    if not isinstance(header, dict) or "tensors" not in header:
        raise CheckpointFormatError("header missing tensor index")
    return header, _aligned(12 + hlen)


def _spans(header: dict, data_len: int) -> dict:
    """Per-tensor checks of checkpoint.py:144-168 (dtype, alignment, size,
    bounds, no overlap); returns name -> (dtype, shape, offset, nbytes, rows)."""
    out, spans = {}, []
    for name, e in header["tensors"].items():
        dtype = e.get("dtype")
        if dtype not in _DTYPES:
            raise CheckpointFormatError(f"tensor {name!r}: unknown dtype {dtype!r}")
        off, nb = int(e["offset"]), int(e["nbytes"])
        shape = tuple(int(d) for d in e["shape"])
        if off % ALIGN:
            raise CheckpointFormatError(f"tensor {name!r}: offset not {ALIGN}-byte aligned")
        if int(np.prod(shape, dtype=np.int64)) * _DTYPES[dtype].itemsize != nb:
            raise CheckpointFormatError(f"tensor {name!r}: nbytes does not match shape")
        if off + nb > data_len:
            raise CheckpointFormatError(f"tensor {name!r}: data extends past end of file")
        spans.append((off, off + nb, name))
        out[name] = (dtype, shape, off, nb, e.get("rows"))
    spans.sort()
    for (_a0, a1, n0), (b0, _b1, n1) in zip(spans, spans[1:]):
        if b0 < a1:
            raise CheckpointFormatError(f"tensors {n0!r} and {n1!r} overlap")
    return out


def read_checkpoint(path: str) -> Checkpoint:
    """checkpoint.py:121-168: parse and validate everything first (a defect
    anywhere raises before any tensor is returned), then copy the tensors out
    of the memory map."""
    m = _Mapped(path)
    try:
        header, start = _parse(m.buf)
        spans = _spans(header, len(m.buf) - start)
        ck = Checkpoint(metadata=header.get("metadata", {}))
        for name, (dtype, shape, off, nb, rows) in spans.items():
            arr = np.frombuffer(m.buf, dtype=_DTYPES[dtype], count=nb // _DTYPES[dtype].itemsize,
                                offset=start + off).reshape(shape).copy()
            ck.tensors[name] = TensorRecord(dtype=dtype, array=arr, rows=rows)
        return ck
    finally:
        m.close()


# ---- layers (pipeline.py:230-281 _store_layer / _load_layer) ---------------------------

def store_layer(ckpt: Checkpoint, layer) -> None:
    """pipeline.py:230-251: packed codes as i4p, scales as f32, the scheme and
    the smoothing plan in the metadata."""
    from .quantize import PER_CHANNEL

    qw, name = layer.qweights, layer.name
    ckpt.add(f"{name}.q4", "i4p", qw.packed, rows=qw.rows)
    f32 = lambda t: (t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)).astype(np.float32)
    if qw.scheme == PER_CHANNEL:
        ckpt.add(f"{name}.s_w", "f32", f32(qw.s_w))
    else:
        ckpt.add(f"{name}.s_wg", "f32", f32(qw.s_wg))
        ckpt.add(f"{name}.s_wc", "f32", f32(qw.s_wc))
    s = layer.plan.s.detach().cpu().numpy() if isinstance(layer.plan.s, torch.Tensor) else np.asarray(layer.plan.s)
    ckpt.metadata.setdefault("layers", {})[name] = {
        "scheme": qw.scheme, "group_size": qw.group_size, "cols": qw.cols,
        "smoothing": {"sigma": layer.plan.sigma, "selected": [int(t) for t in layer.plan.selected],
                      "s": [float(v) for v in s], "objective": layer.plan.objective},
    }


def _layer_from(meta: dict, name: str, get, device, prepare: bool):
    """pipeline.py:254-281 on the GPU: the scale tensors are the stored f32
    values widened to f64, as the reference's `.astype(np.float64)`."""
    from . import gemm as G
    from .pipeline import QuantizedLayer, SmoothingPlan, layer_fused_scales
    from .quantize import PER_CHANNEL, PER_GROUP, QuantizedWeights

    if name not in meta:
        raise CheckpointFormatError(f"no layer {name!r} in checkpoint metadata")
    lm = meta[name]
    dtype, packed, rows = get(f"{name}.q4")
    if dtype != "i4p" or rows is None:
        raise CheckpointFormatError(f"tensor {name + '.q4'!r}: expected i4p with a row count")
    dev = lambda a, dt=None: torch.from_numpy(np.ascontiguousarray(a)).to(device=device, dtype=dt, non_blocking=False)
    f64 = lambda n: dev(get(n)[1], torch.float64)
    if lm["scheme"] == PER_CHANNEL:
        qw = QuantizedWeights(dev(packed), int(rows), int(lm["cols"]), PER_CHANNEL, s_w=f64(f"{name}.s_w"))
    else:
        qw = QuantizedWeights(dev(packed), int(rows), int(lm["cols"]), PER_GROUP, int(lm["group_size"]),
                              s_wg=f64(f"{name}.s_wg"), s_wc=f64(f"{name}.s_wc"))
    sm = lm["smoothing"]
    plan = SmoothingPlan(sigma=float(sm["sigma"]), selected=tuple(int(t) for t in sm["selected"]),
                         s=np.asarray(sm["s"], dtype=np.float64), objective=float(sm["objective"]))
    layer = QuantizedLayer(name=name, qweights=qw, plan=plan)
    if prepare:  # the GPU repack into the tile layout now, not at the first GEMM
        G.prepare(qw, layer_fused_scales(layer))
    return layer


def load_layer(ckpt: Checkpoint, name: str, device="cuda", prepare: bool = True):
    """A QuantizedLayer with its weights on the GPU from a parsed checkpoint."""
    get = lambda n: _tensor(ckpt, n)
    return _layer_from(ckpt.metadata.get("layers", {}), name, get, device, prepare)


def _tensor(ckpt: Checkpoint, n: str):
    rec = ckpt.tensors.get(n)
    if rec is None:
        raise CheckpointFormatError(f"missing tensor {n!r}")
    return rec.dtype, rec.array, rec.rows


def load_layers(path: str, names=None, device="cuda", prepare: bool = True) -> dict:
    """Memory-map a checkpoint file, validate its whole index, and move the
    requested layers (default: all in metadata["layers"]) to the GPU, reading
    only their tensors' byte ranges."""
    m = _Mapped(path)
    try:
        header, start = _parse(m.buf)
        spans = _spans(header, len(m.buf) - start)
        meta = header.get("metadata", {}).get("layers", {})

        def get(n):
            if n not in spans:
                raise CheckpointFormatError(f"missing tensor {n!r}")
            dtype, shape, off, nb, rows = spans[n]
            arr = np.frombuffer(m.buf, dtype=_DTYPES[dtype], count=nb // _DTYPES[dtype].itemsize, offset=start + off)
            return dtype, arr.reshape(shape).copy(), rows  # (the copy outlives the map)

        return {n: _layer_from(meta, n, get, device, prepare) for n in (names if names is not None else sorted(meta))}
    finally:
        m.close()
