"""Tensor-parallel W4A8 linear layers (BASELINE configs[4]: Llama-2-70B linears
N-split / K-split over 2/4/8 B200s of one node, NCCL over NVLink).

Both splits are bit-identical to the single-GPU reference GEMM:

* Column-parallel (N-split): each rank holds W[:, n0:n1] with its per-channel /
  per-group scales. Activations are replicated and every rank runs the same
  deterministic `quant_act_per_token`; no collective on the GEMM path
  (an all-gather of y only if the consumer needs all N).
* Row-parallel (K-split): each rank holds W[k0:k1, :] (group-aligned for
  per-group) and x[:, k0:k1]. The reference's per-token scale uses the FULL
  row (quantize.py:97-98), so the ranks all-reduce MAX the row absmax, quantize
  their shard with the global scale (same codes as unsplit), compute int32
  partial accumulators (GEMM with no epilogue), all-reduce SUM them (exact,
  order-free), and apply the f64 dequant epilogue (gemm.py:182-184 / 200-202).

The per-rank compute is behind `TPOps`; the default is the sm_100a library.
Tests substitute CPU implementations to check the sharding and collective
logic with the gloo backend on CPU.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import torch
import torch.distributed as dist

from . import _lib
from .errors import ConfigError, ShapeError
from .gemm import FusedScales, prepare, run_gemm
from .quantize import PER_CHANNEL, PER_GROUP, QuantizedActivations, QuantizedWeights, as_cuda, attach_rowsum

__all__ = ["shard_nsplit", "shard_ksplit", "TPOps", "ColumnParallelW4A8", "RowParallelW4A8"]


def _rank_world(group=None):
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


def _bounds(total: int, rank: int, world: int, align: int = 1):
    if total % (world * align) != 0:
        raise ConfigError(f"cannot split {total} evenly over {world} ranks with alignment {align}")
    step = total // world
    return rank * step, (rank + 1) * step


def shard_nsplit(qw: QuantizedWeights, rank: int, world: int) -> QuantizedWeights:
    """Columns [n0, n1) of a K x N quantized weight (reference layout)."""
    n0, n1 = _bounds(qw.cols, rank, world)
    sl = slice(n0, n1)
    return QuantizedWeights(
        packed=qw.packed[:, sl].contiguous(), rows=qw.rows, cols=n1 - n0, scheme=qw.scheme,
        group_size=qw.group_size,
        s_w=None if qw.s_w is None else qw.s_w[sl].contiguous(),
        s_wg=None if qw.s_wg is None else qw.s_wg[:, sl].contiguous(),
        s_wc=None if qw.s_wc is None else qw.s_wc[sl].contiguous())


def shard_ksplit(qw: QuantizedWeights, rank: int, world: int) -> QuantizedWeights:
    """Rows [k0, k1) of a K x N quantized weight. The epilogue scales (s_w or
    s_wc) stay global: they were derived from the full column."""
    align = 2 if qw.scheme == PER_CHANNEL else max(2, qw.group_size)
    if qw.scheme == PER_GROUP and qw.group_size % 2:
        raise ConfigError("K-split needs an even group size (two codes per packed byte)")
    k0, k1 = _bounds(qw.rows, rank, world, align)
    packed = qw.packed[k0 // 2:k1 // 2].contiguous()
    s_wg = None
    if qw.s_wg is not None:
        g = qw.group_size
        s_wg = qw.s_wg[k0 // g:k1 // g].contiguous()
    return QuantizedWeights(packed=packed, rows=k1 - k0, cols=qw.cols, scheme=qw.scheme, group_size=qw.group_size,
                            s_w=qw.s_w, s_wg=s_wg, s_wc=qw.s_wc)


class TPOps:
    """Per-rank compute of the TP layers, on the sm_100a library.

    check=True raises DataError for non-finite activations at once (a host
    sync per call, like the reference); check=False (serving / benchmarking)
    ORs the error bits into the per-device deferred status word instead, so a
    layer's launches and collectives stay asynchronous (and graph-capturable);
    `quantize.raise_if_bad(quantize.deferred_status(dev))` reports them later.
    """

    def __init__(self, check: bool = True):
        self.check = check

    def _status(self, dev):
        from .quantize import deferred_status

        return torch.zeros(1, dtype=torch.int32, device=dev) if self.check else deferred_status(dev)

    def _raise(self, status):
        if self.check:
            from .quantize import raise_if_bad

            raise_if_bad(status, "activations")

    def quant(self, x) -> QuantizedActivations:
        from .quantize import quant_act_per_token

        return quant_act_per_token(x, check=self.check)

    def row_absmax(self, x: torch.Tensor) -> torch.Tensor:
        x = as_cuda(x).contiguous()
        m, k = x.shape
        lib = _lib.lib_for_device(x.device)
        out = torch.empty(m, dtype=torch.float64, device=x.device)
        status = self._status(x.device)
        dt = {torch.float16: 0, torch.float32: 1, torch.float64: 2}[x.dtype]
        _lib.check(lib.qqq_act_absmax(_lib.ptr(x), dt, m, k, k, _lib.ptr(out), _lib.ptr(status),
                                      _lib.stream_of(x.device)), "act_absmax")
        self._raise(status)
        return out

    def quant_with_max(self, x: torch.Tensor, row_max: torch.Tensor) -> QuantizedActivations:
        x = as_cuda(x).contiguous()
        m, k = x.shape
        lib = _lib.lib_for_device(x.device)
        kp = (k + 127) // 128 * 128
        q = torch.empty((m, kp), dtype=torch.int8, device=x.device)
        s_a = torch.empty(m, dtype=torch.float64, device=x.device)
        rowsum = torch.empty(m, dtype=torch.int32, device=x.device)
        status = self._status(x.device)
        dt = {torch.float16: 0, torch.float32: 1, torch.float64: 2}[x.dtype]
        _lib.check(lib.qqq_act_quant_with_max(_lib.ptr(x), dt, m, k, k, _lib.ptr(row_max.contiguous()), _lib.ptr(q),
                                              kp, _lib.ptr(s_a), _lib.ptr(rowsum), _lib.ptr(status),
                                              _lib.stream_of(x.device)), "act_quant_with_max")
        aq = QuantizedActivations(q=q[:, :k], s_a=s_a)
        attach_rowsum(aq, rowsum)
        return aq

    def gemm(self, aq, qw, fused) -> torch.Tensor:
        return run_gemm(aq, prepare(qw, fused), qw.cols, with_acc=False).y

    def gemm_acc(self, aq, qw, fused) -> torch.Tensor:
        """int32 accumulator only (no epilogue): the K-split partial."""
        prep = prepare(qw, fused)
        acc_only = type(prep)(prep.mode, prep.w, prep.sc, prep.group, None)
        return run_gemm(aq, acc_only, qw.cols, with_acc=True).acc

    def epilogue(self, acc: torch.Tensor, s_a: torch.Tensor, s_col: torch.Tensor) -> torch.Tensor:
        m, n = acc.shape
        lib = _lib.lib_for_device(acc.device)
        y = torch.empty((m, n), dtype=torch.float16, device=acc.device)
        _lib.check(lib.qqq_dequant_epilogue(_lib.ptr(acc.contiguous()), m, n, n, _lib.ptr(s_a.contiguous()),
                                            _lib.ptr(as_cuda(s_col, torch.float64).contiguous()), _lib.ptr(y), n,
                                            _lib.stream_of(acc.device)), "dequant_epilogue")
        return y


@dataclass
class ColumnParallelW4A8:
    """y[:, n0:n1] = W4A8(x, W[:, n0:n1]); no collective (optional all-gather)."""

    qw: QuantizedWeights
    fused: FusedScales
    group: Optional[object] = None
    ops: TPOps = None

    @classmethod
    def from_full(cls, qw: QuantizedWeights, group=None, ops: TPOps = None, fused_cls=FusedScales):
        rank, world = _rank_world(group)
        shard = shard_nsplit(qw, rank, world)
        return cls(shard, fused_cls.from_quantized(shard), group, ops or TPOps())

    def __call__(self, x, gather: bool = False):
        aq = self.ops.quant(x)
        if aq.q.shape[1] != self.qw.rows:
            raise ShapeError("activation K does not match the weight")
        y = self.ops.gemm(aq, self.qw, self.fused)
        if not gather:
            return y
        rank, world = _rank_world(self.group)
        if world == 1:
            return y
        parts = [torch.empty_like(y) for _ in range(world)]
        dist.all_gather(parts, y.contiguous(), group=self.group)
        return torch.cat(parts, dim=1)


@dataclass
class RowParallelW4A8:
    """y = W4A8(x, W) with K split over the ranks: all-reduce MAX of the row
    absmax, local int32 partial GEMM, exact all-reduce SUM, f64 epilogue."""

    qw: QuantizedWeights
    fused: FusedScales
    group: Optional[object] = None
    ops: TPOps = None

    @classmethod
    def from_full(cls, qw: QuantizedWeights, group=None, ops: TPOps = None, fused_cls=FusedScales):
        rank, world = _rank_world(group)
        shard = shard_ksplit(qw, rank, world)
        return cls(shard, fused_cls.from_quantized(shard), group, ops or TPOps())

    def k_bounds(self):
        rank, world = _rank_world(self.group)
        return _bounds(self.qw.rows * world, rank, world)

    def __call__(self, x_shard):
        _, world = _rank_world(self.group)
        if world == 1:  # the whole K on this rank: the plain quantizer + GEMM (same codes, acc and y)
            return self.ops.gemm(self.ops.quant(x_shard), self.qw, self.fused)
        m = self.ops.row_absmax(x_shard)
        if world > 1:
            dist.all_reduce(m, op=dist.ReduceOp.MAX, group=self.group)
        aq = self.ops.quant_with_max(x_shard, m)
        acc = self.ops.gemm_acc(aq, self.qw, self.fused)
        if world > 1:
            dist.all_reduce(acc, op=dist.ReduceOp.SUM, group=self.group)
        s_col = self.fused.s_w_folded if self.qw.scheme == PER_CHANNEL else self.fused.s_wc
        return self.ops.epilogue(acc, aq.s_a, s_col)
