"""Tensor-parallel (N-split / K-split) host logic on CPU: world_size 2, gloo.

The per-rank compute is the CPU oracle (tests may use it); what is under test
is paper_2406_09904_b200.tp: sharding of the reference packing and scales, the
all-reduce MAX of the per-token absmax, the exact int32 all-reduce of K-split
partials, the all-gather of N-split outputs — all must reproduce the unsplit
reference GEMM bit for bit.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import qqq_oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _to_oracle_qw(qw):
    f = lambda t: None if t is None else t.numpy()
    return O.QuantizedWeights(qw.packed.numpy(), qw.rows, qw.cols, qw.scheme, qw.group_size, s_w=f(qw.s_w),
                              s_wg=f(qw.s_wg), s_wc=f(qw.s_wc))


class OracleFused:
    """FusedScales stand-in built by the oracle (gemm.py:61-69)."""

    def __init__(self, fo):
        self.fo = fo
        self.scheme = fo.scheme
        self.s_w_folded = None if fo.s_w_folded is None else torch.from_numpy(fo.s_w_folded)
        self.s_star = None if fo.s_star is None else torch.from_numpy(fo.s_star)
        self.s_wc = None if fo.s_wc is None else torch.from_numpy(fo.s_wc)

    @classmethod
    def from_quantized(cls, qw):
        return cls(O.FusedScales.from_quantized(_to_oracle_qw(qw)))


class CpuOps:
    def quant(self, x):
        from paper_2406_09904_b200.quantize import QuantizedActivations

        a = O.quant_act_per_token(x.numpy().astype(np.float64))
        return QuantizedActivations(torch.from_numpy(a.q), torch.from_numpy(a.s_a))

    def row_absmax(self, x):
        return torch.from_numpy(np.abs(x.numpy().astype(np.float64)).max(axis=1))

    def quant_with_max(self, x, m):  # quantize.py:97-99 with the global row max
        from paper_2406_09904_b200.quantize import QuantizedActivations

        m = m.numpy()
        s = np.where(m > 0.0, m / 127.0, 1.0)
        q = np.clip(np.rint(x.numpy().astype(np.float64) / s[:, None]), -127, 127).astype(np.int8)
        return QuantizedActivations(torch.from_numpy(q), torch.from_numpy(s))

    def _run(self, aq, qw, fused):
        a = O.QuantizedActivations(aq.q.numpy(), aq.s_a.numpy())
        run = O.w4a8_gemm_per_channel if qw.scheme == "per-channel" else O.w4a8_gemm_per_group
        return run(a, _to_oracle_qw(qw), fused.fo, fast=True)

    def gemm(self, aq, qw, fused):
        return torch.from_numpy(self._run(aq, qw, fused).y)

    def gemm_acc(self, aq, qw, fused):
        return torch.from_numpy(self._run(aq, qw, fused).acc)

    def epilogue(self, acc, s_a, s_col):
        return torch.from_numpy(O._epilogue(acc.numpy(), s_a.numpy(), s_col.numpy()))


def _problem(scheme, m=5, k=512, n=256, seed=3):
    from paper_2406_09904_b200.quantize import QuantizedWeights

    x16, w = O.recipe_r1(m, n, k, seed=seed)
    qo = O.quant_weight_per_channel(w) if scheme == "per-channel" else O.quant_weight_per_group(w, 128)
    f = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a))
    qw = QuantizedWeights(f(qo.packed), qo.rows, qo.cols, qo.scheme, qo.group_size, s_w=f(qo.s_w), s_wg=f(qo.s_wg),
                          s_wc=f(qo.s_wc))
    ref = (O.w4a8_gemm_per_channel if scheme == "per-channel" else O.w4a8_gemm_per_group)(
        O.quant_act_per_token(x16.astype(np.float64)), qo, O.FusedScales.from_quantized(qo), fast=True)
    return x16, qw, ref


def _worker(rank, world, port, scheme, mode, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2406_09904_b200 import tp

        x16, qw, ref = _problem(scheme)
        x = torch.from_numpy(x16)
        if mode == "nsplit":
            layer = tp.ColumnParallelW4A8.from_full(qw, ops=CpuOps(), fused_cls=OracleFused)
            y = layer(x, gather=True)
        else:
            layer = tp.RowParallelW4A8.from_full(qw, ops=CpuOps(), fused_cls=OracleFused)
            k0, k1 = layer.k_bounds()
            y = layer(x[:, k0:k1].contiguous())
        ok = np.array_equal(y.numpy().view(np.uint16), ref.y.view(np.uint16))
        results[rank] = bool(ok)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("scheme", ["per-channel", "per-group"])
@pytest.mark.parametrize("mode", ["nsplit", "ksplit"])
def test_tp_world2_bit_exact(scheme, mode):
    world = 2
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), scheme, mode, results), nprocs=world, join=True)
    assert dict(results) == {0: True, 1: True}


def test_shard_shapes():
    from paper_2406_09904_b200 import tp

    _, qw, _ = _problem("per-group")
    s = tp.shard_ksplit(qw, 1, 2)
    assert s.rows == 256 and s.packed.shape == (128, 256) and s.s_wg.shape == (2, 256)
    s = tp.shard_nsplit(qw, 1, 4)
    assert s.cols == 64 and s.s_wc.shape == (64,)
    with pytest.raises(Exception):
        tp.shard_ksplit(qw, 0, 3)
