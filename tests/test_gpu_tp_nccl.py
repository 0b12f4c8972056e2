"""Tensor parallelism on real GPUs: world_size 2, NCCL, one process per GPU.

ColumnParallelW4A8 (N-split, all-gather) and RowParallelW4A8 (K-split:
all-reduce MAX of the row absmax, int32 partial GEMM, exact all-reduce SUM,
f64 epilogue) on the sm_100a library (TPOps), checked bit-exactly against the
unsplit single-GPU GEMM on rank 0 for both schemes and decode / prefill M.
Needs two visible GPUs; skipped otherwise (the gloo world-2 test covers the
host logic on CPU, tests/test_gpu_config_parity.py the per-rank shards on one
GPU).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, result):
    import torch.distributed as dist

    import paper_2406_09904_b200 as Q
    from paper_2406_09904_b200 import tp

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world)
    ok = True
    try:
        ops = tp.TPOps()
        for scheme in ("per-channel", "per-group"):
            for (k, n, m) in ((4096, 2048, 1), (4096, 2048, 16), (2048, 1024, 300)):
                rng = np.random.default_rng(k + n + m + (scheme == "per-group"))
                w = rng.standard_normal((k, n))
                x = torch.from_numpy(rng.standard_normal((m, k)).astype(np.float16)).cuda()
                qw = Q.quant_weight_per_channel(w) if scheme == "per-channel" else \
                    Q.quant_weight_per_group(w, Q.QuantSpec("per-group", 128))
                fused = Q.FusedScales.from_quantized(qw)
                run = Q.w4a8_gemm_per_channel if scheme == "per-channel" else Q.w4a8_gemm_per_group
                ref = run(Q.quant_act_per_token(x), qw, fused, with_acc=False).y
                sh = tp.shard_nsplit(qw, rank, world)
                col = tp.ColumnParallelW4A8(sh, Q.FusedScales.from_quantized(sh), None, ops)
                y = col(x, gather=True)
                ok &= bool(torch.equal(y.view(torch.int16), ref.view(torch.int16)))
                sk = tp.shard_ksplit(qw, rank, world)
                row = tp.RowParallelW4A8(sk, Q.FusedScales.from_quantized(sk), None, ops)
                k0, k1 = row.k_bounds()
                yr = row(x[:, k0:k1].contiguous())
                ok &= bool(torch.equal(yr.view(torch.int16), ref.view(torch.int16)))
        flag = torch.tensor([1 if ok else 0], device="cuda")
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if rank == 0:
            result["ok"] = bool(flag.item())
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_tp_world2_nccl_bit_exact():
    world = 2
    mgr = mp.Manager()
    result = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), result), nprocs=world, join=True)
    assert result.get("ok") is True
