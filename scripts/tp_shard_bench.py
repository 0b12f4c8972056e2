"""Per-rank compute of the tensor-parallel Llama-2-70B linears (BASELINE
configs[4]) measured on ONE B200: the shard a rank of a P-way split
runs, without the collective. Column-parallel (N-split, no collective):
quant + GEMM of W[:, N/P]. Row-parallel (K-split): row absmax of x[:, K/P] +
quantize with the (all-reduced) max + int32 partial GEMM + f64 epilogue; the
two all-reduces (M f64 MAX, M*N int32 SUM) are not run here, their bytes are
reported. CUDA-graph timed over rotated cold weight replicas.

    python scripts/tp_shard_bench.py > profiles/r01_tp_shards.jsonl
"""
import json, math, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench as B
import paper_2406_09904_b200 as Q
from paper_2406_09904_b200 import _lib, gemm as G, tp as T

dev = torch.device("cuda", 0)
lib = _lib.load()
st = _lib.stream_of(dev)
LAYERS = [("o_proj", 8192, 8192, "row"), ("gate_up", 8192, 28672, "col"), ("down", 28672, 8192, "row")]
for name, k, n, kind in LAYERS:
    qw, fused, _ = B.make_weights(k, n, "per-group", seed=7, device=dev)
    for P in (1, 2, 4, 8):
        shard = T.shard_nsplit(qw, 0, P) if kind == "col" else T.shard_ksplit(qw, 0, P)
        sk, sn = shard.rows, shard.cols
        fs = Q.FusedScales.from_quantized(shard)
        prep = G.prepare(shard, fs)
        R = max(2, math.ceil(2.5 * B.L2_BYTES / (sk * sn / 2)))
        reps = [prep] + [G.PreparedWeights(prep.mode, prep.w.clone(),
                                           None if prep.sc is None else prep.sc.clone(), prep.group,
                                           prep.s_col.clone()) for _ in range(R - 1)]
        for m in (1, 16, 1024):
            x = torch.randn((m, sk), dtype=torch.float16, device=dev)
            y = torch.empty((m, sn), dtype=torch.float16, device=dev)
            G.workspace(dev, lib.qqq_gemm_workspace_bytes(m, sn, sk))
            kp = (sk + 127) // 128 * 128
            q = torch.empty((m, kp), dtype=torch.int8, device=dev)
            s_a = torch.empty(m, dtype=torch.float64, device=dev)
            rsum = torch.empty(m, dtype=torch.int32, device=dev)
            rmax = torch.empty(m, dtype=torch.float64, device=dev)
            status = torch.zeros(1, dtype=torch.int32, device=dev)
            aq = Q.QuantizedActivations(q=q[:, :sk], s_a=s_a)
            Q.quantize.attach_rowsum(aq, rsum)

            def step(p):
                if kind == "col":
                    lib.qqq_act_quant_ex(_lib.ptr(x), 0, m, sk, sk, _lib.ptr(q), kp, _lib.ptr(s_a), _lib.ptr(rsum),
                                         _lib.ptr(status), st)
                    G.run_gemm(aq, p, sn, False, y_out=y)
                else:
                    lib.qqq_act_absmax(_lib.ptr(x), 0, m, sk, sk, _lib.ptr(rmax), _lib.ptr(status), st)
                    # (all-reduce MAX of rmax here)
                    lib.qqq_act_quant_with_max(_lib.ptr(x), 0, m, sk, sk, _lib.ptr(rmax), _lib.ptr(q), kp,
                                               _lib.ptr(s_a), _lib.ptr(rsum), _lib.ptr(status), st)
                    acc_only = G.PreparedWeights(p.mode, p.w, p.sc, p.group, None)
                    part = G.run_gemm(aq, acc_only, sn, True).acc  # int32 partial
                    # (all-reduce SUM of part here)
                    lib.qqq_dequant_epilogue(_lib.ptr(part), m, sn, sn, _lib.ptr(s_a), _lib.ptr(p.s_col), _lib.ptr(y),
                                             sn, st)
            t = B.graph_time_us([(lambda p: (lambda: step(p)))(p) for p in reps], reps=max(2, 40 // R))
            ops = 2.0 * m * sk * sn
            rec = dict(layer=name, K=k, N=n, split="N" if kind == "col" else "K", P=P, M=m, shard=f"{sk}x{sn}",
                       rank_us=round(t, 2), rank_TOPS=round(ops / t / 1e6, 1),
                       allreduce_bytes=0 if kind == "col" or P == 1 else 4 * m * sn + 8 * m)
            print(json.dumps(rec), flush=True)
