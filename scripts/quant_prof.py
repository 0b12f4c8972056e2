"""A few smoothed / plain quantizer launches at one (M, K) for ncu (developer tool)."""
import os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2406_09904_b200 as Q
m, k = int(sys.argv[1]), int(sys.argv[2])
dev = torch.device("cuda", 0)
x = torch.randn((m, k), dtype=torch.float16, device=dev)
s = torch.ones(k, dtype=torch.float64, device=dev)
s[torch.randperm(k, device=dev)[: k // 8]] = 1.7
for _ in range(3):
    Q.quant_act_smoothed(x, s, check=False)
    Q.quant_act_per_token(x, check=False)
torch.cuda.synchronize()
