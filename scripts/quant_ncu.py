"""Few plain launches of the act quantizers (for ncu): smoothed (reciprocal
table), smoothed (IEEE division) and plain, M x K given."""
import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_09904_b200 as Q
m, k = int(sys.argv[1]), int(sys.argv[2])
x = torch.randn((m, k), dtype=torch.float16, device="cuda")
sm = torch.ones(k, dtype=torch.float64, device="cuda")
sm[torch.randperm(k, device="cuda")[: k // 8]] = 1.7
rc = Q.smoothing_reciprocal(sm)
for _ in range(3):
    Q.quant_act_smoothed(x, sm, check=False, recip=rc)
    Q.quant_act_smoothed(x, sm, check=False)
    Q.quant_act_per_token(x, check=False)
torch.cuda.synchronize()
