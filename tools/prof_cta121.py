import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1707_05141_b200 as bf
a = bf.gaussian_tensor(32, 121, 121, 77, seed_mode="add")
for _ in range(2):
    r = bf.svd_tensor(a, bf.JacobiOptions(ordering="round_robin", accumulate_v=False))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
r = bf.svd_tensor(a, bf.JacobiOptions(ordering="round_robin", accumulate_v=False))
e1.record()
torch.cuda.synchronize()
print("121x121 B=32 W-only:", e0.elapsed_time(e1), "ms sweeps", r["sweeps"].double().mean().item())
