"""cfg1 (1000 x 32x32 + V) device time per ordering / tier: serial (register tier, lane = row) vs
round robin (tiled register tier) vs the shared tier."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1707_05141_b200 as bf  # noqa: E402

a = bf.gaussian_tensor(1000, 32, 32, 1_000_000, seed_mode="add")
for order, tier in (("serial", "auto"), ("round_robin", "auto"), ("serial", "shared"), ("round_robin", "shared")):
    opts = bf.JacobiOptions(ordering=order, accumulate_v=True, tier=tier)
    for _ in range(3):
        bf.svd_tensor(a, opts)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        r = bf.svd_tensor(a, opts, rotations=True)
    e1.record()
    torch.cuda.synchronize()
    print(f"{order:12s} {tier:7s} {e0.elapsed_time(e1) / 10:.3f} ms  sweeps {r['sweeps'].float().mean():.2f}")
