"""Device time of one block-Jacobi config (CUDA events, warm-up, L2 flush) -- A/B helper for the
block kernels' staging variants (BF_BLOCK_TMA, read once per process).

    PYTHONPATH=. BF_BLOCK_TMA=4 python tools/time_block.py [gram|direct] [reps]
"""
import json
import os
import sys

import torch

import paper_1707_05141_b200 as bf

method = sys.argv[1] if len(sys.argv) > 1 else "gram"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
a = bf.gaussian_tensor(1000, 256, 256, 4_000_000, seed_mode="add")
opts = bf.BlockJacobiOptions(method=method, block_width=32, tolerance=1e-11 if method == "gram" else None,
                             accumulate_v=True)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
r = bf.block_svd_tensor(a, opts)
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = bf.block_svd_tensor(a, opts)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(json.dumps({"method": method, "tma": os.environ.get("BF_BLOCK_TMA", "default"), "ms": sorted(ts),
                  "sweeps_mean": float(r["sweeps"].double().mean()), "s0": float(r["sigma"][0, 0])}))
