"""Device time of the batched Gaussian sampler (CUDA events): rsvd's sketch (10 000 x 128 x 40)
and a larger stream (1 000 x 256 x 256), float64 and float32.
    PYTHONPATH=. python tools/time_gauss.py
"""
import json

import torch

import paper_1707_05141_b200 as bf

for B, r, c in ((10000, 128, 40), (1000, 256, 256)):
    for dt in (torch.float64, torch.float32):
        bf.gaussian_tensor(B, r, c, 5, dtype=dt)
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            bf.gaussian_tensor(B, r, c, 5, dtype=dt)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        print(json.dumps({"shape": [B, r, c], "dtype": str(dt), "ms": min(ts)}))
