"""Run one hot-path call of a bench config (for ncu captures): python tools/prof_run.py cfg3 [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
gc = bench.GpuConfig(name, bench.CONFIGS[name], torch.device("cuda", 0), 0)
for _ in range(reps):
    gc.step()
torch.cuda.synchronize()
print("done", name)
