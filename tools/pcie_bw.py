"""PCIe copy bandwidth on the box (pinned host <-> device, CUDA events): H2D, D2H, and both
directions at once -- the floor under the e2e legs (cfg3 moves 164 MB in and 328 MB out per step).
    python tools/pcie_bw.py
"""
import json

import torch

MB = 1 << 20
dev = torch.device("cuda")
for nbytes in (164 * MB, 328 * MB):
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    h2 = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d2 = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    res = {}
    for name in ("h2d", "d2h", "both"):
        best = 1e9
        for _ in range(5):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            if name in ("h2d", "both"):
                with torch.cuda.stream(s1):
                    d.copy_(h, non_blocking=True)
            if name in ("d2h", "both"):
                with torch.cuda.stream(s2):
                    h2.copy_(d2, non_blocking=True)
            torch.cuda.current_stream().wait_stream(s1)
            torch.cuda.current_stream().wait_stream(s2)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        res[name] = {"ms": best, "GB/s per direction": nbytes / best / 1e6}
    print(json.dumps({"bytes": nbytes, **res}))
