"""A/B timing of the Gram / direct block path: run with BATCHFACT_B200_LIB pointing at each build."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1707_05141_b200 as bf
from paper_1707_05141_b200.blockjacobi import block_svd_colmajor

tag = os.environ.get("BATCHFACT_B200_LIB", "default") + " tma=" + os.environ.get("BF_BLOCK_TMA", "-")
for method, tol, B in (("gram", 1e-11, 1000), ("direct", None, 500)):
    a = bf.gaussian_tensor(B, 256, 256, 4_000_000, seed_mode="add")
    st = a.transpose(1, 2).contiguous()
    o = bf.BlockJacobiOptions(method=method, block_width=32, tolerance=tol, accumulate_v=True)
    block_svd_colmajor(st, 256, 256, o)
    ts = []
    for _ in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        block_svd_colmajor(st, 256, 256, o)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"{os.path.basename(tag):20s} {method:6s} B={B}: " + " ".join(f"{t:8.2f}" for t in ts) + " ms", flush=True)
