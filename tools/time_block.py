"""Time block Jacobi methods on the cfg4 shape: python tools/time_block.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1707_05141_b200 as bf
from paper_1707_05141_b200.blockjacobi import block_svd_colmajor

for method, tol, B in (("gram", 1e-11, 1000), ("direct", None, 1000), ("direct", None, 200)):
    a = bf.gaussian_tensor(B, 256, 256, 4_000_000, seed_mode="add")
    st = a.transpose(1, 2).contiguous()
    o = bf.BlockJacobiOptions(method=method, block_width=32, tolerance=tol, accumulate_v=True)
    r = block_svd_colmajor(st, 256, 256, o)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = block_svd_colmajor(st, 256, 256, o)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{method:6s} tol={tol} B={B}: {ms:9.2f} ms  {B / ms * 1e3:8.1f} mat/s  sweeps {r['sweeps'].double().mean().item():.2f}"
          f" conv {r['converged'].double().mean().item():.2f}", flush=True)
