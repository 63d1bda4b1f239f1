"""The paper's single published throughput point (batched SVD of 1000 matrices of
512 x 512, 'exceeding 800/400 GFLOP/s' single/double on P100): time our block-Jacobi tier on it.
GFLOP/s here uses the LAPACK-style nominal SVD count 22 n^3 (U, S, V), not the paper's (unstated)
convention."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1707_05141_b200 as bf
from paper_1707_05141_b200.blockjacobi import block_svd_colmajor

B, n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000, 512
a = bf.gaussian_tensor(B, n, n, 9_000_000, seed_mode="add")
st = a.transpose(1, 2).contiguous()
for method, tol in (("gram", 1e-11),):
    o = bf.BlockJacobiOptions(method=method, block_width=32, tolerance=tol, accumulate_v=True)
    r = block_svd_colmajor(st, n, n, o)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = block_svd_colmajor(st, n, n, o)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    gf = B * 22.0 * n ** 3 / (ms * 1e-3) / 1e9
    print(f"512x512 {method} B={B}: {ms:.1f} ms, {B / ms * 1e3:.1f} mat/s, {gf:.0f} GFLOP/s (22 n^3), "
          f"sweeps {r['sweeps'].double().mean().item():.2f}, converged {r['converged'].double().mean().item():.3f}")
