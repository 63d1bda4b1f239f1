"""Per-level SVD timing/sweeps inside the H^2 truncation (diagnostic)."""
import sys, time, json
import torch
from paper_1707_05141_b200 import h2, JacobiOptions, svd_tensor, BlockJacobiOptions, block_svd_tensor

def timed(f, reps=3):
    f(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps): r = f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e3, r

for n, order, eta in ((8192, 8, 1.0), (16384, 8, 1.0), (8192, 11, 2.0)):
    H = h2.build_h2(h2.perturbed_grid(n, seed=0), 0.1, order, eta, 64).to("cuda")
    st = h2._level_struct(H)
    L = H.tree.num_levels
    # leaf-level-like inputs: the leaf U at each level and an inner TE with original T = I
    for l in range(L):
        if H.leaf_U[l] is None: continue
        k = H.ranks[l]
        M = max(H.leaf_rows, k)
        A = torch.zeros(H.leaf_U[l].shape[0], M, k, dtype=torch.float64, device="cuda")
        A[:, :H.leaf_rows] = H.leaf_U[l]
        ms, r = timed(lambda: svd_tensor(A, JacobiOptions(ordering="round_robin", accumulate_v=True)))
        rec = dict(n=n, order=order, level=l, batch=A.shape[0], shape=list(A.shape[1:]), svd_ms=round(ms, 3),
                   sweeps_max=int(r["sweeps"].max()), conv=bool(r["converged"].all()))
        if k > 64:
            kp = (k + 31) // 32 * 32
            Mp = max(M, kp)
            Ap = torch.zeros(A.shape[0], Mp, kp, dtype=torch.float64, device="cuda")
            Ap[:, :M, :k] = A
            ms2, r2 = timed(lambda: block_svd_tensor(Ap, BlockJacobiOptions(block_width=32, method="direct", accumulate_v=True)))
            rec.update(block_ms=round(ms2, 3), block_sweeps=int(r2["sweeps"].max()),
                       sig_diff=float((r2["sigma"][:, :k] - r["sigma"]).abs().max() / r["sigma"][:, 0].max()))
        print(json.dumps(rec), flush=True)
