"""Small invocations of every kernel family for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1707_05141_b200 as bf  # noqa: E402

dev = torch.device("cuda", 0)
for (m, n, order) in [(64, 64, "round_robin"), (40, 40, "round_robin"), (32, 32, "serial"), (33, 17, "round_robin"),
                      (48, 20, "serial")]:
    a = bf.gaussian_tensor(6, m, n, 123 + m, seed_mode="add")
    r = bf.svd_tensor(a, bf.JacobiOptions(ordering=order, accumulate_v=True))
    r2 = bf.svd_tensor(a, bf.JacobiOptions(ordering=order, accumulate_v=True, tier="shared"))
q, rr = bf.qr_tensor(bf.gaussian_tensor(6, 64, 32, 7, seed_mode="add"))
q, rr = bf.qr_tensor(bf.gaussian_tensor(6, 128, 40, 8, seed_mode="add"))
b = bf.block_svd_tensor(bf.gaussian_tensor(3, 128, 128, 9, seed_mode="add"),
                        bf.BlockJacobiOptions(method="gram", block_width=32, tolerance=1e-11, accumulate_v=True))
b = bf.block_svd_tensor(bf.gaussian_tensor(2, 96, 64, 10, seed_mode="add"),
                        bf.BlockJacobiOptions(method="direct", block_width=16, accumulate_v=True))
m5, _ = bf.make_matrix_tensor(4, 128, 128, 1e16, rank=64, seed=5)
t = bf.rsvd_tensor(m5, bf.RsvdOptions(k=32, p=8, seed=5))
b = bf.block_svd_tensor(bf.gaussian_tensor(2, 128, 128, 11, seed_mode="add"),
                        bf.BlockJacobiOptions(method="direct", block_width=32, accumulate_v=True))
r3 = bf.svd_tensor(bf.gaussian_tensor(2, 128, 122, 12, seed_mode="add"),
                   bf.JacobiOptions(ordering="round_robin", accumulate_v=True))  # CTA tier, V in global
# round 2: the fixed-column V replay (64 wide, also inside the direct block method), the float32
# Gaussian stream and f32 rsvd with a device sketch, the wide-pair block pipeline (2k > 64) with
# work counters, the helper re-exports, devices= sharding
QUICK = bool(os.environ.get("BF_SANITIZE_QUICK"))  # racecheck: small batches, no H^2
r64 = bf.svd_tensor(bf.gaussian_tensor(8 if QUICK else 700, 64, 64, 13, seed_mode="add"), bf.JacobiOptions(ordering="round_robin",
                                                                                           accumulate_v=True))
g32 = bf.gaussian_tensor(5, 130, 41, 14, dtype=torch.float32)
t32 = bf.rsvd_tensor(bf.gaussian_tensor(4, 64, 48, 15).float(), bf.RsvdOptions(k=8, p=4, seed=3))
for meth in ("gram", "direct"):
    bw = bf.block_svd_tensor(bf.gaussian_tensor(2, 130, 100, 16, seed_mode="add"),
                             bf.BlockJacobiOptions(method=meth, block_width=48, accumulate_v=True), stats=True)
x = np.random.default_rng(0).standard_normal((20, 9))
bf.householder_vector(x[:, 0]), bf.jacobi_rotation(2.0, 0.5, 1.0), bf.off_orthogonality(x), bf.syrk(x)
bf.gemm(x, x.T, np.ones((20, 20)), alpha=2.0, beta=0.5), bf.frobenius(x)
from paper_1707_05141_b200.blockjacobi import scaled_offdiag  # noqa: E402

scaled_offdiag(x.T @ x)
bf.batch_svd([x, x[:, :5], x], devices=["cuda:0", "cuda:0"])
if QUICK:
    torch.cuda.synchronize()
    print("sanitize workload ok (quick)")
    sys.exit(0)
from paper_1707_05141_b200 import h2  # noqa: E402

g = h2.bmm(torch.randn(3, 30, 17, device=dev, dtype=torch.float64), torch.randn(3, 17, 64, device=dev, dtype=torch.float64))
g = h2.bmm(torch.randn(3, 64, 64, device=dev, dtype=torch.float64), torch.randn(3, 40, 64, device=dev, dtype=torch.float64), tb=True)
H = h2.build_h2(h2.perturbed_grid(700, seed=1), 0.1, 11, 2.0, 64).to("cuda")
Hc, _ = h2.compress(H, 1e-7)
Hc, _ = h2.compress(H, 1e-7, h2.SvdChoice(kind="rsvd", samples=32))
torch.cuda.synchronize()
print("sanitize workload ok")
