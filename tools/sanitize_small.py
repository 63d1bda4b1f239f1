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
from paper_1707_05141_b200 import h2  # noqa: E402

g = h2.bmm(torch.randn(3, 30, 17, device=dev, dtype=torch.float64), torch.randn(3, 17, 64, device=dev, dtype=torch.float64))
g = h2.bmm(torch.randn(3, 64, 64, device=dev, dtype=torch.float64), torch.randn(3, 40, 64, device=dev, dtype=torch.float64), tb=True)
H = h2.build_h2(h2.perturbed_grid(700, seed=1), 0.1, 11, 2.0, 64).to("cuda")
Hc, _ = h2.compress(H, 1e-7)
Hc, _ = h2.compress(H, 1e-7, h2.SvdChoice(kind="rsvd", samples=32))
torch.cuda.synchronize()
print("sanitize workload ok")
