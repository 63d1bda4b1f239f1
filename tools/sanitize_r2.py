"""Tiny invocations of the round-2 kernels for compute-sanitizer racecheck (the full
sanitize_small.py workload exceeds racecheck's time budget): the fixed-column V replay, the
float32 Gaussian stream, the wide-pair block pipeline (2 sweeps), the helper kernels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1707_05141_b200 as bf  # noqa: E402

r64 = bf.svd_tensor(bf.gaussian_tensor(3, 64, 64, 13, seed_mode="add"),
                    bf.JacobiOptions(ordering="round_robin", accumulate_v=True, max_sweeps=3))
g32 = bf.gaussian_tensor(3, 40, 41, 14, dtype=torch.float32)
for meth in ("gram", "direct"):
    bf.block_svd_tensor(bf.gaussian_tensor(1, 100, 100, 16, seed_mode="add"),
                        bf.BlockJacobiOptions(method=meth, block_width=48, accumulate_v=True, max_sweeps=2), stats=True)
x = np.random.default_rng(0).standard_normal((20, 9))
bf.householder_vector(x[:, 0]), bf.off_orthogonality(x), bf.syrk(x), bf.frobenius(x)
torch.cuda.synchronize()
print("sanitize r2 workload ok")
