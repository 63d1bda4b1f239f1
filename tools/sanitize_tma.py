"""Tiny block-Jacobi calls through the tensor-map TMA kernels (bj_gram_tma, bj_rot_tma; odd m
takes the plain-load fallback) for compute-sanitizer (memcheck / racecheck / synccheck):
    compute-sanitizer --tool racecheck python tools/sanitize_tma.py [gram,direct] [max_sweeps]
"""
import sys

import torch

import paper_1707_05141_b200 as bf

methods = sys.argv[1].split(",") if len(sys.argv) > 1 else ["gram", "direct"]
sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
for method in methods:
    for m, n in ((96, 96), (130, 72), (129, 72)):
        a = bf.gaussian_tensor(2, m, n, 77, seed_mode="add")
        r = bf.block_svd_tensor(a, bf.BlockJacobiOptions(method=method, block_width=32, max_sweeps=sweeps,
                                                         accumulate_v=True))
        torch.cuda.synchronize()
        print(method, m, n, float(r["sigma"][0, 0]))
