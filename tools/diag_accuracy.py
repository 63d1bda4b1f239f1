"""Accuracy diagnostics: where does the GPU lose V-orthogonality / reconstruction accuracy
relative to the oracle? Prints residual distributions (p50/p99/max) per variant.

    python tools/diag_accuracy.py

TEST/MEASUREMENT INFRASTRUCTURE: imports the oracle as the checker only.
"""

import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import paper_1707_05141_b200 as bf  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from parity_full import orth_res, recon_res, sigma_stats  # noqa: E402


def d3(x):
    x = np.asarray(x)
    return [float(np.percentile(x, 50)), float(np.percentile(x, 99)), float(x.max())]


def np3(t):
    return t.detach().cpu().numpy()


def svd_variants(name, a, threads=16):
    B, m, n = a.shape
    a_np = np3(a)
    a3 = np.ascontiguousarray(a_np.transpose(0, 2, 1))
    o = orc.batch_svd_stacked(a3, m, n, ordering="round_robin", accumulate_v=True, threads=threads)
    u_o, s_o, v_o = o["u"].transpose(0, 2, 1), o["s"], o["v"].transpose(0, 2, 1)
    def nbias(v):  # mean and std of ||v_j||^2 - 1 over all columns: a systematic drift shows as mean != 0
        d = np.sum(np.asarray(v, np.float64) ** 2, axis=1) - 1.0
        return [float(d.mean()), float(d.std())]

    out = {"oracle": {"orth_u": d3(orth_res(u_o)), "orth_v": d3(orth_res(v_o)),
                      "recon": d3(recon_res(a_np, u_o, s_o, v_o)), "vnorm_bias": nbias(v_o),
                      "rotations": float(o["rotations"].mean()), "sweeps": float(o["sweeps"].mean())}}
    for tier in ("auto", "shared"):
        r = bf.svd_tensor(a, bf.JacobiOptions(ordering="round_robin", accumulate_v=True, tier=tier), rotations=True)
        u, s, v = np3(r["u"]), np3(r["sigma"]), np3(r["v"])
        rot = float(np3(r["rotations"]).mean()) if r["rotations"] is not None else -1.0
        nw, _ = sigma_stats(s, s_o)
        out[tier] = {"orth_u": d3(orth_res(u)), "orth_v": d3(orth_res(v)), "recon": d3(recon_res(a_np, u, s, v)),
                     "sigma_normwise": d3(nw), "vnorm_bias": nbias(v), "rotations": rot,
                     "sweeps": float(np3(r["sweeps"]).mean())}
    print(json.dumps({name: out}), flush=True)


def block_partial(name, a, sweeps, threads=16):
    B, m, n = a.shape
    a_np = np3(a)
    a3 = np.ascontiguousarray(a_np.transpose(0, 2, 1))
    out = {}
    for ms in sweeps:
        r = bf.block_svd_tensor(a, bf.BlockJacobiOptions(method="direct", block_width=32, accumulate_v=True,
                                                         max_sweeps=ms))
        o = orc.batch_block_svd_stacked(a3, m, n, block_width=32, method="direct", tol=None, max_sweeps=ms,
                                        accumulate_v=True, threads=threads)
        s, s_o = np3(r["sigma"]), o["s"]
        nw, _ = sigma_stats(s, s_o)
        v, v_o = np3(r["v"]), o["v"].transpose(0, 2, 1)
        u, u_o = np3(r["u"]), o["u"].transpose(0, 2, 1)
        out[ms] = {"sigma_normwise": d3(nw), "orth_v_gpu": d3(orth_res(v)), "orth_v_oracle": d3(orth_res(v_o)),
                   "recon_gpu": d3(recon_res(a_np, u, s, v)), "recon_oracle": d3(recon_res(a_np, u_o, s_o, v_o))}
    print(json.dumps({name: out}), flush=True)


def main():
    orc.build()
    if len(sys.argv) > 1 and sys.argv[1] == "quick":
        p = bf.gaussian_tensor(500, 256, 64, 4_000_000, seed_mode="add")
        _, r = bf.qr_tensor(p)
        svd_variants("R64_upper", r.contiguous())
        svd_variants("gauss32", bf.gaussian_tensor(500, 32, 32, 1_000_000, seed_mode="add"))
        block_partial("cfg4d_40", bf.gaussian_tensor(40, 256, 256, 4_000_000, seed_mode="add"), [30])
        return
    torch.manual_seed(0)
    a = bf.gaussian_tensor(500, 64, 64, 3_000_000, seed_mode="add")
    svd_variants("gauss64", a)
    # upper-triangular R of 256 x 64 Gaussian pairs: the direct method's inner SVD input
    p = bf.gaussian_tensor(500, 256, 64, 4_000_000, seed_mode="add")
    _, r = bf.qr_tensor(p)
    svd_variants("R64_upper", r.contiguous())
    a40 = bf.gaussian_tensor(500, 40, 40, 5_000_000, seed_mode="add")
    svd_variants("gauss40", a40)
    a4 = bf.gaussian_tensor(40, 256, 256, 4_000_000, seed_mode="add")
    block_partial("cfg4d_40", a4, [1, 2, 30])


if __name__ == "__main__":
    main()
