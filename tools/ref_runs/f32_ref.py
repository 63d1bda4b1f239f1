"""float32 twins of the BASELINE configs: the REFERENCE itself (Python + numpy, /root/reference) on
the same inputs as tools/parity_full.py's cfg*f32, next to the C oracle. Records, per entry, the
reference's sweeps / converged flag and its residuals (||U^T U - I||_F, ||V^T V - I||_F,
||A - U S V^T||_F / ||A||_F), so the GPU's float32 residuals can be gated against the reference's
own, not only against its restatement; and the reference-vs-oracle spread (sigma normwise,
sweeps), the rounding noise floor of the float32 comparison.

Runs in the build container only (needs /root/reference); writes the small fixture the GPU-side
parity tool reads and a summary:
    python tools/ref_runs/f32_ref.py tests/golden/ref_f32_stats.npz > profiles/f32_ref_r02.json
"""

import json
import multiprocessing as mp
import os
import sys

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import numpy as np  # noqa: E402

REF = "/root/reference/pkg/src"
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

# name: (kind, m, n, seed base, ordering / method, entries)
RUNS = {
    "cfg1f32": ("svd", 32, 32, 1_000_000, "serial", range(1000)),
    "cfg1rrf32": ("svd", 32, 32, 1_000_000, "round_robin", range(1000)),
    "cfg3f32": ("svd", 64, 64, 3_000_000, "round_robin", range(5000)),
    "cfg4df32": ("block", 256, 256, 4_000_000, "direct", range(64)),
}


def _res(a, u, s, v):
    a, u, s, v = (np.asarray(x, np.float64) for x in (a, u, s, v))
    ou = np.linalg.norm(u.T @ u - np.eye(u.shape[1]))
    ov = np.linalg.norm(v.T @ v - np.eye(v.shape[1]))
    rc = np.linalg.norm(a - (u * s) @ v.T) / max(np.linalg.norm(a), 1e-300)
    return ou, ov, rc


def ref_entry(args):
    name, i = args
    sys.path.insert(0, REF)
    import importlib

    rsvd = importlib.import_module("batchfact.rsvd")
    kind, m, n, seed, how, _ = RUNS[name]
    a = rsvd.gaussian_matrix(m, n, seed + i, np.float32)
    if kind == "svd":
        jac = importlib.import_module("batchfact.jacobi")
        r = jac.svd(a, jac.JacobiOptions(ordering=how, accumulate_v=True))
    else:
        bj = importlib.import_module("batchfact.blockjacobi")
        r = bj.block_svd(a, bj.BlockJacobiOptions(method=how, block_width=32, accumulate_v=True))
    return (name, i, int(r.sweeps), bool(r.converged), *_res(a, r.u, r.sigma, r.v), np.asarray(r.sigma, np.float32))


def main():
    from oracle import oracle as orc

    orc.build()
    jobs = [(name, i) for name, run in RUNS.items() for i in run[5]]
    with mp.get_context("spawn").Pool(len(os.sched_getaffinity(0))) as pool:
        res = pool.map(ref_entry, jobs, chunksize=8)
    fixture, summary = {}, {"what": "reference (Python/numpy) float32 vs the C oracle on the cfg*f32 inputs", "configs": {}}
    for name, (kind, m, n, seed, how, idx) in RUNS.items():
        rows = [r for r in res if r[0] == name]
        idx = np.array([r[1] for r in rows])
        sw = np.array([r[2] for r in rows], np.int32)
        cv = np.array([r[3] for r in rows], bool)
        ou, ov, rc = (np.array([r[k] for r in rows]) for k in (4, 5, 6))
        sig = np.stack([r[7] for r in rows])
        a3 = np.stack([np.ascontiguousarray(orc.gaussian_matrix(m, n, seed + i, np.float32).T) for i in idx])
        if kind == "svd":
            o = orc.batch_svd_stacked(a3, m, n, ordering=how, accumulate_v=True, threads=8)
        else:
            o = orc.batch_block_svd_stacked(a3, m, n, block_width=32, method=how, accumulate_v=True, threads=8)
        s_o = o["s"].astype(np.float64)
        nw = np.max(np.abs(sig - s_o) / np.maximum(s_o[:, :1], 1e-300), axis=1)
        a_np = a3.transpose(0, 2, 1).astype(np.float64)
        lap = np.linalg.svd(a_np, compute_uv=False)
        ref_lap = np.max(np.abs(sig - lap) / lap[:, :1], axis=1)
        orc_lap = np.max(np.abs(s_o - lap) / lap[:, :1], axis=1)
        dsw = sw - o["sweeps"]
        fixture.update({f"{name}/index": idx, f"{name}/sweeps": sw, f"{name}/converged": cv,
                        f"{name}/orth_u": ou, f"{name}/orth_v": ov, f"{name}/recon": rc})
        if kind == "block":
            fixture[f"{name}/sigma"] = sig
        summary["configs"][name] = {
            "entries": int(len(idx)),
            "ref_max": {"orth_u": float(ou.max()), "orth_v": float(ov.max()), "recon": float(rc.max())},
            "ref_p50": {"orth_u": float(np.median(ou)), "orth_v": float(np.median(ov)), "recon": float(np.median(rc))},
            "ref_vs_oracle_sigma_normwise_max": float(nw.max()),
            "ref_vs_oracle_sigma_normwise_p50": float(np.median(nw)),
            "ref_vs_lapack_sigma_normwise_p50": float(np.median(ref_lap)),
            "oracle_vs_lapack_sigma_normwise_p50": float(np.median(orc_lap)),
            "ref_vs_oracle_sweeps_hist": {str(k): int(v) for k, v in zip(*np.unique(dsw, return_counts=True))},
            "ref_vs_oracle_converged_equal": int(np.sum(cv == o["converged"])),
        }
    np.savez_compressed(sys.argv[1], **fixture)
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main()
