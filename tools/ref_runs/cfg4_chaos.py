"""cfg4 (block Jacobi, Gram, tol 1e-11) convergence chaos: the REFERENCE itself (Python + numpy/
OpenBLAS, /root/reference) against the C oracle on the same entries. Entries whose e_history
hovers at tol decide their converged sweep by rounding; this measures how often the reference and
its own faithful restatement disagree there, the yardstick for GPU-vs-oracle flag/sweep outliers.

Runs in the build container only (needs /root/reference):
    python tools/ref_runs/cfg4_chaos.py profiles/parity_r02.json > profiles/cfg4_chaos_r02.json
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


def ref_entry(i):
    sys.path.insert(0, REF)
    import importlib

    rsvd = importlib.import_module("batchfact.rsvd")
    bj = importlib.import_module("batchfact.blockjacobi")
    a = rsvd.gaussian_matrix(256, 256, 4_000_000 + i)
    r = bj.block_svd(a, bj.BlockJacobiOptions(method="gram", block_width=32, tolerance=1e-11, accumulate_v=True))
    return i, int(r.sweeps), bool(r.converged), [float(e) for e in r.e_history]


def main():
    from oracle import oracle as orc

    par = json.load(open(sys.argv[1]))
    outl = [o["index"] for o in par["configs"]["cfg4"]["flag_or_sweep_outliers"]]
    rng = np.random.default_rng(0)
    others = sorted(set(rng.choice(1000, 60, replace=False).tolist()) - set(outl))[:40]
    idx = sorted(set(outl) | set(others))
    with mp.get_context("spawn").Pool(len(os.sched_getaffinity(0))) as pool:
        ref = pool.map(ref_entry, idx)
    out = []
    for i, sw, cv, eh in ref:
        a = orc.gaussian_matrix(256, 256, 4_000_000 + i)
        o = orc.batch_block_svd_stacked(np.ascontiguousarray(a.T)[None], 256, 256, block_width=32, method="gram",
                                        tol=1e-11, accumulate_v=True)
        out.append({"index": i, "gpu_oracle_outlier": i in outl, "ref_sweeps": sw, "ref_conv": cv,
                    "oracle_sweeps": int(o["sweeps"][0]), "oracle_conv": bool(o["converged"][0]),
                    "ref_e_over_tol_last5": [e / 1e-11 for e in eh[-5:]]})
    dis = [r for r in out if abs(r["ref_sweeps"] - r["oracle_sweeps"]) > 1 or r["ref_conv"] != r["oracle_conv"]]
    summ = {
        "what": "reference (Python/numpy) vs C oracle, cfg4 Gram tol 1e-11: converged/sweeps agreement",
        "entries": len(out),
        "gpu_oracle_outliers_checked": sum(r["gpu_oracle_outlier"] for r in out),
        "ref_vs_oracle_disagree_on_gpu_outliers": sum(1 for r in dis if r["gpu_oracle_outlier"]),
        "ref_vs_oracle_disagree_on_others": sum(1 for r in dis if not r["gpu_oracle_outlier"]),
        "entries_detail": out,
    }
    print(json.dumps(summ, indent=1))


if __name__ == "__main__":
    main()
