"""Time the H^2 compression (truncation + projection phases) over n, for the rank-64 (order 8,
eta 1) and rank-121 (order 11, eta 2) fixtures, full Jacobi vs randomized SVD (§8.3's
Fig. "Compression time"). Prints one JSON line per case."""

import argparse
import json
import time

import torch

from paper_1707_05141_b200 import h2


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ns", default="4096,8192,16384,32768")
    ap.add_argument("--fixtures", default="8:1.0:32,11:2.0:64")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--eps", type=float, default=1e-7)
    ap.add_argument("--kinds", default="full,rsvd")
    ap.add_argument("--oracle-max-n", type=int, default=0, help="also time oracle/h2_ref.compress_ref (CPU) up to this n")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    # one untimed compression of each fixture first: module loading, function attributes and
    # clock ramp otherwise land on the first timed case
    for fx in a.fixtures.split(","):
        order, eta, samples = fx.split(":")
        Hw = h2.build_h2(h2.perturbed_grid(2048, seed=9), 0.1, int(order), float(eta), 64).to("cuda")
        for kind in a.kinds.split(","):
            h2.compress(Hw, a.eps, h2.SvdChoice(kind=kind, samples=int(samples)))
    lines = []
    for fx in a.fixtures.split(","):
        order, eta, samples = fx.split(":")
        order, eta, samples = int(order), float(eta), int(samples)
        for n in [int(x) for x in a.ns.split(",")]:
            t0 = time.perf_counter()
            H = h2.build_h2(h2.perturbed_grid(n, seed=0), 0.1, order, eta, 64)
            tb = time.perf_counter() - t0
            Hd = H.to("cuda")
            cpu_s = None
            if n <= a.oracle_max_n:
                from oracle import h2_ref

                t0 = time.perf_counter()
                h2_ref.compress_ref(H, a.eps)
                cpu_s = time.perf_counter() - t0
            for kind in a.kinds.split(","):
                ch = h2.SvdChoice(kind=kind, samples=samples)
                h2.compress(Hd, a.eps, ch)
                best = None
                for _ in range(a.reps):
                    Hc, rep = h2.compress(Hd, a.eps, ch)
                    tot = rep["truncation_ms"] + rep["projection_ms"]
                    if best is None or tot < best[0]:
                        best = (tot, rep)
                tot, rep = best
                err = h2.estimate_error(Hd, Hc)
                m0, m1 = h2.memory_report(Hd), h2.memory_report(Hc)
                rec = dict(n=n, order=order, eta=eta, svd=kind, samples=samples if kind == "rsvd" else None,
                           build_s=round(tb, 3), truncation_ms=round(rep["truncation_ms"], 3),
                           projection_ms=round(rep["projection_ms"], 3), total_ms=round(tot, 3),
                           ranks_before=rep["ranks_before"], ranks_after=rep["ranks_after"], error=err,
                           lowrank_mb_before=round(m0["lowrank"] / 1e6, 3), lowrank_mb_after=round(m1["lowrank"] / 1e6, 3),
                           dense_mb=round(m0["dense"] / 1e6, 3), oracle_cpu_s=cpu_s if kind == "full" else None,
                           level_svd_ms=[lv["svd_ms"] for lv in rep["levels"]],
                           blocks_lowrank=sum(len(g["t"]) for g in H.coupling.values()),
                           blocks_dense=len(H.dense["t"]), levels=H.tree.num_levels)
                print(json.dumps(rec), flush=True)
                lines.append(rec)
            del Hd
            torch.cuda.empty_cache()
    if a.out:
        with open(a.out, "w") as fh:
            for r in lines:
                fh.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
