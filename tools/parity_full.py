"""Full-config parity: EVERY entry of every BASELINE config through the CUDA path (C ABI) and
the CPU oracle (oracle/: the reference algorithm restated in C, pinned to the reference's own
outputs by tests/golden) on the same inputs.

    python tools/parity_full.py [--configs cfg1,cfg1rr,cfg2,cfg3,cfg4,cfg4d,cfg5] [--out profiles/parity_r02.json]
    python tools/parity_full.py --configs cfg1f32,cfg1rrf32,cfg2f32,cfg3f32,cfg4df32,cfg5f32 \
        --out profiles/parity_f32_r02.json     # float32 twins (gates: see check())

Per config it records (and `check()` gates, SURVEY.md §8c / north_star):
  * sigma: normwise max|ds_i|/s_1 per matrix <= 1e-12 (f64) -- the hard gate; per-value relative
    |ds_i|/s_i as p50/p99/max, next to the oracle-vs-LAPACK floor (numpy.linalg.svd) on the same
    matrices (the floor the per-value figure can be judged against);
  * U, V: equal to the oracle's up to column sign, |du| <= 256 eps s_1/gap_j per column
    (Davis-Kahan scaled; columns with a degenerate gap are excluded);
  * converged flags equal; sweeps within +-1 (same ordering);
  * residuals: max over the batch of ||U^T U - I||_F, ||V^T V - I||_F, ||A - U S V^T||_F/||A||_F for
    the GPU next to the oracle's own maxima on the same batch -- the GPU must not exceed them
    ("residuals no worse than the reference's");
  * QR: elementwise |Q - Q_o|, |R - R_o| vs eps ||A||, ||Q^T Q - I||_F and ||A - QR||_F/||A||_F.

TEST/MEASUREMENT INFRASTRUCTURE: imports the oracle as the checker only.
"""

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

EPS64 = float(np.finfo(np.float64).eps)

# the BASELINE configs (bench.py CONFIGS, same input streams: seed_i = config*1e6 + i)
CONFIGS = {
    "cfg1": dict(kind="svd", m=32, n=32, batch=1000, seed=1_000_000, ordering="serial"),
    "cfg1rr": dict(kind="svd", m=32, n=32, batch=1000, seed=1_000_000, ordering="round_robin"),
    "cfg2": dict(kind="qr", m=64, n=32, batch=10_000, seed=2_000_000),
    "cfg3": dict(kind="svd", m=64, n=64, batch=5000, seed=3_000_000, ordering="round_robin"),
    "cfg4": dict(kind="block", method="gram", tol=1e-11, m=256, n=256, batch=1000, seed=4_000_000),
    "cfg4d": dict(kind="block", method="direct", tol=1e-13, m=256, n=256, batch=1000, seed=4_000_000),
    "cfg5": dict(kind="rsvd", m=128, n=128, batch=10_000, seed=5_000_000, k=32, p=8, rsvd_seed=5),
}
# float32 twins (north_star: "fp64/fp32 matrices"; sigma gate 1e-5 normwise): the same shapes, inputs
# drawn from numpy's float32 stream (rsvd: the f64 test matrices rounded), default f32 tolerances
for _k in ("cfg1", "cfg1rr", "cfg2", "cfg3", "cfg4d", "cfg5"):
    CONFIGS[_k + "f32"] = dict(CONFIGS[_k], dtype="f32")
CONFIGS["cfg4df32"]["tol"] = None  # blockjacobi.py:19-22 default, 1e-5 for float32


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:  # noqa: BLE001
        return os.cpu_count() or 1


# ------------------------------------------------------------------ batched comparison rules


def sigma_stats(s, s_ref):
    """Per-matrix normwise max|ds|/s1 and the flat per-value relative differences."""
    s = np.asarray(s, np.float64)
    s_ref = np.asarray(s_ref, np.float64)
    s1 = np.maximum(np.abs(s_ref[:, :1]), np.finfo(np.float64).tiny)
    normwise = np.max(np.abs(s - s_ref) / s1, axis=1)
    pos = s_ref > 0
    per_value = np.abs(s - s_ref)[pos] / s_ref[pos]
    return normwise, per_value


def dist(x):
    x = np.asarray(x, np.float64)
    if x.size == 0:
        return {"p50": 0.0, "p99": 0.0, "max": 0.0}
    return {"p50": float(np.percentile(x, 50)), "p99": float(np.percentile(x, 99)), "max": float(np.max(x))}


def vec_mismatch_batch(x, x_ref, s_ref, factor=256.0, ncols=None, eps=EPS64):
    """x, x_ref: (B, rows, n) column vectors; s_ref (B, n) descending. Worst err/tol per matrix
    (<= 1 passes): columns compared up to sign, tol = factor eps s1/gap_j (Davis-Kahan)."""
    x = np.asarray(x, np.float64)
    x_ref = np.asarray(x_ref, np.float64)
    s = np.asarray(s_ref, np.float64)
    B, _, n = x.shape
    nc = n if ncols is None else ncols
    s1 = np.maximum(s[:, :1], np.finfo(np.float64).tiny)
    gap = np.full((B, n), np.inf)
    if n > 1:
        d = np.abs(np.diff(s, axis=1))  # sorted: nearest neighbours give the gap
        gap[:, 1:] = np.minimum(gap[:, 1:], d)
        gap[:, :-1] = np.minimum(gap[:, :-1], d)
    else:
        gap[:] = s1
    ok = (s > s1 * 1e3 * eps) & (gap > s1 * 1e3 * eps)
    ok[:, nc:] = False
    sign = np.where(np.einsum("brn,brn->bn", x, x_ref) >= 0, 1.0, -1.0)
    err = np.max(np.abs(x * sign[:, None, :] - x_ref), axis=1)
    tol = factor * eps * s1 / np.where(np.isfinite(gap), gap, s1)
    ratio = np.where(ok, err / tol, 0.0)
    return np.max(ratio, axis=1) if n else np.zeros(B)


def orth_res(q):
    """||Q^T Q - I||_F per matrix; q (B, rows, n)."""
    q = np.asarray(q, np.float64)
    g = np.matmul(q.transpose(0, 2, 1), q)
    g -= np.eye(q.shape[2])[None]
    return np.sqrt(np.sum(g * g, axis=(1, 2)))


def res_pair(g, o, exclude=None):
    """GPU vs oracle residual distribution (max is the gate, p50/p99 show the typical case).
    exclude: entries left out of the gated GPU max (rounding-chaotic Gram entries, see check())."""
    g, o = np.asarray(g, np.float64), np.asarray(o, np.float64)
    keep = np.ones(g.shape[0], bool)
    if exclude is not None and len(exclude):
        keep[np.asarray(exclude)] = False
    return {"gpu_max": float(g[keep].max()), "oracle_max": float(o.max()),
            "gpu_max_all": float(g.max()), "gpu_argmax_all": int(np.argmax(g)), "oracle_argmax": int(np.argmax(o)),
            "gpu_p50": float(np.percentile(g, 50)), "oracle_p50": float(np.percentile(o, 50)),
            "gpu_p99": float(np.percentile(g, 99)), "oracle_p99": float(np.percentile(o, 99))}


def recon_res(a, u, s, v):
    a = np.asarray(a, np.float64)
    r = np.matmul(np.asarray(u, np.float64) * np.asarray(s, np.float64)[:, None, :],
                  np.asarray(v, np.float64).transpose(0, 2, 1))
    na = np.sqrt(np.sum(a * a, axis=(1, 2)))
    d = a - r
    return np.sqrt(np.sum(d * d, axis=(1, 2))) / np.where(na > 0, na, 1.0)


def exact_normwise(a, s, chunk=2000):
    """Per-matrix max|s_i - s_exact_i| / s_exact_1, s_exact = LAPACK (numpy gesdd) in float64 on
    the same input (for float32 twins: how far each implementation is from the exact values)."""
    out = []
    for i in range(0, a.shape[0], chunk):
        sl = np.linalg.svd(np.asarray(a[i:i + chunk], np.float64), compute_uv=False)
        ss = np.asarray(s[i:i + chunk, : sl.shape[1]], np.float64)
        out.append(np.max(np.abs(ss - sl), axis=1) / np.maximum(sl[:, 0], 1e-300))
    return np.concatenate(out) if out else np.zeros(0)


def ref_fixture(name):
    """The reference's own per-entry float32 results on the same inputs (tools/ref_runs/f32_ref.py,
    run where /root/reference exists; committed as tests/golden/ref_f32_stats.npz)."""
    path = os.path.join(ROOT, "tests", "golden", "ref_f32_stats.npz")
    if not os.path.exists(path):
        return None
    z = np.load(path)
    if f"{name}/index" not in z:
        return None
    return {k.split("/", 1)[1]: z[k] for k in z.files if k.startswith(name + "/")}


def lapack_floor(a, s_ref, chunk=2000):
    """Per-value relative difference of the oracle's sigma from LAPACK's (numpy gesdd)."""
    out = []
    for i in range(0, a.shape[0], chunk):
        sl = np.linalg.svd(a[i:i + chunk], compute_uv=False)
        ref = s_ref[i:i + chunk, : sl.shape[1]]
        pos = sl > 0
        out.append((np.abs(ref - sl)[pos] / sl[pos]))
    return np.concatenate(out) if out else np.zeros(0)


# ------------------------------------------------------------------ per-config runs


def _inputs(name, c, dev):
    import paper_1707_05141_b200 as bf

    import torch

    f32 = c.get("dtype") == "f32"
    if c["kind"] == "rsvd":
        a, _ = bf.make_matrix_tensor(c["batch"], c["m"], c["n"], 1e16, rank=64, seed=c["seed"], device=dev)
        if f32:
            a = a.transpose(1, 2).float().contiguous().transpose(1, 2)
    else:
        a = bf.gaussian_tensor(c["batch"], c["m"], c["n"], c["seed"], seed_mode="add",
                               dtype=torch.float32 if f32 else torch.float64, device=dev)
    return a  # (B, m, n) view of column-major storage


def _np(t):
    return t.detach().cpu().numpy()


def run_config(name, threads, dev="cuda"):
    import torch

    import paper_1707_05141_b200 as bf
    from oracle import oracle as orc

    c = CONFIGS[name]
    m, n, B = c["m"], c["n"], c["batch"]
    a = _inputs(name, c, dev)
    a_np = _np(a)  # (B, m, n)
    a3 = np.ascontiguousarray(a_np.transpose(0, 2, 1))  # per-matrix column-major for the oracle
    f32 = c.get("dtype") == "f32"
    eps = float(np.finfo(np.float32 if f32 else np.float64).eps)
    rec = {"config": name, "batch": B, "m": m, "n": n, "dtype": "f32" if f32 else "f64"}
    t0 = time.perf_counter()
    if c["kind"] == "qr":
        q, r = bf.qr_tensor(a)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        qo, ro, bad = orc.batch_qr_stacked(a3, m, n, 16, threads=threads)
        t2 = time.perf_counter()
        q_g, r_g = _np(q), _np(r)
        q_o, r_o = qo.transpose(0, 2, 1), ro.transpose(0, 2, 1)
        scale = np.sqrt(np.sum(a_np * a_np, axis=(1, 2)))
        dq = np.max(np.abs(q_g - q_o), axis=(1, 2)) / (eps * np.maximum(scale, 1.0))
        dr = np.max(np.abs(r_g - r_o), axis=(1, 2)) / (eps * np.maximum(scale, 1.0))
        qr_g = np.matmul(q_g, r_g)
        qr_o = np.matmul(q_o, r_o)
        rec.update({
            "q_vs_oracle_eps_normA": dist(dq), "r_vs_oracle_eps_normA": dist(dr),
            "r_lower_exact_zero": bool(np.all(np.tril(r_g, -1) == 0)),
            "orth_q": res_pair(orth_res(q_g), orth_res(q_o)),
            "recon": res_pair(np.sqrt(np.sum((a_np - qr_g) ** 2, axis=(1, 2))) / scale,
                              np.sqrt(np.sum((a_np - qr_o) ** 2, axis=(1, 2))) / scale),
            "oracle_bad_index": int(bad),
        })
    elif c["kind"] in ("svd", "block"):
        if c["kind"] == "svd":
            r = bf.svd_tensor(a, bf.JacobiOptions(ordering=c["ordering"], accumulate_v=True))
        else:
            r = bf.block_svd_tensor(a, bf.BlockJacobiOptions(method=c["method"], block_width=32, tolerance=c["tol"],
                                                              accumulate_v=True))
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        if c["kind"] == "svd":
            o = orc.batch_svd_stacked(a3, m, n, ordering=c["ordering"], accumulate_v=True, threads=threads)
        else:
            o = orc.batch_block_svd_stacked(a3, m, n, block_width=32, method=c["method"], tol=c["tol"],
                                            accumulate_v=True, threads=threads)
        t2 = time.perf_counter()
        u_g, s_g, v_g = _np(r["u"]), _np(r["sigma"]), _np(r["v"])
        sw_g, cv_g = _np(r["sweeps"]).astype(np.int64), _np(r["converged"]).astype(bool)
        u_o, s_o, v_o = o["u"].transpose(0, 2, 1), o["s"], o["v"].transpose(0, 2, 1)
        sw_o, cv_o = o["sweeps"].astype(np.int64), o["converged"].astype(bool)
        normwise, per_value = sigma_stats(s_g, s_o)
        floor = lapack_floor(a_np, s_o)
        gpu_floor = lapack_floor(a_np, s_g)
        fac = 256.0 if c["kind"] == "svd" else 4096.0
        um = vec_mismatch_batch(u_g, u_o, s_o, fac, eps=eps)
        vm = vec_mismatch_batch(v_g, v_o, s_o, fac, eps=eps)
        dsw = sw_g - sw_o
        odd = np.flatnonzero((cv_g != cv_o) | (np.abs(dsw) > 1))
        chaotic = []
        tol = c.get("tol") or (1e-5 if f32 else 1e-13)
        if c["kind"] == "block":
            eh_all_g = _np(r["e_history"])
            for b in odd:
                eo = o["e_history"][b, : sw_o[b]]
                eg = eh_all_g[b, : sw_g[b]]
                # hovering: e within [tol/10, 100 tol] for >= 2 sweeps on either side (SURVEY §7:
                # Gram's e floor ~ eps kappa^2 sits at tol for these entries)
                hov = np.sum((eo > tol / 10) & (eo < tol * 100)) + np.sum((eg > tol / 10) & (eg < tol * 100))
                if c["method"] == "gram" and hov >= 2:
                    chaotic.append(int(b))
        rec.update({
            "sigma_normwise": dist(normwise), "sigma_per_value_rel": dist(per_value),
            "oracle_vs_lapack_per_value_rel": dist(floor),
            "gpu_vs_lapack_per_value_rel": dist(gpu_floor),
            "u_mismatch_ratio": dist(um), "v_mismatch_ratio": dist(vm),
            "converged_equal": int(np.sum(cv_g == cv_o)), "converged_gpu": int(cv_g.sum()),
            "converged_oracle": int(cv_o.sum()),
            "sweeps_abs_diff_max": int(np.max(np.abs(dsw))) if B else 0,
            "sweeps_diff_hist": {str(k): int(v) for k, v in zip(*np.unique(dsw, return_counts=True))},
            "sweeps_mean": {"gpu": float(sw_g.mean()), "oracle": float(sw_o.mean())},
            "orth_u": res_pair(orth_res(u_g), orth_res(u_o), chaotic),
            "orth_v": res_pair(orth_res(v_g), orth_res(v_o), chaotic),
            "recon": res_pair(recon_res(a_np, u_g, s_g, v_g), recon_res(a_np, u_o, s_o, v_o), chaotic),
            "chaotic_entries": chaotic,
        })
        if f32:
            # float32: the oracle's own distance from the exact singular values can exceed the
            # 1e-5 gate (block direct, tol 1e-5); record both distances per matrix
            ge, oe = exact_normwise(a_np, s_g), exact_normwise(a_np, s_o)
            rec["sigma_normwise_vs_exact"] = {"gpu": dist(ge), "oracle": dist(oe)}
            rec["sigma_f32_fail"] = int(np.sum((normwise > 1e-5) & (ge > oe)))
            fx = ref_fixture(name)
            if fx is not None:
                idx = fx["index"]
                d = sw_g[idx] - fx["sweeps"]
                rec["vs_reference"] = {
                    "entries": int(idx.size),
                    "sweeps_gpu_minus_ref_hist": {str(k): int(v) for k, v in zip(*np.unique(d, return_counts=True))},
                    "sweeps_oracle_minus_ref_hist": {
                        str(k): int(v) for k, v in zip(*np.unique(sw_o[idx] - fx["sweeps"], return_counts=True))},
                    "converged_equal": int(np.sum(cv_g[idx] == fx["converged"])),
                    "ref_max": {"orth_u": float(fx["orth_u"].max()), "orth_v": float(fx["orth_v"].max()),
                                "recon": float(fx["recon"].max())},
                    "full_batch": bool(idx.size == B),
                }
        # entries whose flags or sweep counts differ beyond +-1, with the e history that explains them
        rec["flag_or_sweep_outliers"] = []
        for b in odd[:300]:
            item = {"index": int(b), "sweeps_gpu": int(sw_g[b]), "sweeps_oracle": int(sw_o[b]),
                    "conv_gpu": bool(cv_g[b]), "conv_oracle": bool(cv_o[b])}
            if c["kind"] == "block":
                eo = o["e_history"][b, : sw_o[b]]
                eg = _np(r["e_history"])[b, : sw_g[b]]
                item["oracle_e_over_tol_last5"] = [float(x / tol) for x in eo[-5:]]
                item["gpu_e_over_tol_last5"] = [float(x / tol) for x in eg[-5:]]
                item["marginal"] = int(b) in chaotic
            rec["flag_or_sweep_outliers"].append(item)
        if c["kind"] == "block":
            eh_g, eh_o = _np(r["e_history"]), o["e_history"]
            k = np.minimum(sw_g, sw_o)
            rel = []
            for b in range(B):
                e1, e2 = eh_g[b, : k[b]], eh_o[b, : k[b]]
                big = e2 > 1e-8
                if np.any(big):
                    rel.append(np.max(np.abs(e1[big] - e2[big]) / e2[big]))
            rec["e_history_rel_above_1e-8"] = dist(np.array(rel))
    else:  # rsvd
        opts = bf.RsvdOptions(k=c["k"], p=c["p"], seed=c["rsvd_seed"])
        r = bf.rsvd_tensor(a, opts)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        o = orc.batch_rsvd_stacked(a3, m, n, c["k"], c["p"], seed=c["rsvd_seed"], threads=threads)
        t2 = time.perf_counter()
        u_g, s_g, v_g = _np(r["u"]), _np(r["s"]), _np(r["v"])
        u_o, s_o, v_o = o["u"].transpose(0, 2, 1), o["s"], o["v"].transpose(0, 2, 1)
        normwise, per_value = sigma_stats(s_g, s_o)
        k = c["k"]
        um = vec_mismatch_batch(u_g, u_o, s_o, 4096.0, ncols=k, eps=eps)
        vm = vec_mismatch_batch(v_g, v_o, s_o, 4096.0, ncols=k, eps=eps)
        _, pv_k = sigma_stats(s_g[:, :k], s_o[:, :k])
        rec.update({
            "sigma_normwise": dist(normwise), "sigma_per_value_rel": dist(per_value),
            "sigma_per_value_rel_top_k": dist(pv_k),
            "u_mismatch_ratio_top_k": dist(um), "v_mismatch_ratio_top_k": dist(vm),
            "orth_u": res_pair(orth_res(u_g), orth_res(u_o)),
            "orth_v": res_pair(orth_res(v_g), orth_res(v_o)),
            "recon": res_pair(recon_res(a_np, u_g, s_g, v_g), recon_res(a_np, u_o, s_o, v_o)),
            "oracle_bad_index": int(o["bad"]),
        })
    rec["gpu_call_s"] = t1 - t0
    rec["oracle_s"] = t2 - t1
    rec["oracle_threads"] = threads
    return rec


# ------------------------------------------------------------------ gates


def check(rec):
    """List of failed gates (empty = pass)."""
    bad = []
    name = rec["config"]
    kind = CONFIGS[name]["kind"]

    def res_gate(key):
        g, o = rec[key]["gpu_max"], rec[key]["oracle_max"]
        if rec.get("dtype") == "f32":
            # float32 residuals sit at the stopping tolerance (pairs left just under tol); the maxima
            # of the reference and of its C restatement themselves differ by ~1 % (cfg1f32: 9.15e-6
            # vs 9.08e-6, cfg3f32: 1.757e-5 vs 1.736e-5, profiles/f32_ref_r02.json), so "no worse"
            # is judged against the larger of the two with a 2 % band
            vr = rec.get("vs_reference")
            if vr and vr["full_batch"]:
                o = max(o, vr["ref_max"].get(key, o))
            o *= 1.02
        if g > o:
            bad.append(f"{name}: {key} gpu max {g:.3e} > oracle max {o:.3e}")

    if kind == "qr":
        if rec["q_vs_oracle_eps_normA"]["max"] > 64 or rec["r_vs_oracle_eps_normA"]["max"] > 64:
            bad.append(f"{name}: Q/R elementwise beyond 64 eps ||A||")
        if not rec["r_lower_exact_zero"]:
            bad.append(f"{name}: R has nonzeros below the diagonal")
        res_gate("orth_q")
        res_gate("recon")
        return bad
    f32 = rec.get("dtype") == "f32"
    if f32:
        # float32 (north_star: 1e-5): within 1e-5 normwise of the oracle, or closer to the exact
        # singular values than the oracle is (the reference's own float32 error can exceed 1e-5)
        nfail = rec.get("sigma_f32_fail", int(rec["sigma_normwise"]["max"] > 1e-5))
        if nfail:
            bad.append(f"{name}: {nfail} matrices with sigma > 1e-5 from the oracle and farther "
                       "from exact than the oracle")
    elif rec["sigma_normwise"]["max"] > 1e-12:
        bad.append(f"{name}: sigma normwise {rec['sigma_normwise']['max']:.3e} > 1e-12")
    if kind == "rsvd":
        if rec["u_mismatch_ratio_top_k"]["max"] > 1 or rec["v_mismatch_ratio_top_k"]["max"] > 1:
            bad.append(f"{name}: top-k vectors differ beyond sign")
    else:
        if rec["u_mismatch_ratio"]["max"] > 1 or rec["v_mismatch_ratio"]["max"] > 1:
            bad.append(f"{name}: U/V differ beyond sign")
        # Flags equal and sweeps within +-1. Exception, block Gram only: entries whose
        # e history hovers at tol (within [tol/10, 100 tol] for >= 2 sweeps on either side) decide
        # their converged sweep by rounding. The reference itself (Python/OpenBLAS) disagrees with
        # its faithful C restatement on 35 of 50 such cfg4 entries and on ~7 % of the batch
        # (profiles/cfg4_chaos_r02.json), so these are "chaotic": reported, capped at 10 % of the
        # batch, and left out of the gated residual maxima (their residuals are listed as *_all).
        outl = rec["flag_or_sweep_outliers"]
        if f32:
            # float32 at the default tolerance (1e-6 / 1e-5) converges at the rounding noise floor:
            # the reference and its restatement differ by 2 sweeps on 9 of 5000 cfg3f32 entries
            # (profiles/f32_ref_r02.json); float32 twins gate flags equal and sweeps within +-2
            outl = [o for o in outl if o["conv_gpu"] != o["conv_oracle"] or abs(o["sweeps_gpu"] - o["sweeps_oracle"]) > 2]
        hard = [o for o in outl if not o.get("marginal", False)]
        if hard:
            bad.append(f"{name}: {len(hard)} entries with converged flags / sweeps (+-1) differing, first {hard[0]}")
        if len(outl) > 0.10 * rec["batch"]:
            bad.append(f"{name}: {len(outl)} chaotic flag/sweep outliers (> 10 % of the batch)")
    for key in ("orth_u", "orth_v", "recon"):
        res_gate(key)
    return bad


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default=",".join(k for k in CONFIGS if not k.endswith("f32")))
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "parity_r02.json"))
    ap.add_argument("--threads", type=int, default=host_threads())
    args = ap.parse_args()
    from oracle import oracle as orc

    orc.build()
    out = {"what": "full-config parity, every entry: CUDA path (C ABI) vs the CPU oracle on the same inputs",
           "host_threads": args.threads, "configs": {}}
    failed = []
    for name in args.configs.split(","):
        rec = run_config(name, args.threads)
        rec["failed_gates"] = check(rec)
        failed += rec["failed_gates"]
        out["configs"][name] = rec
        print(json.dumps({name: rec}), flush=True)
    out["all_pass"] = not failed
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as fh:
        json.dump(out, fh, indent=1)
    print("FAILED:" if failed else "ALL PASS", *failed, sep="\n  ")


if __name__ == "__main__":
    main()
