"""Generate the golden fixtures in tests/golden/ by running the REFERENCE itself.

This script imports the reference package ``batchfact`` from
``/root/reference/pkg/src`` (pure Python + numpy; nothing to build) and records its
inputs/outputs for the hot path: QR (qr.py:63-100), Jacobi SVD in both orderings
(jacobi.py:231-290), block Jacobi in both methods (blockjacobi.py:84-174),
randomized SVD (rsvd.py:56-86), the Gaussian sampler (rsvd.py:42-53) and the
prescribed-spectrum generator (testmat.py:83-94).

It runs ONLY in the build container (``/root/reference`` does not exist on the GPU
box). The committed .npz files are what the tests read at run time.

    python tests/golden/make_golden.py
"""

import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

import batchfact  # noqa: E402
import importlib  # noqa: E402

qr = importlib.import_module("batchfact.qr")
jacobi = importlib.import_module("batchfact.jacobi")
blockjacobi = importlib.import_module("batchfact.blockjacobi")
rsvd = importlib.import_module("batchfact.rsvd")
testmat = importlib.import_module("batchfact.testmat")


def gauss(m, n, seed, dtype=np.float64):
    return rsvd.gaussian_matrix(m, n, seed, dtype=dtype)


def pack(prefix, d, out):
    for k, v in d.items():
        out[f"{prefix}{k}"] = np.asarray(v)


def gen_qr():
    cases = []
    cases.append(("eye4", np.eye(4), 16))
    cases.append(("col34", np.array([[3.0], [4.0]]), 16))
    cases.append(("one", np.array([[2.5]]), 16))
    for i, (m, n) in enumerate([(8, 3), (17, 17), (64, 32), (64, 32), (128, 40), (33, 5), (256, 64)]):
        cases.append((f"g{i}_{m}x{n}", gauss(m, n, 2_000_000 + i), 16))
    cases.append(("pw1_64x32", gauss(64, 32, 2_000_100), 1))
    cases.append(("pw5_40x20", gauss(40, 20, 2_000_101), 5))
    a = gauss(12, 6, 2_000_102)
    a[:, 2] = 0.0
    a[:, 4] = a[:, 1]
    cases.append(("rankdef_12x6", a, 16))
    cases.append(("zero_5x3", np.zeros((5, 3)), 16))
    cases.append(("f32_64x32", gauss(64, 32, 2_000_103, np.float32), 16))
    out = {"names": np.array([c[0] for c in cases])}
    for name, a, pw in cases:
        a = np.asfortranarray(a)
        res = qr.qr(a, pw)
        pack(f"{name}/", {"a": a, "pw": pw, "q": res.q, "r": res.r}, out)
    np.savez_compressed(os.path.join(HERE, "qr.npz"), **out)


def gen_svd():
    cases = []
    # (name, a, ordering, accumulate_v, tolerance, max_sweeps)
    cases.append(("kat_3045", np.array([[3.0, 0.0], [4.0, 5.0]]), "serial", True, None, 30))
    cases.append(("kat_diag", np.diag([1.0, 3.0, 2.0]), "serial", True, None, 30))
    cases.append(("one", np.array([[-2.0]]), "serial", True, None, 30))
    cases.append(("col", np.array([[1.0], [2.0], [2.0]]), "round_robin", True, None, 30))
    for order in ("serial", "round_robin"):
        for i in range(6):
            cases.append((f"c1_{order}_{i}", gauss(32, 32, 1_000_000 + i), order, True, None, 30))
        cases.append((f"g_{order}_33x17", gauss(33, 17, 1_100_000), order, True, None, 30))
        cases.append((f"g_{order}_20x7", gauss(20, 7, 1_100_001), order, False, None, 30))
        cases.append((f"g_{order}_64x24", gauss(64, 24, 1_100_002), order, True, None, 30))
        cases.append((f"g_{order}_40x40", gauss(40, 40, 1_100_003), order, True, None, 30))
        a = gauss(16, 8, 1_100_004)
        a[:, 3] = 0.0
        a[:, 6] = 2.0 * a[:, 1]
        cases.append((f"rankdef_{order}_16x8", a, order, True, None, 30))
        cases.append((f"zero_{order}_6x4", np.zeros((6, 4)), order, True, None, 30))
        cases.append((f"ms1_{order}_24x24", gauss(24, 24, 1_100_005), order, True, None, 1))
        cases.append((f"f32_{order}_32x32", gauss(32, 32, 1_100_006, np.float32), order, True, None, 30))
        cases.append((f"tol_{order}_32x16", gauss(32, 16, 1_100_007), order, True, 1e-8, 30))
    for i in range(3):
        cases.append((f"c3_rr_{i}", gauss(64, 64, 3_000_000 + i), "round_robin", True, None, 30))
    spec = testmat.SpectrumSpec(n=32, mode="geometric", cond=1e4)
    a, sig = testmat.make_matrix(32, spec, 7)
    cases.append(("testmat_32_c1e4", a, "serial", True, None, 30))
    out = {"names": np.array([c[0] for c in cases])}
    for name, a, order, accv, tol, ms in cases:
        a = np.asfortranarray(a)
        opts = jacobi.JacobiOptions(tolerance=tol, max_sweeps=ms, ordering=order, accumulate_v=accv)
        res = jacobi.svd(a, opts)
        d = {
            "a": a,
            "ordering": order,
            "accumulate_v": accv,
            "tolerance": -1.0 if tol is None else tol,
            "max_sweeps": ms,
            "u": res.u,
            "sigma": res.sigma,
            "converged": res.converged,
            "sweeps": res.sweeps,
        }
        if res.v is not None:
            d["v"] = res.v
        pack(f"{name}/", d, out)
    out["testmat_32_c1e4/exact_sigma"] = sig
    np.savez_compressed(os.path.join(HERE, "svd.npz"), **out)


def gen_block():
    cases = []
    cases.append(("eye64_gram", np.eye(64), "gram", 16, None, True))
    cases.append(("eye64_direct", np.eye(64), "direct", 16, None, True))
    cases.append(("g96x64_gram", gauss(96, 64, 4_100_000), "gram", 16, 1e-11, True))
    cases.append(("g96x64_direct", gauss(96, 64, 4_100_000), "direct", 16, None, True))
    cases.append(("g128_gram", gauss(128, 128, 4_100_001), "gram", 32, 1e-11, True))
    cases.append(("g128_direct", gauss(128, 128, 4_100_001), "direct", 32, None, True))
    cases.append(("g70x50_gram", gauss(70, 50, 4_100_002), "gram", 8, 1e-11, False))
    cases.append(("g70x50_direct", gauss(70, 50, 4_100_002), "direct", 8, None, False))
    cases.append(("c4_gram_0", gauss(256, 256, 4_000_000), "gram", 32, 1e-11, True))
    cases.append(("c4_direct_0", gauss(256, 256, 4_000_000), "direct", 32, None, True))
    spec = testmat.SpectrumSpec(n=128, mode="geometric", cond=1e7)
    a, sig = testmat.make_matrix(128, spec, 11)
    cases.append(("tm128_c1e7_direct", a, "direct", 32, None, True))
    cases.append(("tm64_c1e7_gram_f32", testmat.make_matrix(64, testmat.SpectrumSpec(n=64, mode="geometric", cond=1e7), 12, dtype=np.float32)[0], "gram", 16, None, False))
    out = {"names": np.array([c[0] for c in cases])}
    for name, a, method, bw, tol, accv in cases:
        t0 = time.time()
        a = np.asfortranarray(a)
        opts = blockjacobi.BlockJacobiOptions(
            block_width=bw, method=method, tolerance=tol, accumulate_v=accv
        )
        res = blockjacobi.block_svd(a, opts)
        d = {
            "a": a,
            "method": method,
            "block_width": bw,
            "tolerance": -1.0 if tol is None else tol,
            "accumulate_v": accv,
            "sigma": res.sigma,
            "converged": res.converged,
            "sweeps": res.sweeps,
            "e_history": np.array(res.e_history, dtype=np.float64),
        }
        if a.shape[0] <= 128:
            d["u"] = res.u
            if res.v is not None:
                d["v"] = res.v
        else:
            d["u_head"] = res.u[:, :8]
        pack(f"{name}/", d, out)
        print(f"  block {name}: {time.time() - t0:.1f}s sweeps={res.sweeps} conv={res.converged}")
    out["tm128_c1e7_direct/exact_sigma"] = sig
    np.savez_compressed(os.path.join(HERE, "block.npz"), **out)


def gen_rsvd():
    cases = []
    spec = testmat.SpectrumSpec(n=128, mode="geometric", cond=1e16, rank=64)
    for i in range(3):
        a, sig = testmat.make_matrix(128, spec, 5_000_000 + i)
        cases.append((f"c5_{i}", a, 32, 8, 5, i, sig))
    a = gauss(64, 48, 5_100_000)
    cases.append(("g64x48", a, 8, 3, 9, 0, None))
    r8 = gauss(50, 8, 5_100_001) @ gauss(8, 30, 5_100_002)
    cases.append(("rank8_50x30", r8, 8, 4, 3, 0, None))
    cases.append(("diag", np.diag(10.0 ** -np.arange(10.0)), 4, 3, 0, 0, None))
    # float32 input: the reference draws its sketch in float32 (rsvd.py:65, dtype=a.dtype)
    a32, _ = testmat.make_matrix(64, testmat.SpectrumSpec(n=48, mode="geometric", cond=1e6, rank=48), 5_100_003)
    cases.append(("f32_64x48", a32.astype(np.float32), 8, 4, 11, 3, None))
    out = {"names": np.array([c[0] for c in cases])}
    for name, a, k, p, seed, index, sig in cases:
        a = np.asfortranarray(a)
        # batch_rsvd derives seed ^ index (rsvd.py:79-86); record the per-entry result
        res = rsvd.rsvd(a, rsvd.RsvdOptions(k=k, p=p, seed=seed ^ index))
        d = {"a": a, "k": k, "p": p, "seed": seed, "index": index, "u": res.u, "s": res.s, "v": res.v}
        if sig is not None:
            d["exact_sigma"] = sig
        pack(f"{name}/", d, out)
    np.savez_compressed(os.path.join(HERE, "rsvd.npz"), **out)


def gen_gauss_testmat():
    out = {}
    seeds = [0, 5, 7, 123456789, (1 << 64) + 3, (1 << 100) + 77]
    for j, s in enumerate(seeds):
        out[f"g{j}/seed_lo"] = np.uint64(s & ((1 << 64) - 1))
        out[f"g{j}/seed_hi"] = np.uint64(s >> 64)
        out[f"g{j}/x"] = gauss(128, 40, s)
        # float32 is numpy's own float ziggurat stream (rsvd.py:52 with dtype=float32)
        out[f"g{j}/x32"] = gauss(128, 40, s, np.float32)
    out["g_count"] = len(seeds)
    spec = testmat.SpectrumSpec(n=128, mode="geometric", cond=1e16, rank=64)
    a, sig = testmat.make_matrix(128, spec, 5_000_000)
    out["tm/a"] = a
    out["tm/sigma"] = sig
    out["tm/p"] = testmat.random_orthonormal(40, 40, 99)
    # the batch error convention (core.py:97-123): lowest failing index
    try:
        batchfact.batch_qr([np.ones((4, 2)), np.ones((2, 3)), np.ones((3, 2)), np.ones((1, 5))])
    except batchfact.BatchError as e:
        out["batch_error_index"] = e.index
    np.savez_compressed(os.path.join(HERE, "gauss_testmat.npz"), **out)


if __name__ == "__main__":
    only = set(sys.argv[1:])  # e.g. `make_golden.py gen_rsvd` regenerates one fixture file
    for fn in (gen_gauss_testmat, gen_qr, gen_svd, gen_rsvd, gen_block):
        if only and fn.__name__ not in only:
            continue
        t0 = time.time()
        fn()
        print(f"{fn.__name__}: {time.time() - t0:.1f}s")
