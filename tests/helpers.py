"""Shared parity helpers: golden loading and the comparison rules of SURVEY.md §8(c)."""

import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

_cache = {}


def golden(name):
    if name not in _cache:
        z = np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False)
        _cache[name] = {k: z[k] for k in z.files}
    return _cache[name]


def case(g, name):
    pre = name + "/"
    return {k[len(pre):]: v for k, v in g.items() if k.startswith(pre)}


def names(g):
    return [str(x) for x in g["names"]]


def eps(dtype):
    return float(np.finfo(dtype).eps)


def sigma_normwise(s, s_ref):
    """max |ds_i| / s_1 (the hard gate: 1e-12 fp64, 1e-5 fp32)."""
    s = np.asarray(s, dtype=np.float64)
    s_ref = np.asarray(s_ref, dtype=np.float64)
    if s_ref.size == 0:
        return 0.0
    scale = max(abs(s_ref[0]), np.finfo(np.float64).tiny)
    return float(np.max(np.abs(s - s_ref)) / scale)


def vec_mismatch(x, x_ref, s_ref, dtype, factor=256.0):
    """Columns compared up to sign; tolerance scaled by sigma_1/gap (Davis-Kahan).

    Returns the worst (error / tolerance) ratio over columns with a nonzero,
    non-degenerate singular value; <= 1 means pass.
    """
    x = np.asarray(x, dtype=np.float64)
    x_ref = np.asarray(x_ref, dtype=np.float64)
    s = np.asarray(s_ref, dtype=np.float64)
    n = x.shape[1]
    if n == 0:
        return 0.0
    s1 = max(s[0], np.finfo(np.float64).tiny)
    worst = 0.0
    e = eps(dtype)
    for j in range(n):
        if s[j] <= s1 * 1e3 * e:
            continue
        others = np.delete(s, j)
        gap = np.min(np.abs(others - s[j])) if others.size else s1
        if gap <= s1 * 1e3 * e:
            continue
        sign = 1.0 if np.dot(x[:, j], x_ref[:, j]) >= 0 else -1.0
        err = np.max(np.abs(sign * x[:, j] - x_ref[:, j]))
        tol = factor * e * s1 / gap
        worst = max(worst, err / tol)
    return worst


def orth_residual(q):
    q = np.asarray(q, dtype=np.float64)
    return float(np.linalg.norm(q.T @ q - np.eye(q.shape[1])))


def recon_residual(a, u, s, v):
    a = np.asarray(a, dtype=np.float64)
    r = np.asarray(u, dtype=np.float64) * np.asarray(s, dtype=np.float64)[None, :] @ np.asarray(v, dtype=np.float64).T
    na = np.linalg.norm(a)
    return float(np.linalg.norm(a - r) / (na if na > 0 else 1.0))
