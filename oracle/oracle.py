"""ctypes front-end of the CPU oracle (oracle.c). TEST INFRASTRUCTURE ONLY.

Importable only from tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs -- never from the product package. Arrays follow the
reference's layout: each matrix column-major; batches are stacked (B, m, n) arrays
whose per-matrix storage is column-major (i.e. built from Fortran-ordered entries).
"""

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

_lib = None


def build(force=False):
    """Compile liboracle.so with the committed Makefile (gcc only)."""
    if force or not os.path.exists(LIB_PATH) or _stale():
        subprocess.run(["make", "-s", "-C", HERE, "liboracle.so"], check=True)


def _stale():
    so = os.path.getmtime(LIB_PATH)
    return any(
        os.path.getmtime(os.path.join(HERE, f)) > so
        for f in ("oracle.c", "oracle_impl.h", "ziggurat_tables.h")
    )


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        P, I, D, U64, I64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_uint64, ctypes.c_int64
        L.orc_gaussian_f64.argtypes = [I, I, U64, U64, P]
        L.orc_gaussian_f32.argtypes = [I, I, U64, U64, P]
        L.orc_philox_raw.argtypes = [U64, U64, I, P]
        L.orc_round_robin.argtypes = [I, P]
        L.orc_rotation.argtypes = [D, D, D, P]
        L.orc_householder_f64.argtypes = [P, I, P]
        L.orc_householder_f64.restype = D
        L.orc_off_orthogonality_f64.argtypes = [P, I, I]
        L.orc_off_orthogonality_f64.restype = D
        L.orc_scaled_offdiag_f64.argtypes = [P, I]
        L.orc_scaled_offdiag_f64.restype = D
        L.orc_syrk_f64.argtypes = [I, I, P, P]
        L.orc_batch_qr.argtypes = [I, I64, I, I, P, P, P, I, I]
        L.orc_batch_qr.restype = I64
        L.orc_batch_svd.argtypes = [I, I64, I, I, P, P, P, P, P, P, P, D, I, I, I]
        L.orc_batch_svd.restype = I64
        L.orc_batch_block_svd.argtypes = [I, I64, I, I, P, P, P, P, P, P, P, I, I, D, I, I]
        L.orc_batch_block_svd.restype = I64
        L.orc_batch_rsvd.argtypes = [I, I64, I, I, I, I, U64, U64, I64, P, P, P, P, P, I]
        L.orc_batch_rsvd.restype = I64
        L.orc_make_matrix_f64.argtypes = [I, I, I, D, I, U64, U64, P, P]
        L.orc_make_matrix_f64.restype = I
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _dt(dtype):
    return 0 if np.dtype(dtype) == np.float64 else 1


def _stack_f(batch):
    """Stack Fortran matrices into a (B, n, m) C-contiguous array (== per-matrix column-major)."""
    batch = [np.asfortranarray(a) for a in batch]
    dtype = batch[0].dtype
    m, n = batch[0].shape
    out = np.empty((len(batch), n, m), dtype=dtype)
    for i, a in enumerate(batch):
        out[i] = a.T
    return out, m, n


def _unstack(arr3):
    """(B, cols, rows) C-order -> list of (rows, cols) Fortran arrays."""
    return [np.asfortranarray(x.T) for x in arr3]


def seed_split(seed):
    seed = int(seed) & ((1 << 128) - 1)
    return seed & ((1 << 64) - 1), seed >> 64


def gaussian_matrix(rows, cols, seed, dtype=np.float64):
    """rsvd.py:42-53: numpy's Philox standard_normal stream in `dtype` (float32 is its own stream)."""
    lo, hi = seed_split(seed)
    f32 = np.dtype(dtype) == np.float32
    out = np.empty((cols, rows), dtype=np.float32 if f32 else np.float64)
    (lib().orc_gaussian_f32 if f32 else lib().orc_gaussian_f64)(rows, cols, lo, hi, _p(out))
    return np.asfortranarray(out.T)


def philox_raw(seed, n):
    lo, hi = seed_split(seed)
    out = np.empty(n, dtype=np.uint64)
    lib().orc_philox_raw(lo, hi, n, _p(out))
    return out


def round_robin(n):
    out = np.empty((n - 1, n // 2, 2), dtype=np.int32)
    lib().orc_round_robin(n, _p(out))
    return out


def rotation(gpp, gpq, gqq):
    cs = np.empty(2)
    lib().orc_rotation(gpp, gpq, gqq, _p(cs))
    return float(cs[0]), float(cs[1])


def householder(x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    v = np.empty_like(x)
    tau = lib().orc_householder_f64(_p(x), len(x), _p(v))
    return v, tau


def off_orthogonality(a):
    a = np.asfortranarray(a, dtype=np.float64)
    return lib().orc_off_orthogonality_f64(_p(a), a.shape[0], a.shape[1])


def scaled_offdiag(g):
    g = np.asfortranarray(g, dtype=np.float64)
    return lib().orc_scaled_offdiag_f64(_p(g), g.shape[0])


def syrk(a):
    a = np.asfortranarray(a, dtype=np.float64)
    g = np.empty((a.shape[1], a.shape[1]), order="F")
    lib().orc_syrk_f64(a.shape[0], a.shape[1], _p(a), _p(g))
    return g


def batch_qr_stacked(a3, m, n, panel_width=16, threads=1):
    """a3: (B, n, m) per-matrix column-major. Returns (q3 (B,n,m), r3 (B,n,n), bad_index)."""
    B = a3.shape[0]
    q = np.empty((B, n, m), dtype=a3.dtype)
    r = np.empty((B, n, n), dtype=a3.dtype)
    bad = lib().orc_batch_qr(_dt(a3.dtype), B, m, n, _p(a3), _p(q), _p(r), panel_width, threads)
    return q, r, bad


def batch_qr(batch, panel_width=16, threads=1):
    a3, m, n = _stack_f(batch)
    q, r, bad = batch_qr_stacked(a3, m, n, panel_width, threads)
    return _unstack(q), _unstack(r), bad


def batch_svd_stacked(a3, m, n, tol=None, max_sweeps=30, ordering="serial", accumulate_v=False, threads=1):
    B = a3.shape[0]
    dt = a3.dtype
    if tol is None:
        tol = 1e-14 if dt == np.float64 else 1e-6
    u = np.empty((B, n, m), dtype=dt)
    s = np.empty((B, n), dtype=dt)
    v = np.empty((B, n, n), dtype=dt) if accumulate_v else None
    sweeps = np.zeros(B, dtype=np.int32)
    conv = np.zeros(B, dtype=np.int32)
    rot = np.zeros(B, dtype=np.int64)
    bad = lib().orc_batch_svd(
        _dt(dt), B, m, n, _p(a3), _p(u), _p(s), _p(v), _p(sweeps), _p(conv), _p(rot),
        float(tol), int(max_sweeps), 0 if ordering == "serial" else 1, threads,
    )
    return dict(u=u, s=s, v=v, sweeps=sweeps, converged=conv.astype(bool), rotations=rot, bad=bad)


def svd(a, tol=None, max_sweeps=30, ordering="serial", accumulate_v=False):
    a3, m, n = _stack_f([a])
    r = batch_svd_stacked(a3, m, n, tol, max_sweeps, ordering, accumulate_v)
    return dict(
        u=np.asfortranarray(r["u"][0].T), sigma=r["s"][0],
        v=None if r["v"] is None else np.asfortranarray(r["v"][0].T),
        sweeps=int(r["sweeps"][0]), converged=bool(r["converged"][0]), rotations=int(r["rotations"][0]),
    )


def batch_block_svd_stacked(a3, m, n, block_width=32, method="direct", tol=None, max_sweeps=30,
                            accumulate_v=False, threads=1):
    B = a3.shape[0]
    dt = a3.dtype
    if tol is None:
        tol = 1e-13 if dt == np.float64 else 1e-5
    u = np.empty((B, n, m), dtype=dt)
    s = np.empty((B, n), dtype=dt)
    v = np.empty((B, n, n), dtype=dt) if accumulate_v else None
    e = np.zeros((B, max_sweeps), dtype=dt)
    sweeps = np.zeros(B, dtype=np.int32)
    conv = np.zeros(B, dtype=np.int32)
    bad = lib().orc_batch_block_svd(
        _dt(dt), B, m, n, _p(a3), _p(u), _p(s), _p(v), _p(sweeps), _p(conv), _p(e),
        int(block_width), 0 if method == "gram" else 1, float(tol), int(max_sweeps), threads,
    )
    return dict(u=u, s=s, v=v, sweeps=sweeps, converged=conv.astype(bool), e_history=e, bad=bad)


def block_svd(a, **kw):
    a3, m, n = _stack_f([a])
    r = batch_block_svd_stacked(a3, m, n, **kw)
    return dict(
        u=np.asfortranarray(r["u"][0].T), sigma=r["s"][0],
        v=None if r["v"] is None else np.asfortranarray(r["v"][0].T),
        sweeps=int(r["sweeps"][0]), converged=bool(r["converged"][0]),
        e_history=r["e_history"][0, : int(r["sweeps"][0])],
    )


def batch_rsvd_stacked(a3, m, n, k, p=8, seed=0, index_base=0, omega3=None, threads=1):
    B = a3.shape[0]
    dt = a3.dtype
    w = k + p
    u = np.empty((B, w, m), dtype=dt)
    s = np.empty((B, w), dtype=dt)
    v = np.empty((B, w, n), dtype=dt)
    lo, hi = seed_split(seed)
    bad = lib().orc_batch_rsvd(
        _dt(dt), B, m, n, k, p, lo, hi, index_base, _p(a3), _p(omega3), _p(u), _p(s), _p(v), threads
    )
    return dict(u=u, s=s, v=v, bad=bad)


def rsvd(a, k, p=8, seed=0):
    a3, m, n = _stack_f([a])
    r = batch_rsvd_stacked(a3, m, n, k, p, seed)
    return dict(u=np.asfortranarray(r["u"][0].T), s=r["s"][0], v=np.asfortranarray(r["v"][0].T), bad=r["bad"])


def make_matrix(m, n, cond, rank, seed, mode="geometric"):
    lo, hi = seed_split(seed)
    a = np.empty((n, m), dtype=np.float64)
    sig = np.empty(n)
    rc = lib().orc_make_matrix_f64(m, n, 0 if mode == "geometric" else 1, float(cond), int(rank), lo, hi, _p(a), _p(sig))
    if rc:
        raise ValueError("make_matrix: bad arguments")
    return np.asfortranarray(a.T), sig
