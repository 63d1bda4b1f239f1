"""The reference's public helper functions, on the device through the C ABI.

batchfact re-exports these next to its batch entry points (/root/reference/pkg/src/batchfact/
__init__.py:3-23; ``scaled_offdiag`` from blockjacobi.py:57):

  householder_vector  qr.py:26-48      -> bf_householder_batched_*
  jacobi_rotation     jacobi.py:68-80  -> bf_jacobi_rotation_batched_f64
  off_orthogonality   jacobi.py:83-99  -> bf_off_orthogonality_batched_*
  scaled_offdiag      blockjacobi.py:57-76 -> bf_scaled_offdiag_batched_*
  syrk                core.py:68-78    -> bf_syrk_batched_*
  gemm                core.py:36-65    -> bf_gemm_batched_* + bf_axpby_*
  frobenius           core.py:81-86    -> bf_frobenius_batched_*
  batch_apply         core.py:97-123   (host orchestration: the same thread-pool contract)

Same signatures, argument checks and error types as the reference; results agree with it to
rounding (the device sums in a different order). Each call is one small batched launch of a
single entry -- these are conveniences around the batched hot path, not part of it.
"""

from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

from . import _lib
from .core import BatchError, as_matrix, ptr, resolve_device, stream_handle, to_host, torch_dtype


def _to_dev(a, dev):
    """numpy (any order) -> contiguous device tensor of the same memory layout as Fortran a."""
    return torch.as_tensor(np.ascontiguousarray(a)).to(dev)


def _colmajor_dev(a, dev):
    """(m, n) numpy -> device (n, m) contiguous == column-major m x n."""
    return torch.as_tensor(np.ascontiguousarray(a.T)).to(dev)


def _scalar(t):
    return float(to_host(t)[0])


def householder_vector(x, *, device=None):
    """Reflector (v, tau) with v[0] = 1 mapping x to (beta, 0, ..., 0) (qr.py:26-48)."""
    x = np.asarray(x)
    if x.ndim != 1 or x.size == 0:
        raise ValueError("householder_vector expects a nonempty vector")
    if x.dtype.type not in (np.float32, np.float64):
        x = x.astype(np.float64)
    L = _lib.load()
    dev = resolve_device(device)
    xd = _to_dev(x, dev)
    v = torch.empty_like(xd)
    tau = torch.empty(1, dtype=xd.dtype, device=dev)
    fn = L.bf_householder_batched_f64 if x.dtype == np.float64 else L.bf_householder_batched_f32
    with torch.cuda.device(dev):
        rc = fn(1, x.size, ptr(xd), ptr(v), ptr(tau), stream_handle(dev))
    _lib.check(rc, "householder_vector")
    return to_host(v).copy(), _scalar(tau)


def jacobi_rotation(g_pp, g_pq, g_qq, *, device=None):
    """Stable rotation (c, s) diagonalising [[g_pp, g_pq], [g_pq, g_qq]] (jacobi.py:68-80)."""
    L = _lib.load()
    dev = resolve_device(device)
    g = torch.tensor([float(g_pp), float(g_pq), float(g_qq)], dtype=torch.float64, device=dev)
    out = torch.empty(2, dtype=torch.float64, device=dev)
    with torch.cuda.device(dev):
        rc = L.bf_jacobi_rotation_batched_f64(1, ptr(g[0:1]), ptr(g[1:2]), ptr(g[2:3]), ptr(out[0:1]),
                                              ptr(out[1:2]), stream_handle(dev))
    _lib.check(rc, "jacobi_rotation")
    c, s = to_host(out)
    return float(c), float(s)


def _offdiag(a, gram, what, device):
    L = _lib.load()
    dev = resolve_device(device)
    ad = _colmajor_dev(a, dev)
    out = torch.empty(1, dtype=ad.dtype, device=dev)
    m, n = a.shape
    f64 = a.dtype == np.float64
    with torch.cuda.device(dev):
        if gram:
            fn = L.bf_off_orthogonality_batched_f64 if f64 else L.bf_off_orthogonality_batched_f32
            rc = fn(1, m, n, ptr(ad), ptr(out), stream_handle(dev))
        else:
            fn = L.bf_scaled_offdiag_batched_f64 if f64 else L.bf_scaled_offdiag_batched_f32
            rc = fn(1, n, ptr(ad), ptr(out), stream_handle(dev))
    _lib.check(rc, what)
    return _scalar(out)


def off_orthogonality(a, *, device=None):
    """Max over column pairs of |<a_i, a_j>| / (||a_i|| ||a_j||); zero columns give 0 (jacobi.py:83-99)."""
    a = as_matrix(a)
    if a.shape[1] < 2:
        return 0.0
    return _offdiag(a, True, "off_orthogonality", device)


def scaled_offdiag(g, *, device=None):
    """Max over i != j of |g_ij| / sqrt(|g_ii| |g_jj|); 0/0 -> 0, x/0 -> inf (blockjacobi.py:57-76)."""
    g = as_matrix(g)
    if g.shape[0] != g.shape[1]:
        raise ValueError(f"scaled_offdiag expects a square matrix, got {g.shape}")
    if g.shape[0] < 2:
        return 0.0
    return _offdiag(g, False, "scaled_offdiag", device)


def syrk(a, *, device=None):
    """Gram matrix a.T @ a, exactly symmetric (upper triangle mirrored, core.py:68-78)."""
    a = as_matrix(a)
    m, k = a.shape
    L = _lib.load()
    dev = resolve_device(device)
    ad = _colmajor_dev(a, dev)
    g = torch.empty((k, k), dtype=ad.dtype, device=dev)
    fn = L.bf_syrk_batched_f64 if a.dtype == np.float64 else L.bf_syrk_batched_f32
    with torch.cuda.device(dev):
        rc = fn(1, m, k, ptr(ad), ptr(g), stream_handle(dev))
    _lib.check(rc, "syrk")
    return np.asfortranarray(to_host(g).T)


def frobenius(a, *, device=None):
    """Frobenius norm; 0.0 for an empty matrix (core.py:81-86)."""
    a = as_matrix(a)
    if a.size == 0:
        return 0.0
    L = _lib.load()
    dev = resolve_device(device)
    ad = _colmajor_dev(a, dev)
    out = torch.empty(1, dtype=ad.dtype, device=dev)
    fn = L.bf_frobenius_batched_f64 if a.dtype == np.float64 else L.bf_frobenius_batched_f32
    with torch.cuda.device(dev):
        rc = fn(1, a.shape[0], a.shape[1], ptr(ad), ptr(out), stream_handle(dev))
    _lib.check(rc, "frobenius")
    return _scalar(out)


def gemm(a, b, c=None, *, alpha=1.0, beta=0.0, trans_a=False, trans_b=False, device=None):
    """alpha * op(a) @ op(b) + beta * c as a new array; c is never written and is ignored when
    beta == 0 (core.py:36-65)."""
    a = as_matrix(a)
    b = as_matrix(b)
    oa_shape = a.shape[::-1] if trans_a else a.shape
    ob_shape = b.shape[::-1] if trans_b else b.shape
    if oa_shape[1] != ob_shape[0]:
        raise ValueError(f"gemm conformance error: op(a) is {oa_shape}, op(b) is {ob_shape}")
    M, K, N = oa_shape[0], oa_shape[1], ob_shape[1]
    dt = np.result_type(a.dtype, b.dtype)
    cc = None
    if beta != 0.0:
        if c is None:
            raise ValueError("gemm: beta != 0 requires c")
        cc = as_matrix(c)
        if cc.shape != (M, N):
            raise ValueError(f"gemm conformance error: c is {cc.shape}, product is {(M, N)}")
    a, b = a.astype(dt, copy=False), b.astype(dt, copy=False)
    L = _lib.load()
    dev = resolve_device(device)
    ad, bd = _colmajor_dev(a, dev), _colmajor_dev(b, dev)
    p = torch.empty((N, M), dtype=torch_dtype(dt), device=dev)  # column-major M x N
    f64 = dt == np.float64
    sh = stream_handle(dev)
    with torch.cuda.device(dev):
        fn = L.bf_gemm_batched_f64 if f64 else L.bf_gemm_batched_f32
        rc = fn(1, M, N, K, ptr(ad), max(a.shape[0], 1), a.size, int(trans_a), ptr(bd), max(b.shape[0], 1), b.size,
                int(trans_b), ptr(p), max(M, 1), M * N, sh)
        _lib.check(rc, "gemm")
        if alpha != 1.0 or beta != 0.0:
            cd = _colmajor_dev(cc.astype(dt, copy=False), dev) if cc is not None else None
            fn = L.bf_axpby_f64 if f64 else L.bf_axpby_f32
            rc = fn(M * N, float(alpha), ptr(p), float(beta), ptr(cd), ptr(p), sh)
            _lib.check(rc, "gemm")
    return np.asfortranarray(to_host(p).T)


def batch_apply(entries, op, *, threads=1):
    """Apply ``op`` to every entry independently; each entry start-to-finish on one worker, so the
    results are bitwise independent of ``threads``; the lowest failing index is raised as
    :class:`BatchError` after the whole batch ran (core.py:97-123). The batched entry points of
    this package do not route through it: a homogeneous group is ONE device call."""
    entries = list(entries)
    results = [None] * len(entries)
    errors = {}

    def run(i):
        try:
            results[i] = op(entries[i])
        except Exception as exc:  # noqa: BLE001 - reported with the batch index
            errors[i] = exc

    if threads > 1 and len(entries) > 1:
        with ThreadPoolExecutor(max_workers=threads) as pool:
            list(pool.map(run, range(len(entries))))
    else:
        for i in range(len(entries)):
            run(i)
    if errors:
        i = min(errors)
        raise BatchError(i, errors[i]) from errors[i]
    return results
