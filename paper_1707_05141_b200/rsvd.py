"""Batched randomized SVD (reference: /root/reference/pkg/src/batchfact/rsvd.py).

``RsvdOptions`` / ``TruncatedSvd`` (rsvd.py:19-39), ``gaussian_matrix`` (rsvd.py:42-53,
numpy Philox4x64-10 + the float64 or float32 ziggurat, reproduced bit-for-bit on the device),
``rsvd`` (Alg. 4, rsvd.py:56-76; the sketch is drawn in the input's dtype, rsvd.py:65) and
``batch_rsvd`` with per-entry seed ``seed ^ i`` (rsvd.py:79-86).
Computation: ``bf_rsvd_batched_*`` / ``bf_gaussian_batched_*``.
"""

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .core import (
    as_matrix,
    as_matrix_view,
    check_batched_tensor,
    colmajor,
    from_colmajor,
    ptr,
    resolve_device,
    resolve_devices,
    run_sharded,
    stream_handle,
    to_host,
    torch_dtype,
    workspace,
    BatchError,
)

_M64 = (1 << 64) - 1
_M128 = (1 << 128) - 1


@dataclass
class RsvdOptions:
    k: int
    p: int = 8  # oversampling
    seed: int = 0
    q_iterations: int = 0  # reserved; subspace iteration is not implemented

    def __post_init__(self):
        if self.k < 1:
            raise ValueError("k must be >= 1")
        if self.p < 0:
            raise ValueError("p must be >= 0")
        if self.q_iterations != 0:
            raise ValueError("q_iterations is reserved and must be 0")


@dataclass
class TruncatedSvd:
    u: np.ndarray  # m x (k+p)
    s: np.ndarray  # length k+p, descending
    v: np.ndarray  # n x (k+p)


def split_seed(seed):
    key = int(seed) & _M128
    return key & _M64, key >> 64


def gaussian_tensor(batch, rows, cols, seed, *, index_base=0, seed_mode="xor", dtype=torch.float64, device=None):
    """(batch, rows, cols) CUDA tensor; entry b is gaussian_matrix(rows, cols, key_b, dtype) with
    key_b = seed ^ (index_base + b) (seed_mode "xor") or seed + index_base + b ("add").
    float32 is numpy's float32 stream (its own ziggurat), not a rounded float64 draw."""
    if rows < 0 or cols < 0:
        raise ValueError("rows and cols must be >= 0")
    if dtype not in (torch.float64, torch.float32):
        raise ValueError(f"dtype must be float64 or float32, got {dtype}")
    L = _lib.load()
    dev = resolve_device(device)
    lo, hi = split_seed(seed)
    out = torch.empty((batch, cols, rows), dtype=dtype, device=dev)
    fn = L.bf_gaussian_batched_f64 if dtype == torch.float64 else L.bf_gaussian_batched_f32
    with torch.cuda.device(dev):
        rc = fn(batch, rows, cols, lo, hi, index_base, 0 if seed_mode == "xor" else 1, ptr(out), stream_handle(dev))
    _lib.check(rc, "gaussian")
    return from_colmajor(out)


def gaussian_matrix(rows, cols, seed, dtype=np.float64, *, device=None):
    """I.i.d. standard normal matrix, bitwise equal to the reference's (rsvd.py:42-53) in
    float64 or float32 (numpy draws float32 with its own float ziggurat)."""
    if rows < 0 or cols < 0:
        raise ValueError("rows and cols must be >= 0")
    dt = np.dtype(dtype)
    if dt not in (np.float64, np.float32):
        raise ValueError(f"dtype must be float64 or float32, got {dt}")
    t = gaussian_tensor(1, rows, cols, seed, dtype=torch_dtype(dt), device=device)
    return np.asfortranarray(to_host(colmajor(t))[0].T)


def _check_width(m, n, opts):
    width = opts.k + opts.p
    if width > min(m, n):
        raise ValueError(f"k + p = {width} exceeds min(m, n) = {min(m, n)} for shape {(m, n)}")


def rsvd_colmajor(store, m, n, opts, *, index_base=0, omega_store=None):
    L = _lib.load()
    dev = store.device
    B = store.shape[0]
    es = store.element_size()
    w = opts.k + opts.p
    u = torch.empty((B, w, m), dtype=store.dtype, device=dev)
    s = torch.empty((B, w), dtype=store.dtype, device=dev)
    v = torch.empty((B, w, n), dtype=store.dtype, device=dev)
    with torch.cuda.device(dev):  # sizes depend on the device (occupancy, SM count)
        nbytes = L.bf_rsvd_workspace_size(B, m, n, opts.k, opts.p, es)
    ws, wsb = workspace(nbytes, dev)
    lo, hi = split_seed(opts.seed)
    fn = L.bf_rsvd_batched_f64 if es == 8 else L.bf_rsvd_batched_f32
    with torch.cuda.device(dev):
        rc = fn(B, m, n, opts.k, opts.p, lo, hi, int(index_base), ptr(store), ptr(omega_store), ptr(u), ptr(s),
                ptr(v), ptr(ws), wsb, stream_handle(dev))
    _lib.check(rc, "rsvd")
    return dict(u=u, s=s, v=v)


def rsvd_tensor(a, opts, *, index_base=0, omega=None):
    """Tensor-native batched rsvd of a (B, m, n) CUDA tensor; entry b uses seed ^ (index_base + b).

    omega (optional): (B, n, k+p) sketch; default draws gaussian_matrix on the device.
    Returns u (B, m, k+p), s (B, k+p), v (B, n, k+p).
    """
    check_batched_tensor(a, "rsvd_tensor")
    B, m, n = a.shape
    _check_width(m, n, opts)
    om = None
    if omega is not None:
        # the kernels read n (k+p) entries per matrix at a fixed stride: validate before the launch
        w = opts.k + opts.p
        if not isinstance(omega, torch.Tensor) or tuple(omega.shape) != (B, n, w):
            raise ValueError(f"omega must be a ({B}, {n}, {w}) tensor, got "
                             f"{tuple(omega.shape) if isinstance(omega, torch.Tensor) else type(omega).__name__}")
        if omega.device != a.device:
            raise ValueError(f"omega is on {omega.device}, a is on {a.device}")
        if omega.dtype != a.dtype:
            raise ValueError(f"omega dtype {omega.dtype} differs from a's {a.dtype}")
        om = colmajor(omega)
    r = rsvd_colmajor(colmajor(a), m, n, opts, index_base=index_base, omega_store=om)
    return dict(u=from_colmajor(r["u"]), s=r["s"], v=from_colmajor(r["v"]))


def batch_rsvd(batch, opts, *, threads=1, device=None, devices=None):
    """Per-entry :func:`rsvd` with per-entry seeds ``opts.seed ^ index`` (rsvd.py:79-86).
    ``devices`` shards the batch over several GPUs; every entry keeps its global index, so the
    sketches (and results) do not depend on the split."""
    del threads
    devs = resolve_devices(device, devices)
    entries = list(batch)
    mats, errors = [], {}
    for i, e in enumerate(entries):
        try:
            a = as_matrix_view(e)
            _check_width(a.shape[0], a.shape[1], opts)
            mats.append(a)
        except Exception as exc:  # noqa: BLE001
            errors[i] = exc
            mats.append(None)
    if errors:
        i = min(errors)
        raise BatchError(i, errors[i]) from errors[i]
    out = [None] * len(mats)
    # contiguous runs of equal shape keep index_base arithmetic exact (seed ^ global index)
    i = 0
    while i < len(mats):
        j = i
        while j + 1 < len(mats) and mats[j + 1].shape == mats[i].shape and mats[j + 1].dtype == mats[i].dtype:
            j += 1
        m, n = mats[i].shape
        run0 = i

        def launch(store, dev, off):
            return rsvd_colmajor(store, m, n, opts, index_base=run0 + off)

        for piece, h in run_sharded(mats, list(range(i, j + 1)), devs, launch):
            for jj, t in enumerate(piece):
                out[t] = TruncatedSvd(u=np.asfortranarray(h["u"][jj].T), s=h["s"][jj].copy(),
                                      v=np.asfortranarray(h["v"][jj].T))
        i = j + 1
    return out


def rsvd(a, opts, *, device=None):
    """Randomized SVD capturing the top k (+p oversampled) triplets of a (rsvd.py:56-76)."""
    try:
        return batch_rsvd([a], opts, device=device)[0]
    except Exception as exc:
        cause = getattr(exc, "cause", None)
        if cause is not None:
            raise cause from None
        raise
