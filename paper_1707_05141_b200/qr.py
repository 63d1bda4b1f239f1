"""Batched Householder QR (reference: /root/reference/pkg/src/batchfact/qr.py).

``batch_qr`` (qr.py:98-100) and ``qr`` (qr.py:63-95) keep the reference's names,
arguments, dataclass and errors; the factorisation itself runs in
``bf_qr_batched_*`` (csrc/qr_kernels.cu) -- one launch per homogeneous group.
"""

from dataclasses import dataclass

import numpy as np
import torch

from .helpers import householder_vector  # noqa: F401  (reference re-exports, on the device)
from . import _lib
from .core import (
    check_batched_tensor,
    colmajor,
    from_colmajor,
    group_entries,
    ptr,
    resolve_devices,
    run_sharded,
    stream_handle,
    workspace,
)

DEFAULT_PANEL_WIDTH = 16


@dataclass
class QrResult:
    q: np.ndarray  # m x n, orthonormal columns
    r: np.ndarray  # n x n, upper triangular with exact zeros below


def _validate(panel_width):
    def v(a):
        m, n = a.shape
        if m < n:
            raise ValueError(f"qr requires m >= n, got {m} x {n}; pass the transpose")
        if panel_width < 1:
            raise ValueError("panel_width must be >= 1")

    return v


def qr_colmajor(store, m, n, panel_width=DEFAULT_PANEL_WIDTH):
    """Core call on column-major storage (B, n, m) -> (q_store (B, n, m), r_store (B, n, n))."""
    L = _lib.load()
    dev = store.device
    B = store.shape[0]
    es = store.element_size()
    q = torch.empty((B, n, m), dtype=store.dtype, device=dev)
    r = torch.empty((B, n, n), dtype=store.dtype, device=dev)
    with torch.cuda.device(dev):  # sizes depend on the device (occupancy, SM count)
        nbytes = L.bf_qr_workspace_size(B, m, n, es)
    ws, wsb = workspace(nbytes, dev)
    fn = L.bf_qr_batched_f64 if es == 8 else L.bf_qr_batched_f32
    with torch.cuda.device(dev):
        rc = fn(B, m, n, ptr(store), ptr(q), ptr(r), int(panel_width), ptr(ws), wsb, stream_handle(dev))
    _lib.check(rc, "qr")
    return q, r


def qr_tensor(a, panel_width=DEFAULT_PANEL_WIDTH):
    """Tensor-native batched QR: a (B, m, n) CUDA tensor -> (Q (B, m, n), R (B, n, n))."""
    check_batched_tensor(a, "qr_tensor")
    B, m, n = a.shape
    _validate(panel_width)(np.empty((m, n)))
    q, r = qr_colmajor(colmajor(a), m, n, panel_width)
    return from_colmajor(q), from_colmajor(r)


def batch_qr(batch, panel_width=DEFAULT_PANEL_WIDTH, *, threads=1, device=None, devices=None):
    """Per-entry :func:`qr` over a batch (qr.py:98-100). ``threads`` is accepted and ignored;
    ``devices`` shards the batch over several GPUs."""
    del threads
    devs = resolve_devices(device, devices)
    groups, mats = group_entries(batch, _validate(panel_width))
    out = [None] * len(mats)
    for (m, n, _), idx in groups.items():
        def launch(store, dev, off):
            q, r = qr_colmajor(store, m, n, panel_width)
            return {"q": q, "r": r}

        for piece, h in run_sharded(mats, idx, devs, launch):
            for j, i in enumerate(piece):
                out[i] = QrResult(q=np.asfortranarray(h["q"][j].T), r=np.asfortranarray(h["r"][j].T))
    return out


def qr(a, panel_width=DEFAULT_PANEL_WIDTH, *, device=None):
    """Reduced QR of one m x n matrix, m >= n (qr.py:63-95)."""
    try:
        return batch_qr([a], panel_width, device=device)[0]
    except Exception as exc:  # surface the reference's per-op error, not the batch wrapper
        cause = getattr(exc, "cause", None)
        if cause is not None:
            raise cause from None
        raise
