"""Batched one-sided block Jacobi SVD (reference: /root/reference/pkg/src/batchfact/blockjacobi.py).

Options (``BlockJacobiOptions``, blockjacobi.py:27-48, default method "direct"),
result (``BlockSvdResult`` with ``e_history``, :51-54) and semantics (round-robin
block-pair order, e computed before the update with pairs at e <= tol skipped,
per-matrix convergence, padding dropped after the sort, :84-168). Computation:
``bf_block_svd_batched_*`` (csrc/block_kernels.cu).
"""

from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch

from .helpers import scaled_offdiag  # noqa: F401  (reference re-exports, on the device)
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
from .jacobi import SvdResult

BLOCK_DEFAULT_TOLERANCE = {
    np.dtype(np.float64): 1e-13,
    np.dtype(np.float32): 1e-5,
}

_METHODS = ("gram", "direct")


@dataclass
class BlockJacobiOptions:
    block_width: int = 32
    method: str = "direct"
    tolerance: Optional[float] = None  # None picks the per-dtype default
    max_sweeps: int = 30
    accumulate_v: bool = False

    def __post_init__(self):
        if self.block_width < 1:
            raise ValueError("block_width must be >= 1")
        if self.method not in _METHODS:
            raise ValueError(f"method must be one of {_METHODS}")
        if self.tolerance is not None and not self.tolerance > 0:
            raise ValueError("tolerance must be positive")
        if self.max_sweeps < 1:
            raise ValueError("max_sweeps must be >= 1")

    def resolve_tolerance(self, dtype):
        if self.tolerance is not None:
            return float(self.tolerance)
        return BLOCK_DEFAULT_TOLERANCE[np.dtype(dtype)]

    def to_c(self, dtype):
        return _lib.BlockOptsC(
            self.resolve_tolerance(dtype),
            int(self.block_width),
            _METHODS.index(self.method),
            int(self.max_sweeps),
            1 if self.accumulate_v else 0,
        )


@dataclass
class BlockSvdResult(SvdResult):
    # max scaled off-diagonal seen in each sweep, for convergence profiling
    e_history: list = field(default_factory=list)


def _validate(a):
    m, n = a.shape
    if m < n:
        raise ValueError(f"block_svd requires m >= n, got {m} x {n}")


def block_svd_colmajor(store, m, n, opts, *, stats=False):
    """One C-ABI call on column-major storage (B, n, m). stats=True also returns the per-matrix
    work counters (B, 4): pair visits, rotated pairs, inner-SVD pair visits, inner rotations."""
    L = _lib.load()
    dev = store.device
    B = store.shape[0]
    es = store.element_size()
    npdt = np.float64 if es == 8 else np.float32
    copts = opts.to_c(npdt)
    u = torch.empty((B, n, m), dtype=store.dtype, device=dev)
    s = torch.empty((B, n), dtype=store.dtype, device=dev)
    v = torch.empty((B, n, n), dtype=store.dtype, device=dev) if opts.accumulate_v else None
    eh = torch.zeros((B, opts.max_sweeps), dtype=store.dtype, device=dev)
    sweeps = torch.empty(B, dtype=torch.int32, device=dev)
    conv = torch.empty(B, dtype=torch.uint8, device=dev)
    with torch.cuda.device(dev):  # sizes depend on the device (occupancy, SM count)
        nbytes = L.bf_block_svd_workspace_size(B, m, n, es, copts)
    ws, wsb = workspace(nbytes, dev)
    st = torch.zeros((B, 4), dtype=torch.int64, device=dev) if stats else None
    fn = L.bf_block_svd_batched_ex_f64 if es == 8 else L.bf_block_svd_batched_ex_f32
    with torch.cuda.device(dev):
        rc = fn(B, m, n, ptr(store), ptr(u), ptr(s), ptr(v), ptr(sweeps), ptr(conv), ptr(eh), ptr(st), copts,
                ptr(ws), wsb, stream_handle(dev))
    _lib.check(rc, "block_svd")
    return dict(u=u, s=s, v=v, sweeps=sweeps, converged=conv, e_history=eh, stats=st)


def block_svd_tensor(a, opts=None, *, stats=False):
    """Tensor-native batched block Jacobi SVD of a (B, m, n) CUDA tensor (stats: see
    :func:`block_svd_colmajor`)."""
    opts = opts or BlockJacobiOptions()
    check_batched_tensor(a, "block_svd_tensor")
    B, m, n = a.shape
    _validate(np.empty((m, n)))
    r = block_svd_colmajor(colmajor(a), m, n, opts, stats=stats)
    return dict(
        u=from_colmajor(r["u"]),
        sigma=r["s"],
        v=None if r["v"] is None else from_colmajor(r["v"]),
        sweeps=r["sweeps"],
        converged=r["converged"].bool(),
        e_history=r["e_history"],
        stats=r["stats"],
    )


def batch_block_svd(batch, opts=None, *, threads=1, device=None, devices=None):
    """Per-entry :func:`block_svd` (blockjacobi.py:171-174); converged entries simply stop.
    ``devices`` shards the batch over several GPUs."""
    del threads
    opts = opts or BlockJacobiOptions()
    devs = resolve_devices(device, devices)
    groups, mats = group_entries(batch, _validate)
    out = [None] * len(mats)
    for (m, n, _), idx in groups.items():
        def launch(store, dev, off):
            r = block_svd_colmajor(store, m, n, opts)
            return {"u": r["u"], "s": r["s"], "v": r["v"], "sweeps": r["sweeps"], "conv": r["converged"],
                    "eh": r["e_history"]}

        for piece, h in run_sharded(mats, idx, devs, launch):
            for j, i in enumerate(piece):
                sw = int(h["sweeps"][j])
                out[i] = BlockSvdResult(
                    u=np.asfortranarray(h["u"][j].T),
                    sigma=h["s"][j].copy(),
                    v=None if h["v"] is None else np.asfortranarray(h["v"][j].T),
                    converged=bool(h["conv"][j]),
                    sweeps=sw,
                    e_history=[float(x) for x in h["eh"][j, :sw]],
                )
    return out


def block_svd(a, opts=None, *, device=None):
    """One-sided block Jacobi SVD of one m x n matrix, m >= n (blockjacobi.py:84-168)."""
    try:
        return batch_block_svd([a], opts, device=device)[0]
    except Exception as exc:
        cause = getattr(exc, "cause", None)
        if cause is not None:
            raise cause from None
        raise
