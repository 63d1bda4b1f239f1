"""Batched one-sided Jacobi SVD (reference: /root/reference/pkg/src/batchfact/jacobi.py).

Same options (``JacobiOptions``, jacobi.py:30-48), result (``SvdResult``, :51-57),
orderings (serial / round_robin, :27) and semantics (skip rule :134/:167, sweep
until a rotation-free sweep :270-281, off-orthogonality fallback :282-283,
stable descending sort and zero-column completion :189-228). Computation runs in
``bf_svd_batched_*``: the register tier (warp per matrix, n <= 32) or the
shared-memory tier (CTA per matrix), chosen by ``tier`` ("auto" by default).
"""

from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from .helpers import jacobi_rotation, off_orthogonality  # noqa: F401  (reference re-exports, on the device)
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

DEFAULT_TOLERANCE = {
    np.dtype(np.float64): 1e-14,
    np.dtype(np.float32): 1e-6,
}

_ORDERINGS = ("serial", "round_robin")
_TIERS = ("auto", "register", "shared")


@dataclass
class JacobiOptions:
    tolerance: Optional[float] = None  # None picks the per-dtype default
    max_sweeps: int = 30
    ordering: str = "serial"
    accumulate_v: bool = False
    tier: str = "auto"  # extension: which memory tier runs the sweeps

    def __post_init__(self):
        if self.tolerance is not None and not self.tolerance > 0:
            raise ValueError("tolerance must be positive")
        if self.max_sweeps < 1:
            raise ValueError("max_sweeps must be >= 1")
        if self.ordering not in _ORDERINGS:
            raise ValueError(f"ordering must be one of {_ORDERINGS}")
        if self.tier not in _TIERS:
            raise ValueError(f"tier must be one of {_TIERS}")

    def resolve_tolerance(self, dtype):
        if self.tolerance is not None:
            return float(self.tolerance)
        return DEFAULT_TOLERANCE[np.dtype(dtype)]

    def to_c(self, dtype):
        return _lib.JacobiOptsC(
            self.resolve_tolerance(dtype),
            int(self.max_sweeps),
            _ORDERINGS.index(self.ordering),
            1 if self.accumulate_v else 0,
            _TIERS.index(self.tier),
        )


@dataclass
class SvdResult:
    u: np.ndarray
    sigma: np.ndarray
    v: Optional[np.ndarray] = None
    converged: bool = True
    sweeps: int = 0


@dataclass
class PairSchedule:
    """(n-1)-step round-robin pairing of n columns, each step a perfect matching."""

    n: int
    steps: list


def round_robin_schedule(n):
    """Circle-method schedule (jacobi.py:102-115); the device kernels evaluate the same
    schedule in closed form (csrc/common.cuh rr_pair)."""
    if n < 2 or n % 2 != 0:
        raise ValueError(f"round-robin schedule needs even n >= 2, got {n}")
    steps = []
    last = n - 1
    for t in range(n - 1):
        # position 0 is fixed; positions 1..n-1 rotate one slot per step
        pos = [0] + [1 + ((j - 1 - t) % last) for j in range(1, n)]
        steps.append([tuple(sorted((pos[i], pos[n - 1 - i]))) for i in range(n // 2)])
    return PairSchedule(n=n, steps=steps)


def _validate(a):
    m, n = a.shape
    if m < n:
        raise ValueError(f"svd requires m >= n, got {m} x {n}; pass the transpose")


def svd_colmajor(store, m, n, opts, *, rotations=False):
    """Core call on column-major storage (B, n, m). Returns device tensors."""
    L = _lib.load()
    dev = store.device
    B = store.shape[0]
    es = store.element_size()
    npdt = np.float64 if es == 8 else np.float32
    copts = opts.to_c(npdt)
    u = torch.empty((B, n, m), dtype=store.dtype, device=dev)
    s = torch.empty((B, n), dtype=store.dtype, device=dev)
    v = torch.empty((B, n, n), dtype=store.dtype, device=dev) if opts.accumulate_v else None
    sweeps = torch.empty(B, dtype=torch.int32, device=dev)
    conv = torch.empty(B, dtype=torch.uint8, device=dev)
    rots = torch.empty(B, dtype=torch.int64, device=dev) if rotations else None
    with torch.cuda.device(dev):  # sizes depend on the device (occupancy, SM count)
        nbytes = L.bf_svd_workspace_size(B, m, n, es, copts)
    ws, wsb = workspace(nbytes, dev)
    fn = L.bf_svd_batched_f64 if es == 8 else L.bf_svd_batched_f32
    with torch.cuda.device(dev):
        rc = fn(B, m, n, ptr(store), ptr(u), ptr(s), ptr(v), ptr(sweeps), ptr(conv), ptr(rots), copts, ptr(ws), wsb,
                stream_handle(dev))
    _lib.check(rc, "svd")
    return dict(u=u, s=s, v=v, sweeps=sweeps, converged=conv, rotations=rots)


def svd_tensor(a, opts=None, *, rotations=False):
    """Tensor-native batched SVD: a (B, m, n) CUDA tensor.

    Returns a dict of device tensors: u (B, m, n), sigma (B, n), v (B, n, n) or None,
    sweeps (B,), converged (B,) bool, rotations (B,) or None.
    """
    opts = opts or JacobiOptions()
    check_batched_tensor(a, "svd_tensor")
    B, m, n = a.shape
    _validate(np.empty((m, n)))
    r = svd_colmajor(colmajor(a), m, n, opts, rotations=rotations)
    return dict(
        u=from_colmajor(r["u"]),
        sigma=r["s"],
        v=None if r["v"] is None else from_colmajor(r["v"]),
        sweeps=r["sweeps"],
        converged=r["converged"].bool(),
        rotations=r["rotations"],
    )


def batch_svd(batch, opts=None, *, threads=1, device=None, devices=None):
    """Per-entry :func:`svd` over a batch (jacobi.py:287-290); flags ride on each result.
    ``devices``: shard the batch over several GPUs (contiguous pieces, one call per device)."""
    del threads
    opts = opts or JacobiOptions()
    devs = resolve_devices(device, devices)
    groups, mats = group_entries(batch, _validate)
    out = [None] * len(mats)
    for (m, n, _), idx in groups.items():
        def launch(store, dev, off):
            r = svd_colmajor(store, m, n, opts)
            return {"u": r["u"], "s": r["s"], "v": r["v"], "sweeps": r["sweeps"], "conv": r["converged"]}

        for piece, h in run_sharded(mats, idx, devs, launch):
            for j, i in enumerate(piece):
                # per-entry views of the (G, n, m) host arrays: column-major (m, n), no copies
                out[i] = SvdResult(
                    u=h["u"][j].T,
                    sigma=h["s"][j],
                    v=None if h["v"] is None else h["v"][j].T,
                    converged=bool(h["conv"][j]),
                    sweeps=int(h["sweeps"][j]),
                )
    return out


def svd(a, opts=None, *, device=None):
    """One-sided Jacobi SVD of one m x n matrix, m >= n (jacobi.py:231-284)."""
    try:
        return batch_svd([a], opts, device=device)[0]
    except Exception as exc:
        cause = getattr(exc, "cause", None)
        if cause is not None:
            raise cause from None
        raise
