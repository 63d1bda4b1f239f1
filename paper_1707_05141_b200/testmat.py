"""Device-side prescribed-spectrum inputs (harness utility; testmat.py:83-94).

The reference's testmat is an input generator, not hot path; the bench uses this to
build config-5 style H-matrix blocks on the GPU instead of on the host.
"""

import torch

from . import _lib
from .core import from_colmajor, ptr, resolve_device, stream_handle, workspace
from .rsvd import split_seed

_MODES = ("geometric", "arithmetic")


def make_matrix_tensor(batch, m, n, cond, rank=None, seed=0, *, mode="geometric", index_base=0, device=None):
    """(batch, m, n) float64 CUDA tensor: entry b = P diag(sigma) Q^T with seed + index_base + b,
    plus the (n,) sigma vector (testmat.py:51-94)."""
    if mode not in _MODES:
        raise ValueError(f"mode must be one of {_MODES}")
    rank = n if rank is None else rank
    L = _lib.load()
    dev = resolve_device(device)
    lo, hi = split_seed(seed)
    a = torch.empty((batch, n, m), dtype=torch.float64, device=dev)
    sig = torch.empty(n, dtype=torch.float64, device=dev)
    with torch.cuda.device(dev):  # sizes depend on the device (occupancy, SM count)
        nbytes = L.bf_make_matrix_workspace_size(batch, m, n)
    ws, wsb = workspace(nbytes, dev)
    with torch.cuda.device(dev):
        rc = L.bf_make_matrix_batched_f64(batch, m, n, _MODES.index(mode), float(cond), int(rank), lo, hi,
                                          int(index_base), ptr(a), ptr(sig), ptr(ws), wsb, stream_handle(dev))
    _lib.check(rc, "make_matrix")
    return from_colmajor(a), sig
