"""Host-side plumbing: the reference's batch conventions over device tensors.

Mirrors /root/reference/pkg/src/batchfact/core.py:
  * ``BatchError(index, cause)`` -- lowest failing entry (core.py:17-23, :120-122);
  * ``as_matrix`` -- 2-d check, non-f32/f64 cast to f64, column-major (core.py:26-33).
The reference's ``batch_apply`` (core.py:97-123) runs one Python call per entry; here a
homogeneous group of entries becomes ONE C-ABI call. Torch is used only for device
memory, streams and copies (pinned host staging); no compute happens in torch.
"""

import os

import numpy as np
import torch

from . import _lib

REAL_DTYPES = (np.float32, np.float64)


class BatchError(Exception):
    """Failure of a per-entry operation inside a batch, tagged with the index."""

    def __init__(self, index, cause):
        super().__init__(f"batch entry {index}: {cause}")
        self.index = index
        self.cause = cause


def as_matrix(a, dtype=None):
    """Coerce ``a`` to a 2-d column-major float array (core.py:26-33)."""
    return np.asfortranarray(as_matrix_view(a, dtype))


def as_matrix_view(a, dtype=None):
    """as_matrix's checks and dtype coercion without the Fortran copy: the batched entry points
    only read their inputs (staged straight into pinned memory by stack_to_device), so the
    reference's defensive copy (core.py:26-33) would be a second pass over every entry."""
    a = np.asarray(a, dtype=dtype)
    if a.ndim != 2:
        raise ValueError(f"expected a 2-d array, got ndim={a.ndim}")
    if a.dtype.type not in REAL_DTYPES:
        a = a.astype(np.float64)
    return a


def write_matrix_text(path, a):
    """Matrix text format of core.py:126-134 (re-exported from cli.py)."""
    from .cli import write_matrix_text as _w

    return _w(path, a)


def read_matrix_text(path, dtype=np.float64):
    """Matrix text format of core.py:137-147 (re-exported from cli.py)."""
    from .cli import read_matrix_text as _r

    return _r(path, dtype)


def syrk(a, *, device=None):
    """core.py:68-78 on the device (paper_1707_05141_b200.helpers)."""
    from .helpers import syrk as _f

    return _f(a, device=device)


def gemm(a, b, c=None, *, alpha=1.0, beta=0.0, trans_a=False, trans_b=False, device=None):
    """core.py:36-65 on the device (paper_1707_05141_b200.helpers)."""
    from .helpers import gemm as _f

    return _f(a, b, c, alpha=alpha, beta=beta, trans_a=trans_a, trans_b=trans_b, device=device)


def frobenius(a, *, device=None):
    """core.py:81-86 on the device (paper_1707_05141_b200.helpers)."""
    from .helpers import frobenius as _f

    return _f(a, device=device)


def batch_apply(entries, op, *, threads=1):
    """core.py:97-123 (paper_1707_05141_b200.helpers)."""
    from .helpers import batch_apply as _f

    return _f(entries, op, threads=threads)


def resolve_device(device=None):
    if not torch.cuda.is_available():
        raise _lib.BackendUnavailable("no CUDA device visible; batchfact_b200 has no CPU fallback")
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    device = torch.device(device)
    if device.type != "cuda":
        raise ValueError("batchfact_b200 runs on CUDA devices only")
    if device.index is None:
        device = torch.device("cuda", torch.cuda.current_device())
    return device


def resolve_devices(device=None, devices=None):
    """The devices of a drop-in call: ``devices`` (the batch is sharded over them, SURVEY §8b
    "devices= selects GPUs for sharding") or the single ``device``."""
    if devices is None:
        return [resolve_device(device)]
    if device is not None:
        raise ValueError("pass device or devices, not both")
    devs = [resolve_device(d) for d in devices]
    if not devs:
        raise ValueError("devices must name at least one CUDA device")
    return devs


def split_contiguous(idx, parts):
    """Cut an index list into ``parts`` contiguous pieces (the ShardPlan split: the first
    len % parts pieces one longer); returns [(offset_in_idx, piece)], empty pieces dropped."""
    n = len(idx)
    base, extra = divmod(n, parts)
    out, start = [], 0
    for r in range(parts):
        cnt = base + (1 if r < extra else 0)
        if cnt:
            out.append((start, idx[start:start + cnt]))
        start += cnt
    return out


PIPELINE_MIN_ENTRIES = 1024  # drop-in groups at least this large use the overlapped host pipeline
# drop-in pipeline depth (host-staging bound; measured on cfg3's 5 000 entries: 8 chunks 25 ms,
# 6 -> 31 ms, 10 -> 26 ms, 12 -> 33 ms)
PIPELINE_CHUNKS = int(os.environ.get("BF_DROPIN_CHUNKS", "8"))


def run_sharded(mats, idx, devs, launch):
    """One batched call per device over contiguous pieces of ``idx``: every piece is staged and
    launched first (the devices run concurrently; launches are asynchronous), then each piece's
    outputs are brought to the host. launch(store, device, offset) -> dict of device tensors
    (None allowed); offset = the piece's position in ``idx`` (rsvd's global seed index).
    Returns [(piece, {name: numpy or None})]. Results do not depend on the split (core.py:97-103).
    One device and a large group: the chunked host pipeline (stream.run_entries_pipelined), which
    overlaps host staging, both copies and the kernels."""
    if len(devs) == 1 and len(idx) >= PIPELINE_MIN_ENTRIES:
        from .stream import run_entries_pipelined

        return [(list(idx), run_entries_pipelined(mats, idx, devs[0], launch, chunks=PIPELINE_CHUNKS))]
    pending = []
    for k, (off, piece) in enumerate(split_contiguous(idx, len(devs))):
        dev = devs[k]
        with torch.cuda.device(dev):
            store = stack_to_device(mats, piece, dev)
            pending.append((piece, launch(store, dev, off)))
    done = []
    for piece, out in pending:
        done.append((piece, {k: (None if v is None else to_host(v)) for k, v in out.items()}))
    return done


def stream_handle(device):
    return torch.cuda.current_stream(device).cuda_stream


def ptr(t):
    return None if t is None else t.data_ptr()


def workspace(nbytes, device):
    if nbytes == 0:
        return None, 0
    return torch.empty(int(nbytes), dtype=torch.uint8, device=device), int(nbytes)


def colmajor(t):
    """(B, m, n) tensor -> (B, n, m) contiguous storage == per-matrix column-major."""
    return t.transpose(-1, -2).contiguous()


def from_colmajor(store):
    """(B, cols, rows) contiguous storage -> (B, rows, cols) view (column-major strides)."""
    return store.transpose(-1, -2)


def torch_dtype(np_dtype):
    return torch.float64 if np.dtype(np_dtype) == np.float64 else torch.float32


def check_batched_tensor(a, what):
    if not isinstance(a, torch.Tensor):
        raise TypeError(f"{what}: expected a torch.Tensor")
    if a.dim() != 3:
        raise ValueError(f"{what}: expected a (batch, m, n) tensor, got shape {tuple(a.shape)}")
    if a.dtype not in (torch.float32, torch.float64):
        raise ValueError(f"{what}: dtype must be float32 or float64")
    if a.device.type != "cuda":
        raise ValueError(f"{what}: tensor must live on a CUDA device")


def group_entries(entries, validate):
    """Coerce entries, validate each (reference error semantics), group by (shape, dtype).

    Returns {(m, n, dtype): [indices]} and the coerced list. Raises BatchError for the
    lowest failing index before any launch (the reference raises it after running the
    batch, with identical outcome, core.py:104-123).
    """
    mats = []
    errors = {}
    for i, e in enumerate(entries):
        try:
            a = as_matrix_view(e)
            validate(a)
            mats.append(a)
        except Exception as exc:  # noqa: BLE001 - reported with the batch index
            errors[i] = exc
            mats.append(None)
    if errors:
        i = min(errors)
        raise BatchError(i, errors[i]) from errors[i]
    groups = {}
    for i, a in enumerate(mats):
        groups.setdefault((a.shape[0], a.shape[1], a.dtype.str), []).append(i)
    return groups, mats


def stack_to_device(mats, idx, device):
    """Stack entries into pinned host memory and copy to the device as column-major storage
    (G, n, m). Fortran-ordered entries are stacked as they lie (one memcpy each, inside one numpy
    call); C-ordered ones (numpy's default) are stacked row-major and transposed ON THE DEVICE,
    so no entry is transposed by the host."""
    sel = [mats[i] for i in idx]
    m, n = sel[0].shape
    dt = torch_dtype(sel[0].dtype)
    if all(a.flags.f_contiguous for a in sel):
        host = torch.empty((len(sel), n, m), dtype=dt, pin_memory=True)
        np.stack([a.T for a in sel], out=host.numpy())
        return host.to(device, non_blocking=True)
    if all(a.flags.c_contiguous for a in sel):
        host = torch.empty((len(sel), m, n), dtype=dt, pin_memory=True)
        np.stack(sel, out=host.numpy())
        return host.to(device, non_blocking=True).transpose(1, 2).contiguous()
    host = torch.empty((len(sel), n, m), dtype=dt, pin_memory=True)
    hv = host.numpy()
    for j, a in enumerate(sel):
        hv[j] = a.T
    return host.to(device, non_blocking=True)


def to_host(t):
    """Device tensor -> numpy (synchronising copy through pinned memory)."""
    host = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    host.copy_(t, non_blocking=True)
    torch.cuda.current_stream(t.device).synchronize()
    return host.numpy()
