"""Batch sharding over ranks: one process per GPU, no collective on the data path.

The reference has no multi-device story: its only parallelism is ``batch_apply``'s
thread pool over independent entries (/root/reference/pkg/src/batchfact/core.py:97-123),
whose contract is that each entry's result is independent of how the batch is split
(core.py:97-103). Sharding keeps that contract across GPUs:

  * a global batch of ``batch`` entries is cut into ``world`` contiguous shards; rank r owns
    entries [start, stop) -- the first ``batch % world`` ranks take one extra entry;
  * each rank runs ONE batched C-ABI call on its shard, on its own device and stream;
  * the only place the global position of an entry matters is rsvd's per-entry seed
    ``seed ^ i`` (rsvd.py:82-85): the shard passes ``index_base = start`` so every entry
    draws the same sketch as in a single-device run (shard-invariant results);
  * the optional final gather (``gather_results``) is the only collective: per-rank
    results padded to the largest shard and exchanged with one all_gather per output
    (NCCL over NVLink on the GPU box, gloo in the CPU tests).

The per-shard operation is a callable ``op(local_store, index_base) -> dict of tensors``
(see :func:`svd_op`, :func:`qr_op`, :func:`block_svd_op`, :func:`rsvd_op`), so the host
logic here is independent of the device code and is tested on CPU with gloo.
"""

from dataclasses import dataclass

import torch


@dataclass(frozen=True)
class ShardPlan:
    """Contiguous split of a global batch over ``world`` ranks."""

    batch: int
    world: int
    rank: int

    def __post_init__(self):
        if self.batch < 0:
            raise ValueError("batch must be >= 0")
        if self.world < 1 or not 0 <= self.rank < self.world:
            raise ValueError(f"rank {self.rank} outside world of {self.world}")

    def bounds(self, rank=None):
        r = self.rank if rank is None else rank
        base, extra = divmod(self.batch, self.world)
        start = r * base + min(r, extra)
        return start, start + base + (1 if r < extra else 0)

    @property
    def start(self):
        return self.bounds()[0]

    @property
    def stop(self):
        return self.bounds()[1]

    @property
    def count(self):
        s, e = self.bounds()
        return e - s

    @property
    def counts(self):
        return [self.bounds(r)[1] - self.bounds(r)[0] for r in range(self.world)]

    @property
    def max_count(self):
        return max(self.counts)


def plan_for(batch, group=None):
    """ShardPlan of this process in ``group`` (or a single-rank plan without torch.distributed)."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        return ShardPlan(batch, dist.get_world_size(group), dist.get_rank(group))
    return ShardPlan(batch, 1, 0)


def local_slice(global_tensor, plan):
    """This rank's entries of a (batch, ...) tensor that every rank holds (e.g. host staging)."""
    if global_tensor.shape[0] != plan.batch:
        raise ValueError(f"expected a batch of {plan.batch}, got {global_tensor.shape[0]}")
    return global_tensor[plan.start:plan.stop]


def run_shard(op, local_store, plan):
    """Run the per-shard op on this rank's entries; ``index_base`` = global start index."""
    if local_store.shape[0] != plan.count:
        raise ValueError(f"rank {plan.rank} owns {plan.count} entries, got {local_store.shape[0]}")
    return op(local_store, plan.start)


def gather_results(result, plan, group=None, keys=None):
    """All-gather per-rank result tensors into global-batch tensors (entry order preserved).

    ``result``: dict name -> tensor whose leading dim is this rank's count (None entries are
    passed through). Shards are padded to ``plan.max_count`` so one equal-size all_gather per
    output suffices. Returns dict name -> (batch, ...) tensor, identical on every rank.
    """
    import torch.distributed as dist

    if plan.world == 1:
        return dict(result)
    out = {}
    for name in keys or list(result):
        t = result[name]
        if t is None:
            out[name] = None
            continue
        if t.shape[0] != plan.count:
            raise ValueError(f"{name}: leading dim {t.shape[0]} != shard size {plan.count}")
        wire = t.view(torch.uint8) if t.dtype == torch.bool else t
        pad = torch.zeros((plan.max_count,) + tuple(wire.shape[1:]), dtype=wire.dtype, device=wire.device)
        pad[: plan.count] = wire
        parts = [torch.empty_like(pad) for _ in range(plan.world)]
        dist.all_gather(parts, pad.contiguous(), group=group)
        full = torch.cat([p[:c] for p, c in zip(parts, plan.counts)], dim=0)
        out[name] = full.view(torch.bool) if t.dtype == torch.bool else full
    return out


# ------------------------------------------------------------------ device ops (one C-ABI call each)


def svd_op(m, n, opts, *, rotations=False):
    from .jacobi import svd_colmajor

    def op(store, index_base):
        del index_base  # Jacobi SVD is position-independent
        return svd_colmajor(store, m, n, opts, rotations=rotations)

    return op


def qr_op(m, n, panel_width=16):
    from .qr import qr_colmajor

    def op(store, index_base):
        del index_base
        q, r = qr_colmajor(store, m, n, panel_width)
        return dict(q=q, r=r)

    return op


def block_svd_op(m, n, opts):
    from .blockjacobi import block_svd_colmajor

    def op(store, index_base):
        del index_base
        return block_svd_colmajor(store, m, n, opts)

    return op


def rsvd_op(m, n, opts):
    from .rsvd import rsvd_colmajor

    def op(store, index_base):
        return rsvd_colmajor(store, m, n, opts, index_base=index_base)

    return op
