"""Multi-rank host logic of the batch sharding (paper_1707_05141_b200/shard.py), world size 2
over gloo on CPU. The per-shard op here is the CPU ORACLE (test infrastructure) standing in
for the device call: what is under test is the split, the global index_base (rsvd's
seed ^ i, rsvd.py:82-85) and the gather -- shard-invariance of every entry's result.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as orc
from paper_1707_05141_b200.shard import ShardPlan, gather_results, local_slice, run_shard


def test_plan_bounds_cover_batch_exactly():
    for batch in (0, 1, 2, 7, 125, 1000, 10_001):
        for world in (1, 2, 3, 8):
            spans = [ShardPlan(batch, world, r).bounds() for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == batch
            for (s0, e0), (s1, _) in zip(spans, spans[1:]):
                assert e0 == s1
            counts = ShardPlan(batch, world, 0).counts
            assert max(counts) - min(counts) <= 1 and sum(counts) == batch


def test_plan_rejects_bad_rank():
    with pytest.raises(ValueError):
        ShardPlan(10, 2, 2)
    with pytest.raises(ValueError):
        ShardPlan(-1, 1, 0)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_svd_op(m, n):
    def op(store, index_base):
        a3 = store.numpy()
        r = orc.batch_svd_stacked(a3, m, n, ordering="round_robin", accumulate_v=True)
        return dict(s=torch.from_numpy(np.ascontiguousarray(r["s"])),
                    sweeps=torch.from_numpy(np.ascontiguousarray(r["sweeps"]).astype(np.int32)),
                    converged=torch.from_numpy(np.ascontiguousarray(r["converged"]).astype(bool)))
    return op


def _oracle_rsvd_op(m, n, k, p, seed):
    def op(store, index_base):
        r = orc.batch_rsvd_stacked(store.numpy(), m, n, k, p, seed=seed, index_base=index_base)
        return dict(s=torch.from_numpy(np.ascontiguousarray(r["s"])))
    return op


def _worker(rank, world, port, batch, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(1234)
        a_svd = torch.from_numpy(rng.standard_normal((batch, 12, 16)))  # (B, n, m) column-major storage
        a_rsvd = torch.from_numpy(rng.standard_normal((batch, 24, 24)))
        plan = ShardPlan(batch, world, rank)
        r1 = gather_results(run_shard(_oracle_svd_op(16, 12), local_slice(a_svd, plan), plan), plan)
        r2 = gather_results(run_shard(_oracle_rsvd_op(24, 24, 4, 2, 7), local_slice(a_rsvd, plan), plan), plan)
        if rank == 0:
            out_q.put({k: v.numpy() for k, v in {**r1, "rsvd_s": r2["s"]}.items()})
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("batch", [7, 1])
def test_gloo_world2_shard_invariance(batch):
    orc.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, batch, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single-process reference: the same global batch in one call
    rng = np.random.default_rng(1234)
    a_svd = rng.standard_normal((batch, 12, 16))
    a_rsvd = rng.standard_normal((batch, 24, 24))
    r = orc.batch_svd_stacked(a_svd, 16, 12, ordering="round_robin", accumulate_v=True)
    np.testing.assert_array_equal(got["s"], r["s"])
    np.testing.assert_array_equal(got["sweeps"], np.asarray(r["sweeps"]).astype(np.int32))
    np.testing.assert_array_equal(got["converged"], np.asarray(r["converged"]).astype(bool))
    rr = orc.batch_rsvd_stacked(a_rsvd, 24, 24, 4, 2, seed=7, index_base=0)
    np.testing.assert_array_equal(got["rsvd_s"], rr["s"])


def test_bench_launcher_spawns_ranks_and_results_are_shard_invariant():
    """`python bench.py --gpus 2` without torchrun re-launches itself under torch.distributed.run
    with 2 ranks (the driver's form); --selftest runs the sharded path over gloo on CPU and checks
    the gathered results against a single-rank run bit for bit."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--selftest"],
                         capture_output=True, text=True, timeout=240, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["selftest"] == "ok" and line["world"] == 2 and line["backend"] == "gloo"
    assert "torch.distributed.run" in line["launcher"]
    for c in line["checks"].values():
        assert c["bitwise_equal"] and len(c["shard_counts"]) == 2
