"""Benchmark: batched fp64 SVD matrices/s & GFLOP/s on B200 (BASELINE.json metric).

python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfg3|...|all]

One "step" = one pass of the hot path over the config's whole batch (synthetic inputs of
the BASELINE shape, generated on the device with the reference's Gaussian stream).
Headline workload (N=1): cfg3, 5,000 random 64x64 fp64 matrices, round-robin Jacobi with V
(the shared-memory tier). The other BASELINE configs are measured in the same run under
"configs" (fewer steps). Multi-GPU (torchrun): every rank runs its own full batch (weak
scaling, no data-path collective); time = max over ranks of the device time.

--impl reference times the CPU oracle (oracle/: the reference algorithm restated in C,
since the reference itself is pure Python and cannot travel) on all host cores, rank 0 only.
"""

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "batched fp64 SVD matrices/sec & GFLOP/s vs size at 1/2/4/8 B200 (vs CPU ref)"
UNIT = "matrices/s"
L2_FLUSH_BYTES = 256 << 20

CONFIGS = {
    "cfg1": dict(kind="svd", m=32, n=32, batch=1000, seed=1_000_000, ordering="serial",
                 desc="batched one-sided Jacobi SVD, 1,000 random 32x32 fp64 (serial ordering, V; register tier)"),
    "cfg2": dict(kind="qr", m=64, n=32, batch=10_000, seed=2_000_000,
                 desc="batched Householder QR, 10,000 random 64x32 fp64 (explicit Q)"),
    "cfg3": dict(kind="svd", m=64, n=64, batch=5000, seed=3_000_000, ordering="round_robin",
                 desc="batched shared-memory Jacobi SVD, 5,000 random 64x64 fp64 (round_robin, V)"),
    "cfg4": dict(kind="block", m=256, n=256, batch=1000, seed=4_000_000,
                 desc="batched block-Jacobi SVD (gram, bw 32, tol 1e-11, V), 1,000 random 256x256 fp64"),
    "cfg4d": dict(kind="block", method="direct", m=256, n=256, batch=1000, seed=4_000_000,
                  desc="batched block-Jacobi SVD, direct method (the reference default: pair QR, inner SVD of R, "
                       "WY apply; bw 32, tol 1e-13, V), 1,000 random 256x256 fp64"),
    "cfg5": dict(kind="rsvd", m=128, n=128, batch=10_000, seed=5_000_000, k=32, p=8,
                 desc="batched randomized SVD k=32 p=8 of 10,000 128x128 geometric-spectrum (cond 1e16, rank 64) blocks"),
}
HEADLINE = "cfg3"


def block_opts(c):
    """cfg4: Gram at tol 1e-11 (BASELINE: tensor-core Gram/rotation); cfg4d: the direct default."""
    import paper_1707_05141_b200 as bf

    if c.get("method", "gram") == "gram":
        return bf.BlockJacobiOptions(method="gram", block_width=32, tolerance=1e-11, accumulate_v=True)
    return bf.BlockJacobiOptions(method="direct", block_width=32, accumulate_v=True)


def load_profile(name):
    """Per-launch DRAM traffic of the config's dominant kernel from the committed ncu --set full
    summary (profiles/ncu_full_r01.json, written by tools/ncu_summary.py)."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "ncu_full_r01.json")))
        return d.get(name, {})
    except Exception:  # noqa: BLE001
        return {}


def load_peaks():
    peaks = {}
    try:
        peaks.update(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))))
    except Exception:  # noqa: BLE001
        peaks["hbm_gbs"] = 6650.0
        peaks["hbm_note"] = "fallback"
    try:
        fp = json.load(open(os.path.join(ROOT, "profiles", "fp64_peak_r01.json")))
        peaks["fp64_tflops"] = fp["dmma_tflops"]
        peaks["fp64_dfma_tflops"] = fp["dfma_tflops"]
    except Exception:  # noqa: BLE001
        peaks["fp64_tflops"] = 37.2
    return peaks


# ----------------------------------------------------------------- algorithmic counts


def jacobi_flops(m, n, sweeps, rotations, accv=True):
    """Paper convention: 6m per pair visit (3 dots), 6m (+6n with V) per rotation."""
    pairs = sweeps * n * (n - 1) // 2
    return 6.0 * m * pairs + (6.0 * m + (6.0 * n if accv else 0.0)) * rotations


def qr_flops(m, n):
    return 4.0 * m * n * n - 4.0 * n ** 3 / 3.0  # geqrf + orgqr


def rsvd_flops(m, n, w, inner):
    return (2.0 * m * n * w + (4.0 * m * w * w - 4.0 * w ** 3 / 3.0) + 2.0 * w * m * n
            + (4.0 * n * w * w - 4.0 * w ** 3 / 3.0) + inner + 2.0 * m * w * w + 2.0 * n * w * w)


# ----------------------------------------------------------------- clocks sampler


class ClockSampler:
    def __init__(self, index):
        self.index = index
        self.samples = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:  # noqa: BLE001
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.samples.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:  # noqa: BLE001
            self.proc.kill()
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[3 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ----------------------------------------------------------------- GPU arm


class GpuConfig:
    """Builds device-resident inputs for one config and runs its hot path once per step."""

    def __init__(self, name, cfg, device, rank, world=1):
        import torch

        from paper_1707_05141_b200.shard import ShardPlan

        import paper_1707_05141_b200 as bf
        from paper_1707_05141_b200.blockjacobi import block_svd_colmajor
        from paper_1707_05141_b200.jacobi import svd_colmajor
        from paper_1707_05141_b200.qr import qr_colmajor
        from paper_1707_05141_b200.rsvd import rsvd_colmajor

        self.k_svd, self.k_qr, self.k_block, self.k_rsvd = svd_colmajor, qr_colmajor, block_svd_colmajor, rsvd_colmajor
        self.bf, self.torch = bf, torch
        self.name, self.cfg, self.dev = name, cfg, device
        m, n, B = cfg["m"], cfg["n"], cfg["batch"]
        # weak scaling: a global batch of world*B entries, contiguous shard of B per rank
        self.plan = ShardPlan(world * B, world, rank)
        seed0 = cfg["seed"] + self.plan.start
        if cfg["kind"] == "rsvd":
            self.a, _ = bf.make_matrix_tensor(B, m, n, 1e16, rank=64, seed=cfg["seed"], index_base=self.plan.start,
                                              device=device)
        else:
            self.a = bf.gaussian_tensor(B, m, n, seed0, seed_mode="add", device=device)
        self.store = self.a.transpose(1, 2).contiguous()  # column-major storage, resident
        torch.cuda.synchronize(device)
        self.out = None

    def step(self):
        bf, c = self.bf, self.cfg
        m, n = c["m"], c["n"]
        if c["kind"] == "svd":
            opts = bf.JacobiOptions(ordering=c["ordering"], accumulate_v=True)
            self.out = self.k_svd(self.store, m, n, opts, rotations=True)
        elif c["kind"] == "qr":
            self.out = self.k_qr(self.store, m, n, 16)
        elif c["kind"] == "block":
            opts = block_opts(c)
            self.out = self.k_block(self.store, m, n, opts)
        else:
            opts = bf.RsvdOptions(k=c["k"], p=c["p"], seed=5)
            self.out = self.k_rsvd(self.store, m, n, opts, index_base=self.plan.start)  # seed ^ global index

    def kernel_name(self):
        c = self.cfg
        if c["kind"] == "svd":
            return "svd_rr_kernel + svd_rr_vkernel" if c["ordering"] == "round_robin" else "svd_reg_kernel"
        if c["kind"] == "block" and c.get("method", "gram") == "direct":
            return "bj_dqr_reg + svd_rr_kernel + svd_rr_vkernel (inner) + bj_dapply_wy + bj_rot_mma"
        return {"qr": "qr_reg_kernel", "block": "bj_gram_mma + svd_rr_kernel (inner) + bj_rot_mma",
                "rsvd": "gemm_mma_kernel + qr_reg_kernel + svd_rr_kernel + svd_rr_vkernel"}[c["kind"]]

    def launches_per_step(self):
        """Our kernels per step, as the ncu launch lists show them (profiles/launches_r01.md)."""
        c = self.cfg
        if c["kind"] == "svd":
            return 2 if c["ordering"] == "round_robin" else 1  # sweep kernel + V replay kernel
        if c["kind"] == "qr":
            return 1
        if c["kind"] == "block":
            nb = c["n"] // 32
            # init + 30 sweeps (launched unconditionally; converged entries exit at once) x (steps x
            # kernels + finalize) + extract. Gram: gram, inner svd (U only), rotation; direct: pair
            # QR, inner svd sweep + V replay, WY apply, V-pair rotation
            per = 3 if c.get("method", "gram") == "gram" else 5
            return 2 + 30 * (per * (nb - 1) + 1)
        return 10  # rsvd: gaussian, 4 DMMA gemms, 2 qr, svd sweep + V replay, sign fix

    def flops(self):
        """Algorithmic flops of the last step (counted from the run's own sweep/rotation counters)."""
        c = self.cfg
        m, n, B = c["m"], c["n"], c["batch"]
        if c["kind"] == "svd":
            sw = self.out["sweeps"].double().sum().item()
            rot = self.out["rotations"].double().sum().item()
            return jacobi_flops(m, n, sw, rot), B * 8.0 * (2 * m * n + n * n + n)
        if c["kind"] == "qr":
            return B * qr_flops(m, n), B * 8.0 * (2 * m * n + n * n)
        if c["kind"] == "block":
            # Gram'd pairs: 2m(2k)^2 each; rotations: (2m + 2n)(2k)^2; inner SVD ~ oracle nominal 1.33 GFLOP/matrix
            sw = self.out["sweeps"].double().sum().item()
            k2 = 64
            pairs = sw * 28
            f = pairs * (2.0 * m * k2 * k2 + (2.0 * m + 2.0 * n) * k2 * k2) + B * 1.33e9
            return f, B * 8.0 * (3 * m * n + n)
        w = c["k"] + c["p"]
        return B * rsvd_flops(m, n, w, 2.909e6), B * 8.0 * (m * n + m * w + n * w + w)

    def device_op(self):
        """The config's batched call as op(dev_store, index_base) -> output tensors (C-ABI call)."""
        c, bf = self.cfg, self.bf
        m, n = c["m"], c["n"]
        if c["kind"] == "svd":
            opts = bf.JacobiOptions(ordering=c["ordering"], accumulate_v=True)

            def op(x, ib):
                r = self.k_svd(x, m, n, opts)
                return [r["u"], r["s"], r["v"], r["sweeps"], r["converged"]]
        elif c["kind"] == "qr":
            def op(x, ib):
                return list(self.k_qr(x, m, n, 16))
        elif c["kind"] == "block":
            opts = block_opts(c)

            def op(x, ib):
                r = self.k_block(x, m, n, opts)
                return [r["u"], r["s"], r["v"], r["sweeps"], r["converged"]]
        else:
            opts = bf.RsvdOptions(k=c["k"], p=c["p"], seed=5)

            def op(x, ib):
                r = self.k_rsvd(x, m, n, opts, index_base=ib)
                return [r["u"], r["s"], r["v"]]
        return op

    def e2e_step(self, host_in, pinned_out, chunks):
        """Public API with HOST buffers: H2D of the inputs, the batched call, D2H of results --
        chunked so the copies overlap the kernels (paper_1707_05141_b200.stream)."""
        from paper_1707_05141_b200.stream import run_host_pipelined

        run_host_pipelined(self.device_op(), host_in, pinned_out, chunks=abs(chunks), device=self.dev,
                           index_base=self.plan.start, taper=chunks > 0)
        return sum(o.numel() * o.element_size() for o in pinned_out)


def time_gpu(gc, steps, warmup, flush):
    torch = gc.torch
    for _ in range(warmup):
        gc.step()
    torch.cuda.synchronize(gc.dev)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    for i in range(steps):
        flush.zero_()  # L2 flush outside the timed window of each step
        starts[i].record()
        gc.step()
        ends[i].record()
    torch.cuda.synchronize(gc.dev)
    return sum(s.elapsed_time(e) for s, e in zip(starts, ends)) / 1e3  # seconds


def time_e2e(gc, steps, chunks):
    torch = gc.torch
    host_in = torch.empty_like(gc.store, device="cpu").pin_memory()
    host_in.copy_(gc.store)
    outs = gc.device_op()(gc.store, gc.plan.start)
    torch.cuda.synchronize(gc.dev)
    pinned = [torch.empty(o.shape, dtype=o.dtype).pin_memory() for o in outs]
    del outs
    gc.e2e_step(host_in, pinned, chunks)  # warm-up (allocator, streams)
    t0 = time.perf_counter()
    d2h = 0
    for _ in range(steps):
        d2h = gc.e2e_step(host_in, pinned, chunks)
    dt = time.perf_counter() - t0
    h2d = host_in.numel() * host_in.element_size()
    return dt, h2d, d2h


# ----------------------------------------------------------------- CPU oracle arm


def cpu_sample(name, cfg, sample, threads):
    """Time the oracle on `sample` matrices of the config (inputs drawn with the same stream)."""
    from oracle import oracle as orc

    from concurrent.futures import ThreadPoolExecutor

    m, n = cfg["m"], cfg["n"]
    a3 = np.empty((sample, n, m))

    def gen(i):  # ctypes drops the GIL: input generation runs on all cores, untimed
        if cfg["kind"] == "rsvd":
            a3[i] = orc.make_matrix(m, n, 1e16, 64, cfg["seed"] + i)[0].T
        else:
            a3[i] = orc.gaussian_matrix(m, n, cfg["seed"] + i).T

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(gen, range(sample)))
    t0 = time.perf_counter()
    if cfg["kind"] == "svd":
        orc.batch_svd_stacked(a3, m, n, ordering=cfg["ordering"], accumulate_v=True, threads=threads)
    elif cfg["kind"] == "qr":
        orc.batch_qr_stacked(a3, m, n, 16, threads=threads)
    elif cfg["kind"] == "block":
        meth = cfg.get("method", "gram")
        orc.batch_block_svd_stacked(a3, m, n, block_width=32, method=meth, tol=1e-11 if meth == "gram" else 1e-13,
                                    accumulate_v=True, threads=threads)
    else:
        orc.batch_rsvd_stacked(a3, m, n, cfg["k"], cfg["p"], seed=5, threads=threads)
    return time.perf_counter() - t0


CPU_SAMPLE = {"cfg1": 1000, "cfg2": 10_000, "cfg3": 5000, "cfg4": 48, "cfg4d": 32, "cfg5": 2000}


def cpu_baseline(name, cfg, threads, sample=None):
    sample = sample or CPU_SAMPLE[name]
    dt = cpu_sample(name, cfg, sample, threads)
    return {"value": sample / dt, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{sample} matrices of {name} ({cfg['m']}x{cfg['n']}), oracle C restatement, {threads} threads, "
                      f"{dt:.2f} s"}


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:  # noqa: BLE001
        return os.cpu_count() or 1


# ----------------------------------------------------------------- main


def free_port():
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def spawn_ranks(n):
    """Re-exec this command under torch.distributed.run with n processes (one per GPU, NCCL)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=HEADLINE, help="headline config (cfg1..cfg5)")
    ap.add_argument("--no-extra", action="store_true", help="skip the other configs")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--e2e-chunks", type=int, default=-12, help="host-buffer pipeline chunks for the e2e leg (negative: equal chunks, no taper)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: every rank runs the config's full batch; strong: the config's batch is split "
                         "over the ranks (contiguous shards, index_base keeps rsvd's seed ^ i global)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `python bench.py --gpus N` without torchrun: launch the N ranks ourselves (one per GPU)
        sys.exit(spawn_ranks(args.gpus))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    name = args.config
    cfg = CONFIGS[name]
    workload = {"workload": cfg["desc"], "config": name, "batch_per_gpu": cfg["batch"], "m": cfg["m"],
                "n": cfg["n"], "l2": "flushed between timed steps (256 MiB memset)",
                "parallelism": f"batch-sharded x{args.gpus} (weak)"}

    if args.impl == "reference":
        if rank != 0:
            return
        thr = host_threads()
        sample = CPU_SAMPLE[name]
        vals = []
        for _ in range(args.warmup):
            cpu_sample(name, cfg, max(1, sample // 8), thr)
        for _ in range(args.steps):
            vals.append(sample / cpu_sample(name, cfg, sample, thr))
        v = float(np.median(vals))
        line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sample / v,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (reference Gaussian stream)", "config": workload,
                "cpu_baseline": {"value": v, "unit": UNIT, "cores": thr, "kind": "port",
                                 "sample": f"{sample} matrices per step, oracle C restatement of the reference "
                                           f"(pure-Python reference cannot travel), {thr} threads"},
                "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    import torch

    dist = None
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    peaks = load_peaks()
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=device)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize(device)

    def max_over_ranks(x):
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    gc = GpuConfig(name, cfg, device, rank, world)
    barrier()
    clocks = ClockSampler(local)
    clocks.start()
    barrier()
    t_dev = time_gpu(gc, args.steps, args.warmup, flush)
    barrier()
    clk = clocks.stop()
    t_max = max_over_ranks(t_dev)
    B = cfg["batch"]
    value = world * B * args.steps / t_max
    flops, bytes_alg = gc.flops()
    ms = 1e3 * t_max / args.steps
    # the headline step is one C-ABI call = the sweep kernel + the V-replay kernel back to back on
    # the current stream; the CUDA-event time of the step is their combined duration (the sweep
    # kernel is ~2/3 of it, profiles/launches_r01.md)
    t_launch = t_dev / args.steps
    achieved_tf = flops / t_launch / 1e12
    prof = load_profile(name)
    # e2e through the public API with host buffers
    e2e_steps = max(5, args.steps)  # host-side timing: more steps than the device leg
    t_e2e, h2d, d2h = time_e2e(gc, e2e_steps, args.e2e_chunks)
    e2e_v = max_over_ranks(t_e2e)
    e2e_value = world * B * e2e_steps / e2e_v

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference Gaussian stream, generated on device)",
            "config": workload, "gflops": flops / t_launch / 1e9,
            "roofline": {"bound": "tensor", "achieved": achieved_tf, "peak": peaks["fp64_tflops"], "unit": "TFLOP/s",
                         "frac": achieved_tf / peaks["fp64_tflops"],
                         "traffic": prof.get("dram_bytes_per_launch"),
                         "kernel": gc.kernel_name(),
                         "traffic_kernel": prof.get("kernel"),
                         "launches_per_step": gc.launches_per_step(),
                         "flops_per_launch": flops, "alg_bytes_per_launch": bytes_alg,
                         "peak_source": "FP64 compute roof: FP64 tensor-core (DMMA) loop measured on this pool, "
                                        "profiles/fp64_peak_r01.json (MEASURED_PEAKS.json has no FP64 entry); the "
                                        "Jacobi kernels issue DFMA, whose measured peak is lower",
                         "dfma_peak": peaks.get("fp64_dfma_tflops"),
                         "frac_of_dfma": achieved_tf / peaks["fp64_dfma_tflops"] if peaks.get("fp64_dfma_tflops") else None,
                         "flops_rule": "SURVEY §8d / PAPER.md:172: 6m per pair visit + (6m+6n) per rotation, from the "
                                       "run's own per-matrix sweep and rotation counters",
                         "traffic_source": prof.get("source"),
                         "hbm_achieved_gbs": bytes_alg / t_launch / 1e9, "hbm_peak_gbs": peaks["hbm_gbs"]},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "path": "host-buffer call (paper_1707_05141_b200.stream.run_host_pipelined: one C-ABI "
                            "bf_svd_batched_f64 call per chunk) with pinned HOST buffers: H2D of A, D2H of U, sigma, "
                            "V, sweeps, converged inside the timed region",
                    "chunks": args.e2e_chunks},
            "gpu_launches": gc.launches_per_step() * args.steps, "clocks": clk}
    del gc
    torch.cuda.empty_cache()

    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(name, cfg, host_threads())

    if not args.no_extra:
        extra = {}
        for other, oc in CONFIGS.items():
            if other == name:
                continue
            g2 = GpuConfig(other, oc, device, rank, world)
            barrier()
            st = 2 if oc["kind"] == "block" else 3
            t2 = time_gpu(g2, st, 3, flush)
            t2m = max_over_ranks(t2)
            f2, b2 = g2.flops()
            ent = {"desc": oc["desc"], "value": world * oc["batch"] * st / t2m, "unit": UNIT,
                   "ms_per_step": 1e3 * t2m / st, "gflops": f2 / (t2 / st) / 1e9,
                   "fp64_frac": f2 / (t2 / st) / 1e12 / peaks["fp64_tflops"],
                   "hbm_frac": b2 / (t2 / st) / 1e9 / peaks["hbm_gbs"]}
            del g2
            torch.cuda.empty_cache()
            if rank == 0 and world == 1 and not args.no_cpu:
                cb = cpu_baseline(other, oc, host_threads())
                ent["cpu_baseline"] = cb
            extra[other] = ent
        line["configs"] = extra
    if rank == 0:
        print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
