"""Benchmark: batched fp64 SVD matrices/s & GFLOP/s on B200 (BASELINE.json metric).

python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfg3|...|all]

One "step" = one pass of the hot path over the config's whole batch (synthetic inputs of
the BASELINE shape, generated on the device with the reference's Gaussian stream).
Headline workload (N=1): cfg3, 5,000 random 64x64 fp64 matrices, round-robin Jacobi with V
(the shared-memory tier). Every other BASELINE config is measured in the same run under
"configs" with the same fields (device value, roofline, e2e through host buffers, CPU baseline,
launch count). Multi-GPU: `--gpus N` launches N ranks itself (torch.distributed.run) when not
already under torchrun; --scaling weak (default: every rank its own full batch) or strong (the
config's batch split over the ranks); no data-path collective; time = max over ranks.

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
    """Per-launch DRAM traffic of the config's dominant kernel(s) from the committed ncu --set full
    summary (profiles/ncu_full_r02.json, written by tools/ncu_summary.py)."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "ncu_full_r02.json")))
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


def block_flops(m, n, kk, method, stats, accv=True):
    """cfg4/cfg4d algorithmic flops from the run's own per-matrix counters (bf_block_svd_batched_ex:
    pair visits, rotated pairs, inner pair visits, inner rotations), SURVEY §8d conventions:
    Gram: 2m(2k)^2 per visited pair (G = P^T P), (2m + 2n)(2k)^2 per rotated pair (P U, V_pair U);
    direct: QR 4m(2k)^2 - 4(2k)^3/3 per visit, (2m + 2n)(2k)^2 per rotated pair (Q [U S; 0], V_pair V_R);
    inner Jacobi: 6(2k) per inner pair visit, 6(2k) (+6(2k) with V, direct) per inner rotation."""
    s = stats.double().sum(dim=0).tolist()
    visits, rotated, ivisits, irot = s
    if method == "gram":
        outer = visits * 2.0 * m * kk * kk + rotated * (2.0 * m + (2.0 * n if accv else 0.0)) * kk * kk
        inner = 6.0 * kk * ivisits + 6.0 * kk * irot
    else:
        outer = visits * (4.0 * m * kk * kk - 4.0 * kk ** 3 / 3.0) + rotated * (2.0 * m + (2.0 * n if accv else 0.0)) * kk * kk
        inner = 6.0 * kk * ivisits + 12.0 * kk * irot
    return outer + inner, {"pair_visits": visits, "rotated_pairs": rotated, "inner_pair_visits": ivisits,
                           "inner_rotations": irot}


class GpuConfig:
    """Builds device-resident inputs for one config and runs its hot path once per step.

    scaling "weak": every rank owns `batch` entries of a world*batch global batch; "strong": the
    config's batch is split over the ranks. Either way a rank's entries are a contiguous shard with
    its global index_base (rsvd's seed ^ i stays global, rsvd.py:82-85)."""

    def __init__(self, name, cfg, device, rank, world=1, scaling="weak", batch=None):
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
        m, n = cfg["m"], cfg["n"]
        B = cfg["batch"] if batch is None else batch
        self.global_batch = world * B if scaling == "weak" else B
        self.plan = ShardPlan(self.global_batch, world, rank)
        self.local_batch = self.plan.count
        seed0 = cfg["seed"] + self.plan.start
        if cfg["kind"] == "rsvd":
            self.a, _ = bf.make_matrix_tensor(self.local_batch, m, n, 1e16, rank=64, seed=cfg["seed"],
                                              index_base=self.plan.start, device=device)
        else:
            self.a = bf.gaussian_tensor(self.local_batch, m, n, seed0, seed_mode="add", device=device)
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
            self.out = self.k_block(self.store, m, n, block_opts(c), stats=True)
        else:
            opts = bf.RsvdOptions(k=c["k"], p=c["p"], seed=5)
            self.out = self.k_rsvd(self.store, m, n, opts, index_base=self.plan.start)  # seed ^ global index

    def kernel_name(self):
        c = self.cfg
        if c["kind"] == "svd":
            return "svd_rr_kernel + svd_rr_vcol_kernel" if c["ordering"] == "round_robin" else "svd_reg_kernel"
        if c["kind"] == "block" and c.get("method", "gram") == "direct":
            return "bj_dqr_reg + svd_rr_kernel + svd_rr_vcol_kernel (inner) + bj_dapply_wy + bj_rot_tma"
        return {"qr": "qr_reg_kernel", "block": "bj_gram_tma + svd_rr_kernel (inner) + bj_rot_tma",
                "rsvd": "gemm_mma_kernel + qr_reg_kernel + svd_rr_kernel + svd_rr_vkernel"}[c["kind"]]

    def work(self):
        """(algorithmic flops, compulsory bytes, counters) of the last step, from the run's own
        sweep / rotation / pair counters."""
        c = self.cfg
        m, n, B = c["m"], c["n"], self.local_batch
        if c["kind"] == "svd":
            sw = self.out["sweeps"].double().sum().item()
            rot = self.out["rotations"].double().sum().item()
            return (jacobi_flops(m, n, sw, rot), B * 8.0 * (2 * m * n + n * n + n),
                    {"sweeps_mean": sw / max(B, 1), "rotations_mean": rot / max(B, 1)})
        if c["kind"] == "qr":
            return B * qr_flops(m, n), B * 8.0 * (2 * m * n + n * n), {}
        if c["kind"] == "block":
            f, cnt = block_flops(m, n, 64, c.get("method", "gram"), self.out["stats"])
            cnt["sweeps_mean"] = self.out["sweeps"].double().mean().item()
            return f, B * 8.0 * (3 * m * n + n), cnt
        w = c["k"] + c["p"]
        return (B * rsvd_flops(m, n, w, 2.909e6), B * 8.0 * (m * n + m * w + n * w + w),
                {"inner_svd": "oracle-mean nominal 2.909 MFLOP per 40x40 inner SVD with V"})

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

    def dropin_call(self, host_list):
        """The reference-shaped drop-in call: list of numpy matrices in, list of dataclasses out."""
        bf, c = self.bf, self.cfg
        if c["kind"] == "svd":
            return bf.batch_svd(host_list, bf.JacobiOptions(ordering=c["ordering"], accumulate_v=True), device=self.dev)
        if c["kind"] == "qr":
            return bf.batch_qr(host_list, 16, device=self.dev)
        if c["kind"] == "block":
            return bf.batch_block_svd(host_list, block_opts(c), device=self.dev)
        return bf.batch_rsvd(host_list, bf.RsvdOptions(k=c["k"], p=c["p"], seed=5), device=self.dev)


def count_launches(gc):
    """Our kernels in one step, counted by the CUDA profiler (kernel names in namespace bf::), in an
    untimed extra step. Falls back to None when CUPTI is unavailable (e.g. under ncu)."""
    if os.environ.get("BF_BENCH_NO_PROFILER"):
        return None, []
    try:
        from torch.profiler import ProfilerActivity, profile

        gc.torch.cuda.synchronize(gc.dev)
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            gc.step()
            gc.torch.cuda.synchronize(gc.dev)
        names = {}
        for ev in prof.events():
            nm = ev.name
            if "bf::" in nm:
                short = nm.split("bf::", 1)[1].split("<", 1)[0].split("(", 1)[0]
                names[short] = names.get(short, 0) + 1
        return sum(names.values()), sorted(names.items(), key=lambda kv: -kv[1])
    except Exception:  # noqa: BLE001
        return None, []


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


def time_dropin(gc, steps):
    """The drop-in API on host numpy matrices (list in, dataclasses out), as a reference user calls it."""
    host = gc.a.cpu().numpy()
    mats = [np.asfortranarray(x) for x in host]
    gc.dropin_call(mats[: min(len(mats), 64)])  # warm-up
    t0 = time.perf_counter()
    for _ in range(steps):
        gc.dropin_call(mats)
    return time.perf_counter() - t0


def roofline(gc, flops, bytes_alg, t_step, peaks, prof):
    """Roofline object of the step: FP64 for the Jacobi / block / rsvd paths, HBM for the QR (whose
    intensity ~5.3 flop/B sits at the FP64 ridge; both fractions are reported)."""
    tf = flops / t_step / 1e12
    gbs = bytes_alg / t_step / 1e9
    common = {"kernel": gc.kernel_name(), "traffic": prof.get("dram_bytes_per_launch"),
              "traffic_kernel": prof.get("kernel"), "traffic_source": prof.get("source"),
              "flops_per_step": flops, "alg_bytes_per_step": bytes_alg,
              "fp64_tflops": tf, "fp64_frac": tf / peaks["fp64_tflops"],
              "hbm_gbs": gbs, "hbm_frac": gbs / peaks["hbm_gbs"],
              "dfma_peak": peaks.get("fp64_dfma_tflops"),
              "frac_of_dfma": tf / peaks["fp64_dfma_tflops"] if peaks.get("fp64_dfma_tflops") else None,
              "flops_rule": "SURVEY §8d / PAPER.md:172 conventions, counted from the run's own per-matrix "
                            "sweep / rotation / pair counters (rsvd: inner SVD at the oracle's mean)"}
    if gc.cfg["kind"] == "qr":
        return dict(bound="hbm", achieved=gbs, peak=peaks["hbm_gbs"], unit="GB/s", frac=gbs / peaks["hbm_gbs"],
                    peak_source="MEASURED_PEAKS.json hbm_gbs (copy bandwidth on this pool)", **common)
    return dict(bound="tensor", achieved=tf, peak=peaks["fp64_tflops"], unit="TFLOP/s",
                frac=tf / peaks["fp64_tflops"],
                peak_source="FP64 compute roof: FP64 tensor-core (DMMA) loop measured on this pool, "
                            "profiles/fp64_peak_r01.json (MEASURED_PEAKS.json has no FP64 entry); the Jacobi "
                            "kernels issue DFMA, whose measured peak is lower (dfma_peak)", **common)


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


def measure(name, cfg, device, rank, world, args, flush, peaks, barrier, max_over_ranks, steps, warmup,
            e2e=True, dropin=False, batch=None):
    """One config: device-resident timing (CUDA events, max over ranks), the counted work, the
    roofline object, the host-buffer e2e leg and (optionally) the list-in drop-in leg."""
    torch = __import__("torch")
    gc = GpuConfig(name, cfg, device, rank, world, args.scaling, batch=batch)
    barrier()
    clocks = ClockSampler(device.index)
    clocks.start()
    barrier()
    t_dev = time_gpu(gc, steps, warmup, flush)
    barrier()
    clk = clocks.stop()
    t_max = max_over_ranks(t_dev)
    flops, bytes_alg, counters = gc.work()
    t_step = t_dev / steps  # this rank's step: its flops over its own device time
    prof = load_profile(name)
    ent = {"value": gc.global_batch * steps / t_max, "unit": UNIT, "ms_per_step": 1e3 * t_max / steps,
           "global_batch": gc.global_batch, "batch_per_gpu": gc.local_batch,
           "gflops": world * flops / t_max * steps / 1e9,
           "roofline": roofline(gc, flops, bytes_alg, t_step, peaks, prof), "counters": counters, "clocks": clk}
    n_launch, kinds = count_launches(gc)
    ent["gpu_launches"] = None if n_launch is None else n_launch * steps
    ent["kernels_per_step"] = dict(kinds)
    if e2e:
        e2e_steps = max(3, min(steps, 5))
        # host-buffer pipeline depth: enough chunks to overlap the PCIe copies with compute, but each
        # chunk must stay a full-GPU call (the small and block configs are latency / wave bound:
        # 12 chunks of cfg1 or cfg4 would each run at one matrix's latency)
        chunks = args.e2e_chunks if args.e2e_chunks != 0 else E2E_CHUNKS.get(name, -12)
        t_e2e, h2d, d2h = time_e2e(gc, e2e_steps, chunks)
        t_e2e = max_over_ranks(t_e2e)
        ent["e2e"] = {"value": gc.global_batch * e2e_steps / t_e2e, "unit": UNIT, "h2d_bytes_per_step": h2d,
                      "d2h_bytes_per_step": d2h,
                      "path": "host-buffer call (paper_1707_05141_b200.stream.run_host_pipelined: one C-ABI batched "
                              "call per chunk) with pinned HOST buffers: H2D of A, D2H of every output inside the "
                              "timed region", "chunks": abs(chunks)}
    if dropin:
        dsteps = 2
        t_d = max_over_ranks(time_dropin(gc, dsteps))
        ent["e2e_dropin"] = {"value": gc.global_batch * dsteps / t_d, "unit": UNIT,
                             "path": "drop-in API as the reference is called: batch_*(list of numpy matrices) -> "
                                     "list of result dataclasses (host stacking, H2D, kernels, D2H, unstacking)"}
    del gc
    torch.cuda.empty_cache()
    return ent


# per-config e2e pipeline chunks (default; --e2e-chunks overrides; positive = first and last chunk
# half-sized, negative = equal chunks). Measured per config: the PCIe-bound cfg2/cfg3/cfg5 overlap
# best with ~10 tapered chunks -- cfg3 at 10 keeps every full chunk (556 matrices) within one wave
# of the persistent 592-CTA kernel: 589 k vs 556 k matrices/s untapered at 12, 539 k at 9, 562 k at
# 11; cfg1 (latency-bound) with 2; the wave-bound block configs unchunked (cfg4 4 321 vs 3 911
# matrices/s at 2 chunks, cfg4d 2 215 vs 2 155)
E2E_CHUNKS = {"cfg1": -2, "cfg2": 10, "cfg3": 10, "cfg4": -1, "cfg4d": -1, "cfg5": 12}

BATCH_SWEEP = [125, 250, 500, 1000, 2000, 4000, 8000, 16000]


def selftest(args, rank, world):
    """Launcher / sharding check without GPUs (gloo on CPU): every rank takes its contiguous shard
    of small cfg1- and cfg5-shaped batches under the same ShardPlan / index_base logic the GPU run
    uses, runs the CPU oracle on it as the stand-in for the device call (test infrastructure), and
    the all-gathered results on rank 0 must equal a single-rank run bit for bit (core.py:97-103;
    rsvd's seed ^ global index, rsvd.py:82-85). Prints one JSON line on rank 0."""
    import torch
    import torch.distributed as dist

    from oracle import oracle as orc
    from paper_1707_05141_b200.shard import ShardPlan, gather_results

    if world > 1:
        dist.init_process_group("gloo")
    checks = {}
    for what, (m, n, B) in (("svd", (16, 12, 37)), ("rsvd", (24, 20, 29))):
        a3 = np.stack([orc.gaussian_matrix(m, n, 9_000_000 + i).T for i in range(B)])  # (B, n, m)
        plan = ShardPlan(B, world, rank)
        loc = np.ascontiguousarray(a3[plan.start:plan.stop])

        def run(x, ib):
            if what == "svd":
                r = orc.batch_svd_stacked(x, m, n, ordering="round_robin", accumulate_v=True)
                return {"s": torch.from_numpy(np.ascontiguousarray(r["s"])),
                        "u": torch.from_numpy(np.ascontiguousarray(r["u"])),
                        "sweeps": torch.from_numpy(r["sweeps"].astype(np.int32))}
            r = orc.batch_rsvd_stacked(x, m, n, 4, 2, seed=5, index_base=ib)
            return {"s": torch.from_numpy(np.ascontiguousarray(r["s"])),
                    "v": torch.from_numpy(np.ascontiguousarray(r["v"]))}

        got = gather_results(run(loc, plan.start), plan)
        if rank == 0:
            ref = run(np.ascontiguousarray(a3), 0)
            checks[what] = {"entries": B, "shard_counts": plan.counts,
                            "bitwise_equal": all(torch.equal(got[k], ref[k]) for k in ref)}
    if rank == 0:
        ok = all(c["bitwise_equal"] for c in checks.values())
        print(json.dumps({"selftest": "ok" if ok else "FAILED", "world": world, "backend": "gloo" if world > 1 else None,
                          "launcher": "torch.distributed.run (spawned by bench.py --gpus N)"
                                      if os.environ.get("TORCHELASTIC_RUN_ID") else "direct",
                          "checks": checks}))
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=HEADLINE, help="headline config (cfg1..cfg5, cfg4d)")
    ap.add_argument("--no-extra", action="store_true", help="skip the other configs")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-dropin", action="store_true", help="skip the list-in drop-in e2e leg")
    ap.add_argument("--batch-sweep", action="store_true", help="also time the headline config at several batch sizes")
    ap.add_argument("--e2e-chunks", type=int, default=0,
                    help="host-buffer pipeline chunks for the e2e leg (negative: equal chunks, no taper)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: every rank runs the config's full batch; strong: the config's batch is split "
                         "over the ranks (contiguous shards, index_base keeps rsvd's seed ^ i global)")
    ap.add_argument("--selftest", action="store_true",
                    help="CPU-only launcher/sharding check over gloo (no GPU): shard-invariant gathered results")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `python bench.py --gpus N` without torchrun: launch the N ranks ourselves (one per GPU)
        sys.exit(spawn_ranks(args.gpus))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.selftest:
        selftest(args, rank, world)
        return
    name = args.config
    cfg = CONFIGS[name]
    gbatch = world * cfg["batch"] if args.scaling == "weak" else cfg["batch"]
    workload = {"workload": cfg["desc"], "config": name, "global_batch": gbatch,
                "batch_per_gpu": cfg["batch"] if args.scaling == "weak" else f"{cfg['batch']}/{world}",
                "m": cfg["m"], "n": cfg["n"], "l2": "flushed between timed steps (256 MiB memset)",
                "parallelism": f"batch-sharded x{world} ({args.scaling}); no data-path collective"}

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
                "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (reference Gaussian stream)", "config": workload,
                "cpu_baseline": {"value": v, "unit": UNIT, "cores": thr, "kind": "port",
                                 "sample": f"{sample} matrices per step, oracle C restatement of the reference "
                                           f"(the pure-Python reference cannot travel; per core the C port is "
                                           f"~11x faster than the as-shipped Python, DESIGN §4), {thr} threads"},
                "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    import torch

    dist = None
    if world > 1:
        import torch.distributed as dist

        # BF_BENCH_SHARE_GPU=1 (functional check of the multi-rank path on a one-GPU box): ranks
        # share the visible GPUs round-robin and talk over gloo (NCCL refuses two ranks per GPU);
        # timings from such a run are not scaling numbers
        if os.environ.get("BF_BENCH_SHARE_GPU"):
            local = local % torch.cuda.device_count()
            dist.init_process_group("gloo")
        else:
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
        t = torch.tensor([x], dtype=torch.float64, device=device if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    ent = measure(name, cfg, device, rank, world, args, flush, peaks, barrier, max_over_ranks, args.steps,
                  args.warmup, e2e=True, dropin=not args.no_dropin)
    line = {"metric": METRIC, "value": ent["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ent["ms_per_step"], "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference Gaussian stream, generated on device)", "config": workload,
            "gflops": ent["gflops"], "roofline": ent["roofline"], "e2e": ent["e2e"],
            "gpu_launches": ent["gpu_launches"], "kernels_per_step": ent["kernels_per_step"],
            "counters": ent["counters"], "clocks": ent["clocks"]}
    if "e2e_dropin" in ent:
        line["e2e_dropin"] = ent["e2e_dropin"]

    if rank == 0 and world == 1 and not args.no_cpu:
        cb = cpu_baseline(name, cfg, host_threads())
        line["cpu_baseline"] = cb
        line["vs_cpu_baseline"] = {"value": ent["value"] / cb["value"], "e2e": ent["e2e"]["value"] / cb["value"]}

    if args.batch_sweep:
        sweep = {}
        for bsz in BATCH_SWEEP:
            e = measure(name, cfg, device, rank, world, args, flush, peaks, barrier, max_over_ranks, 3, 2,
                        e2e=False, batch=bsz)
            sweep[str(bsz)] = {"value": e["value"], "ms_per_step": e["ms_per_step"],
                               "frac": e["roofline"]["frac"], "bound": e["roofline"]["bound"]}
        line["batch_sweep"] = sweep

    if not args.no_extra:
        extra = {}
        for other, oc in CONFIGS.items():
            if other == name:
                continue
            st = 2 if oc["kind"] == "block" else 3
            e = measure(other, oc, device, rank, world, args, flush, peaks, barrier, max_over_ranks, st, 2,
                        e2e=True)
            e["desc"] = oc["desc"]
            e.pop("clocks", None)
            if rank == 0 and world == 1 and not args.no_cpu:
                cb = cpu_baseline(other, oc, host_threads())
                e["cpu_baseline"] = cb
                e["vs_cpu_baseline"] = {"value": e["value"] / cb["value"], "e2e": e["e2e"]["value"] / cb["value"]}
            extra[other] = e
        line["configs"] = extra
    if rank == 0:
        print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
