"""float32 vs float64 device time per BASELINE config shape (CUDA events, warm-up, L2 flushed
between repetitions): float64, float32 as shipped (computed on the float64 tiers where api.cu
promotes it) and float32 on the float32 tiers (BF_F32_NATIVE=1). The measurement behind the
float32-on-float64 design; record: profiles/f32_timing_r02.jsonl.

    PYTHONPATH=. python tools/time_f32.py [--reps 5]
"""

import argparse
import json
import os

import torch

import paper_1707_05141_b200 as bf

CASES = [
    ("cfg1 serial 32x32", "svd", 1000, 32, 32, dict(ordering="serial")),
    ("cfg1 rr 32x32", "svd", 1000, 32, 32, dict(ordering="round_robin")),
    ("cfg3 rr 64x64", "svd", 5000, 64, 64, dict(ordering="round_robin")),
    ("48x48 rr", "svd", 5000, 48, 48, dict(ordering="round_robin")),
    ("cfg2 qr 64x32", "qr", 10000, 64, 32, {}),
    ("cfg4d direct 256", "block", 200, 256, 256, dict(method="direct")),
    ("cfg4 gram 256", "block", 200, 256, 256, dict(method="gram")),
    ("cfg5 rsvd 128 k32", "rsvd", 10000, 128, 128, {}),
]


def run(kind, a, kw):
    if kind == "svd":
        return bf.svd_tensor(a, bf.JacobiOptions(accumulate_v=True, **kw))
    if kind == "qr":
        return bf.qr_tensor(a)
    if kind == "block":
        return bf.block_svd_tensor(a, bf.BlockJacobiOptions(accumulate_v=True, block_width=32, **kw))
    return bf.rsvd_tensor(a, bf.RsvdOptions(k=32, p=8, seed=5))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    out = []
    for name, kind, B, m, n, kw in CASES:
        row = {"case": name, "batch": B}
        for key, dt, native in (("f64_ms", torch.float64, False), ("f32_ms", torch.float32, False),
                                ("f32_native_ms", torch.float32, True)):
            if native:
                os.environ["BF_F32_NATIVE"] = "1"
            else:
                os.environ.pop("BF_F32_NATIVE", None)
            a = bf.gaussian_tensor(B, m, n, 7, seed_mode="add", dtype=dt)
            run(kind, a, kw)
            torch.cuda.synchronize()
            ts = []
            for _ in range(args.reps):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                run(kind, a, kw)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            row[key] = sorted(ts)[len(ts) // 2]
        os.environ.pop("BF_F32_NATIVE", None)
        out.append(row)
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
