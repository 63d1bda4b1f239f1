"""Time hot-path variants with CUDA events (no profiler): python tools/time_variants.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1707_05141_b200 as bf  # noqa: E402
from paper_1707_05141_b200.jacobi import svd_colmajor  # noqa: E402


def t_ms(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def main():
    cases = [(64, 64, 5000, 3_000_000, "round_robin"), (32, 32, 1000, 1_000_000, "serial"),
             (32, 32, 1000, 1_000_000, "round_robin"), (40, 40, 10000, 5_000_000, "round_robin")]
    for m, n, B, seed, order in cases:
        a = bf.gaussian_tensor(B, m, n, seed, seed_mode="add")
        st = a.transpose(1, 2).contiguous()
        for accv in (True, False):
            for tier in ("auto", "shared"):
                o = bf.JacobiOptions(ordering=order, accumulate_v=accv, tier=tier)
                r = svd_colmajor(st, m, n, o, rotations=True)
                sw = r["sweeps"].double().mean().item()
                ms = t_ms(lambda: svd_colmajor(st, m, n, o))
                print(f"{m}x{n} B={B} {order:11s} V={int(accv)} tier={tier:6s}: {ms:8.3f} ms  "
                      f"{B / ms * 1e3:10.0f} mat/s  sweeps {sw:.2f}", flush=True)


if __name__ == "__main__":
    main()
