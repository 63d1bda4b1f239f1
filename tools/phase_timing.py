"""Per-phase clock breakdown of the register-tier W step (instrumented build):
BATCHFACT_B200_LIB=build_var/lib_timing.so python tools/phase_timing.py"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1707_05141_b200 as bf  # noqa: E402
from paper_1707_05141_b200 import _lib  # noqa: E402
from paper_1707_05141_b200.jacobi import svd_colmajor  # noqa: E402

L = _lib.load()
buf = (ctypes.c_ulonglong * 8)()
names = ["products+STS", "barrier1", "reduce+butterfly", "rotation+cs", "barrier2(or)", "apply", "total"]
for m, n, B, seed, order in [(64, 64, 5000, 3_000_000, "round_robin"), (32, 32, 1000, 1_000_000, "serial"),
                             (40, 40, 10000, 5_000_000, "round_robin")]:
    a = bf.gaussian_tensor(B, m, n, seed, seed_mode="add")
    st = a.transpose(1, 2).contiguous()
    o = bf.JacobiOptions(ordering=order, accumulate_v=False)
    svd_colmajor(st, m, n, o)
    torch.cuda.synchronize()
    L.bf_debug_phase_clk(buf, 1)
    r = svd_colmajor(st, m, n, o, rotations=True)
    torch.cuda.synchronize()
    L.bf_debug_phase_clk(buf, 1)
    steps = r["sweeps"].double().sum().item() * (n - 1 if order == "round_robin" else 2 * n - 3)
    print(f"{m}x{n} {order}: cycles per step (thread 0 of each CTA)")
    for i, nm in enumerate(names):
        print(f"   {nm:18s} {buf[i] / steps:8.1f}")
