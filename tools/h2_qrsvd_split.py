"""Split of one upper-level H^2 factorisation (242 x 121 TE, few nodes): QR vs W-only SVD of R."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1707_05141_b200 as bf
from paper_1707_05141_b200.qr import qr_tensor

for B in (1, 4, 16):
    a = bf.gaussian_tensor(B, 242, 121, 5, seed_mode="add")
    def t(f):
        f(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); r = f(); e1.record(); torch.cuda.synchronize()
        return e0.elapsed_time(e1), r
    tq, (q, r) = t(lambda: qr_tensor(a))
    ts, sv = t(lambda: bf.svd_tensor(r.contiguous(), bf.JacobiOptions(ordering="round_robin", accumulate_v=False)))
    print(f"B={B}: qr 242x121 {tq:.3f} ms, svd 121x121 W-only {ts:.3f} ms, sweeps {sv['sweeps'].double().mean().item():.1f}")
