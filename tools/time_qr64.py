"""Time cfg2's QR (10000 x 64x32, f64): python tools/time_qr64.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1707_05141_b200 as bf
from paper_1707_05141_b200.qr import qr_colmajor

a = bf.gaussian_tensor(10000, 64, 32, 2_000_000, seed_mode="add")
st = a.transpose(1, 2).contiguous()
for _ in range(3):
    qr_colmajor(st, 64, 32)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    qr_colmajor(st, 64, 32)
e1.record()
torch.cuda.synchronize()
print(os.path.basename(os.environ.get("BATCHFACT_B200_LIB", "default")), f"qr 10000x64x32: {e0.elapsed_time(e1) / 10:.4f} ms")
