"""Time rsvd's inner QR shape (10000 x 128x40) and the full cfg5 rsvd step: python tools/time_qr40.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1707_05141_b200 as bf
from paper_1707_05141_b200.qr import qr_colmajor

tag = os.environ.get("BF_QR40", "0")
a = bf.gaussian_tensor(10000, 128, 40, 9, seed_mode="add")
st = a.transpose(1, 2).contiguous()
for _ in range(2):
    qr_colmajor(st, 128, 40)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    qr_colmajor(st, 128, 40)
e1.record()
torch.cuda.synchronize()
print(f"BF_QR40={tag} qr 10000x128x40: {e0.elapsed_time(e1) / 5:.3f} ms", flush=True)
m5, _ = bf.make_matrix_tensor(10000, 128, 128, 1e16, rank=64, seed=5)
o = bf.RsvdOptions(k=32, p=8, seed=5)
for _ in range(2):
    bf.rsvd_tensor(m5, o)
torch.cuda.synchronize()
e0.record()
for _ in range(5):
    bf.rsvd_tensor(m5, o)
e1.record()
torch.cuda.synchronize()
print(f"BF_QR40={tag} rsvd cfg5: {e0.elapsed_time(e1) / 5:.3f} ms", flush=True)
