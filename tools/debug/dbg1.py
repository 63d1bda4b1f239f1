import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_1707_05141_b200 as bf
from oracle import oracle as orc
def stack_np(t): return t.transpose(-1,-2).contiguous().cpu().numpy()
B=64
a, sig = bf.make_matrix_tensor(B, 128, 128, 1e16, rank=64, seed=5_000_000)
r = bf.rsvd_tensor(a, bf.RsvdOptions(k=32, p=8, seed=5))
a3 = stack_np(a)
o = orc.batch_rsvd_stacked(a3, 128, 128, 32, 8, seed=5, threads=16)
s = r["s"].cpu().numpy(); sg = sig.cpu().numpy()
eg = np.max(np.abs(s[:, :32]-sg[None,:32])/sg[None,:32], axis=1)
eo = np.max(np.abs(o["s"][:, :32]-sg[None,:32])/sg[None,:32], axis=1)
print("rsvd gpu err per b", np.round(eg,6)); print("oracle err", np.round(eo,6))
b = int(np.argmax(eg)); print("worst b", b, s[b,:34], o["s"][b,:34])
# input check vs oracle make_matrix
ao, so = orc.make_matrix(128,128,1e16,64,5_000_000+b)
print("input diff", np.max(np.abs(a3[b].T-ao)))
# block
Bb = 6
a = bf.gaussian_tensor(Bb, 256, 256, 4_000_000, seed_mode="add")
opts = bf.BlockJacobiOptions(method="gram", block_width=32, tolerance=1e-11, accumulate_v=True)
rb = bf.block_svd_tensor(a, opts)
ob = orc.batch_block_svd_stacked(stack_np(a), 256, 256, block_width=32, method="gram", tol=1e-11, accumulate_v=True, threads=Bb)
for i in range(Bb):
    sw = int(rb["sweeps"][i]); swo = int(ob["sweeps"][i])
    print(i, sw, swo, "gpu e", np.array2string(rb["e_history"][i,:sw].cpu().numpy(), precision=2), "orc e", np.array2string(ob["e_history"][i,:swo], precision=2))
