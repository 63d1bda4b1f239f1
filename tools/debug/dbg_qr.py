import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_1707_05141_b200 as bf
from oracle import oracle as orc
for (m, n) in [(128, 40), (64, 40), (64, 32)]:
    a = bf.gaussian_tensor(4, m, n, 123, seed_mode="add")
    q, r = bf.qr_tensor(a)
    a3 = a.transpose(1, 2).contiguous().cpu().numpy()
    qo, ro, _ = orc.batch_qr_stacked(a3, m, n)
    qg = q.transpose(1, 2).contiguous().cpu().numpy(); rg = r.transpose(1, 2).contiguous().cpu().numpy()
    dr = np.abs(rg - ro).max(axis=(0)); dq = np.abs(qg - qo).max(axis=0)
    print(m, n, "R err", dr.max(), "Q err", dq.max())
    print(" R err by row (first 5 cols)", np.round(np.abs(rg-ro)[0].max(axis=0)[:12], 3))
    print(" Q err by col", np.round(np.abs(qg-qo)[0].max(axis=1)[:12], 3))
