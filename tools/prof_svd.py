"""One svd call for ncu: python tools/prof_svd.py m n B seed ordering accv"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1707_05141_b200 as bf  # noqa: E402
from paper_1707_05141_b200.jacobi import svd_colmajor  # noqa: E402

m, n, B, seed = (int(x) for x in sys.argv[1:5])
order, accv = sys.argv[5], bool(int(sys.argv[6]))
a = bf.gaussian_tensor(B, m, n, seed, seed_mode="add")
st = a.transpose(1, 2).contiguous()
svd_colmajor(st, m, n, bf.JacobiOptions(ordering=order, accumulate_v=accv))
torch.cuda.synchronize()
