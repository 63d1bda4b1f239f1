import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1707_05141_b200 as bf
from paper_1707_05141_b200.blockjacobi import block_svd_colmajor
a = bf.gaussian_tensor(300, 256, 256, 4_000_000, seed_mode="add")
st = a.transpose(1, 2).contiguous()
r = block_svd_colmajor(st, 256, 256, bf.BlockJacobiOptions(method="direct", block_width=32, accumulate_v=True))
torch.cuda.synchronize()
