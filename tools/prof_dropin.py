"""Profile the drop-in list call (batch_svd on 5 000 host 64x64 matrices, cfg3): wall time of one
call and the cProfile hot spots (host staging, result construction, synchronisation).

    PYTHONPATH=. python tools/prof_dropin.py
"""
import time, numpy as np, torch, cProfile, pstats, io
import paper_1707_05141_b200 as bf
a = bf.gaussian_tensor(5000, 64, 64, 3_000_000, seed_mode="add")
host = a.cpu().numpy(); mats = [np.asfortranarray(x) for x in host]
opts = bf.JacobiOptions(ordering="round_robin", accumulate_v=True)
bf.batch_svd(mats[:64], opts)
for _ in range(2): bf.batch_svd(mats, opts)
t=time.perf_counter(); bf.batch_svd(mats, opts); print("call %.1f ms"%((time.perf_counter()-t)*1e3))
pr=cProfile.Profile(); pr.enable(); bf.batch_svd(mats, opts); pr.disable()
s=io.StringIO(); pstats.Stats(pr,stream=s).sort_stats("tottime").print_stats(14); print(s.getvalue()[:3500])
