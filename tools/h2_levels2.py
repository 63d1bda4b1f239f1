import json, torch
from paper_1707_05141_b200 import h2
for n in (4096, 8192):
    H = h2.build_h2(h2.perturbed_grid(n, seed=0), 0.1, 11, 2.0, 64).to("cuda")
    h2.compress(H, 1e-7)
    Hc, rep = h2.compress(H, 1e-7)
    print(n, rep["truncation_ms"], json.dumps(rep["levels"]))
