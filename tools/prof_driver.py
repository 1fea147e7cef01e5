"""Profiling driver (dev tool): runs one warm-up and one profiled instance of a stage.
usage: python tools/prof_driver.py {k1,k2,k3} SCALE"""
import sys
import torch
sys.path.insert(0, ".")
from paper_1603_01876_b200 import capi

stage, S = sys.argv[1], int(sys.argv[2])
n = 1 << S
uv = capi.k0_generate(S, 1)
srt = torch.empty_like(uv)
for rep in range(2):
    capi.k1_sort(uv, S, out=srt)
    if stage in ("k2", "k3"):
        mat = capi.k2_filter(srt, n)
        if stage == "k3":
            capi.k3_pagerank(mat, seed=1, iterations=3)
        mat.close()
torch.cuda.synchronize()
print("done")
