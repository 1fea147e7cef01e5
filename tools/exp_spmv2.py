"""Dev experiment: why the bench's timed-region SpMV differs from a standalone loop."""
import ctypes, json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1603_01876_b200 import capi

S = 24
n = 1 << S
L = capi.lib()
buf = (ctypes.c_char * 65536)()
uv = capi.k0_generate(S, 1)
srt = torch.empty_like(uv)
ranks = torch.empty(n, dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream()

def step(out):
    capi.k1_sort(uv, S, out=srt, stream=st)
    m = capi.k2_filter(srt, n, stream=st, csc=True)
    capi.k3_pagerank(m, seed=1, stream=st, out=out)
    m.close()

import time
from cuda.bindings import runtime as rt

def trim():
    torch.cuda.synchronize()
    err, pool = rt.cudaDeviceGetDefaultMemPool(0)
    rt.cudaMemPoolTrimTo(pool, 0)

def run(tag, steps, out, warm=3, between=None):
    for _ in range(warm):
        step(out)
    torch.cuda.synchronize()
    L.prg_profile_report(None, 0, 1)
    L.prg_profile_enable(1)
    for i in range(steps):
        if between and i:
            between()
        step(out)
    torch.cuda.synchronize()
    L.prg_profile_enable(0)
    L.prg_profile_report(buf, 65536, 1)
    p = json.loads(buf.value.decode())
    sp = p["k3_spmv"]
    print(tag, "spmv %.4f" % (sp[1] / sp[0]), "k3 %.3f" % (p["k3_pagerank"][1] / p["k3_pagerank"][0]), flush=True)

cudart = ctypes.CDLL("libcudart.so.12") if False else None
run("steps5", 5, ranks)
run("steps5_sleep0", 5, ranks, between=lambda: time.sleep(0))
run("steps5_sleep100us", 5, ranks, between=lambda: time.sleep(0.0001))
run("steps5_torchsync", 5, ranks, between=torch.cuda.synchronize)
run("steps5_rtsync", 5, ranks, between=lambda: rt.cudaDeviceSynchronize())
run("steps5_sleep5ms", 5, ranks, between=lambda: time.sleep(0.005))
run("steps5", 5, ranks)
