"""Dev experiment: SpMV launch time under different preceding call sequences."""
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
st = torch.cuda.current_stream()

def spmv(tag, fn, reps=3):
    for i in range(reps):
        L.prg_profile_report(None, 0, 1)
        L.prg_profile_enable(1)
        fn()
        torch.cuda.synchronize()
        L.prg_profile_enable(0)
        L.prg_profile_report(buf, 65536, 1)
        p = json.loads(buf.value.decode())
        sp = p.get("k3_spmv", [1, 0.0])
        print(tag, i, "spmv %.4f" % (sp[1] / sp[0]), "k3 %.3f" % p.get("k3_pagerank", [1, 0])[1], flush=True)

def e1():
    capi.k1_sort(uv, S, out=srt, stream=st)
    m = capi.k2_filter(srt, n, stream=st, csc=True)
    capi.k3_pagerank(m, seed=1, stream=st)
    m.close()

def e2():
    m = capi.k2_filter(srt, n, stream=st, csc=True)
    capi.k3_pagerank(m, seed=1, stream=st)
    m.close()

def e3():
    m = capi.k2_filter(srt, n, stream=st)
    capi.k3_pagerank(m, seed=1, stream=st)
    m.close()

def e4():
    m = capi.k2_filter(srt, n, stream=st, csc=True)
    capi.k3_pagerank(m, seed=1, stream=st)
    capi.k3_pagerank(m, seed=1, stream=st)
    m.close()

for tag, f in (("k1k2csc_k3", e1), ("k2csc_k3", e2), ("k2_k3cold", e3), ("k2csc_k3x2", e4), ("k1k2csc_k3", e1)):
    spmv(tag, f)
