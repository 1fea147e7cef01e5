"""Dev experiment: steady-state SpMV vs allocation settings (run under different env)."""
import ctypes, json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1603_01876_b200 import capi
S = 24; n = 1 << S
L = capi.lib(); buf = (ctypes.c_char * 65536)()
uv = capi.k0_generate(S, 1); srt = torch.empty_like(uv)
st = torch.cuda.current_stream()
capi.k1_sort(uv, S, out=srt, stream=st)
m = capi.k2_filter(srt, n, stream=st, csc=True)
for rep in range(3):
    L.prg_profile_report(None, 0, 1); L.prg_profile_enable(1)
    capi.k3_pagerank(m, seed=1, stream=st)
    torch.cuda.synchronize(); L.prg_profile_enable(0); L.prg_profile_report(buf, 65536, 1)
    p = json.loads(buf.value.decode()); sp = p["k3_spmv"]
    print(os.environ.get("TAG", ""), rep, "spmv %.4f" % (sp[1] / sp[0]), flush=True)
