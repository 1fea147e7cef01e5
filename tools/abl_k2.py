import sys, torch
sys.path.insert(0, ".")
from paper_1603_01876_b200 import capi
S=24; n=1<<S
uv=capi.k0_generate(S,1); srt=capi.k1_sort(uv,S); del uv
L=capi.lib()
import ctypes, json
for i in range(4):
    L.prg_profile_report(None,0,1); L.prg_profile_enable(1)
    m=capi.k2_filter(srt,n); torch.cuda.synchronize(); m.close()
    L.prg_profile_enable(0)
    buf=(ctypes.c_char*65536)(); L.prg_profile_report(buf,65536,1); d=json.loads(buf.value.decode())
    if i: print({k:round(v[1]/v[0],3) for k,v in d.items()})
