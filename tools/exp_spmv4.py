"""Dev experiment: SpMV launch time averaged over pool placements (dummy
stream-ordered allocations of varying size shift where K3's buffers land)."""
import ctypes, json, sys, os, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from cuda.bindings import runtime as rt
from paper_1603_01876_b200 import capi
S = int(os.environ.get("SCALE", "24")); n = 1 << S
L = capi.lib(); buf = (ctypes.c_char * 65536)()
uv = capi.k0_generate(S, 1); srt = torch.empty_like(uv)
st = torch.cuda.current_stream()
capi.k1_sort(uv, S, out=srt, stream=st)
m = capi.k2_filter(srt, n, stream=st, csc=True)
res = []
dummies = []
for shift in (0, 1, 3, 7, 13, 29):
    err, p = rt.cudaMallocAsync(shift * 4096 * 37 + 256, 0)
    dummies.append(p)
    for rep in range(2):
        L.prg_profile_report(None, 0, 1); L.prg_profile_enable(1)
        capi.k3_pagerank(m, seed=1, stream=st)
        torch.cuda.synchronize(); L.prg_profile_enable(0); L.prg_profile_report(buf, 65536, 1)
        p_ = json.loads(buf.value.decode()); sp = p_["k3_spmv"]
        res.append(sp[1] / sp[0])
print(os.environ.get("TAG", ""), "spmv mean %.4f min %.4f max %.4f" % (statistics.mean(res), min(res), max(res)),
      " ".join("%.3f" % x for x in res), flush=True)
