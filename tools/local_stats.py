"""Dev tool: K1 local-sort phase statistics from a -DPRG_LOCAL_STATS=1 build of libprg."""
import ctypes as C, os, subprocess, sys
sys.path.insert(0, ".")
import paper_1603_01876_b200.build as B
out = os.path.join(B.ROOT, "build", "libprg_stats.so")
objs = []
for src in (B.CU_SOURCES if not os.path.exists(out) or "--rebuild" in sys.argv else []):
    o = os.path.join(B.ROOT, "build", f"stats_{src}.o")
    subprocess.run([B.NVCC] + B.NVCC_FLAGS + ["-DPRG_LOCAL_STATS=1", "-c", os.path.join(B.CSRC, src), "-o", o], check=True)
    objs.append(o)
if objs:
    subprocess.run([B.NVCC] + B.ARCH + ["-shared", "-o", out] + objs + ["-lcudart"], check=True)
if len([a for a in sys.argv[1:] if not a.startswith("--")]) < 1:
    sys.exit(0)
from paper_1603_01876_b200 import capi
capi.LIB_PATH = out
import torch
S = int([a for a in sys.argv[1:] if not a.startswith("--")][0])
uv = capi.k0_generate(S, 1)
srt = torch.empty_like(uv)
L = capi.lib()
st = (C.c_ulonglong * 16)()
for rep in range(2):
    L.prg_debug_k1_local_stats(st)
    capi.k1_sort(uv, S, out=srt)
    torch.cuda.synchronize()
L.prg_debug_k1_local_stats(st)
v = list(st)
nseg = v[0]
print(f"segments {nseg} keys {v[1]} avg {v[1]/max(nseg,1):.0f}; cycles/segment load {v[2]/nseg:.0f} sort {v[3]/nseg:.0f} write {v[4]/nseg:.0f}; paths: merge32 {v[5]} merge64 {v[6]} lsd {v[7]}")
print("size hist (<=64,128,256,512,1K,2K,4K,8K+):", v[8:16])
