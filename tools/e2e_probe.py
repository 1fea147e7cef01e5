"""Dev tool: phase times of the host-buffer K3 (prg_k3_pagerank_host) at S=24
(PRG_E2E_DEBUG=1 prints them), pinned host CSR as the bench's e2e uses."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1603_01876_b200 import capi  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 24
n, m = 1 << S, 16 << S
uv = capi.k0_generate(S, 1)
srt = capi.k1_sort(uv, S)
del uv
mat = capi.k2_filter(srt, n)
del srt
L = capi.lib()
ro = torch.empty(n + 1, dtype=torch.int64).pin_memory()
cols = torch.empty(mat.nnz, dtype=torch.int64).pin_memory()
vals = torch.empty(mat.nnz, dtype=torch.float64).pin_memory()
rk = torch.empty(n, dtype=torch.float64).pin_memory()
capi._check(L.prg_matrix_download(mat.handle, ro.data_ptr(), cols.data_ptr(), vals.data_ptr(), None))
nnz = mat.nnz
mat.close()
for i in range(4):
    nrm = C.c_double()
    t0 = time.perf_counter()
    capi._check(L.prg_k3_pagerank_host(n, nnz, ro.data_ptr(), cols.data_ptr(), vals.data_ptr(), 0.85, 20, 1, 0,
                                       rk.data_ptr(), C.byref(nrm)))
    print(f"call {i}: {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
