"""Quick GPU parity sweep (dev tool): K0/K1/K2/K3 device path vs the CPU oracle."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import oracle as O  # noqa: E402  (checker only)
from paper_1603_01876_b200 import capi  # noqa: E402


def rel_l1(a, b):
    return float(np.abs(a - b).sum() / np.abs(b).sum())


def check(S, seed, init, iters=20):
    n = 1 << S
    t0 = time.time()
    uv_ref = O.generate(S, seed, init)
    uv_d = capi.k0_generate(S, seed, init)
    k0_ok = np.array_equal(uv_d.cpu().numpy(), uv_ref)
    srt_d = capi.k1_sort(uv_d, S)
    torch.cuda.synchronize()
    can = O.k1_sort(uv_ref, S)
    k1_ok = np.array_equal(srt_d.cpu().numpy(), can)
    k2o = O.k2(can, n)
    mat = capi.k2_filter(srt_d, n)
    ro, cols, vals, din = mat.download()
    k2_ok = (np.array_equal(ro, k2o.row_offsets) and np.array_equal(cols, k2o.cols)
             and np.array_equal(vals.view(np.int64), k2o.values.view(np.int64)) and np.array_equal(din, k2o.d_in)
             and mat.nnz_raw == k2o.nnz_raw)
    # non-canonical input: ties in arbitrary order
    rng = np.random.default_rng(S)
    nc = can.copy()
    # shuffle within rows by sorting on (u, random)
    order = np.lexsort((rng.random(len(nc)), nc[:, 0]))
    nc = nc[order]
    mat2 = capi.k2_filter(torch.from_numpy(nc).cuda(), n)
    ro2, cols2, vals2, din2 = mat2.download()
    k2nc_ok = np.array_equal(ro2, k2o.row_offsets) and np.array_equal(cols2, k2o.cols) and np.array_equal(vals2, k2o.values)
    rr, nr = O.run_kernel3(k2o.row_offsets, k2o.cols, k2o.values, n, seed=seed, iterations=iters)
    ra, na = O.run_kernel3(k2o.row_offsets, k2o.cols, k2o.values, n, seed=seed, iterations=iters, accurate=True)
    rp, npar = capi.k3_pagerank(mat, seed=seed, iterations=iters, mode=1)
    rp = rp.cpu().numpy()
    par_exact = np.array_equal(rp.view(np.int64), rr.view(np.int64)) and npar == nr
    rt, nt = capi.k3_pagerank(mat, seed=seed, iterations=iters, mode=0)
    rt = rt.cpu().numpy()
    print(f"S={S} seed={seed} init={init[0]}: K0 {k0_ok} K1 {k1_ok} K2 {k2_ok} K2(noncanon) {k2nc_ok} "
          f"nnz={mat.nnz} K3 parity bit-exact {par_exact} (max|d|={np.abs(rp-rr).max():.2e}) "
          f"timed relL1 vs ref {rel_l1(rt, rr):.2e} vs neumaier {rel_l1(rt, ra):.2e}; ref-vs-neumaier {rel_l1(rr, ra):.2e} "
          f"norm {nt!r} vs {nr!r}  [{time.time()-t0:.1f}s]", flush=True)
    return k0_ok and k1_ok and k2_ok and k2nc_ok and par_exact and rel_l1(rt, rr) < 1e-10


if __name__ == "__main__":
    ok = True
    for S, seed, init in [(4, 1, O.GRAPH500), (8, 3, O.GRAPH500), (10, 1, O.GRAPH500), (12, 2, O.UNIFORM),
                          (16, 1, O.GRAPH500), (18, 5, O.GRAPH500)]:
        try:
            ok &= check(S, seed, init)
        except Exception as e:  # keep sweeping
            print(f"S={S} FAILED: {type(e).__name__}: {e}", flush=True)
            ok = False
    print("ALL OK" if ok else "FAILURES")
