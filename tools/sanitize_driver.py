"""Driver for compute-sanitizer runs: one small pass over every
device path — K0, K1 sort engine (all levels + local stage), K2 passes A/B
with the decoupled look-back and spanning-row fix-ups, the CSC build
(renumbering, stable transpose, SELL build), K3 timed mode (slice-claim
counters, split columns), parity and Neumaier modes, the host-buffer e2e path
and the streamed K1 — checked against the oracle so a sanitizer run also
proves the results unchanged.

    compute-sanitizer --tool memcheck python tools/sanitize_driver.py [scale]

Compute-sanitizer is closed on this GPU pool; tests/test_checked.py runs this
driver against the checked library instead (PRG_LIB=build/libprg_checked.so,
device-side PRG_DCHECK bounds / invariant checks) and requires zero failures.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402  (checker)
from paper_1603_01876_b200 import capi  # noqa: E402


def main(scale):
    import torch

    n = 1 << scale
    for seed, init in ((1, O.GRAPH500), (2, O.UNIFORM)):
        uv = capi.k0_generate(scale, seed, init)
        ref_uv = O.generate(scale, seed, init)
        assert np.array_equal(uv.cpu().numpy(), ref_uv)
        srt = capi.k1_sort(uv, scale)
        ref_srt = O.k1_sort(ref_uv, scale)
        assert np.array_equal(srt.cpu().numpy(), ref_srt)
        mat = capi.k2_filter(srt, n)
        ref = O.k2(ref_srt, n)
        ro, cols, vals, din = mat.download()
        assert np.array_equal(ro, ref.row_offsets) and np.array_equal(cols, ref.cols)
        assert np.array_equal(vals.view(np.int64), ref.values.view(np.int64))
        rr, nr = O.run_kernel3(ref.row_offsets, ref.cols, ref.values, n, seed=seed)
        rt, _ = capi.k3_pagerank(mat, seed=seed, mode=0)                 # layout built inside K3
        mat.build_csc()                                                  # K2's CSC build
        rc, _ = capi.k3_pagerank(mat, seed=seed, mode=0)
        assert np.array_equal(rt.cpu().numpy().view(np.int64), rc.cpu().numpy().view(np.int64))
        assert float(np.abs(rc.cpu().numpy() - rr).sum() / rr.sum()) <= 1e-10
        rp, np_ = capi.k3_pagerank(mat, seed=seed, mode=1)
        assert np.array_equal(rp.cpu().numpy().view(np.int64), rr.view(np.int64)) and np_ == nr
        capi.k3_pagerank(mat, seed=seed, mode=2)
        rh, _ = capi.k3_pagerank_host(n, ref.row_offsets, ref.cols, ref.values, seed=seed, mode=0)
        assert np.array_equal(rh.view(np.int64), rt.cpu().numpy().view(np.int64))
        mat.close()
        torch.cuda.synchronize()
    # K1 small-segment kernel: four start vertices in one level-1 bucket, so the second
    # level's 256 children hold 1-4 K keys each (lone children with <= 32 unsorted bits)
    rng = np.random.default_rng(17)
    e = np.column_stack([rng.integers(1, 5, 400000), rng.integers(1, 1025, 400000)]).astype(np.int64)
    assert np.array_equal(capi.k1_sort(torch.from_numpy(e).cuda(), 10).cpu().numpy(), O.k1_sort(e, 10))
    # streamed K1 (one pinned chunk) through the drop-in
    sys.path.insert(0, os.path.join(ROOT, "paper_1603_01876_b200", "python"))
    import tempfile

    import prpipe

    with tempfile.TemporaryDirectory() as d:
        e = prpipe.generate_edges(prpipe.GenConfig(scale=min(scale, 10), seed=3))
        man = prpipe.write_edges(e, os.path.join(d, "in"), num_files=2, scale=min(scale, 10))
        a = prpipe.read_edges(prpipe.sort_edges(man, os.path.join(d, "mem")))
        b = prpipe.read_edges(prpipe.sort_edges(man, os.path.join(d, "ext"), memory_budget_bytes=4096))
        assert a == b
    # checked builds (PRG_LIB=build/libprg_checked.so): no device-side bounds /
    # invariant check may have failed on any path above
    fails = capi.lib().prg_debug_check_failures()
    assert fails == 0, f"{fails} device-side checks failed"
    print(f"sanitize driver ok: S={scale} (checked library: {capi.LIB_PATH.endswith('libprg_checked.so')})")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 12)
