"""Generates tests/golden/*.npz from the REFERENCE implementation itself
(oracle/_ref/libprpipe_ref.so, compiled from /root/reference/proj/src by
oracle/build_ref.sh). Run here (the reference is not present on the GPU box);
the .npz files are committed.

Fixtures (all seeds / scales follow the reference's own tests or BASELINE.json):
  k1k2k3_s10_seed55.npz  — K0 list, std::sort output, K2 CSR + d_in, K3 ranks
                           (S=10 seed 55: tests/test_kernel2_filter.cpp:166-193)
  k1k2k3_s8_seed23.npz   — S=8 seed 23 (tests/test_kernel3_pagerank.cpp:167-174)
  k2k3_er_s12_seed2.npz  — Erdős–Rényi control (uniform initiator), S=12 seed 2
  k3_s16_seed1.npz       — S=16 Kronecker seed 1: K2 stats + final ranks (BASELINE configs[0])
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import oracle as O  # noqa: E402


def make(name, scale, seed, init, k3_seed, keep_edges=True, keep_matrix=True, iters=20):
    n = 1 << scale
    uv = O.ref_generate(scale, seed, init)
    srt, _ = O.ref_k1_sort_core(uv)
    k2, _ = O.ref_k2(srt, n)
    ranks, norm, _ = O.ref_run_kernel3(k2.row_offsets, k2.cols, k2.values, n, iterations=iters, seed=k3_seed,
                                       total_edges=16 * n)
    r0, norm0 = O.ref_init_rank(n, k3_seed)
    step1, norm1 = O.ref_pagerank_step(r0, k2.row_offsets, k2.cols, k2.values, n)
    d = dict(scale=scale, seed=seed, initiator=np.asarray(init), k3_seed=k3_seed, iterations=iters,
             row_offsets=k2.row_offsets, cols=k2.cols, values=k2.values, d_in=k2.d_in, nnz_raw=k2.nnz_raw,
             ranks=ranks, norm1=norm, init_rank=r0, init_norm1=norm0, step1=step1, step1_norm1=norm1)
    if not keep_matrix:
        for key in ("row_offsets", "cols", "values", "init_rank", "step1"):
            d.pop(key)
        d.update(nnz=len(k2.cols), row_offsets_checksum=np.int64(int(k2.row_offsets.sum())),
                 cols_checksum=np.int64(int((k2.cols * np.arange(1, len(k2.cols) + 1, dtype=np.int64)).sum())))
    if keep_edges:
        d.update(edges=uv, sorted_by_u=srt)
    else:
        d.update(edges_checksum=np.int64(np.bitwise_xor.reduce((uv[:, 0] * 1000003 + uv[:, 1]).astype(np.int64))))
    np.savez_compressed(os.path.join(HERE, name), **d)
    print(name, "nnz", k2.nnz, "norm1", repr(norm))


if __name__ == "__main__":
    if not O.have_reference():
        sys.exit("reference library not built (oracle/build_ref.sh needs /root/reference)")
    make("k1k2k3_s10_seed55.npz", 10, 55, O.GRAPH500, 55)
    make("k1k2k3_s8_seed23.npz", 8, 23, O.GRAPH500, 99)
    make("k2k3_er_s12_seed2.npz", 12, 2, O.UNIFORM, 2)
    make("k3_s16_seed1.npz", 16, 1, O.GRAPH500, 1, keep_edges=False, keep_matrix=False)
