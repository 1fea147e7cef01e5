"""The drop-in module `prpipe` (paper_1603_01876_b200/python/prpipe, C++ shim
over the C-ABI) exercised like the reference's own Python tests
(/root/reference/proj/tests/python/test_smoke.py). Host-only pieces (K0,
edge I/O, sizes) run on CPU; K1/K2/K3 need the GPU.
"""
import filecmp
import math
import os

import numpy as np
import pytest

from oracle import oracle as O

prpipe = pytest.importorskip("prpipe")


# ---- CPU: sizes, K0, edge I/O ---------------------------------------------------
def test_derived_sizes_and_memory():
    # test_smoke.py:10-16
    assert prpipe.derived_sizes(22, 16) == (4194304, 67108864)
    assert prpipe.derived_sizes(30, 16) == (1073741824, 17179869184)
    assert prpipe.estimate_memory_bytes(prpipe.GenConfig(scale=19), bytes_per_edge=24) == 201326592
    with pytest.raises(RuntimeError):
        prpipe.derived_sizes(63, 16)


def test_generate_is_deterministic_bounded_and_matches_reference():
    # test_smoke.py:19-25 + bit-exact vs the pinned oracle
    config = prpipe.GenConfig(scale=6, seed=5)
    edges = prpipe.generate_edges(config)
    assert len(edges) == config.edge_count == 1024
    assert all(1 <= u <= 64 and 1 <= v <= 64 for u, v in edges)
    assert edges == prpipe.generate_edges(prpipe.GenConfig(scale=6, seed=5))
    assert np.array_equal(np.array(edges), O.generate(6, 5))
    er = prpipe.generate_edges(prpipe.GenConfig(scale=8, seed=2, initiator=[0.25, 0.25, 0.25, 0.25]))
    assert np.array_equal(np.array(er), O.generate(8, 2, O.UNIFORM))


def test_write_read_roundtrip_and_sharding(tmp_path):
    # test_smoke.py:31-35 + the contiguous split (earlier shards take the remainder)
    edges = prpipe.generate_edges(prpipe.GenConfig(scale=7, seed=9))
    man = prpipe.write_edges(edges, tmp_path / "k0", num_files=3, scale=7)
    assert man.total_edges == len(edges) == 2048
    assert [f.edges for f in man.files] == [683, 683, 682]
    assert prpipe.read_edges(man) == edges
    assert prpipe.read_edges(prpipe.EdgeManifest.load(str(tmp_path / "k0"))) == edges


@pytest.mark.skipif(not O.have_reference(), reason="reference library not built here")
def test_edge_files_byte_identical_to_reference(tmp_path):
    edges = prpipe.generate_edges(prpipe.GenConfig(scale=9, seed=3))
    prpipe.write_edges(edges, tmp_path / "mine", num_files=4, scale=9, sorted_by_start=True)
    O.ref_write_edges(np.array(edges), str(tmp_path / "ref"), 4, 9, True)
    names = sorted(os.listdir(tmp_path / "ref"))
    assert names == sorted(os.listdir(tmp_path / "mine"))
    match, mismatch, errors = filecmp.cmpfiles(tmp_path / "ref", tmp_path / "mine", names, shallow=False)
    assert not mismatch and not errors


def test_edge_io_errors(tmp_path):
    # test_smoke.py:99-100 and the parse-error paths (test_edge_io.cpp:137-172)
    with pytest.raises(RuntimeError):
        prpipe.write_edges([(1, 2)], tmp_path / "x", num_files=2, scale=1)
    d = tmp_path / "bad"
    prpipe.write_edges([(1, 2), (2, 1)], d, num_files=1, scale=1)
    with open(d / "edges_0000.tsv", "w") as f:
        f.write("1\t2\n7\t1\n")  # label outside [1, N]
    with pytest.raises(RuntimeError, match="edges_0000.tsv:2"):
        prpipe.read_edges(prpipe.EdgeManifest.load(str(d)))
    with pytest.raises(RuntimeError, match="missing manifest"):
        prpipe.EdgeManifest.load(str(tmp_path / "nowhere"))


def test_validation_oracle_host_side():
    # dense path (validation.cpp) needs no GPU
    m = prpipe.dense_pagerank_matrix
    assert prpipe.DENSE_CAP == 4096
    assert prpipe.validate([0.5, 0.5], [1.0, 1.0], tol=1e-12)
    assert not prpipe.validate([0.9, 0.1], [0.5, 0.5], tol=1e-3)
    assert callable(m)


# ---- GPU: the reference's smoke tests against the drop-in ---------------------
@pytest.mark.gpu
def test_staged_pipeline(tmp_path):
    # test_smoke.py:28-60
    config = prpipe.GenConfig(scale=7, seed=9)
    edges = prpipe.generate_edges(config)
    manifest = prpipe.write_edges(edges, tmp_path / "k0", num_files=2, scale=config.scale)
    sorted_manifest = prpipe.sort_edges(manifest, tmp_path / "k1")
    assert sorted_manifest.sorted_by_start
    sorted_edges = prpipe.read_edges(sorted_manifest)
    assert sorted(sorted_edges) == sorted(edges)
    assert [u for u, _ in sorted_edges] == sorted(u for u, _ in edges)

    matrix, elapsed, rate = prpipe.run_kernel2(sorted_manifest)
    assert elapsed > 0 and rate > 0
    assert matrix.n == config.vertex_count
    assert all(s == 0.0 or math.isclose(s, 1.0, abs_tol=1e-12) for s in (matrix.row_sum(r) for r in range(matrix.n)))

    pr = prpipe.PageRankConfig(iterations=20, seed=9)
    ranks, elapsed3, rate3 = prpipe.run_kernel3(matrix, pr, sorted_manifest.total_edges)
    assert elapsed3 > 0 and rate3 > 0
    assert len(ranks.values) == matrix.n and all(v >= 0.0 for v in ranks.values)
    assert 0.0 < ranks.norm1 <= 1.0 + 1e-12

    limit_ranks, flag, iters = prpipe.run_to_convergence(matrix, 0.85, 1e-12, 10000, 9)
    assert flag and iters < 10000
    dense = prpipe.dense_pagerank_matrix(matrix, 0.85)
    vec, value, dense_flag, _ = prpipe.principal_eigenvector(dense, tol=1e-12)
    assert dense_flag and value > 0
    assert prpipe.validate(limit_ranks.values, vec, tol=1e-8)

    # bit-exact against the oracle on the same stages
    ref = O.k2(O.k1_sort(np.array(edges), 7), 128)
    assert list(matrix.row_offsets) == list(ref.row_offsets) and list(matrix.cols) == list(ref.cols)
    assert np.array_equal(np.array(matrix.values).view(np.int64), ref.values.view(np.int64))
    rr, _ = O.run_kernel3(ref.row_offsets, ref.cols, ref.values, 128, seed=9)
    assert float(np.abs(np.array(ranks.values) - rr).sum() / rr.sum()) <= 1e-10


@pytest.mark.gpu
def test_sort_edges_under_a_memory_budget(tmp_path):
    """test_kernel1_sort.cpp:79-121: a budget below the list size takes the
    out-of-core route (here: one pinned chunk of budget/16 edges streamed
    through HBM) and must agree with the in-memory sort — bit for bit here, a
    stronger check than the reference's u-sequence + multiset — leaving no
    spill directory behind; :133-144 the output shard count; a non-positive
    budget falls back to default_memory_budget() (kernel1_sort.cpp:135-137)."""
    for scale, seed, files, budget, fan_in in ((10, 33, 4, 4096, 64), (8, 5, 1, 2048, 4)):
        edges = prpipe.generate_edges(prpipe.GenConfig(scale=scale, seed=seed))
        man = prpipe.write_edges(edges, tmp_path / f"in{scale}", num_files=files, scale=scale)
        mem = prpipe.read_edges(prpipe.sort_edges(man, tmp_path / f"mem{scale}"))
        ext_man = prpipe.sort_edges(man, tmp_path / f"ext{scale}", memory_budget_bytes=budget, merge_fan_in=fan_in)
        ext = prpipe.read_edges(ext_man)
        assert ext == mem and ext_man.sorted_by_start
        assert [u for u, _ in ext] == sorted(u for u, _ in edges) and sorted(ext) == sorted(edges)
        assert not os.path.exists(tmp_path / f"ext{scale}" / "spill")
    neg = prpipe.read_edges(prpipe.sort_edges(man, tmp_path / "neg", memory_budget_bytes=-5))
    assert neg == mem
    rows = [(100 - i, i % 100 + 1) for i in range(100)]
    m5 = prpipe.write_edges(rows, tmp_path / "in5", num_files=1, scale=7)
    for budget in (0, 64):  # in memory, and streamed in 4-edge chunks
        out = prpipe.sort_edges(m5, tmp_path / f"out5_{budget}", memory_budget_bytes=budget, num_files=5)
        assert [f.edges for f in out.files] == [20] * 5
        got = prpipe.read_edges(out)
        assert [u for u, _ in got] == sorted(u for u, _ in rows)
    bad = tmp_path / "bad"
    prpipe.write_edges([(1, 2), (2, 1)], bad, num_files=1, scale=1)
    with open(bad / "edges_0000.tsv", "w") as f:
        f.write("1\t2\n9\t1\n")
    with pytest.raises(RuntimeError, match="edges_0000.tsv:2"):  # the reader's own error, streamed route too
        prpipe.sort_edges(prpipe.EdgeManifest.load(str(bad)), tmp_path / "bad_out", memory_budget_bytes=16)


@pytest.mark.gpu
def test_kernel2_worked_case():
    # test_smoke.py:63-73
    edges = [(1, 2), (1, 3), (1, 4), (2, 3), (2, 1), (3, 2), (3, 1), (4, 2)]
    a = prpipe.build_adjacency(edges, 4)
    assert a.total() == 8
    d_in = prpipe.in_degree(a)
    assert d_in == [2, 3, 2, 1]
    s = prpipe.row_normalize(prpipe.zero_columns(a, d_in))
    assert s.value_at(0, 2) == 1.0
    assert s.value_at(1, 0) == 0.5 and s.value_at(1, 2) == 0.5
    assert s.value_at(2, 0) == 1.0
    assert s.row_sum(3) == 0.0


@pytest.mark.gpu
def test_run_pipeline_report(tmp_path):
    # test_smoke.py:76-92
    report = prpipe.run_pipeline(scale=8, seed=4, data_dir=tmp_path / "data", validate=True)
    assert not report["failed"], report["error"]
    assert report["sizes"] == {"vertices": 256, "edges": 4096}
    assert [k["name"] for k in report["kernels"]] == ["k0_generate", "k1_sort", "k2_filter", "k3_pagerank"]
    assert report["kernels"][0]["scoring"] is False
    for k in report["kernels"][1:]:
        assert k["scoring"] is True and k["rate_edges_per_sec"] > 0
    assert report["validation"]["performed"] is True and report["validation"]["passed"] is True


@pytest.mark.gpu
def test_errors_surface_as_exceptions(tmp_path):
    # test_smoke.py:95-100
    with pytest.raises(RuntimeError):
        prpipe.build_adjacency([(2, 1), (1, 2)], 2)  # unsorted
    with pytest.raises(RuntimeError):
        prpipe.write_edges([(1, 2)], tmp_path / "x", num_files=2, scale=1)
    with pytest.raises(RuntimeError):
        prpipe.run_kernel3(prpipe.row_normalize(prpipe.build_adjacency([(1, 2)], 2)),
                           prpipe.PageRankConfig(damping=1.0), 1)


@pytest.mark.gpu
def test_step_api_bit_exact_vs_reference_golden():
    from conftest import golden

    g = golden("k1k2k3_s10_seed55.npz")
    edges = [tuple(map(int, e)) for e in g["sorted_by_u"]]  # the reference's own tie order
    a = prpipe.build_adjacency(edges, 1024)
    s = prpipe.row_normalize(prpipe.zero_columns(a, prpipe.in_degree(a)))
    assert list(s.row_offsets) == list(g["row_offsets"]) and list(s.cols) == list(g["cols"])
    assert np.array_equal(np.array(s.values).view(np.int64), g["values"].view(np.int64))
    r0 = prpipe.init_rank(1024, 55)
    assert np.array_equal(np.array(r0.values).view(np.int64), g["init_rank"].view(np.int64))
    r1 = prpipe.pagerank_step(r0, s, 0.85)
    assert np.array_equal(np.array(r1.values).view(np.int64), g["step1"].view(np.int64))
    assert r1.norm1 == float(g["step1_norm1"])
