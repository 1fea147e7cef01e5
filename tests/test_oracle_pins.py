"""CPU: pin the oracle (oracle/prg_oracle.c) before trusting it.

Two anchors:
  * the reference's own known-answer tests for K1/K2/K3, restated
    (file:line of each original in /root/reference/proj/tests is cited);
  * golden vectors produced by the reference itself (tests/golden/make_golden.py,
    run against oracle/_ref/libprpipe_ref.so) — compared bit for bit.
"""
import numpy as np
import pytest

from conftest import canonical, golden, rel_l1
from oracle import oracle as O

WORKED = np.array([[1, 2], [3, 2], [4, 2], [1, 3], [2, 3], [2, 1], [3, 1], [1, 4]])  # helpers.hpp:19-21


def by_start(uv):
    """helpers.hpp:23-27 (stable here; the tests only depend on u order)."""
    uv = np.asarray(uv).reshape(-1, 2)
    return uv[np.argsort(uv[:, 0], kind="stable")]


# ---- RNG / K0 --------------------------------------------------------------
def test_mix_seed_and_init_rank_single():
    # test_kernel3_pagerank.cpp:62-66: init_rank(1, 5) == [1.0]
    r, norm = O.init_rank(1, 5)
    assert r[0] == 1.0 and norm == 1.0


def test_generate_deterministic_bounded():
    # test_smoke.py:22-29
    e = O.generate(6, 5)
    assert e.shape == (1024, 2)
    assert ((e >= 1) & (e <= 64)).all()
    assert np.array_equal(e, O.generate(6, 5))


@pytest.mark.parametrize("name", ["k1k2k3_s10_seed55.npz", "k1k2k3_s8_seed23.npz"])
def test_generate_matches_reference_golden(name):
    g = golden(name)
    e = O.generate(int(g["scale"]), int(g["seed"]), tuple(g["initiator"]))
    assert np.array_equal(e, g["edges"])


def test_permutation_is_a_permutation():
    p = O.permutation(1 << 10, 3)
    assert np.array_equal(np.sort(p), np.arange(1, (1 << 10) + 1))


# ---- K1 --------------------------------------------------------------------
def test_k1_hand_case():
    # test_kernel1_sort.cpp:29-42
    inp = np.array([[3, 1], [1, 2], [2, 9], [1, 7]])
    out = O.k1_sort(inp, 4)
    assert list(out[:, 0]) == [1, 1, 2, 3]
    assert np.array_equal(canonical(out), canonical(inp))


def test_k1_empty():
    assert O.k1_sort(np.zeros((0, 2), dtype=np.int64), 1).shape == (0, 2)


@pytest.mark.parametrize("name", ["k1k2k3_s10_seed55.npz", "k1k2k3_s8_seed23.npz"])
def test_k1_matches_reference_up_to_tie_order(name):
    # The reference's std::sort leaves ties unordered (kernel1_sort.hpp:23); the
    # u-sequence must match exactly and the (u,v)-canonicalized arrays bit-exactly.
    g = golden(name)
    out = O.k1_sort(g["edges"], int(g["scale"]))
    assert np.array_equal(out[:, 0], g["sorted_by_u"][:, 0])
    assert np.array_equal(out, canonical(g["sorted_by_u"]))


def test_k1_property_rounds():
    # test_kernel1_sort.cpp:150-172 (random sizes/labels; multiset + order)
    rng = np.random.default_rng(0xDECAF)
    for _ in range(20):
        scale = int(rng.integers(1, 7))
        n = 1 << scale
        cnt = int(rng.integers(0, 200))
        inp = rng.integers(1, n + 1, size=(cnt, 2)).astype(np.int64)
        out = O.k1_sort(inp, scale)
        assert (np.diff(out[:, 0]) >= 0).all()
        assert np.array_equal(canonical(out), canonical(inp))


# ---- K2 --------------------------------------------------------------------
def test_k2_duplicate_collapse():
    # test_kernel2_filter.cpp:61-68
    ro, cols, cnt = O.build_adjacency([[1, 2], [1, 2], [2, 3]], 3)
    assert list(cols) == [1, 2] and list(cnt) == [2, 1] and cnt.sum() == 3


def test_k2_empty_and_rejections():
    # :70-76 and :78-85
    ro, cols, cnt = O.build_adjacency(np.zeros((0, 2), dtype=np.int64), 4)
    assert len(cols) == 0 and list(ro) == [0] * 5
    with pytest.raises(ValueError):
        O.build_adjacency([[2, 1], [1, 2]], 2)
    with pytest.raises(ValueError):
        O.build_adjacency([[1, 5]], 4)
    with pytest.raises(ValueError):
        O.build_adjacency([[0, 1]], 4)


def test_k2_in_degree():
    # :87-91
    ro, cols, cnt = O.build_adjacency([[1, 2], [1, 2], [2, 3]], 3)
    assert list(O.in_degree(3, cols, cnt)) == [0, 2, 1]


def test_k2_worked_case():
    # :93-121; acceptance.cpp:61-75
    res = O.k2(by_start(WORKED), 4)
    assert list(res.d_in) == [2, 3, 2, 1]
    assert list(res.row_offsets) == [0, 1, 3, 4, 4]
    assert list(res.cols) == [2, 0, 2, 0]
    assert list(res.values) == [1.0, 0.5, 0.5, 1.0]


def test_k2_all_max_ties_and_unique_max():
    # :123-130 and :132-143
    assert O.k2([[1, 2], [2, 3], [3, 1]], 3).nnz == 0
    ro, cols, cnt = O.build_adjacency([[1, 1], [1, 2], [1, 3], [2, 1], [2, 2], [2, 3], [3, 1]], 3)
    d = O.in_degree(3, cols, cnt)
    assert list(d) == [3, 2, 2]
    fro, fcols, fcnt = O.zero_columns(3, ro, cols, cnt, d)
    assert 0 not in fcols and len(fcols) == 4


def test_k2_normalization():
    # :156-164
    res = O.k2([[1, 2], [1, 3], [1, 3], [1, 3]], 3)
    # column 3 has d_in 3 == max -> filtered; check normalisation directly
    ro, cols, cnt = O.build_adjacency([[1, 2], [1, 3], [1, 3], [1, 3]], 3)
    v = O.row_normalize(3, ro, cnt)
    assert list(v) == [0.25, 0.75]
    assert res.nnz == 0  # column 3 is the max, column 2 is a leaf


def test_k2_conservation_s10():
    # :166-193 (S=10 seed 55)
    g = golden("k1k2k3_s10_seed55.npz")
    ro, cols, cnt = O.build_adjacency(O.k1_sort(g["edges"], 10), 1 << 10)
    assert cnt.sum() == 16384
    res = O.k2(O.k1_sort(g["edges"], 10), 1 << 10)
    sums = np.add.reduceat(res.values, res.row_offsets[:-1][np.diff(res.row_offsets) > 0])
    assert np.allclose(sums, 1.0, atol=1e-12)
    assert ((res.values > 0) & (res.values <= 1)).all()


@pytest.mark.parametrize("name", ["k1k2k3_s10_seed55.npz", "k1k2k3_s8_seed23.npz", "k2k3_er_s12_seed2.npz"])
def test_k2_matches_reference_golden(name):
    g = golden(name)
    s = int(g["scale"])
    for inp in (O.k1_sort(g["edges"], s), g["sorted_by_u"]):  # canonical and reference tie orders
        res = O.k2(inp, 1 << s)
        assert np.array_equal(res.row_offsets, g["row_offsets"])
        assert np.array_equal(res.cols, g["cols"])
        assert np.array_equal(res.values.view(np.int64), g["values"].view(np.int64))
        assert np.array_equal(res.d_in, g["d_in"])
        assert res.nnz_raw == int(g["nnz_raw"])


def test_k2_s16_matches_reference_checksums():
    g = golden("k3_s16_seed1.npz")
    res = O.k2(O.k1_sort(O.generate(16, 1), 16), 1 << 16)
    assert res.nnz == int(g["nnz"]) == 939361
    assert res.nnz_raw == int(g["nnz_raw"]) == 955180
    assert int(res.row_offsets.sum()) == int(g["row_offsets_checksum"])
    assert int((res.cols * np.arange(1, res.nnz + 1, dtype=np.int64)).sum()) == int(g["cols_checksum"])
    assert np.array_equal(res.d_in, g["d_in"]) and res.d_in.max() == 13064


# ---- K3 --------------------------------------------------------------------
def _worked_matrix():
    res = O.k2(by_start(WORKED), 4)
    return res.row_offsets, res.cols, res.values


def test_k3_zero_matrix():
    # test_kernel3_pagerank.cpp:87-93
    r = np.array([0.4, 0.3, 0.2, 0.1])
    out, norm = O.pagerank_step(r, np.zeros(5, np.int64), np.zeros(0, np.int64), np.zeros(0), 4)
    assert np.allclose(out, 0.15 / 4, rtol=1e-15) and abs(norm - 0.15) < 1e-12


def test_k3_permutation_fixed_point():
    # :78-85
    out, norm = O.pagerank_step(np.array([0.5, 0.5]), np.array([0, 1, 2]), np.array([1, 0]), np.array([1.0, 1.0]), 2)
    assert np.allclose(out, 0.5, rtol=1e-15) and abs(norm - 1.0) < 1e-15


def test_k3_worked_spot_value():
    # :95-101
    ro, cols, vals = _worked_matrix()
    out, _ = O.pagerank_step(np.full(4, 0.25), ro, cols, vals, 4)
    assert abs(out[0] - 0.356250) <= 1e-12


def test_k3_linearity_and_mass():
    # :118-129 and :137-149 (S=10 seed 7)
    ro, cols, vals = _worked_matrix()
    r = np.array([0.1, 0.2, 0.3, 0.4])
    a, _ = O.pagerank_step(r, ro, cols, vals, 4)
    b, _ = O.pagerank_step(2 * r, ro, cols, vals, 4)
    assert np.allclose(b, 2 * a, rtol=1e-13)
    res = O.k2(O.k1_sort(O.generate(10, 7), 10), 1 << 10)
    r, prev = O.init_rank(1 << 10, 7)
    for _ in range(20):
        r, norm = O.pagerank_step(r, res.row_offsets, res.cols, res.values, 1 << 10)
        assert 0 < norm <= prev and (r >= 0).all()
        prev = norm


@pytest.mark.parametrize("name", ["k1k2k3_s10_seed55.npz", "k1k2k3_s8_seed23.npz", "k2k3_er_s12_seed2.npz"])
def test_k3_matches_reference_golden_bitwise(name):
    g = golden(name)
    n = 1 << int(g["scale"])
    r0, n0 = O.init_rank(n, int(g["k3_seed"]))
    assert np.array_equal(r0.view(np.int64), g["init_rank"].view(np.int64)) and n0 == float(g["init_norm1"])
    s1, ns1 = O.pagerank_step(r0, g["row_offsets"], g["cols"], g["values"], n)
    assert np.array_equal(s1.view(np.int64), g["step1"].view(np.int64)) and ns1 == float(g["step1_norm1"])
    r, norm = O.run_kernel3(g["row_offsets"], g["cols"], g["values"], n, seed=int(g["k3_seed"]))
    assert np.array_equal(r.view(np.int64), g["ranks"].view(np.int64))
    assert norm == float(g["norm1"])


def test_k3_s16_reference_pin_and_neumaier_drift():
    # BASELINE configs[0]: S=16 seed 1; norm1 0.22149098609600212, drift 3.97e-13
    g = golden("k3_s16_seed1.npz")
    res = O.k2(O.k1_sort(O.generate(16, 1), 16), 1 << 16)
    r, norm = O.run_kernel3(res.row_offsets, res.cols, res.values, 1 << 16, seed=1)
    assert np.array_equal(r.view(np.int64), g["ranks"].view(np.int64))
    assert norm == float(g["norm1"]) == 0.22149098609600212
    ra, _ = O.run_kernel3(res.row_offsets, res.cols, res.values, 1 << 16, seed=1, accurate=True)
    assert 1e-13 < rel_l1(r, ra) < 1e-12


@pytest.mark.skipif(not O.have_reference(), reason="reference library not built here")
def test_oracle_vs_live_reference_s12():
    uv = O.ref_generate(12, 9, O.GRAPH500)
    assert np.array_equal(uv, O.generate(12, 9))
    srt, _ = O.ref_k1_sort_core(uv)
    ref, _ = O.ref_k2(srt, 1 << 12)
    mine = O.k2(O.k1_sort(uv, 12), 1 << 12)
    assert np.array_equal(mine.values.view(np.int64), ref.values.view(np.int64))
    rr, nr, _ = O.ref_run_kernel3(ref.row_offsets, ref.cols, ref.values, 1 << 12, seed=9)
    ro, no = O.run_kernel3(ref.row_offsets, ref.cols, ref.values, 1 << 12, seed=9)
    assert np.array_equal(rr.view(np.int64), ro.view(np.int64)) and nr == no
