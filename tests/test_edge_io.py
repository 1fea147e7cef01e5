"""Host edge I/O of the drop-in (paper_1603_01876_b200/host/edge_io.cpp) against
the reference's own edge_io (compiled from its sources, oracle/_ref) — CPU only.

Restates the reference's tests/test_edge_io.cpp cases (round trips, sharding,
empty input, argument errors, manifest round trip, missing trailing LF,
malformed lines with file:line) and adds the fast path's own hazards: blocks
cut inside a line (multi-MiB shards), single-shard inputs, streaming readers
with tiny buffers, and error precedence across shards — every malformed input
must fail with the reference's exact message, and every good one must give the
reference's exact bytes / edges.
"""
import os

import numpy as np
import pytest

from oracle import oracle as O

prpipe = pytest.importorskip("prpipe")
core = prpipe._core  # test hooks for the streaming classes live on the extension module
need_ref = pytest.mark.skipif(not O.have_reference(), reason="reference library not built here")


def edges_of(scale, seed):
    return [tuple(e) for e in O.generate(scale, seed).tolist()]


def manual(tmp_path, name, text, claimed, scale, extra_files=()):
    """A directory with manifest + shard(s) written by hand (tests/test_edge_io.cpp manual_manifest)."""
    d = tmp_path / name
    prpipe.write_edges([(1, 1)] * max(1, claimed if claimed else 1), d, num_files=1, scale=scale)
    files = [("edges_0000.tsv", text, claimed)] + list(extra_files)
    import json

    man = json.load(open(d / "manifest.json"))
    man["files"] = [{"name": n, "edges": c} for n, _, c in files]
    man["total_edges"] = sum(c for _, _, c in files)
    json.dump(man, open(d / "manifest.json", "w"), indent=2)
    for n, t, _ in files:
        with open(d / n, "wb") as f:
            f.write(t.encode() if isinstance(t, str) else t)
    return d


# ---- the reference's test_edge_io.cpp cases ------------------------------------
def test_roundtrip_sharding_and_remainder(tmp_path):
    e = edges_of(9, 4)
    for files in (1, 3, 4, 7):
        man = prpipe.write_edges(e, tmp_path / f"f{files}", num_files=files, scale=9)
        sizes = [f.edges for f in man.files]
        assert sum(sizes) == len(e) and max(sizes) - min(sizes) <= 1 and sizes == sorted(sizes, reverse=True)
        assert prpipe.read_edges(man) == e
        assert core._stream_manifest(man) == e


def test_empty_input_one_empty_file(tmp_path):
    man = prpipe.write_edges([], tmp_path / "e", num_files=1, scale=1)
    assert man.total_edges == 0 and len(man.files) == 1
    assert os.path.getsize(tmp_path / "e" / "edges_0000.tsv") == 0
    assert prpipe.read_edges(man) == [] and core._stream_manifest(man) == []


def test_argument_errors(tmp_path):
    for args in (([(1, 2), (2, 1)], 3), ([], 2), ([(1, 2), (2, 1)], 0)):
        with pytest.raises(RuntimeError):
            prpipe.write_edges(args[0], tmp_path / "x", num_files=args[1], scale=1)
        with pytest.raises(RuntimeError):
            core._write_streaming(args[0], tmp_path / "y", num_files=args[1], scale=1)


def test_manifest_roundtrip(tmp_path):
    w = prpipe.write_edges([(1, 2), (2, 1), (2, 2)], tmp_path / "m", num_files=2, scale=1, sorted_by_start=True)
    r = prpipe.EdgeManifest.load(str(tmp_path / "m"))
    assert (r.total_edges, r.sorted_by_start, r.scale) == (w.total_edges, w.sorted_by_start, w.scale)
    assert [(f.name, f.edges) for f in r.files] == [(f.name, f.edges) for f in w.files]


def test_missing_trailing_newline_accepted(tmp_path):
    d = manual(tmp_path, "nl", "1\t2\n2\t1", 2, 1)
    assert prpipe.read_edges(prpipe.EdgeManifest.load(str(d))) == [(1, 2), (2, 1)]


# ---- byte identity with the reference ------------------------------------------
@need_ref
@pytest.mark.parametrize("scale,files,sorted_", [(9, 4, True), (12, 1, False), (14, 3, True)])
def test_bytes_identical_to_reference(tmp_path, scale, files, sorted_):
    uv = O.generate(scale, 6)
    prpipe.write_edges([tuple(e) for e in uv.tolist()], tmp_path / "mine", num_files=files, scale=scale,
                       sorted_by_start=sorted_)
    core._write_streaming([tuple(e) for e in uv.tolist()], tmp_path / "stream", num_files=files, scale=scale,
                            sorted_by_start=sorted_)
    O.ref_write_edges(uv, str(tmp_path / "ref"), files, scale, sorted_)
    names = sorted(os.listdir(tmp_path / "ref"))
    for other in ("mine", "stream"):
        assert sorted(os.listdir(tmp_path / other)) == names
        for n in names:
            assert (tmp_path / other / n).read_bytes() == (tmp_path / "ref" / n).read_bytes(), (other, n)


@need_ref
def test_extreme_labels_format_like_to_chars(tmp_path):
    # the writer does not validate labels (the reference's doesn't either): any int64 prints as to_chars does
    big = [(1, 2), (-5, 0), (2**63 - 1, -(2**63)), (10**18, 999999999999), (-1, 10), (123456789, 9)]
    prpipe.write_edges(big, tmp_path / "mine", num_files=2, scale=3)
    O.ref_write_edges(np.array(big, dtype=np.int64), str(tmp_path / "ref"), 2, 3, False)
    for n in sorted(os.listdir(tmp_path / "ref")):
        assert (tmp_path / "mine" / n).read_bytes() == (tmp_path / "ref" / n).read_bytes()


def test_multi_block_single_shard_roundtrip(tmp_path):
    # > 4 MiB in one shard: the bulk reader cuts it into blocks inside lines;
    # > 2^18 edges: the bulk writer formats it in several blocks
    uv = O.generate(19, 8)
    e = [tuple(x) for x in uv.tolist()]
    man = prpipe.write_edges(e, tmp_path / "big", num_files=1, scale=19)
    assert os.path.getsize(tmp_path / "big" / "edges_0000.tsv") > (8 << 20)
    assert prpipe.read_edges(man) == e
    assert core._stream_file(str(tmp_path / "big" / "edges_0000.tsv"), 1 << 19, 200) == e


def test_bulk_reader_is_race_free(tmp_path):
    """Blocks of one shard load concurrently; each block must count and decode
    only its own bytes (a block once peeked at its neighbour's first byte while
    that block was still loading). Repeated reads of multi-block shards must
    all give the same edges."""
    uv = O.generate(19, 11)
    e = [tuple(x) for x in uv.tolist()]
    man = prpipe.write_edges(e, tmp_path / "race", num_files=2, scale=19)
    h = 0x243f6a8885a308d3
    for u, v in e:
        h = ((h ^ ((u * 1000003 + v) & (2**64 - 1))) * 0x100000001b3) & (2**64 - 1)
    for _ in range(25):
        assert core._read_edges_checksum(man) == (len(e), h)


# ---- malformed input: the reference's exact error, line and precedence ---------
def ref_read_error(d):
    import ctypes as C

    f = O._sig(O._ref, "ref_read_edges", C.c_int64, [C.c_char_p, C.c_void_p, C.c_int64, C.POINTER(C.c_int64)])
    line = C.c_int64()
    buf = np.empty(2, dtype=np.int64)
    n = f(str(d).encode(), buf.ctypes.data, 0, C.byref(line))
    return None if n >= 0 else O._ref.ref_last_error().decode()


def ref_stream_error(path, max_label, buffer_bytes):
    import ctypes as C

    f = O._sig(O._ref, "ref_stream_file", C.c_int64,
               [C.c_char_p, C.c_int64, C.c_int64, C.c_void_p, C.c_int64, C.POINTER(C.c_int64)])
    line = C.c_int64()
    buf = np.empty(2, dtype=np.int64)
    n = f(str(path).encode(), max_label, buffer_bytes, buf.ctypes.data, 0, C.byref(line))
    return n if n >= 0 else O._ref.ref_last_error().decode()


BAD = {
    "space": "1 2\n",
    "letter": "1\tx\n",
    "range": "1\t2\n1\t3\n",
    "trailing": "1\t2\t3\n",
    "empty_line": "1\t2\n\n1\t1\n",
    "cr": "1\t2\r\n",
    "plus": "+1\t2\n",
    "leading_space": " 1\t2\n",
    "zero": "0\t1\n",
    "negative": "-1\t1\n",
    "overflow": "1\t99999999999999999999999\n",
    "minus_only": "-\t1\n",
    "tab_end": "1\t\n",
    "no_tab": "12\n",
    "late": "1\t1\n" * 5 + "2\t2\n" * 3 + "1\tz\n",
    "long_line": "1" * (1 << 20) + "\t1\n",
}


@need_ref
@pytest.mark.parametrize("case", sorted(BAD))
def test_malformed_line_same_error_as_reference(tmp_path, case):
    text = BAD[case]
    claimed = text.count("\n") + (0 if text.endswith("\n") else 1)
    d = manual(tmp_path, case, text, claimed, 1 if case != "late" else 2)
    want = ref_read_error(d)
    assert want is not None
    with pytest.raises(RuntimeError) as ei:
        prpipe.read_edges(prpipe.EdgeManifest.load(str(d)))
    assert str(ei.value) == want


@need_ref
@pytest.mark.parametrize("buffer_bytes", [1, 128, 129, 200, 4096])
def test_streaming_reader_same_as_reference(tmp_path, buffer_bytes):
    """EdgeFileReader with small buffers: lines longer than the buffer fail with
    the reference's 'line exceeds' error; good files decode identically."""
    p = tmp_path / "s.tsv"
    good = "".join(f"{u}\t{v}\n" for u, v in O.generate(8, 3).tolist())
    for text in (good, good[:-1], good + "7" * 150 + "\t1\n", "5\t5\n" + "1" * 127 + "\n", "1" * 127):
        p.write_bytes(text.encode())
        want = ref_stream_error(p, 256, buffer_bytes)
        if isinstance(want, str):
            with pytest.raises(RuntimeError) as ei:
                core._stream_file(str(p), 256, buffer_bytes)
            assert str(ei.value) == want
        else:
            assert len(core._stream_file(str(p), 256, buffer_bytes)) == want


@need_ref
def test_error_precedence_across_shards(tmp_path):
    # shard 0 has the wrong count, shard 1 a parse error: the sequential reader reports shard 0
    d = manual(tmp_path, "prec", "1\t1\n1\t2\n", 3, 1, extra_files=[("edges_0001.tsv", "1\tq\n", 1)])
    want = ref_read_error(d)
    with pytest.raises(RuntimeError) as ei:
        prpipe.read_edges(prpipe.EdgeManifest.load(str(d)))
    assert str(ei.value) == want and "edges_0000.tsv" in want
    # count right, parse error late in shard 0, another in shard 1: shard 0's line wins
    d2 = manual(tmp_path, "prec2", "1\t1\n" * 100 + "x\n", 101, 1, extra_files=[("edges_0001.tsv", "y\n", 1)])
    with pytest.raises(RuntimeError) as ei:
        prpipe.read_edges(prpipe.EdgeManifest.load(str(d2)))
    assert str(ei.value) == ref_read_error(d2) and ":101:" in str(ei.value)
    # missing shard after a good one
    d3 = manual(tmp_path, "prec3", "1\t1\n", 1, 1, extra_files=[("edges_0001.tsv", "1\t1\n", 1)])
    os.remove(d3 / "edges_0001.tsv")
    with pytest.raises(RuntimeError) as ei:
        prpipe.read_edges(prpipe.EdgeManifest.load(str(d3)))
    assert str(ei.value) == ref_read_error(d3)


@need_ref
def test_parse_error_inside_a_late_block(tmp_path):
    # a bad line far into a multi-block shard: the line number must be exact
    uv = O.generate(18, 2)
    lines = [f"{u}\t{v}\n" for u, v in uv.tolist()]
    k = len(lines) - 1000
    lines[k] = f"{lines[k][:-1]}\t\n"
    d = manual(tmp_path, "lateblock", "".join(lines), len(lines), 18)
    with pytest.raises(RuntimeError) as ei:
        prpipe.read_edges(prpipe.EdgeManifest.load(str(d)))
    assert str(ei.value) == ref_read_error(d) and f":{k + 1}:" in str(ei.value)
