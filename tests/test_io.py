"""File input (bbtc_edges_read / bbtc_graph_load, SURVEY §8(b) "load"): host-only
parsing checks (-m "not gpu") and one device count of a loaded file (-m gpu).

The karate fixture (SURVEY App. A, 45 triangles) is written in each format; the
parsed pairs must equal the fixture and the oracle's count of them must be 45."""
import numpy as np
import pytest

import inputs
import oracle


def _bb():
    import paper_2009_12457_b200 as bb
    return bb


def write_text(path, s, d, header="# karate\n% also a comment\n\n"):
    with open(path, "w") as f:
        f.write(header)
        for a, b in zip(s.tolist(), d.tolist()):
            f.write(f"{a}\t{b}\n")


def write_mm(path, s, d, n):
    with open(path, "w") as f:
        f.write("%%MatrixMarket matrix coordinate pattern symmetric\n% karate\n")
        f.write(f"{n} {n} {len(s)}\n")
        for a, b in zip(s.tolist(), d.tolist()):
            f.write(f"{b + 1} {a + 1}\n")   # lower triangle, 1-based, as MM symmetric files store it


def write_bin(path, s, d):
    np.stack([s, d], axis=1).astype("<u4").tofile(path)


@pytest.mark.parametrize("fmt", ["text", "mm", "bin"])
def test_read_karate_each_format(tmp_path, fmt):
    bb = _bb()
    s, d = inputs.karate()
    path = tmp_path / f"karate.{fmt}"
    if fmt == "text":
        write_text(path, s, d)
    elif fmt == "mm":
        write_mm(path, s, d, 34)
    else:
        write_bin(path, s, d)
    rs, rd, n_hint = bb.read_edges(path, fmt)
    if fmt == "mm":
        assert n_hint == 34
        rs, rd = rd, rs
    else:
        assert n_hint == 0
    assert np.array_equal(rs, s) and np.array_equal(rd, d)
    total, _, _, _ = oracle.OracleGraph(rs, rd, max(n_hint, 34)).count(2)
    assert total == 45


def test_text_crlf_commas_and_extra_fields(tmp_path):
    bb = _bb()
    p = tmp_path / "g.txt"
    p.write_bytes(b"0,1,7\r\n1 2 0.5\r\n  2\t0\r\n# tail\r\n")
    s, d, _ = bb.read_edges(p, "text")
    assert s.tolist() == [0, 1, 2] and d.tolist() == [1, 2, 0]


def test_empty_text_file(tmp_path):
    bb = _bb()
    p = tmp_path / "e.txt"
    p.write_text("# nothing\n")
    s, d, n = bb.read_edges(p, "text")
    assert len(s) == 0 and len(d) == 0 and n == 0


@pytest.mark.parametrize("body,code,line", [
    ("0 1\n1 x\n", -4, 2),          # malformed second field
    ("0 1\n2\n", -4, 2),            # one id only
    ("0 1\n-3 4\n", -4, 2),         # negative id
    ("0 1\n1 2\n3 4294967295\n", -5, 3),   # reserved id 0xFFFFFFFF
])
def test_text_errors_carry_line(tmp_path, body, code, line):
    bb = _bb()
    p = tmp_path / "bad.txt"
    p.write_text(body)
    with pytest.raises(bb.BBTCError) as ei:
        bb.read_edges(p, "text")
    assert ei.value.code == code
    assert f"bad.txt:{line}:" in str(ei.value)


@pytest.mark.parametrize("body,frag", [
    ("0 1\n", "header"),
    ("%%MatrixMarket matrix array real general\n2 2\n", "coordinate"),
    ("%%MatrixMarket matrix coordinate pattern general\n3 3 2\n1 2\n", "1 of 2"),
    ("%%MatrixMarket matrix coordinate pattern general\n3 3 1\n1 2\n2 3\n", "more entries"),
    ("%%MatrixMarket matrix coordinate pattern general\n3 3 1\n0 2\n", "out of the declared size"),
    ("%%MatrixMarket matrix coordinate pattern general\n3 3 1\n1 4\n", "out of the declared size"),
])
def test_mm_errors(tmp_path, body, frag):
    bb = _bb()
    p = tmp_path / "bad.mtx"
    p.write_text(body)
    with pytest.raises(bb.BBTCError) as ei:
        bb.read_edges(p, "mm")
    assert ei.value.code == -4 and frag in str(ei.value)


def test_bin_errors(tmp_path):
    bb = _bb()
    p = tmp_path / "odd.bin"
    p.write_bytes(b"\x00" * 12)
    with pytest.raises(bb.BBTCError) as ei:
        bb.read_edges(p, "bin")
    assert ei.value.code == -4
    p.write_bytes(np.array([0, 1, 0xFFFFFFFF, 2], "<u4").tobytes())
    with pytest.raises(bb.BBTCError) as ei:
        bb.read_edges(p, "bin")
    assert ei.value.code == -5


def test_missing_file_is_eio(tmp_path):
    bb = _bb()
    with pytest.raises(bb.BBTCError) as ei:
        bb.read_edges(tmp_path / "nope.txt", "text")
    assert ei.value.code == -3


def test_bin_roundtrip_rmat(tmp_path):
    """The generators' binary pair format round-trips a seeded R-MAT list exactly."""
    bb = _bb()
    s, d = inputs.rmat(10, 16, seed=3)
    p = tmp_path / "r.bin"
    write_bin(p, s, d)
    rs, rd, _ = bb.read_edges(p, "bin")
    assert np.array_equal(rs, s) and np.array_equal(rd, d)


@pytest.mark.gpu
@pytest.mark.parametrize("fmt", ["text", "mm", "bin"])
def test_graph_load_counts_karate(tmp_path, fmt):
    bb = _bb()
    s, d = inputs.karate()
    path = tmp_path / f"k.{fmt}"
    {"text": lambda: write_text(path, s, d), "mm": lambda: write_mm(path, s, d, 34),
     "bin": lambda: write_bin(path, s, d)}[fmt]()
    ctx = bb.Context(0)
    g = bb.Graph.load(ctx, path, fmt)
    assert g.n == 34 and g.m == 78
    total, per_task = bb.Plan(ctx, g, 2).count()
    assert total == 45 and per_task.tolist() == [1, 11, 28, 5]


def test_text_and_mm_roundtrip_random(tmp_path):
    """A seeded 200 K-pair list written by numpy as TSV and as MatrixMarket reads back
    exactly (ids up to 2^32 - 2, the largest the ABI accepts)."""
    bb = _bb()
    rng = np.random.default_rng(11)
    s = rng.integers(0, 1 << 20, size=200_000, dtype=np.uint64).astype(np.uint32)
    d = rng.integers(0, 1 << 20, size=200_000, dtype=np.uint64).astype(np.uint32)
    s[:3] = [0xFFFFFFFE, 0, 7]
    d[:3] = [1, 0xFFFFFFFE, 7]
    p = tmp_path / "r.tsv"
    np.savetxt(p, np.stack([s, d], 1), fmt="%d", delimiter="\t", header="random", comments="# ")
    rs, rd, _ = bb.read_edges(p, "text")
    assert np.array_equal(rs, s) and np.array_equal(rd, d)
    n = int(max(s.max(), d.max())) + 1
    m = tmp_path / "r.mtx"
    with open(m, "w") as f:
        f.write(f"%%MatrixMarket matrix coordinate integer general\n{n} {n} {len(s)}\n")
        np.savetxt(f, np.stack([s.astype(np.uint64) + 1, d.astype(np.uint64) + 1, np.ones_like(s)], 1), fmt="%d")
    ms, md, nh = bb.read_edges(m, "mm")
    assert nh == n and np.array_equal(ms, s) and np.array_equal(md, d)


def test_edges_map_matches_read(tmp_path):
    """bbtc_edges_map (memory-mapped host source): the mapping of a binary
    file holds exactly the pairs bbtc_edges_read parses; empty and odd-sized files."""
    bb = _bb()
    s, d = inputs.rmat(11, 16, seed=5)
    p = tmp_path / "m.bin"
    write_bin(p, s, d)
    with bb.EdgeMap(p) as m:
        assert m.n_edges == len(s)
        assert np.array_equal(m.pairs[:, 0], s) and np.array_equal(m.pairs[:, 1], d)
    e = tmp_path / "empty.bin"
    e.write_bytes(b"")
    with bb.EdgeMap(e) as m:
        assert m.n_edges == 0 and m.pairs.shape == (0, 2)
    o = tmp_path / "odd.bin"
    o.write_bytes(b"\x00" * 12)
    with pytest.raises(bb.BBTCError) as ei:
        bb.EdgeMap(o)
    assert ei.value.code == -4
    with pytest.raises(bb.BBTCError) as ei:
        bb.EdgeMap(tmp_path / "nope.bin")
    assert ei.value.code == -3


@pytest.mark.gpu
def test_graph_from_pairs_and_mapped_file(tmp_path):
    """Interleaved pairs (host numpy, a memory-mapped file, a CUDA tensor) build the same
    graph as the split arrays: same n, m and the oracle's per-task counts."""
    import torch
    bb = _bb()
    s, d = inputs.rmat(14, 16, seed=4)
    p = tmp_path / "r14.bin"
    write_bin(p, s, d)
    og = oracle.OracleGraph(s, d, 1 << 14)
    ot, opt, _, _ = og.count(5)
    ctx = bb.Context(0)
    pairs = np.stack([s, d], axis=1)
    graphs = [bb.Graph.from_pairs(ctx, pairs, 1 << 14),
              bb.Graph.load_mapped(ctx, p, 1 << 14),
              bb.Graph.from_pairs(ctx, torch.from_numpy(pairs.view(np.int32)).cuda(), 1 << 14)]
    with bb.EdgeMap(p) as m:
        graphs.append(bb.Graph.from_pairs(ctx, m.pairs, 1 << 14))
    for g in graphs:
        assert g.size() == (og.n, og.m)
        total, per_task = bb.Plan(ctx, g, 5).count()
        assert total == ot and np.array_equal(per_task, opt)
