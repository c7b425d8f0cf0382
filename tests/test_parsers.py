"""Text parsers (parse_edge_list / parse_matrix_market, reference
proj/src/graph.cpp:52-157), now parsed in parallel chunks: the result and the
first error (class, line number) must be what the serial reference grammar
gives, including for inputs large enough to be cut into several chunks."""
import numpy as np
import pytest

import paper_2007_11111_b200 as gt


def _edge_text(m, n, seed, noise=True):
    rng = np.random.default_rng(seed)
    u = rng.integers(0, n, m)
    v = rng.integers(0, n, m)
    lines = []
    for i in range(m):
        if noise and i % 97 == 0:
            lines.append("# comment %d" % i)
        if noise and i % 89 == 0:
            lines.append("   ")
        if noise and i % 83 == 0:
            lines.append("% another comment")
        sep = "\t" if i % 3 == 0 else "  "
        end = "\r" if i % 5 == 0 else ""
        lines.append(f"  {u[i]}{sep}{v[i]}{end}")
    return "\n".join(lines), u, v


def _same_edges(text, fmt, u, v):
    """The parallel host parser returns exactly the pairs, in input order."""
    e, _, _ = gt.parse_text(text, fmt)
    np.testing.assert_array_equal(e[:, 0], u)
    np.testing.assert_array_equal(e[:, 1], v)


def test_edge_list_multi_chunk():
    text, u, v = _edge_text(400_000, 50_000, 3)  # several MB: several chunks
    assert len(text) > 4 << 20
    _same_edges(text, "edges", u, v)


@pytest.mark.gpu
def test_edge_list_graph_via_device_ingest():
    text, u, v = _edge_text(200_000, 30_000, 5)
    g = gt.from_text(text, "edges")
    ref = gt.from_edges(np.stack([u, v], axis=1).astype(np.int64), 30_000)
    assert (g.num_vertices, g.num_edges) == (ref.num_vertices, ref.num_edges)
    for x in range(0, 30_000, 150):
        assert g.neighbors(x) == ref.neighbors(x)


def test_edge_list_first_error_line():
    text, _, _ = _edge_text(400_000, 50_000, 4, noise=False)
    lines = text.split("\n")
    # errors in a late chunk and an early chunk: the early one is reported
    lines[350_000] = "1 2 3"
    lines[123_456] = "7 x"
    with pytest.raises(gt.ParseError, match=r"^line 123457: malformed vertex id 'x'$"):
        gt.parse_text("\n".join(lines), "edges")
    lines[123_456] = "7 8"
    with pytest.raises(gt.ParseError, match=r"^line 350001: expected 'u v', got 3 tokens$"):
        gt.parse_text("\n".join(lines), "edges")
    lines[350_000] = "-1 2"
    with pytest.raises(gt.ParseError, match=r"^line 350001: negative vertex id$"):
        gt.parse_text("\n".join(lines), "edges")


def _mtx(entries, n, nnz=None, field="pattern", extra=()):
    head = [f"%%MatrixMarket matrix coordinate {field} general", "% c", "",
            f"{n} {n} {len(entries) if nnz is None else nnz}"]
    body = []
    for k, (i, j) in enumerate(entries):
        if k % 101 == 0:
            body.append("% mid comment")
        body.append(f"{i + 1} {j + 1}" + (" 1.5" if field != "pattern" else ""))
    return "\n".join(head + body + list(extra))


def test_matrix_market_multi_chunk_and_truncation():
    rng = np.random.default_rng(7)
    n, m = 60_000, 500_000
    u, v = rng.integers(0, n, m), rng.integers(0, n, m)
    ents = list(zip(u.tolist(), v.tolist()))
    _same_edges(_mtx(ents, n, field="real"), "mtx", u, v)
    e, declared, sym = gt.parse_text(_mtx(ents, n, field="real"), "mtx")
    assert declared == n and not sym
    # only nnz entries are read: trailing garbage after them is never parsed
    _same_edges(_mtx(ents, n, nnz=m - 10, extra=["garbage here", "1"]), "mtx", u[: m - 10],
                v[: m - 10])


def test_matrix_market_errors():
    ents = [(k % 50, (k * 7) % 50) for k in range(300_000)]
    text = _mtx(ents, 50)
    lines = text.split("\n")
    # header: 4 lines; body: a comment before every 101 entries
    bad = 4 + 250_000 + 250_000 // 101 + 1  # 1-based line of entry 250000
    lines[bad - 1] = "3 99"
    with pytest.raises(gt.ParseError, match=rf"^line {bad}: entry \(3,99\) out of declared range 50$"):
        gt.parse_text("\n".join(lines), "mtx")
    with pytest.raises(gt.ParseError, match=r"unexpected end of stream: got 300000 of 300001 entries"):
        gt.parse_text(_mtx(ents, 50, nnz=300_001), "mtx")
    with pytest.raises(gt.ParseError, match=r"^line 1: only coordinate format is supported, got 'array'$"):
        gt.parse_text("%%MatrixMarket matrix array real general\n2 2\n", "mtx")
    with pytest.raises(gt.ParseError, match=r"^line 4: expected 2 tokens per entry$"):
        gt.parse_text("%%MatrixMarket matrix coordinate pattern general\n3 3 2\n1 2\n# not a comment\n", "mtx")
