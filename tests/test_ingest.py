"""Native ratings-text ingest (libmfg_b200 mfg_parse_ratings, host code) against
the reference's parsing rules restated in data._parse_stream
(mfg/data.py:164-200): identical values on plain files, and on any line the
fast path does not take, the reference's own acceptance or exact error."""

import io

import numpy as np
import pytest

from paper_2204_14067_b200 import data as D


def _ref(buf: bytes):
    return D._parse_stream(io.BytesIO(buf), "training data")


def _native(buf: bytes):
    return D._parse_native(buf)


def _random_file(rng, n, messy=True):
    lines = []
    for _ in range(n):
        u, i = rng.integers(1, 10**6, size=2)
        r = rng.choice(["%d" % rng.integers(1, 6), "%.1f" % (rng.random() * 5), "%.17g" % rng.normal(3, 2),
                        "%de0" % rng.integers(1, 6), "%d." % rng.integers(1, 6), ".%d" % rng.integers(0, 10),
                        "+%.3f" % rng.random(), "-%.2e" % rng.random()])
        sep = rng.choice([" ", "\t", "  ", " \t "]) if messy else " "
        fields = [str(u), str(i), r]
        if rng.random() < 0.5:
            fields.append(str(rng.integers(10**9, 2 * 10**9)))
        line = sep.join(fields)
        if messy and rng.random() < 0.1:
            line = "  " + line + " \r"
        lines.append(line)
        if messy and rng.random() < 0.05:
            lines.append("   ")
    return ("\n".join(lines) + ("\n" if rng.random() < 0.5 else "")).encode()


@pytest.mark.parametrize("n", [1, 7, 1000, 120_000])
def test_native_parser_matches_reference_rules(n):
    rng = np.random.default_rng(n)
    buf = _random_file(rng, n)
    got = _native(buf)
    assert got is not None
    want = _ref(buf)
    for g, w in zip(got, want):
        assert g.dtype == w.dtype and np.array_equal(g, w)


def test_native_parser_multithreaded_chunks():
    """> 8 MiB: several threads, chunk cuts inside the file; same result."""
    rng = np.random.default_rng(3)
    buf = _random_file(rng, 400_000, messy=False)
    assert len(buf) > 8 << 20
    got = _native(buf)
    want = _ref(buf)
    for g, w in zip(got, want):
        assert np.array_equal(g, w)
    assert D._lib.lib().mfg_count_lines(buf, len(buf)) >= got[0].size


@pytest.mark.parametrize("line, outcome", [
    (b"1_0 2 3", (10, 2, 3.0)),          # Python int() accepts underscores
    (b"1 2 inf", (1, 2, float("inf"))),  # float('inf')
    (b"1 2 1e999", (1, 2, float("inf"))),
    (b"+1 2 3", (1, 2, 3.0)),
    (b"-1 2 3", "positive"),
    (b"0 2 3", "positive"),
    (b"1 2", "expected 3 or 4 fields, got 2"),
    (b"1 2 3 4 5", "expected 3 or 4 fields, got 5"),
    (b"1 x 3", "cannot parse"),
    (b"1 2 3.5.1", "cannot parse"),
])
def test_odd_lines_take_the_reference_path(line, outcome):
    buf = b"5 6 4\n" + line + b"\n7 8 1\n"
    assert _native(buf) is None           # the fast path declines
    if isinstance(outcome, tuple):
        users, items, ratings = D._parse_source(buf, "training data")
        assert (users[1], items[1], ratings[1]) == outcome
        assert np.array_equal(users, _ref(buf)[0])
    else:
        with pytest.raises(D.ParseError) as err:
            D._parse_source(buf, "training data")
        assert "line 2" in str(err.value) and outcome in str(err.value)


def test_empty_and_blank_inputs():
    with pytest.raises(D.EmptyDatasetError):
        D._parse_source(b"", "training data")
    with pytest.raises(D.EmptyDatasetError):
        D._parse_source(b"  \n\t\n", "training data")


def test_instance_file_roundtrip(tmp_path):
    rng = np.random.default_rng(5)
    nnz = 1001
    rows = rng.integers(0, 300, nnz)
    cols = rng.integers(0, 500, nnz)
    for vals in (rng.normal(size=nnz), rng.normal(size=nnz).astype(np.float32)):
        split = D.EvalSplit(300, 500, rng.integers(0, 300, 17), rng.integers(0, 500, 17), rng.normal(size=17), True)
        p = tmp_path / "x.mfgo"
        D.write_instance(p, 300, 500, rows, cols, vals, True, np.arange(300) * 3 + 1, np.arange(500) + 7, split)
        a = D.read_instance(p)
        assert (a["m"], a["n"], a["transposed"]) == (300, 500, True)
        assert np.array_equal(a["rows"], rows) and np.array_equal(a["cols"], cols)
        assert a["vals"].dtype == vals.dtype and np.array_equal(a["vals"], vals)
        assert np.array_equal(a["row_ids"], np.arange(300) * 3 + 1)
        assert np.array_equal(a["col_ids"], np.arange(500) + 7)
        assert np.array_equal(a["test_rows"], split.rows) and np.array_equal(a["test_vals"], split.vals)
    # no ids, no split
    D.write_instance(p, 3, 4, [0, 2], [1, 3], [1.0, 2.0])
    a = D.read_instance(p)
    assert a["row_ids"].size == 0 and a["test_rows"].size == 0 and not a["transposed"]


def test_instance_file_errors(tmp_path):
    p = tmp_path / "bad.mfgo"
    p.write_bytes(b"NOTMAGIC" + b"\0" * 64)
    with pytest.raises(D.DatasetError):
        D.read_instance(p)
    D.write_instance(p, 3, 4, [0, 2], [1, 3], [1.0, 2.0])
    p.write_bytes(p.read_bytes()[:-12])
    with pytest.raises(D.DatasetError):
        D.read_instance(p)


@pytest.mark.gpu
def test_ratings_text_to_instance_on_gpu(tmp_path):
    """load_ratings (native parse + device build) -> save_instance ->
    load_instance reproduces the ObservationSet, id maps and test split."""
    rng = np.random.default_rng(9)
    users = rng.integers(1, 400, 5000) * 7
    items = rng.integers(1, 90, 5000) * 3
    key = np.unique(users * 1000 + items)
    users, items = key // 1000, key % 1000
    r = rng.integers(1, 6, users.size)
    text = "".join(f"{u}\t{i}\t{x}\t{123}\n" for u, i, x in zip(users, items, r)).encode()
    test = "".join(f"{u} {i} {x}\n" for u, i, x in zip(users[:50], items[:50], r[:50])).encode()
    obs, split = D.load_ratings(text, test)
    assert obs.transposed  # fewer items than users -> m <= n by transposing
    p = tmp_path / "i.mfgo"
    D.save_instance(p, obs, split)
    obs2, split2 = D.load_instance(p)
    assert (obs2.m, obs2.n, obs2.transposed) == (obs.m, obs.n, obs.transposed)
    assert np.array_equal(obs2.rows, obs.rows) and np.array_equal(obs2.cols, obs.cols)
    assert np.array_equal(obs2.vals, obs.vals)
    assert np.array_equal(obs2.row_ids, obs.row_ids) and np.array_equal(obs2.col_ids, obs.col_ids)
    assert np.array_equal(split2.rows, split.rows) and np.array_equal(split2.vals, split.vals)
