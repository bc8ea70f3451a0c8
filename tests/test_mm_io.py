"""Matrix Market ingestion: sb_read_matrix_market /
sb_write_matrix_market restate inc/mm_io.hpp and must agree bit for bit with
the reference's own reader (oracle/_ref), duplicates and symmetric expansion
included, with the reference's error messages. CPU only."""
import numpy as np
import pytest

from helpers import random_sparse


def _mtx(tmp_path, name, text):
    p = tmp_path / name
    p.write_text(text)
    return p


CASES = {
    "general_dups.mtx": "%%MatrixMarket matrix coordinate real general\n% comment\n\n4 5 9\n"
                        "1 1 1.5\n2 3 -2.25\n1 1 0.1\n4 5 3e-3\n2 3 1e-17\n2 3 7.0\n3 1 -0.0\n4 4 2\n1 2 0.3\n",
    "symmetric.mtx": "%%MatrixMarket matrix coordinate real symmetric\n5 5 7\n1 1 4\n2 1 -1\n2 2 4\n3 2 -1\n"
                     "3 3 4\n5 3 0.5\n5 5 4\n",
    "empty_rows.mtx": "%%MatrixMarket matrix coordinate real general\n6 6 3\n6 6 1\n1 1 2\n6 6 1e-300\n",
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_reader_matches_reference(sp, ref, tmp_path, name):
    p = _mtx(tmp_path, name, CASES[name])
    A = sp.read_matrix_market(p)
    rp, ci, v = ref.read_matrix_market(p)
    assert np.array_equal(A.row_ptr().astype(np.int64), rp.astype(np.int64))
    assert np.array_equal(A.col_idx(), ci)
    assert np.array_equal(A.values().view(np.uint64), v.view(np.uint64))


def test_round_trip_through_reference(sp, ref, tmp_path):
    A = random_sparse(sp, 60, 11, 0.1, False)
    ours, theirs = tmp_path / "ours.mtx", tmp_path / "theirs.mtx"
    sp.write_matrix_market(A, ours)
    ref.write_matrix_market(A, theirs)
    assert ours.read_text() == theirs.read_text()
    B = sp.read_matrix_market(ours)
    assert B == A


@pytest.mark.parametrize("text,msg", [
    ("%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n", "only coordinate format"),
    ("%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n", "is not real"),
    ("%%MatrixMarket matrix coordinate real hermitian\n1 1 1\n1 1 1\n", "is not general or symmetric"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n", "expected 2 entries, found 1"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1\n", "out of bounds for 2x2"),
    ("hello\n", "malformed header"),
])
def test_errors_match_reference(sp, ref, tmp_path, text, msg):
    p = _mtx(tmp_path, "bad.mtx", text)
    with pytest.raises(Exception) as ours:
        sp.read_matrix_market(p)
    with pytest.raises(Exception) as theirs:
        ref.read_matrix_market(p)
    assert msg in str(ours.value) and msg in str(theirs.value)
    assert str(ours.value).split(": ", 1)[-1] == str(theirs.value).split(": ", 1)[-1]
