"""NEXT N4 output side (paper_2605_01060_b200/output.py): zero-copy Arrow, Alg. 2 async
upload with retry, lifetime rule, idempotent resume, eq:overlap."""
import numpy as np
import pytest

from paper_2605_01060_b200 import output as O


def test_arrow_zero_copy_roundtrip():
    rows = np.random.default_rng(0).standard_normal((1000, 384)).astype(np.float32)
    t = O.arrow_table(rows)
    col = t.column("embedding").chunk(0)
    assert col.type.list_size == 384 and len(col) == 1000
    # the values buffer aliases the numpy rows: no copy (O(1) allocations, lst:zerocopy)
    assert col.values.buffers()[1].address == rows.ctypes.data
    back = O.deserialize(O.serialize(rows))
    assert np.array_equal(back, rows)
    assert O.deserialize(O.serialize(np.zeros((0, 64), np.float32))).shape == (0, 64)


class Flaky(O.LocalStorage):
    def __init__(self, root, fail_first=0, fail_keys=()):
        super().__init__(root)
        self.fail_first, self.fail_keys, self.calls = fail_first, set(fail_keys), 0

    def write(self, path, data):
        self.calls += 1
        if self.calls <= self.fail_first or any(f"/{k:020d}/" in f"/{path}" for k in self.fail_keys):
            raise OSError("transient")
        super().write(path, data)


def test_upload_retry_release_and_resume(tmp_path):
    released = []
    st = Flaky(str(tmp_path), fail_first=2, fail_keys={7})
    up = O.AsyncUploader(st, "run1", workers=4, backoff_s=0.001, release=released.append)
    rng = np.random.default_rng(1)
    data = {k: rng.standard_normal((n, 8)).astype(np.float32) for k, n in [(3, 5), (5, 0), (7, 4), (9, 11)]}
    # partition 9 in two pieces (as with world_size > 1)
    for k, m in data.items():
        if k == 9:
            up.submit(9, 0, 11, m[:6], piece=("p", 9, 0))
            up.submit(9, 6, 11, m[6:], piece=("p", 9, 6))
        else:
            up.submit(k, 0, m.shape[0], m, piece=("p", k, 0))
    up.close()
    # every piece released exactly once, even the one that failed all 3 attempts
    assert sorted(released) == sorted([("p", 3, 0), ("p", 5, 0), ("p", 7, 0), ("p", 9, 0), ("p", 9, 6)])
    assert [p for p, _ in up.failures] == [O.piece_path("run1", 7, 0)]
    assert O.completed(st, "run1") == {3, 5, 9}
    got = np.concatenate([O.deserialize(st.read(O.piece_path("run1", 9, b))) for b in (0, 6)])
    assert np.array_equal(got, data[9])
    assert O.completed(st, "other") == set()


def test_overlap_ratio():
    assert O.overlap_ratio(2.0, 0.5, 0.5) == 1.0                    # I/O hidden behind encode
    assert O.overlap_ratio(1.0, 1.0, 1.0) == pytest.approx(0.5)     # half of the I/O exposed
    assert O.overlap_ratio(0.0, 1.0, 0.0) == 0.0
    assert O.overlap_ratio(1.0, 0.0, 0.0) == 1.0


def test_two_uploaders_piece_markers_and_stale_pieces(tmp_path):
    """world_size 2: each rank has its own uploader and writes only its LPT pieces.  Completion is per
    piece (markers), so a partition split across ranks is complete once both ranks' pieces are durable
    -- no process ever sees all of its rows.  A stale piece left by an earlier run (other piece
    boundaries) is ignored by read_partition and removed by prepare_resume with its incomplete
    partition."""
    st = O.LocalStorage(str(tmp_path))
    rng = np.random.default_rng(2)
    m = rng.standard_normal((10, 4)).astype(np.float32)
    r0 = O.AsyncUploader(st, "run", workers=2)
    r1 = O.AsyncUploader(st, "run", workers=2)
    r0.submit(1, 0, 10, m[:3])           # partition 1: rows [0,3) on rank 0, [3,10) on rank 1
    r1.submit(1, 3, 10, m[3:])
    r1.submit(2, 0, 10, m[:4])           # partition 2: rank 0's piece [4,10) never arrives (crash)
    r0.close()
    r1.close()
    assert O.completed(st, "run") == {1}
    assert np.array_equal(O.read_partition(st, "run", 1), m)
    with pytest.raises(KeyError):
        O.read_partition(st, "run", 2)
    # a stale unmarked piece next to a complete partition is ignored by the reader
    st.write(O.piece_path("run", 1, 5), O.serialize(m[5:]))
    assert np.array_equal(O.read_partition(st, "run", 1), m)
    # resume: complete partitions are kept, incomplete ones are wiped before the re-run
    assert O.prepare_resume(st, "run") == {1}
    assert st.list("run/" + f"{2:020d}") == []
    up = O.AsyncUploader(st, "run", workers=2)
    up.submit(2, 0, 10, m[:5])           # re-run with different boundaries
    up.submit(2, 5, 10, m[5:])
    up.close()
    assert O.completed(st, "run") == {1, 2}
    assert np.array_equal(O.read_partition(st, "run", 2), m)
