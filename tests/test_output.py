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
