"""Output side of SURGE, host-only, over the streaming C ABI:

* zero-copy Arrow serialisation of a polled piece (`lst:zerocopy`): the library-owned
  pinned rows are wrapped as `FixedSizeListArray(float32, d)` without copying;
* asynchronous upload with retry (Alg. 2): a thread pool of W workers, up to 3 attempts with
  2^a s backoff (scaled by `backoff_s` for tests), non-blocking submit;
* the buffer lifetime rule: the polled buffer must outlive every upload that references it --
  the upload closure owns the piece and calls `surge_release` when the write is done;
* idempotent resume: the output path is deterministic (`<run_id>/<key>/<row_begin>.arrow`);
  every durable piece gets a marker `_PIECE.<row_begin>.<n_rows>.<partition_rows>` written after its
  data, so completion is decided per piece, by whichever process (rank) uploaded it: a partition is
  complete when its markers tile [0, partition_rows) exactly.  `completed()` is the O(P) scan a
  restarted run uses to skip partitions; `prepare_resume()` also deletes the files of incomplete
  partitions (their piece boundaries may differ in the re-run), and `read_partition()` reads only
  marked pieces;
* the I/O overlap ratio rho (`eq:overlap`) per SuperBatch.

Tokenisation, real object stores and their latency profiles stay out of scope (SURVEY.md §8 OUT).
"""
from __future__ import annotations

import io
import os
import threading
import time
from concurrent.futures import Future, ThreadPoolExecutor

import numpy as np
import pyarrow as pa
import pyarrow.ipc as ipc


def arrow_table(rows: np.ndarray) -> pa.Table:
    """`lst:zerocopy`: [n x d] float32 C-contiguous -> table with one FixedSizeList column;
    O(1) allocations, the data buffer aliases `rows`."""
    assert rows.dtype == np.float32 and rows.flags["C_CONTIGUOUS"] and rows.ndim == 2
    flat = pa.array(rows.ravel(), type=pa.float32())          # ravel(): a view; pa.array wraps it
    col = pa.FixedSizeListArray.from_arrays(flat, rows.shape[1])
    return pa.table({"embedding": col})


def serialize(rows: np.ndarray) -> bytes:
    sink = io.BytesIO()
    t = arrow_table(rows)
    with ipc.new_file(sink, t.schema) as w:
        w.write_table(t)
    return sink.getvalue()


def deserialize(data: bytes) -> np.ndarray:
    t = ipc.open_file(pa.BufferReader(data)).read_all()
    col = t.column("embedding").combine_chunks()
    d = col.type.list_size
    return np.asarray(col.flatten()).reshape(-1, d)


class LocalStorage:
    """Directory-backed object store: write(path, bytes) (atomic rename), exists(path), list(prefix)."""

    def __init__(self, root: str):
        self.root = root

    def write(self, path: str, data: bytes) -> None:
        full = os.path.join(self.root, path)
        os.makedirs(os.path.dirname(full), exist_ok=True)
        tmp = f"{full}.tmp{threading.get_ident()}"
        with open(tmp, "wb") as f:
            f.write(data)
        os.replace(tmp, full)

    def read(self, path: str) -> bytes:
        with open(os.path.join(self.root, path), "rb") as f:
            return f.read()

    def delete(self, path: str) -> None:
        try:
            os.remove(os.path.join(self.root, path))
        except FileNotFoundError:
            pass

    def exists(self, path: str) -> bool:
        return os.path.exists(os.path.join(self.root, path))

    def list(self, prefix: str):
        base = os.path.join(self.root, prefix)
        if not os.path.isdir(base):
            return []
        return sorted(os.listdir(base))


def piece_path(run_id: str, key: int, row_begin: int) -> str:
    return f"{run_id}/{key:020d}/{row_begin:012d}.arrow"


def marker_path(run_id: str, key: int, row_begin: int, n_rows: int, partition_rows: int) -> str:
    return f"{run_id}/{key:020d}/_PIECE.{row_begin:012d}.{n_rows}.{partition_rows}"


def _pieces(storage, run_id: str, key_dir: str):
    """Marked pieces of one partition directory: sorted [(row_begin, n_rows, partition_rows)]."""
    out = []
    for f in storage.list(f"{run_id}/{key_dir}"):
        if f.startswith("_PIECE."):
            _, b, n, rows = f.split(".")
            out.append((int(b), int(n), int(rows)))
    return sorted(out)


def _covers(pieces) -> bool:
    """The marked pieces tile [0, partition_rows) exactly (in whatever process they were written)."""
    if not pieces:
        return False
    rows = pieces[0][2]
    at = 0
    for b, n, r in pieces:
        if r != rows or b != at:
            return False
        at += n
    return at == rows


def completed(storage, run_id: str) -> set:
    """Resume scan: keys whose every row is durable, from the per-piece markers of all ranks."""
    return {int(name) for name in storage.list(run_id) if _covers(_pieces(storage, run_id, name))}


def prepare_resume(storage, run_id: str) -> set:
    """Before a restarted run (once, on one rank): the complete partitions (to skip), after deleting the
    files of every incomplete one -- the re-run may cut it into different pieces, and a stale piece
    must not survive next to the new ones."""
    done = set()
    for name in storage.list(run_id):
        if _covers(_pieces(storage, run_id, name)):
            done.add(int(name))
        else:
            for f in storage.list(f"{run_id}/{name}"):
                storage.delete(f"{run_id}/{name}/{f}")
    return done


def read_partition(storage, run_id: str, key: int) -> np.ndarray:
    """E_k of a complete partition: its marked pieces in row order (unmarked files are ignored)."""
    pcs = _pieces(storage, run_id, f"{key:020d}")
    if not _covers(pcs):
        raise KeyError(f"partition {key} is not complete")
    parts = [deserialize(storage.read(piece_path(run_id, key, b))) for b, n, _ in pcs if n > 0]
    return np.concatenate(parts) if parts else np.zeros((0, 0), np.float32)


class AsyncUploader:
    """Alg. 2: non-blocking submit of (path, rows) to a W-worker pool, 3 attempts, 2^a backoff.

    `release` is called with the piece once its upload finished (success or final failure) -- the
    lifetime rule of P:413 (the rows alias library-owned memory until then)."""

    def __init__(self, storage, run_id: str, workers: int = 32, attempts: int = 3, backoff_s: float = 1.0,
                 release=None):
        self.storage, self.run_id = storage, run_id
        self.attempts, self.backoff_s = attempts, backoff_s
        self.release = release
        self.pool = ThreadPoolExecutor(max_workers=workers)
        self.pending: dict[str, Future] = {}
        self.lock = threading.Lock()
        self.t_ser = self.t_upl = 0.0
        self.failures: list = []

    def submit(self, key: int, row_begin: int, partition_rows: int, rows: np.ndarray, piece=None) -> Future:
        path = piece_path(self.run_id, key, row_begin)
        fut = self.pool.submit(self._upload_with_retry, path, key, partition_rows, rows, piece)
        with self.lock:
            self.pending[path] = fut
        return fut

    def _write_retry(self, path: str, data: bytes):
        """UploadWithRetry (Alg. 2): up to `attempts` tries, sleeping backoff 2^a between them."""
        err = None
        for a in range(self.attempts):
            try:
                self.storage.write(path, data)
                return None
            except Exception as e:              # noqa: BLE001 -- storage errors are retried
                err = e
                if a + 1 < self.attempts:
                    time.sleep(self.backoff_s * 2 ** a)
        with self.lock:
            self.failures.append((path, repr(err)))
        return err

    def _upload_with_retry(self, path, key, partition_rows, rows, piece):
        try:
            t0 = time.perf_counter()
            data = serialize(rows)
            t1 = time.perf_counter()
            err = self._write_retry(path, data)
            t2 = time.perf_counter()
            with self.lock:
                self.t_ser += t1 - t0
                self.t_upl += t2 - t1
            if err is not None:
                return False
            # the piece is durable: its marker makes it count, whichever rank wrote the other pieces
            row_begin = int(path.rsplit("/", 1)[1].split(".")[0])
            return self._write_retry(marker_path(self.run_id, key, row_begin, rows.shape[0], partition_rows),
                                     b"") is None
        finally:
            if self.release is not None and piece is not None:
                self.release(piece)

    def drain(self):
        with self.lock:
            futs = list(self.pending.values())
        for f in futs:
            f.result()

    def close(self):
        self.drain()
        self.pool.shutdown(wait=True)


def overlap_ratio(t_enc: float, t_ser: float, t_upl: float) -> float:
    """eq:overlap: rho = 1 - max(0, (t_ser + t_upl) - t_enc) / (t_ser + t_upl)."""
    io_t = t_ser + t_upl
    if io_t <= 0:
        return 1.0
    return 1.0 - max(0.0, io_t - t_enc) / io_t


def encode_to_storage(N, h, partitions, uploader: AsyncUploader, skip: set | None = None) -> int:
    """Stream (key, ids, lengths) through libsurge and upload every polled piece asynchronously;
    partitions in `skip` (a resume scan) are not submitted.  Returns the number of submitted texts."""
    skip = skip or set()
    n = 0

    def hand_off(recs):
        for r in recs:
            uploader.submit(int(r.partition_id), int(r.row_begin), int(r.partition_rows), N.flushed_array(r), r)

    for key, ids, lengths in partitions:
        if int(key) in skip:
            continue
        N.surge_submit_partition(h, key, ids, lengths)
        n += len(lengths)
        hand_off(N.surge_poll_flushed(h, 4096, 0))
    N.surge_finish(h)
    while N.surge_pending(h) > 0:
        hand_off(N.surge_poll_flushed(h, 4096, 20))
    hand_off(N.surge_poll_flushed(h, 4096, 0))
    uploader.drain()
    return n
