"""Caller-side driver over the streaming C ABI (submit -> poll -> release).

This is what a user of libsurge writes: it feeds (partition_id, token_ids, lengths) in arrival
order, polls completed pieces and copies them into per-partition matrices.  All encoding work
happens inside libsurge.so.
"""
from __future__ import annotations

import numpy as np

from . import native as N


class SurgeEncoder:
    def __init__(self, enc_cfg, weights_blob, b_min: int, b_max: int, **cfg_kw):
        self.enc_cfg = enc_cfg
        self.cfg = N.make_config(enc_cfg, b_min, b_max, **cfg_kw)
        self.h = N.surge_create(self.cfg, weights_blob, **({"n_weights": cfg_kw.get("n_weights")}
                                                           if "n_weights" in cfg_kw else {}))

    def close(self):
        if self.h is not None:
            N.surge_destroy(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _collect(self, out, recs, keep: bool):
        for r in recs:
            if keep:
                M = out.setdefault(int(r.partition_id), [r.partition_rows, {}])
                M[1][int(r.row_begin)] = N.flushed_array(r).copy()
            N.surge_release(self.h, r)

    def run(self, partitions, keep: bool = True, poll_every: int = 1):
        """Stream (key, ids, lengths) triples through the library; returns {key: [n_k x d] float32}
        (pieces of this rank only when world_size > 1: {key: {row_begin: array}} is kept in .pieces)."""
        out = {}
        for i, (key, ids, lengths) in enumerate(partitions):
            N.surge_submit_partition(self.h, key, ids, lengths)
            if i % poll_every == 0:
                self._collect(out, N.surge_poll_flushed(self.h, 4096, 0), keep)
        N.surge_finish(self.h)
        while N.surge_pending(self.h) > 0:
            self._collect(out, N.surge_poll_flushed(self.h, 4096, 50), keep)
        self._collect(out, N.surge_poll_flushed(self.h, 4096, 0), keep)
        self.pieces = out
        if not keep:
            return None
        res = {}
        d = self.enc_cfg.hidden
        for key, (n, parts) in out.items():
            if sum(p.shape[0] for p in parts.values()) == n:
                res[key] = np.concatenate([parts[b] for b in sorted(parts)]) if n else np.zeros((0, d), np.float32)
        return res

    def stats(self):
        return N.surge_get_stats(self.h)

    def superbatches(self):
        st = self.stats()
        return [dict(N.surge_get_superbatch(self.h, i), members=N.surge_get_superbatch_members(self.h, i))
                for i in range(st["superbatches"])]


def stream(N, h, partitions, consume=None, poll_batch: int = 4096) -> int:
    """Submit (key, ids, lengths) in arrival order on this thread while a second thread polls and
    releases the completed pieces (the threading model of include/surge.h: one producer; poll /
    release from any thread).  A submit that blocks on backpressure -- or on a long run of Safety
    flushes under SURGE_BMAX_SPLIT -- therefore never holds back the release of finished pieces, so
    their pinned buffers return to the pool instead of new ones being page-locked.  `consume(rec)`
    (optional) sees every piece before it is released.  Returns the number of rows delivered."""
    import threading
    done = threading.Event()
    rows = [0]
    err = []

    def poller():
        try:
            while True:
                recs = N.surge_poll_flushed(h, poll_batch, 5)
                for r in recs:
                    rows[0] += int(r.n_rows)
                    if consume is not None:
                        consume(r)
                    N.surge_release(h, r)
                if not recs and done.is_set() and N.surge_pending(h) == 0:
                    for r in N.surge_poll_flushed(h, poll_batch, 0):
                        rows[0] += int(r.n_rows)
                        if consume is not None:
                            consume(r)
                        N.surge_release(h, r)
                    return
        except BaseException as e:   # noqa: BLE001 -- re-raised on the submitting thread
            err.append(e)

    t = threading.Thread(target=poller, daemon=True)
    t.start()
    try:
        for key, ids, lengths in partitions:
            N.surge_submit_partition(h, key, ids, lengths)
        N.surge_finish(h)
    finally:
        done.set()
        t.join()
    if err:
        raise err[0]
    return rows[0]
