"""Oracle over many host cores.  TEST INFRASTRUCTURE ONLY (tests/, bench.py cpu_baseline).

The encoder definition is oracle.encoder.Encoder.encode_text, one text at a time; this module only
spreads independent texts over worker processes (fork; one BLAS thread each), so a 16,384-row
parity sample (SURVEY.md §8(c) "C2: a 16,384-row sample") or the cpu_baseline of BASELINE.md §3
finishes in reasonable time.  No blocking, fusion or reordering of the per-text arithmetic: each
row is exactly what Encoder.encode_text returns for that text.
"""
from __future__ import annotations

import multiprocessing as mp
import os
import time

import numpy as np

_W = {}


def _init(ecfg, weights, ids, starts, ends, pooling):
    from threadpoolctl import threadpool_limits
    from oracle.encoder import Encoder
    _W["lim"] = threadpool_limits(limits=1)
    _W["E"] = Encoder(ecfg, weights)
    _W["ids"], _W["starts"], _W["ends"], _W["pooling"] = ids, starts, ends, pooling


def _run(rows):
    E, ids, s, e = _W["E"], _W["ids"], _W["starts"], _W["ends"]
    return [E.encode_text(ids[s[i]:e[i]], pooling=_W["pooling"]) for i in rows]


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


class OraclePool:
    """A persistent pool of oracle workers over one token stream (text i = ids[starts[i]:ends[i]])."""

    def __init__(self, ecfg, weights, ids, starts, ends, procs: int | None = None, pooling: str = "mean"):
        self.procs = max(1, procs or host_cores())
        self.d = ecfg.hidden
        args = (ecfg, weights, ids, starts, ends, pooling)
        if self.procs == 1:
            _init(*args)
            self.pool = None
        else:
            self.pool = mp.get_context("fork").Pool(self.procs, initializer=_init, initargs=args)

    def encode(self, rows, chunk: int = 16) -> np.ndarray:
        """fp64 oracle embeddings of texts `rows`, in the order of `rows`."""
        rows = [int(r) for r in rows]
        if self.pool is None:
            out = _run(rows)
        else:
            parts = [rows[i:i + chunk] for i in range(0, len(rows), chunk)]
            out = [v for part in self.pool.map(_run, parts) for v in part]
        return np.stack(out) if out else np.zeros((0, self.d))

    def close(self):
        if self.pool is not None:
            self.pool.close()
            self.pool.join()
            self.pool = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def encode_rows(ecfg, weights, ids, starts, ends, rows, procs: int | None = None, pooling: str = "mean",
                chunk: int = 16):
    """fp64 oracle embeddings of texts `rows` (text i = ids[starts[i]:ends[i]]), in the order of
    `rows`.  Returns (float64 [len(rows) x d], seconds, processes used)."""
    rows = [int(r) for r in rows]
    procs = max(1, min(procs or host_cores(), max(1, len(rows) // chunk)))
    t0 = time.perf_counter()
    with OraclePool(ecfg, weights, ids, starts, ends, procs, pooling) as P:
        out = P.encode(rows, chunk)
    return out, time.perf_counter() - t0, procs
