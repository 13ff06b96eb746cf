"""Theorem 1 cost model (§Theorem, `eq:partition-time` P:183, `eq:speedup` P:431-446) and
its fit to measured wall times -- SURVEY.md §8(f) NEXT N3 ("Theorem 1 on B200").

    T_k = c_call + n_k c_enc / G                     (per invocation)
    T(F) = F c_call + N c_enc / G                    (F invocations over N texts)
    alpha = P c_call / (N c_enc / G)                 (IPC-to-compute ratio of PBP)
    speedup(F) = T_PBP / T_SURGE = (1 + alpha) / (1 + alpha F / P)     (eq:speedup)

On B200 the paper's c_ipc (Python process-pool dispatch) becomes c_call: the fixed cost of one
SuperBatch invocation in libsurge (host aggregation + H2D + the chunk's kernel launches + D2H
bookkeeping).  Pure Python, no GPU.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def partition_time(n_k: float, c_call: float, c_enc: float, g: int = 1) -> float:
    """eq:partition-time: wall time of one invocation on n_k texts."""
    return c_call + n_k * c_enc / g


def alpha(p: int, n: int, c_call: float, c_enc: float, g: int = 1) -> float:
    """IPC-to-compute ratio of partition-by-partition processing."""
    return p * c_call / (n * c_enc / g)


def speedup(alpha_: float, f: int, p: int) -> float:
    """eq:speedup: T_PBP / T_SURGE for F invocations vs P."""
    return (1.0 + alpha_) / (1.0 + alpha_ * f / p)


@dataclass
class Fit:
    c_call: float      # s per invocation
    c_enc: float       # s per text (x G)
    residual_rms: float


def fit(invocations, wall_s, n_texts: int, g: int = 1) -> Fit:
    """Least-squares fit of T_i = F_i c_call + N c_enc / G over runs i (same N, varying F)."""
    f = np.asarray(invocations, dtype=np.float64)
    t = np.asarray(wall_s, dtype=np.float64)
    a = np.stack([f, np.full_like(f, n_texts / g)], axis=1)
    (c_call, c_enc), *_ = np.linalg.lstsq(a, t, rcond=None)
    res = t - a @ np.array([c_call, c_enc])
    return Fit(float(c_call), float(c_enc), float(np.sqrt(np.mean(res ** 2))))
