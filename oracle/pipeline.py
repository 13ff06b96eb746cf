"""Oracle: the whole path as a plain definition.  TEST INFRASTRUCTURE ONLY.

Input: partitions {(k_i, T_i)} in arrival order.  Output: k_i -> E_i in R^{n_i x d}
(P:165), produced SuperBatch by SuperBatch as Alg.1 does:

    for each partition: AddPartition  ->  on a flush: concatenate (allTexts), bounds,
    ONE encode of allTexts, slice E[start:end] per member.

The encode of allTexts is, by definition, each text encoded independently
(oracle.encoder); the packed token stream (cu_seqlens) is used only to locate each
text, so any difference against `encode_pbp` is a bookkeeping bug (O4).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import aggregator as agg
from .encoder import Encoder


@dataclass
class SuperBatchResult:
    sb: agg.SuperBatch
    packed: agg.Packed
    lengths: np.ndarray          # int64[S] text lengths in SuperBatch order
    plan: list = field(default_factory=list)   # LPT pieces (world > 1)


@dataclass
class PipelineResult:
    superbatches: list
    empty_keys: list
    peak_buffered: int
    nmax_seen: int
    embeddings: dict             # key -> float64[n_k, d] (only when encode=True)


def run(workload, b_min: int, b_max: int, encoder: Encoder | None = None, world: int = 1,
        rows: dict | None = None, policy: str = agg.LABEL) -> PipelineResult:
    """Drive Alg.1 over `workload` (an iterable of (key, ids, lengths)).

    encoder=None runs the integer path only.  `rows` optionally restricts encoding to
    {key: [row indices within the partition]} (sampled parity at full size).  Under the SPLIT
    policy a member is a piece (rows [row0, row0 + n)) of its partition; E_k is reassembled from
    the pieces by their row offsets ("boundary tracking ensures correct reassembly").
    """
    A = agg.Aggregator(b_min, b_max, policy)
    parts = {}
    results, emb = [], {}

    def on_flush(sb):
        if sb is None:
            return
        ids_list, lens_list = [], []
        for key, n, r0 in zip(sb.keys, sb.sizes, sb.row0):
            ids_k, lens_k = parts[key]
            tok = np.concatenate([[0], np.cumsum(lens_k)])
            ids_list.append(ids_k[tok[r0]:tok[r0 + n]])
            lens_list.append(lens_k[r0:r0 + n])
            if r0 + n == len(lens_k):
                parts.pop(key)
        all_ids = np.concatenate(ids_list)                  # allTexts.extend(texts)
        lengths = np.concatenate(lens_list).astype(np.int64)
        packed = agg.pack(lengths, sb.sizes)               # bounds
        r = SuperBatchResult(sb, packed, lengths)
        if world > 1:
            r.plan, _ = agg.lpt_plan(lengths, sb.sizes, world)
        results.append(r)
        if encoder is not None:                             # E = f(allTexts)
            cu = packed.cu_seqlens
            for j, (start, end, key) in enumerate(sb.bounds()):   # E_k = E[start:end] P:290-291
                r0 = sb.row0[j]
                want = range(r0, r0 + end - start) if rows is None else \
                    [i for i in rows.get(key, []) if r0 <= i < r0 + end - start]
                E = emb.setdefault(key, {})
                for i in want:
                    g = start + i - r0
                    E[i] = encoder.encode_text(all_ids[cu[g]:cu[g + 1]])

    for key, ids, lengths in workload:
        parts[key] = (np.asarray(ids), np.asarray(lengths))
        before = len(A.flushes)
        A.add_partition(key, len(lengths))
        for sb in A.flushes[before:]:          # PREFLUSH / SPLIT may flush more than once per add
            on_flush(sb)
    on_flush(A.finish())
    for k in A.empty_keys:
        parts.pop(k, None)
        emb[k] = {}
    if encoder is not None and rows is None:
        d = encoder.cfg.hidden
        emb = {k: (np.stack([E[i] for i in range(len(E))]) if len(E) else np.zeros((0, d)))
               for k, E in emb.items()}
    return PipelineResult(results, A.empty_keys, A.peak_buffered, A.nmax_seen, emb)


def encode_pbp(workload, encoder: Encoder) -> dict:
    """Partition-by-partition (PBP): one encode per partition, no aggregation."""
    out = {}
    for key, ids, lengths in workload:
        texts, off = [], 0
        for l in np.asarray(lengths):
            texts.append(np.asarray(ids)[off:off + int(l)])
            off += int(l)
        out[key] = encoder.encode_texts(texts)
    return out
