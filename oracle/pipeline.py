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
        rows: dict | None = None) -> PipelineResult:
    """Drive Alg.1 over `workload` (an iterable of (key, ids, lengths)).

    encoder=None runs the integer path only.  `rows` optionally restricts encoding to
    {key: [row indices within the partition]} (sampled parity at full size).
    """
    A = agg.Aggregator(b_min, b_max)
    parts = {}
    results, emb = [], {}

    def on_flush(sb):
        if sb is None:
            return
        ids_list, lens_list = [], []
        for key in sb.keys:
            ids_k, lens_k = parts.pop(key)
            ids_list.append(ids_k)
            lens_list.append(lens_k)
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
                want = range(end - start) if rows is None else rows.get(key, [])
                E = {}
                for i in want:
                    g = start + i
                    E[i] = encoder.encode_text(all_ids[cu[g]:cu[g + 1]])
                emb[key] = E

    for key, ids, lengths in workload:
        parts[key] = (np.asarray(ids), np.asarray(lengths))
        on_flush(A.add_partition(key, len(lengths)))
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
