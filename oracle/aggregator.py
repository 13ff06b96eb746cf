"""Oracle: SuperBatch aggregation (Alg.1), packing, LPT shard plan.  TEST INFRASTRUCTURE ONLY.

Citations are PAPER.md line numbers ("P:n") and SPEC.md ("S:n").
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

EFFICIENCY, SAFETY, END_OF_STREAM = "efficiency", "safety", "end_of_stream"

# What B_max does (readings R2/R3 and R23):
LABEL = "label"          # literal Alg.1: B_max only labels the flush; never split (default)
SPLIT = "split"          # §6: "splitting the oversized partition across consecutive SuperBatches"
PREFLUSH = "preflush"    # §3.2: flush the buffer before a partition that would push it past
                         # B_max; an oversized partition is "emitted ... as its own SuperBatch"


class DuplicateKey(ValueError):
    pass


@dataclass
class SuperBatch:
    """One Flush() of Alg.1: buffered partitions in arrival order."""
    idx: int
    reason: str
    keys: list            # partition keys, arrival order
    sizes: list           # texts per member (n_k, or a piece of it under SPLIT)
    refs: list            # caller payload per member (e.g. partition index)
    row0: list = field(default_factory=list)   # first row of the member within its partition (SPLIT)

    @property
    def total(self) -> int:
        return int(sum(self.sizes))

    def bounds(self):
        """`bounds.append((idx, idx+|texts|, key))` -- P:284-288."""
        out, idx = [], 0
        for key, n in zip(self.keys, self.sizes):
            out.append((idx, idx + n, key))
            idx += n
        return out


class Aggregator:
    """Alg.1 AddPartition / Flush, literal (two-threshold scheme P:304).

    Readings: comparisons are ``>=`` on integer text counts, Safety is
    checked first; B_max only labels the flush (literal Alg.1);
    a partition is never split, an oversized one flushes together with the buffer
    (P:308); zero-text partitions complete immediately and never enter
    the buffer; an empty residual does not flush.
    """

    def __init__(self, b_min: int, b_max: int, policy: str = LABEL):
        if not (0 < b_min < b_max):
            raise ValueError("need 0 < b_min < b_max")
        if policy not in (LABEL, SPLIT, PREFLUSH):
            raise ValueError(policy)
        self.b_min, self.b_max, self.policy = int(b_min), int(b_max), policy
        self.partitions: list = []           # P:262 `partitions <- []`
        self.total = 0                       # P:262 `total <- 0`
        self.flushes: list[SuperBatch] = []
        self.empty_keys: list = []
        self.seen: set = set()
        self.peak_buffered = 0
        self.nmax_seen = 0
        self.finished = False

    def add_partition(self, key, n_texts: int, ref=None):
        """AddPartition(key, texts) -- P:274-280.  Returns the SuperBatch it flushed, or None."""
        if self.finished:
            raise RuntimeError("add after finish")
        if key in self.seen:                 # keys unique and grouped
            raise DuplicateKey(key)
        self.seen.add(key)
        n = int(n_texts)
        if n < 0:
            raise ValueError("n_texts < 0")
        if n == 0:
            self.empty_keys.append(key)
            return None
        if self.policy == SPLIT:
            return self._add_split(key, n, ref)
        if self.policy == PREFLUSH and self.partitions and self.total + n > self.b_max:
            # P:304 "fires only when a single arriving partition would push the running total past
            # B_max": the buffer flushes first, so no SuperBatch but a lone oversized partition
            # ("emitting the partition as its own SuperBatch") exceeds B_max
            self._flush(SAFETY)
        self.partitions.append((key, n, ref, 0))  # P:275 partitions.append((key, copy(texts)))
        self.total += n                           # P:276 total <- total + |texts|
        self.nmax_seen = max(self.nmax_seen, n)
        self.peak_buffered = max(self.peak_buffered, self.total)
        # Lemma, exact integer prefix form: buffer < B_min before the add, plus n_k.
        assert self.total <= self.b_min - 1 + self.nmax_seen, "Lemma bound violated"
        if self.policy == PREFLUSH:              # S <= B_max unless the partition is alone
            assert self.total <= self.b_max or len(self.partitions) == 1
        if self.total >= self.b_max:              # P:277 memory-safety trigger
            return self._flush(SAFETY)
        elif self.total >= self.b_min:            # P:278 efficiency trigger
            return self._flush(EFFICIENCY)
        return None

    def _add_split(self, key, n: int, ref):
        """SPLIT: texts of the arriving partition fill the buffer up to exactly B_max, which
        flushes (the Safety trigger), and the rest continues into the next SuperBatches; the boundary
        records (row0) let the pieces be reassembled ("boundary tracking").  Every SuperBatch
        then holds at most B_max texts (the Lemma's S <= B_max)."""
        self.nmax_seen = max(self.nmax_seen, n)
        row0, last = 0, None
        while self.total + (n - row0) >= self.b_max:
            take = self.b_max - self.total
            self.partitions.append((key, take, ref, row0))
            self.total += take
            self.peak_buffered = max(self.peak_buffered, self.total)
            row0 += take
            last = self._flush(SAFETY)
        if row0 < n:
            self.partitions.append((key, n - row0, ref, row0))
            self.total += n - row0
            self.peak_buffered = max(self.peak_buffered, self.total)
            if self.total >= self.b_min:          # P:278 (total < B_max here)
                last = self._flush(EFFICIENCY)
        return last

    def finish(self):
        """End of stream: Alg.1 line 9 `AddPartition(curKey,curTexts); Flush()`."""
        self.finished = True
        if self.partitions:
            return self._flush(END_OF_STREAM)
        return None

    def _flush(self, reason: str) -> SuperBatch:
        """Flush() -- P:282-296 (the encode/slice/upload part lives in oracle.pipeline)."""
        sb = SuperBatch(len(self.flushes), reason,
                        [p[0] for p in self.partitions], [p[1] for p in self.partitions],
                        [p[2] for p in self.partitions], [p[3] for p in self.partitions])
        self.flushes.append(sb)
        self.partitions, self.total = [], 0      # P:295 partitions <- []; total <- 0
        return sb


def run_aggregator(keys, sizes, b_min: int, b_max: int, policy: str = LABEL) -> Aggregator:
    """Feed a whole arrival sequence through the aggregator and finish."""
    agg = Aggregator(b_min, b_max, policy)
    for i, (k, n) in enumerate(zip(keys, sizes)):
        agg.add_partition(k, int(n), ref=i)
    agg.finish()
    return agg


def theorem_flush_bound(n_texts: int, n_partitions: int, b_min: int) -> int:
    """Theorem: F = ceil(N / B_min) flushes *at most* (P:441); and F <= P trivially."""
    return min(n_partitions, math.ceil(n_texts / b_min))


def memory_bound_bytes(S: int, L: float, d: int) -> float:
    """Lemma M(S) = S*L + S*d*4 bytes (eq:memory P:305)."""
    return S * L + S * d * 4


def fill_ratio_prediction(mu: float, sigma: float, b_min: float) -> float:
    """eq:fill-ratio: E[S/B_min] ~= 1 + sigma^2 / (2 mu B_min)."""
    return 1.0 + sigma * sigma / (2.0 * mu * b_min)


# --------------------------------------------------------------------------- packing

@dataclass
class Packed:
    cu_seqlens: np.ndarray     # int64[S+1]  cu[0]=0, cu[i+1]=cu[i]+len_i
    part_row_off: np.ndarray   # int64[m+1]  first row of member j (Alg.1 `bounds` start)
    part_tok_off: np.ndarray   # int64[m+1]  first token of member j


def pack(lengths: np.ndarray, sizes) -> Packed:
    """Flush's concatenation + `bounds` loop, carried to tokens.

    `lengths` are the SuperBatch's text lengths in member order; `sizes` the member n_k.
    """
    lengths = np.asarray(lengths, dtype=np.int64)
    cu = np.zeros(len(lengths) + 1, dtype=np.int64)
    cu[1:] = np.cumsum(lengths)
    row = np.zeros(len(sizes) + 1, dtype=np.int64)
    row[1:] = np.cumsum(np.asarray(sizes, dtype=np.int64))
    return Packed(cu, row, cu[row])


# --------------------------------------------------------------------------- LPT plan

@dataclass
class Piece:
    member: int        # index of the partition within the SuperBatch
    first_row: int     # global row (SuperBatch order) of its first text
    n_rows: int
    tokens: int
    rank: int = -1


def lpt_plan(lengths: np.ndarray, sizes, world: int):
    """Token-balanced LPT split of one SuperBatch across `world` ranks (north star).

    1. Cut each partition into pieces of <= U = ceil(T/(8G)) tokens at text boundaries
       (greedy: close the piece when the next text would overflow; a text longer than U is
       its own piece).  With G == 1 there is a single piece per partition (reading #19).
    2. Sort pieces by (tokens desc, first_row asc).
    3. Assign each to the rank with minimum (load, rank).
    4. Rank-local order = first_row asc.
    Returns (pieces in global-row order with .rank set, per-rank lists of pieces).
    Pinned (tests/test_oracle_aggregator.py) independently of this code: Graham's LPT bound
    makespan <= (4/3 - 1/(3G)) * OPT against a brute-forced OPT on <= 10-piece instances (an
    ascending or arrival-order schedule breaks it), and Graham's tight instance family reaches
    the ratio exactly.  The tie-breaks (equal tokens -> lower first_row; equal load -> lower
    rank) are this design's reading R16: any tie-break is a valid LPT schedule.
    """
    lengths = np.asarray(lengths, dtype=np.int64)
    T = int(lengths.sum())
    pieces: list[Piece] = []
    row = 0
    if world == 1:
        for j, n in enumerate(sizes):
            pieces.append(Piece(j, row, int(n), int(lengths[row:row + n].sum()), 0))
            row += int(n)
        return pieces, [list(pieces)]
    U = -(-T // (8 * world))
    for j, n in enumerate(sizes):
        first, tok = row, 0
        for i in range(row, row + int(n)):
            l = int(lengths[i])
            if tok > 0 and tok + l > U:
                pieces.append(Piece(j, first, i - first, tok))
                first, tok = i, 0
            tok += l
        row += int(n)
        if row > first:
            pieces.append(Piece(j, first, row - first, tok))
    load = [0] * world
    for p in sorted(pieces, key=lambda p: (-p.tokens, p.first_row)):
        r = min(range(world), key=lambda q: (load[q], q))
        p.rank = r
        load[r] += p.tokens
    per_rank = [[p for p in pieces if p.rank == r] for r in range(world)]  # pieces already row-ordered
    return pieces, per_rank
