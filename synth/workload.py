"""Seeded synthetic partitioned token streams (inputs only -- no method arithmetic).

Recipe:

* Partition sizes (§5.1, §2.1): z_k ~ N(0,1) (numpy PCG64, seed),
  r_k = exp(mu + sigma*z_k), n_k = max(1, round(r_k * N / sum r)), residual N - sum n_k
  added to the largest partition so that sum n_k = N exactly (SPEC.md S:87 rescaling).
  Arrival order = generation order (or ascending for the largest-last variant).
* Text lengths in tokens incl. [CLS]/[SEP]: "synthetic sentences averaging 47 bytes"
   -> bytes ~ U{24..70}, len = 2 + ceil(bytes/4) (mean 14.13).  C1: U{4..32}.
  Long variant (C4, seq <= 512): clip(round(LogNormal(ln 128, 0.6)), 8, 512).
* Token ids: [CLS], then uniform in [id_lo, vocab), then [SEP].
* Partition keys: distinct, non-dense 64-bit values (a bijection of the index).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .configs import WorkloadConfig

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)


@dataclass
class Workload:
    cfg: WorkloadConfig
    seed: int
    keys: np.ndarray        # uint64[P]   partition ids in arrival order
    sizes: np.ndarray       # int64[P]    n_k texts per partition
    lengths: np.ndarray     # int32[N]    tokens per text, partitions concatenated in arrival order
    ids: np.ndarray         # int32[T]    token ids, texts concatenated
    text_off: np.ndarray    # int64[P+1]  first text of partition k in `lengths`
    tok_off: np.ndarray     # int64[P+1]  first token of partition k in `ids`

    @property
    def n_texts(self) -> int:
        return int(self.lengths.shape[0])

    @property
    def n_tokens(self) -> int:
        return int(self.ids.shape[0])

    def partition(self, k: int):
        """(key, ids, lengths) of partition k -- views, not copies."""
        return (int(self.keys[k]),
                self.ids[self.tok_off[k]:self.tok_off[k + 1]],
                self.lengths[self.text_off[k]:self.text_off[k + 1]])

    def __iter__(self):
        for k in range(len(self.sizes)):
            yield self.partition(k)


def partition_sizes(cfg: WorkloadConfig, rng: np.random.Generator) -> np.ndarray:
    P, N = cfg.n_partitions, cfg.n_texts
    z = rng.standard_normal(P)
    r = np.exp(cfg.mu + cfg.sigma * z)
    n = np.maximum(1, np.rint(r * (N / r.sum()))).astype(np.int64)
    res = N - int(n.sum())
    if res >= 0 or n[int(np.argmax(n))] + res >= 1:
        n[int(np.argmax(n))] += res
    else:   # degenerate N ~ P: take the excess from the largest partitions, keeping every n_k >= 1
        if N < len(n):
            raise ValueError("need n_texts >= n_partitions")
        for k in np.argsort(-n, kind="stable"):
            take = min(int(n[k]) - 1, -res)
            n[k] -= take
            res += take
            if res == 0:
                break
    if cfg.order == "ascending":
        n = np.sort(n, kind="stable")
    return n


def text_lengths(cfg: WorkloadConfig, n: int, rng: np.random.Generator, max_position: int) -> np.ndarray:
    if cfg.length_model == "bytes47":
        nbytes = rng.integers(24, 71, size=n)
        lens = 2 + (nbytes + 3) // 4
    elif cfg.length_model == "uniform":
        lens = rng.integers(cfg.len_lo, cfg.len_hi + 1, size=n)
    elif cfg.length_model == "long":
        lens = np.clip(np.rint(rng.lognormal(np.log(128.0), 0.6, size=n)), 8, 512)
    else:
        raise ValueError(cfg.length_model)
    return np.minimum(lens, max_position).astype(np.int32)


def make_workload(cfg: WorkloadConfig, vocab_size: int, max_position: int, seed: int = 0) -> Workload:
    rng = np.random.Generator(np.random.PCG64(seed))
    sizes = partition_sizes(cfg, rng)
    lengths = text_lengths(cfg, int(sizes.sum()), rng, max_position)
    T = int(lengths.sum(dtype=np.int64))
    ids = rng.integers(cfg.id_lo, vocab_size, size=T, dtype=np.int32)
    ends = np.cumsum(lengths, dtype=np.int64)
    ids[ends - lengths] = cfg.cls_id
    ids[ends - 1] = cfg.sep_id
    text_off = np.zeros(len(sizes) + 1, dtype=np.int64)
    text_off[1:] = np.cumsum(sizes)
    tok_off = np.zeros(len(sizes) + 1, dtype=np.int64)
    tok_off[1:] = np.concatenate([[0], ends])[text_off[1:]]
    keys = (np.arange(1, len(sizes) + 1, dtype=np.uint64) * _GOLDEN)
    return Workload(cfg, seed, keys, sizes, lengths, ids, text_off, tok_off)


def random_texts(n: int, vocab_size: int, max_position: int, seed: int,
                 lo: int = 1, hi: int | None = None, cls_id: int = 101, sep_id: int = 102,
                 id_lo: int = 1000):
    """A flat list of n texts (list of int32 arrays) with lengths U{lo..hi} -- for unit tests."""
    rng = np.random.Generator(np.random.PCG64(seed))
    hi = max_position if hi is None else hi
    out = []
    for _ in range(n):
        l = int(rng.integers(lo, hi + 1))
        t = rng.integers(min(id_lo, vocab_size - 1), vocab_size, size=l, dtype=np.int32)
        if l >= 2:
            t[0], t[-1] = cls_id, sep_id
        out.append(t)
    return out


def parity_sample(wl: "Workload", n_rows: int = 16_384, head: int = 4096, seed: int = 0) -> list:
    """Rows of the SURVEY.md §8(c) C2 parity sample: the first `head` rows in stream order, the first
    and last row of every partition, then seeded uniform rows up to `n_rows` distinct rows (sorted)."""
    rows = set(range(min(head, wl.n_texts)))
    for k in range(len(wl.sizes)):
        if wl.sizes[k] > 0:
            rows |= {int(wl.text_off[k]), int(wl.text_off[k + 1]) - 1}
    rng = np.random.default_rng(seed)
    n_rows = min(n_rows, wl.n_texts)
    while len(rows) < n_rows:
        rows |= set(rng.integers(0, wl.n_texts, size=n_rows - len(rows)).tolist())
    return sorted(rows)
