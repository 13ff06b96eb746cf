"""Encoder classes and workload recipes (inputs only).

Encoder shapes: the paper names the models only (all-MiniLM-L6-v2 22M d=384,
bge-base 109M d=768, E5-large 335M d=1024).  The
layer/head/FFN counts are the public BERT-class shapes (SURVEY.md §8(c) reading
#12); param counts reproduce 22.6M / 108.9M / 334.1M.

Workload recipes: PAPER.md §5.1 P:501 (10M texts, P=4,000, log-normal
mu=9.03 sigma=1.72, 47-byte texts), thresholds P:304 (B_min=100K, B_max=500K),
sweeps use B_max=5*B_min.  C1 toy from BASELINE.json configs[0].
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace


@dataclass(frozen=True)
class EncoderConfig:
    name: str
    vocab_size: int
    max_position: int
    type_vocab_size: int
    hidden: int
    layers: int
    heads: int
    ffn: int
    ln_eps: float = 1e-12

    @property
    def head_dim(self) -> int:
        return self.hidden // self.heads

    def n_params(self) -> int:
        d, f = self.hidden, self.ffn
        emb = (self.vocab_size + self.max_position + self.type_vocab_size) * d + 2 * d
        layer = 4 * (d * d + d) + 2 * d + (d * f + f) + (f * d + d) + 2 * d
        return emb + self.layers * layer


@dataclass(frozen=True)
class WorkloadConfig:
    name: str
    n_texts: int                 # N
    n_partitions: int            # P
    sigma: float                 # log-normal sigma of partition sizes
    mu: float = 9.03             # log-normal mu
    length_model: str = "bytes47"  # "bytes47" | "uniform" | "long"
    len_lo: int = 4              # for "uniform"
    len_hi: int = 32
    cls_id: int = 101
    sep_id: int = 102
    id_lo: int = 1000            # ids drawn uniform in [id_lo, vocab)
    b_min: int = 100_000
    b_max: int = 500_000
    order: str = "generated"     # "generated" | "ascending" (largest-last)


ENCODERS = {
    "toy": EncoderConfig("toy", vocab_size=1024, max_position=64, type_vocab_size=2,
                         hidden=64, layers=2, heads=4, ffn=256),
    "minilm": EncoderConfig("minilm", vocab_size=30522, max_position=512, type_vocab_size=2,
                            hidden=384, layers=6, heads=12, ffn=1536),
    "bgebase": EncoderConfig("bgebase", vocab_size=30522, max_position=512, type_vocab_size=2,
                             hidden=768, layers=12, heads=12, ffn=3072),
    "bgelarge": EncoderConfig("bgelarge", vocab_size=30522, max_position=512, type_vocab_size=2,
                              hidden=1024, layers=24, heads=16, ffn=4096),
}

WORKLOADS = {
    # C1 (BASELINE.json configs[0])
    "toy": WorkloadConfig("toy", n_texts=200, n_partitions=8, sigma=1.72,
                          length_model="uniform", len_lo=4, len_hi=32,
                          cls_id=1, sep_id=2, id_lo=4, b_min=64, b_max=320),
    # C1-safety variant: ascending sizes (largest last), B_max=96 (SURVEY §8(d) "Thresholds")
    "toy_safety": WorkloadConfig("toy_safety", n_texts=200, n_partitions=8, sigma=1.72,
                                 length_model="uniform", len_lo=4, len_hi=32,
                                 cls_id=1, sep_id=2, id_lo=4, b_min=64, b_max=96,
                                 order="ascending"),
    # C2 (BASELINE.json configs[1]) -- the bench workload
    "minilm": WorkloadConfig("minilm", n_texts=10_000_000, n_partitions=4000, sigma=1.72),
    "minilm_s1.0": WorkloadConfig("minilm_s1.0", n_texts=10_000_000, n_partitions=4000, sigma=1.0),
    "minilm_s2.5": WorkloadConfig("minilm_s2.5", n_texts=10_000_000, n_partitions=4000, sigma=2.5),
    # C5 skew/scale stress (BASELINE.json configs[4]; tab:sigma-sweep P:764-785, tab:scaling P:1195-1223)
    "c5_s1.0": WorkloadConfig("c5_s1.0", n_texts=100_000_000, n_partitions=40_000, sigma=1.0),
    "c5_s1.72": WorkloadConfig("c5_s1.72", n_texts=100_000_000, n_partitions=40_000, sigma=1.72),
    "c5_s2.5": WorkloadConfig("c5_s2.5", n_texts=100_000_000, n_partitions=40_000, sigma=2.5),
    # C4 long-length variant (seq <= 512)
    "long": WorkloadConfig("long", n_texts=10_000_000, n_partitions=4000, sigma=1.72,
                           length_model="long"),
}


def scaled(w: WorkloadConfig, n_texts: int, n_partitions: int | None = None, **kw) -> WorkloadConfig:
    """Same recipe at a smaller N (and P) -- used for parity-size cases."""
    return replace(w, n_texts=n_texts,
                   n_partitions=n_partitions if n_partitions is not None else w.n_partitions, **kw)
