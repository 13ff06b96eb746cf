"""Random-init BERT-class encoder weights, rounded to bf16 (inputs only).

Pretrained checkpoints are unavailable offline (BASELINE.json north_star), so
weights are seeded random draws rounded RNE to bf16; BOTH the oracle and libsurge
consume exactly these bf16-representable values, so weight quantisation never
enters parity.

Init scale (SURVEY.md §8(c) reading #13): linear matrices and word
embeddings ~N(0,0.02); position/type embeddings ~N(0,0.002); linear biases
~N(0,0.02); LayerNorm gamma ~1+N(0,0.1), beta = 0 ("surge" init, keeps distinct
texts' embeddings discriminable).  The "pin" init additionally draws beta ~N(0,0.1)
so that a dropped beta term cannot hide in a test.

Blob layout (the order `include/surge.h` documents): HF BERT tensor order, each
tensor row-major, bf16 bits as uint16, no padding.
"""
from __future__ import annotations

import numpy as np

from .configs import EncoderConfig


def blob_layout(cfg: EncoderConfig):
    """[(hf_name, shape)] in blob order -- mirrors the table in include/surge.h."""
    d, f = cfg.hidden, cfg.ffn
    out = [
        ("embeddings.word_embeddings.weight", (cfg.vocab_size, d)),
        ("embeddings.position_embeddings.weight", (cfg.max_position, d)),
        ("embeddings.token_type_embeddings.weight", (cfg.type_vocab_size, d)),
        ("embeddings.LayerNorm.weight", (d,)),
        ("embeddings.LayerNorm.bias", (d,)),
    ]
    for l in range(cfg.layers):
        p = f"encoder.layer.{l}."
        out += [
            (p + "attention.self.query.weight", (d, d)), (p + "attention.self.query.bias", (d,)),
            (p + "attention.self.key.weight", (d, d)), (p + "attention.self.key.bias", (d,)),
            (p + "attention.self.value.weight", (d, d)), (p + "attention.self.value.bias", (d,)),
            (p + "attention.output.dense.weight", (d, d)), (p + "attention.output.dense.bias", (d,)),
            (p + "attention.output.LayerNorm.weight", (d,)), (p + "attention.output.LayerNorm.bias", (d,)),
            (p + "intermediate.dense.weight", (f, d)), (p + "intermediate.dense.bias", (f,)),
            (p + "output.dense.weight", (d, f)), (p + "output.dense.bias", (d,)),
            (p + "output.LayerNorm.weight", (d,)), (p + "output.LayerNorm.bias", (d,)),
        ]
    return out


def n_blob_elems(cfg: EncoderConfig) -> int:
    return int(sum(int(np.prod(s)) for _, s in blob_layout(cfg)))


def bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round fp32 -> bf16 (round-to-nearest-even), returned as uint16 bit patterns."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return u.astype(np.uint16)


def bf16_to_f32(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << 16).view(np.float32)


def make_weights(cfg: EncoderConfig, seed: int = 1234, init: str = "surge") -> dict:
    """{hf_name: float32 array of bf16-representable values} in blob order."""
    rng = np.random.Generator(np.random.PCG64(seed))
    out = {}
    for name, shape in blob_layout(cfg):
        if name.endswith("LayerNorm.weight"):
            x = 1.0 + 0.1 * rng.standard_normal(shape)
        elif name.endswith("LayerNorm.bias"):
            x = (0.1 * rng.standard_normal(shape)) if init == "pin" else np.zeros(shape)
        elif "position_embeddings" in name or "token_type_embeddings" in name:
            x = 0.002 * rng.standard_normal(shape)
        else:  # word embeddings, linear weights and biases
            x = 0.02 * rng.standard_normal(shape)
        out[name] = bf16_to_f32(bf16_bits(x.astype(np.float32))).reshape(shape)
    return out


def pack_blob(cfg: EncoderConfig, weights: dict) -> np.ndarray:
    """Flat uint16 bf16 blob in blob_layout order (the libsurge weight input)."""
    parts = []
    for name, shape in blob_layout(cfg):
        w = weights[name]
        assert tuple(w.shape) == tuple(shape), (name, w.shape, shape)
        parts.append(bf16_bits(w).reshape(-1))
    return np.concatenate(parts)
