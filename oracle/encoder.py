"""Oracle: fp64 BERT-class encoder + masked mean-pool + L2 norm.  TEST INFRASTRUCTURE ONLY.

What the method computes for every text, independently of the SuperBatch it lands in
(SURVEY.md §8(c) "plain definition"):  E_k[j] = normalize(meanpool(BERT_theta(text_kj))).

The paper fixes only the model family and output ("all-MiniLM-L6-v2 ... 384-dimensional
L2-normalized embeddings"; bge-base / E5-large P:723-760).  The BERT layer itself
is the public BERT definition the north star names (post-LN, erf-GELU, biased-variance
LayerNorm with eps=1e-12, softmax scale 1/sqrt(d_h), positions restarting at 0 per text,
token type 0); the readings are listed in DESIGN.md ("Readings" #6-#11).

Weights: dict of HF tensor names -> arrays (synth.weights), upcast to fp64 here.
Pinned against transformers BertModel in fp64 (tests/test_oracle_encoder.py).
"""
from __future__ import annotations

import math

import numpy as np
from scipy.special import erf as _erf   # library erf (fp64), pinned against math.erf in tests


def layer_norm(z: np.ndarray, gamma: np.ndarray, beta: np.ndarray, eps: float) -> np.ndarray:
    """LN(z) = gamma * (z - mu) / sqrt(var + eps) + beta, biased variance over the last axis."""
    mu = z.mean(axis=-1, keepdims=True)
    var = ((z - mu) ** 2).mean(axis=-1, keepdims=True)
    return gamma * (z - mu) / np.sqrt(var + eps) + beta


def gelu(x: np.ndarray) -> np.ndarray:
    """Exact GELU: x * 1/2 * (1 + erf(x / sqrt 2))  (BERT hidden_act="gelu"; reading #8)."""
    return x * 0.5 * (1.0 + _erf(x / math.sqrt(2.0)))


def softmax(s: np.ndarray) -> np.ndarray:
    """Explicit softmax along the last axis: subtract row max, exp, divide by the row sum."""
    e = np.exp(s - s.max(axis=-1, keepdims=True))
    return e / e.sum(axis=-1, keepdims=True)


def attention(q: np.ndarray, k: np.ndarray, v: np.ndarray, heads: int) -> np.ndarray:
    """Bidirectional multi-head attention over ONE text's own tokens (block-diagonal; reading #10).

    q,k,v: [l, d].  Per head h: O_h = softmax(Q_h K_h^T / sqrt(d_h)) V_h; output concat_h O_h.
    """
    l, d = q.shape
    dh = d // heads
    out = np.empty((l, d), dtype=np.float64)
    for h in range(heads):
        sl = slice(h * dh, (h + 1) * dh)
        p = softmax(q[:, sl] @ k[:, sl].T / math.sqrt(dh))
        out[:, sl] = p @ v[:, sl]
    return out


def linear(x: np.ndarray, w: np.ndarray, b: np.ndarray) -> np.ndarray:
    """y = x W^T + b  (HF nn.Linear convention, W is [out, in])."""
    return x @ w.T + b


class Encoder:
    """fp64 BERT-class encoder over one text at a time."""

    def __init__(self, cfg, weights: dict):
        self.cfg = cfg
        self.w = {k: np.asarray(v, dtype=np.float64) for k, v in weights.items()}

    def embed(self, ids: np.ndarray) -> np.ndarray:
        """h_t = LN_e(word[id_t] + pos[t] + type[0]), t = 0..l-1 (positions restart per text)."""
        w, l = self.w, len(ids)
        z = (w["embeddings.word_embeddings.weight"][np.asarray(ids, dtype=np.int64)]
             + w["embeddings.position_embeddings.weight"][:l]
             + w["embeddings.token_type_embeddings.weight"][0])
        return layer_norm(z, w["embeddings.LayerNorm.weight"], w["embeddings.LayerNorm.bias"],
                          self.cfg.ln_eps)

    def layer(self, h: np.ndarray, i: int) -> np.ndarray:
        """One post-LN BERT layer (in its order)."""
        w, p, eps = self.w, f"encoder.layer.{i}.", self.cfg.ln_eps
        q = linear(h, w[p + "attention.self.query.weight"], w[p + "attention.self.query.bias"])
        k = linear(h, w[p + "attention.self.key.weight"], w[p + "attention.self.key.bias"])
        v = linear(h, w[p + "attention.self.value.weight"], w[p + "attention.self.value.bias"])
        o = attention(q, k, v, self.cfg.heads)
        h = layer_norm(linear(o, w[p + "attention.output.dense.weight"], w[p + "attention.output.dense.bias"]) + h,
                       w[p + "attention.output.LayerNorm.weight"], w[p + "attention.output.LayerNorm.bias"], eps)
        f = gelu(linear(h, w[p + "intermediate.dense.weight"], w[p + "intermediate.dense.bias"]))
        h = layer_norm(linear(f, w[p + "output.dense.weight"], w[p + "output.dense.bias"]) + h,
                       w[p + "output.LayerNorm.weight"], w[p + "output.LayerNorm.bias"], eps)
        return h

    def hidden_states(self, ids: np.ndarray) -> np.ndarray:
        h = self.embed(ids)
        for i in range(self.cfg.layers):
            h = self.layer(h, i)
        return h

    def encode_text(self, ids: np.ndarray, pooling: str = "mean") -> np.ndarray:
        """One text -> its d-dim unit embedding (pooling "mean": reading #6; "cls": bge's native
        [CLS] pooling)."""
        h = self.hidden_states(ids)
        return cls_pool_l2(h) if pooling == "cls" else mean_pool_l2(h)

    def encode_texts(self, texts) -> np.ndarray:
        """Each text independently (PBP order, P:167 -- no batching, no padding)."""
        if len(texts) == 0:
            return np.zeros((0, self.cfg.hidden))
        return np.stack([self.encode_text(t) for t in texts])


def mean_pool_l2(h: np.ndarray) -> np.ndarray:
    """v = (1/l) sum_t h_t over ALL l tokens incl. [CLS]/[SEP] (reading #6);
    e = v / max(||v||_2, 1e-12) (reading #7, torch F.normalize)."""
    v = h.sum(axis=0) / h.shape[0]
    return v / max(float(np.sqrt((v * v).sum())), 1e-12)


def cls_pool_l2(h: np.ndarray) -> np.ndarray:
    """[CLS] pooling (bge): e = h_0 / max(||h_0||_2, 1e-12)."""
    v = h[0]
    return v / max(float(np.sqrt((v * v).sum())), 1e-12)
