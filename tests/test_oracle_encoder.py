"""Pins for oracle/encoder.py and oracle/pipeline.py (all CPU).

O1 attention (library SDPA + special cases), O2 pool closed forms, O3 unit norm,
O4 SuperBatch invariance, O5 transformers BertModel fp64 (independent library),
O6 LN/GELU values, O13 discriminating power.
"""
import json
import math
import os

import numpy as np
import pytest
import torch

from oracle import encoder as enc
from oracle import pipeline
from synth.configs import ENCODERS, WORKLOADS
from synth.weights import make_weights
from synth.workload import make_workload, random_texts

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def hf_reference(cfg, weights, texts, pooling="mean"):
    """transformers BertModel in fp64 (eager attention, erf GELU, eps 1e-12), then mean (or [CLS])
    pooling + normalize."""
    from transformers import BertConfig, BertModel
    hc = BertConfig(vocab_size=cfg.vocab_size, hidden_size=cfg.hidden, num_hidden_layers=cfg.layers,
                    num_attention_heads=cfg.heads, intermediate_size=cfg.ffn, hidden_act="gelu",
                    max_position_embeddings=cfg.max_position, type_vocab_size=cfg.type_vocab_size,
                    layer_norm_eps=cfg.ln_eps, hidden_dropout_prob=0.0, attention_probs_dropout_prob=0.0)
    hc._attn_implementation = "eager"
    m = BertModel(hc, add_pooling_layer=False).double().eval()
    sd = {k: torch.from_numpy(np.asarray(v, dtype=np.float64)) for k, v in weights.items()}
    missing, unexpected = m.load_state_dict(sd, strict=False)
    assert not unexpected and all("position_ids" in k or "token_type_ids" in k for k in missing), missing
    out = []
    with torch.no_grad():
        for t in texts:
            h = m(input_ids=torch.from_numpy(np.asarray(t, dtype=np.int64))[None]).last_hidden_state[0]
            v = h[0] if pooling == "cls" else h.mean(0)
            out.append(torch.nn.functional.normalize(v, dim=0, eps=1e-12).numpy())
    return np.stack(out)


@pytest.mark.parametrize("init", ["pin", "surge"])
def test_hf_pin_toy(init):
    cfg = ENCODERS["toy"]
    w = make_weights(cfg, seed=99, init=init)
    texts = random_texts(24, cfg.vocab_size, cfg.max_position, seed=1, lo=1, cls_id=1, sep_id=2, id_lo=4)
    texts += [np.array([5], np.int32), np.arange(4, 4 + cfg.max_position, dtype=np.int32)]  # l=1, l=max_pos
    ours = enc.Encoder(cfg, w).encode_texts(texts)
    ref = hf_reference(cfg, w, texts)
    assert np.max(np.abs(ours - ref)) <= 1e-10


def test_hf_pin_minilm_shape():
    cfg = ENCODERS["minilm"]
    w = make_weights(cfg, seed=5, init="pin")
    texts = random_texts(6, cfg.vocab_size, 128, seed=2, lo=1, hi=40)
    ours = enc.Encoder(cfg, w).encode_texts(texts)
    ref = hf_reference(cfg, w, texts)
    assert np.max(np.abs(ours - ref)) <= 1e-10


def test_layer_norm_closed_form():
    g = GOLD["layer_norm"]
    y = enc.layer_norm(np.array(g["x"], float), np.ones(4), np.zeros(4), 0.0)
    assert np.allclose(y, g["y"], atol=1e-12)
    # affine part: gamma scales, beta shifts
    y2 = enc.layer_norm(np.array(g["x"], float), np.full(4, 2.0), np.full(4, 0.5), 0.0)
    assert np.allclose(y2, 2.0 * np.array(g["y"]) + 0.5, atol=1e-12)
    # eps enters under the root
    y3 = enc.layer_norm(np.array([0.0, 2.0]), np.ones(2), np.zeros(2), 3.0)
    assert np.allclose(y3, [-1 / 2, 1 / 2])


def test_gelu_values():
    g = GOLD["gelu"]
    assert np.allclose(enc.gelu(np.array(g["x"])), g["y"], atol=1e-15)
    x = np.linspace(-6, 6, 97)
    assert np.allclose(enc.gelu(x) - enc.gelu(-x), x, atol=1e-14)   # GELU(x) - GELU(-x) = x
    assert np.allclose(enc.gelu(x), [v * 0.5 * (1 + math.erf(v / math.sqrt(2))) for v in x], atol=1e-15)
    assert abs(enc.gelu(np.array([20.0]))[0] - 20.0) < 1e-12


def test_attention_vs_library_and_special_cases():
    rng = np.random.default_rng(0)
    for l in (1, 2, 3, 7, 16, 33):
        for heads, dh in ((4, 16), (2, 32)):
            d = heads * dh
            q, k, v = (rng.standard_normal((l, d)) for _ in range(3))
            ours = enc.attention(q, k, v, heads)
            t = lambda a: torch.from_numpy(a).reshape(l, heads, dh).transpose(0, 1)[None]
            ref = torch.nn.functional.scaled_dot_product_attention(t(q), t(k), t(v))[0].transpose(0, 1).reshape(l, d)
            assert np.max(np.abs(ours - ref.numpy())) <= 1e-12
            if l == 1:
                assert np.array_equal(ours, v)          # softmax of one score is exactly 1
            # permutation equivariance (no positional term inside attention)
            perm = rng.permutation(l)
            assert np.allclose(enc.attention(q[perm], k[perm], v[perm], heads), ours[perm], atol=1e-12)
            # identical keys -> uniform weights -> every output row is the mean of v
            kc = np.repeat(k[:1], l, axis=0)
            assert np.allclose(enc.attention(q, kc, v, heads), np.repeat(v.mean(0, keepdims=True), l, 0), atol=1e-12)


def test_pool_closed_forms():
    rng = np.random.default_rng(1)
    for l in (1, 2, 5, 64):
        a, b = rng.standard_normal(8), rng.standard_normal(8)
        x = a[None] + np.arange(l)[:, None] * b[None]
        m = a + (l - 1) / 2 * b
        assert np.allclose(enc.mean_pool_l2(x), m / np.linalg.norm(m), atol=1e-12)
        c = rng.standard_normal(8)
        assert np.allclose(enc.mean_pool_l2(np.repeat(c[None], l, 0)), c / np.linalg.norm(c), atol=1e-12)
    assert np.array_equal(enc.mean_pool_l2(np.zeros((3, 4))), np.zeros(4))   # max(||v||, 1e-12) guard


@pytest.mark.parametrize("policy,b_max", [("label", None), ("split", 70), ("preflush", 70)])
def test_unit_norm_and_invariance_toy(policy, b_max):
    """O3 unit norm on every row; O4 packed-SuperBatch path == PBP path bit-exactly (also when SPLIT
    cuts partitions across SuperBatches and reassembles them by row offset)."""
    ecfg, wcfg = ENCODERS["toy"], WORKLOADS["toy"]
    w = make_weights(ecfg, seed=1234)
    E = enc.Encoder(ecfg, w)
    wl = make_workload(wcfg, ecfg.vocab_size, ecfg.max_position, seed=0)
    res = pipeline.run(wl, wcfg.b_min, b_max or wcfg.b_max, encoder=E, policy=policy)
    if policy == "split":
        assert any(len(set(sb.sb.keys)) < len(sb.sb.keys) or any(r > 0 for r in sb.sb.row0) for sb in res.superbatches)
    pbp = pipeline.encode_pbp(wl, E)
    assert len(res.superbatches) >= 2
    for key, M in res.embeddings.items():
        assert np.array_equal(M, pbp[key])
        assert np.all(np.abs(np.linalg.norm(M, axis=1) - 1) <= 1e-12)
    assert sum(m.shape[0] for m in res.embeddings.values()) == wcfg.n_texts


def test_discriminating_power_minilm():
    """O13: with the 'surge' init, distinct texts must not collapse (mean cos <= 0.6, max <= 0.9)."""
    cfg = ENCODERS["minilm"]
    w = make_weights(cfg, seed=1234, init="surge")
    wl = make_workload(WORKLOADS["minilm"].__class__(**{**WORKLOADS["minilm"].__dict__, "n_texts": 40, "n_partitions": 4}),
                       cfg.vocab_size, cfg.max_position, seed=0)
    texts = [wl.ids[a:b] for a, b in zip(np.concatenate([[0], np.cumsum(wl.lengths)[:-1]]), np.cumsum(wl.lengths))]
    X = enc.Encoder(cfg, w).encode_texts(texts)
    C = X @ X.T
    off = C[~np.eye(len(X), dtype=bool)]
    assert off.mean() <= 0.6 and off.max() <= 0.9, (off.mean(), off.max())


def test_cls_pooling_pin():
    """[CLS] pooling (bge's native): closed form e = h_0 / ||h_0|| on a known
    matrix, equal to mean pooling for one-token texts, and the full encoder vs transformers' CLS
    hidden state (independent library)."""
    h = np.array([[3.0, 4.0], [10.0, -1.0], [0.5, 0.5]])
    assert np.allclose(enc.cls_pool_l2(h), [0.6, 0.8])
    assert np.allclose(enc.cls_pool_l2(h[:1]), enc.mean_pool_l2(h[:1]))
    cfg = ENCODERS["toy"]
    w = make_weights(cfg, seed=99, init="pin")
    texts = random_texts(12, cfg.vocab_size, cfg.max_position, seed=3, lo=1, cls_id=1, sep_id=2, id_lo=4)
    E = enc.Encoder(cfg, w)
    ours = np.stack([E.encode_text(t, pooling="cls") for t in texts])
    assert np.max(np.abs(ours - hf_reference(cfg, w, texts, pooling="cls"))) <= 1e-10
    assert not np.allclose(ours, E.encode_texts(texts))
