"""Per-kernel GPU tests through the C ABI (device pointers from torch tensors).

Each kernel is compared with (a) the oracle where it computes a step of the method (pack, embed,
pool) and (b) a plain PyTorch fp32 reference of the same op on the same bf16 inputs (GEMM
epilogues, attention).  Shapes span several tiles and ragged tails.
"""
import math

import numpy as np
import pytest
import torch

from oracle import aggregator as oagg
from oracle import encoder as oenc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def N():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2605_01060_b200 import native
    return native


def dev(x, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(x))
    return t.to("cuda") if dtype is None else t.to("cuda", dtype)


def bf16_bits(t: torch.Tensor) -> torch.Tensor:
    return t.to(torch.bfloat16).view(torch.int16)


def from_bits(t: torch.Tensor) -> torch.Tensor:
    return t.view(torch.bfloat16).float()


# n > 8192 runs the multi-CTA scan (one CTA per 8K tile, then the partition offsets); 16384: exact
# tile multiple; 600,000 x 1,000 members: a Safety-flush-sized SuperBatch (sigma = 2.5)
@pytest.mark.parametrize("n,m", [(1, 1), (5, 2), (8191, 3), (8192, 7), (8193, 11), (16384, 0), (16385, 2),
                                 (300_000, 45), (600_000, 1000), (10, 0)])
def test_pack_bit_exact(N, n, m):
    rng = np.random.default_rng(n + m)
    lengths = rng.integers(1, 513, size=n).astype(np.int32)
    if m:
        cuts = np.sort(rng.choice(np.arange(1, n), size=m - 1, replace=False)) if m > 1 else np.array([], int)
        sizes = np.diff(np.concatenate([[0], cuts, [n]])).astype(np.int32)
    else:
        sizes = np.zeros(0, np.int32)
    dl = dev(lengths)
    ds = dev(sizes) if m else torch.zeros(1, dtype=torch.int32, device="cuda")
    cu = torch.full((n + 1,), -7, dtype=torch.int32, device="cuda")
    ro = torch.full((m + 1,), -7, dtype=torch.int32, device="cuda")
    to = torch.full((m + 1,), -7, dtype=torch.int32, device="cuda")
    N.surge_op_pack(dl, n, ds, m, cu, ro, to)
    torch.cuda.synchronize()
    p = oagg.pack(lengths, list(sizes))
    assert np.array_equal(cu.cpu().numpy(), p.cu_seqlens)
    if m:
        assert np.array_equal(ro.cpu().numpy(), p.part_row_off)
        assert np.array_equal(to.cpu().numpy(), p.part_tok_off)


GEMM_CASES = [
    # (M, N, K, epi)   encoder shapes (C2: d=384, ff=1536; C1: d=64, ff=256) and ragged M
    (1, 1152, 384, 0), (127, 1152, 384, 0), (4133, 1152, 384, 0),
    (300, 1536, 384, 1), (4133, 1536, 384, 1),
    (129, 384, 384, 2), (4133, 384, 384, 2), (1000, 384, 1536, 2),
    (77, 192, 64, 0), (300, 256, 64, 1), (300, 64, 64, 2), (333, 64, 256, 2),
    (256, 128, 128, 0), (200, 64, 192, 0),
    # many tiles per CTA (weight-stationary slices, TMEM double buffering) + ragged tails
    (50001, 1152, 384, 0), (50001, 1536, 384, 1), (50001, 384, 384, 2), (20001, 384, 1536, 2),
    # bge-base / bge-large class shapes (N1): streaming 256-column tiles, fp32 pre-LN epilogue (epi 3)
    (3001, 2304, 768, 0), (3001, 3072, 768, 1), (3001, 768, 768, 3), (3001, 768, 3072, 3), (777, 1024, 4096, 3),
    (3001, 4096, 1024, 1), (255, 3072, 768, 1),
]


@pytest.mark.parametrize("M,Nn,K,epi", GEMM_CASES)
def test_gemm_vs_torch(N, M, Nn, K, epi):
    g = torch.Generator(device="cuda").manual_seed(M * 7 + Nn + K + epi)
    A = bf16_bits(torch.randn(M, K, device="cuda", generator=g))
    B = bf16_bits(torch.randn(Nn, K, device="cuda", generator=g) * (1.0 / math.sqrt(K)))
    bias = torch.randn(Nn, device="cuda", generator=g) * 0.1
    res = bf16_bits(torch.randn(M, Nn, device="cuda", generator=g))
    gamma = 1 + 0.1 * torch.randn(Nn, device="cuda", generator=g)
    beta = 0.1 * torch.randn(Nn, device="cuda", generator=g)
    Cc = torch.zeros(M, Nn, dtype=torch.float32 if epi == 3 else torch.int16, device="cuda")
    N.surge_op_gemm(A, B, bias, res, gamma, beta, Cc, M, Nn, K, epi, 1e-12)
    torch.cuda.synchronize()
    acc = from_bits(A) @ from_bits(B).T + bias
    if epi == 3:   # fp32 out: only the fp32 accumulation order differs from torch
        ref = acc + from_bits(res)
        err = (Cc - ref).abs()
        assert bool((err <= 1e-5 * ref.abs() + 1e-4).all()), f"max err {err.max().item():.4g}"
        return
    if epi == 1:
        ref = torch.nn.functional.gelu(acc)
    elif epi == 2:
        ref = torch.nn.functional.layer_norm(acc + from_bits(res), (Nn,), gamma, beta, eps=1e-12)
    else:
        ref = acc
    got = from_bits(Cc)
    err = (got - ref).abs()
    tol = 2 ** -7 * ref.abs() + 2e-3
    assert bool((err <= tol).all()), f"max err {err.max().item():.4g} at {divmod(int(err.argmax()), Nn)}"


def ref_attention(qkv, cu, heads, dh):
    """fp32 SDPA per text; also returns, per output element, max |v| over the text's keys for its
    head (the scale of the bf16 rounding error of P, see test_attention_vs_torch)."""
    d = heads * dh
    out = torch.empty(qkv.shape[0], d, device=qkv.device)
    vmax = torch.empty(qkv.shape[0], d, device=qkv.device)
    for s in range(len(cu) - 1):
        a, b = cu[s], cu[s + 1]
        x = qkv[a:b].view(b - a, 3, heads, dh).permute(1, 2, 0, 3)
        o = torch.nn.functional.scaled_dot_product_attention(x[0][None], x[1][None], x[2][None])[0]
        out[a:b] = o.permute(1, 0, 2).reshape(b - a, d)
        vm = x[2].abs().amax(dim=(1, 2))                      # [heads]
        vmax[a:b] = vm.repeat_interleave(dh)[None, :].expand(b - a, d)
    return out, vmax


@pytest.mark.parametrize("heads,dh,maxlen", [(12, 32, 128), (4, 16, 64), (12, 32, 20), (16, 64, 300), (12, 32, 65),
                                             (16, 64, 512), (12, 32, 257)])
def test_attention_vs_torch(N, heads, dh, maxlen):
    rng = np.random.default_rng(heads * dh + maxlen)
    lens = rng.integers(1, maxlen + 1, size=97).astype(np.int32)
    lens[:6] = [1, 2, 31, min(33, maxlen), min(64, maxlen), min(65, maxlen)]   # tile/long kernel boundary
    # the long kernel's length-class edges (64, 128], (128, 192], (192, 256], (256, 512]
    edges = [e for e in (128, 129, 192, 193, 256, 257) if e <= maxlen]
    lens[6:6 + len(edges)] = edges
    lens[-1] = maxlen
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    T = int(cu[-1])
    g = torch.Generator(device="cuda").manual_seed(5)
    qkv = bf16_bits(torch.randn(T, 3 * heads * dh, device="cuda", generator=g))
    out = torch.zeros(T, heads * dh, dtype=torch.int16, device="cuda")
    N.surge_op_attention(qkv, dev(cu), len(lens), heads, dh, out)
    torch.cuda.synchronize()
    ref, vmax = ref_attention(from_bits(qkv), cu.tolist(), heads, dh)
    err = (from_bits(out) - ref).abs()
    # bf16 output rounding (2^-9 relative, 2^-7 with margin) + P entering P V as bf16: each p_j is
    # rounded to 2^-9 relative and the normaliser uses the unrounded sum, so |dO| <= 2^-8 max_j |v_j|
    tol = 2 ** -7 * ref.abs() + 2 ** -8 * vmax + 1e-3
    assert bool((err <= tol).all()), (err - tol).max().item()
    # length-1 texts: softmax of one score is 1 -> output = v (bit-exact after bf16 rounding of v)
    v0 = from_bits(qkv)[0, 2 * heads * dh:]
    assert torch.equal(from_bits(out)[0], v0)


@pytest.mark.parametrize("d", [64, 384])
def test_meanpool_l2_vs_oracle(N, d):
    rng = np.random.default_rng(d)
    lens = rng.integers(1, 80, size=501).astype(np.int32)
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    T = int(cu[-1])
    x = bf16_bits(torch.from_numpy(rng.standard_normal((T, d)).astype(np.float32)).cuda())
    out = torch.zeros(len(lens), d, device="cuda")
    N.surge_op_meanpool_l2(x, dev(cu), len(lens), d, out)
    torch.cuda.synchronize()
    xf = from_bits(x).cpu().double().numpy()
    ref = np.stack([oenc.mean_pool_l2(xf[cu[i]:cu[i + 1]]) for i in range(len(lens))])
    assert np.max(np.abs(out.cpu().double().numpy() - ref)) <= 2e-6
    assert np.max(np.abs(np.linalg.norm(out.cpu().double().numpy(), axis=1) - 1)) <= 1e-5


@pytest.mark.parametrize("name", ["toy", "minilm"])
def test_embed_ln_vs_oracle(N, name):
    from synth.configs import ENCODERS
    from synth.weights import make_weights, pack_blob
    from synth.workload import random_texts
    e = ENCODERS[name]
    w = make_weights(e, seed=3, init="pin")
    h = N.surge_create(N.make_config(e, 64, 320), pack_blob(e, w))
    try:
        texts = random_texts(40, e.vocab_size, min(e.max_position, 128), seed=4, lo=1)
        lens = np.array([len(t) for t in texts], np.int32)
        cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
        ids = np.concatenate(texts).astype(np.int32)
        x = torch.zeros(int(cu[-1]), e.hidden, dtype=torch.int16, device="cuda")
        N.surge_op_embed_ln(h, dev(ids), dev(cu), len(texts), x)
        torch.cuda.synchronize()
        got = from_bits(x).cpu().double().numpy()
        E = oenc.Encoder(e, w)
        ref = np.concatenate([E.embed(t) for t in texts])
        assert np.max(np.abs(got - ref) - 2 ** -8 * np.abs(ref)) <= 1e-3
    finally:
        N.surge_destroy(h)


@pytest.mark.parametrize("d", [768, 1024])
def test_layernorm_rows_vs_torch(N, d):
    g = torch.Generator(device="cuda").manual_seed(d)
    v = torch.randn(3001, d, device="cuda", generator=g) * 3 + 0.5
    gamma = 1 + 0.1 * torch.randn(d, device="cuda", generator=g)
    beta = 0.1 * torch.randn(d, device="cuda", generator=g)
    y = torch.zeros(3001, d, dtype=torch.int16, device="cuda")
    N.surge_op_layernorm(v, 3001, d, gamma, beta, y, 1e-12)
    torch.cuda.synchronize()
    ref = torch.nn.functional.layer_norm(v, (d,), gamma, beta, eps=1e-12)
    err = (from_bits(y) - ref).abs()
    assert bool((err <= 2 ** -8 * ref.abs() + 1e-4).all()), err.max().item()
