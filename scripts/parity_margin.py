"""Report the parity margin (min cosine, max |delta| vs the fp64 oracle) of the GPU path on sampled
texts of each encoder class -- used to judge numerics changes (e.g. ATT_P_SPLIT) against the
north-star gate (cos >= 0.999, max|delta| <= 1e-2).  SURGE_LIB selects a library variant."""
import numpy as np
import torch

from oracle import encoder as oenc
from paper_2605_01060_b200 import native as N
from synth.configs import ENCODERS
from synth.weights import make_weights, pack_blob

for enc, lmax, n in (("minilm", 20, 300), ("minilm", 128, 120), ("bgebase", 128, 60), ("bgelarge", 512, 16)):
    ecfg = ENCODERS[enc]
    w = make_weights(ecfg, seed=1234)
    rng = np.random.default_rng(3)
    lens = rng.integers(8, lmax + 1, size=n).astype(np.int32)
    ids = rng.integers(1000, ecfg.vocab_size, size=int(lens.sum())).astype(np.int32)
    h = N.surge_create(N.make_config(ecfg, 1000, 5000), pack_blob(ecfg, w))
    out = torch.zeros(n, ecfg.hidden, device="cuda")
    N.surge_encode_packed(h, torch.from_numpy(ids).cuda(), torch.from_numpy(lens).cuda(), lens, n, out)
    torch.cuda.synchronize()
    N.surge_destroy(h)
    got = out.cpu().numpy().astype(np.float64)
    E = oenc.Encoder(ecfg, w)
    off = np.concatenate([[0], np.cumsum(lens)])
    m = min(n, 40 if enc != "bgelarge" else 8)
    ref = np.stack([E.encode_text(ids[off[i]:off[i + 1]]) for i in range(m)])
    g = got[:m]
    cos = (g * ref).sum(1) / (np.linalg.norm(g, axis=1) * np.linalg.norm(ref, axis=1))
    print(f"{enc:9s} len<={lmax:3d}: min cos {cos.min():.7f}  max|d| {np.abs(g - ref).max():.3e}", flush=True)
