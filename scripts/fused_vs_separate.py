"""Max difference between the fused kernels' embeddings and the separate-kernel path (same inputs)."""
import numpy as np
import torch

from paper_2605_01060_b200 import native as N
from synth.configs import ENCODERS
from synth.weights import make_weights, pack_blob

for enc in ("toy", "minilm"):
    ecfg = ENCODERS[enc]
    w = make_weights(ecfg, seed=1234)
    rng = np.random.default_rng(11)
    lens = rng.integers(1, min(64, ecfg.max_position) + 1, size=3000).astype(np.int32)
    ids = rng.integers(4 if enc == "toy" else 1000, ecfg.vocab_size, size=int(lens.sum())).astype(np.int32)
    outs = []
    for mlp, tail in ((1, 1), (0, 0)):
        h = N.surge_create(N.make_config(ecfg, 1000, 5000, chunk_tokens=16384), pack_blob(ecfg, w))
        N.surge_set_option(h, N.SURGE_OPT_MLP_FUSED, mlp)
        N.surge_set_option(h, N.SURGE_OPT_TAIL_FUSED, tail)
        out = torch.zeros(len(lens), ecfg.hidden, device="cuda")
        N.surge_encode_packed(h, torch.from_numpy(ids).cuda(), torch.from_numpy(lens).cuda(), lens, len(lens), out)
        torch.cuda.synchronize()
        N.surge_destroy(h)
        outs.append(out.cpu().numpy().astype(np.float64))
    a, b = outs
    cos = (a * b).sum(1) / (np.linalg.norm(a, axis=1) * np.linalg.norm(b, axis=1))
    print(f"{enc}: fused vs separate: min cos {cos.min():.8f} max|d| {np.abs(a - b).max():.3e}")
