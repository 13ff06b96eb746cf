"""Small runs of the round-2 kernels for compute-sanitizer (scripts/sanitize.sh): the tcgen05 QKV + attention
kernel (MiniLM class, head-split staging), the cluster-pair LayerNorm GEMMs and the long-text attention
(bge-base class, texts of 20..512 tokens over every length-class edge: the tcgen05 kernels when the caller
sets SURGE_ATT_LONG_TC=1, else the mma.sync kernel's length classes)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2605_01060_b200 import native as N  # noqa: E402
from synth.configs import ENCODERS  # noqa: E402
from synth.weights import make_weights, pack_blob  # noqa: E402


def encode(ecfg, lens, ids, **opt):
    h = N.surge_create(N.make_config(ecfg, 1000, 5000, chunk_tokens=4096), pack_blob(ecfg, make_weights(ecfg, seed=1234)))
    try:
        for k, v in opt.items():
            N.surge_set_option(h, getattr(N, k), v)
        out = torch.zeros(len(lens), ecfg.hidden, device="cuda")
        N.surge_encode_packed(h, torch.from_numpy(ids).cuda(), torch.from_numpy(lens).cuda(), lens, len(lens), out)
        torch.cuda.synchronize()
        return out.cpu().numpy()
    finally:
        N.surge_destroy(h)


rng = np.random.default_rng(3)
mini = ENCODERS["minilm"]
lens = rng.integers(1, 129, size=40).astype(np.int32)
ids = rng.integers(1000, mini.vocab_size, size=int(lens.sum())).astype(np.int32)
a = encode(mini, lens, ids, SURGE_OPT_ATT_TC=1)
base = ENCODERS["bgebase"]
lens = np.array([130, 200, 300, 20, 64, 90, 65, 128, 129, 192, 193, 256, 257, 512], dtype=np.int32)   # every length class
ids = rng.integers(1000, base.vocab_size, size=int(lens.sum())).astype(np.int32)
b = encode(base, lens, ids, SURGE_OPT_LN_PAIR=1)
print("new kernels ok", bool(np.isfinite(a).all() and np.isfinite(b).all()))
