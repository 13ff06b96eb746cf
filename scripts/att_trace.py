"""Per-phase cycle counts of the fused QKV + attention epilogue (build with NVCC_EXTRA=-DATT_TRACE).

    NVCC_EXTRA=-DATT_TRACE python paper_2605_01060_b200/build.py --force && python scripts/att_trace.py
Encodes one 262,144-token chunk of C2-shaped texts; CTAs 0-3 print cycles/tile per phase.
"""
import numpy as np
import torch

from paper_2605_01060_b200 import native as N
from synth.configs import ENCODERS
from synth.weights import make_weights, pack_blob

ecfg = ENCODERS["minilm"]
w = make_weights(ecfg, seed=1234)
rng = np.random.default_rng(0)
lens = (2 + np.ceil(rng.integers(24, 71, size=18500) / 4)).astype(np.int32)
ids = rng.integers(1000, ecfg.vocab_size, size=int(lens.sum())).astype(np.int32)
h = N.surge_create(N.make_config(ecfg, 1000, 5000, chunk_tokens=262144), pack_blob(ecfg, w))
out = torch.zeros(len(lens), ecfg.hidden, device="cuda")
d_ids, d_len = torch.from_numpy(ids).cuda(), torch.from_numpy(lens).cuda()
for _ in range(2):
    N.surge_encode_packed(h, d_ids, d_len, lens, len(lens), out)
torch.cuda.synchronize()
N.surge_destroy(h)
print("tokens", int(lens.sum()))
