"""NEXT N2: partition-skew sweep on one B200, the paper's `tab:sigma-sweep`
configuration (MiniLM-L6 class, N = 10M, P = 4,000, log-normal sigma in {1.0, 1.72, 2.5}).

Per sigma: the whole stream through the streaming C ABI from host memory, once partition-by-partition
(PBP, B_min = 1) and once with SURGE's thresholds (B_min = 100K, B_max = 500K); reports texts/s,
the speedup over PBP (the paper: invariant within +-3%), TTFO, safety flushes, n_max and the peak
buffered texts against the Lemma bound B_min - 1 + n_max.

    python scripts/sigma_sweep.py [--n-texts N] [--reps R] [--out profiles/r01/sigma_sweep.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

from synth.configs import ENCODERS, WORKLOADS, scaled  # noqa: E402
from synth.weights import make_weights, pack_blob  # noqa: E402
from synth.workload import make_workload  # noqa: E402
from theorem_b200 import run_stream  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-texts", type=int, default=0)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--out", default="")
    args = ap.parse_args()

    import torch
    from paper_2605_01060_b200 import native as N

    ecfg = ENCODERS["minilm"]
    blob = torch.from_numpy(pack_blob(ecfg, make_weights(ecfg, seed=1234)).view(np.uint8)).cuda()
    rows = []
    for wname in ("minilm_s1.0", "minilm", "minilm_s2.5"):
        wcfg = WORKLOADS[wname]
        if args.n_texts:
            wcfg = scaled(wcfg, n_texts=args.n_texts)
        wl = make_workload(wcfg, ecfg.vocab_size, ecfg.max_position, seed=0)
        parts = [wl.partition(k) for k in range(len(wl.sizes))]
        n, n_max = wl.n_texts, int(wl.sizes.max())
        res = {}
        for mode, b_min, b_max in (("pbp", 1, 2), ("surge", 100_000, 500_000)):
            h = N.surge_create(N.make_config(ecfg, b_min, b_max, weights_on_device=1), blob,
                               n_weights=blob.numel() // 2)
            run_stream(N, h, parts)                   # warm-up
            ts, st = [], None
            for _ in range(args.reps):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                got, st = run_stream(N, h, parts)
                torch.cuda.synchronize()
                ts.append(time.perf_counter() - t0)
                assert got == n
            N.surge_destroy(h)
            res[mode] = {"wall_s": float(np.median(ts)), "texts_per_s": n / float(np.median(ts)),
                         "invocations": int(st["superbatches"]), "safety_flushes": int(st["safety_flushes"]),
                         "ttfo_s": st["ttfo_s"], "peak_buffered_texts": int(st["peak_buffered_texts"]),
                         "lemma_bound": b_min - 1 + n_max}
            assert res[mode]["peak_buffered_texts"] <= res[mode]["lemma_bound"]
        row = {"sigma": wcfg.sigma, "n_texts": n, "partitions": len(wl.sizes), "n_max": n_max,
               "speedup_over_pbp": res["pbp"]["wall_s"] / res["surge"]["wall_s"], **res}
        rows.append(row)
        print(json.dumps(row), flush=True)
    base = rows[1]["speedup_over_pbp"]
    print("| sigma | n_max | SURGE texts/s | PBP texts/s | speedup | vs sigma=1.72 | F | safety | TTFO s | "
          "peak buffered / Lemma bound |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for r in rows:
        s = r["surge"]
        print(f"| {r['sigma']} | {r['n_max']} | {s['texts_per_s']:.4g} | {r['pbp']['texts_per_s']:.4g} | "
              f"{r['speedup_over_pbp']:.3f} | {100 * (r['speedup_over_pbp'] / base - 1):+.1f}% | {s['invocations']} | "
              f"{s['safety_flushes']} | {s['ttfo_s']:.4f} | {s['peak_buffered_texts']} / {s['lemma_bound']} |")
    if args.out:
        with open(args.out, "w") as fh:
            json.dump({"gpu": torch.cuda.get_device_name(0), "runs": rows}, fh, indent=1)


if __name__ == "__main__":
    main()
