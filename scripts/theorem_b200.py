"""NEXT N3: Theorem 1 on B200.

Runs the whole C2 stream (10M texts, P = 4,000 log-normal(sigma=1.72) partitions, MiniLM-L6 class)
through the streaming C ABI (submit / poll / release from host memory, as the bench's e2e) at
partition-by-partition processing (PBP: B_min = 1, one invocation per partition) and at
B_min in {10K, 50K, 100K, 200K, 500K} (B_max = 5 B_min), fits T = F c_call + N c_enc
(paper_2605_01060_b200/costmodel.py, eq:partition-time / eq:speedup P:183) and compares the
measured speedup over PBP with the Theorem's prediction.

    python scripts/theorem_b200.py [--n-texts N] [--reps R] [--out profiles/r01/theorem_b200.json]
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

from paper_2605_01060_b200 import costmodel as cm  # noqa: E402
from synth.configs import ENCODERS, WORKLOADS, scaled  # noqa: E402
from synth.weights import make_weights, pack_blob  # noqa: E402
from synth.workload import make_workload  # noqa: E402


def run_stream(N, h, parts):
    n_rows = 0
    for key, ids, lens in parts:
        N.surge_submit_partition(h, key, ids, lens)
        for r in N.surge_poll_flushed(h, 4096, 0):
            n_rows += r.n_rows
            N.surge_release(h, r)
    N.surge_finish(h)
    while N.surge_pending(h) > 0:
        for r in N.surge_poll_flushed(h, 4096, 20):
            n_rows += r.n_rows
            N.surge_release(h, r)
    for r in N.surge_poll_flushed(h, 4096, 0):
        n_rows += r.n_rows
        N.surge_release(h, r)
    st = N.surge_get_stats(h)
    N.surge_reset(h)
    return n_rows, st


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-texts", type=int, default=0)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--out", default="")
    args = ap.parse_args()

    import torch
    from paper_2605_01060_b200 import native as N

    ecfg = ENCODERS["minilm"]
    wcfg = WORKLOADS["minilm"]
    if args.n_texts:
        wcfg = scaled(wcfg, n_texts=args.n_texts)
    wl = make_workload(wcfg, ecfg.vocab_size, ecfg.max_position, seed=0)
    parts = [wl.partition(k) for k in range(len(wl.sizes))]
    blob = torch.from_numpy(pack_blob(ecfg, make_weights(ecfg, seed=1234)).view(np.uint8)).cuda()
    n, p = wl.n_texts, len(wl.sizes)
    rows = []
    for b_min in (1, 10_000, 50_000, 100_000, 200_000, 500_000):
        b_max = max(5 * b_min, 2)
        cfg = N.make_config(ecfg, b_min, b_max, weights_on_device=1)
        h = N.surge_create(cfg, blob, n_weights=blob.numel() // 2)
        run_stream(N, h, parts)                      # warm-up (pinned pools, workspaces)
        ts, st = [], None
        for _ in range(args.reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            got, st = run_stream(N, h, parts)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
            assert got == n, (got, n)
        N.surge_destroy(h)
        rows.append({"b_min": b_min, "b_max": b_max, "invocations": int(st["superbatches"]),
                     "wall_s": float(np.median(ts)), "wall_s_all": ts, "texts_per_s": n / float(np.median(ts)),
                     "ttfo_s": st["ttfo_s"], "peak_buffered_texts": int(st["peak_buffered_texts"]),
                     "theorem_bound": int(-(-n // b_min)) if b_min > 1 else p})
        print(json.dumps(rows[-1]), flush=True)
    f = cm.fit([r["invocations"] for r in rows], [r["wall_s"] for r in rows], n)
    a = cm.alpha(p, n, f.c_call, f.c_enc)
    t_pbp = rows[0]["wall_s"]
    for r in rows:
        r["speedup_measured"] = t_pbp / r["wall_s"]
        r["speedup_predicted"] = cm.speedup(a, r["invocations"], p)
        r["error_pct"] = 100.0 * (r["speedup_predicted"] - r["speedup_measured"]) / r["speedup_measured"]
    summary = {"n_texts": n, "partitions": p, "c_call_s": f.c_call, "c_enc_s": f.c_enc, "alpha": a,
               "n_star": f.c_call / f.c_enc, "fit_residual_rms_s": f.residual_rms, "runs": rows,
               "gpu": torch.cuda.get_device_name(0)}
    print(json.dumps({k: v for k, v in summary.items() if k != "runs"}), flush=True)
    print("| B_min | F | wall s | texts/s | speedup meas. | speedup pred. | err % | TTFO s | peak buffered |")
    print("|---|---|---|---|---|---|---|---|---|")
    for r in rows:
        print(f"| {r['b_min'] if r['b_min'] > 1 else 'PBP'} | {r['invocations']} | {r['wall_s']:.3f} | "
              f"{r['texts_per_s']:.4g} | {r['speedup_measured']:.3f} | {r['speedup_predicted']:.3f} | "
              f"{r['error_pct']:+.2f} | {r['ttfo_s']:.4f} | {r['peak_buffered_texts']} |")
    if args.out:
        with open(args.out, "w") as fh:
            json.dump(summary, fh, indent=1)


if __name__ == "__main__":
    main()
