"""NEXT N2: the C5 skew / scale stress (BASELINE.json configs[4]: MiniLM-L6 class,
N = 10^8 texts, P = 40,000 log-normal partitions, sigma in {1.0, 1.72, 2.5}) through the streaming
C ABI on one B200, under each B_max reading (include/surge.h SURGE_BMAX_*; R2/R3/R23).

Per (sigma, policy), in its own process (so the host peak RSS is that run's): the whole 10^8-text
stream submitted partition by partition from host memory, every piece polled and released; reports
wall time, texts/s, TTFO (first submit -> first piece pollable), F and the Safety-flush count, n_max,
the largest SuperBatch, peak buffered texts against the Lemma bound (B_min - 1 + n_max;
SPLIT: B_max), the largest pinned output a SuperBatch needs (S_max x d x 4 B, P:480's M(S) term), and
the host peak RSS (VmHWM).

    python scripts/c5_sweep.py [--n-texts N] [--n-partitions P] [--out profiles/r02/c5_sweep.json]
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def one(sigma: str, policy: str, n_texts: int, n_partitions: int) -> dict:
    import torch
    from dataclasses import replace

    from paper_2605_01060_b200 import native as N
    from paper_2605_01060_b200.driver import stream
    from synth.configs import ENCODERS, WORKLOADS
    from synth.weights import make_weights, pack_blob
    from synth.workload import make_workload

    ecfg = ENCODERS["minilm"]
    wcfg = WORKLOADS[f"c5_s{sigma}"]
    if n_texts or n_partitions:
        wcfg = replace(wcfg, n_texts=n_texts or wcfg.n_texts, n_partitions=n_partitions or wcfg.n_partitions)
    t0 = time.perf_counter()
    wl = make_workload(wcfg, ecfg.vocab_size, ecfg.max_position, seed=0)
    t_gen = time.perf_counter() - t0
    parts = [wl.partition(k) for k in range(len(wl.sizes))]
    blob = torch.from_numpy(pack_blob(ecfg, make_weights(ecfg, seed=1234)).view(np.uint16)).cuda()
    pol = N.BMAX_POLICIES[policy]
    h = N.surge_create(N.make_config(ecfg, wcfg.b_min, wcfg.b_max, weights_on_device=1, bmax_policy=pol), blob,
                       n_weights=blob.numel())
    sbs, _ = N.surge_aggregate_ex(wl.sizes, wcfg.b_min, wcfg.b_max, pol)
    s_max = max(sum(m[2] for m in mm) for _, mm in sbs)
    try:
        # warm-up on a prefix (kernels, pinned pools for the common SuperBatch sizes)
        k_warm = int(np.searchsorted(np.cumsum(wl.sizes), 2_000_000)) + 1
        stream(N, h, parts[:k_warm])
        N.surge_reset(h)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        n_rows = stream(N, h, parts)              # submit here, poll + release on a second thread
        t_submit = time.perf_counter() - t0
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        st = N.surge_get_stats(h)
    finally:
        N.surge_destroy(h)
    assert n_rows == wl.n_texts
    n_max = int(wl.sizes.max())
    rss = None
    for line in open("/proc/self/status"):
        if line.startswith("VmHWM:"):
            rss = int(line.split()[1]) / 1e6
    lemma = wcfg.b_min - 1 + n_max
    return {"sigma": float(sigma), "policy": policy, "n_texts": wl.n_texts, "n_partitions": len(wl.sizes),
            "n_tokens": wl.n_tokens, "n_max": n_max, "wall_s": wall, "submit_s": t_submit,
            "texts_per_s": wl.n_texts / wall, "tokens_per_s": wl.n_tokens / wall, "ttfo_s": st["ttfo_s"],
            "superbatches": st["superbatches"], "safety_flushes": st["safety_flushes"],
            "largest_superbatch": s_max, "peak_buffered_texts": st["peak_buffered_texts"],
            "lemma_bound": lemma, "bound_checked": (wcfg.b_max if policy == "split" else lemma),
            "within_bound": st["peak_buffered_texts"] <= (wcfg.b_max if policy == "split" else lemma),
            "peak_inflight_texts": st["peak_inflight_texts"], "max_pinned_output_gb": s_max * ecfg.hidden * 4 / 1e9,
            "host_peak_rss_gb": rss, "encode_ms_total": st["encode_ms_total"], "gen_s": t_gen}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-texts", type=int, default=0)
    ap.add_argument("--n-partitions", type=int, default=0)
    ap.add_argument("--configs", default="1.0:label,1.72:label,1.72:split,2.5:label,2.5:split,2.5:preflush")
    ap.add_argument("--out", default="")
    ap.add_argument("--one", default="", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.one:
        sigma, policy = args.one.split(":")
        print("RESULT " + json.dumps(one(sigma, policy, args.n_texts, args.n_partitions)), flush=True)
        return
    rows = []
    for spec in args.configs.split(","):
        cmd = [sys.executable, os.path.abspath(__file__), "--one", spec, "--n-texts", str(args.n_texts),
               "--n-partitions", str(args.n_partitions)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        res = [ln for ln in r.stdout.splitlines() if ln.startswith("RESULT ")]
        if r.returncode != 0 or not res:
            print(f"{spec}: failed rc={r.returncode}\n{r.stderr[-3000:]}", flush=True)
            continue
        d = json.loads(res[0][7:])
        rows.append(d)
        print(json.dumps(d), flush=True)
    if args.out:
        os.makedirs(os.path.dirname(args.out), exist_ok=True)
        json.dump(rows, open(args.out, "w"), indent=1)
        md = ["| sigma | policy | n_max | texts/s | TTFO s | F | safety | largest SB | peak buffered / bound | "
              "max pinned out GB | host RSS GB |", "|---|---|---|---|---|---|---|---|---|---|---|"]
        for d in rows:
            md.append(f"| {d['sigma']} | {d['policy']} | {d['n_max']} | {d['texts_per_s']:.3e} | {d['ttfo_s']:.4f} | "
                      f"{d['superbatches']} | {d['safety_flushes']} | {d['largest_superbatch']} | "
                      f"{d['peak_buffered_texts']} / {d['bound_checked']} | {d['max_pinned_output_gb']:.2f} | "
                      f"{d['host_peak_rss_gb']:.1f} |")
        open(args.out.replace(".json", ".md"), "w").write("\n".join(md) + "\n")
        print("\n".join(md))


if __name__ == "__main__":
    main()
