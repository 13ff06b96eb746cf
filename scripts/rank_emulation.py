"""Predicted strong scaling of the 10M-text bench from ONE GPU: every rank's share, run one at a time.

At N GPUs each rank runs Alg. 1 over the whole stream and encodes only its LPT pieces of every
SuperBatch (no per-SuperBatch collective), so a rank's step time does not depend on the
other ranks.  This script runs, on one B200, the step of rank r of an N-GPU job (surge_config
rank = r, world_size = N; no process group is needed because the library exchanges nothing) for every
r, and reports max over ranks -- the device time bench.py would take at N GPUs, minus the one-time
NCCL weight broadcast.  Same workload, timing and warm-up rules as bench.py (CUDA events on the
launching stream, inputs resident in HBM).

    python scripts/rank_emulation.py [--worlds 1 2 4 8] [--steps 2] [--warmup 1] [--e2e]

--e2e adds the end-to-end number of every rank: the streaming C ABI from host memory (every rank
submits the WHOLE partition stream -- Alg.1 runs on every rank -- and encodes, copies back, polls and
releases only its own LPT pieces), wall clock per rank, job value = N texts / max over ranks.
"""
from __future__ import annotations

import argparse
import json
import time
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2605_01060_b200 import native as N  # noqa: E402
from synth.configs import ENCODERS, WORKLOADS, scaled  # noqa: E402
from synth.weights import make_weights, pack_blob  # noqa: E402
from synth.workload import make_workload  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--worlds", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--n-texts", type=int, default=0)
    ap.add_argument("--out", default="")
    ap.add_argument("--e2e", action="store_true")
    args = ap.parse_args()

    dev = torch.device("cuda", 0)
    ecfg, wcfg = ENCODERS["minilm"], WORKLOADS["minilm"]
    if args.n_texts:
        wcfg = scaled(wcfg, n_texts=args.n_texts)
    wl = make_workload(wcfg, ecfg.vocab_size, ecfg.max_position, seed=0)
    parts = [wl.partition(k) for k in range(len(wl.sizes))]

    from paper_2605_01060_b200.driver import stream as drive_stream

    def run_stream(h):
        t0 = time.perf_counter()
        n_rows = drive_stream(N, h, parts)    # submit on this thread, poll + release on a second one
        wall = time.perf_counter() - t0
        st = N.surge_get_stats(h)
        N.surge_reset(h)
        return wall, wall, n_rows, st

    blob = torch.from_numpy(pack_blob(ecfg, make_weights(ecfg, seed=1234)).view(np.uint8)).to(dev)
    sizes = wl.sizes.astype(np.int64)
    d_ids = torch.from_numpy(wl.ids).to(dev)
    d_len = torch.from_numpy(wl.lengths).to(dev)
    d_out = torch.empty(wl.n_texts, ecfg.hidden, dtype=torch.float32, device=dev)
    stream = torch.cuda.Stream(device=dev)
    rows = []
    base = None
    for world in args.worlds:
        per_rank = []
        for rank in range(world):
            cfg = N.make_config(ecfg, wcfg.b_min, wcfg.b_max, rank=rank, world_size=world, device=0,
                                weights_on_device=1)
            h = N.surge_create(cfg, blob, n_weights=blob.numel() // 2)

            def step():
                sbs, _ = N.surge_aggregate(sizes, wcfg.b_min, wcfg.b_max)
                for a, b, _r in sbs:
                    t0, t1 = int(wl.text_off[a]), int(wl.text_off[b])
                    k0 = int(wl.tok_off[a])
                    N.surge_encode_superbatch(h, d_ids.data_ptr() + 4 * k0, d_len.data_ptr() + 4 * t0,
                                              wl.lengths[t0:t1], sizes[a:b],
                                              d_out.data_ptr() + 4 * t0 * ecfg.hidden, stream)

            for _ in range(args.warmup):
                step()
            torch.cuda.synchronize()
            st0 = N.surge_get_stats(h)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.steps):
                step()
            e1.record(stream)
            torch.cuda.synchronize()
            st1 = N.surge_get_stats(h)
            ms = e0.elapsed_time(e1) / args.steps
            launches = (st1["kernel_launches"] - st0["kernel_launches"]) // args.steps
            rec = {"rank": rank, "ms_per_step": ms, "launches_per_step": int(launches)}
            if args.e2e:
                run_stream(h)                                  # warm-up (pinned pools)
                wall, t_sub, n_rows, st = run_stream(h)
                rec.update(e2e_s=wall, e2e_submit_s=t_sub, e2e_rows=n_rows, e2e_ttfo_s=st["ttfo_s"])
            per_rank.append(rec)
            N.surge_destroy(h)
        ms_max = max(r["ms_per_step"] for r in per_rank)
        ms_min = min(r["ms_per_step"] for r in per_rank)
        value = wl.n_texts / (ms_max / 1e3)
        if base is None:
            base = value
        row = {"n_gpus": world, "ms_per_step_max": ms_max, "ms_per_step_min": ms_min,
               "texts_per_s": value, "efficiency_vs_1": value / (base * world) if base else None,
               "ranks": per_rank}
        if args.e2e:
            e2e_max = max(r["e2e_s"] for r in per_rank)
            assert sum(r["e2e_rows"] for r in per_rank) == wl.n_texts
            row.update(e2e_s_max=e2e_max, e2e_texts_per_s=wl.n_texts / e2e_max,
                       e2e_over_device=(wl.n_texts / e2e_max) / value,
                       e2e_submit_s_max=max(r["e2e_submit_s"] for r in per_rank))
        rows.append(row)
        print(json.dumps({k: v for k, v in row.items() if k != "ranks"}), flush=True)
    out = {"workload": f"minilm: N={wl.n_texts} texts, P={len(sizes)} sigma=1.72, B_min={wcfg.b_min}",
           "method": "each rank of an N-GPU job run alone on one B200 (rank/world_size in surge_config); "
                     "value = N texts / max over ranks of the step time", "rows": rows}
    if args.out:
        with open(args.out, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
