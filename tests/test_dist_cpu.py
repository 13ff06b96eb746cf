"""Multi-process (world_size 2, gloo, CPU) coverage of the N > 1 host path.

Each rank runs what a libsurge process runs before any kernel: Alg.1 aggregation (surge_aggregate,
P:274-296) over the same partition stream, then the LPT shard plan (surge_lpt_plan) of every
SuperBatch, keeping its own pieces.  The ranks exchange their piece lists over gloo; the union must
cover every row of every SuperBatch exactly once and match the oracle's plan.  The weight blob is
replicated from rank 0 with a broadcast, as bench.py does over NCCL.  A torchrun launch of
`bench.py --impl reference` checks the reference arm's rank behaviour (rank 0 prints one JSON
line, the other ranks exit 0 without work).
"""
from __future__ import annotations

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, world: int, port: int, out_dir: str):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2605_01060_b200 import native as N
        from synth.configs import ENCODERS, WORKLOADS, scaled
        from synth.weights import make_weights, pack_blob
        from synth.workload import make_workload

        ecfg = ENCODERS["toy"]
        wcfg = scaled(WORKLOADS["minilm"], n_texts=20000, n_partitions=60, b_min=2000, b_max=10000)
        wl = make_workload(wcfg, ecfg.vocab_size, ecfg.max_position, seed=7)
        sbs, peak = N.surge_aggregate(wl.sizes, wcfg.b_min, wcfg.b_max)
        mine = []
        for j, (a, b, _r) in enumerate(sbs):
            t0, t1 = int(wl.text_off[a]), int(wl.text_off[b])
            plan = N.surge_lpt_plan(wl.lengths[t0:t1], wl.sizes[a:b], world)
            for i in range(len(plan["rank"])):
                if int(plan["rank"][i]) == rank:
                    mine.append((j, int(plan["first_row"][i]), int(plan["n_rows"][i]), int(plan["tokens"][i])))
        gathered = [None] * world
        dist.all_gather_object(gathered, mine)
        # weights: rank 0 draws, broadcast replicates (bench.py does this over NCCL)
        if rank == 0:
            blob = torch.from_numpy(pack_blob(ecfg, make_weights(ecfg, seed=1234)).view(np.uint8).copy())
        else:
            blob = torch.zeros(2 * sum(int(np.prod(s)) for s in _shapes(ecfg)), dtype=torch.uint8)
        dist.broadcast(blob, src=0)       # bytes: neither gloo nor NCCL reduce/broadcast int16
        ok_blob = bool(np.array_equal(blob.numpy().view(np.uint16),
                                      pack_blob(ecfg, make_weights(ecfg, seed=1234))))
        if rank == 0:
            json.dump({"pieces": gathered, "n_sb": len(sbs), "peak": peak, "blob_ok": ok_blob},
                      open(os.path.join(out_dir, "dist.json"), "w"))
        else:
            assert ok_blob
    finally:
        dist.destroy_process_group()


def _shapes(ecfg):
    from synth.weights import blob_layout
    return [s for _, s in blob_layout(ecfg)]


def test_two_rank_lpt_cover_and_broadcast(tmp_path):
    pytest.importorskip("paper_2605_01060_b200")
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    res = json.load(open(tmp_path / "dist.json"))
    assert res["blob_ok"]
    sys.path.insert(0, ROOT)
    from oracle import aggregator as oagg
    from synth.configs import ENCODERS, WORKLOADS, scaled
    from synth.workload import make_workload
    ecfg = ENCODERS["toy"]
    wcfg = scaled(WORKLOADS["minilm"], n_texts=20000, n_partitions=60, b_min=2000, b_max=10000)
    wl = make_workload(wcfg, ecfg.vocab_size, ecfg.max_position, seed=7)
    A = oagg.run_aggregator([int(k) for k in wl.keys], wl.sizes, wcfg.b_min, wcfg.b_max)
    assert res["n_sb"] == len(A.flushes)
    # exact cover of every SuperBatch's rows by the two ranks, and the oracle's assignment
    k = 0
    lo = 0
    for j, fl in enumerate(A.flushes):
        hi = lo + len(fl.keys)                   # members are consecutive partitions (arrival order)
        t0, t1 = int(wl.text_off[lo]), int(wl.text_off[hi])
        covered = np.zeros(t1 - t0, np.int32)
        loads = [0, 0]
        for rank in (0, 1):
            for (sb, fr, nr, tok) in res["pieces"][rank]:
                if sb != j:
                    continue
                covered[fr:fr + nr] += 1
                loads[rank] += tok
        assert np.all(covered == 1), j
        pieces, _per_rank = oagg.lpt_plan(wl.lengths[t0:t1], wl.sizes[lo:hi], 2)
        want = [0, 0]
        for p in pieces:
            want[p.rank] += p.tokens
        assert loads == want, j
        k += 1
        lo = hi
    assert k == len(A.flushes)


def test_reference_arm_under_torchrun():
    """bench.py --impl reference, 2 ranks: rank 0 prints one JSON line with impl=reference."""
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0",
           "--n-texts", "40000", "--ref-texts", "4"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "texts/s" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"


@pytest.mark.parametrize("gpus", [2, 4])
def test_bench_gpus_n_spawns_ranks(gpus):
    """`bench.py --gpus N` outside torchrun launches the N ranks itself (torch.distributed.run on
    127.0.0.1); --host-only runs each rank's host plan (Alg.1 + LPT through libsurge) over gloo and
    rank 0 reports every rank's share: together they cover the stream exactly, within one LPT piece
    of each other per SuperBatch."""
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    env.pop("WORLD_SIZE", None)
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(gpus), "--host-only",
           "--n-texts", "300000"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_ranks"] == gpus and d["backend"] == "gloo"
    assert sum(d["texts_per_rank"]) == d["n_texts"] == 300_000
    assert sum(d["tokens_per_rank"]) == d["n_tokens"]
    assert max(d["tokens_per_rank"]) - min(d["tokens_per_rank"]) <= d["superbatches"] * d["n_tokens"] / (8 * gpus)


def test_bench_rejects_gpus_world_mismatch():
    """Under a launcher, --gpus must equal the number of ranks (a SCALE run never silently measures
    fewer GPUs than it reports)."""
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="", WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--host-only"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode != 0 and "--gpus 2" in r.stderr


def test_bench_config_overrides():
    """--sigma / --b-min / --b-max reach the workload (config CLI, SURVEY §8(b) surge_config thresholds):
    the host plan runs at the requested skew and thresholds, and no SuperBatch sealed by the efficiency
    trigger exceeds B_max unless it is a single oversized partition (Alg.1)."""
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    env.pop("WORLD_SIZE", None)
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--host-only", "--n-texts", "200000",
           "--sigma", "2.5", "--b-min", "20000", "--b-max", "60000"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][0])
    assert (d["sigma"], d["b_min"], d["b_max"]) == (2.5, 20000, 60000)
    assert d["n_texts"] == 200_000 and sum(d["texts_per_rank"]) == 200_000
    bad = subprocess.run(cmd[:-4] + ["--b-min", "50000", "--b-max", "100"], capture_output=True, text=True,
                         timeout=300, env=env, cwd=ROOT)
    assert bad.returncode != 0 and "B_min <= B_max" in bad.stderr
