"""Parity at BASELINE.json's full size (C2: 10M texts, P = 4,000, sigma = 1.72, MiniLM-L6 class), in the
launch configuration bench.py times (device-resident SuperBatches through surge_encode_superbatch, and
the streaming ABI from host memory as bench.py's e2e):
  * integer parity: Alg. 1 flush decisions (membership, order, reasons) == the oracle's, bit-exact;
  * every one of the 10M rows: finite and unit-norm (|norm - 1| <= 1e-5);
  * the SURVEY §8(c) 16,384-row sample (first 4,096 rows, first and last row of every partition, seeded
    uniform rows) vs the fp64 oracle, one text at a time over all host cores, under the north-star gate;
  * the streaming path returns the same rows bit for bit (sampled partitions) with the right counts.
"""
import numpy as np
import pytest
import torch

from oracle import aggregator as oagg
from oracle import pool as opool
from synth.configs import ENCODERS, WORKLOADS
from synth.weights import make_weights, pack_blob
from synth.workload import make_workload, parity_sample

pytestmark = pytest.mark.gpu

COS_MIN, ABS_MAX, NORM_TOL = 0.999, 1e-2, 1e-5
SAMPLE_ROWS = 16_384


def c2_parity_sample(wl, seed: int = 0):
    """SURVEY.md §8(c) "C2: a 16,384-row sample = the first 4,096 rows in stream order + the first and
    last row of every partition (<= 8,000) + the rest uniformly random (seeded)"."""
    return parity_sample(wl, SAMPLE_ROWS, 4096, seed)


@pytest.fixture(scope="module")
def setup():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2605_01060_b200 import native as N
    ecfg, wcfg = ENCODERS["minilm"], WORKLOADS["minilm"]
    w = make_weights(ecfg, seed=1234)
    wl = make_workload(wcfg, ecfg.vocab_size, ecfg.max_position, seed=0)
    blob = torch.from_numpy(pack_blob(ecfg, w).view(np.uint8)).cuda()
    return N, ecfg, wcfg, w, wl, blob


def test_full_c2_device_path_and_streaming(setup):
    N, ecfg, wcfg, w, wl, blob = setup
    assert wl.n_texts == 10_000_000 and len(wl.sizes) == 4000
    h = N.surge_create(N.make_config(ecfg, wcfg.b_min, wcfg.b_max, weights_on_device=1), blob,
                       n_weights=blob.numel() // 2)
    try:
        sizes = wl.sizes.astype(np.int64)
        sbs, peak = N.surge_aggregate(sizes, wcfg.b_min, wcfg.b_max)
        A = oagg.run_aggregator([int(k) for k in wl.keys], wl.sizes, wcfg.b_min, wcfg.b_max)
        idx = {int(k): i for i, k in enumerate(wl.keys)}
        assert [[idx[int(k)] for k in f.keys] for f in A.flushes] == [list(range(a, b)) for a, b, _ in sbs]
        assert [r for _, _, r in sbs] == [f.reason for f in A.flushes]
        assert peak == A.peak_buffered <= wcfg.b_min - 1 + A.nmax_seen
        d_ids = torch.from_numpy(wl.ids).cuda()
        d_len = torch.from_numpy(wl.lengths).cuda()
        out = torch.empty(wl.n_texts, ecfg.hidden, dtype=torch.float32, device="cuda")
        st = torch.cuda.Stream()
        for a, b, _ in sbs:
            t0, t1, k0 = int(wl.text_off[a]), int(wl.text_off[b]), int(wl.tok_off[a])
            N.surge_encode_superbatch(h, d_ids.data_ptr() + 4 * k0, d_len.data_ptr() + 4 * t0, wl.lengths[t0:t1],
                                      sizes[a:b], out.data_ptr() + 4 * t0 * ecfg.hidden, st)
        torch.cuda.synchronize()
        assert bool(torch.isfinite(out).all())
        norms = out.norm(dim=1)
        assert float((norms - 1).abs().max()) <= NORM_TOL
        # the SURVEY §8(c) C2 parity sample vs the fp64 oracle (all host cores)
        rows = c2_parity_sample(wl)
        assert len(rows) == SAMPLE_ROWS
        ends = np.cumsum(wl.lengths, dtype=np.int64)
        starts = ends - wl.lengths
        ref, secs, procs = opool.encode_rows(ecfg, w, wl.ids, starts, ends, rows)
        print(f"oracle: {len(rows)} rows on {procs} processes in {secs:.1f}s")
        got = out[torch.tensor(rows, device="cuda")].cpu().numpy().astype(np.float64)
        cos = (got * ref).sum(1) / (np.linalg.norm(got, axis=1) * np.linalg.norm(ref, axis=1))
        assert cos.min() >= COS_MIN, cos.min()
        assert np.abs(got - ref).max() <= ABS_MAX
        rng = np.random.default_rng(0)
        parts = rng.choice(len(wl.sizes), size=8, replace=False)
        rows = sorted(set(rows[:16]) | {int(wl.text_off[k]) for k in parts} | {int(wl.text_off[k + 1]) - 1 for k in parts})
        dev_rows = {i: out[i].cpu().numpy() for i in rows}
        del out
        torch.cuda.empty_cache()
        # the streaming ABI (bench.py e2e) on the same stream: counts, and the sampled partitions' rows
        want = {int(wl.keys[k]): k for k in parts}
        seen, n_rows = {}, 0

        def drain(timeout):
            nonlocal n_rows
            for r in N.surge_poll_flushed(h, 4096, timeout):
                n_rows += r.n_rows
                k = want.get(int(r.partition_id))
                if k is not None:
                    arr = N.flushed_array(r)
                    for j in (0, r.n_rows - 1):
                        g = int(wl.text_off[k]) + int(r.row_begin) + j
                        if g in dev_rows:
                            seen[g] = arr[j].copy()
                N.surge_release(h, r)

        for k in range(len(wl.sizes)):
            key, ids, lens = wl.partition(k)
            N.surge_submit_partition(h, key, ids, lens)
            drain(0)
        N.surge_finish(h)
        while N.surge_pending(h) > 0:
            drain(20)
        drain(0)
        assert n_rows == wl.n_texts
        stats = N.surge_get_stats(h)
        assert stats["superbatches"] == len(A.flushes)
        assert len(seen) >= 8
        for g, v in seen.items():
            assert np.array_equal(v, dev_rows[g])
    finally:
        N.surge_destroy(h)


def test_sigma25_safety_superbatch(setup):
    """C2 at sigma = 2.5 (tab:sigma-sweep P:764-785): the Safety branch fires once and carries a
    567,878-text SuperBatch (reading R2/R3: literal Alg. 1, never split).  Integer parity of the whole
    aggregation vs the oracle; that SuperBatch encoded on the device in bench.py's launch configuration:
    every row unit-norm, a 4,096-row sample vs the fp64 oracle (first rows, first/last row of every
    member, seeded uniform rows); the streaming ABI reports the same F, Safety count and Lemma-bounded
    peak, and returns the sampled rows bit for bit."""
    N, ecfg, _, w, _, blob = setup
    wcfg = WORKLOADS["minilm_s2.5"]
    wl = make_workload(wcfg, ecfg.vocab_size, ecfg.max_position, seed=0)
    sizes = wl.sizes.astype(np.int64)
    A = oagg.run_aggregator([int(k) for k in wl.keys], wl.sizes, wcfg.b_min, wcfg.b_max)
    sbs, peak = N.surge_aggregate(sizes, wcfg.b_min, wcfg.b_max)
    assert [r for _, _, r in sbs] == [f.reason for f in A.flushes]
    safety = [j for j, f in enumerate(A.flushes) if f.reason == oagg.SAFETY]
    assert len(safety) == 1 and A.flushes[safety[0]].total == 567_878
    assert peak == A.peak_buffered == 567_878 <= wcfg.b_min - 1 + A.nmax_seen
    a, b, _ = sbs[safety[0]]
    t0, t1, k0, k1 = int(wl.text_off[a]), int(wl.text_off[b]), int(wl.tok_off[a]), int(wl.tok_off[b])
    h = N.surge_create(N.make_config(ecfg, wcfg.b_min, wcfg.b_max, weights_on_device=1), blob,
                       n_weights=blob.numel() // 2)
    try:
        d_ids = torch.from_numpy(wl.ids[k0:k1]).cuda()
        d_len = torch.from_numpy(wl.lengths[t0:t1]).cuda()
        out = torch.empty(t1 - t0, ecfg.hidden, dtype=torch.float32, device="cuda")
        N.surge_encode_superbatch(h, d_ids, d_len, wl.lengths[t0:t1], sizes[a:b], out, torch.cuda.Stream())
        torch.cuda.synchronize()
        assert float((out.norm(dim=1) - 1).abs().max()) <= NORM_TOL
        rows = set(range(1024))
        for k in range(a, b):
            rows |= {int(wl.text_off[k]) - t0, int(wl.text_off[k + 1]) - 1 - t0}
        rng = np.random.default_rng(25)
        while len(rows) < 4096:
            rows |= set(rng.integers(0, t1 - t0, size=4096 - len(rows)).tolist())
        rows = sorted(rows)
        ends = np.cumsum(wl.lengths, dtype=np.int64)
        starts = ends - wl.lengths
        ref, _, _ = opool.encode_rows(ecfg, w, wl.ids, starts, ends, [t0 + r for r in rows])
        got = out[torch.tensor(rows, device="cuda")].cpu().numpy().astype(np.float64)
        cos = (got * ref).sum(1) / (np.linalg.norm(got, axis=1) * np.linalg.norm(ref, axis=1))
        assert cos.min() >= COS_MIN, cos.min()
        assert np.abs(got - ref).max() <= ABS_MAX
        dev = {t0 + r: got[i] for i, r in enumerate(rows[:64])}
        del out
        # streaming ABI over the whole sigma = 2.5 stream
        key_to_k = {int(wl.keys[k]): k for k in range(a, b)}
        seen, n_rows = {}, 0

        def drain(timeout):
            nonlocal n_rows
            for r in N.surge_poll_flushed(h, 4096, timeout):
                n_rows += r.n_rows
                k = key_to_k.get(int(r.partition_id))
                if k is not None:
                    arr, base = N.flushed_array(r), int(wl.text_off[k]) + int(r.row_begin)
                    for g in dev:
                        if base <= g < base + r.n_rows:
                            seen[g] = arr[g - base].astype(np.float64)
                N.surge_release(h, r)

        for k in range(len(wl.sizes)):
            key, ids, lens = wl.partition(k)
            N.surge_submit_partition(h, key, ids, lens)
            drain(0)
        N.surge_finish(h)
        while N.surge_pending(h) > 0:
            drain(20)
        drain(0)
        st = N.surge_get_stats(h)
        assert n_rows == wl.n_texts
        assert st["superbatches"] == len(A.flushes) and st["safety_flushes"] == 1
        assert st["peak_buffered_texts"] == 567_878
        assert len(seen) == len(dev)
        for g, v in seen.items():
            assert np.array_equal(v, dev[g])
    finally:
        N.surge_destroy(h)
