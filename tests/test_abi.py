"""CPU checks of the C ABI: libsurge.so loads, exports every entry point include/surge.h declares,
the host-only LPT plan equals the oracle's bit-exactly, and without a GPU surge_create fails
loudly (no CPU fallback)."""
import os
import re

import numpy as np
import pytest
import torch

from oracle import aggregator as oagg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "surge.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(surge_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2605_01060_b200 import native as N
    declared = header_functions()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(N.lib, name), name
    assert set(declared) == set(N.EXPORTED)
    assert "sm_100a" in N.surge_version()


def test_kernels_are_tcgen05_tma():
    """The built library carries tcgen05 MMA, TMEM loads and TMA loads for sm_100a."""
    import shutil
    import subprocess
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    from paper_2605_01060_b200 import native as N
    sass = subprocess.run([tool, "-sass", N.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass and "UTMALDG" in sass and "LDTM" in sass
    assert "sm_100a" in subprocess.run([tool, "-lelf", N.LIB_PATH], capture_output=True, text=True).stdout


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_create_fails_loudly_without_gpu():
    from paper_2605_01060_b200 import native as N
    from synth.configs import ENCODERS
    from synth.weights import make_weights, pack_blob
    e = ENCODERS["toy"]
    blob = pack_blob(e, make_weights(e))
    with pytest.raises(N.SurgeError) as ei:
        N.surge_create(N.make_config(e, 64, 320), blob)
    assert ei.value.status == N.SURGE_E_CUDA


def test_create_rejects_bad_config():
    from paper_2605_01060_b200 import native as N
    from synth.configs import ENCODERS
    from synth.weights import make_weights, pack_blob
    e = ENCODERS["toy"]
    blob = pack_blob(e, make_weights(e))
    with pytest.raises(N.SurgeError) as ei:
        N.surge_create(N.make_config(e, 100, 100), blob)        # b_max must exceed b_min
    assert ei.value.status == N.SURGE_E_INVALID_ARG
    with pytest.raises(N.SurgeError) as ei:
        N.surge_create(N.make_config(e, 64, 320), blob[:-1])    # wrong blob size
    assert ei.value.status == N.SURGE_E_INVALID_ARG


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_native_lpt_equals_oracle(world):
    from paper_2605_01060_b200 import native as N
    rng = np.random.default_rng(100 + world)
    for _ in range(20):
        sizes = rng.integers(1, 300, size=int(rng.integers(1, 50)))
        lengths = rng.integers(1, 129, size=int(sizes.sum())).astype(np.int32)
        got = N.surge_lpt_plan(lengths, sizes, world)
        pieces, _ = oagg.lpt_plan(lengths, list(sizes), world)
        assert list(got["first_row"]) == [p.first_row for p in pieces]
        assert list(got["n_rows"]) == [p.n_rows for p in pieces]
        assert list(got["member"]) == [p.member for p in pieces]
        assert list(got["tokens"]) == [p.tokens for p in pieces]
        assert list(got["rank"]) == [p.rank for p in pieces]


def test_native_aggregate_equals_oracle():
    """The library's Alg.1 decisions (surge_aggregate, same code as the streaming path) vs the oracle."""
    from paper_2605_01060_b200 import native as N
    from synth.configs import WORKLOADS
    from synth.workload import partition_sizes
    rng = np.random.default_rng(9)
    cases = []
    for _ in range(200):
        P = int(rng.integers(1, 300))
        sizes = np.maximum(0, rng.lognormal(5, 1.7, size=P).astype(np.int64))
        b_min = int(rng.integers(1, 3000))
        cases.append((sizes, b_min, b_min * int(rng.integers(2, 6))))
    w = WORKLOADS["minilm"]
    cases.append((partition_sizes(w, np.random.Generator(np.random.PCG64(0))), w.b_min, w.b_max))
    for sizes, b_min, b_max in cases:
        sbs, peak = N.surge_aggregate(sizes, b_min, b_max)
        A = oagg.run_aggregator(range(len(sizes)), sizes, b_min, b_max)
        assert peak == A.peak_buffered
        assert [r for _, _, r in sbs] == [s.reason for s in A.flushes]
        got = [[k for k in range(a, b) if sizes[k] > 0] for a, b, _ in sbs]
        assert got == [list(s.keys) for s in A.flushes]


def test_nccl_unique_id_without_gpu():
    """K11 plumbing: libsurge resolves NCCL at run time (dlopen) and hands out the 128-byte unique id
    every rank of surge_create_replicated needs; the id is fresh per call."""
    from paper_2605_01060_b200 import native as N
    a, b = N.surge_nccl_unique_id(), N.surge_nccl_unique_id()
    assert len(a) == len(b) == 128 and a != b


@pytest.mark.parametrize("policy", ["label", "split", "preflush"])
def test_native_aggregate_ex_equals_oracle(policy):
    """surge_aggregate_ex (the aggregator the streaming path runs) == the oracle's Alg.1 under every
    B_max reading: SuperBatch reasons, members (partition, row0, rows) and the peak, bit-exact."""
    from oracle import aggregator as oagg
    from paper_2605_01060_b200 import native as N
    rng = np.random.default_rng(11)
    for trial in range(60):
        b_min = int(rng.integers(5, 80))
        b_max = b_min + int(rng.integers(1, 200))
        sizes = rng.integers(0, 5 * b_max, size=int(rng.integers(1, 60)))
        if trial % 2:
            sizes = np.sort(sizes)
        got, peak = N.surge_aggregate_ex(sizes, b_min, b_max, N.BMAX_POLICIES[policy])
        A = oagg.run_aggregator(range(len(sizes)), sizes, b_min, b_max, policy)
        want = [(sb.reason, list(zip(sb.refs, sb.row0, sb.sizes))) for sb in A.flushes]
        assert got == want
        assert peak == A.peak_buffered
    from synth.configs import WORKLOADS, ENCODERS, scaled
    from synth.workload import make_workload
    wl = make_workload(scaled(WORKLOADS["minilm_s2.5"], n_texts=2_000_000, n_partitions=800), 30522, 512, seed=1)
    got, peak = N.surge_aggregate_ex(wl.sizes, 20_000, 100_000, N.BMAX_POLICIES[policy])
    A = oagg.run_aggregator(range(len(wl.sizes)), wl.sizes, 20_000, 100_000, policy)
    assert got == [(sb.reason, list(zip(sb.refs, sb.row0, sb.sizes))) for sb in A.flushes] and peak == A.peak_buffered
