"""Theorem 1 cost model (paper_2605_01060_b200/costmodel.py) against the paper's own numbers."""

import numpy as np
import pytest

from paper_2605_01060_b200 import costmodel as cm



def test_paper_worked_example_minilm():
    """c_ipc 0.087 s, c_enc 0.149 ms, G=4, N=10M, P=4000 -> alpha 0.93, predicted speedup 1.89
    at F=100 (measured 1.92, error < 2%)."""
    a = cm.alpha(4000, 10_000_000, 0.087, 1.49e-4, g=4)
    assert a == pytest.approx(0.934, abs=2e-3)
    s = cm.speedup(a, 100, 4000)
    assert s == pytest.approx(1.89, abs=0.01)
    assert abs(s - 1.92) / 1.92 < 0.02


def test_paper_bge_base_example():
    """bge-base on 2xL4, c_ipc 0.081 s, c_enc 0.215 ms -> alpha 0.301 for G=2 (SURVEY App. A
    item 6: the printed alpha=0.603 needs G=4), predicted 1.29x at F=100 vs measured 1.29x."""
    a = cm.alpha(4000, 10_000_000, 0.081, 2.15e-4, g=2)
    assert a == pytest.approx(0.301, abs=2e-3)
    assert cm.speedup(a, 100, 4000) == pytest.approx(1.29, abs=0.01)


def test_limits():
    # compute-dominated: speedup -> 1; IPC-dominated: speedup -> P / F
    assert cm.speedup(1e-9, 100, 4000) == pytest.approx(1.0)
    assert cm.speedup(1e9, 100, 4000) == pytest.approx(40.0, rel=1e-6)
    assert cm.partition_time(0, 0.5, 1e-3) == 0.5


def test_fit_recovers_exact_parameters():
    n, c_call, c_enc = 10_000_000, 3.1e-4, 3.6e-7
    f = np.array([4000, 1000, 200, 100, 50, 20])
    t = f * c_call + n * c_enc
    r = cm.fit(f, t, n)
    assert r.c_call == pytest.approx(c_call, rel=1e-9)
    assert r.c_enc == pytest.approx(c_enc, rel=1e-9)
    assert r.residual_rms < 1e-12
