#!/usr/bin/env python
"""Isolated timing of the encoder GEMM shapes through surge_op_gemm (tuning aid, GPU only).

    python scripts/gemm_bench.py [M]
"""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_01060_b200 import native as N  # noqa: E402


def main():
    M = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
    dev = torch.device("cuda")
    shapes = [("qkv", 1152, 384, 0), ("out_ln", 384, 384, 2), ("ffn1_gelu", 1536, 384, 1), ("ffn1_bias", 1536, 384, 0),
              ("ffn2_ln", 384, 1536, 2)]
    for name, Nn, K, epi in shapes:
        A = (torch.randn(M, K, device=dev) * 0.5).to(torch.bfloat16).view(torch.int16)
        B = (torch.randn(Nn, K, device=dev) / math.sqrt(K)).to(torch.bfloat16).view(torch.int16)
        bias = torch.randn(Nn, device=dev) * 0.1
        res = torch.randn(M, Nn, device=dev).to(torch.bfloat16).view(torch.int16)
        g, b = torch.ones(Nn, device=dev), torch.zeros(Nn, device=dev)
        C = torch.empty(M, Nn, dtype=torch.int16, device=dev)
        flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        for _ in range(3):
            N.surge_op_gemm(A, B, bias, res, g, b, C, M, Nn, K, epi)
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            N.surge_op_gemm(A, B, bias, res, g, b, C, M, Nn, K, epi)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = sorted(ts)[len(ts) // 2]
        print(f"{name:10s} M={M} N={Nn} K={K}: {ms * 1e3:8.1f} us  {2 * M * Nn * K / ms / 1e9:7.1f} TFLOP/s", flush=True)


if __name__ == "__main__":
    main()
