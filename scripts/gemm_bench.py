#!/usr/bin/env python3
"""Microbenchmark: libelis tcgen05 GEMM (per epilogue) vs cuBLAS (torch.matmul, bf16) on the
encoder's GEMM shapes.  cuBLAS is a yardstick only -- it is never on the hot path.

    python scripts/gemm_bench.py [T]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_09142_b200 import binding  # noqa: E402


def timeit(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e3  # us


def main():
    T = int(sys.argv[1]) if len(sys.argv) > 1 else 43296
    binding.lib()
    shapes = [("qkv", 2304, 768, 0), ("out+ln", 768, 768, 3), ("ffn1", 3072, 768, 1), ("ffn2+ln", 768, 3072, 3),
              ("out+res", 768, 768, 2)]
    print(f"T={T}")
    for name, N, K, epi in shapes:
        A = torch.randn(T, K, device="cuda").to(torch.bfloat16)
        W = (torch.randn(N, K, device="cuda") * 0.03).to(torch.bfloat16)
        b = torch.randn(N, device="cuda") * 0.1
        flops = 2.0 * T * N * K
        if epi == 3:
            h = torch.randn(T, N, device="cuda")
            hb = torch.empty(T, N, device="cuda", dtype=torch.bfloat16)
            g = torch.ones(N, device="cuda")
            be = torch.zeros(N, device="cuda")
            fn = lambda: binding.op_gemm_ln(A, W, b, h, g, be, 1e-12, hb)
        elif epi == 2:
            r = torch.randn(T, N, device="cuda")
            o = torch.empty(T, N, device="cuda")
            fn = lambda: binding.op_gemm(A, W, b, o, 2, residual=r)
        else:
            o = torch.empty(T, N, device="cuda", dtype=torch.bfloat16)
            fn = lambda: binding.op_gemm(A, W, b, o, epi)
        us = timeit(fn)
        cub = timeit(lambda: torch.matmul(A, W.t()))
        print(f"{name:8s} N={N:5d} K={K:5d}  elis {us:8.1f} us {flops / us / 1e6:7.1f} TF/s   "
              f"cuBLAS(matmul only) {cub:8.1f} us {flops / cub / 1e6:7.1f} TF/s")


if __name__ == "__main__":
    main()
