#!/usr/bin/env python3
"""Role-wait breakdown of the tcgen05 GEMM (diagnostic build).

    python -m paper_2505_09142_b200.build --variant=gtrace -DELIS_GEMM_TRACE
    ELIS_LIB=libelis_gtrace.so python scripts/gemm_trace.py [M]
For the four BGE-base GEMM shapes at M tokens (default: the cfg2 step, 43,296), one launch each
through elis_op_gemm / elis_op_gemm_ln; prints per-CTA means (in microseconds at the measured
SM clock) of the producer / MMA / epilogue waits recorded by clock64.
"""
from __future__ import annotations

import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2505_09142_b200 import binding  # noqa: E402

NAMES = ["prod wait(empty)", "mma wait(acc free)", "mma wait(smem full)", "mma span", "epi wait(acc full)",
         "epi pass1", "epi wait(stats)", "epi pass2", "epi span", "tiles"]


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    M = int(args[0]) if args else 43296
    H, F = 768, 3072
    dev = torch.device("cuda")
    lib = binding.lib()
    fn = lib.elis_debug_gemm_trace
    fn.restype = ctypes.c_int
    fn.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
    g = torch.Generator(device="cpu").manual_seed(0)

    def rnd(*shape, scale=0.05):
        return (torch.randn(*shape, generator=g) * scale).to(dev)

    hb = rnd(M, H).bfloat16()
    gg = rnd(M, F).bfloat16()
    shapes = {
        "qkv (bias, bf16 out)": lambda: binding.op_gemm(hb, rnd(3 * H, H).bfloat16(), rnd(3 * H).float(),
                                                         torch.empty(M, 3 * H, dtype=torch.bfloat16, device=dev), 0),
        "ffn1 (bias+GELU)": lambda: binding.op_gemm(hb, rnd(F, H).bfloat16(), rnd(F).float(),
                                                     torch.empty(M, F, dtype=torch.bfloat16, device=dev), 1),
        "out+LN (K=768)": lambda: binding.op_gemm_ln(hb, rnd(H, H).bfloat16(), rnd(H).float(), rnd(M, H).float(),
                                                    torch.ones(H, device=dev), torch.zeros(H, device=dev), 1e-12,
                                                    torch.empty(M, H, dtype=torch.bfloat16, device=dev)),
        "ffn2+LN (K=3072)": lambda: binding.op_gemm_ln(gg, rnd(H, F).bfloat16(), rnd(H).float(), rnd(M, H).float(),
                                                      torch.ones(H, device=dev), torch.zeros(H, device=dev), 1e-12,
                                                      torch.empty(M, H, dtype=torch.bfloat16, device=dev)),
    }
    if "--r16" in sys.argv:  # fp16 operands, fp16 residual stream (EPI_BIAS_RESID16_LN)
        hh, gh = hb.half(), gg.half()
        shapes = {
            "qkv fp16": lambda: binding.op_gemm(hh, rnd(3 * H, H).half(), rnd(3 * H).float(),
                                                torch.empty(M, 3 * H, dtype=torch.half, device=dev), 0),
            "out+LN16 (K=768)": lambda: binding.op_gemm_ln16(hh, rnd(H, H).half(), rnd(H).float(), rnd(M, H).half(),
                                                            torch.ones(H, device=dev), torch.zeros(H, device=dev),
                                                            1e-12),
            "ffn2+LN16 (K=3072)": lambda: binding.op_gemm_ln16(gh, rnd(H, F).half(), rnd(H).float(), rnd(M, H).half(),
                                                              torch.ones(H, device=dev), torch.zeros(H, device=dev),
                                                              1e-12),
        }
    if "--fp8" in sys.argv:  # E4M3 operands (kind::f8f6f4) on the same shapes
        def f8(*shape, scale=4.0):
            return (torch.randn(*shape, generator=g) * scale).to(torch.float8_e4m3fn).view(torch.uint8).to(dev)
        h8, g8 = f8(M, H), f8(M, F)
        cs = lambda n: torch.full((n,), 1e-3, device=dev)
        shapes = {
            "qkv fp8": lambda: binding.op_gemm_f8(h8, f8(3 * H, H), cs(3 * H), rnd(3 * H).float(),
                                                 torch.empty(M, 3 * H, dtype=torch.bfloat16, device=dev), 0),
            "ffn1 fp8 (GELU, e4m3 out)": lambda: binding.op_gemm_f8(h8, f8(F, H), cs(F), rnd(F).float(),
                                                                   torch.empty(M, F, dtype=torch.uint8, device=dev),
                                                                   1, 16.0),
            "ffn2+LN fp8": lambda: binding.op_gemm_ln_f8(g8, f8(H, F), cs(H), rnd(H).float(), rnd(M, H).float(),
                                                        torch.ones(H, device=dev), torch.zeros(H, device=dev),
                                                        1e-12, torch.empty(M, H, dtype=torch.uint8, device=dev), 8.0),
        }
    clk_ghz = None
    for name, call in shapes.items():
        call()
        torch.cuda.synchronize()
        assert fn(None, 0, 1) == 0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        call()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        buf = np.zeros(1024 * 16, np.int64)
        assert fn(buf.ctypes.data, buf.size, 0) == 0
        t = buf.reshape(1024, 16)
        used = t[:, 8] > 0
        t = t[used | (t[:, 3] > 0)]
        span = t[:, 8][t[:, 8] > 0].mean()
        if clk_ghz is None:
            clk_ghz = span / (ms * 1e6) * 1e3 / 1e3  # cycles per ns ~ GHz (epilogue span ~ launch)
        mma = t[t[:, 3] > 0]
        epi = t[t[:, 8] > 0]
        row = {
            NAMES[0]: t[:, 0].mean(), NAMES[1]: mma[:, 1].mean(), NAMES[2]: mma[:, 2].mean(),
            NAMES[3]: mma[:, 3].mean(), NAMES[4]: epi[:, 4].mean(), NAMES[5]: epi[:, 5].mean(),
            NAMES[6]: epi[:, 6].mean(), NAMES[7]: epi[:, 7].mean(), NAMES[8]: epi[:, 8].mean(),
        }
        print(f"{name}: launch {ms * 1e3:.1f} us, CTAs {len(t)}, tiles/MMA-CTA {mma[:, 9].mean():.2f}")
        print("   " + "  ".join(f"{k} {v / (clk_ghz * 1e3):.1f}" for k, v in row.items()) + "  (us)")


if __name__ == "__main__":
    main()
