"""Time the exact-fp32 head FC (elis_op_fc_f32) at the head's shapes; ELIS_FC_SPLIT_MAX=1 forces
no split-K.  python scripts/fc_bench.py"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_09142_b200 import binding  # noqa: E402

res = {"split_max": os.environ.get("ELIS_FC_SPLIT_MAX", "default")}
for n, N, K in [(256, 1024, 768), (256, 1024, 1024), (16, 1024, 1024), (1311, 1024, 1024), (4096, 1024, 1024)]:
    X = torch.randn(n, K, device="cuda")
    W = torch.randn(N, K, device="cuda") * 0.03
    b = torch.randn(N, device="cuda")
    Y = torch.empty(n, N, device="cuda")
    for _ in range(5):
        binding.op_fc_f32(X, W, b, Y, 1)
    torch.cuda.synchronize()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(50):
        binding.op_fc_f32(X, W, b, Y, 1)
    e.record()
    torch.cuda.synchronize()
    us = a.elapsed_time(e) / 50 * 1e3
    res[f"{n}x{N}x{K}_us"] = round(us, 2)
    res[f"{n}x{N}x{K}_tflops"] = round(2 * n * N * K / us / 1e6, 2)
print(json.dumps(res))
