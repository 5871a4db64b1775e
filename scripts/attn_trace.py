#!/usr/bin/env python3
"""Phase breakdown of the persistent tcgen05 attention engine (diagnostic build).

    python -m paper_2505_09142_b200.build --variant=atrace -DELIS_ATTN_TRACE
    ELIS_LIB=libelis_atrace.so python scripts/attn_trace.py [n_requests]

One fp16 elis_op_attention_f16 launch over trace-shaped BGE-base requests (cfg2: 256); every
pipeline's %globaltimer stamps (TMA producer, MMA issuer, softmax warp 0) are summed per phase:
where a pipeline's time goes between the kernel's first and last stamp.
"""
from __future__ import annotations

import ctypes
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2505_09142_b200 import binding, inputs  # noqa: E402

PIPES, EVENTS = 512, 2048
# (role, start code, end code) -> phase name
PHASES = {
    (0, 1, 2): "producer: wait Q slot free",
    (0, 3, 4): "producer: wait K/V stage free",
    (1, 10, 11): "mma: wait Q loaded",
    (1, 12, 13): "mma: wait K loaded + S released",
    (1, 14, 15): "mma: wait P (softmax) + V",
    (2, 20, 21): "softmax: wait S",
    (2, 21, 26): "softmax: S loads (LDTM + wait)",
    (2, 21, 28): "softmax: block (S loads, max, exp2, wait PV_{g-1}, P)",
    (2, 28, 22): "softmax: arrive",
    (2, 21, 22): "softmax: inactive warp block",
    (2, 23, 24): "softmax: wait O (last PV)",
    (2, 24, 25): "softmax: epilogue stores",
    (2, 22, 20): "softmax: between blocks",
    (2, 25, 20): "softmax: next item start",
    (2, 22, 23): "softmax: to epilogue",
}


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    H, nh = 768, 12
    L = inputs.trace_lengths(n, seed=0)[0].astype(np.int32)
    T = int(L.sum())
    rng = np.random.default_rng(0)
    x = torch.from_numpy(rng.normal(0, 1, (3 * nh, T, 64)).astype(np.float32)).to(torch.float16).cuda()
    ctx = torch.empty(T, H, dtype=torch.float16, device="cuda")
    lt = torch.from_numpy(L).cuda()
    lib = binding.lib()
    fn = lib.elis_debug_attn_trace
    fn.restype = ctypes.c_int
    fn.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
    binding.op_attention(x, lt, H, nh, ctx, f16=True)
    fn(None, None, 1)
    binding.op_attention(x, lt, H, nh, ctx, f16=True)
    torch.cuda.synchronize()
    tr = np.zeros(PIPES * EVENTS, np.uint64)
    cnt = np.zeros(PIPES * 4, np.uint32)
    assert fn(tr.ctypes.data, cnt.ctypes.data, 0) == 0
    tr = tr.reshape(PIPES, 4, EVENTS // 4)
    cnt = cnt.reshape(PIPES, 4)
    t_all = [int(v >> 8) for p in range(PIPES) for r in range(3) for v in tr[p, r, :min(cnt[p, r], EVENTS // 4)]]
    t0, t1 = min(t_all), max(t_all)
    print(f"n={n} T={T}: kernel span {1e-3 * (t1 - t0):.1f} us over {int((cnt[:, 2] > 0).sum())} pipelines")
    tot = defaultdict(float)
    npipes = 0
    for p in range(PIPES):
        if cnt[p, 2] == 0:
            continue
        npipes += 1
        for role in range(3):
            ev = [(int(v >> 8), int(v & 0xFF)) for v in tr[p, role, :min(cnt[p, role], EVENTS // 4)]]
            for (ta, ca), (tb, cb) in zip(ev, ev[1:]):
                name = PHASES.get((role, ca, cb))
                if name:
                    tot[name] += tb - ta
    for name in sorted(tot, key=lambda k: -tot[k]):
        print(f"  {name:32s} {1e-3 * tot[name] / npipes:8.1f} us per pipeline")


if __name__ == "__main__":
    main()
