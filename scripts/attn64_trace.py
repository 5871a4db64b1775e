#!/usr/bin/env python3
"""Phase breakdown of the 64-key-block tcgen05 attention engine (diagnostic build).

    python -m paper_2505_09142_b200.build --variant=atrace -DELIS_ATTN_TRACE
    ELIS_LIB=libelis_atrace.so python scripts/attn64_trace.py [n_requests]

One fp16 elis_op_attention_f16 launch over trace-shaped BGE-base requests (256 = cfg2, 1311 = the
cfg5 due set); thread 0 of every CTA stamped %globaltimer at its phase boundaries: the per-CTA
time in each phase, averaged, and the kernel span.
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

CTAS, EV = 1 << 16, 48
PHASES = {(1, 2): "setup (barriers, TMEM alloc)", (2, 3): "wait Q / K_0 / V_0 loads", (3, 4): "issue S_0",
          (2, 4): "setup -> first wait (non-issuer view)", (4, 5): "wait S_j", (5, 6): "softmax (thread 0's warp)",
          (6, 7): "barrier (all warps' P)", (7, 8): "wait K/V_j loaded (issuer)", (8, 4): "issue PV_j + S_j+1",
          (7, 4): "issue PV_j + S_j+1", (4, 9): "-", (8, 9): "issue last PV", (9, 10): "wait last PV",
          (10, 11): "epilogue"}


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    H, nh = 768, 12
    L = inputs.trace_lengths(n, seed=0)[0].astype(np.int32)
    T = int(L.sum())
    rng = np.random.default_rng(0)
    x = torch.from_numpy(rng.normal(0, 1, (3 * nh, T, 64)).astype(np.float32)).to(torch.float16).cuda()
    ctx = torch.empty(T, H, dtype=torch.float16, device="cuda")
    lt = torch.from_numpy(L).cuda()
    fn = binding.lib().elis_debug_attn64_trace
    fn.restype = ctypes.c_int
    fn.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
    binding.op_attention(x, lt, H, nh, ctx, f16=True)
    binding.op_attention(x, lt, H, nh, ctx, f16=True)
    torch.cuda.synchronize()
    tr = np.zeros(CTAS * EV, np.uint64)
    cnt = np.zeros(CTAS, np.uint32)
    assert fn(tr.ctypes.data, cnt.ctypes.data) == 0
    tr = tr.reshape(CTAS, EV)
    ctas = int((cnt > 0).sum())
    t0 = min(int(tr[c, 0] >> 8) for c in range(CTAS) if cnt[c])
    t1 = max(int(tr[c, min(cnt[c], EV) - 1] >> 8) for c in range(CTAS) if cnt[c])
    tot = defaultdict(float)
    life = 0.0
    blocks = 0
    for c in range(CTAS):
        k = min(int(cnt[c]), EV)
        if k < 2:
            continue
        ev = [(int(v >> 8), int(v & 0xFF)) for v in tr[c, :k]]
        life += ev[-1][0] - ev[0][0]
        blocks += sum(1 for _, code in ev if code == 5)
        for (ta, ca), (tb, cb) in zip(ev, ev[1:]):
            tot[PHASES.get((ca, cb), f"{ca}->{cb}")] += tb - ta
    print(f"n={n} T={T}: kernel span {1e-3 * (t1 - t0):.1f} us, {ctas} CTAs, {blocks} 64-key blocks, "
          f"mean CTA lifetime {1e-3 * life / ctas:.2f} us")
    for name in sorted(tot, key=lambda k: -tot[k]):
        print(f"  {name:40s} {1e-3 * tot[name] / ctas:8.3f} us per CTA  ({1e-3 * tot[name] / max(blocks, 1):.3f} us per block)")


if __name__ == "__main__":
    main()
