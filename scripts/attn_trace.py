#!/usr/bin/env python3
"""Phase breakdown of the tcgen05 attention CTAs (diagnostic build).

    python -m paper_2505_09142_b200.build --variant=trace -DELIS_ATTN_TRACE
    ELIS_LIB=libelis_trace.so python scripts/attn_trace.py
Runs one BGE-base predict on the cfg2 workload and reads the %globaltimer stamps thread 0 of each
CTA wrote in the last attention launch: start, after setup, S_0 ready, P_0 in TMEM, O_0 ready,
block-0 fold done, end.
"""
from __future__ import annotations

import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2505_09142_b200 import binding, inputs  # noqa: E402


def main():
    cfg = inputs.CONFIGS["base"]
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    L = inputs.trace_lengths(n, seed=0)[0]
    tok = inputs.make_tokens(L, seed=0)
    T = int(L.sum())
    p = binding.Predictor(cfg, inputs.flatten_weights(cfg, inputs.make_weights(cfg)), T, n)
    dev = torch.device("cuda:0")
    t_tok, t_len = torch.from_numpy(tok).to(dev), torch.from_numpy(L.astype(np.int32)).to(dev)
    out = torch.empty(n, dtype=torch.float32, device=dev)
    lib = binding.lib()
    fn = lib.elis_debug_attn_trace
    fn.restype = ctypes.c_int
    fn.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
    for _ in range(2):
        p.predict_remaining(t_tok, t_len, T, out)
    torch.cuda.synchronize()
    assert fn(None, 0, 1) == 0
    p.predict_remaining(t_tok, t_len, T, out)
    torch.cuda.synchronize()
    cap = 1 << 16
    buf = np.zeros(cap * 8, np.uint64)
    assert fn(buf.ctypes.data, cap * 8, 0) == 0
    t = buf.reshape(cap, 8)
    t = t[t[:, 0] != 0].astype(np.int64)
    t0 = t[:, 0].min()
    st = t[:, :7] - t0
    nkb = t[:, 7] & 0xFF
    Ls = (t[:, 7] >> 8) & 0xFFFFFF
    sm = t[:, 7] >> 32
    span = st[:, 6].max()
    print(f"CTAs {len(t)}  launch span {span / 1e3:.1f} us  SMs {len(np.unique(sm))}")
    names = ["setup", "S0 wait", "softmax0", "PV0 wait", "fold0", "rest"]
    d = np.diff(st, axis=1)
    life = st[:, 6] - st[:, 0]
    print(f"lifetime us: mean {life.mean() / 1e3:.2f} p50 {np.median(life) / 1e3:.2f} p90 {np.percentile(life, 90) / 1e3:.2f}")
    for k in sorted(np.unique(nkb)):
        m = nkb == k
        print(f"nkb={k}: {m.sum():5d} CTAs  life {life[m].mean() / 1e3:6.2f} us  " +
              "  ".join(f"{nm} {d[m, i].mean() / 1e3:5.2f}" for i, nm in enumerate(names)))
    # concurrency: CTAs resident per SM over time
    ev = np.concatenate([np.stack([st[:, 0], np.ones(len(st))], 1), np.stack([st[:, 6], -np.ones(len(st))], 1)])
    ev = ev[np.argsort(ev[:, 0], kind="stable")]
    c = np.cumsum(ev[:, 1])
    dt = np.diff(ev[:, 0], append=ev[-1, 0])
    print(f"mean resident CTAs (all SMs) {np.sum(c * dt) / span:.1f}  (148 x 4 = 592 slots)")
    # startup gaps: first start per SM, last end per SM
    first = np.array([st[sm == s, 0].min() for s in np.unique(sm)])
    last = np.array([st[sm == s, 6].max() for s in np.unique(sm)])
    print(f"per-SM first start us: max {first.max() / 1e3:.2f}; last end us: min {last.min() / 1e3:.2f} max {last.max() / 1e3:.2f}")


if __name__ == "__main__":
    main()
