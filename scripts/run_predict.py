#!/usr/bin/env python3
"""Run elis_predict_remaining `--iters` times on one workload (for ncu captures / quick timing).

    python scripts/run_predict.py --config base --n 256 --lengths trace --iters 3
Each predict is 1 + 12 x 5 + 10 launches for BGE-base (meta, embed_ln, per layer qkv / attention /
out / ffn1 / ffn2, pool, 8 head fc); use `ncu -k regex:<kernel> -s <skip> -c <count>`.
"""
from __future__ import annotations

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2505_09142_b200 import binding, inputs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="base")
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--lengths", default="trace")
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--time", action="store_true", help="print per-kernel ms from the library profiler")
    ap.add_argument("--precision", default="bf16", choices=["bf16", "fp8", "fp16"])
    ap.add_argument("--pooling", default="mean", choices=["mean", "cls"])
    ap.add_argument("--cls-last-layer", action="store_true", help="CLS pooling: last layer on CLS rows only")
    ap.add_argument("--residual16", action="store_true", help="fp16 residual stream (with --precision fp16)")
    a = ap.parse_args()
    cfg = inputs.CONFIGS[a.config]
    if a.pooling == "cls":
        cfg = inputs.EncoderConfig(**{**cfg.to_dict(), "pooling": inputs.POOL_CLS})
    if a.lengths == "trace":
        L = inputs.trace_lengths(a.n, seed=0)[0]
    elif a.lengths == "uniform":
        L = inputs.uniform_lengths(a.n, seed=0)
    else:
        L = np.full(a.n, int(a.lengths.split(":")[1]), np.int32)
    tok = inputs.make_tokens(L, seed=0)
    T = int(L.sum())
    p = binding.Predictor(cfg, inputs.flatten_weights(cfg, inputs.make_weights(cfg)), max_tokens=T, max_requests=a.n,
                         precision=a.precision, cls_last_layer=a.cls_last_layer, residual16=a.residual16)
    dev = torch.device("cuda:0")
    t_tok = torch.from_numpy(tok).to(dev)
    t_len = torch.from_numpy(L.astype(np.int32)).to(dev)
    out = torch.empty(a.n, dtype=torch.float32, device=dev)
    if a.time:
        p.profile_enable(True)
    for _ in range(a.iters):
        p.predict_remaining(t_tok, t_len, T, out)
    torch.cuda.synchronize()
    binding.check(p.sync_status(), "predict")
    if a.time:
        prof = p.profile_read()
        print({k: round(ms / a.iters, 4) for k, (ms, _) in prof.items()})
    print(f"T={T} pred[0:4]={out[:4].tolist()}")


if __name__ == "__main__":
    main()
