#!/usr/bin/env python3
"""Run elis_predict_remaining `--iters` times on one workload (for ncu captures / quick timing).

    python scripts/run_predict.py --config base --n 256 --lengths trace --iters 3
    python scripts/run_predict.py --workload cfg5 --iters 2   # bench.py's default step: due window 0 of the
                                                              # 65,536-slot table + the select over the table
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
    ap.add_argument("--precision", default="auto", choices=["auto", "bf16", "fp8", "fp16"])
    ap.add_argument("--workload", default=None, choices=["cfg5"], help="cfg5: bench.py's default step (window 0)")
    ap.add_argument("--cap", type=int, default=256)
    ap.add_argument("--pooling", default="mean", choices=["mean", "cls"])
    ap.add_argument("--cls-last-layer", action="store_true", help="CLS pooling: last layer on CLS rows only")
    ap.add_argument("--dump", default=None, help="save predictions + final hidden states (.npz) for bitwise A/B")
    ap.add_argument("--residual", default=None, choices=["fp16", "fp32"], help="residual stream (default: the library's)")
    a = ap.parse_args()
    cfg = inputs.CONFIGS[a.config]
    if a.pooling == "cls":
        cfg = inputs.EncoderConfig(**{**cfg.to_dict(), "pooling": inputs.POOL_CLS})
    slots = gen = None
    if a.workload == "cfg5":
        import bench
        ba = bench.parse([])
        Lt, gen, tok_t, offs = bench.table_population(ba)
        slots = bench.due_windows(ba.inflight, ba.due)[0]
        L = Lt[slots]
        tok = np.concatenate([tok_t[offs[i]:offs[i + 1]] for i in slots])
        a.n = len(slots)
    elif a.lengths == "trace":
        L = inputs.trace_lengths(a.n, seed=0)[0]
    elif a.lengths == "uniform":
        L = inputs.uniform_lengths(a.n, seed=0)
    else:
        L = np.full(a.n, int(a.lengths.split(":")[1]), np.int32)
    if slots is None:
        tok = inputs.make_tokens(L, seed=0)
    T = int(L.sum())
    p = binding.Predictor(cfg, inputs.flatten_weights(cfg, inputs.make_weights(cfg)), max_tokens=T, max_requests=a.n,
                         precision=a.precision, cls_last_layer=a.cls_last_layer,
                         residual16=None if a.residual is None else a.residual == "fp16")
    dev = torch.device("cuda:0")
    t_tok = torch.from_numpy(tok).to(dev)
    t_len = torch.from_numpy(L.astype(np.int32)).to(dev)
    out = torch.empty(a.n, dtype=torch.float32, device=dev)
    if slots is not None:
        table = torch.zeros(len(gen), dtype=torch.float32, device=dev)
        d_slots = torch.from_numpy(slots).to(dev)
        d_gen = torch.from_numpy(gen).to(dev)
        ids = torch.empty(a.cap, dtype=torch.int32, device=dev)
    if a.time:
        p.profile_enable(True)
    for _ in range(a.iters):
        if slots is None:
            p.predict_remaining(t_tok, t_len, T, out)
        else:
            p.predict_remaining(t_tok, t_len, T, table, out_slot=d_slots)
            p.isrtf_select(table, d_gen, a.cap, ids)
    torch.cuda.synchronize()
    binding.check(p.sync_status(), "predict")
    if a.time:
        prof = p.profile_read()
        print({k: round(ms / a.iters, 4) for k, (ms, _) in prof.items()})
    if a.dump:
        hid = torch.empty(T * cfg.hidden, dtype=torch.float32, device=dev)
        p.get_hidden(hid)
        torch.cuda.synchronize()
        pred = out if slots is None else table[torch.from_numpy(slots).to(dev)]
        np.savez(a.dump, pred=pred.cpu().numpy(), hidden=hid.cpu().numpy())
    print(f"T={T} n={a.n} pred[0:4]={(out if slots is None else table[torch.from_numpy(slots[:4]).to(dev)])[:4].tolist()}")


if __name__ == "__main__":
    main()
