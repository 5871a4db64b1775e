#!/usr/bin/env python3
"""Parity sweep of the predictor against the fp64 oracle over many seeded workloads (evidence for
DESIGN.md R21 / R23): for each seed and length recipe, the max relative prediction error and the
max absolute final-hidden error of every precision path, one JSON line per (seed, recipe).

    python scripts/parity_sweep.py [--seeds 8] [--n 24] [--paths fp16-r16,fp16,bf16]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import head as ohead  # noqa: E402  (test infrastructure: the checker)
from paper_2505_09142_b200 import binding, inputs  # noqa: E402


def run(cfg, flat, L, tokens, path):
    prec, r16 = ("fp16", True) if path == "fp16-r16" else (path, False)
    T = int(L.sum())
    P = binding.Predictor(cfg, flat, T, len(L), precision=prec, residual16=r16)
    out = torch.empty(len(L), device="cuda")
    P.predict_remaining(torch.from_numpy(tokens).cuda(), torch.from_numpy(L).cuda(), T, out)
    hid = torch.empty(T, cfg.hidden, device="cuda")
    P.get_hidden(hid)
    binding.check(P.sync_status(), "predict")
    r = out.cpu().numpy().astype(np.float64), hid.cpu().numpy().astype(np.float64)
    P.close()
    return r


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seeds", type=int, default=8)
    ap.add_argument("--n", type=int, default=24)
    ap.add_argument("--paths", default="fp16-r16,fp16,bf16")
    a = ap.parse_args()
    cfg = inputs.CONFIGS["base"]
    W = inputs.make_weights(cfg, seed=0)
    flat = inputs.flatten_weights(cfg, W)
    paths = a.paths.split(",")
    worst = {p: [0.0, 0.0] for p in paths}
    for seed in range(100, 100 + a.seeds):
        for recipe in ("trace", "uniform"):
            if recipe == "trace":
                L = inputs.trace_lengths(a.n, seed=seed)[0].astype(np.int32)
            else:
                L = inputs.uniform_lengths(a.n, 32, 512, seed=seed).astype(np.int32)
                L = L[: max(4, a.n // 3)]   # uniform requests are long: fewer per set
            tokens = inputs.make_tokens(L, seed=seed)
            t0 = time.time()
            ref, hs = ohead.predict_with_hidden(tokens, L, W, cfg)
            ref_h = np.concatenate(hs)
            t_or = time.time() - t0
            row = {"seed": seed, "recipe": recipe, "n": int(len(L)), "tokens": int(L.sum()),
                   "pred_range": [float(ref.min()), float(ref.max())], "oracle_s": round(t_or, 1)}
            for p in paths:
                g, h = run(cfg, flat, L, tokens, p)
                rel = np.abs(g - ref) / np.maximum(np.abs(ref), 1.0)
                he = float(np.abs(h - ref_h).max())
                row[p] = {"pred_rel_max": float(rel.max()), "pred_rel_mean": float(rel.mean()), "hidden_abs_max": he}
                worst[p] = [max(worst[p][0], float(rel.max())), max(worst[p][1], he)]
            print(json.dumps(row), flush=True)
    print(json.dumps({"summary": {p: {"pred_rel_max": v[0], "hidden_abs_max": v[1],
                                      "meets_bars": v[0] <= 1e-2 and v[1] <= 2e-2} for p, v in worst.items()},
                      "bars": {"pred_rel": 1e-2, "hidden_abs": 2e-2}, "seeds": a.seeds, "n": a.n}), flush=True)


if __name__ == "__main__":
    main()
