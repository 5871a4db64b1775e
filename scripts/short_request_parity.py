#!/usr/bin/env python3
"""Prediction error of the short requests of the cfg2 workload (256 trace-shaped BGE-base requests,
one call) vs the fp64 oracle, per operand / residual precision: every request of <= 64 tokens (the
ones whose mean pool averages the fewest rows) and 16 longer ones.

    python scripts/short_request_parity.py > profiles/rNN_short_request_parity.jsonl
"""
from __future__ import annotations

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import head as ohead  # noqa: E402
from paper_2505_09142_b200 import binding, inputs  # noqa: E402


def main():
    n = 256
    L, _, _ = inputs.trace_lengths(n, seed=0)
    tokens = inputs.make_tokens(L, seed=0)
    cfg = inputs.CONFIGS["base"]
    W = inputs.make_weights(cfg, seed=0)
    flat = inputs.flatten_weights(cfg, W)
    short = [int(i) for i in np.where(L <= 64)[0]]
    longer = [int(i) for i in np.argsort(L)[np.linspace(len(short), n - 1, 16).astype(int)]]
    sample = sorted(set(short + longer))
    ref = ohead.predict(tokens, L, W, cfg, requests=sample)
    for prec, r16 in (("fp16", True), ("fp16", False), ("bf16", False)):
        P = binding.Predictor(cfg, flat, int(L.sum()), n, precision=prec, residual16=r16)
        out = torch.empty(n, device="cuda")
        P.predict_remaining(torch.from_numpy(tokens).cuda(), torch.from_numpy(L.astype(np.int32)).cuda(), int(L.sum()),
                            out)
        assert P.sync_status() == 0
        gpu = out.cpu().numpy().astype(np.float64)[sample]
        P.close()
        abs_err = np.abs(gpu - ref)
        rel = abs_err / np.maximum(np.abs(ref), 1.0)
        w = int(np.argmax(rel))
        print(json.dumps({"precision": prec, "residual": "fp16" if r16 else "fp32", "requests": len(sample),
                          "short_requests": len(short), "rel_max": float(rel.max()), "rel_p90": float(np.quantile(rel, 0.9)),
                          "abs_max_tokens": float(abs_err.max()), "over_1e-2": int((rel > 1e-2).sum()),
                          "worst": {"request": sample[w], "L": int(L[sample[w]]), "gpu": float(gpu[w]), "oracle": float(ref[w])}}))


if __name__ == "__main__":
    main()
