#!/usr/bin/env python3
"""Latency of one elis_predict_remaining for small due sets (the cfg4 stream simulator's regime:
a handful of requests per scheduling iteration), eager and replayed from a captured CUDA graph.

    python scripts/small_predict_latency.py [--ns 1,4,16,64] [--iters 200]

Prints one JSON line per n: mean device time per call (CUDA events around `iters` back-to-back
calls) and the number of library kernel launches per call.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2505_09142_b200 import binding, inputs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ns", default="1,4,16,64")
    ap.add_argument("--iters", type=int, default=200)
    ap.add_argument("--config", default="base")
    a = ap.parse_args()
    cfg = inputs.CONFIGS[a.config]
    flat = inputs.flatten_weights(cfg, inputs.make_weights(cfg))
    dev = torch.device("cuda:0")
    for n in (int(x) for x in a.ns.split(",")):
        L = np.asarray(inputs.trace_lengths(n, seed=1)[0], np.int32)
        T = int(L.sum())
        tok = inputs.make_tokens(L, seed=1)
        p = binding.Predictor(cfg, flat, max_tokens=T, max_requests=n)
        t_tok = torch.from_numpy(tok).to(dev)
        t_len = torch.from_numpy(L).to(dev)
        out = torch.empty(n, dtype=torch.float32, device=dev)
        st = torch.cuda.Stream()
        res = {"n": n, "tokens": T}
        with torch.cuda.stream(st):
            for _ in range(5):
                p.predict_remaining(t_tok, t_len, T, out, stream=st)
            st.synchronize()
            l0 = p.launch_count()
            p.predict_remaining(t_tok, t_len, T, out, stream=st)
            res["launches_per_call"] = p.launch_count() - l0
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(a.iters):
                p.predict_remaining(t_tok, t_len, T, out, stream=st)
            e1.record(st)
            st.synchronize()
            res["eager_ms"] = round(e0.elapsed_time(e1) / a.iters, 4)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=st):
                p.predict_remaining(t_tok, t_len, T, out, stream=st)
            for _ in range(5):
                g.replay()
            e0.record(st)
            for _ in range(a.iters):
                g.replay()
            e1.record(st)
            st.synchronize()
            res["graph_ms"] = round(e0.elapsed_time(e1) / a.iters, 4)
        binding.check(p.sync_status(), "predict")
        res["pdl"] = os.environ.get("ELIS_PDL", "1") != "0"
        print(json.dumps(res), flush=True)
        p.close()


if __name__ == "__main__":
    main()
