"""Latency of the ISRTF select paths on one B200 (cfg5 table: 65,536 slots, cap 256 by default):
single-GPU elis_isrtf_select, elis_isrtf_select_dist over NCCL (world 1) and over peer memory
(world 1, and world 2/4/8 ranks sharing the device, each with its own stream), CUDA events,
median of `iters` back-to-back calls.

    python scripts/select_latency.py [--n 65536] [--cap 256] [--iters 200]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_09142_b200 import binding, inputs  # noqa: E402


def predictor():
    cfg = inputs.CONFIGS["tiny"]
    return binding.Predictor(cfg, inputs.flatten_weights(cfg, inputs.make_weights(cfg, seed=0)), 1024, 1024)


def timed(fn, iters, streams):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        a = [torch.cuda.Event(enable_timing=True) for _ in streams]
        b = [torch.cuda.Event(enable_timing=True) for _ in streams]
        for e, s in zip(a, streams):
            e.record(s)
        fn()
        for e, s in zip(b, streams):
            e.record(s)
        torch.cuda.synchronize()
        ts.append(max(x.elapsed_time(y) for x, y in zip(a, b)) * 1e3)
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=65536)
    ap.add_argument("--cap", type=int, default=256)
    ap.add_argument("--iters", type=int, default=200)
    a = ap.parse_args()
    n, cap = a.n, a.cap
    pred = torch.from_numpy(inputs.random_predictions(n, seed=1)).cuda()
    gen_np, _, _ = inputs.random_sched_state(n, seed=2)
    gen = torch.from_numpy(gen_np).cuda()
    res = {"n": n, "cap": cap}
    st = torch.cuda.current_stream()
    ids = torch.empty(cap, dtype=torch.int32, device="cuda")

    P = predictor()
    res["single_us"] = timed(lambda: P.isrtf_select(pred, gen, cap, ids, stream=st), a.iters, [st])
    P.dist_attach(0, 1, binding.nccl_unique_id())
    res["dist_nccl_w1_us"] = timed(lambda: P.isrtf_select_dist(pred, gen, 0, cap, ids, stream=st), a.iters, [st])
    binding.peer_attach_local([P])
    res["dist_peer_w1_us"] = timed(lambda: P.isrtf_select_dist(pred, gen, 0, cap, ids, stream=st), a.iters, [st])
    P.close()
    for world in (2, 4, 8):
        Ps = [predictor() for _ in range(world)]
        binding.peer_attach_local(Ps)
        streams = [torch.cuda.Stream() for _ in range(world)]
        nl = n // world
        outs = [torch.empty(cap, dtype=torch.int32, device="cuda") for _ in range(world)]

        def call():
            for r in range(world):
                Ps[r].isrtf_select_dist(pred[r * nl:(r + 1) * nl], gen[r * nl:(r + 1) * nl], r * nl, cap, outs[r],
                                        stream=streams[r])
        torch.cuda.synchronize()
        res[f"dist_peer_w{world}_shared_gpu_us"] = timed(call, a.iters, streams)
        assert all(bool((o == outs[0]).all()) for o in outs)
        for p in Ps:
            p.close()
    print(json.dumps(res))


if __name__ == "__main__":
    main()
