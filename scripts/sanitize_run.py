#!/usr/bin/env python3
"""Small end-to-end calls for compute-sanitizer (memcheck / racecheck / synccheck):
cfg1 (tiny encoder, 16 x 64 tokens, select cap 4) and a ~1k-token BGE-base call on the default
path (fp16 operands + fp16 residual stream: tcgen05 GEMMs with the LN cluster exchange, tcgen05
attention, 3xTF32 head), then the ISRTF select over 65,536 keys.

    compute-sanitizer --tool memcheck python scripts/sanitize_run.py
"""
from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2505_09142_b200 import binding, inputs  # noqa: E402


def run(name, lengths, cap):
    cfg = inputs.CONFIGS[name]
    W = inputs.make_weights(cfg, seed=0)
    L = np.asarray(lengths, np.int32)
    tok = inputs.make_tokens(L, seed=1)
    P = binding.Predictor(cfg, inputs.flatten_weights(cfg, W), int(L.sum()), len(L))
    out = torch.empty(len(L), device="cuda")
    P.predict_remaining(torch.from_numpy(tok).cuda(), torch.from_numpy(L).cuda(), int(L.sum()), out)
    ids = torch.empty(cap, dtype=torch.int32, device="cuda")
    P.isrtf_select(out, torch.zeros(len(L), dtype=torch.int32, device="cuda"), cap, ids)
    assert P.sync_status() == 0, binding.lib().elis_last_error()
    print(name, "ok", out.cpu().numpy()[:4], ids.cpu().numpy()[:4])
    return P


def main():
    torch.cuda.set_device(0)
    run("tiny", [64] * 16, 4).close()
    P = run("base", [300, 128, 65, 200, 33, 7, 129, 140], 4)
    keys = torch.from_numpy(inputs.random_predictions(65536, seed=2, kind="spread")).cuda()
    gen = torch.zeros(65536, dtype=torch.int32, device="cuda")
    ids = torch.empty(256, dtype=torch.int32, device="cuda")
    P.isrtf_select(keys, gen, 256, ids)
    assert P.sync_status() == 0
    print("select 65536 ok", ids.cpu().numpy()[:4])
    P.close()


if __name__ == "__main__":
    main()
