"""Write paper_2505_09142_b200/head_calibration.json.  TEST INFRASTRUCTURE ONLY.

Random-init predictions sit near 0, clamp to ties and make ISRTF degenerate to
FCFS order.  This committed script calls only oracle/ to measure the raw
(uncalibrated) head output on a fixed 64-request trace-shaped calibration set
and stores an affine (scale, offset) for the LAST head layer so that
predictions spread as 256 +- 64 tokens (SURVEY.md Sec. 8c "Head calibration").
The constants are part of the weights: both sides consume them identically.

    python -m oracle.calibrate_head [tiny base large]
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

from paper_2505_09142_b200 import inputs
from . import head as ohead

CALIB_SEED = 77
CALIB_N = 64
TARGET_MEAN, TARGET_STD = 256.0, 64.0


def calibrate(name: str, pooling: int = inputs.POOL_MEAN, n: int = CALIB_N):
    cfg = inputs.EncoderConfig(**{**inputs.CONFIGS[name].to_dict(), "pooling": pooling})
    W = inputs.make_weights(cfg, seed=0, calibrated=False)
    L, _, _ = inputs.trace_lengths(n, seed=CALIB_SEED)
    tok = inputs.make_tokens(L, seed=CALIB_SEED)
    raw = ohead.predict(tok, L, W, cfg)
    scale = TARGET_STD / float(raw.std())
    offset = TARGET_MEAN - scale * float(raw.mean())
    return {"scale": scale, "offset": offset, "raw_mean": float(raw.mean()),
            "raw_std": float(raw.std()), "n": n, "seed": CALIB_SEED}


def main(argv):
    names = argv or ["tiny", "base"]
    path = inputs._CALIB_PATH
    table = {}
    if os.path.exists(path):
        with open(path) as f:
            table = json.load(f)
    for name in names:
        for pooling in (inputs.POOL_MEAN, inputs.POOL_CLS):
            key = f"{name}/pool{pooling}"
            table[key] = calibrate(name, pooling)
            print(key, table[key], flush=True)
    with open(path, "w") as f:
        json.dump(table, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1:])
