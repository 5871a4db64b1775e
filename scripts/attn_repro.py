"""Tiny op_attention call (BGE-base heads: d = 64, 12 heads) for debugging and A/B of the attention
engines (ELIS_ATTN_ENGINE selects one per process).

    python scripts/attn_repro.py 1,2,63,64,65,130,7,512,200,33 [--f16] [--ramp] [--dump ctx.npy]
    python scripts/attn_repro.py trace:256

--ramp scales the keys x6 from position 64 and x12 from 192 (the lazy O rescale path); --dump saves
ctx as raw 16-bit words.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2505_09142_b200 import binding, inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("lengths", nargs="?", default="1,2,63,64,65,130,7,512,200,33")
ap.add_argument("--f16", action="store_true")
ap.add_argument("--ramp", action="store_true")
ap.add_argument("--seed", type=int, default=0)
ap.add_argument("--dump", default=None)
a = ap.parse_args()
d, nh = 64, 12
H = d * nh
if a.lengths.startswith("trace:"):
    lengths = np.asarray(inputs.trace_lengths(int(a.lengths[6:]), seed=0)[0], np.int32)
else:
    lengths = np.array([int(x) for x in a.lengths.split(",")], np.int32)
T = int(lengths.sum())
rng = np.random.default_rng(a.seed)
x = rng.normal(0, 1.0, (T, 3 * H)).astype(np.float32)
if a.ramp:
    starts = inputs.offsets(lengths)
    for i, L in enumerate(lengths):
        pos = np.arange(L)
        x[starts[i]:starts[i + 1], H:2 * H] *= np.where(pos >= 192, 12.0, np.where(pos >= 64, 6.0, 1.0))[:, None]
dt = torch.float16 if a.f16 else torch.bfloat16
qkv = torch.from_numpy(x).to(dt).cuda().view(T, 3, nh, d).permute(1, 2, 0, 3).contiguous()  # head-major planes
ctx = torch.full((T, H), float("nan"), dtype=dt, device="cuda")
binding.op_attention(qkv, torch.from_numpy(lengths).cuda(), H, nh, ctx, f16=a.f16)
torch.cuda.synchronize()
if a.dump:
    np.save(a.dump, ctx.view(torch.int16).cpu().numpy())
print("ok", lengths.tolist()[:12], "nan rows:", int(torch.isnan(ctx.float()).any(1).sum()))
