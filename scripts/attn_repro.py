"""Tiny op_attention call (the per-op parity test's lengths) for debugging attention engines."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2505_09142_b200 import binding
d, nh = 64, 12
H = d * nh
arg = sys.argv[1] if len(sys.argv) > 1 else "1,2,63,64,65,130,7,512,200,33"
if arg.startswith("trace:"):
    from paper_2505_09142_b200 import inputs
    lengths = np.asarray(inputs.trace_lengths(int(arg[6:]), seed=0)[0], np.int32)
else:
    lengths = np.array([int(x) for x in arg.split(",")], np.int32)
T = int(lengths.sum())
qkv = torch.randn(3 * T * H, device="cuda").to(torch.bfloat16)
ctx = torch.full((T, H), float("nan"), dtype=torch.bfloat16, device="cuda")
binding.op_attention(qkv, torch.from_numpy(lengths).cuda(), H, nh, ctx)
torch.cuda.synchronize()
print("ok", lengths.tolist()[:12], "nan rows:", int(torch.isnan(ctx.float()).any(1).sum()))
