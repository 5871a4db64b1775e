"""fp16 operands: the same tcgen05 kernels with fp16 instead of
bf16 weights, activations and attention operands -- 3 more mantissa bits at the same speed.
Held to the north_star bars (predictions 1e-2 relative, hidden 2e-2 absolute) against the fp64
oracle, on the trace-shaped workload where the bf16 path's largest relative error (a request
predicted ~22 tokens) exceeds 1e-2."""
import numpy as np
import pytest

from paper_2505_09142_b200 import inputs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

PRED_RTOL = 1e-2
HIDDEN_ATOL = 2e-2
# bf16 operands (elis.h ELIS_PREC_BF16, not the default): DESIGN.md R21 bounds their prediction
# error by 8x the fp16 path's (bf16 keeps 8 significand bits, fp16 11: unit roundoff 2^-9 vs 2^-12)
# -- 8 x 0.63% (the fp16 worst case) ~ 5%, measured 5.8%; the bar is 8% relative and 2 tokens
# absolute.  The hidden-state bar is the north_star's 2e-2 (bf16 measured <= 0.019).
BF16_PRED_RTOL = 8e-2
BF16_PRED_ATOL_TOKENS = 2.0


def _run(cfg, flat, L, tokens, precision):
    from paper_2505_09142_b200 import binding
    T = int(L.sum())
    P = binding.Predictor(cfg, flat, T, len(L), precision=precision, residual16=False)
    out = torch.full((len(L),), float("nan"), device="cuda")
    P.predict_remaining(torch.from_numpy(tokens).cuda(), torch.from_numpy(L).cuda(), T, out)
    hid = torch.empty(T, cfg.hidden, device="cuda")
    P.get_hidden(hid)
    assert P.sync_status() == 0
    r = out.cpu().numpy().astype(np.float64), hid.cpu().numpy().astype(np.float64)
    P.close()
    return r


@pytest.mark.parametrize("seed,n", [(5, 24), (11, 16)])
def test_predict_fp16_base_parity(cuda_lib, seed, n):
    from oracle import head as ohead
    cfg = inputs.CONFIGS["base"]
    W = inputs.make_weights(cfg, seed=0)
    flat = inputs.flatten_weights(cfg, W)
    L, _, _ = inputs.trace_lengths(n, seed=seed)
    L = L.astype(np.int32)
    tokens = inputs.make_tokens(L, seed=seed)
    ref, hs = ohead.predict_with_hidden(tokens, L, W, cfg)
    ref_h = np.concatenate(hs)
    res = {prec: _run(cfg, flat, L, tokens, prec) for prec in ("bf16", "fp16")}
    for prec, (p, h) in res.items():
        rel = np.abs(p - ref) / np.maximum(np.abs(ref), 1.0)
        print(f"{prec}: pred rel max {rel.max():.4g} mean {rel.mean():.4g} abs max {np.abs(p - ref).max():.4g}; "
              f"hidden max abs {np.abs(h - ref_h).max():.4g}")
    # bf16 is held to its own documented bound on the same (hardest measured) workload
    pb, hb = res["bf16"]
    rel_b = np.abs(pb - ref) / np.maximum(np.abs(ref), 1.0)
    assert rel_b.max() <= BF16_PRED_RTOL, rel_b.max()
    assert np.abs(pb - ref).max() <= BF16_PRED_ATOL_TOKENS, np.abs(pb - ref).max()
    assert np.abs(hb - ref_h).max() <= HIDDEN_ATOL
    p16, h16 = res["fp16"]
    rel = np.abs(p16 - ref) / np.maximum(np.abs(ref), 1.0)
    assert rel.max() <= PRED_RTOL, rel.max()
    assert np.abs(h16 - ref_h).max() <= HIDDEN_ATOL
    # fp16 carries 8x finer operand rounding than bf16: its errors must be clearly smaller
    p16_err = np.abs(p16 - ref).mean()
    assert p16_err < 0.5 * np.abs(res["bf16"][0] - ref).mean()


def test_fp16_select_bit_exact(cuda_lib):
    """ISRTF selection on the fp16 path's predictions is the oracle's, bit for bit."""
    from paper_2505_09142_b200 import binding
    from oracle.select import isrtf_select
    cfg = inputs.CONFIGS["base"]
    W = inputs.make_weights(cfg, seed=0)
    L, gen, _ = inputs.trace_lengths(64, seed=21)
    L = L.astype(np.int32)
    tokens = inputs.make_tokens(L, seed=21)
    T = int(L.sum())
    P = binding.Predictor(cfg, inputs.flatten_weights(cfg, W), T, len(L), precision="fp16", residual16=False)
    out = torch.empty(len(L), device="cuda")
    P.predict_remaining(torch.from_numpy(tokens).cuda(), torch.from_numpy(L).cuda(), T, out)
    ids = torch.empty(16, dtype=torch.int32, device="cuda")
    P.isrtf_select(out, torch.from_numpy(gen.astype(np.int32)).cuda(), 16, ids)
    assert P.sync_status() == 0
    o_ids, _, _, _ = isrtf_select(out.cpu().numpy(), gen.astype(np.int32), 16)
    np.testing.assert_array_equal(ids.cpu().numpy(), o_ids)
    P.close()
