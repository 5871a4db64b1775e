"""CLS-only last layer: with CLS pooling (P:138 reading, R2) only
row 0 of each request reaches the head, so the last layer's attention, out-projection and FFN
run on the n CLS rows.  Exact in the method's arithmetic: the pruned forward must match the fp64
oracle to the same bars as the unpruned one, and the CLS rows of the final hidden states too."""
import numpy as np
import pytest

from paper_2505_09142_b200 import inputs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

CLS_PRED_RTOL = {"bf16": 3e-2, "fp16": 1e-2}   # DESIGN.md "Tolerances" (CLS rows)
HIDDEN_ATOL = 2e-2


def _predict(cfg, flat, L, tokens, **kw):
    from paper_2505_09142_b200 import binding
    T = int(L.sum())
    kw.setdefault("residual16", False)  # the fp32 stream on both sides of the comparison
    P = binding.Predictor(cfg, flat, T, len(L), **kw)
    out = torch.full((len(L),), float("nan"), device="cuda")
    P.predict_remaining(torch.from_numpy(tokens).cuda(), torch.from_numpy(L).cuda(), T, out)
    hid = torch.empty(T, cfg.hidden, device="cuda")
    P.get_hidden(hid)
    assert P.sync_status() == 0
    r = out.cpu().numpy().astype(np.float64), hid.cpu().numpy().astype(np.float64)
    P.close()
    return r


@pytest.mark.parametrize("precision", ["bf16", "fp16"])
def test_cls_last_layer_parity(cuda_lib, precision):
    from oracle import head as ohead
    cfg = inputs.EncoderConfig(**{**inputs.CONFIGS["base"].to_dict(), "pooling": inputs.POOL_CLS})
    W = inputs.make_weights(cfg, seed=0)
    flat = inputs.flatten_weights(cfg, W)
    L = np.array([1, 2, 31, 64, 127, 128, 129, 257, 400, 512, 77, 5], np.int32)
    tokens = inputs.make_tokens(L, seed=12)
    full, hfull = _predict(cfg, flat, L, tokens, precision=precision)
    pr, hpr = _predict(cfg, flat, L, tokens, precision=precision, cls_last_layer=True)
    ref, hs = ohead.predict_with_hidden(tokens, L, W, cfg)
    cls_rows = inputs.offsets(L)[:-1]
    ref_cls = np.stack([h[0] for h in hs])
    r_pr = np.abs(pr - ref) / np.maximum(np.abs(ref), 1.0)
    r_full = np.abs(full - ref) / np.maximum(np.abs(ref), 1.0)
    print(f"{precision}: pruned rel max {r_pr.max():.4g}, unpruned {r_full.max():.4g}; CLS hidden pruned "
          f"{np.abs(hpr[cls_rows] - ref_cls).max():.4g} unpruned {np.abs(hfull[cls_rows] - ref_cls).max():.4g}")
    assert r_pr.max() <= CLS_PRED_RTOL[precision]
    assert np.abs(hpr[cls_rows] - ref_cls).max() <= HIDDEN_ATOL
    # the non-CLS rows are untouched by the pruned layer: they hold layer L-1 states, not final ones
    assert not np.allclose(np.delete(hpr, cls_rows, axis=0), np.delete(hfull, cls_rows, axis=0))


def test_cls_last_layer_fp8_close_to_unpruned(cuda_lib):
    from oracle import fp8 as ofp8
    cfg = inputs.EncoderConfig(**{**inputs.CONFIGS["base"].to_dict(), "pooling": inputs.POOL_CLS})
    W = inputs.make_weights(cfg, seed=0)
    flat = inputs.flatten_weights(cfg, W)
    L = np.array([40, 200, 512, 3, 129], np.int32)
    tokens = inputs.make_tokens(L, seed=13)
    pr, _ = _predict(cfg, flat, L, tokens, precision="fp8", cls_last_layer=True)
    ref8, _ = ofp8.predict_with_hidden_fp8(tokens, L, W, cfg)
    rel = np.abs(pr - ref8) / np.maximum(np.abs(ref8), 1.0)
    print("fp8 pruned vs fp8 oracle rel", rel.max())
    assert np.isfinite(pr).all() and rel.max() <= 0.3
