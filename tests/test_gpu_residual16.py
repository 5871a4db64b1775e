"""fp16 residual stream (elis_config.residual16; SURVEY.md Sec. 8b `residual_fp32 = 0`, DESIGN.md
R23): with fp16 operands the residual between layers is the fp16 copy the GEMMs already read, so
the LayerNorm GEMM epilogues (EPI_BIAS_RESID16_LN) move 2 bytes per element instead of 4 + 4 + 2.
Held to the north_star bars (predictions 1e-2 relative, hidden 2e-2 absolute) against the fp64
oracle on the trace-shaped workloads the fp16 path is tested on, plus batch invariance and the
per-op epilogue against the fp32-residual epilogue."""
import numpy as np
import pytest

from paper_2505_09142_b200 import inputs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

PRED_RTOL = 1e-2
HIDDEN_ATOL = 2e-2


def _run(cfg, flat, L, tokens, residual16, precision="fp16"):
    from paper_2505_09142_b200 import binding
    T = int(L.sum())
    P = binding.Predictor(cfg, flat, T, len(L), precision=precision, residual16=residual16)
    out = torch.full((len(L),), float("nan"), device="cuda")
    P.predict_remaining(torch.from_numpy(tokens).cuda(), torch.from_numpy(L).cuda(), T, out)
    hid = torch.empty(T, cfg.hidden, device="cuda")
    P.get_hidden(hid)
    assert P.sync_status() == 0
    r = out.cpu().numpy().astype(np.float64), hid.cpu().numpy().astype(np.float64)
    P.close()
    return r


@pytest.mark.parametrize("seed,n", [(5, 24), (11, 16), (3, 32)])
def test_residual16_base_parity(cuda_lib, seed, n):
    from oracle import head as ohead
    cfg = inputs.CONFIGS["base"]
    W = inputs.make_weights(cfg, seed=0)
    flat = inputs.flatten_weights(cfg, W)
    L, _, _ = inputs.trace_lengths(n, seed=seed)
    L = L.astype(np.int32)
    tokens = inputs.make_tokens(L, seed=seed)
    ref, hs = ohead.predict_with_hidden(tokens, L, W, cfg)
    ref_h = np.concatenate(hs)
    res = {r16: _run(cfg, flat, L, tokens, r16) for r16 in (False, True)}
    for r16, (p, h) in res.items():
        rel = np.abs(p - ref) / np.maximum(np.abs(ref), 1.0)
        print(f"residual16={r16}: pred rel max {rel.max():.4g} mean {rel.mean():.4g}; "
              f"hidden max abs {np.abs(h - ref_h).max():.4g} rms {np.sqrt(((h - ref_h) ** 2).mean()):.3g}")
    p, h = res[True]
    rel = np.abs(p - ref) / np.maximum(np.abs(ref), 1.0)
    assert rel.max() <= PRED_RTOL, rel.max()
    assert np.abs(h - ref_h).max() <= HIDDEN_ATOL, np.abs(h - ref_h).max()


def test_residual16_batch_invariance_and_select(cuda_lib):
    """pred_i is bitwise the same alone and inside a ragged batch; the ISRTF batch on those
    predictions is the oracle select's."""
    from paper_2505_09142_b200 import binding
    from oracle.select import isrtf_select
    cfg = inputs.CONFIGS["base"]
    W = inputs.make_weights(cfg, seed=0)
    flat = inputs.flatten_weights(cfg, W)
    L, gen, _ = inputs.trace_lengths(96, seed=17)
    L = L.astype(np.int32)
    tokens = inputs.make_tokens(L, seed=17)
    T = int(L.sum())
    P = binding.Predictor(cfg, flat, T, len(L), precision="fp16", residual16=True)
    out = torch.empty(len(L), device="cuda")
    P.predict_remaining(torch.from_numpy(tokens).cuda(), torch.from_numpy(L).cuda(), T, out)
    ids = torch.empty(8, dtype=torch.int32, device="cuda")
    P.isrtf_select(out, torch.from_numpy(gen.astype(np.int32)).cuda(), 8, ids)
    assert P.sync_status() == 0
    gpu = out.cpu().numpy()
    o_ids, _, _, _ = isrtf_select(gpu, gen.astype(np.int32), 8)
    np.testing.assert_array_equal(ids.cpu().numpy(), o_ids)
    offs = inputs.offsets(L)
    for i in (0, 7, int(np.argmax(L)), len(L) - 1):
        t1 = tokens[offs[i]:offs[i + 1]]
        one = torch.empty(1, device="cuda")
        P.predict_remaining(torch.from_numpy(t1).cuda(), torch.from_numpy(L[i:i + 1]).cuda(), int(L[i]), one)
        assert P.sync_status() == 0
        assert one.item() == gpu[i], (i, one.item(), gpu[i])
    P.close()


def test_residual16_config_rules(cuda_lib):
    """residual16 needs fp16 operands and no CLS-only last layer (ELIS_ERR_CONFIG otherwise)."""
    from paper_2505_09142_b200 import binding
    cfg = inputs.CONFIGS["base"]
    flat = inputs.flatten_weights(cfg, inputs.make_weights(cfg, seed=0))
    with pytest.raises(binding.ElisError):
        binding.Predictor(cfg, flat, 1024, 8, precision="bf16", residual16=True)


def test_residual16_cls_pooling_parity(cuda_lib):
    """CLS pooling (P:138 reading) over the fp16 stream: the pooled row is read from the fp16
    buffer (k_pool<__half>); fp16 operands hold CLS to the 1e-2 bar (DESIGN.md Tolerances)."""
    from oracle import head as ohead
    cfg = inputs.EncoderConfig(**{**inputs.CONFIGS["base"].to_dict(), "pooling": inputs.POOL_CLS})
    W = inputs.make_weights(cfg, seed=0)
    flat = inputs.flatten_weights(cfg, W)
    L, _, _ = inputs.trace_lengths(16, seed=9)
    L = L.astype(np.int32)
    tokens = inputs.make_tokens(L, seed=9)
    ref, hs = ohead.predict_with_hidden(tokens, L, W, cfg)
    p, h = _run(cfg, flat, L, tokens, True)
    rel = np.abs(p - ref) / np.maximum(np.abs(ref), 1.0)
    print(f"CLS residual16: pred rel max {rel.max():.4g}; hidden max abs {np.abs(h - np.concatenate(hs)).max():.4g}")
    assert rel.max() <= PRED_RTOL, rel.max()
    assert np.abs(h - np.concatenate(hs)).max() <= HIDDEN_ATOL
