"""Pins of oracle/fp8.py (the FP8 variant's definition, R20) against the E4M3 format's
closed forms, an independent library conversion, and the unquantised oracle."""
import numpy as np
import pytest

from oracle import encoder as oenc
from oracle import fp8
from paper_2505_09142_b200 import inputs


def test_e4m3_table_closed_forms():
    t = fp8.e4m3_values()
    assert len(t) == 127 and np.all(np.diff(t) > 0)
    assert t[0] == 0.0 and t[1] == 2.0 ** -9                 # smallest subnormal
    assert t[7] == 7 * 2.0 ** -9 and t[8] == 2.0 ** -6       # largest subnormal, smallest normal
    assert t[-1] == 448.0                                    # 1.75 * 2^8
    assert np.sum((t >= 1) & (t < 2)) == 8                   # 3 mantissa bits per binade
    np.testing.assert_array_equal(t[t >= 1][:8], 1 + np.arange(8) / 8)


def test_round_e4m3_rules():
    t = fp8.e4m3_values()
    np.testing.assert_array_equal(fp8.round_e4m3(t), t)                   # representable -> itself
    np.testing.assert_array_equal(fp8.round_e4m3(-t), -t)
    # ties to the even code: 1 + 1/16 sits between 1 (code even) and 1.125 (odd)
    assert fp8.round_e4m3(np.array(1.0625)) == 1.0
    assert fp8.round_e4m3(np.array(1.1875)) == 1.25                      # between 1.125 (odd) and 1.25
    assert fp8.round_e4m3(np.array(2.0 ** -10)) == 0.0                   # half the smallest subnormal
    assert fp8.round_e4m3(np.array(3 * 2.0 ** -10)) == 2 * 2.0 ** -9     # 1.5 subnormal steps -> even
    assert fp8.round_e4m3(np.array(1e6)) == 448.0 and fp8.round_e4m3(np.array(-500.0)) == -448.0
    assert fp8.round_e4m3(np.array(464.0 - 1e-9)) == 448.0               # saturating, not overflowing


def test_round_e4m3_is_nearest_by_brute_force():
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.normal(0, 1, 4000), rng.normal(0, 100, 2000), rng.normal(0, 0.01, 2000)])
    x = x[np.abs(x) <= 448]
    r = fp8.round_e4m3(x)
    t = np.concatenate([-fp8.e4m3_values()[::-1], fp8.e4m3_values()])
    best = np.abs(x[:, None] - t[None, :]).min(axis=1)
    np.testing.assert_array_equal(np.abs(r - x), best)
    normal = np.abs(x) >= 2.0 ** -6
    assert np.all(np.abs(r - x)[normal] <= np.abs(x[normal]) * 2.0 ** -4)


def test_round_e4m3_matches_torch_float8():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(1)
    x = np.concatenate([rng.normal(0, 3, 20000), rng.uniform(-448, 448, 5000)]).astype(np.float32)
    ref = torch.from_numpy(x).to(torch.float8_e4m3fn).float().numpy().astype(np.float64)
    np.testing.assert_array_equal(fp8.round_e4m3(x.astype(np.float64)), ref)


def test_quant_weight_row_scale():
    rng = np.random.default_rng(2)
    w = rng.normal(0, 0.02, (16, 64))
    w[3] = 0.0
    q = fp8.quant_weight(w)
    amax = np.abs(w).max(axis=1)
    for r in range(16):
        if amax[r] > 0:
            assert np.abs(q[r]).max() == pytest.approx(amax[r], rel=1e-15)    # the row max is exact
    assert np.all(q[3] == 0)
    s = np.where(amax > 0, amax / 448, 1)[:, None]
    normal = np.abs(w) / s >= 2.0 ** -6
    assert np.all(np.abs(q - w)[normal] <= (np.abs(w) * 2.0 ** -4)[normal] * (1 + 1e-12))


def test_fp8_layer_reduces_to_oracle_without_rounding(monkeypatch):
    """With the E4M3 rounding replaced by the identity, the FP8 forward is the fp64 oracle
    bit for bit (no dropped or reordered term)."""
    cfg = inputs.CONFIGS["tiny"]
    W = inputs.make_weights(cfg, seed=0)
    tokens = inputs.make_tokens(np.array([37], np.int32), seed=3)
    monkeypatch.setattr(fp8, "round_e4m3", lambda x: np.asarray(x, np.float64))
    Wq = fp8.quantize_weights(W, cfg)
    for k in W:
        np.testing.assert_allclose(np.asarray(Wq[k], np.float64), np.asarray(W[k], np.float64), rtol=1e-15, atol=0)
    np.testing.assert_allclose(fp8.encode_fp8(tokens, Wq, cfg), oenc.encode(tokens, W, cfg), rtol=0, atol=1e-12)


def test_fp8_forward_error_is_bounded():
    """The quantised forward stays near the fp64 one (each GEMM input carries <= 2^-4 relative
    rounding): a sanity band, not a parity claim."""
    cfg = inputs.CONFIGS["tiny"]
    W = inputs.make_weights(cfg, seed=0)
    tokens = inputs.make_tokens(np.array([40], np.int32), seed=4)
    h8 = fp8.encode_fp8(tokens, fp8.quantize_weights(W, cfg), cfg)
    h = oenc.encode(tokens, W, cfg)
    err = np.abs(h8 - h)
    assert 1e-4 < err.max() < 0.5
