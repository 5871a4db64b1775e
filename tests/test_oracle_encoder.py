"""Pins for oracle/encoder.py and oracle/head.py against things other than themselves.

Each test cites what fixes the expected value:
  * closed forms (LayerNorm statistics, softmax row sums, erf-GELU values,
    L = 1 attention, Wq = Wk = 0 attention);
  * invariants (permutation equivariance without positions, padding invariance
    of the varlen encoding -- BASELINE.json north_star);
  * a library routine with identical weights: HF ``transformers.BertModel``
    (fp64, eager attention) for the whole encoder, ``torch.nn.Sequential`` for
    the head.  These are independent implementations of BERT / an MLP, not a
    re-typing of the oracle's formulas.
"""
import math

import numpy as np
import pytest

from paper_2505_09142_b200 import inputs
from oracle import encoder as oenc
from oracle import head as ohead

TINY = inputs.CONFIGS["tiny"]


def small_cfg(**kw):
    base = dict(name="t", num_layers=2, hidden=64, num_heads=4, intermediate=256)
    base.update(kw)
    return inputs.EncoderConfig(**base)


# ---------------------------------------------------------------- closed forms

def test_layernorm_mean0_var1():
    """gamma = 1, beta = 0: each row has mean 0 and variance var/(var + eps) (closed form)."""
    rng = np.random.default_rng(0)
    x = rng.normal(3.0, 2.5, size=(17, 768))
    eps = 1e-12
    y = oenc.layer_norm(x, np.ones(768), np.zeros(768), eps)
    assert np.max(np.abs(y.mean(axis=1))) < 1e-14
    var_in = x.var(axis=1)
    np.testing.assert_allclose(y.var(axis=1), var_in / (var_in + eps), rtol=0, atol=1e-13)
    # a large eps makes the eps term visible: variance = var / (var + eps)
    y2 = oenc.layer_norm(x, np.ones(768), np.zeros(768), 5.0)
    np.testing.assert_allclose(y2.var(axis=1), var_in / (var_in + 5.0), rtol=1e-12)


def test_layernorm_affine():
    """gamma, beta act per column after normalisation: LN(x; g, b) = g * LN(x; 1, 0) + b."""
    rng = np.random.default_rng(1)
    x = rng.normal(size=(5, 32))
    g, b = rng.normal(size=32), rng.normal(size=32)
    base = oenc.layer_norm(x, np.ones(32), np.zeros(32), 1e-12)
    np.testing.assert_allclose(oenc.layer_norm(x, g, b, 1e-12), base * g + b, rtol=0, atol=1e-14)


def test_softmax_rows_sum_to_one_and_shift_invariant():
    rng = np.random.default_rng(2)
    s = rng.normal(0, 30, size=(64, 300))
    p = oenc.softmax_rows(s)
    assert np.max(np.abs(p.sum(axis=1) - 1.0)) < 1e-15 * 300
    assert (p >= 0).all()
    np.testing.assert_allclose(oenc.softmax_rows(s + 1234.5), p, rtol=1e-12, atol=1e-300)
    # two equal logits and the rest -inf-ish -> 1/2, 1/2
    t = np.array([[5.0, 5.0, -1e4, -1e4]])
    np.testing.assert_allclose(oenc.softmax_rows(t), [[0.5, 0.5, 0.0, 0.0]], atol=1e-300)


def test_gelu_erf_values():
    """GELU(z) = z * Phi(z): Phi(1) = 0.8413447460685429, Phi(-1) = 0.15865525393145707."""
    z = np.array([0.0, 1.0, -1.0, 8.0, -8.0, 2.0])
    g = oenc.gelu(z)
    expect = [0.0, 0.8413447460685429, -0.15865525393145707, 8.0, -8.0 * 6.22096057427178e-16,
              2.0 * 0.9772498680518208]
    np.testing.assert_allclose(g, expect, rtol=1e-13, atol=1e-15)  # 1+erf cancels near -8
    for v in np.linspace(-5, 5, 41):
        assert abs(oenc.gelu(np.array([v]))[0] - 0.5 * v * (1 + math.erf(v / math.sqrt(2)))) < 1e-15


def test_attention_single_token_is_v():
    """L = 1: softmax of one score is 1, so ctx = v exactly."""
    rng = np.random.default_rng(3)
    q, k, v = rng.normal(size=(3, 1, 64))
    np.testing.assert_array_equal(oenc.attention(q, k, v, 4), v)


def test_attention_zero_scores_is_mean_v():
    """q = 0 (Wq = 0): all scores equal, so every row of ctx = mean over tokens of v."""
    rng = np.random.default_rng(4)
    L, H = 37, 64
    k, v = rng.normal(size=(2, L, H))
    ctx = oenc.attention(np.zeros((L, H)), k, v, 4)
    np.testing.assert_allclose(ctx, np.broadcast_to(v.mean(axis=0), (L, H)), rtol=0, atol=1e-14)


def test_attention_heads_independent():
    """Changing head 1's v columns leaves head 0's output columns untouched."""
    rng = np.random.default_rng(5)
    q, k, v = rng.normal(size=(3, 20, 64))
    a = oenc.attention(q, k, v, 4)
    v2 = v.copy()
    v2[:, 16:32] += 3.0
    b = oenc.attention(q, k, v2, 4)
    np.testing.assert_array_equal(a[:, :16], b[:, :16])
    assert np.abs(a[:, 16:32] - b[:, 16:32]).max() > 1.0


# ---------------------------------------------------------------- invariants

def test_permutation_equivariance_without_positions():
    """Zero position embeddings: the encoder is permutation-equivariant over tokens
    (bidirectional, no causal mask) and the mean pool is permutation-invariant."""
    cfg = small_cfg()
    W = inputs.make_weights(cfg, seed=3, calibrated=False)
    W["embeddings.position_embeddings.weight"] = np.zeros_like(W["embeddings.position_embeddings.weight"])
    rng = np.random.default_rng(6)
    tok = rng.integers(1000, 30000, 23)
    perm = rng.permutation(23)
    h = oenc.encode(tok, W, cfg)
    hp = oenc.encode(tok[perm], W, cfg)
    np.testing.assert_allclose(hp, h[perm], rtol=0, atol=1e-12)
    np.testing.assert_allclose(ohead.pool(hp, ohead.POOL_MEAN), ohead.pool(h, ohead.POOL_MEAN), atol=1e-13)


def test_positions_matter():
    """With positions the output depends on token order (guards against dropped Pos[t])."""
    cfg = small_cfg()
    W = inputs.make_weights(cfg, seed=3, calibrated=False)
    tok = np.arange(1000, 1010)
    h = oenc.encode(tok, W, cfg)
    hr = oenc.encode(tok[::-1], W, cfg)
    assert np.abs(hr - h[::-1]).max() > 1e-3


# ---------------------------------------------------------------- library pins

def _hf_model(cfg, W):
    torch = pytest.importorskip("torch")
    transformers = pytest.importorskip("transformers")
    hf_cfg = transformers.BertConfig(
        vocab_size=cfg.vocab_size, hidden_size=cfg.hidden, num_hidden_layers=cfg.num_layers,
        num_attention_heads=cfg.num_heads, intermediate_size=cfg.intermediate,
        hidden_act="gelu", max_position_embeddings=cfg.max_position,
        type_vocab_size=cfg.type_vocab_size, layer_norm_eps=cfg.ln_eps,
        hidden_dropout_prob=0.0, attention_probs_dropout_prob=0.0)
    hf_cfg._attn_implementation = "eager"
    m = transformers.BertModel(hf_cfg, add_pooling_layer=False).double().eval()
    sd = {k: torch.from_numpy(np.asarray(v, dtype=np.float64)) for k, v in W.items()
          if not k.startswith("head.")}
    missing, unexpected = m.load_state_dict(sd, strict=False)
    assert not unexpected
    assert all("position_ids" in k or "token_type_ids" in k for k in missing), missing
    return m


@pytest.mark.parametrize("cfgname", ["tiny", "odd"])
def test_encoder_matches_hf_bert_fp64(cfgname):
    """Whole encoder (embedding, 2 post-LN blocks) == HF BertModel fp64, same weights."""
    torch = pytest.importorskip("torch")
    cfg = TINY if cfgname == "tiny" else small_cfg(hidden=96, num_heads=3, intermediate=200, num_layers=3)
    W = inputs.make_weights(cfg, seed=1, calibrated=False)
    m = _hf_model(cfg, W)
    rng = np.random.default_rng(7)
    for L in (1, 2, 31, 64, 130):
        tok = rng.integers(1000, cfg.vocab_size, L)
        tok[0] = inputs.CLS_ID
        ours = oenc.encode(tok, W, cfg)
        with torch.no_grad():
            ref = m(input_ids=torch.from_numpy(tok[None].astype(np.int64)),
                    token_type_ids=torch.zeros(1, L, dtype=torch.long)).last_hidden_state[0].numpy()
        assert np.abs(ours - ref).max() < 1e-10, (L, np.abs(ours - ref).max())


def test_padding_invariance_vs_hf_padded_batch():
    """Varlen encoding == padded batch with a key mask (BASELINE.json: 'padding
    invariance of the varlen encoding'); the oracle encodes each request alone."""
    torch = pytest.importorskip("torch")
    cfg = TINY
    W = inputs.make_weights(cfg, seed=2, calibrated=False)
    m = _hf_model(cfg, W)
    lengths = np.array([5, 64, 1, 33, 17], dtype=np.int32)
    tok = inputs.make_tokens(lengths, seed=5)
    ours = oenc.encode_packed(tok, lengths, W, cfg)
    Lmax = int(lengths.max())
    ids = np.zeros((len(lengths), Lmax), dtype=np.int64)
    mask = np.zeros((len(lengths), Lmax), dtype=np.int64)
    starts = inputs.offsets(lengths)
    for i, L in enumerate(lengths):
        ids[i, :L] = tok[starts[i]:starts[i + 1]]
        mask[i, :L] = 1
    with torch.no_grad():
        ref = m(input_ids=torch.from_numpy(ids), attention_mask=torch.from_numpy(mask),
                token_type_ids=torch.zeros_like(torch.from_numpy(ids))).last_hidden_state.numpy()
    for i, L in enumerate(lengths):
        assert np.abs(ours[i] - ref[i, :L]).max() < 1e-10
    # and packing order does not matter: encoding a sub-batch gives the same rows
    sub = oenc.encode_packed(tok, lengths, W, cfg, requests=[3])
    np.testing.assert_array_equal(sub[0], ours[3])


@pytest.mark.parametrize("pooling", [ohead.POOL_MEAN, ohead.POOL_CLS])
def test_head_matches_torch_sequential(pooling):
    """Pool + 8 FC (ReLU after the first 7) == torch.nn.Sequential fp64 with the same weights."""
    torch = pytest.importorskip("torch")
    cfg = inputs.EncoderConfig(**{**TINY.to_dict(), "pooling": pooling})
    W = inputs.make_weights(cfg, seed=4, calibrated=True)
    rng = np.random.default_rng(8)
    h = rng.normal(size=(29, cfg.hidden))
    layers = []
    dims = [cfg.hidden] + [cfg.head_hidden] * (cfg.head_layers - 1) + [1]
    for j in range(cfg.head_layers):
        lin = torch.nn.Linear(dims[j], dims[j + 1]).double()
        with torch.no_grad():
            lin.weight.copy_(torch.from_numpy(np.asarray(W[f"head.fc{j + 1}.weight"], np.float64)))
            lin.bias.copy_(torch.from_numpy(np.asarray(W[f"head.fc{j + 1}.bias"], np.float64)))
        layers.append(lin)
        if j < cfg.head_layers - 1:
            layers.append(torch.nn.ReLU())
    seq = torch.nn.Sequential(*layers)
    ht = torch.from_numpy(h)
    p_ref = ht.mean(dim=0) if pooling == ohead.POOL_MEAN else ht[0]
    with torch.no_grad():
        y_ref = float(seq(p_ref[None])[0, 0])
    y = ohead.head(ohead.pool(h, pooling), W, cfg)
    assert abs(y - y_ref) <= 1e-10 * max(1.0, abs(y_ref))


def test_mean_pool_is_arithmetic_mean_and_cls_is_row0():
    h = np.arange(12.0).reshape(4, 3)
    np.testing.assert_array_equal(ohead.pool(h, ohead.POOL_MEAN), [4.5, 5.5, 6.5])
    np.testing.assert_array_equal(ohead.pool(h, ohead.POOL_CLS), [0.0, 1.0, 2.0])


def test_predict_batch_independence():
    """pred_i does not depend on the other requests of the batch."""
    cfg = TINY
    W = inputs.make_weights(cfg, seed=0)
    lengths = np.array([40, 12, 64], dtype=np.int32)
    tok = inputs.make_tokens(lengths, seed=9)
    all3 = ohead.predict(tok, lengths, W, cfg)
    starts = inputs.offsets(lengths)
    alone = ohead.predict(tok[starts[1]:starts[2]], lengths[1:2], W, cfg)
    assert all3[1] == alone[0]
