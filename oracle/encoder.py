"""Oracle: BGE/BERT bidirectional encoder forward in fp64, one request at a time.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Follows PAPER.md Sec. 3.1 / 4.2: the predictor's encoder is "BGE
(BAAI/bge-base-en-v1.5)" producing "768-dimensional embeddings"
(P:123); the paper gives no internals, so the BERT-base conventions of
DESIGN.md reading R1 are written out step by step below (post-LN blocks,
erf-GELU, LayerNorm eps 1e-12 inside the square root, learned absolute
positions restarting at 0 for every request, token type 0).

Each request is encoded independently over its own L_i tokens (the varlen
semantics: no padding, no cross-request attention).  Library primitives used:
numpy matmul and scipy.special.erf.  No blocking, fusion or reordering.
"""
from __future__ import annotations

import numpy as np
from scipy.special import erf


def layer_norm(x: np.ndarray, gamma: np.ndarray, beta: np.ndarray, eps: float) -> np.ndarray:
    """LN(v) = (v - mean(v)) / sqrt(mean((v - mean)^2) + eps) * gamma + beta  (population variance)."""
    x = np.asarray(x, dtype=np.float64)
    mu = x.mean(axis=-1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    return (x - mu) / np.sqrt(var + eps) * np.asarray(gamma, np.float64) + np.asarray(beta, np.float64)


def gelu(z: np.ndarray) -> np.ndarray:
    """GELU(z) = 1/2 z (1 + erf(z / sqrt 2))  (exact, erf form)."""
    return 0.5 * z * (1.0 + erf(z / np.sqrt(2.0)))


def linear(x: np.ndarray, w: np.ndarray, b: np.ndarray) -> np.ndarray:
    """nn.Linear: x W^T + b, weight stored [out, in]."""
    return np.asarray(x, np.float64) @ np.asarray(w, np.float64).T + np.asarray(b, np.float64)


def softmax_rows(s: np.ndarray) -> np.ndarray:
    """Row softmax with the row max subtracted first."""
    m = s.max(axis=-1, keepdims=True)
    e = np.exp(s - m)
    return e / e.sum(axis=-1, keepdims=True)


def attention(q: np.ndarray, k: np.ndarray, v: np.ndarray, num_heads: int) -> np.ndarray:
    """Bidirectional multi-head attention over ONE request's L tokens (no mask).

    q, k, v: [L, H].  For each head h: S = q_h k_h^T / sqrt(d); P = softmax(S);
    ctx_h = P v_h; heads concatenated back to [L, H]."""
    L, H = q.shape
    d = H // num_heads
    ctx = np.empty((L, H), dtype=np.float64)
    for h in range(num_heads):
        sl = slice(h * d, (h + 1) * d)
        s = q[:, sl] @ k[:, sl].T / np.sqrt(d)
        p = softmax_rows(s)
        ctx[:, sl] = p @ v[:, sl]
    return ctx


def embed(tokens: np.ndarray, W: dict, cfg) -> np.ndarray:
    """x_t = Word[tok_t] + Pos[t] + Type[0], t = 0..L-1, then the embedding LayerNorm."""
    tokens = np.asarray(tokens, dtype=np.int64)
    L = tokens.shape[0]
    x = (np.asarray(W["embeddings.word_embeddings.weight"], np.float64)[tokens]
         + np.asarray(W["embeddings.position_embeddings.weight"], np.float64)[:L]
         + np.asarray(W["embeddings.token_type_embeddings.weight"], np.float64)[0])
    return layer_norm(x, W["embeddings.LayerNorm.weight"], W["embeddings.LayerNorm.bias"], cfg.ln_eps)


def encoder_layer(h: np.ndarray, W: dict, l: int, cfg) -> np.ndarray:
    """One post-LN BERT block:
        q, k, v = h Wq^T + bq, h Wk^T + bk, h Wv^T + bv
        h <- LN1(h + Attn(q, k, v) Wo^T + bo)
        h <- LN2(h + GELU(h W1^T + b1) W2^T + b2)"""
    p = f"encoder.layer.{l}."
    q = linear(h, W[p + "attention.self.query.weight"], W[p + "attention.self.query.bias"])
    k = linear(h, W[p + "attention.self.key.weight"], W[p + "attention.self.key.bias"])
    v = linear(h, W[p + "attention.self.value.weight"], W[p + "attention.self.value.bias"])
    ctx = attention(q, k, v, cfg.num_heads)
    a = linear(ctx, W[p + "attention.output.dense.weight"], W[p + "attention.output.dense.bias"])
    h = layer_norm(h + a, W[p + "attention.output.LayerNorm.weight"],
                   W[p + "attention.output.LayerNorm.bias"], cfg.ln_eps)
    g = gelu(linear(h, W[p + "intermediate.dense.weight"], W[p + "intermediate.dense.bias"]))
    f = linear(g, W[p + "output.dense.weight"], W[p + "output.dense.bias"])
    h = layer_norm(h + f, W[p + "output.LayerNorm.weight"], W[p + "output.LayerNorm.bias"], cfg.ln_eps)
    return h


def encode(tokens: np.ndarray, W: dict, cfg) -> np.ndarray:
    """Final hidden states [L, H] (fp64) of one request."""
    h = embed(tokens, W, cfg)
    for l in range(cfg.num_layers):
        h = encoder_layer(h, W, l, cfg)
    return h


def encode_packed(tokens: np.ndarray, lengths: np.ndarray, W: dict, cfg, requests=None):
    """Encode every request of a packed batch independently.

    Returns a list of [L_i, H] fp64 arrays (for the selected ``requests`` if given)."""
    lengths = np.asarray(lengths, dtype=np.int64)
    starts = np.concatenate([[0], np.cumsum(lengths)])
    idx = range(len(lengths)) if requests is None else requests
    return [encode(tokens[starts[i]:starts[i + 1]], W, cfg) for i in idx]
