"""Oracle: the FP8 (E4M3) variant of the encoder forward, fp64.  TEST INFRASTRUCTURE ONLY.

SURVEY.md Sec. 8f row f4(i) ("FP8 E4M3 encoder GEMMs ... looser tolerance"); the quantisation
scheme is DESIGN.md reading R20 (the paper never states a precision, R12):

  * E4M3 (OCP FP8, "fn" variant): 1 sign, 4 exponent bits (bias 7), 3 mantissa bits; finite
    values only, largest 448; subnormals are multiples of 2^-9.  Conversion = round to nearest,
    ties to an even mantissa, saturating to +-448.
  * weights: per output row r, s_r = max|W[r, :]| / 448 (1 for a zero row);
    W~[r, :] = s_r * E4M3(W[r, :] / s_r).
  * activations entering a GEMM (static power-of-two scales a):
        LayerNorm outputs (QKV and FFN1 inputs)  a = 8
        attention outputs (out-projection input) a = 16
        GELU outputs (FFN2 input)                a = 16
    x~ = E4M3(a x) / a.
  * everything else as oracle/encoder.py: attention, residual stream, LayerNorm and the head
    unquantised (the GPU keeps them in bf16 / fp32).

Each block is oracle/encoder.py's post-LN BERT block with x~ / W~ substituted at the four GEMM
inputs, in the same order; no other change.  The E4M3 rounding is written out from the format's
definition (enumerate every finite code, take the nearest, break ties to the even code).
"""
from __future__ import annotations

import numpy as np

from . import encoder, head

E4M3_MAX = 448.0
SCALE_HIDDEN = 8.0    # LayerNorm outputs -> QKV, FFN1
SCALE_CTX = 16.0      # attention outputs -> out-projection
SCALE_GELU = 16.0     # GELU outputs -> FFN2


def e4m3_values() -> np.ndarray:
    """All non-negative finite E4M3 values, indexed by their 7-bit code (exponent << 3 | mantissa);
    code 0x7F is NaN in the fn variant and is excluded."""
    vals = []
    for code in range(0x7F):
        e, m = code >> 3, code & 7
        vals.append(m / 8.0 * 2.0 ** -6 if e == 0 else (1.0 + m / 8.0) * 2.0 ** (e - 7))
    return np.array(vals, dtype=np.float64)


_TABLE = e4m3_values()   # strictly increasing, code order == value order


def round_e4m3(x: np.ndarray) -> np.ndarray:
    """Round to the nearest E4M3 value (ties to the even code), saturating at +-448."""
    x = np.asarray(x, dtype=np.float64)
    a = np.minimum(np.abs(x), E4M3_MAX)
    hi = np.clip(np.searchsorted(_TABLE, a, side="left"), 0, len(_TABLE) - 1)   # first value >= a
    lo = np.maximum(hi - 1, 0)
    d_lo, d_hi = a - _TABLE[lo], _TABLE[hi] - a
    pick_hi = (d_hi < d_lo) | ((d_hi == d_lo) & (hi % 2 == 0))
    r = np.where(pick_hi, _TABLE[hi], _TABLE[lo])
    return np.copysign(r, x)


def quant_act(x: np.ndarray, scale: float) -> np.ndarray:
    """x~ = E4M3(scale x) / scale."""
    return round_e4m3(np.asarray(x, np.float64) * scale) / scale


def quant_weight(w: np.ndarray) -> np.ndarray:
    """Per-output-row scaled E4M3: W~[r] = s_r E4M3(W[r] / s_r), s_r = max|W[r]| / 448."""
    w = np.asarray(w, dtype=np.float64)
    amax = np.abs(w).max(axis=1, keepdims=True)
    s = np.where(amax > 0, amax / E4M3_MAX, 1.0)
    return round_e4m3(w / s) * s


def quantize_weights(W: dict, cfg) -> dict:
    """The weight dict with every encoder GEMM matrix replaced by its W~."""
    Wq = dict(W)
    for l in range(cfg.num_layers):
        p = f"encoder.layer.{l}."
        for n in ("attention.self.query.weight", "attention.self.key.weight", "attention.self.value.weight",
                  "attention.output.dense.weight", "intermediate.dense.weight", "output.dense.weight"):
            Wq[p + n] = quant_weight(W[p + n])
    return Wq


def encoder_layer_fp8(h: np.ndarray, Wq: dict, l: int, cfg) -> np.ndarray:
    """oracle/encoder.py encoder_layer with the quantised GEMM inputs (Wq from quantize_weights)."""
    p = f"encoder.layer.{l}."
    hq = quant_act(h, SCALE_HIDDEN)
    q = encoder.linear(hq, Wq[p + "attention.self.query.weight"], Wq[p + "attention.self.query.bias"])
    k = encoder.linear(hq, Wq[p + "attention.self.key.weight"], Wq[p + "attention.self.key.bias"])
    v = encoder.linear(hq, Wq[p + "attention.self.value.weight"], Wq[p + "attention.self.value.bias"])
    ctx = encoder.attention(q, k, v, cfg.num_heads)
    a = encoder.linear(quant_act(ctx, SCALE_CTX), Wq[p + "attention.output.dense.weight"],
                       Wq[p + "attention.output.dense.bias"])
    h = encoder.layer_norm(h + a, Wq[p + "attention.output.LayerNorm.weight"],
                           Wq[p + "attention.output.LayerNorm.bias"], cfg.ln_eps)
    g = encoder.gelu(encoder.linear(quant_act(h, SCALE_HIDDEN), Wq[p + "intermediate.dense.weight"],
                                    Wq[p + "intermediate.dense.bias"]))
    f = encoder.linear(quant_act(g, SCALE_GELU), Wq[p + "output.dense.weight"], Wq[p + "output.dense.bias"])
    return encoder.layer_norm(h + f, Wq[p + "output.LayerNorm.weight"], Wq[p + "output.LayerNorm.bias"], cfg.ln_eps)


def encode_fp8(tokens: np.ndarray, Wq: dict, cfg) -> np.ndarray:
    h = encoder.embed(tokens, Wq, cfg)
    for l in range(cfg.num_layers):
        h = encoder_layer_fp8(h, Wq, l, cfg)
    return h


def predict_with_hidden_fp8(tokens: np.ndarray, lengths: np.ndarray, W: dict, cfg, requests=None):
    """(predictions fp64 [k], final hidden states list) of the FP8 forward + the fp64 head."""
    Wq = quantize_weights(W, cfg)
    lengths = np.asarray(lengths, dtype=np.int64)
    starts = np.concatenate([[0], np.cumsum(lengths)])
    idx = range(len(lengths)) if requests is None else requests
    hs = [encode_fp8(tokens[starts[i]:starts[i + 1]], Wq, cfg) for i in idx]
    preds = np.array([head.head(head.pool(h, cfg.pooling), W, cfg) for h in hs], dtype=np.float64)
    return preds, hs
