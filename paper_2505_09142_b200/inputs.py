"""Seeded synthetic inputs shared by the CUDA path, the oracle and the bench.

This module holds NO arithmetic of the method (no encoder, head, key packing or
selection).  It only draws random numbers in the shapes the paper's workload has
and lays them out in the canonical order both sides consume.  It is the one
module the oracle and the product path share.

Shapes follow PAPER.md:
  * encoder = BGE (BAAI/bge-base-en-v1.5), a BERT-base encoder, 768-d
    (Sec. 3.1); BGE-large / tiny sizes come from BASELINE.json configs.
  * head = "eight FC layers", ReLU, hidden 1024 (Sec. 4.2).
  * a request's input is "the prompt attached with the answer" and is
    re-encoded after every 50-token window.

Weights are random (no checkpoint is available offline).  Encoder values are
rounded to bf16-representable fp32 so both sides consume identical numbers;
head values are plain fp32.
"""
from __future__ import annotations

import json
import os
from dataclasses import dataclass, asdict

import numpy as np

MASTER_SEED = 250509142
SUB_WEIGHTS, SUB_TOKENS, SUB_LENGTHS, SUB_ARRIVALS, SUB_OUTPUTS, SUB_PRED = 0, 1, 2, 3, 4, 5

VOCAB = 30522
MAX_POSITION = 512
TYPE_VOCAB = 2
LN_EPS = 1e-12
CLS_ID = 101
SEP_ID = 102
HEAD_LAYERS = 8
HEAD_HIDDEN = 1024
WINDOW_K = 50  # P:175 "optimal window size is 50 tokens"

POOL_MEAN = 0
POOL_CLS = 1


@dataclass(frozen=True)
class EncoderConfig:
    name: str
    num_layers: int
    hidden: int
    num_heads: int
    intermediate: int
    vocab_size: int = VOCAB
    max_position: int = MAX_POSITION
    type_vocab_size: int = TYPE_VOCAB
    ln_eps: float = LN_EPS
    head_layers: int = HEAD_LAYERS
    head_hidden: int = HEAD_HIDDEN
    pooling: int = POOL_MEAN

    @property
    def head_dim(self) -> int:
        return self.hidden // self.num_heads

    def to_dict(self):
        return asdict(self)


CONFIGS = {
    # BASELINE.json configs[0]
    "tiny": EncoderConfig("tiny", 2, 128, 4, 512),
    # BGE-base = BERT-base -- BASELINE.json configs[1], [3], [4]
    "base": EncoderConfig("base", 12, 768, 12, 3072),
    # BGE-large -- BASELINE.json configs[2]
    "large": EncoderConfig("large", 24, 1024, 16, 4096),
}


def _rng(*sub: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([MASTER_SEED, *sub])))


def round_to_bf16(x: np.ndarray) -> np.ndarray:
    """Round fp32 values to the nearest bf16-representable fp32 (ties to even).

    Data preparation only: makes the encoder weights exactly representable in
    the bf16 operands the GPU path uses, so both sides see identical numbers."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).reshape(x.shape)


def weight_shapes(cfg: EncoderConfig):
    """Canonical order: HF BertModel state_dict order (no pooler), then head fc1..fc8."""
    H, F = cfg.hidden, cfg.intermediate
    s = [
        ("embeddings.word_embeddings.weight", (cfg.vocab_size, H)),
        ("embeddings.position_embeddings.weight", (cfg.max_position, H)),
        ("embeddings.token_type_embeddings.weight", (cfg.type_vocab_size, H)),
        ("embeddings.LayerNorm.weight", (H,)),
        ("embeddings.LayerNorm.bias", (H,)),
    ]
    for l in range(cfg.num_layers):
        p = f"encoder.layer.{l}."
        s += [
            (p + "attention.self.query.weight", (H, H)),
            (p + "attention.self.query.bias", (H,)),
            (p + "attention.self.key.weight", (H, H)),
            (p + "attention.self.key.bias", (H,)),
            (p + "attention.self.value.weight", (H, H)),
            (p + "attention.self.value.bias", (H,)),
            (p + "attention.output.dense.weight", (H, H)),
            (p + "attention.output.dense.bias", (H,)),
            (p + "attention.output.LayerNorm.weight", (H,)),
            (p + "attention.output.LayerNorm.bias", (H,)),
            (p + "intermediate.dense.weight", (F, H)),
            (p + "intermediate.dense.bias", (F,)),
            (p + "output.dense.weight", (H, F)),
            (p + "output.dense.bias", (H,)),
            (p + "output.LayerNorm.weight", (H,)),
            (p + "output.LayerNorm.bias", (H,)),
        ]
    dims = [H] + [cfg.head_hidden] * (cfg.head_layers - 1) + [1]
    for j in range(cfg.head_layers):
        s += [(f"head.fc{j + 1}.weight", (dims[j + 1], dims[j])),
              (f"head.fc{j + 1}.bias", (dims[j + 1],))]
    return s


def weight_count(cfg: EncoderConfig) -> int:
    return int(sum(int(np.prod(shape)) for _, shape in weight_shapes(cfg)))


_CALIB_PATH = os.path.join(os.path.dirname(__file__), "head_calibration.json")


def head_calibration(cfg: EncoderConfig):
    """(scale, offset) for the last head layer, written by oracle/calibrate_head.py.

    Random-init predictions sit near 0 and would clamp to ties; the committed
    calibration scales the final layer so predictions spread around 256 +- 64
    tokens (SURVEY.md Sec. 8c "Head calibration").  Missing entry -> (1, 0)."""
    try:
        with open(_CALIB_PATH) as f:
            table = json.load(f)
    except FileNotFoundError:
        return 1.0, 0.0
    key = f"{cfg.name}/pool{cfg.pooling}"
    if key not in table:
        return 1.0, 0.0
    return float(table[key]["scale"]), float(table[key]["offset"])


def make_weights(cfg: EncoderConfig, seed: int = 0, calibrated: bool = True) -> dict:
    """Random-init weights (HF BERT init: N(0, 0.02); LN gamma 1 + U(+-0.1), beta N(0, 0.02);
    head: He-normal, zero bias).  Encoder values bf16-representable, head plain fp32."""
    rng = _rng(SUB_WEIGHTS, seed)
    out = {}
    for name, shape in weight_shapes(cfg):
        if name.startswith("head."):
            if name.endswith("weight"):
                fan_in = shape[1]
                w = rng.standard_normal(shape) * np.sqrt(2.0 / fan_in)
            else:
                w = np.zeros(shape)
            out[name] = w.astype(np.float32)
            continue
        if "LayerNorm.weight" in name:
            w = 1.0 + rng.uniform(-0.1, 0.1, size=shape)
        else:
            w = rng.standard_normal(shape) * 0.02
        out[name] = round_to_bf16(w.astype(np.float32))
    if calibrated:
        scale, offset = head_calibration(cfg)
        last = f"head.fc{cfg.head_layers}."
        out[last + "weight"] = (out[last + "weight"] * np.float32(scale)).astype(np.float32)
        out[last + "bias"] = (out[last + "bias"] + np.float32(offset)).astype(np.float32)
    return out


def flatten_weights(cfg: EncoderConfig, w: dict) -> np.ndarray:
    parts = []
    for name, shape in weight_shapes(cfg):
        a = np.asarray(w[name], dtype=np.float32)
        assert a.shape == tuple(shape), (name, a.shape, shape)
        parts.append(a.reshape(-1))
    return np.ascontiguousarray(np.concatenate(parts), dtype=np.float32)


def unflatten_weights(cfg: EncoderConfig, flat: np.ndarray) -> dict:
    out, off = {}, 0
    for name, shape in weight_shapes(cfg):
        n = int(np.prod(shape))
        out[name] = flat[off:off + n].reshape(shape)
        off += n
    assert off == flat.size
    return out


# ----------------------------------------------------------------------------- requests

def trace_lengths(n: int, seed: int = 0):
    """Trace-shaped (prompt + partial response) lengths and tokens generated so far.

    prompt p ~ round(LogNormal(ln 48, 1.0)) clipped [4, 384]; total response
    r ~ round(LogNormal(ln 180, 0.8)) clipped [1, 1536]; generated g is a multiple
    of the 50-token window (re-predicts happen at window boundaries);
    L = clip(2 + p + g, 32, 512) ([CLS] + prompt + [SEP] + response so far).
    Returns (lengths int32 [n], generated int32 [n], total_response int32 [n])."""
    rng = _rng(SUB_LENGTHS, seed)
    p = np.clip(np.rint(rng.lognormal(np.log(48.0), 1.0, n)), 4, 384).astype(np.int64)
    r = np.clip(np.rint(rng.lognormal(np.log(180.0), 0.8, n)), 1, 1536).astype(np.int64)
    g = WINDOW_K * np.floor(rng.uniform(0.0, 1.0, n) * r / WINDOW_K).astype(np.int64)
    L = np.clip(2 + p + g, 32, MAX_POSITION)
    return L.astype(np.int32), g.astype(np.int32), r.astype(np.int32)


def uniform_lengths(n: int, lo: int = 32, hi: int = 512, seed: int = 0):
    rng = _rng(SUB_LENGTHS, 1000 + seed)
    return rng.integers(lo, hi + 1, n).astype(np.int32)


def make_tokens(lengths: np.ndarray, seed: int = 0) -> np.ndarray:
    """Packed token ids [sum(lengths)]: [CLS] first, [SEP] last, the rest uniform in
    [1000, 30521] (avoids BERT special ids)."""
    rng = _rng(SUB_TOKENS, seed)
    lengths = np.asarray(lengths, dtype=np.int64)
    T = int(lengths.sum())
    tok = rng.integers(1000, VOCAB, T).astype(np.int32)
    starts = np.concatenate([[0], np.cumsum(lengths)[:-1]]).astype(np.int64)
    if T:
        tok[starts] = CLS_ID
        ends = starts + lengths - 1
        multi = lengths > 1
        tok[ends[multi]] = SEP_ID
    return tok


def offsets(lengths: np.ndarray) -> np.ndarray:
    """Start of each request in the packed token array (data layout, not method)."""
    lengths = np.asarray(lengths, dtype=np.int64)
    return np.concatenate([[0], np.cumsum(lengths)]).astype(np.int64)


def random_predictions(n: int, seed: int = 0, kind: str = "mixed") -> np.ndarray:
    """fp32 'predictions' for select-only tests: heavy ties, zeros, negatives, -0, NaN, inf."""
    rng = _rng(SUB_PRED, seed)
    if kind == "spread":
        return rng.normal(256.0, 64.0, n).astype(np.float32)
    v = rng.normal(120.0, 80.0, n).astype(np.float32)
    r = rng.uniform(0, 1, n)
    v[r < 0.30] = np.rint(v[r < 0.30] / 16.0) * 16.0          # ties
    v[(r >= 0.30) & (r < 0.35)] = 0.0
    v[(r >= 0.35) & (r < 0.38)] = -0.0
    v[(r >= 0.38) & (r < 0.42)] = -np.abs(v[(r >= 0.38) & (r < 0.42)])
    v[(r >= 0.42) & (r < 0.44)] = np.nan
    v[(r >= 0.44) & (r < 0.45)] = np.inf
    return v.astype(np.float32)


# ----------------------------------------------------------------------------- request streams

# Average LLM latencies over 500 prompts on A100 (ms), PAPER.md tab:ml-models.
MODEL_AVG_LATENCY_MS = {"opt6.7": 1315.5, "opt13": 2643.2, "lam7": 6522.2, "lam13": 8610.2, "vic": 2964.9}
GAMMA_ALPHA, GAMMA_BETA_S = 0.73, 10.41  # FabriX inter-arrival fit


def average_request_rate(avg_latency_ms: float, batch_size: int) -> float:
    """Requests/s that keep a backend of `batch_size` busy: (1000 / avg latency) x batch size
    (P:481, P:492 -- the formula's braces are garbled in the source; R17)."""
    return 1000.0 / avg_latency_ms * batch_size


def arrival_times_ms(n: int, rate_per_s: float, alpha: float = 1.0, seed: int = 0) -> np.ndarray:
    """Cumulative arrival times (ms) with Gamma(alpha, 1 / (alpha * rate)) inter-arrivals:
    alpha = 1 is a Poisson process (BASELINE.json configs[3]); alpha = 0.73 is the FabriX shape
     rescaled to the requested mean rate."""
    rng = _rng(SUB_ARRIVALS, 7000 + seed)
    gaps_s = rng.gamma(alpha, 1.0 / (alpha * rate_per_s), n)
    return np.cumsum(gaps_s) * 1000.0


def stream_requests(n: int, seed: int = 0):
    """n synthetic requests: prompt token ids ([CLS] + prompt + [SEP]) and true total output
    lengths (trace-shaped: prompt ~ LogNormal(ln 48, 1), response ~ LogNormal(ln 180, 0.8)).
    Returns (list of int32 prompt arrays, int32 total outputs)."""
    rng = _rng(SUB_OUTPUTS, seed)
    p = np.clip(np.rint(rng.lognormal(np.log(48.0), 1.0, n)), 4, 384).astype(np.int64)
    r = np.clip(np.rint(rng.lognormal(np.log(180.0), 0.8, n)), 1, 1536).astype(np.int32)
    prompts = []
    for i in range(n):
        t = rng.integers(1000, VOCAB, p[i] + 2).astype(np.int32)
        t[0], t[-1] = CLS_ID, SEP_ID
        prompts.append(t)
    return prompts, r


def response_tokens(job_id: int, total: int, seed: int = 0) -> np.ndarray:
    """The (synthetic) tokens the served LLM generates for job `job_id`."""
    rng = _rng(SUB_OUTPUTS, 100000 + seed, job_id)
    return rng.integers(1000, VOCAB, total).astype(np.int32)


NOISY_MAE_SCHEDULE = (19.9, 16.0, 12.5, 9.5, 7.0, 5.0)  # SPEC S:209 (tokens; anchored at P:359's MAE 19.923)


def noisy_remaining(job_id: int, total: int, generated: int, seed: int = 0,
                    mae_schedule=NOISY_MAE_SCHEDULE, window: int = WINDOW_K) -> float:
    """NoisyIterative priority source: max(0, total + e - generated) with
    e ~ Laplace(scale = mae_schedule[min(step, last)]), step = generated // window, seeded per
    (job id, step) so a replay is independent of scheduling order.  A stand-in for the trained
    predictor's error (its weights are not available): the draw is an input, not method arithmetic."""
    step = generated // window
    scale = mae_schedule[min(step, len(mae_schedule) - 1)]
    e = _rng(SUB_PRED, 200000 + seed, job_id, step).laplace(0.0, scale)
    return max(0.0, float(total) + float(e) - float(generated))


def random_sched_state(n: int, seed: int = 0, frac_running: float = 0.05, frac_empty: float = 0.05):
    """generated (int32, <0 = empty slot), order (unique uint32 rank of (arrival, id)),
    running (uint8) for select tests."""
    rng = _rng(SUB_ARRIVALS, seed)
    gen = (WINDOW_K * rng.integers(0, 20, n)).astype(np.int32)
    gen[rng.uniform(0, 1, n) < frac_empty] = -1
    order = rng.permutation(n).astype(np.uint32)
    running = (rng.uniform(0, 1, n) < frac_running).astype(np.uint8)
    running[gen < 0] = 0
    return gen, order, running
