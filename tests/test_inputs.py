"""The synthetic workload generators against the numbers the paper prints."""
import numpy as np

from paper_2505_09142_b200 import inputs


def test_gamma_interarrivals_match_fabrix_fit():
    """Gamma(alpha = 0.73, beta = 10.41 s): mean alpha*beta = 7.5993 s, variance
    alpha*beta^2 = 79.11 s^2.  arrival_times_ms parametrises by rate: 1 / 7.5993 s."""
    a, b = inputs.GAMMA_ALPHA, inputs.GAMMA_BETA_S
    t = inputs.arrival_times_ms(400000, rate_per_s=1.0 / (a * b), alpha=a, seed=3)
    gaps = np.diff(np.concatenate([[0.0], t])) / 1000.0
    assert abs(gaps.mean() - 7.5993) / 7.5993 < 0.01
    assert abs(gaps.var() - 79.11) / 79.11 < 0.03


def test_poisson_rate():
    t = inputs.arrival_times_ms(200000, rate_per_s=0.4646, alpha=1.0, seed=4)
    gaps = np.diff(np.concatenate([[0.0], t])) / 1000.0
    assert abs(gaps.mean() - 1 / 0.4646) / (1 / 0.4646) < 0.01
    assert abs(gaps.std() / gaps.mean() - 1.0) < 0.01     # exponential: CV = 1


def test_average_request_rate_formula():
    """(1000 / avg latency ms) x batch: lam13 (8,610.2 ms) at batch 4 is
    0.4646 req/s; 120 / 8.61 = 13.9 req/s at batch 120."""
    assert round(inputs.average_request_rate(8610.2, 4), 4) == 0.4646
    assert round(inputs.average_request_rate(8610.0, 120), 1) == 13.9


def test_trace_lengths_shape():
    L, g, r = inputs.trace_lengths(20000, seed=0)
    assert L.min() >= 32 and L.max() <= 512
    assert (g % inputs.WINDOW_K == 0).all() and (g <= r).all()
    assert 150 < L.mean() < 190          # mean 169.9


def test_tokens_layout():
    L = np.array([1, 5, 3], np.int32)
    t = inputs.make_tokens(L, seed=0)
    assert t.size == 9 and t[0] == inputs.CLS_ID and t[1] == inputs.CLS_ID and t[5] == inputs.SEP_ID
    assert t[6] == inputs.CLS_ID and t[8] == inputs.SEP_ID


def test_weights_bf16_representable_and_count():
    cfg = inputs.CONFIGS["tiny"]
    W = inputs.make_weights(cfg, seed=0)
    flat = inputs.flatten_weights(cfg, W)
    assert flat.size == inputs.weight_count(cfg)
    enc = flat[: flat.size - sum(int(np.prod(s)) for n, s in inputs.weight_shapes(cfg) if n.startswith("head."))]
    np.testing.assert_array_equal(inputs.round_to_bf16(enc), enc)


def test_noisy_remaining_spec():
    """max(0, total + e - generated), e ~ Laplace(MAE of the step), seeded
    per (job, step): deterministic, error MAE per step equals the schedule (Laplace mean absolute
    deviation = scale), non-increasing with the step."""
    a = inputs.noisy_remaining(7, 120, 100, seed=3)
    assert a == inputs.noisy_remaining(7, 120, 100, seed=3) and a >= 0.0
    maes = []
    for step in range(7):
        g = 50 * step
        err = np.array([inputs.noisy_remaining(j, 100000, g) - (100000 - g) for j in range(4000)])
        maes.append(np.abs(err).mean())
        want = inputs.NOISY_MAE_SCHEDULE[min(step, 5)]
        assert abs(maes[-1] - want) < 0.06 * want
    assert all(maes[i + 1] <= maes[i] * 1.05 for i in range(6))
    assert inputs.noisy_remaining(1, 10, 10) >= 0.0
