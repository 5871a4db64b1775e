"""ISRTF / FCFS select on the B200 (key pack + radix top-k + preempt flags): bit-exact
against oracle/select.py on identical fp32 predictions -- random, tie-heavy, zeros,
negatives, -0, NaN, +inf, empty slots, caps {1, n-1, n, n+3, 4096}, preempt on/off."""
import numpy as np
import pytest

from paper_2505_09142_b200 import inputs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def predictors(cuda_lib):
    from paper_2505_09142_b200 import binding
    cfg = inputs.CONFIGS["tiny"]
    flat = inputs.flatten_weights(cfg, inputs.make_weights(cfg, seed=0))
    p0 = binding.Predictor(cfg, flat, 1024, 1024)
    p1 = binding.Predictor(cfg, flat, 1024, 1024, head_predicts_total=True)
    yield {False: p0, True: p1}
    p0.close()
    p1.close()


def gpu_select(P, pred, gen, cap, policy, allow, order, running):
    n = len(pred)
    ids = torch.full((cap,), -7, dtype=torch.int32, device="cuda")
    pre = torch.full((max(n, 1),), 9, dtype=torch.uint8, device="cuda")
    cnt = torch.full((1,), -7, dtype=torch.int32, device="cuda")
    nan = torch.full((1,), -7, dtype=torch.int32, device="cuda")
    P.isrtf_select(torch.from_numpy(pred).cuda(), torch.from_numpy(gen).cuda(), cap, ids, policy=policy,
                   allow_preempt=allow, order=None if order is None else torch.from_numpy(order).cuda(),
                   running=None if running is None else torch.from_numpy(running).cuda(), out_preempted=pre,
                   out_count=cnt, out_nan_count=nan)
    torch.cuda.synchronize()
    return ids.cpu().numpy(), int(cnt.item()), pre.cpu().numpy()[:n], int(nan.item())


CASES = []
for seed in range(24):
    rng = np.random.default_rng(seed)
    n = int(rng.choice([1, 2, 5, 16, 100, 256, 1000, 4096, 20000, 65536]))
    cap = int(rng.choice([1, max(1, n - 1), n, n + 3, 4, 64, 256, 1024, 4096]))
    CASES.append((seed, n, min(cap, 4096)))


@pytest.mark.parametrize("seed,n,cap", CASES)
def test_select_bit_exact(predictors, seed, n, cap):
    from oracle.select import isrtf_select
    rng = np.random.default_rng(seed)
    policy = int(rng.integers(0, 2))
    allow = bool(rng.integers(0, 2))
    hpt = bool(rng.integers(0, 2))
    pred = inputs.random_predictions(n, seed=seed, kind="mixed" if seed % 3 else "spread")
    gen, order, running = inputs.random_sched_state(n, seed=seed)
    use_order = order if seed % 2 else None
    ids, cnt, pre, nan = gpu_select(predictors[hpt], pred, gen, cap, policy, allow, use_order, running)
    o_ids, o_cnt, o_pre, o_nan = isrtf_select(pred, gen, cap, policy, allow, use_order, running, hpt)
    np.testing.assert_array_equal(ids, o_ids)
    assert cnt == o_cnt
    np.testing.assert_array_equal(pre, o_pre)
    if policy == 0:
        assert nan == o_nan


def test_select_all_ties_and_empty(predictors):
    from oracle.select import isrtf_select
    P = predictors[False]
    n = 5000
    pred = np.full(n, 42.0, np.float32)          # every key ties: order decides
    gen = np.zeros(n, np.int32)
    order = np.random.default_rng(0).permutation(n).astype(np.uint32)
    ids, cnt, _, _ = gpu_select(P, pred, gen, 300, 0, True, order, None)
    o_ids, _, _, _ = isrtf_select(pred, gen, 300, order=order)
    np.testing.assert_array_equal(ids, o_ids)
    gen[:] = -1                                  # no eligible slot: EmptyBuffer no-op
    ids, cnt, _, _ = gpu_select(P, pred, gen, 8, 0, True, None, None)
    assert cnt == 0 and (ids == -1).all()


def test_select_spec_vectors(predictors):
    P = predictors[False]
    ids, _, _, _ = gpu_select(P, np.float32([30, 200, 10]), np.zeros(3, np.int32), 3, 0, True, None, None)
    assert list(ids) == [2, 0, 1]
    ids, _, _, _ = gpu_select(P, np.float32([200, 10, 400, 30]), np.zeros(4, np.int32), 2, 0, True, None, None)
    assert list(ids) == [1, 3]
    ids, cnt, _, _ = gpu_select(P, np.float32([5]), np.zeros(1, np.int32), 4, 0, True, None, None)
    assert list(ids) == [0, -1, -1, -1] and cnt == 1
