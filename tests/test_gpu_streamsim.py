"""Closed-loop stream simulator with the GPU hot path in the loop (SURVEY.md f1,
BASELINE.json configs[3]) replayed through the fp64 oracle simulator: given the same
priorities, every scheduling decision -- hence every first-execution and finish time -- must be
identical (bit-exact selects + the same window rules, Alg. 1)."""
import numpy as np
import pytest

from paper_2505_09142_b200 import inputs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def tiny_predictor(cuda_lib):
    from paper_2505_09142_b200 import binding
    cfg = inputs.CONFIGS["tiny"]
    P = binding.Predictor(cfg, inputs.flatten_weights(cfg, inputs.make_weights(cfg, seed=0)), 64 * 512, 64)
    yield P
    P.close()


def make_stream(n, mult, seed):
    prompts, totals = inputs.stream_requests(n, seed=seed)
    totals = np.minimum(totals, 400)   # keep the test short
    tpot = 0.95 * inputs.MODEL_AVG_LATENCY_MS["lam13"] / float(totals.mean())
    rate = mult * inputs.average_request_rate(inputs.MODEL_AVG_LATENCY_MS["lam13"], 4)
    arr = inputs.arrival_times_ms(n, rate, alpha=1.0, seed=seed)
    return prompts, totals, arr, 0.05 * inputs.MODEL_AVG_LATENCY_MS["lam13"], tpot


def replay(totals, arr, policy, cap, ttft, tpot, allow, priority, workers=1, **starv):
    from oracle import scheduler, sim
    jobs = [sim.SimJob(i, float(arr[i]), int(totals[i])) for i in range(len(totals))]
    if workers == 1 and not starv:
        r = sim.simulate(jobs, policy, cap=cap, K=50, ttft=ttft, tpot=tpot, allow_preempt=allow, priority=priority)
    else:
        r = scheduler.simulate_nodes(jobs, workers, policy, cap=cap, K=50, ttft=ttft, tpot=tpot,
                                     allow_preempt=allow, priority=priority, **starv)
    return np.array([r[i][0] for i in range(len(jobs))]), np.array([r[i][1] for i in range(len(jobs))])


@pytest.mark.parametrize("source,policy,allow", [("gpu", 0, True), ("oracle", 0, True), ("gpu", 0, False),
                                                 ("none", 1, True), ("sjf", 0, False)])
def test_stream_sim_matches_oracle_replay(tiny_predictor, source, policy, allow):
    from oracle import sim
    from paper_2505_09142_b200.streamsim import StreamSim
    prompts, totals, arr, ttft, tpot = make_stream(120, 3.0, seed=1)
    S = StreamSim(tiny_predictor, policy=policy, cap=4, ttft_ms=ttft, tpot_ms=tpot, allow_preempt=allow,
                  priority=source if source != "none" else "gpu")
    res = S.run(prompts, totals, arr)
    assert np.isfinite(res.finish).all() and (res.finish >= res.first).all()
    if source == "gpu" and policy == 0:
        prio = lambda job, g: res.recorded[(job.id, g)]
    elif source == "sjf":
        prio = lambda job, g: float(np.float32(job.total))   # the profiled total length
    else:
        prio = sim.oracle_remaining
    first, finish = replay(totals, arr, policy, 4, ttft, tpot, allow, prio)
    np.testing.assert_array_equal(res.first, first)
    np.testing.assert_array_equal(res.finish, finish)


def test_srtf_beats_fcfs_on_the_stream(tiny_predictor):
    """With true remaining as priority (SRTF bound) mean JCT is below FCFS."""
    from paper_2505_09142_b200.streamsim import StreamSim
    prompts, totals, arr, ttft, tpot = make_stream(150, 5.0, seed=2)
    f = StreamSim(tiny_predictor, policy=1, cap=4, ttft_ms=ttft, tpot_ms=tpot).run(prompts, totals, arr)
    s = StreamSim(tiny_predictor, policy=0, cap=4, ttft_ms=ttft, tpot_ms=tpot, priority="oracle").run(
        prompts, totals, arr)
    assert s.jct.mean() < f.jct.mean()


@pytest.mark.parametrize("workers,source,starv", [
    (3, "gpu", {}), (3, "oracle", {}), (8, "gpu", {"boost_after": 2, "boost_amount": 40.0}),
    (1, "gpu", {"boost_after": 1, "boost_amount": 25.0, "preempt_margin": 10.0}),
    (4, "oracle", {"preempt_margin": 30.0})])
def test_multi_worker_stream_matches_oracle_replay(tiny_predictor, workers, source, starv):
    """Per-node Priority Buffers + least-loaded balancer + starvation control on the GPU
     replayed through oracle/scheduler.simulate_nodes."""
    from oracle import sim
    from paper_2505_09142_b200.streamsim import StreamSim
    prompts, totals, arr, ttft, tpot = make_stream(160, 3.0 * workers, seed=3 + workers)
    S = StreamSim(tiny_predictor, policy=0, cap=4, ttft_ms=ttft, tpot_ms=tpot, priority=source,
                  workers=workers, **starv)
    res = S.run(prompts, totals, arr)
    assert np.isfinite(res.finish).all() and (res.finish >= res.first).all()
    prio = (lambda job, g: res.recorded[(job.id, g)]) if source == "gpu" else sim.oracle_remaining
    first, finish = replay(totals, arr, 0, 4, ttft, tpot, True, prio, workers, **starv)
    np.testing.assert_array_equal(res.first, first)
    np.testing.assert_array_equal(res.finish, finish)


def test_fcfs_multi_worker_matches_oracle(tiny_predictor):
    from oracle import sim
    from paper_2505_09142_b200.streamsim import StreamSim
    prompts, totals, arr, ttft, tpot = make_stream(140, 6.0, seed=11)
    res = StreamSim(tiny_predictor, policy=1, cap=2, ttft_ms=ttft, tpot_ms=tpot, workers=5).run(prompts, totals, arr)
    first, finish = replay(totals, arr, 1, 2, ttft, tpot, True, sim.oracle_remaining, 5)
    np.testing.assert_array_equal(res.first, first)
    np.testing.assert_array_equal(res.finish, finish)


def test_token_arena_path_equals_host_sequences(tiny_predictor):
    """The device-resident token arena (prompts uploaded once, generated tokens appended per window,
    due set gathered on the device) feeds the predictor exactly the sequences the host path builds:
    every recorded priority is bitwise equal."""
    from paper_2505_09142_b200.streamsim import StreamSim
    prompts, totals, arr, ttft, tpot = make_stream(150, 3.0, seed=4)
    runs = [StreamSim(tiny_predictor, cap=4, ttft_ms=ttft, tpot_ms=tpot, arena=a).run(prompts, totals, arr)
            for a in (True, False)]
    assert runs[0].recorded == runs[1].recorded
    np.testing.assert_array_equal(runs[0].finish, runs[1].finish)
