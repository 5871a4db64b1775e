"""The in-flight table path of the north_star workload (BASELINE.json configs[4]; SURVEY.md Sec. 8a
rows a0, a13, 8e): each rank encodes its cost-balanced slice of the due set, and
elis_predict_remaining_dist writes every rank's predictions into every rank's replica of the
table (peer memory: one fused head-output kernel storing over NVLink + epoch flags; or NCCL);
then every rank selects over the whole table.

One B200 runs the protocol for real: several ranks share the device, each with its own predictor,
region and stream, their fused kernels waiting on each other's flags.  Expected values: the
single-GPU elis_predict_remaining of the same requests (bitwise: the path is batch-invariant),
the fp64 oracle's predictions (1e-2 relative), and the oracle select over the table."""
import numpy as np
import pytest

from paper_2505_09142_b200 import inputs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

SENTINEL = -12345.0


def _predictor(name="tiny", max_tokens=64 * 512, max_requests=256, **kw):
    from paper_2505_09142_b200 import binding
    cfg = inputs.CONFIGS[name]
    W = inputs.make_weights(cfg, seed=0)
    return cfg, W, binding.Predictor(cfg, inputs.flatten_weights(cfg, W), max_tokens, max_requests, **kw)


def _population(F, seed):
    L, gen, _ = inputs.trace_lengths(F, seed=seed)
    tok = inputs.make_tokens(L, seed=seed)
    return L, gen, tok, inputs.offsets(L)


def _slice(tok, offs, L, slots):
    t = np.concatenate([tok[offs[i]:offs[i + 1]] for i in slots]) if len(slots) else np.zeros(0, np.int32)
    return t.astype(np.int32), L[slots].astype(np.int32)


def _reference_table(P, F, L, tok, offs, windows):
    """Single-GPU elis_predict_remaining into one table, window by window."""
    table = torch.full((F,), SENTINEL, device="cuda")
    for sl in windows:
        t, l = _slice(tok, offs, L, sl)
        P.predict_remaining(torch.from_numpy(t).cuda(), torch.from_numpy(l).cuda(), int(l.sum()), table,
                            out_slot=torch.from_numpy(sl).cuda())
    assert P.sync_status() == 0
    return table.cpu().numpy()


@pytest.mark.parametrize("world,empty_rank", [(1, None), (2, None), (3, 1), (4, None), (8, 5)])
def test_predict_dist_peer_local_ranks(cuda_lib, world, empty_rank):
    from paper_2505_09142_b200 import binding
    cfg, W, Pref = _predictor()
    F, due = 700, 90
    L, gen, tok, offs = _population(F, seed=31)
    windows = [((k * due + np.arange(due)) % F).astype(np.int32) for k in range(4)]  # 4 calls: both parities
    ref = _reference_table(Pref, F, L, tok, offs, windows)
    Pref.close()
    Ps = [_predictor()[2] for _ in range(world)]
    binding.peer_attach_local(Ps)
    streams = [torch.cuda.Stream() for _ in range(world)]
    tables = [torch.full((F,), SENTINEL, device="cuda") for _ in range(world)]
    for sl in windows:
        b = binding.cost_split(L[sl], world, cfg)
        args = []
        for r in range(world):
            # a rank with nothing to encode (its slice dropped) still takes part in the exchange
            mine = sl[b[r]:b[r + 1]] if r != empty_rank else sl[:0]
            t, l = _slice(tok, offs, L, mine)
            args.append((torch.from_numpy(t).cuda(), torch.from_numpy(l).cuda(), int(l.sum()),
                         torch.from_numpy(mine.copy()).cuda()))
        torch.cuda.synchronize()
        for r in range(world):   # enqueue every rank before any can finish
            t, l, T, s = args[r]
            Ps[r].predict_remaining_dist(t if T else None, l if T else None, T, tables[r], s, stream=streams[r])
        torch.cuda.synchronize()
    for r in range(world):
        assert Ps[r].sync_status() == 0
        got = tables[r].cpu().numpy()
        if empty_rank is None:
            np.testing.assert_array_equal(got, ref, err_msg=f"rank {r}")
        else:   # the empty rank's slots of each window keep the sentinel; everything else matches
            miss = got == SENTINEL
            assert miss.sum() > F - len(windows) * due   # slots outside every window + the dropped ones
            np.testing.assert_array_equal(got[~miss], ref[~miss])
    for P in Ps:
        P.close()


def test_predict_dist_nccl_world1_and_peer_agree(cuda_lib):
    from paper_2505_09142_b200 import binding
    cfg, W, P0 = _predictor()
    F, due = 400, 120
    L, gen, tok, offs = _population(F, seed=32)
    sl = np.arange(due, dtype=np.int32) * 3 % F
    ref = _reference_table(P0, F, L, tok, offs, [sl])
    P0.close()
    t, l = _slice(tok, offs, L, sl)
    for transport in ("nccl", "peer"):
        _, _, P = _predictor()
        if transport == "nccl":
            P.dist_attach(0, 1, binding.nccl_unique_id())
        else:
            binding.peer_attach_local([P])
        table = torch.full((F,), SENTINEL, device="cuda")
        for _ in range(3):
            P.predict_remaining_dist(torch.from_numpy(t).cuda(), torch.from_numpy(l).cuda(), int(l.sum()), table,
                                     torch.from_numpy(sl).cuda())
        assert P.sync_status() == 0
        np.testing.assert_array_equal(table.cpu().numpy(), ref, err_msg=transport)
        P.close()


def test_predict_dist_base_default_precision_vs_oracle(cuda_lib):
    """BGE-base at the ABI default precision (fp16 operands + fp16 residual stream): two ranks
    sharing the GPU encode the cost-balanced halves of a ragged due set; both replicas of the
    table hold the oracle's predictions within the north_star's 1e-2 relative bar."""
    from oracle import head as ohead
    from paper_2505_09142_b200 import binding
    cfg = inputs.CONFIGS["base"]
    W = inputs.make_weights(cfg, seed=0)
    F = 64
    L = np.array([1, 7, 33, 64, 65, 127, 128, 129, 200, 300, 511, 512, 40, 90], np.int32)
    slots = np.array([3, 60, 17, 0, 44, 5, 9, 31, 22, 63, 50, 12, 38, 27], np.int32)
    tok = inputs.make_tokens(L, seed=33)
    offs = inputs.offsets(L)
    ref = ohead.predict(tok, L, W, cfg)
    Ps = [binding.Predictor(cfg, inputs.flatten_weights(cfg, W), int(L.sum()), len(L)) for _ in range(2)]
    binding.peer_attach_local(Ps)
    b = binding.cost_split(L, 2, cfg)
    assert 0 < b[1] < len(L)
    streams = [torch.cuda.Stream() for _ in range(2)]
    tables = [torch.full((F,), SENTINEL, device="cuda") for _ in range(2)]
    # every rank's device inputs stay referenced until both ranks finished: a temporary freed after
    # the call returns could be handed to the other rank's next allocation (another stream) while
    # this rank's kernels still read it
    args = []
    for r in range(2):
        a, e = b[r], b[r + 1]
        t = tok[offs[a]:offs[e]]
        args.append((torch.from_numpy(t).cuda(), torch.from_numpy(L[a:e].copy()).cuda(), int(t.size),
                     torch.from_numpy(slots[a:e].copy()).cuda()))
    torch.cuda.synchronize()
    for r in range(2):
        t, l, T, s = args[r]
        Ps[r].predict_remaining_dist(t, l, T, tables[r], s, stream=streams[r])
    torch.cuda.synchronize()
    for r in range(2):
        assert Ps[r].sync_status() == 0
        got = tables[r].cpu().numpy().astype(np.float64)
        rel = np.abs(got[slots] - ref) / np.maximum(np.abs(ref), 1.0)
        assert rel.max() <= 1e-2, (r, rel.max())
        assert (np.delete(got, slots) == SENTINEL).all()
    np.testing.assert_array_equal(tables[0].cpu().numpy(), tables[1].cpu().numpy())
    for P in Ps:
        P.close()


@pytest.mark.parametrize("F,due,cap", [(5000, 100, 256), (65536, 64, 256), (300, 50, 4)])
def test_iteration_table_host_matches_device_path_and_oracle(cuda_lib, F, due, cap):
    """elis_iteration_table_host (host due tokens in, ids out) == device calls, and its batch is the
    oracle select over the resulting table (cached keys + the re-predicted due set)."""
    from oracle.select import isrtf_select
    cfg, W, P = _predictor(max_requests=max(due, 1))
    L, gen, tok, offs = _population(F, seed=34)
    base = inputs.random_predictions(F, seed=35, kind="spread")
    sl = ((7 * np.arange(due)) % F).astype(np.int32)
    t, l = _slice(tok, offs, L, sl)
    d_gen = torch.from_numpy(gen).cuda()
    table_a = torch.from_numpy(base.copy()).cuda()
    P.predict_remaining(torch.from_numpy(t).cuda(), torch.from_numpy(l).cuda(), int(l.sum()), table_a,
                        out_slot=torch.from_numpy(sl).cuda())
    ids_a = torch.empty(cap, dtype=torch.int32, device="cuda")
    P.isrtf_select(table_a, d_gen, cap, ids_a)
    table_b = torch.from_numpy(base.copy()).cuda()
    h_ids = np.full(cap, -7, np.int32)
    h_cnt = np.zeros(1, np.int32)
    P.iteration_table_host(t, l, sl, table_b, d_gen, cap, h_ids, h_cnt)
    assert P.sync_status() == 0
    tb = table_b.cpu().numpy()
    np.testing.assert_array_equal(tb, table_a.cpu().numpy())
    np.testing.assert_array_equal(h_ids, ids_a.cpu().numpy())
    o_ids, o_cnt, _, _ = isrtf_select(tb, gen, cap)
    np.testing.assert_array_equal(h_ids, o_ids)
    assert h_cnt[0] == o_cnt
    P.close()
