"""Shape-agnostic predict (elis_predict_remaining_dev): n and total_tokens read
on the device, every kernel sized for the capacity and exiting beyond the device values -- the same
bits as elis_predict_remaining, and ONE captured CUDA graph replays iterations whose due sets differ
in size (the closed loop of row f1)."""
import numpy as np
import pytest

from paper_2505_09142_b200 import inputs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _predictor(name, max_tokens, max_requests, **kw):
    from paper_2505_09142_b200 import binding
    cfg = inputs.CONFIGS[name]
    if kw.pop("cls", False):
        cfg = inputs.EncoderConfig(**{**cfg.to_dict(), "pooling": inputs.POOL_CLS})
    W = inputs.make_weights(cfg, seed=0)
    return binding.Predictor(cfg, inputs.flatten_weights(cfg, W), max_tokens, max_requests, **kw)


@pytest.mark.parametrize("name,kw", [("tiny", {}), ("base", {}), ("base", {"cls": True, "cls_last_layer": True})])
def test_dev_dims_equal_host_shapes(cuda_lib, name, kw):
    P = _predictor(name, 8192, 64, **kw)
    cap_tok = torch.zeros(8192, dtype=torch.int32, device="cuda")
    cap_len = torch.zeros(64, dtype=torch.int32, device="cuda")
    dims = torch.zeros(2, dtype=torch.int32, device="cuda")
    for seed, n in ((1, 1), (2, 17), (3, 64), (4, 5)):
        L, _, _ = inputs.trace_lengths(n, seed=seed)
        L = np.minimum(L, 8192 // 64).astype(np.int32) if n == 64 else L.astype(np.int32)
        tok = inputs.make_tokens(L, seed=seed)
        T = int(L.sum())
        ref = torch.full((n,), float("nan"), device="cuda")
        P.predict_remaining(torch.from_numpy(tok).cuda(), torch.from_numpy(L).cuda(), T, ref)
        cap_tok[:T] = torch.from_numpy(tok).cuda()
        cap_len[:n] = torch.from_numpy(L).cuda()
        dims.copy_(torch.tensor([n, T], dtype=torch.int32))
        got = torch.full((64,), float("nan"), device="cuda")
        P.predict_remaining_dev(cap_tok, cap_len, dims, got)
        assert P.sync_status() == 0
        assert torch.equal(got[:n], ref), (name, n)
        assert torch.isnan(got[n:]).all()            # nothing written past n
    dims.copy_(torch.tensor([65, 100], dtype=torch.int32))   # n beyond max_requests: sticky, no crash
    P.predict_remaining_dev(cap_tok, cap_len, dims, torch.empty(64, device="cuda"))
    assert P.sync_status() == 7 and P.device_error_bits() & 64
    P.close()


def test_one_graph_replays_variable_due_sets(cuda_lib):
    """Capture predict_dev (into the in-flight table through out_slot) + the ISRTF select once;
    replay it for due sets of different sizes: the table and the batch equal the eager calls."""
    P = _predictor("base", 16384, 128)
    F, cap = 2048, 16
    gen = torch.zeros(F, dtype=torch.int32, device="cuda")
    table_g = torch.from_numpy(inputs.random_predictions(F, seed=5, kind="spread")).cuda()
    table_e = table_g.clone()
    tok = torch.zeros(16384, dtype=torch.int32, device="cuda")
    lens = torch.zeros(128, dtype=torch.int32, device="cuda")
    slots = torch.zeros(128, dtype=torch.int32, device="cuda")
    dims = torch.zeros(2, dtype=torch.int32, device="cuda")
    ids_g = torch.empty(cap, dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):  # warm-up (launch attributes set outside the capture)
        P.predict_remaining_dev(tok, lens, dims, table_g, out_slot=slots, stream=s)
        P.isrtf_select(table_g, gen, cap, ids_g, stream=s)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        P.predict_remaining_dev(tok, lens, dims, table_g, out_slot=slots, stream=s)
        P.isrtf_select(table_g, gen, cap, ids_g, stream=s)
    rng = np.random.default_rng(9)
    for it, n in enumerate((3, 40, 1, 128, 17)):
        L, _, _ = inputs.trace_lengths(n, seed=20 + it)
        L = np.minimum(L, 16384 // 128).astype(np.int32) if n == 128 else L.astype(np.int32)
        t = inputs.make_tokens(L, seed=20 + it)
        sl = rng.choice(F, n, replace=False).astype(np.int32)
        T = int(L.sum())
        tok[:T] = torch.from_numpy(t).cuda()
        lens[:n] = torch.from_numpy(L).cuda()
        slots[:n] = torch.from_numpy(sl).cuda()
        dims.copy_(torch.tensor([n, T], dtype=torch.int32))
        g.replay()
        torch.cuda.synchronize()
        ids_e = torch.empty(cap, dtype=torch.int32, device="cuda")
        P.predict_remaining(torch.from_numpy(t).cuda(), torch.from_numpy(L).cuda(), T, table_e,
                            out_slot=torch.from_numpy(sl).cuda())
        P.isrtf_select(table_e, gen, cap, ids_e)
        assert P.sync_status() == 0
        assert torch.equal(table_g, table_e), n
        assert torch.equal(ids_g, ids_e), n
    P.close()
