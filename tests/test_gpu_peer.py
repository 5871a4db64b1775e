"""Peer-memory transport of elis_isrtf_select_dist (include/elis.h "multi-GPU over peer memory";
SURVEY.md Sec. 8a row a13, 8e "B200-native stretch"): local top-cap ->
NVLink stores into every rank's region + epoch flags -> acquire -> identical merge, one kernel.

One B200 is enough to run the protocol for real: several ranks share the device, each with its
own predictor, region and stream, and their fused kernels run concurrently and wait on each
other's flags.  (1) ranks in one process (elis_peer_attach_local); (2) two processes mapping
each other's region through CUDA IPC (elis_peer_attach), handles exchanged over gloo -- the path
bench.py takes at N > 1.  Expected values: the oracle select over the concatenated slots, with
global ids (tie-break rank = global slot index, or the caller's global order)."""
import os

import numpy as np
import pytest

from paper_2505_09142_b200 import inputs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _predictor():
    from paper_2505_09142_b200 import binding
    cfg = inputs.CONFIGS["tiny"]
    return binding.Predictor(cfg, inputs.flatten_weights(cfg, inputs.make_weights(cfg, seed=0)), 1024, 1024)


def _split(n, world):
    b = np.linspace(0, n, world + 1).round().astype(int)
    return [(int(b[r]), int(b[r + 1] - b[r])) for r in range(world)]


def _oracle(pred, gen, cap, allow, running, order=None):
    from oracle.select import isrtf_select
    n = pred.shape[0]
    order = np.arange(n, dtype=np.uint32) if order is None else order
    return isrtf_select(pred, gen, cap, 0, allow, order, running)


@pytest.mark.parametrize("world,n,cap,allow", [(2, 256, 4, True), (2, 8192, 256, False), (3, 1000, 64, True),
                                               (4, 65536, 1024, True), (8, 4096, 16, False), (1, 300, 128, True)])
def test_peer_select_local_ranks_match_oracle(cuda_lib, world, n, cap, allow):
    from paper_2505_09142_b200 import binding
    Ps = [_predictor() for _ in range(world)]
    binding.peer_attach_local(Ps)
    streams = [torch.cuda.Stream() for _ in range(world)]
    parts = _split(n, world)
    # three calls with fresh inputs each: both parities of the double-buffered regions are reused
    for it in range(3):
        pred = inputs.random_predictions(n, seed=97 * it + n)
        gen, order, running = inputs.random_sched_state(n, seed=97 * it + n + 1)
        o_ids, o_cnt, o_pre, _ = _oracle(pred, gen, cap, allow, running)
        outs = []
        for r, (off, nl) in enumerate(parts):
            d = dict(pred=torch.from_numpy(pred[off:off + nl].copy()).cuda(),
                     gen=torch.from_numpy(gen[off:off + nl].copy()).cuda(),
                     run=torch.from_numpy(running[off:off + nl].copy()).cuda(),
                     ids=torch.full((cap,), -7, dtype=torch.int32, device="cuda"),
                     cnt=torch.zeros(1, dtype=torch.int32, device="cuda"),
                     pre=torch.full((max(nl, 1),), 9, dtype=torch.uint8, device="cuda"))
            outs.append(d)
        torch.cuda.synchronize()
        for r, (off, nl) in enumerate(parts):   # enqueue every rank before any can finish
            d = outs[r]
            Ps[r].isrtf_select_dist(d["pred"], d["gen"], off, cap, d["ids"], allow_preempt=allow, running=d["run"],
                                    out_preempted=d["pre"], out_count=d["cnt"], stream=streams[r])
        torch.cuda.synchronize()
        for r, (off, nl) in enumerate(parts):
            assert Ps[r].sync_status() == 0
            d = outs[r]
            np.testing.assert_array_equal(d["ids"].cpu().numpy(), o_ids, err_msg=f"rank {r} iteration {it}")
            assert int(d["cnt"].item()) == o_cnt
            np.testing.assert_array_equal(d["pre"].cpu().numpy()[:nl], o_pre[off:off + nl])
    for P in Ps:
        P.close()


def test_peer_select_equals_nccl_transport(cuda_lib):
    """world 1: the peer kernel and the NCCL path (pack -> all-gather -> unpack -> merge) agree
    bit for bit, including the caller's global order and FCFS."""
    from paper_2505_09142_b200 import binding
    n, cap, off = 5000, 256, 123
    pred = inputs.random_predictions(n, seed=5)
    gen, order, running = inputs.random_sched_state(n, seed=6)
    order = order + np.uint32(off)
    res = []
    for transport in ("nccl", "peer"):
        P = _predictor()
        if transport == "nccl":
            P.dist_attach(0, 1, binding.nccl_unique_id())
        else:
            binding.peer_attach_local([P])
        for policy in (binding.POLICY_ISRTF, binding.POLICY_FCFS):
            ids = torch.full((cap,), -7, dtype=torch.int32, device="cuda")
            cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
            pre = torch.zeros(n, dtype=torch.uint8, device="cuda")
            P.isrtf_select_dist(torch.from_numpy(pred).cuda(), torch.from_numpy(gen).cuda(), off, cap, ids,
                                policy=policy, allow_preempt=False, order=torch.from_numpy(order).cuda(),
                                running=torch.from_numpy(running).cuda(), out_preempted=pre, out_count=cnt)
            assert P.sync_status() == 0
            res.append((transport, policy, ids.cpu().numpy(), int(cnt.item()), pre.cpu().numpy()))
        P.close()
    for (_, pol, a_ids, a_cnt, a_pre), (_, pol2, b_ids, b_cnt, b_pre) in zip(res[:2], res[2:]):
        assert pol == pol2
        np.testing.assert_array_equal(a_ids, b_ids)
        assert a_cnt == b_cnt
        np.testing.assert_array_equal(a_pre, b_pre)


def test_peer_select_missing_rank_times_out(cuda_lib):
    """A rank that never calls: the waiting rank gives up (10 s bound) with the sticky
    ELIS_ERR_PEER_TIMEOUT and an empty batch instead of hanging the GPU."""
    from paper_2505_09142_b200 import binding
    Ps = [_predictor() for _ in range(2)]
    binding.peer_attach_local(Ps)
    n, cap = 64, 4
    pred = torch.from_numpy(inputs.random_predictions(n, seed=1)).cuda()
    gen = torch.zeros(n, dtype=torch.int32, device="cuda")
    ids = torch.full((cap,), -7, dtype=torch.int32, device="cuda")
    cnt = torch.full((1,), -7, dtype=torch.int32, device="cuda")
    Ps[0].isrtf_select_dist(pred, gen, 0, cap, ids, out_count=cnt)
    assert Ps[0].sync_status() == 8  # ELIS_ERR_PEER_TIMEOUT
    assert (ids.cpu().numpy() == -1).all() and int(cnt.item()) == 0
    assert Ps[0].sync_status() == 0  # cleared
    for P in Ps:
        P.close()


def _ipc_worker(rank, world, port, n, cap, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2505_09142_b200 import binding
        torch.cuda.set_device(0)
        P = _predictor()
        h = P.peer_export(rank, world)
        hs = [None] * world
        dist.all_gather_object(hs, h)
        P.peer_attach(hs)
        parts = _split(n, world)
        off, nl = parts[rank]
        got = []
        for it in range(4):
            pred = inputs.random_predictions(n, seed=11 * it + 3)
            gen, order, running = inputs.random_sched_state(n, seed=11 * it + 4)
            ids = torch.full((cap,), -7, dtype=torch.int32, device="cuda")
            cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
            pre = torch.zeros(nl, dtype=torch.uint8, device="cuda")
            P.isrtf_select_dist(torch.from_numpy(pred[off:off + nl].copy()).cuda(),
                                torch.from_numpy(gen[off:off + nl].copy()).cuda(), off, cap, ids,
                                running=torch.from_numpy(running[off:off + nl].copy()).cuda(), out_preempted=pre,
                                out_count=cnt)
            st = P.sync_status()
            got.append((st, ids.cpu().numpy(), int(cnt.item()), pre.cpu().numpy()))
        dist.barrier()   # no rank unmaps a region another rank may still be writing
        P.close()
        q.put((rank, got))
    except Exception as e:  # surfaced by the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_peer_select_two_processes_cuda_ipc(cuda_lib):
    """Two processes on one B200, regions mapped through cudaIpcOpenMemHandle: the exact
    multi-process path bench.py uses at N > 1 (there, one GPU per rank over NVLink)."""
    import socket

    import torch.multiprocessing as mp
    world, n, cap = 2, 3000, 64
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_worker, args=(r, world, port, n, cap, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    parts = _split(n, world)
    for r in range(world):
        assert not isinstance(res[r], str), res[r]
        for it, (st, ids, cnt, pre) in enumerate(res[r]):
            pred = inputs.random_predictions(n, seed=11 * it + 3)
            gen, order, running = inputs.random_sched_state(n, seed=11 * it + 4)
            o_ids, o_cnt, o_pre, _ = _oracle(pred, gen, cap, True, running)
            assert st == 0
            np.testing.assert_array_equal(ids, o_ids, err_msg=f"rank {r} it {it}")
            assert cnt == o_cnt
            off, nl = parts[r]
            np.testing.assert_array_equal(pre, o_pre[off:off + nl])
