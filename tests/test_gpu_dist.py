"""elis_isrtf_select_dist on one B200 (world = 1 NCCL communicator): the full local top-cap ->
pack -> ncclAllGather -> unpack -> merge -> preempt-flag path, bit-exact against the oracle
select over the same slots with global ids.  (world_size 2 of the same decomposition runs on
CPU with gloo in tests/test_dist_gloo.py; one GPU per rank is required by NCCL.)"""
import numpy as np
import pytest

from paper_2505_09142_b200 import inputs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.mark.parametrize("n,cap,offset,allow", [(256, 4, 0, True), (8192, 256, 8192, False), (65536, 1024, 0, True),
                                                (100, 128, 300, True)])
def test_select_dist_world1_matches_oracle(cuda_lib, n, cap, offset, allow):
    from paper_2505_09142_b200 import binding
    from oracle.select import isrtf_select
    cfg = inputs.CONFIGS["tiny"]
    P = binding.Predictor(cfg, inputs.flatten_weights(cfg, inputs.make_weights(cfg, seed=0)), 1024, 1024)
    P.dist_attach(0, 1, binding.nccl_unique_id())
    pred = inputs.random_predictions(n, seed=n)
    gen, order, running = inputs.random_sched_state(n, seed=n)
    ids = torch.full((cap,), -7, dtype=torch.int32, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
    pre = torch.zeros(n, dtype=torch.uint8, device="cuda")
    P.isrtf_select_dist(torch.from_numpy(pred).cuda(), torch.from_numpy(gen).cuda(), offset, cap, ids,
                        allow_preempt=allow, running=torch.from_numpy(running).cuda(), out_preempted=pre,
                        out_count=cnt)
    assert P.sync_status() == 0
    o_ids, o_cnt, o_pre, _ = isrtf_select(pred, gen, cap, 0, allow, np.arange(n, dtype=np.uint32) + offset,
                                          running)
    got = ids.cpu().numpy()
    exp = np.where(o_ids >= 0, o_ids + offset, -1)
    np.testing.assert_array_equal(got, exp)
    assert int(cnt.item()) == o_cnt
    np.testing.assert_array_equal(pre.cpu().numpy(), o_pre)
    P.close()
