"""Device-resident token arena (include/elis.h elis_arena_*): prompts
uploaded once, generated tokens appended per window, the due set's predictor inputs gathered on
the device -- bit-identical to the host construction of "the prompt attached with the answer"
 with the harness's truncation rule (R7, streamsim.build_sequence)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).cuda()


@pytest.mark.parametrize("seed", [0, 1])
def test_arena_gather_matches_host_sequences(cuda_lib, seed):
    from paper_2505_09142_b200 import binding
    from paper_2505_09142_b200.streamsim import build_sequence, seq_len
    rng = np.random.default_rng(seed)
    F = 300
    A = binding.Arena(F)
    prompts = [np.concatenate([[101], rng.integers(1000, 30522, int(rng.integers(0, 400))), [102]]).astype(np.int32)
               for _ in range(F)]
    responses = [rng.integers(1000, 30522, 1400).astype(np.int32) for _ in range(F)]
    gen = np.zeros(F, np.int64)
    slots = np.arange(F, dtype=np.int32)
    A.set_prompts(_dev(slots), _dev(np.concatenate(prompts)), _dev([len(p) for p in prompts]))
    out = torch.empty(F * 512, dtype=torch.int32, device="cuda")
    lens = torch.empty(F, dtype=torch.int32, device="cuda")
    dims = torch.empty(2, dtype=torch.int32, device="cuda")
    for rnd in range(30):  # windows: a random subset of jobs generates 1..50 tokens (ring wraps past 512)
        who = np.sort(rng.choice(F, int(rng.integers(1, F)), replace=False)).astype(np.int32)
        cnt = rng.integers(0, 51, who.size).astype(np.int32)
        cnt = np.minimum(cnt, 1400 - gen[who]).astype(np.int32)
        A.append(_dev(who), _dev(np.concatenate([responses[j][gen[j]:gen[j] + c] for j, c in zip(who, cnt)])),
                 _dev(cnt))
        gen[who] += cnt
        due = rng.permutation(F)[: int(rng.integers(1, 64))].astype(np.int32)
        A.gather(_dev(due), 512, out, lens[:due.size], dims)
        assert A.sync_status() == 0
        want = [build_sequence(prompts[j], responses[j], int(gen[j])) for j in due]
        L = lens[:due.size].cpu().numpy()
        np.testing.assert_array_equal(L, [w.size for w in want])
        assert (L == [seq_len(prompts[j].size, int(gen[j])) for j in due]).all()
        np.testing.assert_array_equal(dims.cpu().numpy(), [due.size, int(L.sum())])
        np.testing.assert_array_equal(out[:int(L.sum())].cpu().numpy(), np.concatenate(want))
    assert gen.max() > 520  # the truncation and the ring wrap were exercised
    A.close()


def test_arena_errors_are_sticky(cuda_lib):
    from paper_2505_09142_b200 import binding
    A = binding.Arena(8)
    A.set_prompts(_dev([9]), _dev([101, 5, 102]), _dev([3]))          # slot out of range
    assert A.sync_status() == 7
    assert A.sync_status() == 0                                        # cleared after reporting
    A.set_prompts(_dev([2]), _dev(np.full(600, 7)), _dev([600]))       # prompt longer than 512
    assert A.sync_status() == 7
    out = torch.empty(1024, dtype=torch.int32, device="cuda")
    lens = torch.empty(1, dtype=torch.int32, device="cuda")
    A.gather(_dev([5]), 512, out, lens)                                 # slot 5 never got a prompt
    assert A.sync_status() == 7
    with pytest.raises(binding.ElisError):
        A.gather(_dev([1]), 513, out, lens)                             # host-validated max_len
    A.close()
