"""CPU-side checks of the C-ABI library: it loads, exports every symbol the headers
declare, and its host-only logic (weight count, config validation) agrees with the
input generator.  No compute calls (there is no GPU here)."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2505_09142_b200 import binding, inputs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_functions():
    names = []
    for h in ("elis.h", "elis_ops.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names += re.findall(r"\b(elis_[a-z0-9_]+)\s*\(", src)
    return sorted(set(names))


def test_library_exports_every_declared_symbol():
    L = binding.lib()
    names = _declared_functions()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing


def test_abi_version():
    assert binding.lib().elis_abi_version() == binding.ABI_VERSION == 5


@pytest.mark.parametrize("name", ["tiny", "base", "large"])
def test_weight_count_matches_generator(name):
    cfg = inputs.CONFIGS[name]
    c = binding.make_config(cfg, 1024, 16)
    assert binding.lib().elis_weight_count(ctypes.byref(c)) == inputs.weight_count(cfg)


def test_invalid_configs_rejected():
    L = binding.lib()
    base = inputs.CONFIGS["base"]
    for bad in (dict(hidden=100), dict(num_heads=5), dict(max_position=1024), dict(intermediate=100),
                dict(max_tokens=0)):
        c = binding.make_config(base, 1024, 16)
        for k, v in bad.items():
            setattr(c, k, v)
        assert L.elis_weight_count(ctypes.byref(c)) == 0
        h = ctypes.c_void_p()
        w = np.zeros(4, np.float32)
        assert L.elis_predictor_create(ctypes.byref(c), w.ctypes.data, 4, ctypes.byref(h)) == 2  # ELIS_ERR_CONFIG


def test_create_validates_weight_count_and_device():
    L = binding.lib()
    c = binding.make_config(inputs.CONFIGS["tiny"], 1024, 16)
    h = ctypes.c_void_p()
    w = np.zeros(10, np.float32)
    assert L.elis_predictor_create(ctypes.byref(c), w.ctypes.data, 10, ctypes.byref(h)) == 1  # count mismatch
    n = L.elis_weight_count(ctypes.byref(c))
    w = np.zeros(n, np.float32)
    st = L.elis_predictor_create(ctypes.byref(c), w.ctypes.data, n, ctypes.byref(h))
    import torch
    if not torch.cuda.is_available():
        assert st == 3  # ELIS_ERR_UNSUPPORTED_DEVICE: no device here
        assert b"device" in L.elis_last_error()
    else:
        assert st == 0
        L.elis_predictor_destroy(h)


def test_status_strings():
    L = binding.lib()
    for s in range(8):
        assert L.elis_status_string(s)


def test_null_argument_errors_without_gpu():
    L = binding.lib()
    # NULL predictor: host-validated, returns immediately
    assert L.elis_predict_remaining(None, None, None, 1, 1, None, None, None) == 1
    assert L.elis_isrtf_select(None, None, None, 1, 1, None, None, None) == 1
    assert L.elis_sync_status(None) == 1


def test_precision_validation():
    """FP8 needs head dim 64 and 256-multiples; unknown precisions fail."""
    L = binding.lib()
    ok = binding.make_config(inputs.CONFIGS["base"], 1024, 16, precision="fp8")
    assert L.elis_weight_count(ctypes.byref(ok)) == inputs.weight_count(inputs.CONFIGS["base"])
    tiny = binding.make_config(inputs.CONFIGS["tiny"], 1024, 16, precision="fp8")
    assert L.elis_weight_count(ctypes.byref(tiny)) == 0
    bad = binding.make_config(inputs.CONFIGS["base"], 1024, 16)
    bad.precision = 7
    assert L.elis_weight_count(ctypes.byref(bad)) == 0


def test_cls_last_layer_validation():
    """The CLS-only last layer requires CLS pooling and head dim 64."""
    L = binding.lib()
    cls_cfg = inputs.EncoderConfig(**{**inputs.CONFIGS["base"].to_dict(), "pooling": inputs.POOL_CLS})
    ok = binding.make_config(cls_cfg, 1024, 16, cls_last_layer=True)
    assert L.elis_weight_count(ctypes.byref(ok)) > 0
    mean = binding.make_config(inputs.CONFIGS["base"], 1024, 16, cls_last_layer=True)
    assert L.elis_weight_count(ctypes.byref(mean)) == 0
    tiny = inputs.EncoderConfig(**{**inputs.CONFIGS["tiny"].to_dict(), "pooling": inputs.POOL_CLS})
    assert L.elis_weight_count(ctypes.byref(binding.make_config(tiny, 1024, 16, cls_last_layer=True))) == 0


def _declared_arity():
    """name -> number of parameters, parsed from the headers' prototypes."""
    out = {}
    for h in ("elis.h", "elis_ops.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"\b(elis_[a-z0-9_]+)\s*\(([^;{]*?)\)\s*;", src, flags=re.S):
            params = m.group(2).strip()
            out[m.group(1)] = 0 if params in ("", "void") else params.count(",") + 1
    return out


def test_binding_signatures_match_the_headers():
    """Every function the binding declares takes as many arguments as its C prototype (catches a
    changed prototype the ctypes table did not follow)."""
    L = binding.lib()
    arity = _declared_arity()
    checked = 0
    for name, n in arity.items():
        fn = getattr(L, name, None)
        if fn is None or fn.argtypes is None:
            continue
        assert len(fn.argtypes) == n, (name, len(fn.argtypes), n)
        checked += 1
    assert checked >= 25


def test_residual16_validation():
    """residual16 (ABI v4) needs fp16 operands and no CLS-only last layer."""
    L = binding.lib()
    base = inputs.CONFIGS["base"]
    ok = binding.make_config(base, 1024, 16, precision="fp16", residual16=True)
    assert L.elis_weight_count(ctypes.byref(ok)) == inputs.weight_count(base)
    bad = binding.make_config(base, 1024, 16, precision="bf16", residual16=True)
    assert L.elis_weight_count(ctypes.byref(bad)) == 0
    cls_cfg = inputs.EncoderConfig(**{**base.to_dict(), "pooling": inputs.POOL_CLS})
    both = binding.make_config(cls_cfg, 1024, 16, precision="fp16", residual16=True, cls_last_layer=True)
    assert L.elis_weight_count(ctypes.byref(both)) == 0


def _brute_split(L, world, cfg):
    """The SURVEY.md 8e rule written out: boundary r = the index whose prefix cost is closest to
    r/world of the total (ties -> smaller index), searched from the previous boundary on."""
    H, F, nl = cfg.hidden, cfg.intermediate, cfg.num_layers
    c = [nl * (2.0 * (4 * H * H + 2 * H * F) * x + 4.0 * H * x * x) for x in L.tolist()]
    pre = [0.0]
    for v in c:
        pre.append(pre[-1] + v)
    b = [0]
    for r in range(1, world):
        tgt = pre[-1] * r / world
        cands = range(b[-1], len(L) + 1)
        b.append(min(cands, key=lambda i: (abs(pre[i] - tgt), i)))
    b.append(len(L))
    return np.array(b, np.int32), c


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("kind", ["trace", "uniform", "tiny"])
def test_cost_split_matches_definition_and_balances(world, kind):
    """elis_cost_split (host function of the C ABI, no GPU): equal to the written-out quantile rule,
    contiguous, and every slice's cost within one request of total / world."""
    cfg = inputs.CONFIGS["base"]
    if kind == "trace":
        L, _, _ = inputs.trace_lengths(1311, seed=world)
    elif kind == "uniform":
        L = inputs.uniform_lengths(500, seed=world)
    else:
        L = np.array([512, 1, 1, 3], np.int32)
    got = binding.cost_split(L, world, cfg)
    exp, c = _brute_split(L, world, cfg)
    np.testing.assert_array_equal(got, exp)
    assert got[0] == 0 and got[-1] == len(L) and (np.diff(got) >= 0).all()
    if kind != "tiny":
        tot, cmax = sum(c), max(c)
        for r in range(world):
            assert abs(sum(c[got[r]:got[r + 1]]) - tot / world) <= cmax + 1e-6 * tot
    # BGE-base constants of SURVEY.md 8e: c(L) = 169.87e6 L + 36,864 L^2
    assert abs(c[0] - (169.869312e6 * int(L[0]) + 36864.0 * int(L[0]) ** 2)) < 1.0


def test_cost_split_edge_cases():
    cfg = inputs.CONFIGS["base"]
    np.testing.assert_array_equal(binding.cost_split(np.zeros(0, np.int32), 4, cfg), [0, 0, 0, 0, 0])
    np.testing.assert_array_equal(binding.cost_split(np.array([100], np.int32), 3, cfg), [0, 0, 1, 1])
    with pytest.raises(binding.ElisError):
        binding.cost_split(np.array([1, 2], np.int32), 0, cfg)
