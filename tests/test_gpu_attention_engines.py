"""The optional 64-key attention engines are bitwise equal to the default one.

ELIS_ATTN_ENGINE selects the engine once per process, so each engine runs in its own subprocess
(scripts/attn_repro.py) on the same seeded ragged input: 65 = persistent 4-CTA/SM item loop, 66 =
early S with P in shared memory.  Both keep every MMA, the softmax and the
epilogue rounding of the default 64-key engine, so their ctx must match it bit for bit -- bf16 and
fp16 planes, with keys ramped so the lazy O rescale runs in part of the rows.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LENGTHS = "1,2,31,63,64,65,130,7,512,200,33,511,257,100,3,129,96,97"


def _dump(engine, path, f16, ramp):
    env = dict(os.environ, ELIS_ATTN_ENGINE=engine)
    cmd = [sys.executable, os.path.join(ROOT, "scripts", "attn_repro.py"), LENGTHS, "--dump", str(path), "--seed", "3"]
    cmd += (["--f16"] if f16 else []) + (["--ramp"] if ramp else [])
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=180)
    assert r.returncode == 0, r.stderr[-2000:]
    return np.load(path)


@pytest.mark.parametrize("f16,ramp", [(False, False), (True, False), (True, True)])
def test_optional_attention_engines_bitwise_equal(cuda_lib, tmp_path, f16, ramp):
    ref = _dump("64", tmp_path / "e64.npy", f16, ramp)
    for engine in ("65", "66"):
        got = _dump(engine, tmp_path / f"e{engine}.npy", f16, ramp)
        assert np.array_equal(got, ref), engine
