#!/usr/bin/env python3
"""Minimax polynomial for 2^f on [-1/2, 1/2] (relative error), used by the attention softmax's
FMA-pipe exp2 (csrc/attention.cu, exp2_poly2).  Linear program on a dense grid, then the fp32
Horner evaluation is re-checked.

    python scripts/fit_exp2.py [degree]      # default 3 -> max rel err 7.5e-5
"""
import sys

import numpy as np
from scipy.optimize import linprog


def fit(deg: int):
    f = np.linspace(-0.5, 0.5, 4001)
    y = 2.0 ** f
    A = np.stack([f ** k / y for k in range(deg + 1)], 1)
    n = A.shape[0]
    a_ub = np.vstack([np.hstack([A, -np.ones((n, 1))]), np.hstack([-A, -np.ones((n, 1))])])
    b_ub = np.concatenate([np.ones(n), -np.ones(n)])
    c = np.zeros(deg + 2)
    c[-1] = 1.0
    r = linprog(c, A_ub=a_ub, b_ub=b_ub, bounds=[(None, None)] * (deg + 2))
    co = r.x[:-1].astype(np.float32)
    ff = np.linspace(-0.5, 0.5, 100001).astype(np.float32)
    p = np.zeros_like(ff)
    for k in range(deg, -1, -1):
        p = (p * ff + co[k]).astype(np.float32)
    err = np.abs(p / 2.0 ** ff.astype(np.float64) - 1).max()
    return co, err


if __name__ == "__main__":
    d = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    co, err = fit(d)
    print("coefficients c0..c%d:" % d, [f"{float(x):.10g}" for x in co], f"max rel err {err:.3g}")
