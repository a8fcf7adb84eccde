"""Pins of oracle/ops.py against the paper's definitions -- CPU only."""
import json
import os

import numpy as np
import pytest

from oracle import ops
from tvs_synth import random_field

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "operators.json")))


def test_forward_backward_examples():
    g = GOLD["forward_diff"]
    assert ops.dplus_x(np.array([g["in"]], float))[0].tolist() == g["out"]
    assert ops.dplus_y(np.array([g["in"]], float).T)[:, 0].tolist() == g["out"]
    g = GOLD["backward_diff"]
    assert ops.dminus_x(np.array([g["in"]], float))[0].tolist() == g["out"]
    assert ops.dminus_y(np.array([g["in"]], float).T)[:, 0].tolist() == g["out"]


def test_neumann_examples():
    for key, fn in (("dneum_x", ops.dneum_x), ("dneum_y", ops.dneum_y)):
        g = GOLD[key]
        assert fn(np.array(g["in"], float)).tolist() == g["out"]


def test_laplacian_impulse():
    u = np.zeros((5, 5))
    u[2, 2] = 1.0
    lap = ops.laplacian(u)
    g = GOLD["laplacian_impulse_5x5"]
    assert lap[2, 2] == g["out_centre"]
    for (i, j) in ((1, 2), (3, 2), (2, 1), (2, 3)):
        assert lap[i, j] == g["out_neighbours"]
    assert abs(lap).sum() == 8


@pytest.mark.parametrize("shape", [(2, 2), (3, 5), (6, 4), (7, 9)])
def test_adjointness(shape):
    """div = -grad^* and multidiv = -multigrad^* (P:603), to round-off."""
    u = random_field(shape, 1)
    p = random_field((2,) + shape, 2)
    assert abs(ops.inner(ops.grad(u), p) + ops.inner(u, ops.div(p))) < 1e-12
    uu = random_field((2,) + shape, 3)
    pp = random_field((2, 2) + shape, 4)
    assert abs(ops.inner(ops.multigrad(uu), pp) + ops.inner(uu, ops.multidiv(pp))) < 1e-12


def test_dminus_is_minus_dplus_transpose():
    for n in (2, 3, 5, 8):
        dp = np.array([ops.dplus_x(np.eye(n)[k][None, :])[0] for k in range(n)]).T
        dm = np.array([ops.dminus_x(np.eye(n)[k][None, :])[0] for k in range(n)]).T
        assert np.array_equal(dm, -dp.T)


def test_laplacian_is_neumann_tridiagonal():
    """Delta = D-D+ per axis is the 1D Neumann Laplacian (ends -1, interior -2)."""
    n = 6
    lap = np.array([ops.dminus_x(ops.dplus_x(np.eye(n)[k][None, :]))[0] for k in range(n)]).T
    ref = -2 * np.eye(n) + np.eye(n, k=1) + np.eye(n, k=-1)
    ref[0, 0] = ref[-1, -1] = -1
    assert np.array_equal(lap, ref)
