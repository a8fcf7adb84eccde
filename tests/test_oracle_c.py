"""Pins of the plain C11 oracle (oracle/c/tvo.c, NumPy-free, threaded per subdomain) -- no GPU.

The C oracle is pinned like the NumPy one, against what the paper and the mathematics fix
(hand-derived operator values, adjointness, the Penrose identities of Delta^dagger on non-square
grids, the projection's properties, the layout / partition-of-unity examples, Schwarz 1 x 1 =
Chambolle, the constant-image fixed point, the exact ROF solution of a step, weak duality and a
closing gap, DD -> single-domain convergence), and then against the NumPy oracle: two oracles
written independently from the same passages agree to rounding on ragged layouts."""
import json
import os

import numpy as np
import pytest

from oracle import c_oracle as C, layout, ops, solvers as S, spectral
from tvs_synth import random_field, random_image, step_image

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "operators.json")))


def test_operator_examples():
    """Hand-derived values (operators.json)."""
    u = np.array([GOLD["forward_diff"]["in"]], np.float64)
    assert np.allclose(C.grad(u)[0][0], GOLD["forward_diff"]["out"])
    p = np.stack([np.array([GOLD["backward_diff"]["in"]], np.float64), np.zeros((1, 3))])
    assert np.allclose(C.div(p)[0], GOLD["backward_diff"]["out"])
    d = np.array(GOLD["dneum_x"]["in"], np.float64)
    t = C.tau0(d)
    assert np.allclose(t[1], GOLD["dneum_x"]["out"])
    assert np.allclose(-t[0], GOLD["dneum_y"]["out"])
    imp = np.zeros((5, 5))
    imp[2, 2] = 1.0
    lap = C.div(C.grad(imp))
    assert lap[2, 2] == GOLD["laplacian_impulse_5x5"]["out_centre"]
    assert lap[1, 2] == lap[3, 2] == lap[2, 1] == lap[2, 3] == GOLD["laplacian_impulse_5x5"]["out_neighbours"]


@pytest.mark.parametrize("shape", [(6, 4), (5, 9), (2, 2)])
def test_adjointness(shape):
    """<grad u, p> = -<u, div p> (div = -grad^*)."""
    u = random_field(shape, 1, 1.0)
    p = random_field((2,) + shape, 2, 1.0)
    assert abs(np.sum(C.grad(u) * p) + np.sum(u * C.div(p))) < 1e-12


@pytest.mark.parametrize("shape", [(4, 6), (5, 7), (3, 3)])
def test_penrose_identities(shape):
    """X = Delta^dagger satisfies the four Penrose identities with Delta = div grad -- they fix the
    pseudo-inverse uniquely; non-square grids catch the printed sigma pairing (reading A2)."""
    n = shape[0] * shape[1]
    E = np.eye(n).reshape((n,) + shape)
    Lm = np.stack([C.div(C.grad(e)).ravel() for e in E], axis=1)
    X = np.stack([C.lap_pinv(e).ravel() for e in E], axis=1)
    for a, b in ((Lm @ X @ Lm, Lm), (X @ Lm @ X, X), (Lm @ X, (Lm @ X).T), (X @ Lm, (X @ Lm).T)):
        assert np.abs(a - b).max() < 1e-10


def test_projection_properties():
    """P is idempotent, self-adjoint, divergence-free, annihilates gradients."""
    w = random_field((2, 7, 9), 5, 1.0)
    v = random_field((2, 7, 9), 6, 1.0)
    pw = C.project(w)
    assert np.abs(C.div(pw)).max() < 1e-10
    assert np.abs(C.project(pw) - pw).max() < 1e-12
    assert abs(np.sum(pw * v) - np.sum(w * C.project(v))) < 1e-12
    assert np.abs(C.project(C.grad(random_field((7, 9), 7, 1.0)))).max() < 1e-12


def test_layout_examples():
    g = GOLD["layout_10_m2_s2"]
    assert [list(C.layout_range(g["n"], g["m"], g["s"], k)) for k in range(g["m"])] == g["ranges"]
    b = GOLD["pou_band_s2"]
    assert np.allclose([C.layout_theta(10, 2, 2, 0, x) for x in (4, 5)], b["theta_left_band"])
    assert np.allclose([C.layout_theta(10, 2, 2, 1, x) for x in (4, 5)], b["theta_right_band"])
    for n, m, s in ((50, 3, 4), (37, 5, 2)):
        for x in range(n):   # partition of unity
            assert abs(sum(C.layout_theta(n, m, s, k, x) for k in range(m)) - 1.0) < 1e-15


def test_schwarz_1x1_is_chambolle():
    """One subdomain (theta = 1, alpha_hat = 1): S sweeps of K updates = S K Chambolle
    iterations (Alg. 1) -- against the NumPy oracle's independent Chambolle loops."""
    d0 = random_image(12, 10, 7).astype(np.float64)
    tau, p, _ = C.step1(d0, 0.05, (1, 1, 0, 0), 5, 4)
    tb, pb = S.chambolle_tfs(d0, 0.05, 20)
    assert np.abs(tau - tb).max() < 1e-12 and np.abs(p - pb).max() < 1e-12
    d, _, _ = C.step2(d0, tb, 0.1, (1, 1, 0, 0), 5, 4)
    db, _ = S.chambolle_irv2(d0, tb, 0.1, 20)
    assert np.abs(d - db).max() < 1e-12


def test_constant_image_is_a_fixed_point():
    d0 = np.full((9, 11), 0.37)
    tau, p, st = C.step1(d0, 0.05, (2, 2, 3, 3), 3, 3)
    assert np.abs(tau).max() < 1e-14 and np.abs(p).max() == 0.0
    d, _, _ = C.step2(d0, tau, 0.1, (2, 2, 3, 3), 3, 3)
    assert np.abs(d - d0).max() < 1e-14


def test_rof_step_closed_form():
    """tau = 0 reduces IRV2 to ROF; the vertical step has the exact solution 1/(aL), 1 - 1/(aR)."""
    g = GOLD["rof_step"]
    d0 = step_image(g["n2"], g["left"] + g["right"], g["left"]).astype(np.float64)
    tau = np.zeros((2, g["n2"] + 1, g["left"] + g["right"] + 1))
    d, _, _ = C.step2(d0, tau, 1.0 / g["alpha"], (1, 1, 0, 0), 1, 4000)
    assert np.abs(d[:, :g["left"]] - g["low"]).max() < 1e-6
    assert np.abs(d[:, g["left"]:] - g["high"]).max() < 1e-6


def test_gap_closes_and_feasibility():
    """The C oracle's own energies: gap >= 0 and decreasing over longer single-domain runs; the dual
    stays in the unit balls."""
    d0 = random_image(10, 12, 9).astype(np.float64)
    tau, _, _ = C.step1(d0, 0.05, (1, 1, 0, 0), 1, 200)
    gaps = []
    for k in (5, 50, 2000):
        _, p, st = C.step2(d0, tau, 0.1, (1, 1, 0, 0), 1, k)
        gaps.append(st["gap"])
        assert np.sqrt(p[0] ** 2 + p[1] ** 2).max() <= 1.0 + 1e-12
    assert min(gaps) >= -1e-10 and gaps[0] > gaps[1] > gaps[2] and gaps[2] < 1e-2 * gaps[0]


def test_dd_converges_to_single_domain():
    """The 2 x 2 Schwarz iterate approaches the single-domain solution as the sweeps grow."""
    d0 = random_image(12, 12, 8).astype(np.float64)
    tau, _, _ = C.step1(d0, 0.05, (1, 1, 0, 0), 1, 100)
    ref, _, _ = C.step2(d0, tau, 0.1, (1, 1, 0, 0), 1, 20000)
    e = [np.abs(C.step2(d0, tau, 0.1, (2, 2, 4, 4), n, 10)[0] - ref).max() for n in (10, 300)]
    assert e[1] < 0.2 * e[0]


@pytest.mark.parametrize("shape,L", [((21, 19), (2, 3, 3, 4)), ((24, 20), (2, 2, 4, 4)),
                                     ((37, 53), (3, 2, 3, 5)), ((40, 18), (4, 1, 4, 0)),
                                     ((5, 9), (1, 2, 0, 2))])
def test_agrees_with_numpy_oracle(shape, L):
    """Two oracles written independently from the same passages: tau, p, d, p2 and the energies
    agree to rounding on ragged layouts (both steps)."""
    d0 = random_image(*shape, seed=shape[0] * 5 + shape[1]).astype(np.float64)
    lay = layout.Layout(shape[0], shape[1], *L)
    tc, pc, s1 = C.step1(d0, 0.05, L, 3, 3)
    tn, pn, i1 = S.dd_step1(d0, 0.05, lay, 3, 3)
    assert np.abs(tc - tn).max() < 1e-12 and np.abs(pc - pn).max() < 1e-12
    dc, qc, s2 = C.step2(d0, tn, 0.1, L, 3, 4)
    dn, qn, i2 = S.dd_step2(d0, tn, 0.1, lay, 3, 4)
    assert np.abs(dc - dn).max() < 1e-12 and np.abs(qc - qn).max() < 1e-12
    ptau0 = spectral.project(S.tau0(d0))
    assert abs(s1["E"] - S.primal_energy_tfs(tn, ptau0, 0.05)) < 1e-10 * abs(s1["E"])
    alpha, g, _ = S.irv2_data(d0, tn, 0.1)
    assert abs(s2["E"] - S.primal_energy_irv2(dn, d0, g, alpha)) < 1e-10 * abs(s2["E"])
    assert abs(s1["gap"] - S.duality_gap(tn, pn)) < 1e-10 * abs(s1["E"])
    assert abs(s2["D"] - i2["dual_energy"]) < 1e-10 * abs(s2["D"])


def test_threads_do_not_change_the_result():
    """One task per subdomain on POSIX threads: bitwise the sequential result."""
    d0 = random_image(33, 35, 4).astype(np.float64)
    L = (2, 3, 2, 2)
    t1, p1, _ = C.step1(d0, 0.05, L, 3, 2, threads=1)
    t4, p4, _ = C.step1(d0, 0.05, L, 3, 2, threads=4)
    assert np.array_equal(t1, t4) and np.array_equal(p1, p4)
    d1, q1, _ = C.step2(d0, t1, 0.1, L, 3, 4, threads=1)
    d4, q4, _ = C.step2(d0, t1, 0.1, L, 3, 4, threads=6)
    assert np.array_equal(d1, d4) and np.array_equal(q1, q4)


def test_config1_end_to_end_agrees():
    """BASELINE config 1 (64^2 disk on a ramp, 2 x 2, s = 4, 20 x 20 per step) end to end."""
    from tvs_synth import CONFIGS
    c = CONFIGS["c1"]
    d0 = c.image().astype(np.float64)
    L = (c.m2, c.m1, c.overlap, c.overlap)
    lay = layout.Layout(c.n, c.n, *L)
    tc, _, _ = C.step1(d0, c.delta, L, c.sweeps, c.inner, threads=4)
    dc, _, _ = C.step2(d0, tc, c.lam, L, c.sweeps, c.inner, threads=4)
    dn, tn, _, _ = S.dd_denoise(d0, c.delta, c.lam, lay, (c.sweeps, c.inner), (c.sweeps, c.inner))
    assert np.abs(tc - tn).max() < 1e-11 and np.abs(dc - dn).max() < 1e-11
    assert np.abs(ops.div(tc)).max() < 1e-10   # tau in K
