"""Pins of oracle/solvers.py: tau_0, g, Alg. 1-5, energies (no GPU)."""
import json
import os

import numpy as np
import pytest

from oracle import layout, ops, solvers as S, spectral
from tvs_synth import random_field, random_image, step_image, disk_on_ramp

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "operators.json")))


def test_tau0_divergence_structure():
    """Interior div tau_0 = 0 (mixed differences commute); boundary dual rows/cols are not, so
    tau_0 is not in K in general -- the reason for pre-projecting (reading A1)."""
    d = random_image(7, 9, 3)
    dv = ops.div(S.tau0(d))
    assert np.abs(dv[1:-1, 1:-1]).max() < 1e-15
    assert np.abs(dv).max() > 0.1


def test_g_round_trip():
    """g(tau_0(d_0)) = d_0 - mean (reading A3, C-12): backward-difference integration inverts tau_0."""
    d = random_image(8, 11, 5).astype(np.float64)
    g = S.g_from_tau(S.tau0(d), 8, 11)
    assert np.abs(g - (d - d.mean())).max() < 1e-13


def test_schwarz_1x1_equals_chambolle():
    """Alg. 2 with M = 1x1 (theta = 1, alpha-hat = 1) is S*K Chambolle iterations."""
    d0 = random_image(12, 10, 7).astype(np.float64)
    lay = layout.Layout(12, 10, 1, 1, 0, 0)
    ta, pa, _ = S.dd_step1(d0, 0.05, lay, 5, 4)
    tb, pb = S.chambolle_tfs(d0, 0.05, 20)
    assert np.abs(ta - tb).max() < 1e-12 and np.abs(pa - pb).max() < 1e-12
    da, _, _ = S.dd_step2(d0, tb, 0.1, lay, 5, 4)
    db, _ = S.chambolle_irv2(d0, tb, 0.1, 20)
    assert np.abs(da - db).max() < 1e-12


@pytest.mark.parametrize("m2,m1", [(2, 2), (1, 3), (3, 1)])
def test_localized_tfs_equals_full_grid(m2, m1):
    """Alg. 5 (localized, block-DCT projection) == Alg. 4 (full grid) per subdomain."""
    d0 = random_image(12, 10, 7)
    lay = layout.Layout(12, 10, m2, m1, 2, 2)
    n2t, n1t = 13, 11
    whole = S.full_rect(n2t, n1t)
    p = 0.3 * random_field((2, 2, n2t, n1t), 9)
    f = spectral.project(S.tau0(d0)) / 0.05
    r = f - spectral.project(ops.multidiv(p))
    for m in lay.subdomains():
        s = lay.rect(m, True)
        q0 = 0.2 * random_field((2, 2) + S.rect_shape(s), 11) * S.restrict(lay.theta(m, True), whole, s)
        vl = S._tfs_inner_local(m, lay, p, r, q0, 3, 0.125)
        vg = S.tfs_inner_global(m, lay, p, f, S.extend(q0, s, whole), 3, 0.125)
        assert np.abs(S.extend(vl, s, whole) - vg).max() < 1e-12


@pytest.mark.parametrize("m2,m1", [(2, 2), (1, 3), (3, 1)])
def test_localized_irv2_equals_full_grid(m2, m1):
    d0 = random_image(12, 10, 7)
    lay = layout.Layout(12, 10, m2, m1, 2, 2)
    whole = S.full_rect(12, 10)
    _, _, f = S.irv2_data(d0, S.tau0(d0), 0.1)
    p = 0.3 * random_field((2, 12, 10), 4)
    for m in lay.subdomains():
        s = lay.rect(m, False)
        q0 = 0.2 * random_field((2,) + S.rect_shape(s), 11) * S.restrict(lay.theta(m, False), whole, s)
        vl = S._irv2_inner_local(m, lay, p, f, q0, 4, 0.125)
        vg = S.irv2_inner_global(m, lay, p, f, S.extend(q0, s, whole), 4, 0.125)
        assert np.abs(S.extend(vl, s, whole) - vg).max() < 1e-12


def test_constant_image_fixed_point():
    d0 = np.full((10, 12), 0.37)
    lay = layout.Layout(10, 12, 2, 2, 3, 3)
    tau, p1, _ = S.dd_step1(d0, 0.05, lay, 3, 3)
    assert np.abs(tau).max() == 0 and np.abs(p1).max() == 0
    d, p2, _ = S.dd_step2(d0, tau, 0.1, lay, 3, 3)
    assert np.abs(d - d0).max() < 1e-15


def test_feasibility_and_far_boundary():
    """|p_k| <= 1 pointwise every sweep (B^h); the x-dual on the last column and the
    y-dual on the last row never move (D+ is 0 there)."""
    d0 = random_image(14, 12, 2)
    lay = layout.Layout(14, 12, 2, 2, 4, 4)
    tau, p1, _ = S.dd_step1(d0, 0.05, lay, 4, 5)
    for k in range(2):
        assert np.sqrt(p1[k, 0] ** 2 + p1[k, 1] ** 2).max() <= 1 + 1e-12
        assert np.all(p1[k, 0][:, -1] == 0) and np.all(p1[k, 1][-1, :] == 0)
    d, p2, _ = S.dd_step2(d0, tau, 0.1, lay, 4, 5)
    assert np.sqrt(p2[0] ** 2 + p2[1] ** 2).max() <= 1 + 1e-12
    assert np.all(p2[0][:, -1] == 0) and np.all(p2[1][-1, :] == 0)


def test_tau_divergence_free():
    d0 = random_image(10, 9, 4)
    lay = layout.Layout(10, 9, 2, 2, 3, 3)
    tau, _, _ = S.dd_step1(d0, 0.05, lay, 3, 4)
    assert np.abs(ops.div(tau)).max() < 1e-10


def test_single_domain_monotone_and_gap():
    """Chambolle's dual energy is non-increasing for t <= 1/8 and the duality gap
    (C-15) is >= 0 and decreases towards 0."""
    d0 = random_image(10, 12, 6)
    _, _, e1 = S.chambolle_tfs(d0, 0.05, 60, trace=True)
    assert all(b <= a + 1e-9 * a for a, b in zip(e1, e1[1:]))
    tau, _ = S.chambolle_tfs(d0, 0.05, 400)
    _, _, e2 = S.chambolle_irv2(d0, tau, 0.1, 60, trace=True)
    assert all(b <= a + 1e-9 * a for a, b in zip(e2, e2[1:]))
    gaps = []
    for it in (20, 200, 2000):
        d, p = S.chambolle_irv2(d0, tau, 0.1, it)
        g = S.g_from_tau(tau, 10, 12)
        gaps.append(S.duality_gap(d - g, p))
    assert min(gaps) >= -1e-10 and gaps[0] > gaps[1] > gaps[2]
    gt = []
    for it in (20, 200, 2000):
        t, p = S.chambolle_tfs(d0, 0.05, it)
        gt.append(S.duality_gap(t, p))
    assert min(gt) >= -1e-10 and gt[0] > gt[1] > gt[2]


def test_rof_step_closed_form():
    """tau = 0 reduces IRV2 to ROF; the vertical step has the exact solution 1/(aL), 1 - 1/(aR)."""
    g = GOLD["rof_step"]
    d0 = step_image(g["n2"], g["left"] + g["right"], g["left"])
    tau = np.zeros((2, g["n2"] + 1, g["left"] + g["right"] + 1))
    d, _ = S.chambolle_irv2(d0, tau, 1.0 / g["alpha"], 4000)
    assert np.abs(d[:, :g["left"]] - g["low"]).max() < 1e-6
    assert np.abs(d[:, g["left"]:] - g["high"]).max() < 1e-6


def test_dd_irv2_converges_to_single_domain():
    """Alg. 2 converges to the single-domain solution (O(n^-1/2)) on a tiny image."""
    d0 = random_image(16, 16, 8)
    tau = S.tau0(d0) * 0.0
    lay = layout.Layout(16, 16, 2, 2, 4, 4)
    d_ref, _ = S.chambolle_irv2(d0, tau, 0.1, 20000)
    errs = []
    for sweeps in (20, 200, 800):
        d, _, _ = S.dd_step2(d0, tau, 0.1, lay, sweeps, 10)
        errs.append(np.abs(d - d_ref).max())
    assert errs[0] > errs[1] > errs[2] and errs[2] < 2e-3


def test_dd_tfs_converges_to_single_domain():
    d0 = random_image(10, 10, 9)
    lay = layout.Layout(10, 10, 2, 2, 3, 3)
    t_ref, _ = S.chambolle_tfs(d0, 0.05, 6000)
    errs = []
    for sweeps in (10, 60, 240):
        t, _, _ = S.dd_step1(d0, 0.05, lay, sweeps, 10)
        errs.append(np.abs(t - t_ref).max())
    assert errs[0] > errs[1] > errs[2]


def test_dd_energy_monotone_diagnostic():
    """Reading A18: monotone DD energy is a diagnostic (held in all our runs)."""
    d0 = disk_on_ramp(32, 11)
    lay = layout.Layout(32, 32, 2, 2, 4, 4)
    _, _, info = S.dd_step1(d0, 0.05, lay, 10, 5, trace=True)
    e = info["energies"]
    assert all(b <= a * (1 + 1e-9) for a, b in zip(e, e[1:]))
    tau = S.dd_step1(d0, 0.05, lay, 10, 5)[0]
    _, _, info2 = S.dd_step2(d0, tau, 0.1, lay, 10, 5, trace=True)
    e = info2["energies"]
    assert all(b <= a * (1 + 1e-9) for a, b in zip(e, e[1:]))


# ----------------------------------------------------------------------------- IRV1 (NEXT row 2)

def test_xi_is_smoothed_unit_normal_of_a_ramp():
    """tau_0 = grad^perp d_0 so tau_0^perp = (tau_2, -tau_1) = grad d_0 and xi of Eq.
    defXi2:discrete is the smoothed unit normal: for the x-ramp d_0 = c j every
    interior xi equals (c / sqrt(c^2 + eps), 0).  Pins the perp orientation and the eps placement."""
    c, eps = 0.3, 1e-3
    d0 = c * np.tile(np.arange(9, dtype=np.float64), (7, 1))
    xi = S.xi_from_tau(S.tau0(d0), 7, 9, eps)
    assert np.allclose(xi[0][:, 1:], c / np.sqrt(c * c + eps), atol=1e-15)
    assert np.abs(xi[1]).max() == 0.0
    assert np.all(xi[0][:, 0] == 0.0)      # tau_0's zero Neumann column


def test_xi_strictly_inside_unit_ball():
    """||xi||_inf < 1 holds automatically for eps > 0 (Rem. IRPW11)."""
    tau = random_field((2, 12, 15), 4, 3.0)
    xi = S.xi_from_tau(tau, 11, 14, 1e-3)
    assert np.sqrt(xi[0] ** 2 + xi[1] ** 2).max() < 1.0


def test_irv1_with_zero_tangent_field_is_rof():
    """tau = 0 gives xi = 0, so IRV1 and IRV2 (g = 0) are both the ROF dual of
    Chambolle 2004 with alpha = 1/mu = 1/lambda (reading A4): identical iterates."""
    d0 = random_image(9, 11, 3).astype(np.float64)
    tau = np.zeros((2, 10, 12))
    d1, p1 = S.chambolle_irv1(d0, tau, 0.1, 1e-3, 50)
    d2, p2 = S.chambolle_irv2(d0, tau, 0.1, 50)
    assert np.abs(d1 - d2).max() < 1e-14 and np.abs(p1 - p2).max() < 1e-14


def test_irv1_weak_duality_gap_closes():
    """Weak duality between Eq. IRPXi and the dual of Cor. irdual:
    E(d) >= G(p) for every feasible p; Chambolle's iterates drive E(d(p)) - G(p) to 0.  A wrong
    sign or a dropped div xi in f or in the recovery d = d_0 - (div p + div xi)/alpha leaves a
    gap that does not close."""
    d0 = disk_on_ramp(16, 1001).astype(np.float64)
    tau, _ = S.chambolle_tfs(d0, 0.05, 300)
    mu, eps = 0.1, 1e-3
    alpha, dxi, f = S.irv1_data(d0, tau, mu, eps)
    gaps = []
    for it in (10, 100, 3000):
        d, p = S.chambolle_irv1(d0, tau, mu, eps, it)
        gaps.append(S.primal_energy_irv1(d, d0, dxi, alpha) - S.dual_value_irv1(p, d0, f, alpha))
    assert min(gaps) >= -1e-9
    assert gaps[0] > gaps[1] > gaps[2] and gaps[2] < 1e-3 * gaps[0]


def test_irv1_schwarz_1x1_equals_chambolle_and_dd_converges():
    """Alg. 2 with one subdomain is plain Chambolle (alpha_hat = 1, theta = 1), and the 2 x 2 DD
    iterate approaches the single-domain IRV1 solution."""
    d0 = random_image(12, 12, 8).astype(np.float64)
    tau, _ = S.chambolle_tfs(d0, 0.05, 100)
    one = layout.Layout(12, 12, 1, 1, 0, 0)
    d_dd, _, _ = S.dd_step2(d0, tau, 0.1, one, 6, 5, variant="irv1")
    d_ch, _ = S.chambolle_irv1(d0, tau, 0.1, 1e-3, 30)
    assert np.abs(d_dd - d_ch).max() < 1e-13
    ref, _ = S.chambolle_irv1(d0, tau, 0.1, 1e-3, 20000)
    lay = layout.Layout(12, 12, 2, 2, 4, 4)
    e = [np.abs(S.dd_step2(d0, tau, 0.1, lay, n, 10, variant="irv1")[0] - ref).max()
         for n in (10, 300)]
    assert e[1] < 0.2 * e[0]


# ----------------------------------------------------------------------------- stopping rules (NEXT 3)

def test_stopping_rules_bracket_the_fixed_schedule():
    """tol = 0 never fires (the fixed schedule, reading A10); a huge tol fires after the first
    comparison (step 2: after sweep 1, step 1: before sweep 2's inner loop, i.e. 1 sweep run); the
    sweep at which criterion 1 fires is the first n with |D_n^{1/2} - D_{n+1}^{1/2}| below
    |Omega|^{1/2} tol, recomputed here from the traced energies."""
    d0 = random_image(14, 13, 3).astype(np.float64)
    lay = layout.Layout(14, 13, 2, 2, 3, 3)
    tau, _ = S.chambolle_tfs(d0, 0.05, 50)
    _, _, i0 = S.dd_step2(d0, tau, 0.1, lay, 12, 4, stop=(1, 0.0))
    assert i0["sweeps_run"] == 12
    _, _, i1 = S.dd_step2(d0, tau, 0.1, lay, 12, 4, stop=(1, 1e9))
    assert i1["sweeps_run"] == 1
    _, _, tr = S.dd_step2(d0, tau, 0.1, lay, 12, 4, trace=True)
    e = [S.ops.inner(S.step2_data(d0, tau, 0.1)[1], S.step2_data(d0, tau, 0.1)[1])] + tr["energies"]
    crit = [abs(np.sqrt(a) - np.sqrt(b)) / np.sqrt(14 * 13) for a, b in zip(e, e[1:])]
    tol = 0.5 * (crit[4] + crit[5])
    assert crit[5] < tol and all(c > tol for c in crit[:5])   # the criterion decreases here
    _, _, i2 = S.dd_step2(d0, tau, 0.1, lay, 12, 4, stop=(1, tol))
    assert i2["sweeps_run"] == 6
    _, _, j0 = S.dd_step1(d0, 0.05, lay, 4, 3, stop=(2, 0.0))
    assert j0["sweeps_run"] == 4
    _, _, j1 = S.dd_step1(d0, 0.05, lay, 4, 3, stop=(2, 1e30))
    assert j1["sweeps_run"] == 1


def test_reported_dual_energy_is_the_objective():
    """info['dual_energy'] is D(p) of Eqs. tfsdualdis / ir2dualdis of the returned p."""
    d0 = random_image(10, 11, 5).astype(np.float64)
    lay = layout.Layout(10, 11, 2, 2, 3, 3)
    tau, p1, i1 = S.dd_step1(d0, 0.05, lay, 3, 3)
    assert abs(i1["dual_energy"] - S.dual_energy_tfs(p1, i1["f"])) < 1e-10 * i1["dual_energy"]
    d, p2, i2 = S.dd_step2(d0, tau, 0.1, lay, 3, 3)
    assert abs(i2["dual_energy"] - S.dual_energy_irv2(p2, i2["f"])) < 1e-10 * i2["dual_energy"]
