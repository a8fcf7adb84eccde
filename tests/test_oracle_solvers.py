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


# ----------------------------------------------------------------------------- primal energies / gaps (C-13, C-15)

def _feasible(shape, seed):
    """Random dual with every row strictly inside the unit ball (|p_k| <= 1, Eq. eq:DefDisB)."""
    q = random_field(shape, seed, 1.0)
    nrm = np.sqrt(q[..., 0, :, :] ** 2 + q[..., 1, :, :] ** 2) if q.ndim == 4 else np.sqrt(q[0] ** 2 + q[1] ** 2)
    scale = 0.99 / np.maximum(nrm, 1.0)
    return q * (scale[:, None] if q.ndim == 4 else scale)


def _curl_minus(psi):
    """curl^- psi = (D-_y psi, -D-_x psi): divergence-free on any grid (div curl^- = 0, SURVEY C-4)."""
    return np.stack([ops.dminus_y(psi), -ops.dminus_x(psi)])


def test_tfs_energy_gap_identity_for_any_feasible_dual():
    """For EVERY feasible p, with tau(p) = P tau_0 - delta P multidiv p:
    E_1(tau) - G_1(p) = sum_k (TV(tau_k) + <p_k, grad tau_k>) = duality_gap(tau, p) >= 0.
    Three independently written formulas (primal_energy_tfs, dual_value_tfs, duality_gap) must agree
    to rounding: a dropped 1/2, tau_0 in place of P tau_0, or a wrong sign breaks the identity."""
    d0 = random_image(9, 12, 11).astype(np.float64)
    delta = 0.05
    ptau0 = spectral.project(S.tau0(d0))
    for seed in (1, 2, 3):
        p = _feasible((2, 2, 10, 13), 40 + seed)
        tau = ptau0 - delta * spectral.project(ops.multidiv(p))
        e = S.primal_energy_tfs(tau, ptau0, delta)
        g = S.dual_value_tfs(p, ptau0, delta)
        gap = S.duality_gap(tau, p)
        assert gap >= 0.0
        assert abs((e - g) - gap) < 1e-10 * max(1.0, abs(e))
    # tau_0 instead of P tau_0 in the primal data term (the slip of Alg. 1, reading A1) breaks it
    tau0 = S.tau0(d0)
    assert abs(S.primal_energy_tfs(tau, tau0, delta) - S.dual_value_tfs(p, ptau0, delta) - gap) > 1e-3


def test_irv2_energy_gap_identity_for_any_feasible_dual():
    """Same identity for step 2 (Eq. modifiedStep2, dual P:504-510, d = d_0 - div p/alpha
    P:509): E_2(d) - G_2(p) = TV(d - g) + <p, grad(d - g)> = duality_gap(d - g, p) >= 0."""
    d0 = random_image(11, 8, 12).astype(np.float64)
    tau, _ = S.chambolle_tfs(d0, 0.05, 30)
    alpha, g, f = S.irv2_data(d0, tau, 0.1)
    for seed in (4, 5, 6):
        p = _feasible((2, 11, 8), 50 + seed)
        d = d0 - ops.div(p) / alpha
        e = S.primal_energy_irv2(d, d0, g, alpha)
        gv = S.dual_value_irv2(p, d0, g, alpha)
        gap = S.duality_gap(d - g, p)
        assert gap >= 0.0
        assert abs((e - gv) - gap) < 1e-10 * max(1.0, abs(e))


def test_channelwise_tv_dual_attains_zero_gap():
    """The row-wise unit balls of the dual (Alg. 1 row-wise projection P:790) are the dual of
    the CHANNEL-WISE vector TV (reading A15): p_k = -grad u_k/|grad u_k| attains the sup, so the gap
    is 0 to rounding; an isotropic TV would leave sqrt(sum_k |.|^2) - sum_k |.| < 0 here."""
    u = random_field((2, 7, 9), 61, 1.0)
    gr = ops.multigrad(u)
    nrm = np.sqrt(gr[:, 0] ** 2 + gr[:, 1] ** 2)
    p = -gr / np.maximum(nrm, 1e-300)[:, None]
    assert abs(S.duality_gap(u, p)) < 1e-12 * S.tv(u)
    assert abs(S.tv(u) - sum(S.tv(u[k]) for k in range(2))) < 1e-13 * S.tv(u)


def test_tfs_gap_closes_and_bounds_hold_over_chambolle_iterates():
    """Weak duality across iterates: E_1(tau(p_a)) >= G_1(p_b) for all pairs; G_1 is monotone
    (Alg. 1 decreases D); the gap closes over Chambolle's iterates."""
    d0 = disk_on_ramp(16, 1001).astype(np.float64)
    delta = 0.05
    ptau0 = spectral.project(S.tau0(d0))
    es, gs, gaps = [], [], []
    for it in (5, 50, 500, 5000):
        tau, p = S.chambolle_tfs(d0, delta, it)
        es.append(S.primal_energy_tfs(tau, ptau0, delta))
        gs.append(S.dual_value_tfs(p, ptau0, delta))
        gaps.append(S.duality_gap(tau, p))
    assert min(es) >= max(gs) - 1e-9
    assert all(b >= a - 1e-12 for a, b in zip(gs, gs[1:]))
    assert gaps[0] > gaps[1] > gaps[2] > gaps[3] and gaps[3] < 2e-2 * gaps[0]


def test_irv2_gap_closes_over_chambolle_iterates():
    d0 = disk_on_ramp(16, 1001).astype(np.float64)
    tau, _ = S.chambolle_tfs(d0, 0.05, 300)
    alpha, g, _ = S.irv2_data(d0, tau, 0.1)
    es, gs, gaps = [], [], []
    for it in (5, 50, 500, 5000):
        d, p = S.chambolle_irv2(d0, tau, 0.1, it)
        es.append(S.primal_energy_irv2(d, d0, g, alpha))
        gs.append(S.dual_value_irv2(p, d0, g, alpha))
        gaps.append(S.duality_gap(d - g, p))
    assert min(es) >= max(gs) - 1e-9
    assert all(b >= a - 1e-12 for a, b in zip(gs, gs[1:]))
    assert gaps[0] > gaps[1] > gaps[2] > gaps[3] and gaps[3] < 2e-2 * gaps[0]


def test_tfs_primal_energy_is_minimised_at_the_dual_solution():
    """Pins E_1's weights independently of the dual algebra: the long-run Chambolle tau* (computed
    without primal_energy_tfs) minimises E_1 over K up to its gap: E_1(tau* + w) >= E_1(tau*) - gap
    for divergence-free w = curl^- psi, and along the ray c tau* (in K; TV is differentiable along
    it).  Doubling the fit weight moves the minimiser along that ray, so one of c = 1 +- 0.02
    lowers the mis-written energy.  (Fitting tau_0 instead of P tau_0 only adds the constant
    ||(I - P) tau_0||^2 / (2 delta) on K; the identity test above catches that slip.)"""
    d0 = disk_on_ramp(16, 1001).astype(np.float64)
    delta = 0.05
    ptau0 = spectral.project(S.tau0(d0))
    tau, p = S.chambolle_tfs(d0, delta, 20000)
    gap = S.duality_gap(tau, p)
    e0 = S.primal_energy_tfs(tau, ptau0, delta)
    for seed in range(4):
        w = _curl_minus(random_field((17, 17), 70 + seed, 1.0))
        w *= 0.05 / np.abs(w).max()
        assert np.abs(ops.div(w)).max() < 1e-13
        for sgn in (1.0, -1.0):
            assert S.primal_energy_tfs(tau + sgn * w, ptau0, delta) >= e0 - gap - 1e-9
    for c in (0.98, 1.02):
        assert S.primal_energy_tfs(c * tau, ptau0, delta) >= e0 - gap - 1e-9
    wrong = lambda t: S.tv(t) + ops.inner(t - ptau0, t - ptau0) / delta   # noqa: E731 (1/delta)
    assert min(wrong(c * tau) for c in (0.98, 1.02)) < wrong(tau) - 1e-9


def test_irv2_primal_energy_is_minimised_at_the_dual_solution():
    """E_2(d* + h) >= E_2(d*) - gap for perturbations h of the long-run Chambolle d*, including the
    ray d = g + mean(u) + c (u - mean(u)), u = d* - g, along which TV(d - g) is differentiable; a
    dropped 1/2 (alpha ||d - d_0||^2) moves the minimiser along that ray, so one of c = 1 +- 0.02
    lowers the mis-written energy."""
    d0 = disk_on_ramp(16, 1001).astype(np.float64)
    tau, _ = S.chambolle_tfs(d0, 0.05, 300)
    alpha, g, _ = S.irv2_data(d0, tau, 0.1)
    d, p = S.chambolle_irv2(d0, tau, 0.1, 20000)
    gap = S.duality_gap(d - g, p)
    e0 = S.primal_energy_irv2(d, d0, g, alpha)
    for seed in range(4):
        h = random_field((16, 16), 80 + seed, 0.02)
        for sgn in (1.0, -1.0):
            assert S.primal_energy_irv2(d + sgn * h, d0, g, alpha) >= e0 - gap - 1e-9
    u = d - g
    ray = [g + u.mean() + c * (u - u.mean()) for c in (0.98, 1.02)]
    assert all(S.primal_energy_irv2(x, d0, g, alpha) >= e0 - gap - 1e-9 for x in ray)
    wrong = lambda x: S.tv(x - g) + alpha * ops.inner(x - d0, x - d0)   # noqa: E731
    assert min(wrong(x) for x in ray) < wrong(d) - 1e-9


def test_threaded_subdomains_are_bitwise_identical():
    """One task per subdomain on threads (the paper's threading) combines the local solves
    in subdomain order: the DD iterates are bitwise those of the sequential loop."""
    d0 = random_image(21, 19, 13).astype(np.float64)
    lay = layout.Layout(21, 19, 2, 3, 3, 4)
    t1, p1, _ = S.dd_step1(d0, 0.05, lay, 3, 2)
    t4, p4, _ = S.dd_step1(d0, 0.05, lay, 3, 2, workers=4)
    assert np.array_equal(t1, t4) and np.array_equal(p1, p4)
    a1, q1, _ = S.dd_step2(d0, t1, 0.1, lay, 3, 4)
    a4, q4, _ = S.dd_step2(d0, t1, 0.1, lay, 3, 4, workers=4)
    assert np.array_equal(a1, a4) and np.array_equal(q1, q4)
