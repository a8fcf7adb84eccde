"""Full-size parity at BASELINE configs 4 (8192^2, 8 strips, s = 32) and 5 (32768^2, 16 x 16,
s = 32), in the launch configuration of the library (SURVEY 8(d) "sampled parity").

The oracle cannot run these schedules end to end, so the CUDA path is compared with it on outputs
the oracle can compute one subdomain at a time: after the first outer sweep (p^0 = 0, qhat = 0,
Alg. 2) the dual on the rows/columns covered by a single subdomain m is exactly
p^1 = alpha_hat * qhat_m, and qhat_m is the local solve of m alone (Alg. 3 / Alg. 5 with
omega0 = R_{S+} r^0).  After the full schedule the checks are properties that hold at any size:
feasibility |p_k| <= 1, finiteness, d = d_0 - div p / alpha on sampled
windows, div tau = 0.

Inputs: the seeded synthetic images of tvs_synth; step 2 is fed the oracle's
projected tangent field P tau_0 (config 4) or tau = 0 (config 5: IRV2 reduces to the ROF dual,
P:472-510 with g constant)."""
import numpy as np
import pytest

from oracle import layout as olayout, ops, solvers as S, spectral
from tvs_synth import CONFIGS

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-4


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2602_17494_b200 as pkg
    c = pkg.Context(0)
    yield c
    c.close()


_IMG = {}


def _log(kind, **kw):
    import json
    import os
    path = os.environ.get("TVS_PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps({"check": kind, **{k: (float(v) if isinstance(v, (float, np.floating))
                                                     else v) for k, v in kw.items()}}) + "\n")


def _image(name):
    if name not in _IMG:
        _IMG[name] = CONFIGS[name].image()
    return _IMG[name]


def _core(ranges, a, n):
    """Rows (inclusive) of axis range a covered by no other subdomain, clipped to [0, n-1]."""
    lo = ranges[a - 1][1] + 1 if a > 0 else 0
    hi = ranges[a + 1][0] - 1 if a + 1 < len(ranges) else n - 1
    return lo, min(hi, n - 1)


def _layout(c):
    return (c.m2, c.m1, c.overlap, c.overlap)


# ----------------------------------------------------------------------------- config 4

_TAU4 = {}


@pytest.mark.parametrize("variant,strips", [("irv2", (0, 5, 7)), ("irv1", (0, 5))])
def test_config4_step2_first_sweep_sampled(ctx, variant, strips):
    c = CONFIGS["c4"]
    img = _image("c4")
    d0 = img.astype(np.float64)
    n = c.n
    lay = olayout.Layout(n, n, *_layout(c))
    if "tau" not in _TAU4:
        _TAU4["tau"] = spectral.project(S.tau0(d0)).astype(np.float32)
    tau32 = _TAU4["tau"]
    d_g, p_g, _ = ctx.tv_stokes_step2(torch.from_numpy(tau32).cuda(), torch.from_numpy(img).cuda(),
                                      c.lam, _layout(c), (1, c.inner, c.t), want_p=True,
                                      variant=variant, eps=1e-3)
    alpha, f, shift = S.step2_data(d0, tau32.astype(np.float64), c.lam, variant, 1e-3)
    full = S.full_rect(n, n)
    ry = [(a, min(b, n - 1)) for a, b in lay.ry]
    for a in strips:
        m = (a, 0)
        s = lay.rect(m, extended=False)
        sp = S.rect_plus(s, n, n)
        omega0 = S.restrict(f, full, sp)                     # p^0 = 0
        v = S.irv2_local_iterations(lay, m, omega0, np.zeros((2,) + S.rect_shape(s)), c.inner, c.t)
        lo, hi = _core(ry, a, n)
        y0 = s[0][0]
        p_ref = lay.alpha_hat * v[:, lo - y0:hi - y0 + 1, :]
        p_gpu = p_g[:, lo:hi + 1, :].cpu().numpy().astype(np.float64)
        e_p = np.abs(p_gpu - p_ref).max()
        # d on rows whose div stencil (rows i-1, i) lies in the core
        d_ref = d0[lo + 1:hi] - (ops.div(p_ref)[1:-1] + shift[lo + 1:hi]) / alpha
        e_d = np.abs(d_g[lo + 1:hi].cpu().numpy() - d_ref).max()
        _log(f"c4_step2_{variant}_sweep1", m=list(m), p_err=e_p, d_err=e_d)
        assert e_p <= TOL, (m, e_p)
        assert e_d <= TOL, (m, e_d)


def test_config4_step2_full_schedule_properties(ctx):
    c = CONFIGS["c4"]
    img = _image("c4")
    n = c.n
    tau = torch.zeros((2, n + 1, n + 1), device="cuda")
    d_g, p_g, st = ctx.tv_stokes_step2(tau, torch.from_numpy(img).cuda(), c.lam, _layout(c),
                                       (c.sweeps, c.inner, c.t), want_p=True)
    assert st.pixel_updates > 0
    assert torch.isfinite(p_g).all() and torch.isfinite(d_g).all()
    # |p_k| <= 1 up to fp32 rounding of the update and of theta (sum theta = 1 +- ulp)
    assert float(torch.sqrt(p_g[0] ** 2 + p_g[1] ** 2).max()) <= 1.0 + 1e-5
    alpha = 1.0 / c.lam
    for r0, c0 in ((0, 0), (n // 3, n // 2), (n - 300, n - 300)):
        pw = p_g[:, r0:r0 + 300, c0:c0 + 300].cpu().numpy().astype(np.float64)
        d_chk = img[r0:r0 + 300, c0:c0 + 300].astype(np.float64) - ops.div(pw) / alpha
        err = np.abs(d_g[r0:r0 + 300, c0:c0 + 300].cpu().numpy() - d_chk)[1:-1, 1:-1].max()
        assert err <= 1e-5, ((r0, c0), err)


def test_config4_step1_first_sweep_sampled(ctx):
    """Step 1 at 8192^2: one sweep of two Alg. 5 updates (the second applies the local
    projection, kernel (b), to a full 1056 x 8193 strip); tau = delta r^1 must be divergence-free."""
    c = CONFIGS["c4"]
    img = _image("c4")
    d0 = img.astype(np.float64)
    n = c.n
    nt = n + 1
    lay = olayout.Layout(n, n, *_layout(c))
    tau_g, p_g, _ = ctx.tv_stokes_step1(torch.from_numpy(img).cuda(), c.delta, _layout(c),
                                        (1, 2, c.t), want_p=True)
    f = spectral.project(S.tau0(d0)) / c.delta
    p0 = np.zeros((2, 2, nt, nt))
    for a in (0, 4):
        m = (a, 0)
        s = lay.rect(m, extended=True)
        v = S._tfs_inner_local(m, lay, p0, f, np.zeros((2, 2) + S.rect_shape(s)), 2, c.t)
        lo, hi = _core(lay.ry, a, nt)
        y0 = s[0][0]
        p_ref = lay.alpha_hat * v[:, :, lo - y0:hi - y0 + 1, :]
        p_gpu = p_g.reshape(2, 2, nt, nt)[:, :, lo:hi + 1, :].cpu().numpy().astype(np.float64)
        e_p = np.abs(p_gpu - p_ref).max()
        assert e_p <= TOL, (m, e_p)
    # tau = delta r^1 is divergence-free up to the fp32 projection error
    e_div = np.abs(ops.div(tau_g.cpu().numpy().astype(np.float64))).max()
    _log("c4_step1_div_tau", div=e_div)
    assert e_div <= TOL, e_div
    # the global projection alone at full size: sweeps = 1, inner = 0 leaves p = 0 and
    # tau = P tau_0 = delta f (element-wise parity of the 8193^2 projection)
    tau_p, _, _ = ctx.tv_stokes_step1(torch.from_numpy(img).cuda(), c.delta, _layout(c), (1, 0, c.t))
    e_P = np.abs(tau_p.cpu().numpy().astype(np.float64) - c.delta * f).max()
    _log("c4_global_P", err=e_P)
    assert e_P <= TOL, e_P


# ----------------------------------------------------------------------------- config 5

def test_config5_step2_sampled_and_properties(ctx):
    """32768^2 (1.07 G pixels), 16 x 16 subdomains of ~2080^2, on one GPU."""
    c = CONFIGS["c5"]
    img = _image("c5")
    n = c.n
    lay = olayout.Layout(n, n, *_layout(c))
    d0_dev = torch.from_numpy(img).cuda()
    tau = torch.zeros((2, n + 1, n + 1), device="cuda")
    d_g, p_g, _ = ctx.tv_stokes_step2(tau, d0_dev, c.lam, _layout(c), (1, c.inner, c.t),
                                      want_p=True)
    ry = [(a, min(b, n - 1)) for a, b in lay.ry]
    rx = [(a, min(b, n - 1)) for a, b in lay.rx]
    for m in ((0, 0), (7, 9), (15, 15)):
        s = lay.rect(m, extended=False)
        sp = S.rect_plus(s, n, n)
        (y0, _), (x0, _) = s
        (py0, py1), (px0, px1) = sp
        crop = img[py0:py1 + 1, px0:px1 + 1].astype(np.float64)
        # tau = 0 integrates to g = 0 (reading A3), so f = alpha d_0; p^0 = 0 gives omega0 = R f
        _, _, omega0 = S.irv2_data(crop, np.zeros((2,) + tuple(x + 1 for x in crop.shape)), c.lam)
        v = S.irv2_local_iterations(lay, m, omega0, np.zeros((2,) + S.rect_shape(s)), c.inner, c.t)
        ylo, yhi = _core(ry, m[0], n)
        xlo, xhi = _core(rx, m[1], n)
        p_ref = lay.alpha_hat * v[:, ylo - y0:yhi - y0 + 1, xlo - x0:xhi - x0 + 1]
        p_gpu = p_g[:, ylo:yhi + 1, xlo:xhi + 1].cpu().numpy().astype(np.float64)
        e_p = np.abs(p_gpu - p_ref).max()
        _log("c5_step2_sweep1", m=list(m), p_err=e_p)
        assert e_p <= TOL, (m, e_p)
    del d_g, p_g
    # full schedule: properties that hold at any size
    d_g, p_g, st = ctx.tv_stokes_step2(tau, d0_dev, c.lam, _layout(c), (c.sweeps, c.inner, c.t),
                                       want_p=True)
    assert torch.isfinite(d_g).all()
    nrm = torch.sqrt(p_g[0] ** 2 + p_g[1] ** 2)
    assert float(nrm.max()) <= 1.0 + 1e-5
    del nrm
    alpha = 1.0 / c.lam
    for r0, c0 in ((0, 0), (n // 2, n // 3), (n - 256, n - 256)):
        pw = p_g[:, r0:r0 + 256, c0:c0 + 256].cpu().numpy().astype(np.float64)
        d_chk = img[r0:r0 + 256, c0:c0 + 256].astype(np.float64) - ops.div(pw) / alpha
        err = np.abs(d_g[r0:r0 + 256, c0:c0 + 256].cpu().numpy() - d_chk)[1:-1, 1:-1].max()
        assert err <= 1e-5, ((r0, c0), err)


# ----------------------------------------------------------------------------- config 5, 1-GPU size

def test_config5_weak1_step1_sampled(ctx):
    """Config 5 at its one-GPU weak-scaling size (11585^2, 16 x 16 subdomains of ~745^2, s = 32;
    reading A16): the 11586^2 global projection P tau_0 element-wise, one sweep of two Alg. 5
    updates on three subdomains (corner, edge, interior), div tau = 0.  N = 11586 > 4096, so every
    projection batch runs the chirp-z x-DCTs."""
    c = CONFIGS["c5w1"]
    img = _image("c5w1")
    d0 = img.astype(np.float64)
    n = c.n
    nt = n + 1
    lay = olayout.Layout(n, n, *_layout(c))
    d0_dev = torch.from_numpy(img).cuda()
    tau_p, _, _ = ctx.tv_stokes_step1(d0_dev, c.delta, _layout(c), (1, 0, c.t))
    f = spectral.project(S.tau0(d0)) / c.delta
    e_P = np.abs(tau_p.cpu().numpy().astype(np.float64) - c.delta * f).max()
    _log("c5w1_global_P", err=e_P)
    assert e_P <= TOL, e_P
    del tau_p
    tau_g, p_g, _ = ctx.tv_stokes_step1(d0_dev, c.delta, _layout(c), (1, 2, c.t), want_p=True)
    p0 = np.zeros((2, 2, nt, nt))
    for m in ((0, 0), (0, 7), (9, 6)):
        s = lay.rect(m, extended=True)
        v = S._tfs_inner_local(m, lay, p0, f, np.zeros((2, 2) + S.rect_shape(s)), 2, c.t)
        ylo, yhi = _core(lay.ry, m[0], nt)
        xlo, xhi = _core(lay.rx, m[1], nt)
        (y0, _), (x0, _) = s
        p_ref = lay.alpha_hat * v[:, :, ylo - y0:yhi - y0 + 1, xlo - x0:xhi - x0 + 1]
        p_gpu = (p_g.reshape(2, 2, nt, nt)[:, :, ylo:yhi + 1, xlo:xhi + 1]
                 .cpu().numpy().astype(np.float64))
        e_p = np.abs(p_gpu - p_ref).max()
        _log("c5w1_step1_sweep1", m=list(m), p_err=e_p)
        assert e_p <= TOL, (m, e_p)
    e_div = np.abs(ops.div(tau_g.cpu().numpy().astype(np.float64))).max()
    _log("c5w1_step1_div_tau", div=e_div)
    assert e_div <= TOL, e_div


def test_config4_bench_schedule_energies_oracle_evaluated(ctx):
    """The bench workload exactly (config 4, 30 x 20 per step, both steps, bench.py's headline):
    the library's E_1, D_1, gap_1 (step 1) and E_2, D_2, gap_2 (step 2) -- fixed-order fp64
    reductions on the device -- against the oracle's energy functions evaluated in fp64 on the
    library's own outputs tau, p^1, d, p^2 (E_1 P:249, D_TFS P:675 with f = P tau_0 / delta from
    the oracle's global projection, E_2 P:475-479 with g from the oracle's integration of tau, D_IRV2
    P:679, gap SURVEY C-15), at the north star's 1e-4 relative; and weak duality G <= E for both
    steps with the oracle's dual objectives (Cor. tfsdual P:240-250, the ROF dual P:504-510)."""
    c = CONFIGS["c4"]
    d0 = _image("c4")
    L = _layout(c)
    d0_dev = torch.from_numpy(d0).cuda()
    tau_g, p1_g, s1 = ctx.tv_stokes_step1(d0_dev, c.delta, L, (c.sweeps, c.inner, c.t), want_p=True)
    d_g, p2_g, s2 = ctx.tv_stokes_step2(tau_g, d0_dev, c.lam, L, (c.sweeps, c.inner, c.t), want_p=True)
    torch.cuda.synchronize()
    assert s1.pixel_updates > 0 and s2.pixel_updates > 0
    tau = tau_g.cpu().numpy().astype(np.float64)
    p1 = p1_g.cpu().numpy().astype(np.float64).reshape(2, 2, *tau.shape[1:])
    d = d_g.cpu().numpy().astype(np.float64)
    p2 = p2_g.cpu().numpy().astype(np.float64)
    del tau_g, p1_g, d_g, p2_g
    d0 = d0.astype(np.float64)
    ptau0 = spectral.project(S.tau0(d0))
    e1 = S.primal_energy_tfs(tau, ptau0, c.delta)
    dd1 = S.dual_energy_tfs(p1, ptau0 / c.delta)
    g1 = S.duality_gap(tau, p1)
    G1 = S.dual_value_tfs(p1, ptau0, c.delta)
    del ptau0
    alpha, g, f2 = S.irv2_data(d0, tau, c.lam)
    e2 = S.primal_energy_irv2(d, d0, g, alpha)
    dd2 = S.dual_energy_irv2(p2, f2)
    g2 = S.duality_gap(d - g, p2)
    G2 = S.dual_value_irv2(p2, d0, g, alpha)
    r = {"E1": _rel_(s1.primal_energy, e1), "D1": _rel_(s1.dual_energy, dd1),
         "E2": _rel_(s2.primal_energy, e2), "D2": _rel_(s2.dual_energy, dd2)}
    _log("c4_bench_schedule_energies", gap1=s1.gap, gap1_ref=g1, gap2=s2.gap, gap2_ref=g2,
         G1=G1, G2=G2, **{k + "_rel": v for k, v in r.items()})
    assert all(v <= TOL for v in r.values()), r
    assert abs(s1.gap - g1) <= TOL * e1, (s1.gap, g1)
    assert abs(s2.gap - g2) <= TOL * e2, (s2.gap, g2)
    # weak duality on the oracle's side (fp64): the dual objective never exceeds the primal
    assert G1 <= e1 * (1 + 1e-12), (G1, e1)
    assert G2 <= e2 * (1 + 1e-12), (G2, e2)


def _rel_(a, b):
    return abs(a - b) / abs(b)
