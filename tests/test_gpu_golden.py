"""GPU parity against stored fp64 oracle outputs on BASELINE workloads whose schedules the oracle
cannot rerun inside a test.  Every stored value was written by a committed script under
tests/golden/ that calls only ``oracle/`` (and ``tvs_synth`` for the seeded image):

* c3_full_schedule.npz (make_c3_full.py): config 3 end to end with the FULL bench schedule
  (2048^2, 8 x 8, overlap 16, 50 sweeps x 10 inner per step) -- tau / d at windows over every
  overlap-band crossing and seeded points, and the final energies;
* c4_short_schedule.npz (make_c4_short.py): config 4 at full size (8192^2, 8 strips), 2 sweeps x 2
  (step 1) and 2 x 4 (step 2): the second sweep starts from a nonzero dual;
* c5_step1_sampled.npz (make_c5_sampled.py): config 5 at full size (32768^2, 16 x 16) on one GPU:
  P tau_0 on sampled full rows, and the first sweep's local solves of three subdomains.

Tolerances: the north star's 1e-4 max-abs on tau / d and 1e-4 relative on the primal energies;
the dual p (non-unique minimiser, reading A20) at the diagnostic 1e-2."""
import os

import numpy as np
import pytest

from oracle import layout as olayout
from tvs_synth import CONFIGS

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")
TOL = 1e-4
P_TOL = 1e-2


def _load(name):
    path = os.path.join(GOLD, name)
    if not os.path.exists(path):
        pytest.skip(f"{name} not generated (tests/golden/make_*.py)")
    return np.load(path)


def _log(kind, **kw):
    import json
    path = os.environ.get("TVS_PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps({"check": kind, **{k: float(v) for k, v in kw.items()}}) + "\n")


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2602_17494_b200 as pkg
    c = pkg.Context(0)
    yield c
    c.close()


def _rel(a, b):
    return abs(a - b) / abs(b)


def test_config3_full_bench_schedule(ctx):
    """The bench's config-3 workload end to end (tv_stokes_denoise, 50 x 10 per step) vs the
    oracle's full schedule: tau, d at the stored points, E1 / E2 / D1 / D2 and the gaps."""
    g = _load("c3_full_schedule.npz")
    c = CONFIGS["c3"]
    L = (c.m2, c.m1, c.overlap, c.overlap)
    it = (c.sweeps, c.inner, c.t)
    d0 = torch.from_numpy(c.image()).cuda()
    tau, p1, s1 = ctx.tv_stokes_step1(d0, c.delta, L, it, want_p=True)
    d, p2, s2 = ctx.tv_stokes_step2(tau, d0, c.lam, L, it, want_p=True)
    torch.cuda.synchronize()
    ty, tx = torch.from_numpy(g["tau_rows"]).long().cuda(), torch.from_numpy(g["tau_cols"]).long().cuda()
    dy, dx = torch.from_numpy(g["d_rows"]).long().cuda(), torch.from_numpy(g["d_cols"]).long().cuda()
    e_tau = float(np.abs(tau[:, ty, tx].cpu().numpy().astype(np.float64) - g["tau"]).max())
    e_d = float(np.abs(d[dy, dx].cpu().numpy().astype(np.float64) - g["d"]).max())
    e_p1 = float(np.abs(p1.reshape(2, 2, c.n + 1, c.n + 1)[:, :, ty, tx].cpu().numpy() - g["p1"]).max())
    e_p2 = float(np.abs(p2[:, dy, dx].cpu().numpy() - g["p2"]).max())
    r = {"E1": _rel(s1.primal_energy, float(g["E1"])), "E2": _rel(s2.primal_energy, float(g["E2"])),
         "D1": _rel(s1.dual_energy, float(g["D1"])), "D2": _rel(s2.dual_energy, float(g["D2"]))}
    _log("c3_full_schedule", tau_err=e_tau, d_err=e_d, p1_err=e_p1, p2_err=e_p2, **{k + "_rel": v for k, v in r.items()},
         gap1=s1.gap, gap1_ref=float(g["gap1"]), gap2=s2.gap, gap2_ref=float(g["gap2"]))
    assert e_tau <= TOL, e_tau
    assert e_d <= TOL, e_d
    assert e_p1 <= P_TOL and e_p2 <= P_TOL, (e_p1, e_p2)
    assert all(v <= TOL for v in r.values()), r
    assert abs(s1.gap - float(g["gap1"])) <= TOL * float(g["E1"])
    assert abs(s2.gap - float(g["gap2"])) <= TOL * float(g["E2"])


def test_config4_short_schedule_full_size(ctx):
    """Config 4 at 8192^2 with two sweeps per step: tau / d on the stored rows x columns (every
    strip overlap's first / middle / last row), energies and gaps."""
    g = _load("c4_short_schedule.npz")
    c = CONFIGS["c4"]
    L = (c.m2, c.m1, c.overlap, c.overlap)
    it1 = (int(g["it1"][0]), int(g["it1"][1]), c.t)
    it2 = (int(g["it2"][0]), int(g["it2"][1]), c.t)
    d0 = torch.from_numpy(c.image()).cuda()
    tau, _, s1 = ctx.tv_stokes_step1(d0, c.delta, L, it1)
    d, _, s2 = ctx.tv_stokes_step2(tau, d0, c.lam, L, it2)
    torch.cuda.synchronize()
    tr, tc = torch.from_numpy(g["tau_rows"]).long().cuda(), torch.from_numpy(g["tau_cols"]).long().cuda()
    dr, dc = torch.from_numpy(g["d_rows"]).long().cuda(), torch.from_numpy(g["d_cols"]).long().cuda()
    e_tau = float(np.abs(tau[:, tr][:, :, tc].cpu().numpy().astype(np.float64) - g["tau"]).max())
    e_d = float(np.abs(d[dr][:, dc].cpu().numpy().astype(np.float64) - g["d"]).max())
    r = {"E1": _rel(s1.primal_energy, float(g["E1"])), "E2": _rel(s2.primal_energy, float(g["E2"])),
         "D1": _rel(s1.dual_energy, float(g["D1"])), "D2": _rel(s2.dual_energy, float(g["D2"]))}
    _log("c4_short_schedule", tau_err=e_tau, d_err=e_d, **{k + "_rel": v for k, v in r.items()})
    assert e_tau <= TOL, e_tau
    assert e_d <= TOL, e_d
    assert all(v <= TOL for v in r.values()), r
    assert abs(s1.gap - float(g["gap1"])) <= TOL * float(g["E1"])
    assert abs(s2.gap - float(g["gap2"])) <= TOL * float(g["E2"])


def test_config5_step1_full_size_sampled(ctx):
    """Config 5 step 1 at 32768^2 on ONE GPU (subdomain groups bound the scratch): the 32769^2
    global projection P tau_0 (a 0-update sweep leaves tau = P tau_0) on the stored full rows, and
    after one sweep of two Alg. 5 updates the dual on the rows / columns covered by a single
    subdomain, p^1 = alpha_hat qhat_m, for the three stored subdomains."""
    g = _load("c5_step1_sampled.npz")
    c = CONFIGS["c5"]
    n, nt = c.n, c.n + 1
    L = (c.m2, c.m1, c.overlap, c.overlap)
    lay = olayout.Layout(n, n, *L)
    d0 = torch.from_numpy(c.image()).cuda()
    tau, _, _ = ctx.tv_stokes_step1(d0, c.delta, L, (0, 1, c.t))   # no sweep: tau = P tau_0
    rows = torch.from_numpy(g["ptau0_rows"]).long().cuda()
    cols = torch.from_numpy(g["ptau0_cols"]).long().cuda()
    e_P = float(np.abs(tau[:, rows][:, :, cols].cpu().numpy().astype(np.float64) - g["ptau0"]).max())
    del tau
    _log("c5_global_P", err=e_P)
    assert e_P <= TOL, e_P
    inner = int(g["inner"])
    tau, p, _ = ctx.tv_stokes_step1(d0, c.delta, L, (1, inner, c.t), want_p=True)
    del tau
    p = p.reshape(2, 2, nt, nt)

    def core(ranges, a):
        lo = ranges[a - 1][1] + 1 if a > 0 else 0
        hi = ranges[a + 1][0] - 1 if a + 1 < len(ranges) else nt - 1
        return lo, hi

    for key in ("0_0", "7_9", "15_15"):
        iy, ix = (int(v) for v in key.split("_"))
        r, cc, q = g[f"q_{key}_rows"], g[f"q_{key}_cols"], g[f"q_{key}"]
        ylo, yhi = core(lay.ry, iy)
        xlo, xhi = core(lay.rx, ix)
        sel = (r >= ylo) & (r <= yhi) & (cc >= xlo) & (cc <= xhi)   # single-subdomain points
        assert sel.sum() > 1000, key
        pr = p[:, :, torch.from_numpy(r[sel]).long().cuda(), torch.from_numpy(cc[sel]).long().cuda()]
        e = float(np.abs(pr.cpu().numpy().astype(np.float64) - lay.alpha_hat * q[:, :, sel]).max())
        _log("c5_step1_sweep1", m=iy * 16 + ix, p_err=e)
        assert e <= TOL, (key, e)
