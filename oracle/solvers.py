"""TV-Stokes dual iterations: Chambolle (Alg. 1), overlapping Schwarz (Alg. 2) with the IRV2
inner loop (Alg. 3) and the TFS inner loops (Alg. 4 full-grid, Alg. 5 localized), fp64.

Oracle: test infrastructure only (see oracle/__init__.py).  Each function cites the passage it
follows; readings A1..A21 are listed in DESIGN.md.  Rectangles are ((y0, y1), (x0, x1)) inclusive
0-based global indices.  Fields: scalar (n2, n1); vector (2, n2, n1) with [0] = x-component;
2x2 multi-field (2, 2, n2, n1) with [k] = row p_k.
"""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import ops, spectral
from .layout import Layout


def map_subdomains(fn, subs, workers=1):
    """[fn(m) for m in subs], optionally on ``workers`` threads: one task per subdomain, the
    paper's own parallelisation ("multi-threading, where each thread processes only a local
    portion of the image").  The local solves of one outer sweep are independent
    (Alg. 2 is additive) and their results are combined by the caller in subdomain
    order, so the output is bitwise the same for every ``workers``.  NumPy releases the GIL in
    its kernels; BLAS threads are split between the workers."""
    subs = list(subs)
    if workers <= 1 or len(subs) <= 1:
        return [fn(m) for m in subs]
    from threadpoolctl import threadpool_limits
    workers = min(workers, len(subs))
    with threadpool_limits(limits=max(1, (os.cpu_count() or 1) // workers), user_api="blas"):
        with ThreadPoolExecutor(max_workers=workers) as ex:
            return list(ex.map(fn, subs))

# ----------------------------------------------------------------------------- rect helpers


def rect_plus(rect, n2, n1):
    """A_+ (reading A12): one more row below and one more column to the right,
    clipped at the global edge (grid n2 x n1)."""
    (y0, y1), (x0, x1) = rect
    return (y0, min(y1 + 1, n2 - 1)), (x0, min(x1 + 1, n1 - 1))


def rect_shape(rect):
    (y0, y1), (x0, x1) = rect
    return (y1 - y0 + 1, x1 - x0 + 1)


def restrict(arr, outer, inner):
    """R_inner of an array living on rectangle ``outer`` (last two axes are (y, x))."""
    (oy0, _), (ox0, _) = outer
    (iy0, iy1), (ix0, ix1) = inner
    return arr[..., iy0 - oy0:iy1 - oy0 + 1, ix0 - ox0:ix1 - ox0 + 1]


def extend(arr, inner, outer):
    """E_inner into rectangle ``outer``: zero outside ``inner``."""
    (oy0, oy1), (ox0, ox1) = outer
    (iy0, iy1), (ix0, ix1) = inner
    out = np.zeros(arr.shape[:-2] + (oy1 - oy0 + 1, ox1 - ox0 + 1), dtype=np.float64)
    out[..., iy0 - oy0:iy1 - oy0 + 1, ix0 - ox0:ix1 - ox0 + 1] = arr
    return out


def full_rect(n2, n1):
    return (0, n2 - 1), (0, n1 - 1)


# ----------------------------------------------------------------------------- data of the steps


def tau0(d0):
    """tau_0 = (-D_y^{neum-} d_0, D_x^{neum-} d_0)^T on Omega~ (Eq. def:backdiffNeumann)."""
    return np.stack([-ops.dneum_y(d0), ops.dneum_x(d0)])


def g_from_tau(tau, n2, n1):
    """g on Omega with backward differences (D-_x g, D-_y g)^T = (R_Omega tau)^perp, reading A3
    (P:681 and P:689): g_{i,j} - g_{i,j-1} = tau_2[i,j] (j >= 1), g_{i,j} - g_{i-1,j} = -tau_1[i,j]
    (i >= 1), g_{0,0} = 0, integrated along row 0 then down each column; returned zero-mean
    (the constant does not change the minimiser)."""
    t1 = np.asarray(tau[0], np.float64)
    t2 = np.asarray(tau[1], np.float64)
    g = np.zeros((n2, n1), dtype=np.float64)
    for j in range(1, n1):
        g[0, j] = g[0, j - 1] + t2[0, j]
    for i in range(1, n2):
        g[i, :] = g[i - 1, :] - t1[i, :n1]
    return g - g.mean()


def rowwise_update(v, psi, theta, t):
    """v_k <- (theta v_k + t theta psi_k) / (theta + t |psi_k|) per row k (Alg. 3/5, P:1349-1352,
    P:1746-1749); theta = 0 gives v = 0 (reading A13).  Works for v of shape (2, ..) [one row] or
    (2, 2, ..) [two rows]."""
    v = np.asarray(v, np.float64)
    psi = np.asarray(psi, np.float64)
    if v.ndim == 3:
        nrm = np.sqrt(psi[0] ** 2 + psi[1] ** 2)
        den = theta + t * nrm
        out = np.zeros_like(v)
        ok = theta > 0
        for c in range(2):
            out[c][ok] = (theta[ok] * v[c][ok] + t * theta[ok] * psi[c][ok]) / den[ok]
        return out
    return np.stack([rowwise_update(v[k], psi[k], theta, t) for k in range(v.shape[0])])


# ----------------------------------------------------------------------------- Alg. 1 (single domain)


def chambolle_tfs(d0, delta, iters, t=0.125, p0=None, trace=False):
    """Alg. 1 with tau_0 pre-projected (reading A1, decision P:252):
    psi = multigrad(P multidiv p - delta^{-1} P tau_0); p_k <- (p_k + t psi_k)/(1 + t |psi_k|)."""
    n2, n1 = d0.shape
    f = spectral.project(tau0(d0)) / delta
    p = np.zeros((2, 2, n2 + 1, n1 + 1)) if p0 is None else np.array(p0, np.float64)
    one = np.ones((n2 + 1, n1 + 1))
    energies = []
    for _ in range(iters):
        r = spectral.project(ops.multidiv(p)) - f
        if trace:
            energies.append(ops.inner(r, r))
        p = rowwise_update(p, ops.multigrad(r), one, t)
    tau = delta * (f - spectral.project(ops.multidiv(p)))      # tau = P tau0 - delta P multidiv p
    return (tau, p, energies) if trace else (tau, p)


def irv2_data(d0, tau, lam):
    """alpha = 1/lambda (reading A4), g from tau (A3), f = alpha (d_0 - g) (Eq. ir2dualdis)."""
    n2, n1 = d0.shape
    alpha = 1.0 / lam
    g = g_from_tau(tau, n2, n1)
    return alpha, g, alpha * (np.asarray(d0, np.float64) - g)


def xi_from_tau(tau, n2, n1, eps):
    """xi^h of Eq. defXi2:discrete: tau_perp = R_Omega (tau_2, -tau_1) and
    xi = tau_perp / sqrt(|tau_perp|^2 + eps) pointwise on Omega (N2 x N1)."""
    t1 = np.asarray(tau[0], np.float64)[:n2, :n1]
    t2 = np.asarray(tau[1], np.float64)[:n2, :n1]
    den = np.sqrt(t2 ** 2 + t1 ** 2 + eps)
    return np.stack([t2 / den, -t1 / den])


def irv1_data(d0, tau, mu, eps):
    """IRV1 (Eq. ir1dualdis): alpha = 1/mu, xi from tau (Eq. defXi2:discrete),
    f = alpha d_0 - div xi.  Returns (alpha, div xi, f)."""
    n2, n1 = d0.shape
    alpha = 1.0 / mu
    dxi = ops.div(xi_from_tau(tau, n2, n1, eps))
    return alpha, dxi, alpha * np.asarray(d0, np.float64) - dxi


def step2_data(d0, tau, lam, variant="irv2", eps=1e-3):
    """Data of the step-2 dual min ||div p - f||^2 and the shift of the primal recovery
    d = d_0 - (div p + shift) / alpha: IRV2 (f = alpha (d_0 - g), shift 0) or IRV1
    (f = alpha d_0 - div xi, shift = div xi, Eq. tau_hat)."""
    if variant == "irv1":
        alpha, dxi, f = irv1_data(d0, tau, lam, eps)
        return alpha, f, dxi
    alpha, _, f = irv2_data(d0, tau, lam)
    return alpha, f, np.zeros_like(f)


def chambolle_irv1(d0, tau, mu, eps, iters, t=0.125, trace=False):
    """Chambolle's iteration for the IRV1 dual (Cor. irdual P:403-417, Eq. ir1dualdis):
    psi = grad(div p - f), p <- (p + t psi)/(1 + t |psi|); d = d_0 - (div p + div xi)/alpha."""
    n2, n1 = d0.shape
    alpha, dxi, f = irv1_data(d0, tau, mu, eps)
    p = np.zeros((2, n2, n1))
    one = np.ones((n2, n1))
    energies = []
    for _ in range(iters):
        r = ops.div(p) - f
        if trace:
            energies.append(ops.inner(r, r))
        p = rowwise_update(p, ops.grad(r), one, t)
    d = np.asarray(d0, np.float64) - (ops.div(p) + dxi) / alpha
    return (d, p, energies) if trace else (d, p)


def chambolle_irv2(d0, tau, lam, iters, t=0.125, trace=False):
    """Chambolle's iteration for the IRV2 dual: psi = grad(div p - f);
    p <- (p + t psi)/(1 + t |psi|); d = d_0 - div p / alpha."""
    n2, n1 = d0.shape
    alpha, g, f = irv2_data(d0, tau, lam)
    p = np.zeros((2, n2, n1))
    one = np.ones((n2, n1))
    energies = []
    for _ in range(iters):
        r = ops.div(p) - f
        if trace:
            energies.append(ops.inner(r, r))
        p = rowwise_update(p, ops.grad(r), one, t)
    d = np.asarray(d0, np.float64) - ops.div(p) / alpha
    return (d, p, energies) if trace else (d, p)


# ----------------------------------------------------------------------------- local projection


def local_projection(w, s_plus, n2t, n1t, cuts_y, cuts_x):
    """R_{S+} P E_{S+} w (Eq. locglobprojpart1) for w on S+ (shape (2, ..)).

    q = div_T E w on T = (S+)_+ (reading: T = S+ plus one row/column, clipped -- resDiv P:1417);
    phi = R_T Delta^dagger E_T q via the literal block-DCT sum (Eq. invLaplLowCapLong);
    result = w - R_{S+} grad_T phi (resGrad P:1421-1425)."""
    t_rect = rect_plus(s_plus, n2t, n1t)
    q = ops.div(extend(w, s_plus, t_rect))
    phi = spectral.lap_pinv_block(q, t_rect[0], t_rect[1], t_rect[0], t_rect[1],
                                  n2t, n1t, cuts_y, cuts_x)
    return np.asarray(w, np.float64) - restrict(ops.grad(phi), t_rect, s_plus)


# ----------------------------------------------------------------------------- Schwarz, step 2


def _irv2_inner_local(m, lay, p, f, qhat_m, inner, t):
    """Alg. 3 for Lambda = div on Omega, localized to Omega_m / Omega_{m,+}
    (resDiv/resGrad):
    omega0 = R_{S+}(f - div p + div(theta_m p)),  psi = R_S grad_{S+}(div_{S+} E v - omega0)."""
    n2, n1 = lay.n2, lay.n1
    s = lay.rect(m, extended=False)
    sp = rect_plus(s, n2, n1)
    th = lay.theta_rect(m, extended=False)
    p_s = restrict(p, full_rect(n2, n1), s)
    omega0 = (restrict(f - ops.div(p), full_rect(n2, n1), sp)
              + ops.div(extend(th * p_s, s, sp)))
    return irv2_local_iterations(lay, m, omega0, qhat_m, inner, t)


def irv2_local_iterations(lay, m, omega0, v0, inner, t):
    """The inner loop of the localized Alg. 3 given omega0 on S+ = R_{S+}(...):
    ``inner`` times psi = R_S grad_{S+}(div_{S+} E v - omega0); v <- (theta v + t theta psi) /
    (theta + t |psi|).  Only arrays on S / S+ are touched."""
    s = lay.rect(m, extended=False)
    sp = rect_plus(s, lay.n2, lay.n1)
    th = lay.theta_rect(m, extended=False)
    v = np.array(v0, np.float64)
    for _ in range(inner):
        u = ops.div(extend(v, s, sp)) - omega0
        psi = restrict(ops.grad(u), sp, s)
        v = rowwise_update(v, psi, th, t)
    return v


def irv2_inner_global(m, lay, p, f, v0_full, inner, t):
    """Alg. 3 literally on the full grid Omega:
    psi = Lambda^*(-Lambda(v + sum_{l != m} theta_l p) + f) with Lambda = div, Lambda^* = -grad."""
    th = lay.theta(m, extended=False)
    others = p - th * p                       # sum_{l != m} theta_l p, since sum theta = 1
    v = np.array(v0_full, np.float64)
    for _ in range(inner):
        psi = -ops.grad(-ops.div(v + others) + f)
        v = rowwise_update(v, psi, th, t)
    return v


def stop_rule(criterion, tol, d_prev, d_next, npts, cfac):
    """Outer stopping tests between consecutive dual energies:
    1 -- |D_n^{1/2} - D_{n+1}^{1/2}| < (cfac |Gamma|)^{1/2} tol (section 5.2: cfac = 2 for TFS,
    P:915-919; 1 for IRV1/IRV2); 2 -- |D_n^2 - D_{n+1}^2| / |Gamma| < tol (section 6.3,
    P:1776, printed with squares, reading A19).  0 never stops (fixed schedule, A10)."""
    if criterion == 1:
        return abs(np.sqrt(d_prev) - np.sqrt(d_next)) < np.sqrt(cfac * npts) * tol
    if criterion == 2:
        return abs(d_prev ** 2 - d_next ** 2) / npts < tol
    return False


def dd_step2(d0, tau, lam, lay: Layout, sweeps, inner, t=0.125, warm="qhat", trace=False,
             subdomains=None, variant="irv2", eps=1e-3, stop=(0, 0.0), workers=1):
    """Alg. 2 for step 2 on Gamma = Omega with the localized Alg. 3; IRV2 (default,
    the variant the paper adopts) or IRV1 (``variant='irv1'``, xi smoothing ``eps``).

    Warm start v^0 = R_S qhat_m from the previous sweep, qhat = 0 initially (reading A9;
    ``warm='theta_p'`` uses R_S theta_m p^n instead).  Fixed schedule, no stopping test (A10).
    ``workers`` > 1 runs the local solves of a sweep on threads (map_subdomains; same result).
    Returns (d, p, info) with d = d_0 - (div p + shift) / alpha (IRV1: Eq. tau_hat)."""
    n2, n1 = d0.shape
    alpha, f, shift = step2_data(d0, tau, lam, variant, eps)
    p = np.zeros((2, n2, n1))
    qhat = {}
    for m in lay.subdomains():
        qhat[m] = np.zeros((2,) + rect_shape(lay.rect(m, extended=False)))
    energies = []
    e_prev = ops.inner(f, f)                  # D(p^0) = ||div 0 - f||^2
    sweeps_run = sweeps
    for n in range(sweeps):
        acc = np.zeros_like(p)

        def local(m, p=p):
            s = lay.rect(m, extended=False)
            if warm == "qhat":
                v0 = qhat[m]
            else:
                v0 = restrict(lay.theta(m, False) * p, full_rect(n2, n1), s)
            return _irv2_inner_local(m, lay, p, f, v0, inner, t)

        subs = lay.subdomains()
        for m, q in zip(subs, map_subdomains(local, subs, workers)):
            qhat[m] = q
            acc += extend(q, lay.rect(m, extended=False), full_rect(n2, n1))
        p = (1.0 - lay.alpha_hat) * p + lay.alpha_hat * acc
        if trace or stop[0]:
            r = ops.div(p) - f
            energies.append(ops.inner(r, r))
            if stop_rule(stop[0], stop[1], e_prev, energies[-1], n2 * n1, 1.0):
                sweeps_run = n + 1
                break
            e_prev = energies[-1]
    d = np.asarray(d0, np.float64) - (ops.div(p) + shift) / alpha
    r = ops.div(p) - f
    info = {"alpha": alpha, "shift": shift, "f": f, "energies": energies, "qhat": qhat,
            "sweeps_run": sweeps_run, "dual_energy": ops.inner(r, r)}
    return d, p, info


# ----------------------------------------------------------------------------- Schwarz, step 1


def _tfs_inner_local(m, lay, p, r_global, qhat_m, inner, t):
    """Alg. 5, localized TFS inner loop on Omega~_m / Omega~_{m,+}:
    omega0_loc = R_{S+}(f - P multidiv sum_{l != m} theta_l p)
               = R_{S+} r + R_{S+} P E_{S+} multidiv_{S+} E_S (theta_m p)   (r = f - P multidiv p);
    then tfs_local_iterations."""
    n2t, n1t = lay.n2 + 1, lay.n1 + 1
    cy = spectral.cut_points(n2t, lay.m2)
    cx = spectral.cut_points(n1t, lay.m1)
    s = lay.rect(m, extended=True)
    sp = rect_plus(s, n2t, n1t)
    whole = full_rect(n2t, n1t)
    th = lay.theta_rect(m, extended=True)
    tp = th * restrict(p, whole, s)
    w_m = ops.multidiv(extend(tp, s, sp))
    omega0 = restrict(r_global, whole, sp) + local_projection(w_m, sp, n2t, n1t, cy, cx)
    return tfs_local_iterations(lay, m, omega0, qhat_m, inner, t)


def tfs_local_iterations(lay, m, omega0, v0, inner, t):
    """The inner loop of Alg. 5 given omega0 on S+: ``inner`` times
    psi = R_S E multigrad_{S+}(R_{S+} P E_{S+} multidiv_{S+} E_S v - omega0);
    v_k <- (theta v_k + t theta psi_k)/(theta + t |psi_k|).  Only arrays on S / S+ / T."""
    n2t, n1t = lay.n2 + 1, lay.n1 + 1
    cy = spectral.cut_points(n2t, lay.m2)
    cx = spectral.cut_points(n1t, lay.m1)
    s = lay.rect(m, extended=True)
    sp = rect_plus(s, n2t, n1t)
    th = lay.theta_rect(m, extended=True)
    v = np.array(v0, np.float64)
    for _ in range(inner):
        w = ops.multidiv(extend(v, s, sp))
        pw = local_projection(w, sp, n2t, n1t, cy, cx)
        psi = restrict(ops.multigrad(pw - omega0), sp, s)
        v = rowwise_update(v, psi, th, t)
    return v


def tfs_inner_global(m, lay, p, f, v0_full, inner, t):
    """Alg. 4 on the full grid Omega~:
    omega0 = f - P multidiv sum_{l != m} theta_l p;  psi = multigrad(P multidiv v - omega0)."""
    th = lay.theta(m, extended=True)
    others = p - th * p
    omega0 = f - spectral.project(ops.multidiv(others))
    v = np.array(v0_full, np.float64)
    for _ in range(inner):
        psi = ops.multigrad(spectral.project(ops.multidiv(v)) - omega0)
        v = rowwise_update(v, psi, th, t)
    return v


def dd_step1(d0, delta, lay: Layout, sweeps, inner, t=0.125, warm="qhat", trace=False,
             stop=(0, 0.0), workers=1):
    """Alg. 2 for TFS on Gamma = Omega~ with the localized Alg. 5.

    f = delta^{-1} P tau_0.  The global residual r^n = f - P multidiv p^n is
    evaluated once per outer sweep (reading A11 of P:1761-1766).  Output
    tau = P tau_0 - delta P multidiv p^S = delta r^S (Cor. tfsdual / Eq. tfs_dualPK).
    ``workers`` > 1 runs the local solves of a sweep on threads (map_subdomains; same result)."""
    n2, n1 = d0.shape
    n2t, n1t = n2 + 1, n1 + 1
    whole = full_rect(n2t, n1t)
    f = spectral.project(tau0(d0)) / delta
    p = np.zeros((2, 2, n2t, n1t))
    qhat = {m: np.zeros((2, 2) + rect_shape(lay.rect(m, True))) for m in lay.subdomains()}
    energies = []
    e_prev = None
    sweeps_run = sweeps
    for n in range(sweeps):
        r = f - spectral.project(ops.multidiv(p))
        if stop[0]:                          # D_TFS(p^n) = ||r^n||^2 (Eq. tfsdualdis)
            e = ops.inner(r, r)
            if e_prev is not None and stop_rule(stop[0], stop[1], e_prev, e, n2t * n1t, 2.0):
                sweeps_run = n
                break
            e_prev = e
        acc = np.zeros_like(p)

        def local(m, p=p, r=r):
            s = lay.rect(m, extended=True)
            if warm == "qhat":
                v0 = qhat[m]
            else:
                v0 = restrict(lay.theta(m, True) * p, whole, s)
            return _tfs_inner_local(m, lay, p, r, v0, inner, t)

        subs = lay.subdomains()
        for m, q in zip(subs, map_subdomains(local, subs, workers)):
            qhat[m] = q
            acc += extend(q, lay.rect(m, extended=True), whole)
        p = (1.0 - lay.alpha_hat) * p + lay.alpha_hat * acc
        if trace:
            rr = spectral.project(ops.multidiv(p)) - f
            energies.append(ops.inner(rr, rr))
    tau = delta * (f - spectral.project(ops.multidiv(p)))
    return tau, p, {"f": f, "energies": energies, "qhat": qhat, "sweeps_run": sweeps_run,
                    "dual_energy": ops.inner(tau, tau) / delta ** 2}


def dd_denoise(d0, delta, lam, lay: Layout, it1, it2, t=0.125, workers=1):
    """Step 1 then step 2 on the same splitting; it = (sweeps, inner)."""
    tau, p1, _ = dd_step1(d0, delta, lay, it1[0], it1[1], t, workers=workers)
    d, p2, info = dd_step2(d0, tau, lam, lay, it2[0], it2[1], t, workers=workers)
    return d, tau, p1, p2


# ----------------------------------------------------------------------------- energies


def tv(u):
    """Channel-wise discrete TV: sum_k sum_px |grad u_k| (reading A15)."""
    u = np.asarray(u, np.float64)
    if u.ndim == 2:
        gr = ops.grad(u)
        return float(np.sum(np.sqrt(gr[0] ** 2 + gr[1] ** 2)))
    return sum(tv(u[k]) for k in range(u.shape[0]))


def dual_energy_tfs(p, f):
    """D_TFS(p) = || P multidiv p - f ||^2 (Eq. tfsdualdis)."""
    r = spectral.project(ops.multidiv(p)) - f
    return ops.inner(r, r)


def dual_energy_irv2(p, f):
    """D_IRV2(p) = || div p - f ||^2 with f = alpha (d_0 - g), g zero-mean."""
    r = ops.div(p) - f
    return ops.inner(r, r)


def primal_energy_tfs(tau, ptau0, delta):
    """E_1 = TV(tau) + ||tau - P tau_0||^2 / (2 delta)."""
    dlt = np.asarray(tau, np.float64) - ptau0
    return tv(tau) + ops.inner(dlt, dlt) / (2.0 * delta)


def primal_energy_irv2(d, d0, g, alpha):
    """E_2 = TV(d - g) + alpha/2 ||d - d_0||^2 (Eq. modifiedStep2)."""
    dd = np.asarray(d, np.float64) - d0
    return tv(np.asarray(d, np.float64) - g) + 0.5 * alpha * ops.inner(dd, dd)


def primal_energy_irv1(d, d0, dxi, alpha):
    """E = TV(d) + <d, div xi> + alpha/2 ||d - d_0||^2 (Eq. IRPXi)."""
    d = np.asarray(d, np.float64)
    dd = d - d0
    return tv(d) + ops.inner(d, dxi) + 0.5 * alpha * ops.inner(dd, dd)


def dual_value_tfs(p, ptau0, delta):
    """Dual objective of Cor. tfsdual in the projected-data form: with
    D_TFS(p) = ||P multidiv p - delta^{-1} P tau_0||^2 (Eq. tfsdualdis),
    G_1(p) = ||P tau_0||^2 / (2 delta) - (delta / 2) D_TFS(p) <= min E_1 (weak duality); at the
    recovered tau = P tau_0 - delta P multidiv p, E_1(tau) - G_1(p) equals the C-15 gap."""
    f = np.asarray(ptau0, np.float64) / delta
    return ops.inner(ptau0, ptau0) / (2.0 * delta) - 0.5 * delta * dual_energy_tfs(p, f)


def dual_value_irv2(p, d0, g, alpha):
    """Dual objective of the ROF problem of Eq. modifiedStep2 (dual P:504-510): with
    D_IRV2(p) = ||div p - alpha (d_0 - g)||^2 (Eq. ir2dualdis),
    G_2(p) = alpha/2 ||d_0 - g||^2 - D_IRV2(p) / (2 alpha) <= min E_2 (weak duality)."""
    h = np.asarray(d0, np.float64) - g
    return 0.5 * alpha * ops.inner(h, h) - dual_energy_irv2(p, alpha * h) / (2.0 * alpha)


def dual_value_irv1(p, d0, f, alpha):
    """The dual function whose maximiser Cor. irdual characterises:
    G(p) = alpha/2 ||d_0||^2 - ||div p - f||^2 / (2 alpha) <= min E (weak duality)."""
    r = ops.div(p) - f
    return 0.5 * alpha * ops.inner(d0, d0) - ops.inner(r, r) / (2.0 * alpha)


def duality_gap(u, p):
    """sum_k sum_px (|grad u_k| + p_k . grad u_k) >= 0 for |p_k| <= 1 (SURVEY C-15):
    TV(u) = sup_{|p|<=1} <u, div p> = sup -<grad u, p>, so the gap vanishes iff p attains it."""
    u = np.asarray(u, np.float64)
    p = np.asarray(p, np.float64)
    if u.ndim == 2:
        gr = ops.grad(u)
        return float(np.sum(np.sqrt(gr[0] ** 2 + gr[1] ** 2) + p[0] * gr[0] + p[1] * gr[1]))
    return sum(duality_gap(u[k], p[k]) for k in range(u.shape[0]))
