"""Overlapping layout, partition of unity and coloring weight (section 6.1).

Readings: A6 -- s is the width of the band shared by adjacent subdomains, layout is
defined on Omega~ and Omega_m = Omega~_m cap Omega; A7 -- separable linear
ramps across each band; A8 -- core cuts c_k = floor(k N / M).
Oracle: test infrastructure only (see oracle/__init__.py).
"""
import numpy as np


class LayoutError(ValueError):
    pass


def ranges_1d(n, m, s):
    """Inclusive index ranges of the M subdomains of an axis of length n (0-based).

    Subdomain k = [c_k - floor(s/2), c_{k+1} - 1 + ceil(s/2)] clipped to [0, n-1] (A8), so
    adjacent subdomains share a band of exactly s points (A6; SPEC S:502 example)."""
    if m < 1 or n < 2:
        raise LayoutError("need m >= 1 and n >= 2")
    cuts = [k * n // m for k in range(m + 1)]
    if m > 1:
        if s < 1:
            raise LayoutError("overlap must be >= 1 for M > 1")
        if min(cuts[k + 1] - cuts[k] for k in range(m)) <= s:
            raise LayoutError("core width must exceed the overlap (A17)")
    out = []
    for k in range(m):
        lo = cuts[k] - (s // 2 if k > 0 else 0)
        hi = cuts[k + 1] - 1 + ((s + 1) // 2 if k < m - 1 else 0)
        out.append((max(0, lo), min(n - 1, hi)))
    return out


def theta_1d(n, m, s):
    """1D partition of unity, shape (m, n) (reading A7 of properties (i)-(iii)).

    Across the band [L, R] between subdomains k and k+1 (R - L + 1 = s):
    theta_k(x) = (R - x + 1)/(s + 1), theta_{k+1}(x) = (x - L + 1)/(s + 1); 1 elsewhere inside
    the subdomain, 0 outside it."""
    rg = ranges_1d(n, m, s)
    th = np.zeros((m, n), dtype=np.float64)
    for k, (lo, hi) in enumerate(rg):
        th[k, lo:hi + 1] = 1.0
    for k in range(m - 1):
        left, right = rg[k + 1][0], rg[k][1]      # band [L, R]
        for x in range(left, right + 1):
            th[k, x] = (right - x + 1) / (s + 1.0)
            th[k + 1, x] = (x - left + 1) / (s + 1.0)
    return th


def alpha_hat(m2, m1):
    """Coloring relaxation: 1 if M1 = M2 = 1; 1/2 if one of them is 1; 1/4 otherwise."""
    if m1 == 1 and m2 == 1:
        return 1.0
    if m1 == 1 or m2 == 1:
        return 0.5
    return 0.25


class Layout:
    """M2 x M1 overlapping subdomains of Omega~ ((N2+1) x (N1+1)) and of Omega (N2 x N1)."""

    def __init__(self, n2, n1, m2, m1, s_y, s_x):
        self.n2, self.n1, self.m2, self.m1 = n2, n1, m2, m1
        self.s_y, self.s_x = s_y, s_x
        # layout lives on Omega~ (A6); Omega ranges are the same ranges clipped
        self.ry = ranges_1d(n2 + 1, m2, s_y)
        self.rx = ranges_1d(n1 + 1, m1, s_x)
        self.ty = theta_1d(n2 + 1, m2, s_y)
        self.tx = theta_1d(n1 + 1, m1, s_x)
        self.alpha_hat = alpha_hat(m2, m1)

    def subdomains(self):
        return [(a, b) for a in range(self.m2) for b in range(self.m1)]

    def rect(self, m, extended):
        """Inclusive (rows, cols) of Gamma_m: on Omega~ if ``extended`` else Omega~_m cap Omega."""
        a, b = m
        (y0, y1), (x0, x1) = self.ry[a], self.rx[b]
        if not extended:
            y1, x1 = min(y1, self.n2 - 1), min(x1, self.n1 - 1)
        return (y0, y1), (x0, x1)

    def theta(self, m, extended):
        """theta_m on the whole grid (Omega~ or Omega): separable product theta_y * theta_x."""
        a, b = m
        th = self.ty[a][:, None] * self.tx[b][None, :]
        if not extended:
            th = th[:self.n2, :self.n1]
        return th

    def theta_rect(self, m, extended):
        """theta_m restricted to its own rectangle Gamma_m (the same products as ``theta``)."""
        a, b = m
        (y0, y1), (x0, x1) = self.rect(m, extended)
        return self.ty[a][y0:y1 + 1, None] * self.tx[b][None, x0:x1 + 1]
