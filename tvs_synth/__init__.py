"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of the method's arithmetic (no difference operators, no DCT, no
projection, no dual update).  It only draws images and states the workload table, so that the
fp64 oracle (``oracle/``) and the CUDA path (``paper_2602_17494_b200``) can consume the very same
fp32 pixels without sharing any code that computes the method.

Recipes follow BASELINE.json ``configs`` and SURVEY.md section 8(d):

* RNG: counter-based splitmix64.  Every draw is ``mix(key(seed, stream) + (counter+1)*GOLDEN)``,
  so the noise of pixel k is independent of image size, tiling or process count.
* Noise: Box-Muller on the counter pair (2k, 2k+1) of stream ``"noise"``.
* Geometry (disk, ellipses, Voronoi sites and ramps): sequential counters of stream ``"geom"``.
* Every image is clipped to [0, 1] after the noise and stored as fp32.

The paper's own test images ("Image 10" P:1771) are not distributed; these
synthetic images stand in for them (sigma = 0.1 matches the paper's DD run sigma^2 = 0.01).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_STREAMS = {"noise": 1, "geom": 2, "aux": 3}


def _mix(z: np.ndarray) -> np.ndarray:
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def _key(seed: int, stream: str) -> np.uint64:
    with np.errstate(over="ignore"):
        return _mix(np.uint64(seed) * _GOLDEN + np.uint64(_STREAMS[stream]))


def uniform(seed: int, stream: str, counters: np.ndarray) -> np.ndarray:
    """U[0,1) doubles (53 bits) for the given uint64 counters of (seed, stream)."""
    k = _key(seed, stream)
    c = np.asarray(counters, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = _mix(k + (c + np.uint64(1)) * _GOLDEN)
    return (z >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def gaussian_field(seed: int, n2: int, n1: int, sigma: float, row0: int = 0) -> np.ndarray:
    """N(0, sigma^2) per pixel via Box-Muller on counters (2k, 2k+1), k = i*n1 + j."""
    out = np.empty((n2, n1), dtype=np.float64)
    # chunk rows to bound temporaries for large images
    step = max(1, (1 << 22) // max(n1, 1))
    for a in range(0, n2, step):
        b = min(n2, a + step)
        k = (np.arange(row0 + a, row0 + b, dtype=np.uint64)[:, None] * np.uint64(n1)
             + np.arange(n1, dtype=np.uint64)[None, :])
        u1 = uniform(seed, "noise", k * np.uint64(2))
        u2 = uniform(seed, "noise", k * np.uint64(2) + np.uint64(1))
        out[a:b] = sigma * np.sqrt(-2.0 * np.log1p(-u1)) * np.cos(2.0 * np.pi * u2)
    return out


class _Seq:
    """Sequential draws from the 'geom' stream."""

    def __init__(self, seed: int):
        self.seed, self.c = seed, 0

    def u(self, n: int = 1, lo: float = 0.0, hi: float = 1.0) -> np.ndarray:
        v = uniform(self.seed, "geom", np.arange(self.c, self.c + n, dtype=np.uint64))
        self.c += n
        return lo + (hi - lo) * v


def disk_on_ramp(n: int = 64, seed: int = 1001, sigma: float = 0.1) -> np.ndarray:
    """Config 1: disk r=20 (0.8) centred (31.5, 31.5) on a ramp 0.1..0.4 along x, + noise."""
    i = np.arange(n, dtype=np.float64)[:, None]
    j = np.arange(n, dtype=np.float64)[None, :]
    img = 0.1 + 0.3 * j / (n - 1) + 0.0 * i
    c = (n - 1) / 2.0
    img = np.where((i - c) ** 2 + (j - c) ** 2 <= 20.0 ** 2, 0.8, img)
    img = img + gaussian_field(seed, n, n, sigma)
    return np.clip(img, 0.0, 1.0).astype(np.float32)


def ellipses_on_sinusoid(n: int = 512, seed: int = 1002, sigma: float = 0.08,
                         count: int = 12) -> np.ndarray:
    """Config 2: 12 seeded ellipses (U[0,1] intensity) on 0.5 + 0.2 sin(2pi j/128) cos(2pi i/128)."""
    i = np.arange(n, dtype=np.float64)[:, None]
    j = np.arange(n, dtype=np.float64)[None, :]
    img = 0.5 + 0.2 * np.sin(2 * np.pi * j / 128.0) * np.cos(2 * np.pi * i / 128.0)
    g = _Seq(seed)
    for _ in range(count):
        cy, cx = g.u(2, 0.0, n)
        ay, ax = g.u(2, n / 32.0, n / 8.0)
        ang = g.u(1, 0.0, np.pi)[0]
        val = g.u(1)[0]
        ca, sa = np.cos(ang), np.sin(ang)
        dx, dy = j - cx, i - cy
        xr = ca * dx + sa * dy
        yr = -sa * dx + ca * dy
        img = np.where((xr / ax) ** 2 + (yr / ay) ** 2 <= 1.0, val, img)
    img = img + gaussian_field(seed, n, n, sigma)
    return np.clip(img, 0.0, 1.0).astype(np.float32)


def ellipses_rect(n2: int = 270, n1: int = 480, seed: int = 1010, sigma: float = 0.1,
                  count: int = 12) -> np.ndarray:
    """Stand-in for the paper's DD validation image (Image 10, 270 x 480, sigma^2 = 0.01, P:1771;
    not distributed): the config-2 recipe on a rectangle -- seeded ellipses (U[0,1] intensity,
    semi-axes U[min/32, min/8]) on 0.5 + 0.2 sin(2pi j/128) cos(2pi i/128), Gaussian noise
    sigma = 0.1, clipped to [0, 1]."""
    i = np.arange(n2, dtype=np.float64)[:, None]
    j = np.arange(n1, dtype=np.float64)[None, :]
    img = 0.5 + 0.2 * np.sin(2 * np.pi * j / 128.0) * np.cos(2 * np.pi * i / 128.0)
    g = _Seq(seed)
    m = min(n2, n1)
    for _ in range(count):
        cy, cx = g.u(1, 0.0, n2)[0], g.u(1, 0.0, n1)[0]
        ay, ax = g.u(2, m / 32.0, m / 8.0)
        ang = g.u(1, 0.0, np.pi)[0]
        val = g.u(1)[0]
        ca, sa = np.cos(ang), np.sin(ang)
        dx, dy = j - cx, i - cy
        xr = ca * dx + sa * dy
        yr = -sa * dx + ca * dy
        img = np.where((xr / ax) ** 2 + (yr / ay) ** 2 <= 1.0, val, img)
    img = img + gaussian_field(seed, n2, n1, sigma)
    return np.clip(img, 0.0, 1.0).astype(np.float32)


def _voronoi_geometry(n, cells, seed):
    g = int(round(np.sqrt(cells)))
    assert g * g == cells
    geo = _Seq(seed)
    # stratum (a, b) covers rows [a*n/g, (a+1)*n/g) and cols [b*n/g, (b+1)*n/g)
    edges = np.arange(g + 1, dtype=np.float64) * (n / g)
    u = geo.u(2 * cells).reshape(g, g, 2)
    sy = edges[:-1, None] + u[..., 0] * (n / g)
    sx = edges[None, :-1] + u[..., 1] * (n / g)
    prm = geo.u(3 * cells).reshape(g, g, 3)
    c0 = 0.2 + 0.6 * prm[..., 0]
    ga = -1e-3 + 2e-3 * prm[..., 1]
    gb = -1e-3 + 2e-3 * prm[..., 2]
    return g, sy, sx, c0, ga, gb


def _voronoi_rows(args):
    """Rows [r0, r1) of the Voronoi image (+ noise, clipped) -- exact for any row split."""
    n, cells, seed, sigma, r0_all, r1_all = args
    g, sy, sx, c0, ga, gb = _voronoi_geometry(n, cells, seed)
    out = np.empty((r1_all - r0_all, n), dtype=np.float32)
    cols = np.arange(n, dtype=np.float64)
    bcol = np.minimum((cols * g / n).astype(np.int64), g - 1)
    step = max(1, (1 << 21) // n)
    for r0 in range(r0_all, r1_all, step):
        r1 = min(r1_all, r0 + step)
        rows = np.arange(r0, r1, dtype=np.float64)
        arow = np.minimum((rows * g / n).astype(np.int64), g - 1)
        best = np.full((r1 - r0, n), np.inf)
        bidx = np.zeros((r1 - r0, n), dtype=np.int64)
        for da in range(-2, 3):
            for db in range(-2, 3):
                a = arow[:, None] + da
                b = bcol[None, :] + db
                ok = (a >= 0) & (a < g) & (b >= 0) & (b < g)
                ac = np.clip(a, 0, g - 1)
                bc = np.clip(b, 0, g - 1)
                d2 = (rows[:, None] - sy[ac, bc]) ** 2 + (cols[None, :] - sx[ac, bc]) ** 2
                idx = ac * g + bc
                d2 = np.where(ok, d2, np.inf)
                better = (d2 < best) | ((d2 == best) & (idx < bidx))
                best = np.where(better, d2, best)
                bidx = np.where(better, idx, bidx)
        ka, kb = bidx // g, bidx % g
        img = (c0[ka, kb] + ga[ka, kb] * (cols[None, :] - sx[ka, kb])
               + gb[ka, kb] * (rows[:, None] - sy[ka, kb]))
        img += gaussian_field(seed, r1 - r0, n, sigma, row0=r0)
        out[r0 - r0_all:r1 - r0_all] = np.clip(img, 0.0, 1.0)
    return out


def voronoi(n: int, cells: int, seed: int, sigma: float = 0.1, workers: int = 0) -> np.ndarray:
    """Configs 3-5: jittered-grid Voronoi, each cell an affine ramp, + noise.

    ``workers`` > 1 splits the rows over processes; the result is bit-identical for any split
    (every pixel depends only on its coordinates and the seed)."""
    import os
    if workers == 0:
        workers = min(16, os.cpu_count() or 1) if n >= 4096 else 1
    if workers <= 1:
        return _voronoi_rows((n, cells, seed, sigma, 0, n))
    from concurrent.futures import ProcessPoolExecutor
    bounds = [(n * k) // workers for k in range(workers + 1)]
    jobs = [(n, cells, seed, sigma, bounds[k], bounds[k + 1]) for k in range(workers)]
    with ProcessPoolExecutor(max_workers=workers) as ex:
        parts = list(ex.map(_voronoi_rows, jobs))
    return np.concatenate(parts, axis=0)


@dataclass(frozen=True)
class Config:
    """One BASELINE.json workload: image recipe, layout and schedule."""
    name: str
    n: int
    m2: int
    m1: int
    overlap: int
    sweeps: int
    inner: int
    seed: int
    delta: float = 0.05
    lam: float = 0.1          # TV weight; alpha = 1/lambda
    t: float = 0.125
    cells: int = 0
    extra: dict = field(default_factory=dict)

    def image(self) -> np.ndarray:
        if self.name == "c1":
            return disk_on_ramp(self.n, self.seed)
        if self.name == "c2":
            return ellipses_on_sinusoid(self.n, self.seed)
        return voronoi(self.n, self.cells, self.seed)


CONFIGS = {
    "c1": Config("c1", 64, 2, 2, 4, 20, 20, 1001),
    "c2": Config("c2", 512, 4, 4, 8, 50, 10, 1002),
    "c3": Config("c3", 2048, 8, 8, 16, 50, 10, 1003, cells=64),
    "c4": Config("c4", 8192, 8, 1, 32, 30, 20, 1004, cells=1024),
    "c5": Config("c5", 32768, 16, 16, 32, 20, 10, 1005, cells=16384),
    # config-5 weak-scaling sizes at 1 / 2 / 4 GPUs (16 x 16 subdomains at every size, reading A16)
    "c5w1": Config("c5w1", 11585, 16, 16, 32, 20, 10, 1006, cells=16384),
    "c5w2": Config("c5w2", 16384, 16, 16, 32, 20, 10, 1007, cells=16384),
    "c5w4": Config("c5w4", 23170, 16, 16, 32, 20, 10, 1008, cells=16384),
}


def random_image(n2: int, n1: int, seed: int) -> np.ndarray:
    """Small i.i.d. U[0,1] test image (fp32) for unit tests."""
    k = np.arange(n2 * n1, dtype=np.uint64)
    return uniform(seed, "aux", k).reshape(n2, n1).astype(np.float32)


def random_field(shape, seed: int, scale: float = 1.0) -> np.ndarray:
    """i.i.d. U[-scale, scale] fp64 array of any shape for operator tests."""
    n = int(np.prod(shape))
    k = np.arange(n, dtype=np.uint64)
    return (scale * (2.0 * uniform(seed, "aux", k) - 1.0)).reshape(shape)


def step_image(n2: int, n1: int, left: int) -> np.ndarray:
    """Vertical step: 0 on the first ``left`` columns, 1 elsewhere (ROF closed-form pin)."""
    img = np.zeros((n2, n1), dtype=np.float32)
    img[:, left:] = 1.0
    return img
