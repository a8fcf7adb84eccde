#!/usr/bin/env python3
"""Writes tests/golden/c5_step1_sampled.npz: fp64 oracle values for BASELINE config 5 at full size
(32768 x 32768 Voronoi-16384, 16 x 16 subdomains, overlap 32, delta 0.05, t 1/8), step 1:

* P tau_0 (the global projection of Eq. formula:PKh) on sampled rows -- every core cut
  row of the layout, its neighbours, the first / last rows, and 24 seeded rows -- at the first,
  middle and last 512 columns and every 32nd;
* the first outer sweep's local solves qhat_m (Alg. 5) of three subdomains -- corner
  (0, 0), interior (7, 9) and the far corner (15, 15), which touches the extra row and column of
  Omega~ -- after 2 inner updates.  With p^0 = 0 and qhat = 0 (reading A9), omega0_m = R_{S+} f,
  f = delta^{-1} P tau_0 (the local projection of theta_m p^0 = 0 vanishes), and
  the second update applies the literal block-DCT local projection (Eq. invLaplLowCapLong) to a
  nonzero field.  Stored at 32 x 32 windows (corners, band crossings, centre) + 4000 seeded points.

Calls only ``oracle/`` (and ``tvs_synth`` for the image).  Runtime about 30-60 min and ~40 GB of
host memory on 8 cores (two 32769^3 DCT products and nine literal local projections).
Usage: python tests/golden/make_c5_sampled.py [out.npz]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import layout as olayout, ops, solvers as S, spectral  # noqa: E402
from tvs_synth import CONFIGS  # noqa: E402

SUBS = [(0, 0), (7, 9), (15, 15)]
INNER = 2


def windows(shape, seed, w=32, nrand=4000):
    """Local (row, col) indices: 32 x 32 windows at the four corners, the centre and the band
    crossings of the tile, plus seeded scattered points."""
    a, b = shape
    pts = set()
    for cy in (0, a // 2, a - w, 16, a - 48):
        for cx in (0, b // 2, b - w, 16, b - 48):
            for i in range(max(0, cy), min(a, cy + w)):
                for j in range(max(0, cx), min(b, cx + w)):
                    pts.add(i * b + j)
    rng = np.random.default_rng(seed)
    pts.update(int(k) for k in rng.integers(0, a * b, size=nrand))
    k = np.array(sorted(pts), dtype=np.int64)
    return (k // b).astype(np.int32), (k % b).astype(np.int32)


def ptau0_columns(n):
    """Columns stored for P tau_0: the first, middle and last 512 and every 32nd."""
    cols = set(range(512)) | set(range(n // 2 - 256, n // 2 + 256)) | set(range(n - 512, n)) \
        | set(range(0, n, 32))
    return np.array(sorted(cols), dtype=np.int32)


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(os.path.dirname(__file__), "c5_step1_sampled.npz")
    c = CONFIGS["c5"]
    n = c.n
    n2t = n + 1
    lay = olayout.Layout(n, n, c.m2, c.m1, c.overlap, c.overlap)
    t0 = time.time()
    d0 = c.image().astype(np.float64)
    print(f"image {time.time() - t0:.0f} s", flush=True)
    cuts = spectral.cut_points(n2t, c.m2)
    rng = np.random.default_rng(55)
    sample_rows = sorted(set([0, 1, n2t - 2, n2t - 1] + [r + d for r in cuts[1:-1] for d in (-1, 0, 1)]
                             + [int(r) for r in rng.integers(0, n2t, size=24)]))
    need = set(sample_rows)
    rects = {}
    for (iy, ix) in SUBS:
        m = (iy, ix)
        s = lay.rect(m, True)
        sp = S.rect_plus(s, n2t, n2t)
        rects[m] = (s, sp)
        need.update(range(sp[0][0], sp[0][1] + 1))
    t0 = time.time()
    tau0 = S.tau0(d0)
    del d0
    need = np.asarray(sorted(need), dtype=np.int64)
    q, w_rows = ops.div(tau0), tau0[:, need]
    del tau0
    rows, ptau0 = spectral.project_rows_div(q, w_rows, need)
    del q
    print(f"P tau_0 on {len(rows)} rows: {time.time() - t0:.0f} s", flush=True)
    at = {int(r): k for k, r in enumerate(rows)}
    f_rows = ptau0 / c.delta
    pcols = ptau0_columns(n2t)
    res = {"ptau0_rows": np.array(sample_rows, np.int32), "ptau0_cols": pcols,
           "ptau0": ptau0[:, [at[r] for r in sample_rows]][:, :, pcols].astype(np.float32)}
    for (iy, ix) in SUBS:
        m = (iy, ix)
        s, sp = rects[m]
        omega0 = np.stack([f_rows[:, at[r], sp[1][0]:sp[1][1] + 1] for r in range(sp[0][0], sp[0][1] + 1)],
                          axis=1)
        t1 = time.time()
        v0 = np.zeros((2, 2) + S.rect_shape(s))
        q = S.tfs_local_iterations(lay, m, omega0, v0, INNER, c.t)
        print(f"subdomain {m}: {time.time() - t1:.0f} s", flush=True)
        wr, wc = windows(S.rect_shape(s), 100 + 16 * iy + ix)
        key = f"{iy}_{ix}"
        res[f"q_{key}_rows"] = wr + s[0][0]
        res[f"q_{key}_cols"] = wc + s[1][0]
        res[f"q_{key}"] = q[:, :, wr, wc].astype(np.float32)
    res["inner"] = np.array(INNER)
    np.savez_compressed(out, **res)
    print(f"wrote {out}", flush=True)


if __name__ == "__main__":
    main()
