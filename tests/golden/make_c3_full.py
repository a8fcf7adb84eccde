#!/usr/bin/env python3
"""Writes tests/golden/c3_full_schedule.npz: the fp64 oracle on BASELINE config 3 with the FULL
bench schedule (2048 x 2048 Voronoi-64, 8 x 8 subdomains, overlap 16, 50 sweeps x 10 inner per
step, delta 0.05, lambda 0.1, t 1/8), end to end (step 1, then step 2 fed the oracle's tau).

Calls only ``oracle/`` (and ``tvs_synth`` for the seeded image); nothing here touches the CUDA
path.  Stored: tau (2 planes on Omega~), d (Omega) as fp32 (rounding 3e-8, far below the 1e-4
tolerance) and the duals p1 (4 planes), p2 (2 planes) as fp16 (diagnostic, tolerance 1e-2) at
(i) 16 x 16 windows centred on every crossing of the layout's core cuts (these cover every
overlap band crossing, where the Schwarz combine and the partition of unity act) and on every
subdomain centre, and (ii) 20000 seeded scattered points; plus the scalars E1, E2 (primal
energies), D1, D2 (dual energies) and the duality gaps of both steps.

Runtime: about 15-30 min on 8 host cores (one thread per subdomain; the literal block-DCT local
projection dominates).
Usage: python tests/golden/make_c3_full.py [out.npz]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import layout as olayout, ops, solvers as S, spectral  # noqa: E402
from tvs_synth import CONFIGS  # noqa: E402


def sample_points(n, cuts, seed, nrand=20000, w=16):
    """(rows, cols) index arrays on an n x n grid: windows at cut crossings / core centres plus
    seeded scattered points (deduplicated, sorted)."""
    centres = sorted(set(cuts[1:-1]) | {(cuts[k] + cuts[k + 1]) // 2 for k in range(len(cuts) - 1)}
                     | {0, n - 1})
    pts = set()
    for cy in centres:
        for cx in centres:
            y0 = min(max(cy - w // 2, 0), n - w)
            x0 = min(max(cx - w // 2, 0), n - w)
            for i in range(y0, y0 + w):
                for j in range(x0, x0 + w):
                    pts.add(i * n + j)
    rng = np.random.default_rng(seed)
    pts.update(int(k) for k in rng.integers(0, n * n, size=nrand))
    k = np.array(sorted(pts), dtype=np.int64)
    return (k // n).astype(np.int32), (k % n).astype(np.int32)


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(os.path.dirname(__file__), "c3_full_schedule.npz")
    c = CONFIGS["c3"]
    img = c.image()
    d0 = img.astype(np.float64)
    n = c.n
    lay = olayout.Layout(n, n, c.m2, c.m1, c.overlap, c.overlap)
    t0 = time.time()
    workers = os.cpu_count() or 1   # one task per subdomain on threads (bitwise the same result)
    tau, p1, info1 = S.dd_step1(d0, c.delta, lay, c.sweeps, c.inner, c.t, workers=workers)
    t1 = time.time()
    print(f"step 1: {t1 - t0:.0f} s", flush=True)
    d, p2, info2 = S.dd_step2(d0, tau, c.lam, lay, c.sweeps, c.inner, c.t, workers=workers)
    t2 = time.time()
    print(f"step 2: {t2 - t1:.0f} s", flush=True)
    ptau0 = spectral.project(S.tau0(d0))
    alpha, g, _ = S.irv2_data(d0, tau, c.lam)
    e1 = S.primal_energy_tfs(tau, ptau0, c.delta)
    e2 = S.primal_energy_irv2(d, d0, g, alpha)
    gap1 = S.duality_gap(tau, p1)
    gap2 = S.duality_gap(d - g, p2)
    cuts = spectral.cut_points(n + 1, c.m2)
    ty, tx = sample_points(n + 1, cuts, 31)
    dy, dx = sample_points(n, [min(k, n) for k in cuts], 32)
    np.savez_compressed(
        out,
        tau_rows=ty, tau_cols=tx, tau=tau[:, ty, tx].astype(np.float32),
        p1=p1[:, :, ty, tx].astype(np.float16),
        d_rows=dy, d_cols=dx, d=d[dy, dx].astype(np.float32), p2=p2[:, dy, dx].astype(np.float16),
        E1=e1, E2=e2, D1=info1["dual_energy"], D2=info2["dual_energy"], gap1=gap1, gap2=gap2,
        max_abs_div_tau=float(np.abs(ops.div(tau)).max()),
        schedule=np.array([c.sweeps, c.inner]), seconds=np.array([t1 - t0, t2 - t1]))
    print(f"wrote {out}: E1 {e1:.10e} E2 {e2:.10e} D1 {info1['dual_energy']:.6e} "
          f"D2 {info2['dual_energy']:.6e} gap1 {gap1:.4e} gap2 {gap2:.4e}", flush=True)


if __name__ == "__main__":
    main()
