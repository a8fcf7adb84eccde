#!/usr/bin/env python3
"""Writes tests/golden/c4_short_schedule.npz: the fp64 oracle end to end on BASELINE config 4 at
full size (8192 x 8192 Voronoi-1024, 8 horizontal strips, overlap 32, delta 0.05, lambda 0.1,
t 1/8) with a SHORTENED schedule: step 1 two outer sweeps x two Alg. 5 updates, then step 2 (fed
the oracle's tau) two sweeps x four Alg. 3 updates.  The second sweep of each step starts from a
nonzero p^1, so omega0_m = R_{S+}(r^1 + P_loc multidiv theta_m p^1) and the combine of
overlapping strips are exercised at full size -- the full 30 x 20 schedule is out of the oracle's
reach (~3e15 MAC for step 1).

Calls only ``oracle/`` (and ``tvs_synth``).  Stored: tau (2 planes on Omega~) and d (Omega) as fp32
(rounding 3e-8 against the 1e-4 tolerance) on a grid of rows (first / middle / last row of every
32-row strip overlap, the first and last rows, 6 seeded rows) x columns (first, middle and last
256, every 16th), and the scalars E1, E2, D1, D2, gap1, gap2.
Runtime about 20-40 min on 8 cores (the literal block-DCT local projections dominate).
Usage: python tests/golden/make_c4_short.py [out.npz]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import layout as olayout, solvers as S, spectral  # noqa: E402
from tvs_synth import CONFIGS  # noqa: E402

IT1 = (2, 2)
IT2 = (2, 4)


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(os.path.dirname(__file__), "c4_short_schedule.npz")
    c = CONFIGS["c4"]
    n = c.n
    d0 = c.image().astype(np.float64)
    lay = olayout.Layout(n, n, c.m2, c.m1, c.overlap, c.overlap)
    workers = os.cpu_count() or 1
    t0 = time.time()
    tau, p1, info1 = S.dd_step1(d0, c.delta, lay, IT1[0], IT1[1], c.t, workers=workers)
    t1 = time.time()
    print(f"step 1: {t1 - t0:.0f} s", flush=True)
    d, p2, info2 = S.dd_step2(d0, tau, c.lam, lay, IT2[0], IT2[1], c.t, workers=workers)
    print(f"step 2: {time.time() - t1:.0f} s", flush=True)
    ptau0 = info1["f"] * c.delta
    alpha, g, _ = S.irv2_data(d0, tau, c.lam)
    e1 = S.primal_energy_tfs(tau, ptau0, c.delta)
    e2 = S.primal_energy_irv2(d, d0, g, alpha)
    gap1 = S.duality_gap(tau, p1)
    gap2 = S.duality_gap(d - g, p2)
    # rows: every overlap band's first, middle and last row, the first / last rows, 6 seeded rows;
    # columns: the first, middle and last 256 plus every 16th
    rows = {0, 1, n - 1, n}
    for k in range(len(lay.ry) - 1):
        a, b = lay.ry[k + 1][0], lay.ry[k][1]
        rows.update((a, (a + b) // 2, b))
    rng = np.random.default_rng(44)
    rows.update(int(r) for r in rng.integers(0, n, size=6))
    tr = np.array(sorted(rows), dtype=np.int32)
    cols = set(range(0, 256)) | set(range(n // 2 - 128, n // 2 + 128)) | set(range(n - 255, n + 1)) \
        | set(range(0, n + 1, 16))
    tc = np.array(sorted(cols), dtype=np.int32)
    dr, dc = tr[tr < n], tc[tc < n]
    np.savez_compressed(out, tau_rows=tr, tau_cols=tc, tau=tau[:, tr][:, :, tc].astype(np.float32),
                        d_rows=dr, d_cols=dc, d=d[dr][:, dc].astype(np.float32), E1=e1, E2=e2,
                        D1=info1["dual_energy"], D2=info2["dual_energy"], gap1=gap1, gap2=gap2,
                        it1=np.array(IT1), it2=np.array(IT2))
    print(f"wrote {out}: E1 {e1:.10e} E2 {e2:.10e} gap1 {gap1:.4e} gap2 {gap2:.4e}", flush=True)


if __name__ == "__main__":
    main()
