"""Pins of oracle/layout.py: layout (A6/A8), partition of unity (A7), alpha-hat."""
import json
import os

import numpy as np
import pytest

from oracle import layout

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "operators.json")))


def test_spec_layout_example():
    g = GOLD["layout_10_m2_s2"]
    assert [list(r) for r in layout.ranges_1d(g["n"], g["m"], g["s"])] == g["ranges"]


def test_pou_band_values():
    th = layout.theta_1d(10, 2, 2)
    g = GOLD["pou_band_s2"]
    assert np.allclose(th[0, 4:6], g["theta_left_band"], atol=1e-15)
    assert np.allclose(th[1, 4:6], g["theta_right_band"], atol=1e-15)


def test_alpha_hat_table():
    for m2, m1, a in GOLD["alpha_hat"]["cases"]:
        assert layout.alpha_hat(m2, m1) == a


@pytest.mark.parametrize("n,m,s", [(65, 2, 4), (513, 4, 8), (2049, 8, 16), (8193, 8, 32),
                                   (32769, 16, 32), (30, 3, 3), (25, 5, 1)])
def test_pou_properties(n, m, s):
    """(i) sum = 1, theta >= 0; (ii) supp in Gamma_m; (iii) |grad theta| <= 1/(s+1); bands = s wide."""
    rg = layout.ranges_1d(n, m, s)
    th = layout.theta_1d(n, m, s)
    assert np.abs(th.sum(0) - 1).max() < 1e-14 and th.min() >= 0
    for k, (lo, hi) in enumerate(rg):
        assert np.all(th[k, :lo] == 0) and np.all(th[k, hi + 1:] == 0)
        assert np.all(th[k, lo:hi + 1] > 0)
        assert np.abs(np.diff(th[k])).max() <= 1.0 / (s + 1) + 1e-15 or m == 1
    for k in range(m - 1):
        assert rg[k][1] - rg[k + 1][0] + 1 == s
    assert rg[0][0] == 0 and rg[-1][1] == n - 1


def test_layout_rejects_bad_overlap():
    with pytest.raises(layout.LayoutError):
        layout.ranges_1d(20, 4, 5)          # core width 5 <= s
    with pytest.raises(layout.LayoutError):
        layout.ranges_1d(20, 2, 0)


def test_survey_config_sizes():
    """Per-axis subdomain sizes of SURVEY.md section 8 (layout on Omega~)."""
    sizes = lambda n, m, s: sorted({hi - lo + 1 for lo, hi in layout.ranges_1d(n, m, s)})
    assert sizes(65, 2, 4) == [34, 35]
    assert sizes(513, 4, 8) == [132, 133, 136]
    assert sizes(2049, 8, 16) == [264, 265, 272]
    assert sizes(8193, 8, 32) == [1040, 1041, 1056]
