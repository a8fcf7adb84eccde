"""The C-ABI library loads and exports every symbol include/tvstokes.h declares; host-only
entry points agree with the paper's layout rules (no compute calls: no GPU needed)."""
import os
import re

import numpy as np
import pytest

import paper_2602_17494_b200 as pkg
from paper_2602_17494_b200 import build as pbuild
from oracle import layout as olayout

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    pbuild.build()
    return pkg.load_library()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "tvstokes.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:tvs_status|const char \*)\s*(\w+)\s*\(", src, flags=re.M)))


def test_header_declares_expected(lib):
    assert set(declared_symbols()) == set(pkg.ABI_SYMBOLS)


def test_library_exports_every_declared_symbol(lib):
    for name in declared_symbols():
        assert hasattr(lib, name), name
    out = os.popen(f"nm -D --defined-only {pkg.LIB_PATH}").read()
    for name in declared_symbols():
        assert re.search(rf"\bT {name}\b", out), name


def test_library_is_sm100a(lib):
    out = os.popen(f"cuobjdump --list-elf {pkg.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out


@pytest.mark.parametrize("n,m,s", [(10, 2, 2), (65, 2, 4), (513, 4, 8), (2049, 8, 16),
                                   (8193, 8, 32), (31, 3, 3), (101, 4, 5)])
def test_layout_matches_oracle(lib, n, m, s):
    ref = olayout.ranges_1d(n, m, s)
    th = olayout.theta_1d(n, m, s)
    for k in range(m):
        assert pkg.layout_range(n, m, s, k) == ref[k]
        for x in sorted({0, n - 1, ref[k][0], ref[k][1], (ref[k][0] + ref[k][1]) // 2}):
            assert abs(pkg.layout_theta(n, m, s, k, x) - th[k, x]) < 1e-15


def test_layout_errors(lib):
    with pytest.raises(pkg.TvsError) as e:
        pkg.layout_range(20, 4, 5, 0)
    assert e.value.code == 2


def test_owned_rows_partition(lib):
    L = (8, 8, 16, 16)
    for world in (1, 2, 4, 8):
        rows = [pkg.owned_rows(2048, 2048, L, r, world) for r in range(world)]
        assert rows[0][0] == 0 and rows[-1][1] == 2049
        assert all(rows[i][1] == rows[i + 1][0] for i in range(world - 1))
