"""Pins of oracle/spectral.py: DCT, Delta^dagger (Penrose identities), P_K properties."""
import json
import os

import numpy as np
import pytest
import scipy.fft

from oracle import ops, spectral
from tvs_synth import random_field

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "operators.json")))


def _dense(fn, shape_in):
    n = int(np.prod(shape_in))
    cols = []
    for k in range(n):
        e = np.zeros(n)
        e[k] = 1.0
        cols.append(np.asarray(fn(e.reshape(shape_in))).ravel())
    return np.array(cols).T


def test_dct2_example_and_library():
    assert np.allclose(spectral.dct_matrix(2), GOLD["dct_2"]["out"], atol=1e-16)
    for n in (3, 7, 16, 65):
        c = spectral.dct_matrix(n)
        # orthonormal DCT-II is scipy's type-2 'ortho' transform (library special case)
        ref = scipy.fft.dct(np.eye(n), type=2, norm="ortho", axis=0)
        assert np.abs(c - ref).max() < 1e-13
        assert np.abs(c @ c.T - np.eye(n)).max() < 1e-13


def test_dct_diagonalises_neumann_laplacian():
    """C_N L C_N^T = diag(-sigma_k^2) -- the reason form:DiscInvLapl holds."""
    for n in (4, 9):
        lap = -2 * np.eye(n) + np.eye(n, k=1) + np.eye(n, k=-1)
        lap[0, 0] = lap[-1, -1] = -1
        c = spectral.dct_matrix(n)
        assert np.abs(c @ lap @ c.T - np.diag(-spectral.sigma(n) ** 2)).max() < 1e-13


@pytest.mark.parametrize("shape", [(3, 3), (4, 6), (5, 7), (6, 4)])
def test_lap_pinv_penrose(shape):
    """The four Penrose identities determine Delta^dagger uniquely (reading A2 pairing)."""
    A = _dense(ops.laplacian, shape)
    X = _dense(spectral.lap_pinv, shape)
    assert np.abs(A @ X @ A - A).max() < 1e-12
    assert np.abs(X @ A @ X - X).max() < 1e-12
    assert np.abs((A @ X) - (A @ X).T).max() < 1e-12
    assert np.abs((X @ A) - (X @ A).T).max() < 1e-12
    assert np.abs(X - np.linalg.pinv(A)).max() < 1e-11
    assert np.abs(spectral.lap_pinv(np.ones(shape))).max() < 1e-13   # constant -> 0


@pytest.mark.parametrize("shape", [(4, 6), (5, 7)])
def test_printed_sigma_pairing_is_wrong_on_nonsquare(shape):
    """Reading A2: the printed index pairing of form:DiscInvLaplTild fails on non-square grids."""
    A = _dense(ops.laplacian, shape)
    Xp = _dense(lambda q: spectral.lap_pinv(q, printed_pairing=True), shape)
    assert np.abs(Xp - np.linalg.pinv(A)).max() > 0.1


def _feasible_shape():
    return (9, 12)


def test_projection_properties():
    """Prop. DisProj: idempotent, self-adjoint; div P w = 0; P grad = 0; ||Pw||<=||w||."""
    sh = _feasible_shape()
    w = random_field((2,) + sh, 5)
    u = random_field((2,) + sh, 6)
    pw = spectral.project(w)
    assert np.abs(ops.div(pw)).max() < 1e-10
    assert np.abs(spectral.project(pw) - pw).max() < 1e-12
    assert abs(ops.inner(pw, u) - ops.inner(w, spectral.project(u))) < 1e-11
    phi = random_field(sh, 7)
    assert np.abs(spectral.project(ops.grad(phi))).max() < 1e-11
    assert ops.inner(pw, pw) <= ops.inner(w, w) + 1e-12
    # curl fields (D-_y psi, -D-_x psi) are divergence free (mixed differences commute) -> fixed
    psi = random_field(sh, 8)
    curl = np.stack([ops.dminus_y(psi), -ops.dminus_x(psi)])
    assert np.abs(ops.div(curl)).max() < 1e-12
    assert np.abs(spectral.project(curl) - curl).max() < 1e-11


def test_projection_dimension():
    """dim K^h = dim Null(div) = 2 n - rank(div) = 2n - (n - 1) = n + 1 (Null(grad) = constants)."""
    sh = (5, 6)
    n = sh[0] * sh[1]
    Pm = _dense(spectral.project, (2,) + sh)
    assert round(np.trace(Pm)) == n + 1
    assert np.abs(Pm @ Pm - Pm).max() < 1e-11
    assert np.abs(Pm - Pm.T).max() < 1e-11


@pytest.mark.parametrize("m2,m1", [(1, 1), (2, 2), (3, 2)])
def test_block_dct_equals_restricted_global(m2, m1):
    """Eq. invLaplLowCapLong equals R_B Delta^dagger E_A computed globally."""
    n2, n1 = 17, 20
    cy, cx = spectral.cut_points(n2, m2), spectral.cut_points(n1, m1)
    a = ((3, 9), (5, 14))
    b = ((0, 6), (11, 19))
    qa = random_field((7, 10), 9)
    blk = spectral.lap_pinv_block(qa, a[0], a[1], b[0], b[1], n2, n1, cy, cx)
    full = np.zeros((n2, n1))
    full[3:10, 5:15] = qa
    ref = spectral.lap_pinv(full)[0:7, 11:20]
    assert np.abs(blk - ref).max() < 1e-13


def test_row_restricted_pinv_and_projection():
    """lap_pinv_rows / project_rows (output rows of the same formulas, for config-5 sizes) equal the
    corresponding rows of lap_pinv / project on square and non-square grids."""
    from tvs_synth import random_field
    for shape in ((9, 9), (8, 13), (17, 6)):
        q = random_field(shape, 3 + shape[0], 1.0)
        rows = [0, 2, shape[0] - 1]
        assert np.abs(spectral.lap_pinv_rows(q, rows) - spectral.lap_pinv(q)[rows]).max() < 1e-12
        w = random_field((2,) + shape, 9 + shape[1], 1.0)
        r, pw = spectral.project_rows(w, [shape[0] - 1, 1, 3])
        assert list(r) == [1, 3, shape[0] - 1]
        assert np.abs(pw - spectral.project(w)[:, r]).max() < 1e-12
