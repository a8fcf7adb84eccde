"""Moore-Penrose Delta^dagger via the orthonormal DCT-II and the projection P_K.

Oracle: test infrastructure only (see oracle/__init__.py).  fp64 throughout.
"""
import numpy as np

from . import ops

_DCT_CACHE = {}


def dct_matrix(n):
    """C_N of Eq. form:DCTmat: row k = sqrt(2/N) * w_k * cos(k (2j+1) pi / (2N)),
    w_0 = 1/sqrt(2), else 1 (0-based k, j).  Orthogonal."""
    c = _DCT_CACHE.get(n)
    if c is None:
        k = np.arange(n, dtype=np.float64)[:, None]
        j = np.arange(n, dtype=np.float64)[None, :]
        c = np.sqrt(2.0 / n) * np.cos(k * (2.0 * j + 1.0) * np.pi / (2.0 * n))
        c[0, :] *= 1.0 / np.sqrt(2.0)
        if n <= 8192:
            _DCT_CACHE[n] = c
    return c


def sigma(n):
    """sigma_{N,k} = (2/h) sin(k pi / (2N)), 0-based k (h = 1)."""
    return 2.0 * np.sin(np.arange(n, dtype=np.float64) * np.pi / (2.0 * n))


_LAM_CACHE = {}


def spectral_inverse(n2, n1, printed_pairing=False):
    """The diagonal (Delta~)^dagger of Eq. form:DiscInvLaplTild.

    Reading A2: row index i (y-frequency) pairs with sigma_{N~2, i} and column j with
    sigma_{N~1, j} (dimension-consistent with C_{N2} d C_{N1}^T).  The printed formula pairs
    i with N~1 and j with N~2; ``printed_pairing=True`` reproduces it literally (only used by the
    test that shows it fails the Penrose identities on non-square grids).
    """
    if not printed_pairing and (n2, n1) in _LAM_CACHE:   # cached: pure function of (n2, n1)
        return _LAM_CACHE[(n2, n1)]
    if printed_pairing:
        # literal: entry (i, j) -> -1/(sigma_{N1,i}^2 + sigma_{N2,j}^2); only defined if the
        # index ranges fit, i.e. used on grids where it can be evaluated
        si = 2.0 * np.sin(np.arange(n2)[:, None] * np.pi / (2.0 * n1))
        sj = 2.0 * np.sin(np.arange(n1)[None, :] * np.pi / (2.0 * n2))
    else:
        si = sigma(n2)[:, None]
        sj = sigma(n1)[None, :]
    den = si ** 2 + sj ** 2
    lam = np.zeros((n2, n1), dtype=np.float64)
    nz = den != 0.0
    nz[0, 0] = False
    lam[nz] = -1.0 / den[nz]
    if not printed_pairing and n2 * n1 <= 8192 * 8192:
        lam.setflags(write=False)
        _LAM_CACHE[(n2, n1)] = lam
    return lam


def lap_pinv(q, printed_pairing=False):
    """(Delta)^dagger q = C^{-1} (Delta~)^dagger C q (Eqs. form:DiscInvLapl P:611-612,
    eq:DCT2D P:627-629, eq:DCT2Dinv P:649-651), with C q = C_{N2} q C_{N1}^T."""
    n2, n1 = q.shape
    c2, c1 = dct_matrix(n2), dct_matrix(n1)
    x = c2 @ np.asarray(q, np.float64) @ c1.T
    y = spectral_inverse(n2, n1, printed_pairing) * x
    return c2.T @ y @ c1


def project(w):
    """P_{K^h} w = w - grad (Delta)^dagger div w (Eq. formula:PKh)."""
    return np.asarray(w, np.float64) - ops.grad(lap_pinv(ops.div(w)))


def project_multi(w):
    """P applied to a 2-vector field (shape (2, n2, n1)); identical to ``project``."""
    return project(w)


def lap_pinv_rows(q, rows):
    """Rows ``rows`` of (Delta)^dagger q (the restriction R_B of Eq. form:DiscInvLapl, P:611-625,
    to the rows B of the output): C_{N2}[:, B]^T ((Delta~)^dagger * (C_{N2} q C_{N1}^T)) C_{N1}.
    Same formula as lap_pinv with only the needed output rows formed -- for grids too large to
    hold the full result next to the DCT matrices (config 5: N~ = 32769)."""
    n2, n1 = q.shape
    rows = np.asarray(rows, dtype=np.int64)
    c2 = dct_matrix(n2)
    c1 = c2 if n1 == n2 else dct_matrix(n1)
    x = c2 @ (np.asarray(q, np.float64) @ c1.T)
    for a in range(0, n2, 1024):   # x *= (Delta~)^dagger, a row block of the diagonal at a time
        b = min(n2, a + 1024)
        si = sigma(n2)[a:b, None] ** 2
        den = si + sigma(n1)[None, :] ** 2
        lam = np.zeros_like(den)
        nz = den != 0.0
        lam[nz] = -1.0 / den[nz]
        x[a:b] *= lam
    return (c2[:, rows].T @ x) @ c1


def project_rows(w, rows):
    """Rows ``rows`` of P_{K^h} w = w - grad (Delta)^dagger div w (Eq. formula:PKh);
    grad = (D+_x, D+_y) needs phi on rows r and r + 1 (zero D+_y on the last row).
    Returns (sorted rows, (2, len(rows), n1))."""
    w = np.asarray(w, np.float64)
    rows = np.asarray(sorted(set(int(r) for r in rows)), dtype=np.int64)
    return project_rows_div(ops.div(w), w[:, rows], rows)


def project_rows_div(q, w_rows, rows):
    """project_rows given q = div w and the rows of w (sorted ``rows``): lets a caller free w
    before the DCT products (config 5: 32769^2 planes)."""
    n2, n1 = q.shape
    rows = np.asarray(rows, dtype=np.int64)
    need = np.asarray(sorted(set(rows.tolist()) | set(min(int(r) + 1, n2 - 1) for r in rows)), dtype=np.int64)
    phi = lap_pinv_rows(q, need)
    at = {int(r): k for k, r in enumerate(need)}
    out = np.empty((2, len(rows), n1))
    for k, r in enumerate(rows):
        pr = phi[at[int(r)]]
        out[0, k] = w_rows[0, k] - np.concatenate([pr[1:] - pr[:-1], [0.0]])
        out[1, k] = w_rows[1, k] - ((phi[at[int(r) + 1]] - pr) if r < n2 - 1 else 0.0)
    return rows, out


def cut_points(n, m):
    """Near-uniform core cuts c_k = floor(k n / M), k = 0..M (reading A8)."""
    return [k * n // m for k in range(m + 1)]


def lap_pinv_block(q_a, a_rows, a_cols, b_rows, b_cols, n2, n1, cuts_y, cuts_x):
    """R_B (Delta)^dagger E_A q_A by the literal block-DCT sum of Eq. invLaplLowCapLong
    (P:1669-1677), derived via Lemma lmChainOp and Eq. locglobprojpart3
    (P:1491-1503):

        sum_{lambda2, lambda1} ([C_{N2}]^{lambda2}_{m2})^T
            ( R_{A~_lambda} (Delta~)^dagger E_{A~_lambda} )
            ( [C_{N2}]^{k2}_{lambda2} d_k ([C_{N1}]^{k1}_{lambda1})^T ) [C_{N1}]^{lambda1}_{m1}

    ``a_rows``/``a_cols`` (and ``b_*``) are (first, last) inclusive index ranges on Omega~ of the
    source block A_k and target block B_m; the A~ tiling of frequency space is the product of the
    core partitions ``cuts_y`` x ``cuts_x``.  Each block [C]^{k}_{lambda} is the
    sub-matrix of C_N with rows in A~_lambda and columns in A_k.
    """
    c2, c1 = dct_matrix(n2), dct_matrix(n1)
    lam_full = spectral_inverse(n2, n1)
    ay = slice(a_rows[0], a_rows[1] + 1)
    ax = slice(a_cols[0], a_cols[1] + 1)
    by = slice(b_rows[0], b_rows[1] + 1)
    bx = slice(b_cols[0], b_cols[1] + 1)
    q_a = np.asarray(q_a, np.float64)
    out = np.zeros((b_rows[1] - b_rows[0] + 1, b_cols[1] - b_cols[0] + 1), dtype=np.float64)
    for l2 in range(len(cuts_y) - 1):
        fy = slice(cuts_y[l2], cuts_y[l2 + 1])
        c2_k = c2[fy, ay]                        # [C_{N2}]^{k2}_{lambda2}
        c2_m = c2[fy, by]                        # [C_{N2}]^{lambda2}_{m2}
        for l1 in range(len(cuts_x) - 1):
            fx = slice(cuts_x[l1], cuts_x[l1 + 1])
            c1_k = c1[fx, ax]                    # [C_{N1}]^{k1}_{lambda1}
            c1_m = c1[fx, bx]                    # [C_{N1}]^{lambda1}_{m1}
            blk = c2_k @ q_a @ c1_k.T
            blk = lam_full[fy, fx] * blk         # R_{A~} (Delta~)^dagger E_{A~} (diagonal)
            out += c2_m.T @ blk @ c1_m
    return out
