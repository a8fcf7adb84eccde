"""Finite-difference calculus of PAPER.md section 4.1, fp64, h = 1.

Arrays are indexed [i, j] = [row (y), column (x)], 0-based (the paper is 1-based).
A vector field is an array of shape (2, n2, n1): [0] = x-component, [1] = y-component
(grad = (D+_x, D+_y)^T, Eq. defGradDis).  A 2x2 multi-field has shape (2, 2, n2, n1):
[k] is the k-th 2-vector row p_k (multidiv acts row-wise).
Oracle: test infrastructure only (see oracle/__init__.py).
"""
import numpy as np


def dplus_x(u):
    """(D+_x u)_{i,j} = u_{i,j+1} - u_{i,j} for j < N1, 0 at j = N1."""
    out = np.zeros_like(u, dtype=np.float64)
    out[:, :-1] = u[:, 1:] - u[:, :-1]
    return out


def dplus_y(u):
    """(D+_y u)_{i,j} = u_{i+1,j} - u_{i,j} for i < N2, 0 at i = N2."""
    out = np.zeros_like(u, dtype=np.float64)
    out[:-1, :] = u[1:, :] - u[:-1, :]
    return out


def dminus_x(u):
    """Three-case backward difference: u_1 | u_j - u_{j-1} | -u_{N1-1}."""
    n = u.shape[1]
    assert n >= 2
    out = np.empty_like(u, dtype=np.float64)
    out[:, 0] = u[:, 0]
    out[:, 1:n - 1] = u[:, 1:n - 1] - u[:, 0:n - 2]
    out[:, n - 1] = -u[:, n - 2]
    return out


def dminus_y(u):
    """Three-case backward difference in y."""
    n = u.shape[0]
    assert n >= 2
    out = np.empty_like(u, dtype=np.float64)
    out[0, :] = u[0, :]
    out[1:n - 1, :] = u[1:n - 1, :] - u[0:n - 2, :]
    out[n - 1, :] = -u[n - 2, :]
    return out


def grad(u):
    """grad u = (D+_x u, D+_y u)^T (Eq. defGradDis)."""
    return np.stack([dplus_x(u), dplus_y(u)])


def div(p):
    """div p = D-_x p_1 + D-_y p_2 (Eq. defDivDis); div = -grad^* (P:597)."""
    return dminus_x(p[0]) + dminus_y(p[1])


def multigrad(u):
    """Row-wise gradient of a 2-vector field: (grad u_1, grad u_2)^T."""
    return np.stack([grad(u[0]), grad(u[1])])


def multidiv(p):
    """Row-wise divergence of a 2x2 field: (div p_1, div p_2)^T."""
    return np.stack([div(p[0]), div(p[1])])


def laplacian(u):
    """Delta = div grad."""
    return div(grad(u))


def dneum_x(d):
    """D_x^{neum-}: X(Omega) -> X(Omega~) (Eq. def:backdiffNeumann).

    0 on the first and last column j = 1, N1+1; d_{i,j} - d_{i,j-1} for j = 2..N1, i <= N2;
    the mirrored extra row i = N2+1 repeats row N2's differences.
    """
    n2, n1 = d.shape
    out = np.zeros((n2 + 1, n1 + 1), dtype=np.float64)
    dd = np.asarray(d, dtype=np.float64)
    out[:n2, 1:n1] = dd[:, 1:] - dd[:, :-1]
    out[n2, 1:n1] = dd[n2 - 1, 1:] - dd[n2 - 1, :-1]
    return out


def dneum_y(d):
    """D_y^{neum-}: 0 on rows 1 and N2+1; mirrored extra column j = N1+1."""
    n2, n1 = d.shape
    out = np.zeros((n2 + 1, n1 + 1), dtype=np.float64)
    dd = np.asarray(d, dtype=np.float64)
    out[1:n2, :n1] = dd[1:, :] - dd[:-1, :]
    out[1:n2, n1] = dd[1:, n1 - 1] - dd[:-1, n1 - 1]
    return out


def inner(a, b):
    """<a, b> with h = 1: plain sum of products over all entries."""
    return float(np.sum(np.asarray(a, np.float64) * np.asarray(b, np.float64)))
