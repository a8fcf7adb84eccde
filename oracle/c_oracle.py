"""ctypes binding of the plain C11 fp64 oracle ``oracle/c/tvo.c`` (test infrastructure only; see
oracle/__init__.py).  The C oracle is the NumPy-free implementation the north star asks for, with
the tvo_* calls of SURVEY 8(b) ("Oracle": the library's three calls with double and host
pointers), threaded one task per subdomain.  It is compiled in-tree with gcc (by
``__graft_entry__.build()`` or on first use here) and pinned by tests/test_oracle_c.py: the same
pins as the NumPy oracle, plus agreement of the two independently written oracles."""
import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "c", "tvo.c")
LIB = os.path.join(HERE, "c", "libtvo.so")
_lib = None


def build(force=False):
    """gcc -O2 -std=c11 -pthread -shared: oracle/c/libtvo.so (no GPU, no NumPy)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.run(["gcc", "-O2", "-std=c11", "-Wall", "-pthread", "-shared", "-fPIC", "-o", LIB,
                        SRC, "-lm"], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB)
        D, I = ctypes.POINTER(ctypes.c_double), ctypes.c_int
        I4 = ctypes.c_int * 4
        L.tvo_step1.argtypes = [D, I, I, ctypes.c_double, I4, I, I, ctypes.c_double, I, D, D, D]
        L.tvo_step2.argtypes = [D, D, I, I, ctypes.c_double, I4, I, I, ctypes.c_double, I, D, D, D]
        L.tvo_grad.argtypes = [D, I, I, D]
        L.tvo_div.argtypes = [D, I, I, D]
        L.tvo_lap_pinv.argtypes = [D, I, I, D]
        L.tvo_project.argtypes = [D, I, I, D]
        L.tvo_tau0.argtypes = [D, I, I, D]
        L.tvo_layout_range.argtypes = [I, I, I, I, ctypes.POINTER(I), ctypes.POINTER(I)]
        L.tvo_layout_theta.argtypes = [I, I, I, I, I]
        L.tvo_layout_theta.restype = ctypes.c_double
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _arr(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class OracleError(RuntimeError):
    pass


def _ck(st, what):
    if st:
        raise OracleError(f"{what}: status {st}")


def grad(u):
    u = _arr(u)
    out = np.empty((2,) + u.shape)
    lib().tvo_grad(_p(u), u.shape[0], u.shape[1], _p(out))
    return out


def div(p):
    p = _arr(p)
    out = np.empty(p.shape[1:])
    lib().tvo_div(_p(p), p.shape[1], p.shape[2], _p(out))
    return out


def lap_pinv(q):
    q = _arr(q)
    out = np.empty(q.shape)
    _ck(lib().tvo_lap_pinv(_p(q), q.shape[0], q.shape[1], _p(out)), "tvo_lap_pinv")
    return out


def project(w):
    w = _arr(w)
    out = np.empty(w.shape)
    _ck(lib().tvo_project(_p(w), w.shape[1], w.shape[2], _p(out)), "tvo_project")
    return out


def tau0(d0):
    d0 = _arr(d0)
    out = np.empty((2, d0.shape[0] + 1, d0.shape[1] + 1))
    lib().tvo_tau0(_p(d0), d0.shape[0], d0.shape[1], _p(out))
    return out


def layout_range(n, m, s, k):
    lo, hi = ctypes.c_int(), ctypes.c_int()
    _ck(lib().tvo_layout_range(n, m, s, k, ctypes.byref(lo), ctypes.byref(hi)), "tvo_layout_range")
    return lo.value, hi.value


def layout_theta(n, m, s, k, x):
    return lib().tvo_layout_theta(n, m, s, k, x)


def step1(d0, delta, layout, sweeps, inner, t=0.125, threads=1):
    """tvo_step1: returns (tau (2, n2+1, n1+1), p (2, 2, n2+1, n1+1), stats {E, D, gap})."""
    d0 = _arr(d0)
    n2, n1 = d0.shape
    tau = np.empty((2, n2 + 1, n1 + 1))
    p = np.empty((2, 2, n2 + 1, n1 + 1))
    st = np.empty(3)
    _ck(lib().tvo_step1(_p(d0), n2, n1, delta, (ctypes.c_int * 4)(*layout), sweeps, inner, t,
                        threads, _p(tau), _p(p), _p(st)), "tvo_step1")
    return tau, p, {"E": st[0], "D": st[1], "gap": st[2]}


def step2(d0, tau, lam, layout, sweeps, inner, t=0.125, threads=1):
    """tvo_step2 (IRV2): returns (d, p (2, n2, n1), stats {E, D, gap})."""
    d0, tau = _arr(d0), _arr(tau)
    n2, n1 = d0.shape
    d = np.empty((n2, n1))
    p = np.empty((2, n2, n1))
    st = np.empty(3)
    _ck(lib().tvo_step2(_p(tau), _p(d0), n2, n1, lam, (ctypes.c_int * 4)(*layout), sweeps, inner, t,
                        threads, _p(d), _p(p), _p(st)), "tvo_step2")
    return d, p, {"E": st[0], "D": st[1], "gap": st[2]}
