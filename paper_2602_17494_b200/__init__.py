"""Thin Python binding of the B200-native TV-Stokes library (include/tvstokes.h).

Argument marshalling only: every step of the method runs in the CUDA kernels of
``libtvstokes.so`` (built in-tree by ``build.py`` / ``__graft_entry__.build()``).  There is no
CPU fallback: if the library is missing or no CUDA device is present, calls raise.
PyTorch is used only for device memory and streams.

Names follow the C-ABI: ``tv_stokes_step1``, ``tv_stokes_step2``, ``tv_stokes_denoise``,
``tv_stokes_denoise_host``.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

HERE = os.path.dirname(os.path.abspath(__file__))
# TVS_LIB_PATH: an alternative build of the same library (A/B experiments of build-time variants)
LIB_PATH = os.environ.get("TVS_LIB_PATH") or os.path.join(HERE, "libtvstokes.so")

# exported symbols declared in include/tvstokes.h
ABI_SYMBOLS = [
    "tvs_create", "tvs_destroy", "tvs_last_error", "tvs_nccl_unique_id", "tvs_owned_rows",
    "tvs_layout_range", "tvs_layout_theta", "tv_stokes_step1", "tv_stokes_step2",
    "tv_stokes_denoise", "tv_stokes_denoise_host", "tvs_set_profiling", "tvs_kernel_times",
    "tvs_reset_kernel_times", "tvs_selftest_gemm", "tvs_dist_rows", "tv_stokes_step2_irv1",
    "tvs_set_stopping", "tvs_create_virtual_group", "tvs_set_trace",
]

STATUS = {0: "TVS_OK", 1: "TVS_EINVAL", 2: "TVS_ELAYOUT", 4: "TVS_ENUMERIC", 5: "TVS_ECUDA",
          6: "TVS_ENCCL", 7: "TVS_ENOMEM"}
KERNEL_FAMILIES = ["sweep2", "sweep1", "prediv", "proj_fwd_gemm", "proj_solve", "proj_inv_gemm",
                   "other", "proj_fwd_czt", "proj_inv_czt"]


class TvsError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class Layout(ctypes.Structure):
    _fields_ = [("m2", ctypes.c_int32), ("m1", ctypes.c_int32),
                ("overlap_y", ctypes.c_int32), ("overlap_x", ctypes.c_int32)]


class Iters(ctypes.Structure):
    _fields_ = [("sweeps", ctypes.c_int32), ("inner", ctypes.c_int32), ("t", ctypes.c_float)]


class Stats(ctypes.Structure):
    _fields_ = [("seconds", ctypes.c_double), ("pixel_updates", ctypes.c_int64),
                ("launches", ctypes.c_int64), ("flops_proj", ctypes.c_double),
                ("bytes_sweep", ctypes.c_double), ("dual_energy", ctypes.c_double),
                ("sweeps_run", ctypes.c_int64), ("primal_energy", ctypes.c_double),
                ("gap", ctypes.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libtvstokes.so (fails loudly if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"libtvstokes.so not found at {path}: run __graft_entry__.build() "
                           "(the product path has no CPU fallback)")
    lib = ctypes.CDLL(path)
    P = ctypes.c_void_p
    i32, f32 = ctypes.c_int32, ctypes.c_float
    LP, IP = ctypes.POINTER(Layout), ctypes.POINTER(Iters)
    lib.tvs_create.argtypes = [ctypes.POINTER(P), ctypes.c_int, ctypes.c_int, P, ctypes.c_int]
    lib.tvs_destroy.argtypes = [P]
    lib.tvs_create_virtual_group.argtypes = [ctypes.POINTER(P), ctypes.c_int, ctypes.c_int]
    lib.tvs_last_error.argtypes = [P]
    lib.tvs_last_error.restype = ctypes.c_char_p
    lib.tvs_nccl_unique_id.argtypes = [P]
    lib.tvs_owned_rows.argtypes = [i32, i32, ctypes.POINTER(Layout), ctypes.c_int, ctypes.c_int,
                                   ctypes.POINTER(i32), ctypes.POINTER(i32)]
    lib.tvs_dist_rows.argtypes = [i32, i32, LP, i32, ctypes.c_int, ctypes.c_int, ctypes.c_int32 * 16]
    lib.tvs_layout_range.argtypes = [i32, i32, i32, i32, ctypes.POINTER(i32), ctypes.POINTER(i32)]
    lib.tvs_layout_theta.argtypes = [i32, i32, i32, i32, i32, ctypes.POINTER(ctypes.c_double)]
    lib.tv_stokes_step1.argtypes = [P, P, i32, i32, f32, LP, IP, P, P,
                                    ctypes.POINTER(Stats), P]
    lib.tv_stokes_step2.argtypes = [P, P, P, i32, i32, f32, LP, IP, P, P,
                                    ctypes.POINTER(Stats), P]
    lib.tv_stokes_step2_irv1.argtypes = [P, P, P, i32, i32, f32, f32, LP, IP, P, P,
                                         ctypes.POINTER(Stats), P]
    lib.tv_stokes_denoise.argtypes = [P, P, i32, i32, f32, f32, LP, IP, IP, P, P,
                                      ctypes.POINTER(Stats), ctypes.POINTER(Stats), P]
    lib.tv_stokes_denoise_host.argtypes = lib.tv_stokes_denoise.argtypes
    lib.tvs_set_profiling.argtypes = [P, ctypes.c_int]
    lib.tvs_set_stopping.argtypes = [P, i32, ctypes.c_double]
    lib.tvs_set_trace.argtypes = [P, ctypes.POINTER(ctypes.c_double), i32, ctypes.POINTER(i32)]
    arr7i = ctypes.c_int64 * len(KERNEL_FAMILIES)
    arr7d = ctypes.c_double * len(KERNEL_FAMILIES)
    lib.tvs_kernel_times.argtypes = [P, arr7i, arr7d, arr7d, arr7d]
    lib.tvs_reset_kernel_times.argtypes = [P]
    lib.tvs_selftest_gemm.argtypes = [P, i32, i32, i32, i32, ctypes.c_uint64,
                                      ctypes.POINTER(ctypes.c_double)]
    for name in ABI_SYMBOLS:
        if name != "tvs_last_error":
            getattr(lib, name).restype = ctypes.c_int
    _lib = lib
    return lib


# ----------------------------------------------------------------------------- host-only helpers

def layout_range(n, m, s, k):
    lib = load_library()
    lo, hi = ctypes.c_int32(), ctypes.c_int32()
    st = lib.tvs_layout_range(n, m, s, k, ctypes.byref(lo), ctypes.byref(hi))
    if st:
        raise TvsError(st, "tvs_layout_range")
    return lo.value, hi.value


def layout_theta(n, m, s, k, x):
    lib = load_library()
    th = ctypes.c_double()
    st = lib.tvs_layout_theta(n, m, s, k, x, ctypes.byref(th))
    if st:
        raise TvsError(st, "tvs_layout_theta")
    return th.value


def owned_rows(n2, n1, layout, rank, world):
    lib = load_library()
    a, b = ctypes.c_int32(), ctypes.c_int32()
    st = lib.tvs_owned_rows(n2, n1, ctypes.byref(_layout(layout)), rank, world, ctypes.byref(a), ctypes.byref(b))
    if st:
        raise TvsError(st, "tvs_owned_rows")
    return a.value, b.value


DIST_FIELDS = ["k0", "k1", "R0", "R1", "E0", "E1", "V0", "V1", "us0", "us1", "ur0", "ur1",
               "ds0", "ds1", "dr0", "dr1"]


def dist_rows(n2, n1, layout, step, rank, world):
    """Slab decomposition rows of `rank` (host only; see tvs_dist_rows in include/tvstokes.h)."""
    lib = load_library()
    out = (ctypes.c_int32 * 16)()
    st = lib.tvs_dist_rows(n2, n1, ctypes.byref(_layout(layout)), step, rank, world, out)
    if st:
        raise TvsError(st, "tvs_dist_rows")
    return dict(zip(DIST_FIELDS, list(out)))


def nccl_unique_id():
    lib = load_library()
    buf = (ctypes.c_uint8 * 128)()
    st = lib.tvs_nccl_unique_id(buf)
    if st:
        raise TvsError(st, "tvs_nccl_unique_id")
    return bytes(buf)


def _layout(L):
    if isinstance(L, Layout):
        return L
    m2, m1, sy, sx = L
    return Layout(m2, m1, sy, sx)


def _iters(it):
    if isinstance(it, Iters):
        return it
    sweeps, inner, t = it
    return Iters(sweeps, inner, t)


# ----------------------------------------------------------------------------- context


@dataclass
class KernelTimes:
    counts: list
    ms: list
    bytes: list
    flops: list


class Context:
    """Owns a tvs_ctx on one CUDA device.  Arrays are torch CUDA float32 tensors (device entry
    points) or numpy float32 arrays (``*_host``)."""

    def __init__(self, device: int = 0, rank: int = 0, world: int = 1, nccl_id: bytes = None):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("tvstokes needs a CUDA device (no CPU fallback)")
        self.lib = load_library()
        self.device = device
        h = ctypes.c_void_p()
        idbuf = (ctypes.c_uint8 * 128).from_buffer_copy(nccl_id) if nccl_id else None
        st = self.lib.tvs_create(ctypes.byref(h), rank, world, idbuf, device)
        if st:
            raise TvsError(st, "tvs_create")
        self.h = h

    @classmethod
    def virtual_group(cls, world: int, device: int = 0):
        """`world` contexts on one GPU forming a virtual slab group (tvs_create_virtual_group):
        drive each from its own thread and stream; exchanges are device-to-device copies."""
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("tvstokes needs a CUDA device (no CPU fallback)")
        lib = load_library()
        hs = (ctypes.c_void_p * world)()
        st = lib.tvs_create_virtual_group(hs, world, device)
        if st:
            raise TvsError(st, "tvs_create_virtual_group")
        out = []
        for r in range(world):
            c = cls.__new__(cls)
            c.lib, c.device, c.h = lib, device, ctypes.c_void_p(hs[r])
            c.vrank = r
            out.append(c)
        return out

    def close(self):
        if getattr(self, "h", None):
            self.lib.tvs_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st, what):
        if st:
            raise TvsError(st, f"{what}: {self.lib.tvs_last_error(self.h).decode()}")

    @staticmethod
    def _ptr(t):
        return ctypes.c_void_p(t.data_ptr()) if t is not None else None

    def _stream(self, stream):
        import torch
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        return ctypes.c_void_p(s.cuda_stream)

    def _dev(self, x, shape):
        import torch
        assert isinstance(x, torch.Tensor) and x.is_cuda and x.dtype == torch.float32, \
            "expected a CUDA float32 tensor"
        assert x.is_contiguous() and tuple(x.shape) == tuple(shape), (x.shape, shape)
        return x

    def tv_stokes_step1(self, d0, delta, layout, iters, want_p=False, stream=None):
        import torch
        n2, n1 = d0.shape
        self._dev(d0, (n2, n1))
        tau = torch.empty((2, n2 + 1, n1 + 1), device=d0.device, dtype=torch.float32)
        p = torch.empty((4, n2 + 1, n1 + 1), device=d0.device, dtype=torch.float32) if want_p else None
        st = Stats()
        self._check(self.lib.tv_stokes_step1(self.h, self._ptr(d0), n2, n1, float(delta),
                                             ctypes.byref(_layout(layout)), ctypes.byref(_iters(iters)), self._ptr(tau),
                                             self._ptr(p), ctypes.byref(st), self._stream(stream)),
                    "tv_stokes_step1")
        return tau, p, st

    def tv_stokes_step2(self, tau, d0, lam, layout, iters, want_p=False, stream=None,
                        variant="irv2", eps=1e-3):
        """Step 2: ``variant='irv2'`` (tv_stokes_step2, lam = 1/alpha) or ``'irv1'``
        (tv_stokes_step2_irv1, lam = mu = 1/alpha, xi smoothing ``eps``)."""
        import torch
        n2, n1 = d0.shape
        self._dev(d0, (n2, n1))
        self._dev(tau, (2, n2 + 1, n1 + 1))
        d = torch.empty((n2, n1), device=d0.device, dtype=torch.float32)
        p = torch.empty((2, n2, n1), device=d0.device, dtype=torch.float32) if want_p else None
        st = Stats()
        L, it = ctypes.byref(_layout(layout)), ctypes.byref(_iters(iters))
        if variant == "irv1":
            self._check(self.lib.tv_stokes_step2_irv1(self.h, self._ptr(tau), self._ptr(d0), n2, n1,
                                                      float(lam), float(eps), L, it, self._ptr(d),
                                                      self._ptr(p), ctypes.byref(st),
                                                      self._stream(stream)), "tv_stokes_step2_irv1")
        elif variant == "irv2":
            self._check(self.lib.tv_stokes_step2(self.h, self._ptr(tau), self._ptr(d0), n2, n1,
                                                 float(lam), L, it, self._ptr(d), self._ptr(p),
                                                 ctypes.byref(st), self._stream(stream)),
                        "tv_stokes_step2")
        else:
            raise ValueError(f"unknown step-2 variant {variant!r}")
        return d, p, st

    def tv_stokes_denoise(self, d0, delta, lam, layout, it1, it2, want_tau=False, stream=None,
                          out=None):
        import torch
        n2, n1 = d0.shape
        self._dev(d0, (n2, n1))
        d = out if out is not None else torch.empty((n2, n1), device=d0.device, dtype=torch.float32)
        tau = torch.empty((2, n2 + 1, n1 + 1), device=d0.device, dtype=torch.float32) if want_tau else None
        s1, s2 = Stats(), Stats()
        self._check(self.lib.tv_stokes_denoise(self.h, self._ptr(d0), n2, n1, float(delta),
                                               float(lam), ctypes.byref(_layout(layout)),
                                               ctypes.byref(_iters(it1)), ctypes.byref(_iters(it2)), self._ptr(d), self._ptr(tau),
                                               ctypes.byref(s1), ctypes.byref(s2),
                                               self._stream(stream)), "tv_stokes_denoise")
        return d, tau, s1, s2

    def tv_stokes_denoise_host(self, d0, delta, lam, layout, it1, it2, out=None, stream=None):
        """Host (numpy float32) in, host out: the H2D/D2H copies are inside the call."""
        import numpy as np
        d0 = np.ascontiguousarray(d0, dtype=np.float32)
        n2, n1 = d0.shape
        d = out if out is not None else np.empty((n2, n1), dtype=np.float32)
        s1, s2 = Stats(), Stats()
        self._check(self.lib.tv_stokes_denoise_host(
            self.h, ctypes.c_void_p(d0.ctypes.data), n2, n1, float(delta), float(lam),
            ctypes.byref(_layout(layout)), ctypes.byref(_iters(it1)), ctypes.byref(_iters(it2)),
            ctypes.c_void_p(d.ctypes.data), None,
            ctypes.byref(s1), ctypes.byref(s2), self._stream(stream)), "tv_stokes_denoise_host")
        return d, s1, s2

    def selftest_gemm(self, M, N, K, impl, seed=1):
        err = ctypes.c_double()
        self._check(self.lib.tvs_selftest_gemm(self.h, M, N, K, impl, seed, ctypes.byref(err)),
                    "tvs_selftest_gemm")
        return err.value

    def set_stopping(self, criterion: int, tol: float = 0.0):
        """Outer-loop stopping rule (tvs_set_stopping): 0 fixed schedule, 1 the sqrt(D) criterion
        of section 5.2, 2 the D^2 criterion of section 6.3."""
        self._check(self.lib.tvs_set_stopping(self.h, int(criterion), float(tol)), "tvs_set_stopping")

    def set_trace(self, cap: int):
        """Per-sweep (E, D, gap) of the Schwarz iterates of the following calls (tvs_set_trace);
        read them with ``trace()`` after a call; cap = 0 turns it off."""
        import numpy as np
        self._trace_buf = np.zeros((max(cap, 1), 3))
        self._trace_n = ctypes.c_int32(0)
        self._check(self.lib.tvs_set_trace(
            self.h, self._trace_buf.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) if cap else None,
            int(cap), ctypes.byref(self._trace_n)), "tvs_set_trace")

    def trace(self):
        """(n_entries, 3) array of the last traced call: columns E, D, gap."""
        return self._trace_buf[: self._trace_n.value].copy()

    def set_profiling(self, on: bool):
        self._check(self.lib.tvs_set_profiling(self.h, 1 if on else 0), "tvs_set_profiling")

    def reset_kernel_times(self):
        self._check(self.lib.tvs_reset_kernel_times(self.h), "tvs_reset_kernel_times")

    def kernel_times(self) -> KernelTimes:
        n = len(KERNEL_FAMILIES)
        c = (ctypes.c_int64 * n)()
        ms, by, fl = (ctypes.c_double * n)(), (ctypes.c_double * n)(), (ctypes.c_double * n)()
        self._check(self.lib.tvs_kernel_times(self.h, c, ms, by, fl), "tvs_kernel_times")
        return KernelTimes(list(c), list(ms), list(by), list(fl))


_default_ctx = None


def default_context():
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


def tv_stokes_step1(d0, delta, layout, iters, **kw):
    return default_context().tv_stokes_step1(d0, delta, layout, iters, **kw)


def tv_stokes_step2(tau, d0, lam, layout, iters, **kw):
    return default_context().tv_stokes_step2(tau, d0, lam, layout, iters, **kw)


def tv_stokes_denoise(d0, delta, lam, layout, it1, it2, **kw):
    return default_context().tv_stokes_denoise(d0, delta, lam, layout, it1, it2, **kw)


def tv_stokes_denoise_host(d0, delta, lam, layout, it1, it2, **kw):
    return default_context().tv_stokes_denoise_host(d0, delta, lam, layout, it1, it2, **kw)
