"""Brute-force pair sums in plain C (oracle/bf.c) -- TEST INFRASTRUCTURE ONLY.

ctypes wrapper of the O12 building block u_t = sum_{s: t != s} q_s G_p(t - s) (P:172,
Eq. hms_d2) with the Ewald sums of oracle/pgf.py restated in C + OpenMP, so that
AIM-vs-brute-force checks on meshes of 10^3-10^6 nodes finish in seconds.  The shared object is
compiled with gcc on first use (and by __graft_entry__.build()); it is pinned against
oracle/pgf.py and against closed forms in tests/test_oracle_bf.py.
"""
import ctypes
import os
import subprocess

import numpy as np

from .pgf import PgfSpec

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "bf.c")
_LIB = os.path.join(_HERE, "_build", "libbf.so")
_lib = None


def build(force=False):
    """Compile oracle/bf.c -> oracle/_build/libbf.so (gcc -O2 -fopenmp)."""
    if not force and os.path.exists(_LIB) and os.path.getmtime(_LIB) >= os.path.getmtime(_SRC):
        return _LIB
    os.makedirs(os.path.dirname(_LIB), exist_ok=True)
    tmp = _LIB + ".%d.tmp" % os.getpid()
    subprocess.run(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-o", tmp, _SRC, "-lm"], check=True)
    os.replace(tmp, _LIB)
    return _LIB


class _Spec(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int), ("ax", ctypes.c_int * 3), ("L", ctypes.c_double * 3),
                ("alpha", ctypes.c_double), ("nreal", ctypes.c_int * 3), ("mrec", ctypes.c_int * 3)]


def _load():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.POINTER
        _lib.bf_potential.argtypes = [P(_Spec), ctypes.c_int64, P(ctypes.c_double), ctypes.c_int64,
                                      P(ctypes.c_double), P(ctypes.c_double), P(ctypes.c_double)]
        _lib.bf_pgf_points.argtypes = [P(_Spec), ctypes.c_int64, P(ctypes.c_double), ctypes.c_int,
                                       P(ctypes.c_double)]
    return _lib


def _cspec(spec):
    if spec.dim == 0:
        raise ValueError("bf.c covers periodic kernels only (free space: 1/|r| in oracle.pgf)")
    s = _Spec()
    s.dim = spec.dim
    ax = list(spec.axes) + list(spec.free)
    for i in range(3):
        s.ax[i] = ax[i]
        s.L[i] = float(spec.L[i]) if i < spec.dim else 0.0
        s.nreal[i] = int(spec.n_real[i]) if i < spec.dim else 0
        s.mrec[i] = int(spec.m_recip[i]) if i < spec.dim else 0
    s.alpha = float(spec.alpha)
    return s


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def pgf(r, spec):
    """G_p(r) at points r [P,3] (r not a lattice vector); same definition as oracle.pgf.pgf."""
    r = np.ascontiguousarray(np.atleast_2d(r), dtype=np.float64)
    out = np.zeros(r.shape[0])
    cs = _cspec(spec)
    _load().bf_pgf_points(ctypes.byref(cs), r.shape[0], _dp(r), 0, _dp(out))
    return out


def pgf_self(spec):
    """G_p^reg(0) (reading R13); same definition as oracle.pgf.pgf_self."""
    out = np.zeros(1)
    r = np.zeros((1, 3))
    cs = _cspec(spec)
    _load().bf_pgf_points(ctypes.byref(cs), 1, _dp(r), 1, _dp(out))
    return float(out[0])


def potential(targets, sources, q, spec):
    """sum_k q_k G_p(t_n - s_k) over pairs with t_n != s_k (as oracle.pgf.pgf_potential)."""
    t = np.ascontiguousarray(np.atleast_2d(targets), dtype=np.float64)
    s = np.ascontiguousarray(np.atleast_2d(sources), dtype=np.float64)
    q = np.ascontiguousarray(q, dtype=np.float64)
    out = np.zeros(t.shape[0])
    cs = _cspec(spec)
    st = _load().bf_potential(ctypes.byref(cs), t.shape[0], _dp(t), s.shape[0], _dp(s), _dp(q), _dp(out))
    if st != 0:
        raise ValueError("bf_potential: reciprocal range too large")
    return out
