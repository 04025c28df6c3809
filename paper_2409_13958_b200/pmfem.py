"""Thin ctypes binding of libpmfem (include/pmfem.h): argument marshalling only.

Every step of the H_eff path runs in the library's CUDA kernels; PyTorch supplies device
memory and streams.  There is no CPU fallback: if the shared library is missing or cannot be
loaded, importing this module raises.
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# PMFEM_LIB=checked loads the build with device-side bounds asserts (build.py --checked)
LIB_PATH = os.path.join(_HERE, "lib", "libpmfem_checked.so" if os.environ.get("PMFEM_LIB") == "checked"
                        else "libpmfem.so")

if not os.path.exists(LIB_PATH):
    raise ImportError("libpmfem.so not built (%s); run __graft_entry__.build() or "
                      "python paper_2409_13958_b200/build.py" % LIB_PATH)
_lib = ctypes.CDLL(LIB_PATH)

STATUS = {0: "PMFEM_OK", 1: "PMFEM_E_INVALID_ARG", 2: "PMFEM_E_MESH", 3: "PMFEM_E_PBC_AMBIGUOUS",
          4: "PMFEM_E_PBC_INCONSISTENT", 5: "PMFEM_E_OUTSIDE_GRID", 6: "PMFEM_E_RER_TOO_LARGE",
          7: "PMFEM_E_PGF_NOT_CONVERGED", 8: "PMFEM_E_STATE", 9: "PMFEM_E_CUDA", 10: "PMFEM_E_NCCL",
          11: "PMFEM_E_OOM"}

SYMBOLS = ["pmfem_setup", "pmfem_setup_dist", "pmfem_nccl_unique_id", "pmfem_build_pgf", "pmfem_llg_rk4",
           "pmfem_llg_am2", "pmfem_set_anisotropy", "pmfem_build_pgf_bloch", "pmfem_demag", "pmfem_exchange",
           "pmfem_heff", "pmfem_build_bloch", "pmfem_demag_bloch", "pmfem_exchange_bloch", "pmfem_heff_bloch",
           "pmfem_heff_host", "pmfem_query", "pmfem_get_order", "pmfem_export", "pmfem_set_timing",
           "pmfem_get_timing", "pmfem_last_error", "pmfem_destroy"]


class PmfemError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__("%s: %s" % (STATUS.get(status, status), msg))
        self.status = status


class _Mesh(ctypes.Structure):
    _fields_ = [("n_nodes", ctypes.c_int64), ("xyz", ctypes.POINTER(ctypes.c_double)),
                ("n_tets", ctypes.c_int64), ("tets", ctypes.POINTER(ctypes.c_int32)),
                ("region", ctypes.POINTER(ctypes.c_int32)), ("n_regions", ctypes.c_int32),
                ("Ms", ctypes.POINTER(ctypes.c_double)), ("Aex", ctypes.POINTER(ctypes.c_double))]


class _Periodicity(ctypes.Structure):
    _fields_ = [("periodic", ctypes.c_int32 * 3), ("lattice", (ctypes.c_double * 3) * 3),
                ("match_tol", ctypes.c_double)]


class _Grid(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32 * 3), ("order", ctypes.c_int32), ("rer_scale", ctypes.c_double),
                ("z0_ring", ctypes.c_int32)]


class _Info(ctypes.Structure):
    _fields_ = [("n_nodes", ctypes.c_int64), ("n_parents", ctypes.c_int64), ("n_parents_local", ctypes.c_int64),
                ("periodic_dims", ctypes.c_int32), ("touching", ctypes.c_int32), ("protruding", ctypes.c_int32),
                ("grid", ctypes.c_int32 * 3), ("fft", ctypes.c_int32 * 3),
                ("nnz_ring1", ctypes.c_int64), ("nnz_z0", ctypes.c_int64), ("nnz_cbox", ctypes.c_int64),
                ("bytes_per_eval_algorithmic", ctypes.c_double), ("setup_seconds", ctypes.c_double),
                ("pgf_seconds", ctypes.c_double), ("kernel_bytes", ctypes.c_double * 8),
                ("launches_per_eval", ctypes.c_int32), ("fft_fused", ctypes.c_int32),
                ("comm_bytes_per_eval", ctypes.c_double), ("k2_tile", ctypes.c_int32 * 3),
                ("slab_world", ctypes.c_int32), ("cbox_format", ctypes.c_int32),
                ("cbox_packed_units", ctypes.c_int64), ("pgf_achieved_rel_err", ctypes.c_double)]


_vp = ctypes.c_void_p
_lib.pmfem_setup.argtypes = [ctypes.POINTER(_vp), ctypes.POINTER(_Mesh), ctypes.POINTER(_Periodicity),
                             ctypes.POINTER(_Grid), ctypes.c_int]
_lib.pmfem_setup_dist.argtypes = [ctypes.POINTER(_vp), ctypes.POINTER(_Mesh), ctypes.POINTER(_Periodicity),
                                  ctypes.POINTER(_Grid), ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
_lib.pmfem_nccl_unique_id.argtypes = [ctypes.c_void_p]
_lib.pmfem_build_pgf.argtypes = [_vp, ctypes.c_double]
for _n in ("pmfem_demag", "pmfem_exchange", "pmfem_heff", "pmfem_heff_host"):
    getattr(_lib, _n).argtypes = [_vp, _vp, _vp, _vp]
_lib.pmfem_llg_rk4.argtypes = [_vp, _vp, ctypes.c_int64, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                              ctypes.c_void_p, _vp]
_lib.pmfem_llg_am2.argtypes = [_vp, _vp, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                               ctypes.c_double, ctypes.c_void_p, ctypes.c_double, _vp,
                               ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]
_lib.pmfem_set_anisotropy.argtypes = [_vp, ctypes.c_int, ctypes.c_double, ctypes.c_void_p]
_lib.pmfem_build_pgf_bloch.argtypes = [_vp, ctypes.c_void_p, ctypes.c_double]
_lib.pmfem_build_bloch.argtypes = [_vp, ctypes.c_void_p, ctypes.c_double]
for _n in ("pmfem_demag_bloch", "pmfem_exchange_bloch", "pmfem_heff_bloch"):
    getattr(_lib, _n).argtypes = [_vp, _vp, _vp, _vp, _vp, _vp]
_lib.pmfem_query.argtypes = [_vp, ctypes.POINTER(_Info)]
_lib.pmfem_get_order.argtypes = [_vp, ctypes.POINTER(ctypes.c_int64)]
_lib.pmfem_export.argtypes = [_vp, ctypes.c_char_p, _vp, ctypes.POINTER(ctypes.c_int64)]
_lib.pmfem_set_timing.argtypes = [_vp, ctypes.c_int]
_lib.pmfem_get_timing.argtypes = [_vp, ctypes.POINTER(ctypes.c_float)]
_lib.pmfem_last_error.argtypes = [_vp]
_lib.pmfem_last_error.restype = ctypes.c_char_p
_lib.pmfem_destroy.argtypes = [_vp]
for _n in SYMBOLS:
    if _n not in ("pmfem_last_error", "pmfem_destroy"):
        getattr(_lib, _n).restype = ctypes.c_int

_EXPORT_DTYPES = {"parent": np.int64, "lca": np.int64, "shift": np.int32, "ring1_rowptr": np.int64,
                  "ring1_col": np.int32, "z0_rowptr": np.int64, "z0_col": np.int32, "cbox_rowptr": np.int64,
                  "cbox_col": np.int32, "stencil_s": np.int32, "perm": np.int64, "dist_bounds": np.int64}
_EXPORT_DTYPES.update({"cbox_device_rowptr": np.int64, "cbox_device_col": np.int32,
                       "cbox_device_val": np.float32, "cbox_device_chunks": np.int64,
                       "cbox_device_format": np.int64, "slab_kranges": np.int64,
                       "dist_planes": np.int64, "dist_ghost": np.int64, "axis_perm": np.int64})
for _k in ("r1", "z0", "cbox"):
    _EXPORT_DTYPES["bloch_%s_rowptr" % _k] = np.int64
    _EXPORT_DTYPES["bloch_%s_col" % _k] = np.int32
for _k in "mqu":
    _EXPORT_DTYPES["send_%s_ptr" % _k] = np.int64
    _EXPORT_DTYPES["recv_%s_ptr" % _k] = np.int64
    _EXPORT_DTYPES["send_%s_idx" % _k] = np.int32
    _EXPORT_DTYPES["recv_%s_idx" % _k] = np.int32

KERNELS = ["K1_local_in", "K2_anterp", "K3_fft_conv", "K4_interp_corr", "K5_grad_sum"]


def _ptr(a, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def _dev_ptr(t, rows=None, device=None):
    """Device pointer of a contiguous float32 CUDA tensor [rows, 3] on `device` (the ABI takes
    no row count: a wrong shape or device would read/write out of bounds, so it is checked here)."""
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()):
        raise TypeError("expected a contiguous float32 CUDA tensor")
    if rows is not None and tuple(t.shape) != (rows, 3):
        raise ValueError("expected shape (%d, 3), got %s" % (rows, tuple(t.shape)))
    if device is not None and t.device.index != device:
        raise ValueError("tensor on cuda:%s, context on cuda:%d" % (t.device.index, device))
    return ctypes.c_void_p(t.data_ptr())


def _host_ptr(t, rows):
    """Host pointer of a contiguous float32 CPU tensor [rows, 3]."""
    import torch
    if not (isinstance(t, torch.Tensor) and not t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()):
        raise TypeError("expected a contiguous float32 CPU tensor")
    if tuple(t.shape) != (rows, 3):
        raise ValueError("expected shape (%d, 3), got %s" % (rows, tuple(t.shape)))
    return _vp(t.data_ptr())


class Context:
    """Owns a pmfem_ctx.  device=-1 builds a host-only context (setup artifacts, no fields)."""

    def __init__(self, xyz, tets, periodic, lattice, grid_n, Ms=637.0, Aex=1.4e-6, order=1,
                 rer_scale=2.0, z0_ring=1, device=0, region=None, match_tol=0.0, rank=0, world=1,
                 nccl_id=None):
        xyz = np.ascontiguousarray(xyz, dtype=np.float64)
        tets = np.ascontiguousarray(tets, dtype=np.int32)
        Ms = np.ascontiguousarray(np.atleast_1d(Ms), dtype=np.float64)
        Aex = np.ascontiguousarray(np.atleast_1d(Aex), dtype=np.float64)
        self._keep = [xyz, tets, Ms, Aex]
        m = _Mesh(xyz.shape[0], _ptr(xyz, ctypes.c_double), tets.shape[0], _ptr(tets, ctypes.c_int32),
                  None, Ms.size, _ptr(Ms, ctypes.c_double), _ptr(Aex, ctypes.c_double))
        if region is not None:
            region = np.ascontiguousarray(region, dtype=np.int32)
            self._keep.append(region)
            m.region = _ptr(region, ctypes.c_int32)
        # lattice: 3 periods (the diagonal) or 3x3 lattice vectors (rows; must be diagonal)
        lat = np.asarray(lattice, dtype=np.float64)
        if lat.shape == (3,):
            lat = np.diag(lat)
        if lat.shape != (3, 3):
            raise ValueError("lattice must be 3 periods or a 3x3 matrix of lattice vectors")
        latc = ((ctypes.c_double * 3) * 3)(*[(ctypes.c_double * 3)(*[float(v) for v in row]) for row in lat])
        p = _Periodicity((ctypes.c_int32 * 3)(*[int(bool(v)) for v in periodic]), latc, float(match_tol))
        g = _Grid((ctypes.c_int32 * 3)(*[int(v) for v in grid_n]), int(order), float(rer_scale), int(z0_ring))
        h = _vp()
        if world == 1:
            st = _lib.pmfem_setup(ctypes.byref(h), ctypes.byref(m), ctypes.byref(p), ctypes.byref(g), int(device))
        else:
            idbuf = None
            if nccl_id is not None:
                idbuf = ctypes.create_string_buffer(bytes(nccl_id), 128)
            st = _lib.pmfem_setup_dist(ctypes.byref(h), ctypes.byref(m), ctypes.byref(p), ctypes.byref(g),
                                       int(device), idbuf, int(rank), int(world))
        self.rank, self.world = rank, world
        if st != 0:
            raise PmfemError(st, _lib.pmfem_last_error(None).decode())
        self._h = h
        self.device = device
        self._keep = None
        info = self.query()
        self.n_parents = info["n_parents"]
        self.n_parents_local = info["n_parents_local"]
        self.n_nodes = info["n_nodes"]

    def _check(self, st):
        if st != 0:
            raise PmfemError(st, _lib.pmfem_last_error(self._h).decode())

    def close(self):
        if getattr(self, "_h", None):
            _lib.pmfem_destroy(self._h)
            self._h = None

    __del__ = close

    def build_pgf(self, target_rel_err=1e-12):
        self._check(_lib.pmfem_build_pgf(self._h, float(target_rel_err)))

    def build_pgf_bloch(self, k0, target_rel_err=1e-12):
        """NEXT-4: the modulated Bloch kernel table + complex spectrum (exports kernel_bloch,
        spectrum_bloch as complex [P2][P1][P0])."""
        k = (ctypes.c_double * 3)(*[float(v) for v in k0])
        self._check(_lib.pmfem_build_pgf_bloch(self._h, ctypes.cast(k, ctypes.c_void_p), float(target_rel_err)))
        P = self.query()["fft"]
        K = self.export("kernel_bloch")
        G = self.export("spectrum_bloch")
        shape = (P[2], P[1], P[0])
        return (K[0::2] + 1j * K[1::2]).reshape(shape), (G[0::2] + 1j * G[1::2]).reshape(shape)

    def build_bloch(self, k0, target_rel_err=1e-12):
        """NEXT-4 complex field path: the Bloch kernel and the phased operators for k0 (rad/cm,
        user frame); then demag_bloch / exchange_bloch / heff_bloch."""
        k = (ctypes.c_double * 3)(*[float(v) for v in k0])
        self._check(_lib.pmfem_build_bloch(self._h, ctypes.cast(k, ctypes.c_void_p), float(target_rel_err)))

    def _eval_bloch(self, fn, m_re, m_im, H_re, H_im, stream):
        import torch
        H_re = torch.empty_like(m_re) if H_re is None else H_re
        H_im = torch.empty_like(m_im) if H_im is None else H_im
        n = self.n_parents_local
        self._check(fn(self._h, _dev_ptr(m_re, n, self.device), _dev_ptr(m_im, n, self.device),
                       _dev_ptr(H_re, n, self.device), _dev_ptr(H_im, n, self.device), self._stream(stream)))
        return H_re, H_im

    def demag_bloch(self, m_re, m_im, H_re=None, H_im=None, stream=None):
        return self._eval_bloch(_lib.pmfem_demag_bloch, m_re, m_im, H_re, H_im, stream)

    def exchange_bloch(self, m_re, m_im, H_re=None, H_im=None, stream=None):
        return self._eval_bloch(_lib.pmfem_exchange_bloch, m_re, m_im, H_re, H_im, stream)

    def heff_bloch(self, m_re, m_im, H_re=None, H_im=None, stream=None):
        return self._eval_bloch(_lib.pmfem_heff_bloch, m_re, m_im, H_re, H_im, stream)

    def _stream(self, stream):
        if stream is None:
            import torch
            stream = torch.cuda.current_stream(self.device)
        return _vp(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))

    def _eval(self, fn, m, H, stream):
        import torch
        if H is None:
            H = torch.empty_like(m)
        n = self.n_parents_local
        fn_st = fn(self._h, _dev_ptr(m, n, self.device), _dev_ptr(H, n, self.device), self._stream(stream))
        self._check(fn_st)
        return H

    def demag(self, m, H=None, stream=None):
        return self._eval(_lib.pmfem_demag, m, H, stream)

    def exchange(self, m, H=None, stream=None):
        return self._eval(_lib.pmfem_exchange, m, H, stream)

    def heff(self, m, H=None, stream=None):
        return self._eval(_lib.pmfem_heff, m, H, stream)

    def heff_host(self, m_host, H_host=None, stream=None):
        """m_host, H_host: float32 [N',3] host arrays (numpy or pinned torch CPU tensors)."""
        import torch
        if isinstance(m_host, np.ndarray):
            m_host = torch.from_numpy(np.ascontiguousarray(m_host, dtype=np.float32))
        if H_host is None:
            H_host = torch.empty_like(m_host)
        n = self.n_parents_local
        self._check(_lib.pmfem_heff_host(self._h, _host_ptr(m_host, n), _host_ptr(H_host, n), self._stream(stream)))
        return H_host

    def llg_rk4(self, m, steps, dt, alpha, gamma=1.7595e7, H_applied=(0.0, 0.0, 0.0), stream=None):
        """`steps` RK4 steps of the LLG equation on m (float32 CUDA tensor [N'_local, 3], in place)."""
        hap = (ctypes.c_double * 3)(*[float(v) for v in H_applied])
        self._check(_lib.pmfem_llg_rk4(self._h, _dev_ptr(m, self.n_parents_local, self.device), int(steps), float(dt), float(alpha), float(gamma),
                                       ctypes.cast(hap, ctypes.c_void_p), self._stream(stream)))
        return m

    def set_anisotropy(self, kind, K=0.0, axis=(0.0, 0.0, 1.0)):
        """NEXT-2 anisotropy used by the LLG integrators: kind 0 none, 1 uniaxial (axis), 2 cubic."""
        ax = (ctypes.c_double * 3)(*[float(v) for v in axis])
        self._check(_lib.pmfem_set_anisotropy(self._h, int(kind), float(K), ctypes.cast(ax, ctypes.c_void_p)))

    def llg_am2(self, m, t_end, dt0, tol, alpha, gamma=1.7595e7, H_applied=(0.0, 0.0, 0.0), dt_max=0.0,
                stream=None):
        """Adaptive AM2 predictor-corrector LLG integration of m (in place) to t_end; returns
        (accepted, rejected) step counts."""
        hap = (ctypes.c_double * 3)(*[float(v) for v in H_applied])
        acc, rej = ctypes.c_int64(0), ctypes.c_int64(0)
        self._check(_lib.pmfem_llg_am2(self._h, _dev_ptr(m, self.n_parents_local, self.device), float(t_end),
                                       float(dt0), float(tol), float(alpha), float(gamma),
                                       ctypes.cast(hap, ctypes.c_void_p), float(dt_max), self._stream(stream),
                                       ctypes.byref(acc), ctypes.byref(rej)))
        return acc.value, rej.value

    def query(self):
        info = _Info()
        self._check(_lib.pmfem_query(self._h, ctypes.byref(info)))
        out = {k: getattr(info, k) for k, _ in _Info._fields_}
        for k in ("grid", "fft", "kernel_bytes", "k2_tile"):
            out[k] = list(out[k])
        return out

    def get_order(self):
        """rank-local internal row i -> original (user) node index of its parent."""
        a = np.zeros(self.n_parents_local, dtype=np.int64)
        self._check(_lib.pmfem_get_order(self._h, _ptr(a, ctypes.c_int64)))
        return a

    def internal_to_parent_rank(self):
        """rank-local internal row i -> parent rank (parents numbered by increasing original index)."""
        parents = self.export("parent")
        return np.searchsorted(parents, self.get_order())

    def export(self, name):
        cnt = ctypes.c_int64(0)
        self._check(_lib.pmfem_export(self._h, name.encode(), None, ctypes.byref(cnt)))
        dt = _EXPORT_DTYPES.get(name, np.float64)
        a = np.zeros(cnt.value, dtype=dt)
        if cnt.value:
            self._check(_lib.pmfem_export(self._h, name.encode(), a.ctypes.data_as(_vp), ctypes.byref(cnt)))
        return a

    def set_timing(self, enable=True):
        self._check(_lib.pmfem_set_timing(self._h, int(bool(enable))))

    def timing(self):
        a = (ctypes.c_float * 8)()
        self._check(_lib.pmfem_get_timing(self._h, a))
        return dict(zip(KERNELS, list(a)[:5]))


def nccl_unique_id():
    """128-byte NCCL unique id (rank 0 creates it; broadcast it with torch.distributed)."""
    buf = ctypes.create_string_buffer(128)
    st = _lib.pmfem_nccl_unique_id(buf)
    if st != 0:
        raise PmfemError(st, _lib.pmfem_last_error(None).decode())
    return bytes(buf.raw)


def library_symbols():
    """Exported symbols declared in include/pmfem.h (for the ABI test)."""
    return {n: hasattr(_lib, n) for n in SYMBOLS}
