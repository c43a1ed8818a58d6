"""Thin Python binding of libpodp's C ABI (include/podp.h) -- argument marshalling only.

Every step of the on-line path (assembly, LU solve, MPT forms, certificate, selection) runs in the CUDA kernels
of libpodp.so; this module only converts NumPy/PyTorch buffers into the pointers the ABI expects.  There is no
CPU fallback: if libpodp.so is missing or a call fails, an exception is raised.
PyTorch is used for device memory and streams only.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, os.environ.get("PODP_LIB_NAME", "libpodp.so"))  # env: dev A/B builds only

PODP_OK = 0
FLAG_DEFAULT = 0
FLAG_OUT_R = 1 << 0
FLAG_OUT_P = 1 << 1
FLAG_NO_PIVOT = 1 << 2
FLAG_PENCIL = 1 << 3
FLAG_LU_LL = 1 << 8
FLAG_LU_BLK = 1 << 9
FLAG_LU_DYN = 1 << 10
FLAG_LU_GENERIC = 1 << 11
FLAG_MPT_GEMM = 1 << 13
FLAG_MPT_PAIR = 1 << 14
R_MAX = 128
STATUS_NAMES = {0: "PODP_OK", 1: "PODP_ERR_ARG", 2: "PODP_ERR_CUDA", 3: "PODP_ERR_OOM", 4: "PODP_ERR_UNSUPPORTED",
                5: "PODP_ERR_NONFINITE", 6: "PODP_ERR_NOT_HERMITIAN", 7: "PODP_ERR_NO_CANDIDATES"}
EXPORTED = ["podp_create", "podp_create_batch", "podp_create_perdir", "podp_eval", "podp_eval_host", "podp_select", "podp_n_obj", "podp_r",
            "podp_last_launch_count", "podp_destroy", "podp_last_error", "podp_version", "podp_profile_enable",
            "podp_profile_read", "podp_invariants", "podp_coil_voltage", "podp_release_workspace"]


class PodpError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {message}")
        self.status = status
        self.message = message


class podp_operators(ctypes.Structure):
    _fields_ = [("r", ctypes.c_int32), ("nu", ctypes.c_double), ("alpha", ctypes.c_double),
                ("alpha_lb", ctypes.c_double)] + [
        (n, ctypes.POINTER(ctypes.c_double)) for n in ("K", "M", "K_R", "b0", "b1", "N0", "S", "H", "G", "M_I")]


class podp_perdir_operators(ctypes.Structure):
    _DP = ctypes.POINTER(ctypes.c_double)
    _fields_ = [("m", ctypes.c_int32 * 3), ("nu", ctypes.c_double), ("alpha", ctypes.c_double),
                ("alpha_lb", ctypes.c_double), ("K", _DP * 9), ("C", _DP * 9), ("b0", _DP * 3), ("b1", _DP * 3),
                ("H", _DP * 9), ("N0", _DP), ("S", _DP), ("G", _DP * 9)]


_lib = None


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libpodp.so (in-tree).  Raises FileNotFoundError if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path)
    P = ctypes.c_void_p
    i32, i64, dbl = ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    lib.podp_create.argtypes = [ctypes.POINTER(podp_operators), ctypes.c_int, P, ctypes.POINTER(P)]
    lib.podp_create_batch.argtypes = [i32, ctypes.POINTER(podp_operators), ctypes.c_int, P, ctypes.POINTER(P)]
    lib.podp_create_perdir.argtypes = [ctypes.POINTER(podp_perdir_operators), ctypes.c_int, P, ctypes.POINTER(P)]
    lib.podp_eval.argtypes = [P, P, i64, P, P, P, P, P, ctypes.c_int, P]
    lib.podp_eval_host.argtypes = [P, P, i64, P, P, P, P, ctypes.c_int, P]
    lib.podp_select.argtypes = [P, P, P, i64, P, i32, i32, dbl, P, P, P, P, P, P]
    lib.podp_n_obj.argtypes = [P]
    lib.podp_r.argtypes = [P]
    lib.podp_destroy.argtypes = [P]
    for fn in ("podp_create", "podp_create_batch", "podp_create_perdir", "podp_eval", "podp_eval_host", "podp_select", "podp_destroy"):
        getattr(lib, fn).restype = ctypes.c_int
    lib.podp_n_obj.restype = i32
    lib.podp_r.restype = i32
    lib.podp_last_launch_count.restype = i32
    lib.podp_last_error.restype = ctypes.c_char_p
    lib.podp_invariants.argtypes = [P, P, i64, P, P, P]
    lib.podp_invariants.restype = ctypes.c_int
    lib.podp_coil_voltage.argtypes = [P, P, i64, P, P, i32, P, P]
    lib.podp_coil_voltage.restype = ctypes.c_int
    lib.podp_profile_enable.argtypes = [ctypes.c_int]
    lib.podp_profile_enable.restype = ctypes.c_int
    lib.podp_profile_read.argtypes = [P, P, P, i32, i32]
    lib.podp_profile_read.restype = i32
    lib.podp_version.restype = ctypes.c_char_p
    lib.podp_release_workspace.argtypes = [ctypes.c_int]
    lib.podp_release_workspace.restype = ctypes.c_int
    _lib = lib
    return lib


def release_workspace(device: int = 0):
    """Return the library's unused workspace memory on `device` to the driver (podp_release_workspace)."""
    _check(load_library().podp_release_workspace(device))


def profile_enable(on: bool = True):
    """Record CUDA event pairs around each libpodp kernel launch (bench instrumentation)."""
    load_library().podp_profile_enable(1 if on else 0)


def profile_read(reset: bool = True) -> dict:
    """{kernel name: (total ms, launches)} accumulated since the last reset; call when streams are idle."""
    lib = load_library()
    n_max = 16
    names = ctypes.create_string_buffer(32 * n_max)
    ms = np.zeros(n_max)
    cnt = np.zeros(n_max, dtype=np.int64)
    n = lib.podp_profile_read(names, ms.ctypes.data, cnt.ctypes.data, n_max, 1 if reset else 0)
    out = {}
    for i in range(n):
        nm = names.raw[32 * i:32 * (i + 1)].split(b"\0")[0].decode()
        out[nm] = (float(ms[i]), int(cnt[i]))
    return out


def invariants(T1, I, stream=None):
    """NEXT row N4: eigenvalues (ascending) of Rt and I per output row.  T1, I: (..., 6) float64 CUDA
    tensors from Evaluator.eval.  Returns (eigR, eigI) of shape (..., 3)."""
    import torch
    T1c, Ic = T1.contiguous(), I.contiguous()
    n = T1c.numel() // 6
    eR = torch.empty(T1c.shape[:-1] + (3,), dtype=torch.float64, device=T1c.device)
    eI = torch.empty_like(eR)
    _check(load_library().podp_invariants(ctypes.c_void_p(T1c.data_ptr()), ctypes.c_void_p(Ic.data_ptr()), n,
                                          ctypes.c_void_p(eR.data_ptr()), ctypes.c_void_p(eI.data_ptr()),
                                          _stream_handle(stream)))
    return eR, eI


def coil_voltage(T1, I, h_ex, h_ms, stream=None):
    """NEXT row N4: V = h_ms^T (Rt + i I) h_ex for each coil pair (eqn:meas_voltage).
    h_ex, h_ms: (n_coil, 3) real background fields at the object.  Returns complex128 (..., n_coil)."""
    import torch
    h_ex = np.ascontiguousarray(h_ex, dtype=np.float64).reshape(-1, 3)
    h_ms = np.ascontiguousarray(h_ms, dtype=np.float64).reshape(-1, 3)
    if h_ex.shape != h_ms.shape:
        raise ValueError("h_ex and h_ms must have the same shape (n_coil, 3)")
    T1c, Ic = T1.contiguous(), I.contiguous()
    n = T1c.numel() // 6
    V = torch.empty(T1c.shape[:-1] + (h_ex.shape[0],), dtype=torch.complex128, device=T1c.device)
    _check(load_library().podp_coil_voltage(ctypes.c_void_p(T1c.data_ptr()), ctypes.c_void_p(Ic.data_ptr()), n,
                                            ctypes.c_void_p(h_ex.ctypes.data), ctypes.c_void_p(h_ms.ctypes.data),
                                            h_ex.shape[0], ctypes.c_void_p(V.data_ptr()), _stream_handle(stream)))
    return V


def scale_signature(omega, outputs: dict, s: float) -> tuple:
    """Remark 6.2: M[s alpha B, omega] = s^3 M[alpha B, s^2 omega].  Given a signature evaluated on
    the grid `omega` for object alpha B, returns the grid omega / s^2 and the outputs scaled by s^3 for the
    scaled object s alpha B -- a dictionary entry at zero extra solves (NEXT row N4)."""
    f = float(s) ** 3
    return omega / float(s) ** 2, {k: (v * f if k in ("T1", "I", "Delta") else v) for k, v in outputs.items()}


def _check(st: int):
    if st != PODP_OK:
        raise PodpError(st, load_library().podp_last_error().decode())


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _c128(x, shape) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(x, dtype=np.complex128))
    if a.shape != shape:
        raise ValueError(f"expected shape {shape}, got {a.shape}")
    return a


def _f64(x, shape) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    if a.shape != shape:
        raise ValueError(f"expected shape {shape}, got {a.shape}")
    return a


def _marshal(o, keep: list) -> podp_operators:
    """Duck-typed operator object (attributes K, M, K_R?, M_I?, b0, b1, N0, S, H, G, nu, alpha, alpha_lb)."""
    r = int(np.asarray(o.K).shape[0])
    st = podp_operators()
    st.r = r
    st.nu, st.alpha, st.alpha_lb = float(o.nu), float(o.alpha), float(o.alpha_lb)
    arrays = dict(K=_c128(o.K, (r, r)), M=_c128(o.M, (r, r)), b0=_c128(o.b0, (r, 3)), b1=_c128(o.b1, (r, 3)),
                  N0=_f64(o.N0, (3, 3)), S=_f64(o.S, (3, 3)), H=_c128(o.H, (3, r)),
                  G=_c128(o.G, (6 + 2 * r, 6 + 2 * r)))
    for name in ("K_R", "M_I"):
        x = getattr(o, name, None)
        if x is not None:
            arrays[name] = _c128(x, (r, r))
    for k, a in arrays.items():
        keep.append(a)
        setattr(st, k, _dptr(a))
    return st


def _stream_handle(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


class Evaluator:
    """podp_create / podp_create_batch + podp_eval / podp_eval_host / podp_select on one device."""

    @classmethod
    def per_direction(cls, Kb, Cb, b0, b1, Hb, N0, S, Gx, nu: float, alpha: float, alpha_lb: float,
                      device: int = 0, stream=None) -> "Evaluator":
        """NEXT row N1, literal form (podp_create_perdir): Kb[i][j], Cb[i][j] the M_i x M_j blocks K_ij^M and
        C_ij^M / nu; b0[i], b1[i] length M_i; Hb[i][j] the length-M_j rows h_i^(j); Gx[i][j] the direction Grams
        W_i^H W_j ((2 + 2 M_i) x (2 + 2 M_j)).  Argument marshalling only."""
        lib = load_library()
        m = [int(np.asarray(b0[i]).shape[0]) for i in range(3)]
        st = podp_perdir_operators()
        keep: list = []

        def put(a):
            keep.append(a)
            return _dptr(a)
        for i in range(3):
            st.m[i] = m[i]
            st.b0[i] = put(_c128(b0[i], (m[i],)))
            st.b1[i] = put(_c128(b1[i], (m[i],)))
            for j in range(3):
                st.K[3 * i + j] = put(_c128(Kb[i][j], (m[i], m[j])))
                st.C[3 * i + j] = put(_c128(Cb[i][j], (m[i], m[j])))
                st.H[3 * i + j] = put(_c128(Hb[i][j], (m[j],)))
                st.G[3 * i + j] = put(_c128(Gx[i][j], (2 + 2 * m[i], 2 + 2 * m[j])))
        st.N0 = put(_f64(N0, (3, 3)))
        st.S = put(_f64(S, (3, 3)))
        st.nu, st.alpha, st.alpha_lb = float(nu), float(alpha), float(alpha_lb)
        h = ctypes.c_void_p()
        import torch
        with torch.cuda.device(device):
            _check(lib.podp_create_perdir(ctypes.byref(st), device, _stream_handle(stream), ctypes.byref(h)))
        self = cls.__new__(cls)
        self._h = h
        self.device = device
        self.n_obj = int(lib.podp_n_obj(h))
        self.r = int(lib.podp_r(h))
        self.m = m
        return self

    def __init__(self, ops, device: int = 0, stream=None):
        lib = load_library()
        ops_list = list(ops) if isinstance(ops, (list, tuple)) else [ops]
        keep: list = []
        arr = (podp_operators * len(ops_list))(*[_marshal(o, keep) for o in ops_list])
        h = ctypes.c_void_p()
        import torch
        with torch.cuda.device(device):
            _check(lib.podp_create_batch(len(ops_list), arr, device, _stream_handle(stream), ctypes.byref(h)))
        self._h = h
        self.device = device
        self.n_obj = int(lib.podp_n_obj(h))
        self.r = int(lib.podp_r(h))

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            load_library().podp_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def alloc_outputs(self, F: int, info: bool = True, want_P: bool = False):
        import torch
        dev = torch.device("cuda", self.device)
        n = self.n_obj
        out = dict(T1=torch.empty((n, F, 6), dtype=torch.float64, device=dev),
                   I=torch.empty((n, F, 6), dtype=torch.float64, device=dev),
                   Delta=torch.empty((n, F, 6), dtype=torch.float64, device=dev))
        if info:
            out["info"] = torch.empty((n, F), dtype=torch.int32, device=dev)
        if want_P:
            out["P"] = torch.empty((n, F, 3, self.r), dtype=torch.complex128, device=dev)
        return out

    def eval(self, omega, out: dict | None = None, flags: int = 0, info: bool = True, want_P: bool = False,
             stream=None) -> dict:
        """omega: 1-D float64 CUDA tensor (device-resident).  Asynchronous on `stream`."""
        import torch
        if not (isinstance(omega, torch.Tensor) and omega.is_cuda and omega.dtype == torch.float64 and omega.dim() == 1):
            raise TypeError("omega must be a 1-D float64 CUDA tensor")
        omega = omega.contiguous()
        F = omega.shape[0]
        if out is None:
            out = self.alloc_outputs(F, info=info, want_P=want_P)
        if want_P:
            flags |= FLAG_OUT_P
        lib = load_library()
        p = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p()  # noqa: E731
        _check(lib.podp_eval(self._h, p(omega), F, p(out["T1"]), p(out["I"]), p(out["Delta"]), p(out.get("info")),
                             p(out.get("P")), flags, _stream_handle(stream)))
        return out

    def launches_last_call(self) -> int:
        return int(load_library().podp_last_launch_count())

    def eval_host(self, omega_h: np.ndarray, flags: int = 0, out: dict | None = None, stream=None) -> dict:
        """End-to-end entry: host omega in, host outputs back (podp_eval_host; synchronises)."""
        omega_h = np.ascontiguousarray(omega_h, dtype=np.float64)
        F = omega_h.shape[0]
        n = self.n_obj
        if out is None:
            out = dict(T1=np.empty((n, F, 6)), I=np.empty((n, F, 6)), Delta=np.empty((n, F, 6)),
                       info=np.empty((n, F), dtype=np.int32))
        lib = load_library()
        vp = lambda a: ctypes.c_void_p(a.ctypes.data) if a is not None else ctypes.c_void_p()  # noqa: E731
        _check(lib.podp_eval_host(self._h, vp(omega_h), F, vp(out["T1"]), vp(out["I"]), vp(out["Delta"]),
                                  vp(out.get("info")), flags, _stream_handle(stream)))
        return out

    def select(self, omega, Delta, snap, n_star: int = 2, theta: float = 0.0, stream=None):
        """One Algorithm-1 selection step on device-resident omega (F) and Delta (F x 6) of one object."""
        import torch
        F = omega.shape[0]
        if Delta.shape[-2:] != (F, 6) or not Delta.is_contiguous():
            raise ValueError("Delta must be a contiguous F x 6 tensor")
        snap = np.ascontiguousarray(snap, dtype=np.float64)
        n_int = len(snap) - 1
        n_new = ctypes.c_int32()
        om_new = np.empty(n_star)
        idx_new = np.empty(n_star, dtype=np.int64)
        lam = ctypes.c_double()
        lam_n = np.empty(max(n_int, 1))
        lib = load_library()
        _check(lib.podp_select(self._h, ctypes.c_void_p(omega.data_ptr()), ctypes.c_void_p(Delta.data_ptr()), F,
                               ctypes.c_void_p(snap.ctypes.data), len(snap), n_star, float(theta),
                               ctypes.byref(n_new), ctypes.c_void_p(om_new.ctypes.data),
                               ctypes.c_void_p(idx_new.ctypes.data), ctypes.byref(lam),
                               ctypes.c_void_p(lam_n.ctypes.data), _stream_handle(stream)))
        k = n_new.value
        return om_new[:k].copy(), idx_new[:k].copy(), lam.value, lam_n[:n_int].copy()
