"""ctypes binding of the in-tree CUDA library ``libddmgnn_b200.so`` (C ABI in
include/ddmgnn_b200.h).

There is no fallback: if the shared library is missing or no sm_100 device is
present, every compute entry point raises.  Build the library with
``python -c "import __graft_entry__ as g; g.build()"`` (or ``make -C
paper_2402_08296_b200/csrc``).
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# DDMGNN_B200_LIB selects an alternative in-tree build (kernel experiments)
LIB_PATH = os.environ.get("DDMGNN_B200_LIB") or os.path.join(_HERE, "libddmgnn_b200.so")

PRECOND_NONE = 0
LEVEL_ONE = 1
LEVEL_TWO = 2
ASM_ONE = 3
ASM_TWO = 4
IC0 = 5
FLEXIBLE = 0x100  # OR into the pcg level: opt-in flexible CG (Polak-Ribiere beta)
LEGACY_STREAM = 1  # cudaStreamLegacy

_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_int = ctypes.c_int
_dbl = ctypes.c_double
_vp = ctypes.c_void_p
_ctx = ctypes.c_void_p
_pd = ctypes.POINTER(ctypes.c_double)
_pi64 = ctypes.POINTER(ctypes.c_int64)
_pi32 = ctypes.POINTER(ctypes.c_int32)
_pf = ctypes.POINTER(ctypes.c_float)
_pint = ctypes.POINTER(ctypes.c_int)
_pvp = ctypes.POINTER(ctypes.c_void_p)

HOST_PRECOND_FN = ctypes.CFUNCTYPE(_int, _vp, _pd, _pd, _i64)

# (name, restype, argtypes) for every symbol declared in include/ddmgnn_b200.h
SIGNATURES = [
    ("ddmgnn_last_error", ctypes.c_char_p, []),
    ("ddmgnn_version", _int, []),
    ("ddmgnn_create", _int, [_int, ctypes.POINTER(_ctx)]),
    ("ddmgnn_destroy", None, [_ctx]),
    ("ddmgnn_stream", _vp, [_ctx]),
    ("ddmgnn_set_matrix", _int, [_ctx, _i64, _i64, _pi64, _pi32, _pd]),
    ("ddmgnn_set_geometry", _int, [_ctx, _i64, _pd]),
    ("ddmgnn_set_decomposition", _int, [_ctx, _i64, _pi64, _pi64]),
    ("ddmgnn_set_model", _int, [_ctx, _int, _int, _dbl, _pd, _i64]),
    ("ddmgnn_set_coarse_inverse", _int, [_ctx, _i64, _pd]),
    ("ddmgnn_set_batch_cap", _int, [_ctx, _i64]),
    ("ddmgnn_alloc_local_inverses", _int, [_ctx, _pi64, ctypes.POINTER(_vp)]),
    ("ddmgnn_set_ic0", _int, [_ctx]),
    ("ddmgnn_export_ic0", _int, [_ctx, _pi64, _pi32, _pi32, _pd]),
    ("ddmgnn_build", _int, [_ctx]),
    ("ddmgnn_info", _int, [_ctx, _pi64, _int]),
    ("ddmgnn_export_local_graph", _int, [_ctx, _i64, _pi64, _pi32, _pi32, _pf]),
    ("ddmgnn_apply", _int, [_ctx, _vp, _vp, _int, _vp, _int]),
    ("ddmgnn_apply_host", _int, [_ctx, _pd, _pd, _int]),
    ("ddmgnn_launch_gnn_only", _int, [_ctx, _vp, _vp]),
    ("ddmgnn_apply_status", _int, [_ctx, _vp]),
    ("ddmgnn_spmv", _int, [_ctx, _vp, _vp, _vp]),
    ("ddmgnn_pcg", _int, [_ctx, _vp, _vp, _vp, _dbl, _int, _int, _int, _vp, _pint, _pd, _pint]),
    ("ddmgnn_pcg_host_precond", _int,
     [_ctx, _pd, _pd, _pd, _dbl, _int, _int, HOST_PRECOND_FN, _vp, _pint, _pd, _pint]),
    ("ddmgnn_local_outputs", _int, [_ctx, ctypes.POINTER(_vp), ctypes.POINTER(_vp),
                                    ctypes.POINTER(_vp)]),
    ("ddmgnn_set_pou", _int, [_ctx, _i64, _pd]),
    ("ddmgnn_gather", _int, [_vp, _vp, _i64, _vp, _vp]),
    ("ddmgnn_scatter", _int, [_vp, _vp, _i64, _vp, _vp]),
    ("ddmgnn_dot", _int, [_i64, _vp, _vp, _vp, _vp, _vp]),
    ("ddmgnn_dot_diff", _int, [_i64, _vp, _vp, _vp, _vp, _vp, _vp]),
    ("ddmgnn_axpy2", _int, [_i64, _dbl, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    ("ddmgnn_xpby", _int, [_i64, _vp, _dbl, _vp, _vp]),
    ("ddmgnn_dense_gemv", _int, [_i64, _vp, _vp, _vp, _vp]),
    ("ddmgnn_pcg_scalars", _int, [_int, _vp, _vp, _vp]),
    ("ddmgnn_axpy2_dev", _int, [_i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    ("ddmgnn_xpby_dev", _int, [_i64, _vp, _vp, _vp, _vp]),
    ("ddmgnn_prolong", _int, [_i64, _int, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    ("ddmgnn_peer_put", _int, [_int, _int, _int, _pvp, _vp, _vp, _pi64, _pvp, _pi64, _vp]),
    ("ddmgnn_peer_wait", _int, [_int, _int, _int, _pvp, _pi64, _vp, _vp, _vp, _int, _vp]),
    ("ddmgnn_peer_ack", _int, [_int, _int, _int, _pvp, _pi64, _vp]),
    ("ddmgnn_peer_allgather", _int, [_int, _int, _int, _pvp, _pvp, _vp, _i64, _vp]),
    ("ddmgnn_peer_allreduce", _int, [_int, _int, _int, _pvp, _pvp, _vp, _int, _vp]),
    ("ddmgnn_peer_alloc", _int, [_int, _i64, ctypes.POINTER(_vp)]),
    ("ddmgnn_peer_free", _int, [_vp]),
    ("ddmgnn_ipc_get", _int, [_vp, ctypes.c_char_p]),
    ("ddmgnn_ipc_open", _int, [_int, ctypes.c_char_p, ctypes.POINTER(_vp)]),
    ("ddmgnn_ipc_close", _int, [_vp]),
]

_lib = None


def load() -> ctypes.CDLL:
    """Load the CUDA library (raises ImportError if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} not found: build the CUDA extension first "
                "(python -c 'import __graft_entry__ as g; g.build()')")
        lib = ctypes.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(status: int) -> None:
    if status == 0:
        return
    msg = load().ddmgnn_last_error().decode("utf-8", "replace")
    if status == 1:
        raise ValueError(msg)
    raise RuntimeError(msg)


def dptr(a: np.ndarray):
    return a.ctypes.data_as(_pd)


def i64ptr(a: np.ndarray):
    return a.ctypes.data_as(_pi64)


def i32ptr(a: np.ndarray):
    return a.ctypes.data_as(_pi32)


class Context:
    """Owns one ``ddmgnn_ctx`` (device-resident matrix, layout, weights, buffers)."""

    def __init__(self, device: int = 0):
        lib = load()
        h = _ctx()
        check(lib.ddmgnn_create(int(device), ctypes.byref(h)))
        self._h = h
        self.device = int(device)
        self._lib = lib

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            self._lib.ddmgnn_destroy(self._h)
            self._h = _ctx()

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter shutdown
            pass

    @property
    def stream(self) -> int:
        return int(self._lib.ddmgnn_stream(self._h) or 0)

    def set_matrix(self, a):
        indptr = np.ascontiguousarray(a.indptr, dtype=np.int64)
        indices = np.ascontiguousarray(a.indices, dtype=np.int32)
        data = np.ascontiguousarray(a.data, dtype=np.float64)
        check(self._lib.ddmgnn_set_matrix(self._h, a.shape[0], int(indptr[-1]), i64ptr(indptr),
                                          i32ptr(indices), dptr(data)))

    def set_geometry(self, coords):
        c = np.ascontiguousarray(coords, dtype=np.float64)
        check(self._lib.ddmgnn_set_geometry(self._h, c.shape[0], dptr(c)))

    def set_decomposition(self, subdomains):
        sizes = np.array([s.size for s in subdomains], dtype=np.int64)
        sub_ptr = np.concatenate(([0], np.cumsum(sizes))).astype(np.int64)
        sub_idx = np.ascontiguousarray(np.concatenate(subdomains), dtype=np.int64)
        check(self._lib.ddmgnn_set_decomposition(self._h, len(subdomains), i64ptr(sub_ptr),
                                                 i64ptr(sub_idx)))

    def set_model(self, k_bar, d, alpha, flat):
        f = np.ascontiguousarray(flat, dtype=np.float64)
        check(self._lib.ddmgnn_set_model(self._h, int(k_bar), int(d), float(alpha), dptr(f),
                                         f.size))

    def set_coarse_inverse(self, inv):
        m = np.ascontiguousarray(inv, dtype=np.float64)
        check(self._lib.ddmgnn_set_coarse_inverse(self._h, m.shape[0], dptr(m)))

    def alloc_local_inverses(self, off: np.ndarray) -> int:
        o = np.ascontiguousarray(off, dtype=np.int64)
        ptr = _vp()
        check(self._lib.ddmgnn_alloc_local_inverses(self._h, i64ptr(o), ctypes.byref(ptr)))
        return ptr.value

    def set_ic0(self):
        check(self._lib.ddmgnn_set_ic0(self._h))

    def export_ic0(self):
        nnz = ctypes.c_int64(0)
        check(self._lib.ddmgnn_export_ic0(self._h, ctypes.byref(nnz), None, None, None))
        n = self.info()["n"]
        ip = np.zeros(n + 1, dtype=np.int32)
        ix = np.zeros(max(1, nnz.value), dtype=np.int32)
        dv = np.zeros(max(1, nnz.value), dtype=np.float64)
        check(self._lib.ddmgnn_export_ic0(self._h, ctypes.byref(nnz), i32ptr(ip), i32ptr(ix),
                                          dptr(dv)))
        return ip, ix[: nnz.value], dv[: nnz.value]

    def set_batch_cap(self, cap):
        check(self._lib.ddmgnn_set_batch_cap(self._h, int(cap)))

    def build(self):
        check(self._lib.ddmgnn_build(self._h))

    def gnn_launches(self) -> int:
        """Kernel launches of one GNN forward: per constant-bank chunk the CTA
        kernel, one launch per cluster size in use, and for flat-path subdomains
        a restriction prologue (first chunk) plus two launches per layer."""
        i = self.info()
        n, nl_max = 0, i["lmax"]
        for ch in range(i["n_chunks"]):
            nl = min(nl_max, i["k_bar"] - ch * nl_max)
            n += (i["K"] > i["n_big"]) + i["cluster_launches"]
            if i["n_big"] > i["n_cluster"]:
                n += 2 * nl + (1 if ch == 0 else 0)
        return n

    def info(self) -> dict:
        out = np.zeros(14, dtype=np.int64)
        check(self._lib.ddmgnn_info(self._h, i64ptr(out), 14))
        keys = ("n", "K", "V", "E", "E_pad", "k_max", "slices", "k_bar", "d", "lmax",
                "n_chunks", "n_big", "n_cluster", "cluster_launches")
        return dict(zip(keys, (int(x) for x in out)))

    def export_local_graph(self, sub: int):
        ne = ctypes.c_int64(0)
        check(self._lib.ddmgnn_export_local_graph(self._h, int(sub), ctypes.byref(ne), None,
                                                  None, None))
        n = ne.value
        src = np.zeros(max(n, 1), dtype=np.int32)
        dst = np.zeros(max(n, 1), dtype=np.int32)
        vec = np.zeros((max(n, 1), 3), dtype=np.float32)
        check(self._lib.ddmgnn_export_local_graph(self._h, int(sub), ctypes.byref(ne),
                                                  i32ptr(src), i32ptr(dst),
                                                  vec.ctypes.data_as(_pf)))
        return src[:n], dst[:n], vec[:n]

    def apply_host(self, r: np.ndarray, level: int, out: np.ndarray | None = None) -> np.ndarray:
        r = np.ascontiguousarray(r, dtype=np.float64)
        z = np.empty_like(r) if out is None else out
        check(self._lib.ddmgnn_apply_host(self._h, dptr(r), dptr(z), int(level)))
        return z

    def apply_device(self, r_ptr: int, z_ptr: int, level: int, stream: int = 0,
                     sync_check: bool = True):
        check(self._lib.ddmgnn_apply(self._h, _vp(r_ptr), _vp(z_ptr), int(level),
                                     _vp(stream or None), int(bool(sync_check))))

    def launch_gnn_only(self, r_ptr: int, stream: int = 0):
        check(self._lib.ddmgnn_launch_gnn_only(self._h, _vp(r_ptr), _vp(stream or None)))

    def apply_status(self, stream: int = 0):
        """Raise the reference's error if a launch since the last check saw a
        non-finite model state (synchronises the stream)."""
        check(self._lib.ddmgnn_apply_status(self._h, _vp(stream or None)))

    def set_pou(self, pou):
        w = np.ascontiguousarray(pou, dtype=np.float64)
        check(self._lib.ddmgnn_set_pou(self._h, w.size, dptr(w)))

    def local_outputs(self):
        """Device pointers (zloc, scale, r0r) written by launch_gnn_only."""
        z, s, r = _vp(), _vp(), _vp()
        check(self._lib.ddmgnn_local_outputs(self._h, ctypes.byref(z), ctypes.byref(s),
                                             ctypes.byref(r)))
        return z.value, s.value, r.value

    def spmv_device(self, x_ptr: int, y_ptr: int, stream: int = 0):
        check(self._lib.ddmgnn_spmv(self._h, _vp(x_ptr), _vp(y_ptr), _vp(stream or None)))

    def pcg(self, b, u0, tol, max_iter, level, device_ptrs=False, u_out=None, stream=0,
            flexible=False):
        """Returns (u, iterations, history, converged)."""
        it = ctypes.c_int(0)
        conv = ctypes.c_int(0)
        hist = np.zeros(max(0, max_iter) + 1, dtype=np.float64)
        if flexible:
            level = int(level) | FLEXIBLE
        if device_ptrs:
            status = self._lib.ddmgnn_pcg(self._h, _vp(b), _vp(u0 or None), _vp(u_out), float(tol),
                                          int(max_iter), int(level), 1, _vp(stream or None),
                                          ctypes.byref(it), dptr(hist), ctypes.byref(conv))
            check(status)
            return u_out, it.value, hist[: it.value + 1].tolist(), bool(conv.value)
        b = np.ascontiguousarray(b, dtype=np.float64)
        u = np.empty_like(b)
        u0a = None if u0 is None else np.ascontiguousarray(u0, dtype=np.float64)
        status = self._lib.ddmgnn_pcg(self._h, _vp(b.ctypes.data),
                                      _vp(None if u0a is None else u0a.ctypes.data),
                                      _vp(u.ctypes.data), float(tol), int(max_iter), int(level), 0,
                                      _vp(stream or None), ctypes.byref(it), dptr(hist),
                                      ctypes.byref(conv))
        check(status)
        return u, it.value, hist[: it.value + 1].tolist(), bool(conv.value)

    def pcg_host_precond(self, b, u0, tol, max_iter, fn, flexible=False):
        b = np.ascontiguousarray(b, dtype=np.float64)
        n = b.shape[0]
        u = np.empty_like(b)
        u0a = None if u0 is None else np.ascontiguousarray(u0, dtype=np.float64)
        err = []

        def cb(_user, r_p, z_p, nn):
            try:
                r = np.ctypeslib.as_array(r_p, shape=(nn,)).copy()
                z = np.asarray(fn(r), dtype=np.float64)
                if z.shape != (nn,):
                    raise ValueError(f"preconditioner returned shape {z.shape}, expected ({nn},)")
                np.ctypeslib.as_array(z_p, shape=(nn,))[:] = z
                return 0
            except BaseException as exc:  # re-raised after the C call returns
                err.append(exc)
                return 1

        cfn = HOST_PRECOND_FN(cb)
        it = ctypes.c_int(0)
        conv = ctypes.c_int(0)
        hist = np.zeros(max(0, max_iter) + 1, dtype=np.float64)
        status = self._lib.ddmgnn_pcg_host_precond(
            self._h, dptr(b), None if u0a is None else dptr(u0a), dptr(u), float(tol),
            int(max_iter), int(bool(flexible)), cfn, None, ctypes.byref(it), dptr(hist),
            ctypes.byref(conv))
        if err:
            raise err[0]
        check(status)
        assert u.shape == (n,)
        return u, it.value, hist[: it.value + 1].tolist(), bool(conv.value)
