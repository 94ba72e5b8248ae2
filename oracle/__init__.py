"""fp64 CPU oracle for InfraredGP's FFP (arXiv 2508.19737) — TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2508_19737_b200``) never imports it and shares no code with it.

This module is a thin ctypes marshalling layer over ``oracle/igp_oracle.c``
(plain C, double precision); every step of the method lives in that file, each
function citing the PAPER.md passage it follows.  ``liboracle.so`` is compiled
with gcc on first use if it is missing (``build()`` in ``__graft_entry__`` also
compiles it).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "igp_oracle.c")
_SRCS = [_SRC, os.path.join(_HERE, "birch_oracle.c")]
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

MODE_FULL = 0
MODE_PRE_SIGMOID = 1
MODE_LINEAR = 2

THETA = 0.1  # (alpha, theta) = (1, 0.1)
ALPHA = 1.0
EPS = 1e-3  # "epsilon = 0.001 in our experiment"

_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so (gcc, -O2, OpenMP, no fast-math)."""
    if force or not os.path.exists(_LIB_PATH) or any(os.path.getmtime(_LIB_PATH) < os.path.getmtime(s)
                                                      for s in _SRCS):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        # -ffp-contract=off: no implicit fma; birch_oracle.c uses explicit fma() where it means one
        subprocess.check_call(
            ["gcc", "-O2", "-fPIC", "-shared", "-fopenmp", "-fno-fast-math", "-ffp-contract=off", "-std=c11",
             "-Wall", "-o", tmp, *_SRCS, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is not None:
        return _lib
    build()
    lib = ctypes.CDLL(_LIB_PATH)
    P = ctypes.c_void_p
    i32, i64, u64, f64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double
    lib.oracle_build_csr.argtypes = [P, i64, i32, P, P, P]
    lib.oracle_build_csr.restype = i64
    lib.oracle_corrected_degree.argtypes = [i32, f64, f64]
    lib.oracle_corrected_degree.restype = f64
    lib.oracle_philox4x32_10.argtypes = [P, P, P]
    lib.oracle_philox4x32_10.restype = None
    lib.oracle_philox_bits.argtypes = [u64, u64, i64, P]
    lib.oracle_philox_bits.restype = None
    lib.oracle_box_muller.argtypes = [ctypes.c_uint32, ctypes.c_uint32, P]
    lib.oracle_box_muller.restype = None
    lib.oracle_normal.argtypes = [u64, u64, i64, P]
    lib.oracle_normal.restype = None
    lib.oracle_normal_at.argtypes = [u64, u64, P, i64, P]
    lib.oracle_normal_at.restype = None
    lib.oracle_propagate.argtypes = [P, P, i32, i32, P, P, f64, f64, i32, P]
    lib.oracle_propagate.restype = None
    lib.oracle_zscore_columns.argtypes = [P, i32, i32]
    lib.oracle_zscore_columns.restype = None
    lib.oracle_row_l2.argtypes = [P, i32, i32]
    lib.oracle_row_l2.restype = None
    lib.oracle_embed.argtypes = [P, P, i32, i32, i32, f64, f64, f64, f64, P, u64, u64, i32, i32, P]
    lib.oracle_embed.restype = ctypes.c_int
    lib.oracle_embed_ddof.argtypes = [P, P, i32, i32, i32, f64, f64, f64, f64, P, u64, u64, i32, i32, i32, P]
    lib.oracle_embed_ddof.restype = ctypes.c_int
    lib.oracle_zscore_columns_ddof.argtypes = [P, i32, i32, i32]
    lib.oracle_zscore_columns_ddof.restype = None
    lib.oracle_embed_f32.argtypes = [P, P, i32, i32, i32, f64, f64, f64, f64, P, u64, u64, i32, i32, P]
    lib.oracle_embed_f32.restype = ctypes.c_int
    lib.oracle_birch_new.argtypes = [i32, f64, i32]
    lib.oracle_birch_new.restype = P
    lib.oracle_birch_free.argtypes = [P]
    lib.oracle_birch_free.restype = None
    lib.oracle_birch_partial_fit.argtypes = [P, P, i64]
    lib.oracle_birch_partial_fit.restype = ctypes.c_int
    lib.oracle_birch_num_clusters.argtypes = [P]
    lib.oracle_birch_num_clusters.restype = i64
    lib.oracle_birch_clusters.argtypes = [P, P, P, P, P, P]
    lib.oracle_birch_clusters.restype = None
    lib.oracle_birch_shape.argtypes = [P, P, P, P]
    lib.oracle_birch_shape.restype = None
    lib.oracle_birch_predict.argtypes = [P, P, i64, i32, P, i64, P]
    lib.oracle_birch_predict.restype = ctypes.c_int
    _lib = lib
    return lib


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data) if a.size else ctypes.c_void_p(0)


class OracleError(ValueError):
    pass


def build_csr(edges, num_nodes: int):
    """Canonical CSR of the undirected simple graph on ``num_nodes`` nodes.

    ``edges``: int array [E, 2] (duplicates / either orientation / self loops allowed).
    Returns (row_ptr int32[N+1], col_idx int32[2M], M)."""
    lib = _load()
    e = np.ascontiguousarray(np.asarray(edges, dtype=np.int32).reshape(-1, 2))
    E = e.shape[0]
    rp = np.zeros(max(num_nodes, 0) + 1, dtype=np.int32)
    ci = np.zeros(max(2 * E, 1), dtype=np.int32)
    m = ctypes.c_int64(0)
    nnz = lib.oracle_build_csr(_ptr(e), E, int(num_nodes), _ptr(rp), _ptr(ci), ctypes.byref(m))
    if nnz == -2:
        raise OracleError("num_nodes must be positive")
    if nnz == -1:
        raise OracleError("edge index out of range")
    return rp, ci[:nnz].copy(), int(m.value)


def corrected_degree(deg, tau: float, eps: float = EPS) -> np.ndarray:
    """Eq. (1) (tau < 0) / D + tau I (tau >= 0), element-wise, fp64."""
    lib = _load()
    deg = np.asarray(deg, dtype=np.int64).ravel()
    return np.array([lib.oracle_corrected_degree(int(x), float(tau), float(eps)) for x in deg])


def philox4x32_10(ctr, key) -> np.ndarray:
    lib = _load()
    c = np.ascontiguousarray(np.asarray(ctr, dtype=np.uint32))
    k = np.ascontiguousarray(np.asarray(key, dtype=np.uint32))
    out = np.zeros(4, dtype=np.uint32)
    lib.oracle_philox4x32_10(_ptr(c), _ptr(k), _ptr(out))
    return out


def philox_bits(seed: int, sub: int, count: int) -> np.ndarray:
    lib = _load()
    out = np.zeros(count, dtype=np.uint32)
    lib.oracle_philox_bits(seed, sub, count, _ptr(out))
    return out


def box_muller(r_even: int, r_odd: int) -> np.ndarray:
    """The Box-Muller transform of one raw pair (n_even, n_odd), fp64."""
    lib = _load()
    out = np.zeros(2, dtype=np.float64)
    lib.oracle_box_muller(int(r_even), int(r_odd), _ptr(out))
    return out


def normal(seed: int, sub: int, count: int) -> np.ndarray:
    """X ~ N(0,1), fp64, draw k of the (seed, sub) stream (count % 4 == 0)."""
    lib = _load()
    out = np.zeros(count, dtype=np.float64)
    lib.oracle_normal(seed, sub, count, _ptr(out))
    return out


def normal_at(seed: int, sub: int, index) -> np.ndarray:
    """Elements ``index`` (flat, any order) of the ``normal(seed, sub, .)`` stream, fp64."""
    lib = _load()
    idx = np.ascontiguousarray(np.asarray(index, dtype=np.int64).ravel())
    if idx.size and idx.min() < 0:
        raise OracleError("negative stream index")
    out = np.zeros(idx.size, dtype=np.float64)
    lib.oracle_normal_at(seed, sub, _ptr(idx), idx.size, _ptr(out))
    return out


def propagate(row_ptr, col_idx, Dtau, Z, theta=THETA, alpha=ALPHA, nthreads=1) -> np.ndarray:
    """One application of Eq. (3): theta Z + alpha D^{-1/2} A D^{-1/2} Z (fp64)."""
    lib = _load()
    rp = np.ascontiguousarray(row_ptr, dtype=np.int32)
    ci = np.ascontiguousarray(col_idx, dtype=np.int32)
    Dt = np.ascontiguousarray(Dtau, dtype=np.float64)
    Z = np.ascontiguousarray(Z, dtype=np.float64)
    if Z.ndim == 1:
        Z = Z[:, None]
    N, d = Z.shape
    P = np.zeros((N, d), dtype=np.float64)
    lib.oracle_propagate(_ptr(rp), _ptr(ci), N, d, _ptr(Dt), _ptr(Z), theta, alpha, nthreads, _ptr(P))
    return P


def zscore_columns(T, ddof: int = 0) -> np.ndarray:
    """Column z-score (ZNorm), std over N - ddof (reading A2: ddof = 0)."""
    lib = _load()
    T = np.array(T, dtype=np.float64, order="C", copy=True)
    if T.ndim == 1:
        T = T[:, None]
    lib.oracle_zscore_columns_ddof(_ptr(T), T.shape[0], T.shape[1], int(ddof))
    return T


def row_l2(Z) -> np.ndarray:
    """Optional post-op (not in the paper, reading A12): rows scaled to unit L2 norm."""
    lib = _load()
    Z = np.array(Z, dtype=np.float64, order="C", copy=True)
    if Z.ndim == 1:
        Z = Z[None, :]
    lib.oracle_row_l2(_ptr(Z), Z.shape[0], Z.shape[1])
    return Z


def embed(row_ptr, col_idx, num_nodes: int, d: int, steps: int, tau: float, seed: int = 0,
          sub: int = 0, theta=THETA, alpha=ALPHA, eps=EPS, Z0=None, mode=MODE_FULL,
          nthreads: int = 1, fp32_twin: bool = False, ddof: int = 0) -> np.ndarray:
    """Alg. 1 lines 1-6 in fp64; returns Z~ (or Z^(L) / linear output per ``mode``).

    ``fp32_twin=True`` runs ``oracle_embed_f32`` instead: the same steps with float storage
    and arithmetic (fp64 column statistics), used only to report the fp32 drift floor."""
    lib = _load()
    rp = np.ascontiguousarray(row_ptr, dtype=np.int32)
    ci = np.ascontiguousarray(col_idx, dtype=np.int32)
    out = np.zeros((num_nodes, d), dtype=np.float64)
    z0p = ctypes.c_void_p(0)
    if Z0 is not None:
        Z0 = np.ascontiguousarray(Z0, dtype=np.float64).reshape(num_nodes, d)
        z0p = _ptr(Z0)
    if fp32_twin:
        if ddof:
            raise OracleError("the fp32 twin uses the population std (ddof = 0)")
        rc = lib.oracle_embed_f32(_ptr(rp), _ptr(ci), num_nodes, d, steps, tau, theta, alpha, eps, z0p, seed, sub,
                                  mode, nthreads, _ptr(out))
    else:
        rc = lib.oracle_embed_ddof(_ptr(rp), _ptr(ci), num_nodes, d, steps, tau, theta, alpha, eps, z0p, seed, sub,
                                   mode, nthreads, int(ddof), _ptr(out))
    if rc != 0:
        raise OracleError(f"oracle_embed rejected its arguments (rc={rc})")
    return out


def input_theta(seed: int, sub: int, num_nodes: int, d: int) -> np.ndarray:
    """Theta = X / sqrt(d), X the Philox/Box-Muller stream (Alg. 1 l.2, reading A1)."""
    return normal(seed, sub, num_nodes * d).reshape(num_nodes, d) / np.sqrt(d)


# ---------------------------------------------------------------- BIRCH (Alg. 1 l.7, Alg. 2 l.9-11)
class Birch:
    """The oracle's CF tree (oracle/birch_oracle.c): ``partial_fit`` inserts rows in order,
    ``clusters()`` returns the leaf entries (the K-agnostic clusters) in leaf-chain order,
    ``predict`` labels rows by their nearest cluster centroid.  fp64 throughout."""

    def __init__(self, d: int, threshold: float = 0.5, branching: int = 50):
        self._lib = _load()
        self.d = d
        self._h = self._lib.oracle_birch_new(d, float(threshold), int(branching))
        if not self._h:
            raise OracleError("oracle_birch_new rejected its arguments")

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            self._lib.oracle_birch_free(h)
            self._h = None

    def partial_fit(self, X):
        X = np.ascontiguousarray(X, dtype=np.float64).reshape(-1, self.d)
        rc = self._lib.oracle_birch_partial_fit(self._h, _ptr(X), X.shape[0])
        if rc != 0:
            raise OracleError(f"oracle_birch_partial_fit failed (rc={rc})")
        return self

    fit = partial_fit  # a fresh tree: fit == partial_fit on all rows in order

    def clusters(self):
        """(centroids [K,d], sqn [K], n [K], LS [K,d], SS [K])"""
        K = int(self._lib.oracle_birch_num_clusters(self._h))
        cen = np.zeros((K, self.d))
        ls = np.zeros((K, self.d))
        sqn, n, ss = np.zeros(K), np.zeros(K), np.zeros(K)
        self._lib.oracle_birch_clusters(self._h, _ptr(cen), _ptr(sqn), _ptr(n), _ptr(ls), _ptr(ss))
        return cen, sqn, n, ls, ss

    def shape(self):
        dep, nodes, pts = ctypes.c_int32(0), ctypes.c_int32(0), ctypes.c_int64(0)
        self._lib.oracle_birch_shape(self._h, ctypes.byref(dep), ctypes.byref(nodes), ctypes.byref(pts))
        return dep.value, nodes.value, pts.value

    def predict(self, X):
        cen, sqn, _, _, _ = self.clusters()
        return birch_predict(cen, sqn, X)


def birch_predict(cen, sqn, X) -> np.ndarray:
    """label_i = argmin_j sqn_j - 2 c_j . x_i (first minimum), fp64."""
    lib = _load()
    cen = np.ascontiguousarray(cen, dtype=np.float64)
    sqn = np.ascontiguousarray(sqn, dtype=np.float64)
    K, d = cen.shape
    X = np.ascontiguousarray(X, dtype=np.float64).reshape(-1, d)
    out = np.zeros(X.shape[0], dtype=np.int32)
    rc = lib.oracle_birch_predict(_ptr(cen), _ptr(sqn), K, d, _ptr(X), X.shape[0], _ptr(out))
    if rc != 0:
        raise OracleError(f"oracle_birch_predict rejected its arguments (rc={rc})")
    return out
