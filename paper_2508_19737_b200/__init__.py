"""B200-native InfraredGP feed-forward propagation (arXiv 2508.19737), Python binding.

A thin ctypes layer over ``libigp.so`` (the C ABI in ``include/igp.h``): argument
marshalling only — every step of the method runs in the library's sm_100a
kernels.  PyTorch supplies device memory and streams.  There is no CPU
fallback: importing this package without the built library, or calling it
without a CUDA device, raises.

    import torch, paper_2508_19737_b200 as igp
    g = igp.build_graph(edges_cuda_int32_Ex2, num_nodes)
    Z = igp.embed(g, tau=-1.0, d=64, steps=60, seed=0)     # torch.float32 [N, 64] on cuda

Method: Alg. 1 lines 1-6: D_tau by Eq. (1),
Theta ~ N(0, 1/d), L layers Z <- ZNorm(tanh(phi * Z)) with Eq. (3)
 and Eq. (4), output sigmoid(Z^(L)).
"""
from __future__ import annotations

import ctypes
import os

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libigp.so")

MODES = {"full": 0, "pre_sigmoid": 1, "linear": 2}
FLAG_TIME_LAYERS = 1
FLAG_ROW_L2 = 2

IGP_OK = 0
_STATUS = {0: "IGP_OK", 2: "IGP_ERR_INPUT", 4: "IGP_ERR_NUMERICAL", 5: "IGP_ERR_CUDA", 6: "IGP_ERR_OOM",
           7: "IGP_ERR_UNSUPPORTED"}


class IGPError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


class EmbedOpts(ctypes.Structure):
    _fields_ = [("tau", ctypes.c_float), ("d", ctypes.c_int32), ("steps", ctypes.c_int32),
                ("seed", ctypes.c_uint64), ("subsequence", ctypes.c_uint64), ("theta", ctypes.c_float),
                ("alpha", ctypes.c_float), ("eps", ctypes.c_float), ("mode", ctypes.c_int32),
                ("flags", ctypes.c_uint32), ("d_z0", ctypes.c_void_p), ("ddof", ctypes.c_int32)]


# name -> (restype, argtypes); mirrors include/igp.h
_P, _i32, _i64, _u64, _f32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_float
SIGNATURES = {
    "igp_build_graph": (ctypes.c_int, [_P, _i64, _i32, _P, ctypes.POINTER(_P)]),
    "igp_build_graph_ex": (ctypes.c_int, [_P, _i64, _i32, ctypes.c_uint32, _P, ctypes.POINTER(_P)]),
    "igp_graph_add_edges": (ctypes.c_int, [_P, _P, _i64, _P]),
    "igp_graph_info": (ctypes.c_int, [_P, ctypes.POINTER(_i32), ctypes.POINTER(_i64), ctypes.POINTER(_i64)]),
    "igp_graph_status": (ctypes.c_int, [_P]),
    "igp_graph_copy_csr": (ctypes.c_int, [_P, _P, _P, _P, _P]),
    "igp_destroy_graph": (ctypes.c_int, [_P]),
    "igp_destroy_graph_async": (ctypes.c_int, [_P, _P]),
    "igp_embed_opts_default": (None, [ctypes.POINTER(EmbedOpts)]),
    "igp_embed": (ctypes.c_int, [_P, _f32, _i32, _i32, _u64, _P, _P]),
    "igp_embed_ex": (ctypes.c_int, [_P, ctypes.POINTER(EmbedOpts), _P, _P]),
    "igp_embed_host": (ctypes.c_int, [_P, _i64, _i32, ctypes.POINTER(EmbedOpts), _P, _P]),
    "igp_layer_timer_reset": (ctypes.c_int, []),
    "igp_layer_timer_read": (ctypes.c_int, [ctypes.POINTER(_f32), ctypes.POINTER(_i64)]),
    "igp_philox_bits": (ctypes.c_int, [_u64, _u64, _i64, _P, _P]),
    "igp_philox_normal": (ctypes.c_int, [_u64, _u64, _i64, _P, _P]),
    "igp_birch_create": (ctypes.c_int, [_i32, ctypes.c_double, _i32, ctypes.POINTER(_P)]),
    "igp_birch_partial_fit": (ctypes.c_int, [_P, _P, _i64, _P]),
    "igp_birch_info": (ctypes.c_int, [_P, ctypes.POINTER(_i64), ctypes.POINTER(_i32), ctypes.POINTER(_i64),
                                      ctypes.POINTER(_i64)]),
    "igp_birch_clusters": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, _P]),
    "igp_birch_predict": (ctypes.c_int, [_P, _P, _i64, _P, _P]),
    "igp_birch_predict_ex": (ctypes.c_int, [_P, _P, _i64, _P, _i32, ctypes.POINTER(_i64), _P]),
    "igp_birch_destroy": (ctypes.c_int, [_P]),
    "igp_status_string": (ctypes.c_char_p, [ctypes.c_int]),
    "igp_last_error_message": (ctypes.c_char_p, []),
    "igp_kernel_launch_count": (_u64, []),
    "igp_version": (ctypes.c_char_p, []),
    "igp_trim_memory": (ctypes.c_int, []),
}

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python paper_2508_19737_b200/_build.py` "
                      "(there is no CPU fallback)")
_lib = ctypes.CDLL(LIB_PATH)
for _name, (_res, _args) in SIGNATURES.items():
    _fn = getattr(_lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args


def lib() -> ctypes.CDLL:
    return _lib


def _check(status: int):
    if status != IGP_OK:
        raise IGPError(status, _lib.igp_last_error_message().decode())


def _stream_ptr(stream) -> ctypes.c_void_p:
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _require_cuda(t: torch.Tensor, dtype, name: str):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if t.dtype != dtype or not t.is_contiguous():
        raise TypeError(f"{name} must be a contiguous {dtype} tensor")


class Graph:
    """Device CSR handle (igp_graph_t).  Owns row_ptr / col_idx on the device.

    ``nnz`` / ``num_edges`` are read lazily (igp_graph_info): for a graph built with
    ``async_build=True`` the first access waits for the build and raises on a range error."""

    def __init__(self, handle: ctypes.c_void_p, device: torch.device, num_nodes: int):
        self._h = handle
        self.device = device
        self.num_nodes = int(num_nodes)
        self._nnz = None

    @property
    def handle(self):
        if self._h is None:
            raise ValueError("graph was destroyed")
        return self._h

    def _info(self):
        if self._nnz is None:
            n, nnz, m = _i32(), _i64(), _i64()
            _check(_lib.igp_graph_info(self.handle, ctypes.byref(n), ctypes.byref(nnz), ctypes.byref(m)))
            self._nnz = nnz.value
        return self._nnz

    @property
    def nnz(self) -> int:
        return self._info()

    @property
    def num_edges(self) -> int:
        return self._info() // 2

    def status(self):
        """igp_graph_status: wait for the build / last merge; raises IGPError on a range error."""
        _check(_lib.igp_graph_status(self.handle))

    def csr(self, stream=None, degrees: bool = False):
        """(row_ptr int32[N+1], col_idx int32[nnz]) copies on the graph's device; with
        ``degrees=True`` also deg int32[N] (igp_graph_copy_csr's d_deg)."""
        rp = torch.empty(self.num_nodes + 1, dtype=torch.int32, device=self.device)
        ci = torch.empty(max(self.nnz, 1), dtype=torch.int32, device=self.device)
        deg = torch.empty(self.num_nodes, dtype=torch.int32, device=self.device) if degrees else None
        _check(_lib.igp_graph_copy_csr(self.handle, ctypes.c_void_p(rp.data_ptr()), ctypes.c_void_p(ci.data_ptr()),
                                       ctypes.c_void_p(deg.data_ptr() if degrees else 0), _stream_ptr(stream)))
        return (rp, ci[: self.nnz], deg) if degrees else (rp, ci[: self.nnz])

    def add_edges(self, edges: torch.Tensor, stream=None):
        """igp_graph_add_edges: merge new edges (CUDA int32 [E, 2]) into this graph in place."""
        _require_cuda(edges, torch.int32, "edges")
        with torch.cuda.device(self.device):
            _check(_lib.igp_graph_add_edges(self.handle, ctypes.c_void_p(edges.data_ptr()), edges.shape[0],
                                            _stream_ptr(stream)))
        self._nnz = None
        return self

    def close(self, stream=None):
        """Destroy the handle: with ``stream`` in stream order (igp_destroy_graph_async, no host
        sync; all work on the graph must be on / ordered before that stream), else after a
        device sync (igp_destroy_graph)."""
        if self._h is not None:
            if stream is None:
                _lib.igp_destroy_graph(self._h)
            else:
                with torch.cuda.device(self.device):
                    _lib.igp_destroy_graph_async(self._h, _stream_ptr(stream))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


BUILD_NO_REORDER = 1
BUILD_ASYNC = 2
BUILD_REORDER_COMMUNITY = 4
BUILD_REORDER_DEGREE = 8
ORDERS = {"auto": 0, "none": BUILD_NO_REORDER, "degree": BUILD_REORDER_DEGREE, "community": BUILD_REORDER_COMMUNITY}


def build_graph(edges: torch.Tensor, num_nodes: int, stream=None, reorder: bool = True,
                async_build: bool = False, order: str | None = None) -> Graph:
    """igp_build_graph_ex: canonical CSR of the undirected simple graph.

    ``edges``: CUDA int32 tensor [E, 2] (duplicates / both orientations / self loops allowed).
    ``order``: row order of the filter steps: "auto" (default: "community" once N x 128 B
    exceeds half the L2, else "degree"), "degree" (IGP_BUILD_REORDER_DEGREE), "community"
    (IGP_BUILD_REORDER_COMMUNITY) or "none" (IGP_BUILD_NO_REORDER; also ``reorder=False``).
    ``async_build=True`` returns without any host sync (IGP_BUILD_ASYNC); range errors surface
    from ``Graph.status()`` / ``nnz``."""
    _require_cuda(edges, torch.int32, "edges")
    if edges.dim() != 2 or edges.shape[1] != 2:
        raise ValueError("edges must have shape [E, 2]")
    h = _P()
    if order is None:
        order = "auto" if reorder else "none"
    flags = ORDERS[order] | (BUILD_ASYNC if async_build else 0)
    with torch.cuda.device(edges.device):
        _check(_lib.igp_build_graph_ex(ctypes.c_void_p(edges.data_ptr()), edges.shape[0], int(num_nodes),
                                       flags, _stream_ptr(stream), ctypes.byref(h)))
    return Graph(h, edges.device, num_nodes)


def layer_timer_reset():
    """igp_layer_timer_reset: forget the filter-step intervals recorded so far."""
    _check(_lib.igp_layer_timer_reset())


def layer_timer_read():
    """igp_layer_timer_read: (total ms, launches) of the filter-step intervals recorded by
    embeds with ``time_layers=True`` since the last reset (waits for them to complete)."""
    ms, n = _f32(), _i64()
    _check(_lib.igp_layer_timer_read(ctypes.byref(ms), ctypes.byref(n)))
    return ms.value, n.value


def make_opts(tau: float, d: int, steps: int, seed: int = 0, *, subsequence: int = 0, theta: float = 0.1,
              alpha: float = 1.0, eps: float = 1e-3, mode: str = "full", time_layers: bool = False,
              row_l2: bool = False, z0: torch.Tensor | None = None, ddof: int = 0) -> EmbedOpts:
    o = EmbedOpts()
    _lib.igp_embed_opts_default(ctypes.byref(o))
    o.tau, o.d, o.steps, o.seed, o.subsequence = float(tau), int(d), int(steps), int(seed), int(subsequence)
    o.theta, o.alpha, o.eps, o.mode, o.ddof = float(theta), float(alpha), float(eps), MODES[mode], int(ddof)
    o.flags = (FLAG_TIME_LAYERS if time_layers else 0) | (FLAG_ROW_L2 if row_l2 else 0)
    if z0 is not None:  # caller-provided Z^(0) (CUDA float32 [N, d]) instead of Theta
        _require_cuda(z0, torch.float32, "z0")
        o.d_z0 = z0.data_ptr()
    return o


def embed(graph: Graph, tau: float, d: int, steps: int, seed: int = 0, *, out: torch.Tensor | None = None,
          stream=None, **kw) -> torch.Tensor:
    """igp_embed_ex: Alg. 1 l.1-6; returns Z~ as CUDA float32 [N, d] (asynchronous on ``stream``)."""
    o = make_opts(tau, d, steps, seed, **kw)
    z0 = kw.get("z0")
    if z0 is not None and tuple(z0.shape) != (graph.num_nodes, int(d)):
        raise ValueError("z0 must have shape [N, d]")
    if out is None:
        out = torch.empty((graph.num_nodes, int(d)), dtype=torch.float32, device=graph.device)
    _require_cuda(out, torch.float32, "out")
    if tuple(out.shape) != (graph.num_nodes, int(d)):
        raise ValueError("out must have shape [N, d]")
    with torch.cuda.device(graph.device):
        _check(_lib.igp_embed_ex(graph.handle, ctypes.byref(o), ctypes.c_void_p(out.data_ptr()), _stream_ptr(stream)))
    return out


def embed_host(edges, num_nodes: int, tau: float, d: int, steps: int, seed: int = 0, *, out=None, stream=None,
               **kw) -> torch.Tensor:
    """igp_embed_host: end to end from HOST edges (int32 [E, 2], pinned recommended) to a HOST
    float32 [N, d] result; copies, build, embed and the stream sync happen inside the call."""
    e = edges if isinstance(edges, torch.Tensor) else torch.from_numpy(edges)
    if e.is_cuda or e.dtype != torch.int32 or not e.is_contiguous():
        raise TypeError("edges must be a contiguous host int32 tensor/array")
    if out is None:
        out = torch.empty((int(num_nodes), int(d)), dtype=torch.float32, pin_memory=True)
    if out.is_cuda or out.dtype != torch.float32 or not out.is_contiguous():
        raise TypeError("out must be a contiguous host float32 tensor")
    o = make_opts(tau, d, steps, seed, **kw)
    _check(_lib.igp_embed_host(ctypes.c_void_p(e.data_ptr()), e.shape[0] if e.dim() == 2 else 0, int(num_nodes),
                               ctypes.byref(o), ctypes.c_void_p(out.data_ptr()), _stream_ptr(stream)))
    return out


def philox_bits(seed: int, subsequence: int, count: int, device="cuda", stream=None) -> torch.Tensor:
    """Raw Philox4x32-10 words as int32 (bit pattern of the uint32 draws)."""
    out = torch.empty(max(count, 1), dtype=torch.int32, device=device)
    _check(_lib.igp_philox_bits(seed, subsequence, count, ctypes.c_void_p(out.data_ptr()), _stream_ptr(stream)))
    return out[:count]


def philox_normal(seed: int, subsequence: int, count: int, device="cuda", stream=None) -> torch.Tensor:
    out = torch.empty(max(count, 4), dtype=torch.float32, device=device)
    _check(_lib.igp_philox_normal(seed, subsequence, count, ctypes.c_void_p(out.data_ptr()), _stream_ptr(stream)))
    return out[:count]


class Birch:
    """BIRCH CF tree on the device (igp_birch_t; Alg. 1 l.7, Alg. 2 l.9-11): ``partial_fit``
    inserts rows (CUDA float32 [m, d]) in order, ``predict`` labels rows by their nearest
    cluster, ``clusters`` returns the leaf entries (K-agnostic clusters) in label order."""

    def __init__(self, d: int, threshold: float = 0.5, branching: int = 50, device=None):
        self.d = int(d)
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        h = _P()
        with torch.cuda.device(self.device):
            _check(_lib.igp_birch_create(self.d, float(threshold), int(branching), ctypes.byref(h)))
        self._h = h

    def _rows(self, X):
        _require_cuda(X, torch.float32, "X")
        if X.dim() != 2 or X.shape[1] != self.d:
            raise ValueError(f"X must have shape [m, {self.d}]")
        return X

    def partial_fit(self, X: torch.Tensor, stream=None):
        X = self._rows(X)
        with torch.cuda.device(self.device):
            _check(_lib.igp_birch_partial_fit(self._h, ctypes.c_void_p(X.data_ptr()), X.shape[0], _stream_ptr(stream)))
        return self

    fit = partial_fit

    def info(self):
        """(K clusters, depth, nodes, points)"""
        k, dep, nodes, pts = _i64(), _i32(), _i64(), _i64()
        with torch.cuda.device(self.device):
            _check(_lib.igp_birch_info(self._h, ctypes.byref(k), ctypes.byref(dep), ctypes.byref(nodes),
                                       ctypes.byref(pts)))
        return k.value, dep.value, nodes.value, pts.value

    def clusters(self, stream=None):
        """(centroids [K, d], sqn [K], n [K], LS [K, d], SS [K]) as CUDA float64 tensors."""
        K = self.info()[0]
        f = dict(dtype=torch.float64, device=self.device)
        cen, ls = torch.empty((K, self.d), **f), torch.empty((K, self.d), **f)
        sqn, n, ss = torch.empty(K, **f), torch.empty(K, **f), torch.empty(K, **f)
        ptr = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
        with torch.cuda.device(self.device):
            _check(_lib.igp_birch_clusters(self._h, ptr(cen), ptr(sqn), ptr(n), ptr(ls), ptr(ss), _stream_ptr(stream)))
        return cen, sqn, n, ls, ss

    PATHS = {"auto": 0, "fp64": 1, "tensor": 2}  # IGP_PREDICT_*

    def predict(self, X: torch.Tensor, stream=None, out: torch.Tensor | None = None, path: str = "auto",
                return_ambiguous: bool = False):
        """Labels (int32 [m]).  path: "fp64" (CUDA cores, every distance in fp64), "tensor"
        (tcgen05 3xTF32 scores, certified; uncertified rows re-solved in fp64), "auto" (tensor
        where d allows).  The labels are the same on every path.  With return_ambiguous, also
        the number of rows solved in fp64 (synchronises)."""
        X = self._rows(X)
        if path not in self.PATHS:
            raise ValueError(f"path must be one of {sorted(self.PATHS)}")
        if out is None:
            out = torch.empty(X.shape[0], dtype=torch.int32, device=self.device)
        _require_cuda(out, torch.int32, "out")
        if out.dim() != 1 or out.shape[0] < X.shape[0]:
            raise ValueError("out must be int32 [m]")
        amb = _i64()
        with torch.cuda.device(self.device):
            _check(_lib.igp_birch_predict_ex(self._h, ctypes.c_void_p(X.data_ptr()), X.shape[0],
                                             ctypes.c_void_p(out.data_ptr()), self.PATHS[path],
                                             ctypes.byref(amb) if return_ambiguous else None, _stream_ptr(stream)))
        return (out, amb.value) if return_ambiguous else out

    def close(self):
        if getattr(self, "_h", None) is not None:
            _lib.igp_birch_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def trim_memory():
    """igp_trim_memory: return the library's cached pool memory on the current device to the driver."""
    _check(_lib.igp_trim_memory())


def kernel_launch_count() -> int:
    return int(_lib.igp_kernel_launch_count())


def version() -> str:
    return _lib.igp_version().decode()
