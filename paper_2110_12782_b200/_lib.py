"""ctypes binding of libnetmfp.so (include/netmfp.h) — argument marshalling only.

Every compute call goes to the CUDA library; there is no Python or CPU
fallback.  If the shared library is missing or cannot be loaded, importing
this module raises.  Buffers may be torch tensors (CUDA -> NETMFP_MEM_DEVICE,
CPU -> NETMFP_MEM_HOST) or numpy arrays (host); all buffers of one call must
live in the same memory space.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libnetmfp.so")

MEM_DEVICE, MEM_HOST = 0, 1
LOG_TRUNC, LOG_LOG1P = 0, 1
OK, ERR_ARG, ERR_CUDA, ERR_NUMERIC, ERR_OOM, ERR_NCCL = 0, 1, 2, 3, 4, 5

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libnetmfp.so not built ({LIB_PATH}); run __graft_entry__.build() "
                      "or python -m paper_2110_12782_b200.build")
_L = C.CDLL(LIB_PATH)

_p = C.c_void_p
_i64 = C.c_int64
_i32 = C.c_int32
_d = C.c_double
_u64 = C.c_uint64


class Params(C.Structure):
    """netmfp_params (include/netmfp.h) — Alg. 5 inputs."""
    _fields_ = [("alpha", _d), ("k", _i32), ("s1", _i32), ("q", _i32), ("T", _i32), ("b", _d),
                ("d", _i32), ("s2", _i32), ("s3", _i32), ("z", _i32), ("prop_order", _i32),
                ("mu", _d), ("theta", _d), ("seed", _u64), ("logmode", _i32)]


_SIGS = {
    "netmfp_ctx_create": (C.c_int, [C.c_int, _p, C.POINTER(_p)]),
    "netmfp_ctx_destroy": (C.c_int, [_p]),
    "netmfp_ctx_launches": (_i64, [_p]),
    "netmfp_ctx_profile": (C.c_int, [_p, C.c_int, C.c_char_p]),
    "netmfp_ctx_profile_read": (C.c_int, [_p, C.c_char_p, C.c_size_t]),
    "netmfp_last_error": (C.c_char_p, []),
    "netmfp_version": (C.c_char_p, []),
    "netmfp_build_csr": (C.c_int, [_p, _i64, _p, _p, _i64, C.c_int, C.POINTER(_p)]),
    "netmfp_graph_info": (C.c_int, [_p, C.POINTER(_i64), C.POINTER(_i64), C.POINTER(_i64)]),
    "netmfp_graph_export": (C.c_int, [_p, _p, _p, _p, _p, C.c_int]),
    "netmfp_graph_free": (C.c_int, [_p]),
    "netmfp_partition_rows": (C.c_int, [_p, _i64, _i32, _p]),
    "netmfp_spmm": (C.c_int, [_p, _p, _d, _d, _p, _i64, _p, _i64, _i64, C.c_int]),
    "netmfp_gaussian": (C.c_int, [_p, _i64, _i64, C.c_uint64, _p, _i64, C.c_int]),
    "netmfp_gram": (C.c_int, [_p, _i64, _p, _i64, _i64, _p, _i64, _i64, _p, C.c_int]),
    "netmfp_orthonormalize": (C.c_int, [_p, _i64, _i64, _p, _i64, _p, _i64, _i32, C.c_int]),
    "netmfp_sym_eig": (C.c_int, [_p, _p, _i64, _p, _p, _i32, C.c_int]),
    "netmfp_eig": (C.c_int, [_p, _p, _d, _i32, _i32, _i32, _u64, _p, _i64, _p, C.c_int]),
    "netmfp_factor_pair": (C.c_int, [_p, _p, _d, _i32, _p, _i64, _p, _i32, _p, _i64, _p, C.c_int]),
    "netmfp_sketch_svd": (C.c_int, [_p, _i64, _p, _i64, _p, _i32, _d, _i32, _i32, _i32, _i32, _u64,
                                    _i32, _p, _i64, _p, _p, _i64, _p, _i64, _p, C.c_int]),
    "netmfp_propagate": (C.c_int, [_p, _p, _p, _i64, _i32, _i32, _d, _d, C.c_int]),
    "netmfp_cheb_coeffs": (C.c_int, [_i32, _d, _d, _p]),
    "netmfp_embed": (C.c_int, [_p, _p, C.POINTER(Params), _p, _i64, _p, _p, C.c_int]),
    "netmfp_embed_edges": (C.c_int, [_p, _i64, _p, _p, _i64, C.POINTER(Params), _p, _i64, _p, C.c_int]),
    "netmfp_dist_unique_id": (C.c_int, [_p]),
    "netmfp_dist_init": (C.c_int, [_p, _p, _i32, _i32]),
    "netmfp_dist_build_csr": (C.c_int, [_p, _i64, _p, _p, _i64, _p, C.c_int, C.POINTER(_p)]),
    "netmfp_graph_rows": (C.c_int, [_p, C.POINTER(_i64), C.POINTER(_i64), C.POINTER(_i64)]),
    "netmfp_build_csr_rows": (C.c_int, [_p, _i64, _p, _p, _i64, _i64, _i64, C.c_int, C.POINTER(_p)]),
    "netmfp_dist_init_ops": (C.c_int, [_p, _p, _i32, _i32]),
    "netmfp_dist_stats": (C.c_int, [_p, C.POINTER(_i64), C.POINTER(_i64)]),
}
DIST_ID_BYTES = 128
for _name, (_res, _args) in _SIGS.items():
    _f = getattr(_L, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_SIGS)

# Objects freed during interpreter shutdown must not call into the library
# after the CUDA runtime has been torn down.
_SHUTDOWN = [False]


def _on_exit():
    _SHUTDOWN[0] = True


import atexit  # noqa: E402

atexit.register(_on_exit)


class NetmfpError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"netmfp error {code}: {msg}")
        self.code = code


def _check(rc):
    if rc != OK:
        raise NetmfpError(rc, _L.netmfp_last_error().decode())


# ---------------------------------------------------------------- buffers
def _is_torch(x):
    return type(x).__module__.startswith("torch")


def _mem(x):
    if x is None:
        return None
    if _is_torch(x):
        return MEM_DEVICE if x.is_cuda else MEM_HOST
    return MEM_HOST


def _ptr(x):
    if x is None:
        return None
    if _is_torch(x):
        return x.data_ptr()
    return x.ctypes.data


def _ld(x, dtype_name):
    """Leading dimension of a row-major 2-D buffer (stride(1) == 1)."""
    if _is_torch(x):
        assert x.dim() == 2 and x.stride(1) == 1, "row-major 2-D buffer required"
        assert str(x.dtype).endswith(dtype_name), f"{dtype_name} buffer required, got {x.dtype}"
        return x.stride(0)
    assert x.ndim == 2 and x.strides[1] == x.itemsize and x.dtype.name == dtype_name
    return x.strides[0] // x.itemsize


def _same_mem(*xs):
    ms = {_mem(x) for x in xs if x is not None}
    assert len(ms) == 1, "all buffers of one call must be in the same memory space"
    return ms.pop()


# ---------------------------------------------------------------- objects
class Context:
    """netmfp_ctx: device + stream (defaults to torch's current stream)."""

    def __init__(self, device: int = 0, stream=None):
        h = _p()
        if stream is None:
            try:
                import torch
                stream = torch.cuda.current_stream(device).cuda_stream
            except Exception:
                stream = None
        _check(_L.netmfp_ctx_create(device, stream, C.byref(h)))
        self.h = h
        self.device = device

    @property
    def launches(self) -> int:
        return int(_L.netmfp_ctx_launches(self.h))

    def profile(self, enable: bool = True, kernels: str = ""):
        """Time matching kernel launches with CUDA events (see netmfp_ctx_profile)."""
        _check(_L.netmfp_ctx_profile(self.h, 1 if enable else 0, kernels.encode()))

    def profile_read(self) -> dict:
        """{kernel: (launches, total_ms)} since the last read."""
        buf = C.create_string_buffer(1 << 16)
        _check(_L.netmfp_ctx_profile_read(self.h, buf, len(buf)))
        out = {}
        for line in buf.value.decode().splitlines():
            name, cnt, ms = line.split()
            out[name] = (int(cnt), float(ms))
        return out

    def close(self):
        if getattr(self, "h", None) and not _SHUTDOWN[0]:
            _L.netmfp_ctx_destroy(self.h)
        self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Graph:
    """netmfp_graph: device-resident CSR owned by the library."""

    def __init__(self, h):
        self.h = h
        n, nnz, nh = _i64(), _i64(), _i64()
        _check(_L.netmfp_graph_info(h, C.byref(n), C.byref(nnz), C.byref(nh)))
        self.n, self.nnz, self.n_heavy = n.value, nnz.value, nh.value

    def export(self, ctx: Context):
        rowptr = np.empty(self.n + 1, dtype=np.int64)
        col = np.empty(max(self.nnz, 1), dtype=np.int32)
        deg = np.empty(self.n, dtype=np.int32)
        _check(_L.netmfp_graph_export(ctx.h, self.h, rowptr.ctypes.data, col.ctypes.data,
                                      deg.ctypes.data, MEM_HOST))
        return rowptr, col[: self.nnz], deg

    def close(self):
        if getattr(self, "h", None) and not _SHUTDOWN[0]:
            _L.netmfp_graph_free(self.h)
        self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------- calls
def netmfp_build_csr(ctx: Context, n: int, src, dst) -> Graph:
    mem = _same_mem(src, dst)
    h = _p()
    _check(_L.netmfp_build_csr(ctx.h, n, _ptr(src), _ptr(dst), len(src), mem, C.byref(h)))
    g = Graph(h)
    g.ctx = ctx  # keep the creating context alive as long as the graph
    return g


def netmfp_dist_unique_id() -> bytes:
    """A fresh communicator id (rank 0 creates it; share it, e.g. with
    torch.distributed.broadcast_object_list)."""
    buf = C.create_string_buffer(DIST_ID_BYTES)
    _check(_L.netmfp_dist_unique_id(buf))
    return buf.raw


def netmfp_dist_init(ctx: Context, uid: bytes, nranks: int, rank: int) -> None:
    buf = C.create_string_buffer(bytes(uid), DIST_ID_BYTES)
    _check(_L.netmfp_dist_init(ctx.h, buf, nranks, rank))


_ALLRED = C.CFUNCTYPE(C.c_int, _p, _p, _i64, _i32)
_BCAST = C.CFUNCTYPE(C.c_int, _p, _p, _i64, _i32, _i32)


class CommOps(C.Structure):
    """netmfp_comm_ops (include/netmfp.h): host-staged communicator callbacks."""
    _fields_ = [("user", _p), ("allreduce_sum", _ALLRED), ("broadcast", _BCAST)]


_DT_CTYPES = {0: C.c_float, 1: C.c_double, 2: C.c_int64, 3: C.c_int32, 4: C.c_uint8}


def netmfp_dist_init_ops(ctx: Context, nranks: int, rank: int, allreduce_sum, broadcast) -> None:
    """Join a host-staged communicator: allreduce_sum(a) and broadcast(a, root)
    act in place on numpy views of the library's host staging buffers (e.g.
    torch.distributed gloo calls on torch.from_numpy(a)); collective over ranks."""
    def _view(buf, count, dt):
        return np.ctypeslib.as_array((_DT_CTYPES[dt] * count).from_address(buf))

    def _ar(user, buf, count, dt):
        try:
            allreduce_sum(_view(buf, count, dt))
            return 0
        except Exception:  # reported as NETMFP_ERR_NCCL by the library
            return 1

    def _bc(user, buf, count, dt, root):
        try:
            broadcast(_view(buf, count, dt), root)
            return 0
        except Exception:
            return 1

    ops = CommOps(None, _ALLRED(_ar), _BCAST(_bc))
    ctx._comm_ops = ops  # keep the callbacks alive as long as the context
    _check(_L.netmfp_dist_init_ops(ctx.h, C.byref(ops), nranks, rank))


def netmfp_dist_stats(ctx: Context):
    """(bytes received in collectives, collectives) since the last call."""
    b, k = _i64(), _i64()
    _check(_L.netmfp_dist_stats(ctx.h, C.byref(b), C.byref(k)))
    return b.value, k.value


def netmfp_dist_build_csr(ctx: Context, n: int, src, dst, bounds=None) -> Graph:
    """This rank's rows of the row-partitioned CSR (collective)."""
    mem = _same_mem(src, dst)
    h = _p()
    b = None if bounds is None else np.ascontiguousarray(bounds, dtype=np.int64)
    _check(_L.netmfp_dist_build_csr(ctx.h, n, _ptr(src), _ptr(dst), len(src), None if b is None else b.ctypes.data,
                                    mem, C.byref(h)))
    g = Graph(h)
    g.ctx = ctx
    return g


def netmfp_build_csr_rows(ctx: Context, n: int, src, dst, row0: int, row1: int) -> Graph:
    """CSR of rows [row0, row1) with global column ids (one rank's partition)."""
    mem = _same_mem(src, dst)
    h = _p()
    _check(_L.netmfp_build_csr_rows(ctx.h, n, _ptr(src), _ptr(dst), len(src), row0, row1, mem, C.byref(h)))
    g = Graph(h)
    g.ctx = ctx
    return g


def netmfp_graph_rows(g: Graph):
    """(first global row, n, vol(G))."""
    r0, ng, vol = _i64(), _i64(), _i64()
    _check(_L.netmfp_graph_rows(g.h, C.byref(r0), C.byref(ng), C.byref(vol)))
    return r0.value, ng.value, vol.value


def netmfp_partition_rows(rowptr: np.ndarray, parts: int) -> np.ndarray:
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
    bounds = np.empty(parts + 1, dtype=np.int64)
    _check(_L.netmfp_partition_rows(rowptr.ctypes.data, rowptr.size - 1, parts, bounds.ctypes.data))
    return bounds


def netmfp_spmm(ctx, g: Graph, a: float, b: float, X, Y, cols=None):
    mem = _same_mem(X, Y)
    cols = X.shape[1] if cols is None else cols
    _check(_L.netmfp_spmm(ctx.h, g.h, a, b, _ptr(X), _ld(X, "float32"), _ptr(Y), _ld(Y, "float32"),
                          cols, mem))
    return Y


def netmfp_gaussian(ctx, seed, Omega):
    mem = _same_mem(Omega)
    _check(_L.netmfp_gaussian(ctx.h, Omega.shape[0], Omega.shape[1], seed, _ptr(Omega), _ld(Omega, "float32"), mem))
    return Omega


def netmfp_gram(ctx, A, B, G):
    mem = _same_mem(A, B, G)
    _check(_L.netmfp_gram(ctx.h, A.shape[0], _ptr(A), _ld(A, "float32"), A.shape[1], _ptr(B),
                          _ld(B, "float32"), B.shape[1], _ptr(G), mem))
    return G


def netmfp_orthonormalize(ctx, Y, Q, passes=2):
    mem = _same_mem(Y, Q)
    _check(_L.netmfp_orthonormalize(ctx.h, Y.shape[0], Y.shape[1], _ptr(Y), _ld(Y, "float32"), _ptr(Q),
                                    _ld(Q, "float32"), passes, mem))
    return Q


def netmfp_sym_eig(ctx, S, lam, V, abs_order=True):
    mem = _same_mem(S, lam, V)
    _check(_L.netmfp_sym_eig(ctx.h, _ptr(S), S.shape[0], _ptr(lam), _ptr(V), 1 if abs_order else 0, mem))
    return lam, V


def netmfp_eig(ctx, g: Graph, alpha, k, s1, q, seed, U, lam):
    mem = _same_mem(U, lam)
    _check(_L.netmfp_eig(ctx.h, g.h, alpha, k, s1, q, seed, _ptr(U), _ld(U, "float32"), _ptr(lam), mem))
    return U, lam


def netmfp_factor_pair(ctx, g: Graph, alpha, T, U, lam, F, Cm):
    mem = _same_mem(U, lam, F, Cm)
    k = lam.shape[0]
    _check(_L.netmfp_factor_pair(ctx.h, g.h, alpha, T, _ptr(U), _ld(U, "float32"), _ptr(lam), k,
                                 _ptr(F), _ld(F, "float32"), _ptr(Cm), mem))
    return F, Cm


def netmfp_sketch_svd(ctx, F, Cm, scale, d, s2, s3, z, seed, logmode=LOG_TRUNC, U=None, sigma=None,
                      E=None, Ysk=None, Zsk=None):
    mem = _same_mem(F, Cm, U, sigma, E, Ysk, Zsk)
    n, k = F.shape[0], Cm.shape[0]
    _check(_L.netmfp_sketch_svd(ctx.h, n, _ptr(F), _ld(F, "float32"), _ptr(Cm), k, scale, d, s2, s3, z,
                                seed, logmode, _ptr(U), _ld(U, "float32") if U is not None else 0,
                                _ptr(sigma), _ptr(E), _ld(E, "float32") if E is not None else 0,
                                _ptr(Ysk), _ld(Ysk, "float32") if Ysk is not None else 0, _ptr(Zsk), mem))
    return U, sigma, E


def netmfp_propagate(ctx, g: Graph, E, order, mu, theta):
    mem = _mem(E)
    _check(_L.netmfp_propagate(ctx.h, g.h, _ptr(E), _ld(E, "float32"), E.shape[1], order, mu, theta, mem))
    return E


def netmfp_cheb_coeffs(order, mu, theta) -> np.ndarray:
    c = np.empty(order + 1, dtype=np.float64)
    _check(_L.netmfp_cheb_coeffs(order, mu, theta, c.ctypes.data))
    return c


def make_params(**kw) -> Params:
    p = Params()
    for f, _ in Params._fields_:
        setattr(p, f, kw[f])
    return p


def netmfp_embed(ctx, g: Graph, params: Params, E, sigma=None, lam=None):
    mem = _same_mem(E, sigma, lam)
    _check(_L.netmfp_embed(ctx.h, g.h, C.byref(params), _ptr(E), _ld(E, "float32"), _ptr(sigma),
                           _ptr(lam), mem))
    return E


def netmfp_embed_edges(ctx, n, src, dst, params: Params, E, sigma=None):
    mem = _same_mem(src, dst, E, sigma)
    _check(_L.netmfp_embed_edges(ctx.h, n, _ptr(src), _ptr(dst), len(src), C.byref(params), _ptr(E),
                                 _ld(E, "float32"), _ptr(sigma), mem))
    return E


def version() -> str:
    return _L.netmfp_version().decode()
