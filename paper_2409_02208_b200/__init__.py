"""B200-native CBM multiply (arXiv 2409.02208 hot path) — Python binding.

The product is ``libcbm_b200.so`` (C++ host library + sm_100a CUDA kernels,
built in-tree by ``make -C paper_2409_02208_b200`` / ``__graft_entry__.build()``)
behind the C ABI of ``include/cbm_b200.h``. This module is a thin ctypes
mirror of the reference library's API for that path, keeping its names,
argument meaning and error behaviour:

=====================================  =========================================
reference (``/root/reference/proj``)   here
=====================================  =========================================
``build_cbm`` (builder.hpp:99)          :func:`build_cbm`
``build_cbm_normalized`` (:104-106)     :func:`build_cbm_normalized`
``count_scalar_ops`` (kernels.hpp:22)   :func:`count_scalar_ops`
``spmm`` / ``spmm_into`` (:34-39)       :meth:`DeviceCbm.spmm` / :meth:`DeviceCbm.spmm_into`
``spmv`` / ``spmv_into`` (:28-44)       :meth:`DeviceCbm.spmv` / :meth:`DeviceCbm.spmv_into`
``std::invalid_argument``               :class:`ValueError`
=====================================  =========================================

There is no CPU fallback: importing fails loudly when the shared library is
missing, and every multiply runs in the CUDA kernels.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

__all__ = [
    "CsrBinaryMatrix", "CbmMatrix", "DeviceCbm", "build_cbm", "build_cbm_normalized",
    "count_scalar_ops", "plan_dense", "generate_graph", "generate_dense", "CbmError", "FormatError",
    "load_cbm", "save_cbm", "dense_matmul", "csr_operator", "VIRTUAL_PARENT",
    "library_path", "gemm_parts", "ipc_handle", "ipc_open", "ipc_close",
]

VIRTUAL_PARENT = 0xFFFFFFFF
_HERE = os.path.dirname(os.path.abspath(__file__))
library_path = os.path.join(_HERE, "libcbm_b200.so")
if os.environ.get("CBM_B200_LIB"):  # dev tool: A/B a second in-tree build of the library
    library_path = os.path.join(_HERE, os.path.basename(os.environ["CBM_B200_LIB"]))

if not os.path.exists(library_path):
    raise ImportError(
        f"{library_path} is missing: build it with `make -C {_HERE}` or "
        "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")

_lib = C.CDLL(library_path)

OK, EINVAL, ECUDA, ENOMEM, ELOGIC, EFORMAT = 0, 1, 2, 3, 4, 5


class CbmError(RuntimeError):
    """Non-argument failure from the library (CUDA, memory, builder logic)."""

    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class _CsrView(C.Structure):
    _fields_ = [("n_rows", C.c_uint32), ("n_cols", C.c_uint32),
                ("row_ptr", C.c_void_p), ("col_idx", C.c_void_p)]


class _CbmView(C.Structure):
    _fields_ = [("n_rows", C.c_uint32), ("n_cols", C.c_uint32), ("nnz", C.c_uint64),
                ("alpha", C.c_uint64), ("is_normalized", C.c_int32),
                ("parent", C.c_void_p), ("topo_order", C.c_void_p), ("row_ptr", C.c_void_p),
                ("col_idx", C.c_void_p), ("values", C.c_void_p), ("row_scale", C.c_void_p),
                ("col_scale", C.c_void_p)]


class _Options(C.Structure):
    _fields_ = [("device", C.c_int32), ("order_faithful", C.c_int32),
                ("split_threshold", C.c_uint32), ("chunk", C.c_uint32), ("prescale", C.c_int32),
                ("kernel", C.c_int32), ("max_segments", C.c_int32),
                ("flatten_gain", C.c_int32), ("prefetch", C.c_int32), ("tile", C.c_int32),
                ("tile_rows", C.c_uint32), ("tile_stage", C.c_uint32), ("tile_vec", C.c_int32),
                ("dense", C.c_int32), ("dense_min", C.c_uint32), ("hub", C.c_int32)]


class _Info(C.Structure):
    _fields_ = [("n_rows", C.c_uint32), ("n_cols", C.c_uint32), ("nnz_delta", C.c_uint64),
                ("nnz_effective", C.c_uint64), ("n_flattened", C.c_uint32),
                ("n_levels", C.c_uint32), ("n_roots", C.c_uint32), ("n_interior", C.c_uint32),
                ("n_items", C.c_uint32), ("n_chunk_items", C.c_uint32),
                ("max_row_deltas", C.c_uint32), ("device_bytes", C.c_uint64),
                ("launches_per_call", C.c_uint32), ("is_normalized", C.c_int32),
                ("order_faithful", C.c_int32), ("tile_active", C.c_int32),
                ("tile_blocks", C.c_uint32), ("tile_max_rows", C.c_uint32),
                ("tile_max_staged", C.c_uint32), ("tile_cut_rows", C.c_uint32),
                ("tile_deltas", C.c_uint64), ("tile_staged_deltas", C.c_uint64),
                ("tile_staged_rows", C.c_uint64), ("dense_active", C.c_int32),
                ("dense_tiles", C.c_uint32), ("dense_chunks", C.c_uint64),
                ("dense_entries", C.c_uint64), ("cold_entries", C.c_uint64),
                ("hub_active", C.c_int32), ("hub_rows", C.c_uint32),
                ("hub_entries", C.c_uint64), ("hub_chunks", C.c_uint64)]


class _Stats(C.Structure):
    _fields_ = [("t_edges", C.c_double), ("t_arborescence", C.c_double),
                ("t_deltas", C.c_double), ("t_total", C.c_double),
                ("candidate_edges", C.c_uint64), ("rounds", C.c_uint32)]


_vp, _i64, _u64, _i32 = C.c_void_p, C.c_int64, C.c_uint64, C.c_int32
_sig = {
    "cbm_b200_last_error": (C.c_char_p, []),
    "cbm_b200_build": (C.c_int, [C.POINTER(_CsrView), _u64, _i32, _i32, _i32, C.POINTER(_vp)]),
    "cbm_b200_build_ex": (C.c_int, [C.POINTER(_CsrView), _u64, _i32, _i32, _i32, _i32,
                                    C.POINTER(_vp)]),
    "cbm_b200_host_view": (C.c_int, [_vp, C.POINTER(_CbmView)]),
    "cbm_b200_host_branches": (C.c_int, [_vp, C.POINTER(_vp), C.POINTER(_u64)]),
    "cbm_b200_host_stats": (C.c_int, [_vp, C.POINTER(_Stats)]),
    "cbm_b200_host_free": (None, [_vp]),
    "cbm_b200_load_cbm1": (C.c_int, [C.c_char_p, C.POINTER(_vp)]),
    "cbm_b200_save_cbm1": (C.c_int, [C.POINTER(_CbmView), C.c_char_p]),
    "cbm_b200_count_ops": (C.c_int, [C.POINTER(_CbmView), C.POINTER(_u64), C.POINTER(_u64)]),
    "cbm_b200_default_options": (None, [C.POINTER(_Options)]),
    "cbm_b200_upload": (C.c_int, [C.POINTER(_CbmView), C.POINTER(_Options), C.POINTER(_vp)]),
    "cbm_b200_upload_cbm1": (C.c_int, [C.c_char_p, C.POINTER(_Options), C.POINTER(_vp)]),
    "cbm_b200_free": (None, [_vp]),
    "cbm_b200_reserve": (C.c_int, [_vp, _i64]),
    "cbm_b200_reserve_on": (C.c_int, [_vp, _i64, _vp]),
    "cbm_b200_spmm_ex": (C.c_int, [_vp, _vp, _i64, _i64, _i64, _vp, _i64, _i64, _i64, C.c_uint32,
                                   _vp]),
    "cbm_b200_column_slab": (C.c_int, [_i64, C.c_int32, C.c_int32, C.POINTER(_i64),
                                       C.POINTER(_i64)]),
    "cbm_b200_spmm_sharded": (C.c_int, [C.POINTER(_vp), C.c_int32, _vp, _i64, _i64, _vp, _i64,
                                        _i64]),
    "cbm_b200_spmm": (C.c_int, [_vp, _vp, _i64, _i64, _i64, _vp, _i64, _i64, _i64, _vp]),
    "cbm_b200_spmm_host": (C.c_int, [_vp, _vp, _i64, _i64, _vp, _i64, _i64, _vp]),
    "cbm_b200_spmv": (C.c_int, [_vp, _vp, _i64, _i64, _vp, _i64, _i64, _vp]),
    "cbm_b200_get_info": (C.c_int, [_vp, C.POINTER(_Info)]),
    "cbm_b200_plan_dense": (C.c_int, [C.POINTER(_CbmView), C.c_uint32, C.POINTER(_u64)]),
    "cbm_b200_plan_hub": (C.c_int, [C.POINTER(_CbmView), C.c_int32, C.POINTER(_u64)]),
    "cbm_b200_dense_matmul": (C.c_int, [_vp, _i64, _i64, _vp, _i64, _vp, _vp]),
    "cbm_b200_gcn_forward": (C.c_int, [_vp, _vp, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _vp]),
    "cbm_b200_gemm_parts": (C.c_int, [C.POINTER(_vp), C.POINTER(_i64), _i32, _i64, _vp, _i64,
                                      C.POINTER(_vp), _i32, _i64, _i32, _vp]),
    "cbm_b200_ipc_handle": (C.c_int, [_vp, C.c_char_p, C.POINTER(_u64)]),
    "cbm_b200_ipc_open": (C.c_int, [C.c_char_p, _i32, C.POINTER(_vp)]),
    "cbm_b200_ipc_close": (C.c_int, [_vp]),
    "cbm_b200_gen_graph": (C.c_int, [C.c_char_p, C.POINTER(C.c_double), _i32, _u64,
                                     C.POINTER(_vp)]),
    "cbm_b200_csr_get": (C.c_int, [_vp, C.POINTER(_CsrView)]),
    "cbm_b200_csr_free": (None, [_vp]),
    "cbm_b200_gen_dense": (C.c_int, [_i32, _u64, _u64, C.c_double, C.c_double, _u64, _vp]),
}
for _name, (_res, _args) in _sig.items():
    _fn = getattr(_lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args

EXPORTED_SYMBOLS = tuple(_sig)


class FormatError(CbmError):
    """cbm::format_error (io.hpp:19-22): bad or truncated CBM1 container."""


def _check(rc: int):
    if rc == OK:
        return
    msg = _lib.cbm_b200_last_error().decode()
    if rc == EINVAL:
        raise ValueError(msg)
    if rc == EFORMAT:
        raise FormatError(rc, msg)
    raise CbmError(rc, msg)



# ---------------------------------------------------------------------------
# Host containers
# ---------------------------------------------------------------------------
@dataclass
class CsrBinaryMatrix:
    """Pattern CSR (csr.hpp:14-40): row_ptr u64[n_rows+1], col_idx u32[nnz]."""
    n_rows: int
    n_cols: int
    row_ptr: np.ndarray
    col_idx: np.ndarray

    def __post_init__(self):
        self.row_ptr = np.ascontiguousarray(self.row_ptr, dtype=np.uint64)
        self.col_idx = np.ascontiguousarray(self.col_idx, dtype=np.uint32)

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    @classmethod
    def from_rows(cls, n_cols: int, rows) -> "CsrBinaryMatrix":
        rp = [0]
        ci = []
        for r in rows:
            r = sorted(set(int(c) for c in r))
            ci.extend(r)
            rp.append(len(ci))
        return cls(len(rows), n_cols, np.array(rp, np.uint64), np.array(ci, np.uint32))

    def _view(self) -> _CsrView:
        return _CsrView(self.n_rows, self.n_cols, self.row_ptr.ctypes.data,
                        self.col_idx.ctypes.data)

    def dense(self) -> np.ndarray:
        d = np.zeros((self.n_rows, self.n_cols), np.float32)
        for i in range(self.n_rows):
            d[i, self.col_idx[self.row_ptr[i]:self.row_ptr[i + 1]]] = 1.0
        return d


@dataclass
class CbmMatrix:
    """A built CBM (CbmMatrix, builder.hpp:66-74), host arrays."""
    n_rows: int
    n_cols: int
    alpha: int
    is_normalized: bool
    parent: np.ndarray
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray
    row_scale: np.ndarray | None = None
    topo_order: np.ndarray | None = None
    branch_ptr: np.ndarray | None = None
    build_stats: dict | None = None
    # normalized row block of a larger matrix (sharding.row_partition): the
    # per-column scale of the delta values; row_scale then scales its own rows
    col_scale: np.ndarray | None = None

    def __post_init__(self):
        self.parent = np.ascontiguousarray(self.parent, np.uint32)
        self.row_ptr = np.ascontiguousarray(self.row_ptr, np.uint64)
        self.col_idx = np.ascontiguousarray(self.col_idx, np.uint32)
        self.values = np.ascontiguousarray(self.values, np.float32)
        if self.row_scale is not None:
            self.row_scale = np.ascontiguousarray(self.row_scale, np.float32)
        if self.col_scale is not None:
            self.col_scale = np.ascontiguousarray(self.col_scale, np.float32)

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def _view(self) -> _CbmView:
        return _CbmView(self.n_rows, self.n_cols, self.nnz, self.alpha, int(self.is_normalized),
                        self.parent.ctypes.data,
                        self.topo_order.ctypes.data if self.topo_order is not None else None,
                        self.row_ptr.ctypes.data, self.col_idx.ctypes.data,
                        self.values.ctypes.data,
                        self.row_scale.ctypes.data if self.is_normalized else None,
                        self.col_scale.ctypes.data
                        if self.is_normalized and self.col_scale is not None else None)


def _copy(ptr, n, dtype):
    if n == 0:
        return np.zeros(0, dtype)
    buf = (C.c_char * (n * np.dtype(dtype).itemsize)).from_address(ptr)
    return np.frombuffer(buf, dtype=dtype, count=n).copy()


def _from_host_handle(h) -> CbmMatrix:
    try:
        v = _CbmView()
        _check(_lib.cbm_b200_host_view(h, C.byref(v)))
        bp, nb = _vp(), _u64()
        _check(_lib.cbm_b200_host_branches(h, C.byref(bp), C.byref(nb)))
        st = _Stats()
        _check(_lib.cbm_b200_host_stats(h, C.byref(st)))
        m, z = v.n_rows, v.nnz
        return CbmMatrix(
            n_rows=m, n_cols=v.n_cols, alpha=v.alpha, is_normalized=bool(v.is_normalized),
            parent=_copy(v.parent, m, np.uint32), row_ptr=_copy(v.row_ptr, m + 1, np.uint64),
            col_idx=_copy(v.col_idx, z, np.uint32), values=_copy(v.values, z, np.float32),
            row_scale=_copy(v.row_scale, m, np.float32) if v.is_normalized else None,
            topo_order=_copy(v.topo_order, m, np.uint32),
            branch_ptr=_copy(bp.value, nb.value + 1, np.uint64),
            build_stats={"t_edges": st.t_edges, "t_arborescence": st.t_arborescence,
                         "t_deltas": st.t_deltas, "t_total": st.t_total,
                         "candidate_edges": st.candidate_edges, "rounds": st.rounds})
    finally:
        _lib.cbm_b200_host_free(h)


def _build(a: CsrBinaryMatrix, alpha, normalized, degree_mode, threads, algo=0) -> CbmMatrix:
    h = _vp()
    view = a._view()
    _check(_lib.cbm_b200_build_ex(C.byref(view), alpha, int(normalized), degree_mode,
                                  threads, algo, C.byref(h)))
    return _from_host_handle(h)


def load_cbm(path) -> CbmMatrix:
    """load_cbm (io.hpp:57): read and fully validate a CBM1 container."""
    h = _vp()
    _check(_lib.cbm_b200_load_cbm1(str(path).encode(), C.byref(h)))
    return _from_host_handle(h)


def save_cbm(c: CbmMatrix, path) -> None:
    """save_cbm (io.hpp:52): write a CBM1 container the reference can load."""
    v = c._view()
    _check(_lib.cbm_b200_save_cbm1(C.byref(v), str(path).encode()))


_ALGO = {"heap": 0, "rounds": 1}


def build_cbm(a: CsrBinaryMatrix, alpha: int = 0, threads: int = 1,
              arborescence: str = "heap") -> CbmMatrix:
    """build_cbm (builder.hpp:99): same chain and delta matrix as the reference."""
    return _build(a, alpha, False, 0, threads, _ALGO[arborescence])


def build_cbm_normalized(a: CsrBinaryMatrix, alpha: int = 0, threads: int = 1,
                         degree_mode: str = "augmented", arborescence: str = "heap") -> CbmMatrix:
    """build_cbm_normalized (builder.hpp:104-106): represents D^-1/2 (A+I) D^-1/2."""
    mode = {"augmented": 0, "original": 1}[degree_mode]
    return _build(a, alpha, True, mode, threads, _ALGO[arborescence])


def csr_operator(a: CsrBinaryMatrix, normalized: bool = False) -> CbmMatrix:
    """The UNCOMPRESSED matrix in CBM form (every parent virtual, one +1 delta
    per nonzero; normalized: the pattern of A + I with column and row scales),
    for timing the GPU CSR SpMM comparator with the same kernel (the paper's
    runtime-reduction metric; csr_spmm_into, kernels.cpp:152)."""
    rp, ci = a.row_ptr, a.col_idx
    scale = None
    if normalized:
        if a.n_rows != a.n_cols:
            raise ValueError("normalized_adjacency_csr: matrix must be square")
        rows = []
        for x in range(a.n_rows):
            r = ci[rp[x]:rp[x + 1]]
            if not np.any(r == x):
                r = np.sort(np.append(r, np.uint32(x)))
            rows.append(r)
        lens = np.array([len(r) for r in rows], np.uint64)
        rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
        ci = np.concatenate(rows).astype(np.uint32) if rows else np.zeros(0, np.uint32)
        deg = np.diff(rp).astype(np.float64)
        scale = (np.float32(1.0) / np.sqrt(deg).astype(np.float32)).astype(np.float32)
        vals = scale[ci]
    else:
        vals = np.ones(ci.size, np.float32)
    return CbmMatrix(a.n_rows, a.n_cols, 0, normalized,
                     np.full(a.n_rows, VIRTUAL_PARENT, np.uint32), rp, ci, vals, scale)


def count_scalar_ops(c: CbmMatrix) -> tuple[int, int]:
    """count_scalar_ops (kernels.cpp:66-68): (multiply_adds, update_adds)."""
    a, b = _u64(), _u64()
    v = c._view()
    _check(_lib.cbm_b200_count_ops(C.byref(v), C.byref(a), C.byref(b)))
    return a.value, b.value


def plan_dense(c: CbmMatrix, dense_min: int = 0) -> dict:
    """Host-only plan of the dense-block layout: what an upload
    with dense=1 would put on the tensor cores."""
    st = (_u64 * 6)()
    v = c._view()
    _check(_lib.cbm_b200_plan_dense(C.byref(v), dense_min, st))
    keys = ("tiles", "chunks", "dense_entries", "cold_entries", "padded_slots", "max_tile_rows")
    return dict(zip(keys, (int(x) for x in st)))


def plan_hub(c: CbmMatrix, mode: int = -1) -> dict:
    """Host-only plan of the hub-row panel: what an upload with
    hub=mode would take off the streaming kernel."""
    st = (_u64 * 6)()
    v = c._view()
    _check(_lib.cbm_b200_plan_hub(C.byref(v), mode, st))
    keys = ("active", "rows", "entries", "chunks", "pieces", "rest_deltas")
    return dict(zip(keys, (int(x) for x in st)))


def generate_graph(kind: str, params, seed: int) -> CsrBinaryMatrix:
    """Seeded synthetic graph (see include/cbm_b200.h and DESIGN.md §Workloads)."""
    p = (C.c_double * len(params))(*[float(x) for x in params])
    h = _vp()
    _check(_lib.cbm_b200_gen_graph(kind.encode(), p, len(params), seed, C.byref(h)))
    try:
        v = _CsrView()
        _check(_lib.cbm_b200_csr_get(h, C.byref(v)))
        rp = _copy(v.row_ptr, v.n_rows + 1, np.uint64)
        return CsrBinaryMatrix(v.n_rows, v.n_cols, rp, _copy(v.col_idx, int(rp[-1]), np.uint32))
    finally:
        _lib.cbm_b200_csr_free(h)


_DENSE_KIND = {"uniform": 0, "int": 1, "normal": 2, "glorot": 3}


def generate_dense(kind: str, rows: int, cols: int, seed: int, lo: float = -1.0,
                   hi: float = 1.0, out: np.ndarray | None = None) -> np.ndarray:
    """Seeded dense fill; "uniform" reproduces the reference's random_dense."""
    if out is None:
        out = np.empty((rows, cols), np.float32)
    assert out.dtype == np.float32 and out.flags.c_contiguous and out.size == rows * cols
    _check(_lib.cbm_b200_gen_dense(_DENSE_KIND[kind], rows, cols, lo, hi, seed,
                                   out.ctypes.data if out.size else None))
    return out


def column_slab(d: int, world: int, rank: int) -> tuple[int, int]:
    """[lo, hi) columns of `rank` of `world` (cbm_b200_column_slab)."""
    lo, hi = _i64(), _i64()
    _check(_lib.cbm_b200_column_slab(d, world, rank, C.byref(lo), C.byref(hi)))
    return lo.value, hi.value


def spmm_sharded(ops, x: np.ndarray, y: np.ndarray | None = None) -> np.ndarray:
    """Y = A X on host arrays with the columns split over `ops` (one DeviceCbm
    of the same matrix per device; cbm_b200_spmm_sharded)."""
    ops = list(ops)
    if not ops:
        raise ValueError("spmm_sharded: no handles")
    x = np.ascontiguousarray(x, np.float32)
    if x.ndim != 2:
        raise ValueError("spmm: operand must be 2-D")
    if y is None:
        y = np.empty((ops[0].n_rows, x.shape[1]), np.float32)
    hs = (_vp * len(ops))(*[o._h for o in ops])
    _check(_lib.cbm_b200_spmm_sharded(hs, len(ops), x.ctypes.data, x.shape[0], x.shape[1],
                                      y.ctypes.data, y.shape[0], y.shape[1]))
    return y


def dense_matmul(a, b, stream=None):
    """dense_matmul (dense.hpp:48-50) on CUDA float32 tensors, reference-exact."""
    torch = _torch()
    a, b = a.contiguous(), b.contiguous()
    if a.shape[1] != b.shape[0]:
        raise ValueError("dense_matmul: inner dimensions differ")
    c = torch.empty((a.shape[0], b.shape[1]), dtype=torch.float32, device=a.device)
    s = DeviceCbm._stream(stream)
    _check(_lib.cbm_b200_dense_matmul(a.data_ptr(), a.shape[0], a.shape[1], b.data_ptr(),
                                      b.shape[1], c.data_ptr(), s))
    return c


def _ptr(t):
    return t if isinstance(t, int) else t.data_ptr()


def gemm_parts(parts, part_k, m, b, outs, ldc, ordered=True, stream=None):
    """C = [A_0 | ... | A_{P-1}] . B written to every buffer of `outs`
    (cbm_b200_gemm_parts: the fused all-gather + GEMM of the multi-GPU GCN).
    `parts` / `outs` are CUDA tensors or raw device pointers (e.g. peer
    buffers from ipc_open); A_p is m x part_k[p] row-major, B is a CUDA
    tensor sum(part_k) x n, C has leading dimension ldc (floats)."""
    b = b.contiguous()
    n = b.shape[1]
    if b.shape[0] != sum(part_k):
        raise ValueError("dense_matmul: inner dimensions differ")
    pa = (_vp * len(parts))(*[_ptr(t) for t in parts])
    pk = (_i64 * len(part_k))(*[int(k) for k in part_k])
    po = (_vp * len(outs))(*[_ptr(t) for t in outs])
    _check(_lib.cbm_b200_gemm_parts(pa, pk, len(parts), m, b.data_ptr(), n, po, len(outs), ldc,
                                    int(ordered), DeviceCbm._stream(stream)))


def ipc_handle(t) -> tuple[bytes, int]:
    """(64-byte CUDA IPC handle of the allocation holding CUDA tensor `t`,
    byte offset of `t` inside that allocation)."""
    buf = C.create_string_buffer(64)
    off = _u64()
    _check(_lib.cbm_b200_ipc_handle(_ptr(t), buf, C.byref(off)))
    return buf.raw, int(off.value)


def ipc_open(handle, device: int = -1) -> int:
    """Map a peer's buffer from ipc_handle's (handle, offset); returns the
    device pointer of the peer's tensor (base + offset). Unmap the base with
    ipc_close(ptr - offset)."""
    raw, off = handle
    p = _vp()
    _check(_lib.cbm_b200_ipc_open(C.create_string_buffer(raw, 64), device, C.byref(p)))
    return int(p.value) + int(off)


def ipc_close(base_ptr: int):
    _check(_lib.cbm_b200_ipc_close(base_ptr))


# ---------------------------------------------------------------------------
# Device operator
# ---------------------------------------------------------------------------
def _torch():
    import torch  # device memory and streams only; plumbing, not the product
    return torch


class DeviceCbm:
    """A CBM uploaded once into the device layout."""

    def __init__(self, c: CbmMatrix | None, device: int | None = None,
                 order_faithful: bool = False, split_threshold: int = 0, chunk: int = 0,
                 prescale: int = -1, kernel: str = "auto", max_segments: int = 0,
                 flatten_gain: int = -1, prefetch: bool = False, tile: int = -1,
                 tile_rows: int = 0, tile_stage: int = 0, tile_vec: int = 0,
                 dense: int = -1, dense_min: int = 0, hub: int = -1, _cbm1_path=None):
        opt = _Options()
        _lib.cbm_b200_default_options(C.byref(opt))
        opt.device = -1 if device is None else int(device)
        opt.order_faithful = int(order_faithful)
        opt.split_threshold = split_threshold
        opt.chunk = chunk
        opt.prescale = prescale
        if kernel not in ("auto", "scalar"):
            raise ValueError("kernel must be 'auto' or 'scalar'")
        opt.kernel = {"auto": 0, "scalar": 1}[kernel]
        opt.max_segments = max_segments
        opt.flatten_gain = flatten_gain
        opt.prefetch = int(prefetch)
        opt.tile = int(tile)
        opt.tile_rows = tile_rows
        opt.tile_stage = tile_stage
        opt.tile_vec = tile_vec
        opt.dense = int(dense)
        opt.dense_min = dense_min
        opt.hub = int(hub)
        self._h = _vp()
        if _cbm1_path is not None:
            _check(_lib.cbm_b200_upload_cbm1(str(_cbm1_path).encode(), C.byref(opt),
                                             C.byref(self._h)))
            info = self.info()
            self.n_rows, self.n_cols = info["n_rows"], info["n_cols"]
            self.is_normalized = bool(info["is_normalized"])
        else:
            view = c._view()
            _check(_lib.cbm_b200_upload(C.byref(view), C.byref(opt), C.byref(self._h)))
            self.n_rows, self.n_cols = c.n_rows, c.n_cols
            self.is_normalized = c.is_normalized
        self.device = opt.device

    @classmethod
    def from_cbm1(cls, path, **options) -> "DeviceCbm":
        """A CBM1 container file straight to the device (cbm_b200_upload_cbm1:
        mapped, validated like load_cbm, uploaded)."""
        return cls(None, _cbm1_path=path, **options)

    def close(self, _free=_lib.cbm_b200_free):
        if getattr(self, "_h", None):
            _free(self._h)
            self._h = None

    __del__ = close

    def info(self) -> dict:
        i = _Info()
        _check(_lib.cbm_b200_get_info(self._h, C.byref(i)))
        return {k: getattr(i, k) for k, _ in _Info._fields_}

    def reserve(self, d_max: int, stream=None):
        """Pre-size the workspace of `stream` (default: the current stream)."""
        _check(_lib.cbm_b200_reserve_on(self._h, d_max, self._stream(stream)))

    @staticmethod
    def _stream(stream):
        if stream is None:
            return _torch().cuda.current_stream().cuda_stream
        return getattr(stream, "cuda_stream", stream)

    def spmm_into(self, x, y, stream=None, relu: bool = False):
        """Y = A X on CUDA float32 tensors (row-major; Y fully overwritten);
        relu=True fuses relu_inplace (dense.cpp:51-54) into the epilogue."""
        xs, ys = x.stride(), y.stride()
        if x.dim() != 2 or y.dim() != 2 or xs[1] != 1 or ys[1] != 1:
            raise ValueError("spmm: operands must be 2-D row-major")
        if relu:
            _check(_lib.cbm_b200_spmm_ex(self._h, x.data_ptr(), x.shape[0], x.shape[1], xs[0],
                                         y.data_ptr(), y.shape[0], y.shape[1], ys[0], 1,
                                         self._stream(stream)))
            return
        _check(_lib.cbm_b200_spmm(self._h, x.data_ptr(), x.shape[0], x.shape[1], xs[0],
                                  y.data_ptr(), y.shape[0], y.shape[1], ys[0],
                                  self._stream(stream)))

    def spmm(self, x, stream=None, relu: bool = False):
        torch = _torch()
        y = torch.empty((self.n_rows, x.shape[1]), dtype=torch.float32, device=x.device)
        self.spmm_into(x, y, stream, relu)
        return y

    def spmv_into(self, v, u, stream=None):
        vv = v.reshape(v.shape[0], -1) if v.dim() == 1 else v
        uu = u.reshape(u.shape[0], -1) if u.dim() == 1 else u
        _check(_lib.cbm_b200_spmv(self._h, vv.data_ptr(), vv.shape[0], vv.shape[1],
                                  uu.data_ptr(), uu.shape[0], uu.shape[1], self._stream(stream)))

    def spmv(self, v, stream=None):
        torch = _torch()
        u = torch.empty((self.n_rows, 1), dtype=torch.float32, device=v.device)
        self.spmv_into(v, u, stream)
        return u

    def spmm_host(self, x: np.ndarray, y: np.ndarray | None = None, stream=None) -> np.ndarray:
        """The drop-in for spmm_into on host DenseMatrix data: H2D, multiply, D2H."""
        x = np.ascontiguousarray(x, np.float32)
        if y is None:
            y = np.empty((self.n_rows, x.shape[1] if x.ndim == 2 else 1), np.float32)
        s = self._stream(stream) if stream is not None else None
        _check(_lib.cbm_b200_spmm_host(self._h, x.ctypes.data, x.shape[0], x.shape[1],
                                       y.ctypes.data, y.shape[0], y.shape[1], s))
        return y

    def gcn_forward(self, x, w0, w1, stream=None):
        """gcn_forward (gcn.cpp:22-33) on CUDA float32 tensors (packed row-major)."""
        torch = _torch()
        x, w0, w1 = (t.contiguous() for t in (x, w0, w1))
        if w0.shape[0] != x.shape[1] or w1.shape[0] != w0.shape[1]:
            raise ValueError("dense_matmul: inner dimensions differ")
        out = torch.empty((x.shape[0], w1.shape[1]), dtype=torch.float32, device=x.device)
        _check(_lib.cbm_b200_gcn_forward(self._h, x.data_ptr(), x.shape[0], x.shape[1],
                                         w0.data_ptr(), w0.shape[1], w1.data_ptr(), w1.shape[1],
                                         out.data_ptr(), self._stream(stream)))
        return out

    def spmm_host_ptr(self, x_ptr, x_rows, x_cols, y_ptr, y_rows, y_cols, stream=None):
        _check(_lib.cbm_b200_spmm_host(self._h, x_ptr, x_rows, x_cols, y_ptr, y_rows, y_cols,
                                       self._stream(stream) if stream is not None else None))
