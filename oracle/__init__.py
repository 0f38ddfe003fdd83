"""TEST INFRASTRUCTURE ONLY — the parity oracle and the reference CPU path.

Importable only from tests/, ``__graft_entry__.smoke()`` and bench.py's
``cpu_baseline`` / ``--impl reference`` legs, as the checker or the timed CPU
baseline. The product package (``paper_2409_02208_b200``) never imports this.

Two native libraries back it, both built by ``oracle/Makefile``:

* ``oracle/liboracle.so`` — our plain-C restatement of the reference hot path
  (``oracle/cbm_oracle.c``; cites ``proj/src/kernels.cpp`` line by line).
* ``oracle/_ref/libcbmref.so`` — the UNMODIFIED reference library compiled from
  ``/root/reference/proj/src`` (f32 build) plus ``oracle/ref_capi.cpp``.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
VIRTUAL_PARENT = 0xFFFFFFFF

_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")


def _load(path: str) -> C.CDLL:
    if not os.path.exists(path):
        raise OSError(f"{path} missing: run `make -C oracle` (or __graft_entry__.build())")
    return C.CDLL(path)


# --------------------------------------------------------------------------
# Restated oracle (plain C)
# --------------------------------------------------------------------------
_orc = None


def restated() -> C.CDLL:
    global _orc
    if _orc is None:
        lib = _load(os.path.join(_HERE, "liboracle.so"))
        lib.oracle_spmm.argtypes = [C.c_uint32, C.c_uint32, _u32p, _u32p, _u64p, _u32p,
                                    _f32p, C.c_void_p, C.c_int, _f32p, C.c_uint64, _f32p,
                                    C.c_uint64]
        lib.oracle_csr_spmm.argtypes = [C.c_uint32, C.c_uint32, _u64p, _u32p, _f32p, _f32p,
                                        C.c_uint64, _f32p, C.c_uint64]
        lib.oracle_dense_matmul.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, _f32p, _f32p,
                                            _f32p]
        lib.oracle_random_dense.argtypes = [C.c_uint32, C.c_uint32, C.c_double, C.c_double,
                                            C.c_uint64, _f32p]
        lib.oracle_random_binary.argtypes = [C.c_uint32, C.c_uint32, C.c_double, C.c_uint64,
                                             _u64p, _u32p]
        lib.oracle_random_binary.restype = C.c_uint64
        lib.oracle_csr_spmm_f64.argtypes = [C.c_uint32, C.c_uint32, _u64p, _u32p, C.c_void_p,
                                            C.c_int, _f32p, C.c_uint64,
                                            np.ctypeslib.ndpointer(np.float64,
                                                                   flags="C_CONTIGUOUS"),
                                            C.c_uint64]
        lib.oracle_gen_graph.argtypes = [C.c_int, C.POINTER(C.c_double), C.c_uint64,
                                         C.POINTER(_OracleGraph)]
        lib.oracle_graph_free.argtypes = [C.POINTER(_OracleGraph)]
        lib.oracle_gen_dense.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_double,
                                         C.c_double, C.c_uint64, _f32p]
        _orc = lib
    return _orc


class _OracleGraph(C.Structure):
    _fields_ = [("n_rows", C.c_uint32), ("n_cols", C.c_uint32), ("nnz", C.c_uint64),
                ("row_ptr", C.POINTER(C.c_uint64)), ("col_idx", C.POINTER(C.c_uint32))]


_GRAPH_KINDS = {"community": 0, "pa_triangle": 1, "clique_overlay": 2}
_DENSE_KINDS = {"int": 1, "normal": 2, "glorot": 3}


def oracle_gen_graph(kind: str, params, seed: int):
    """Restated seeded graph generators (oracle/gen_oracle.c): returns
    (n, row_ptr u64[n+1], col_idx u32[nnz]) — the same CSR the product's
    generate_graph draws (pinned by tests/test_oracle_gen.py)."""
    if kind == "random_binary":
        rows, cols, dens = params
        rp, ci = oracle_random_binary(int(rows), int(cols), float(dens), seed)
        return int(rows), int(cols), rp, ci
    lib = restated()
    p = (C.c_double * len(params))(*[float(v) for v in params])
    g = _OracleGraph()
    rc = lib.oracle_gen_graph(_GRAPH_KINDS[kind], p, seed, C.byref(g))
    if rc != 0:
        raise RuntimeError(f"oracle_gen_graph({kind}) failed ({rc})")
    try:
        n = g.n_rows
        rp = np.ctypeslib.as_array(g.row_ptr, shape=(n + 1,)).copy()
        ci = (np.ctypeslib.as_array(g.col_idx, shape=(g.nnz,)).copy() if g.nnz
              else np.zeros(0, np.uint32))
    finally:
        lib.oracle_graph_free(C.byref(g))
    return n, g.n_cols if g.n_cols else n, rp, ci


def oracle_gen_dense(kind: str, rows: int, cols: int, seed: int, lo: float = -8.0,
                     hi: float = 8.0) -> np.ndarray:
    """Restated seeded dense operands: "int" (below(hi-lo+1)+lo), "normal"
    (Box–Muller N(0,1)), "glorot" (Glorot-uniform rows x cols weight)."""
    out = np.empty((rows, cols), np.float32)
    rc = restated().oracle_gen_dense(_DENSE_KINDS[kind], rows, cols, lo, hi, seed, out)
    if rc != 0:
        raise ValueError(f"oracle_gen_dense({kind}) failed")
    return out


def topo_order_from_parents(parent: np.ndarray) -> np.ndarray:
    """Any parents-first order (BFS by depth); the oracle's bits do not depend
    on which one (each update reads only its own, already final, parent)."""
    parent = np.asarray(parent, dtype=np.uint32)
    m = parent.shape[0]
    depth = np.full(m, -1, dtype=np.int64)
    roots = parent == VIRTUAL_PARENT
    depth[roots] = 0
    frontier = np.nonzero(roots)[0]
    order = np.argsort(np.where(roots, -1, parent.astype(np.int64)), kind="stable")
    par_sorted = parent[order]
    # CSR of children
    nr = int(roots.sum())
    ch_par = par_sorted[nr:].astype(np.int64)
    ch = order[nr:]
    ptr = np.searchsorted(ch_par, np.arange(m + 1))
    out = [frontier]
    while frontier.size:
        nxt = [ch[ptr[p]:ptr[p + 1]] for p in frontier]
        frontier = np.concatenate(nxt) if nxt else np.zeros(0, np.int64)
        if frontier.size:
            out.append(frontier)
    topo = np.concatenate(out).astype(np.uint32)
    if topo.shape[0] != m:
        raise ValueError("parent links contain a cycle")
    return topo


def oracle_spmm(cbm: "RefCbmArrays", x: np.ndarray) -> np.ndarray:
    """Restated spmm_into (proj/src/kernels.cpp:105-123), f32, no FMA."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    if x.shape[0] != cbm.n_cols:
        raise ValueError("spmm: inner dimensions differ")
    d = x.shape[1]
    y = np.empty((cbm.n_rows, d), dtype=np.float32)
    topo = cbm.topo_order if cbm.topo_order is not None else topo_order_from_parents(cbm.parent)
    scale = cbm.row_scale if cbm.normalized else None
    restated().oracle_spmm(cbm.n_rows, d, cbm.parent, topo, cbm.row_ptr, cbm.col_idx,
                           cbm.values,
                           scale.ctypes.data if scale is not None else None,
                           int(cbm.normalized), x, d, y, d)
    return y


def oracle_csr_spmm(row_ptr, col_idx, values, x) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float32)
    m = row_ptr.shape[0] - 1
    y = np.empty((m, x.shape[1]), dtype=np.float32)
    restated().oracle_csr_spmm(m, x.shape[1], np.ascontiguousarray(row_ptr, np.uint64),
                               np.ascontiguousarray(col_idx, np.uint32),
                               np.ascontiguousarray(values, np.float32), x, x.shape[1], y,
                               x.shape[1])
    return y


def oracle_exact_spmm(row_ptr, col_idx, x, scale=None, add_identity=False) -> np.ndarray:
    """A x (or S (A + I) S x) in double over the represented pattern (the
    graph's CSR): the yardstick when f32 sequential sums drift."""
    x = np.ascontiguousarray(x, np.float32)
    m = row_ptr.shape[0] - 1
    y = np.empty((m, x.shape[1]), np.float64)
    sc = np.ascontiguousarray(scale, np.float32) if scale is not None else None
    restated().oracle_csr_spmm_f64(m, x.shape[1], np.ascontiguousarray(row_ptr, np.uint64),
                                   np.ascontiguousarray(col_idx, np.uint32),
                                   sc.ctypes.data if sc is not None else None,
                                   int(add_identity), x, x.shape[1], y, x.shape[1])
    return y


def judge_parity(got, ref, tol, exact_fn=None, sample_cols=8):
    """SURVEY §8d Gate 2 with a fallback for long rows: pass when
    max|G-R|/max|R| <= tol against the reference R. Otherwise (the reference's
    own sequential f32 sums drift on rows of ~1e6 entries) `exact_fn(cols)`
    gives the double-precision product on a column sample; pass when the device
    result is within tol of it, and report how far the reference is from it."""
    got = np.asarray(got, np.float32)
    ref = np.asarray(ref, np.float32)
    den = float(np.abs(ref).max()) if ref.size else 0.0
    err = float(np.abs(got.astype(np.float64) - ref).max()) / den if den > 0 else 0.0
    out = {"ok": err <= tol, "mode": f"normwise max|G-R|/max|R| <= {tol:g}", "normwise_err": err}
    if err <= tol or exact_fn is None:
        return out
    d = got.shape[1]
    cols = np.unique(np.linspace(0, d - 1, min(d, sample_cols)).astype(np.int64))
    e = exact_fn(cols)
    den_e = float(np.abs(e).max()) or 1.0
    g_e = float(np.abs(got[:, cols].astype(np.float64) - e).max()) / den_e
    r_e = float(np.abs(ref[:, cols].astype(np.float64) - e).max()) / den_e
    out.update({"ok": g_e <= tol, "mode": f"normwise vs the f64 product <= {tol:g} "
                "(reference's own f32 drift exceeds tol)",
                "exact_err": g_e, "reference_exact_err": r_e, "exact_cols": cols.tolist()})
    return out


def oracle_dense_matmul(a, b) -> np.ndarray:
    a = np.ascontiguousarray(a, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    c = np.empty((a.shape[0], b.shape[1]), np.float32)
    restated().oracle_dense_matmul(a.shape[0], a.shape[1], b.shape[1], a, b, c)
    return c


def oracle_random_dense(rows, cols, lo, hi, seed) -> np.ndarray:
    out = np.empty((rows, cols), np.float32)
    restated().oracle_random_dense(rows, cols, lo, hi, seed, out)
    return out


def oracle_random_binary(rows, cols, density, seed):
    rp = np.zeros(rows + 1, np.uint64)
    ci = np.zeros(max(1, rows * cols), np.uint32)
    nnz = restated().oracle_random_binary(rows, cols, density, seed, rp, ci)
    return rp, ci[:nnz].copy()


def oracle_gcn_forward(cbm: "RefCbmArrays", x, w0, w1) -> np.ndarray:
    """gcn_forward (proj/src/gcn.cpp:22-33) from restated pieces."""
    h = oracle_dense_matmul(x, w0)
    h = oracle_spmm(cbm, h)
    h = np.where(h < 0, np.float32(0), h)   # relu_inplace (dense.cpp:51-54): -0.0 stays
    h = oracle_spmm(cbm, h)
    return oracle_dense_matmul(h, w1)


# --------------------------------------------------------------------------
# Reference library (compiled from /root/reference sources)
# --------------------------------------------------------------------------
@dataclass
class RefCbmArrays:
    """Plain arrays of a reference CbmMatrix (builder.hpp:66-74)."""
    n_rows: int
    n_cols: int
    alpha: int
    normalized: bool
    parent: np.ndarray
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray
    row_scale: np.ndarray | None = None
    topo_order: np.ndarray | None = None
    branch_ptr: np.ndarray | None = None
    extra: dict = field(default_factory=dict)


_ref = None


def ref_available() -> bool:
    return os.path.exists(os.path.join(_HERE, "_ref", "libcbmref.so"))


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        lib = _load(os.path.join(_HERE, "_ref", "libcbmref.so"))
        vp = C.c_void_p
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_csr_from_arrays.restype = vp
        lib.ref_csr_from_arrays.argtypes = [C.c_uint32, C.c_uint32, _u64p, _u32p]
        for fn, args in (("ref_gen_random_binary", [C.c_uint32, C.c_uint32, C.c_double, C.c_uint64]),
                         ("ref_gen_block_graph", [C.c_uint32] * 3),
                         ("ref_gen_community_graph", [C.c_uint32] * 4 + [C.c_uint64]),
                         ("ref_gen_citation_graph", [C.c_uint32, C.c_uint64, C.c_uint64])):
            getattr(lib, fn).restype = vp
            getattr(lib, fn).argtypes = args
        lib.ref_csr_dims.argtypes = [vp, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                     C.POINTER(C.c_uint64)]
        lib.ref_csr_export.argtypes = [vp, _u64p, _u32p]
        lib.ref_csr_free.argtypes = [vp]
        lib.ref_build_cbm.restype = vp
        lib.ref_build_cbm.argtypes = [vp, C.c_uint64, C.c_int, C.c_int]
        lib.ref_cbm_from_arrays.restype = vp
        lib.ref_cbm_from_arrays.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, C.c_int, _u32p,
                                            _u64p, _u32p, _f32p, C.c_void_p]
        lib.ref_cbm_dims.argtypes = [vp, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                     C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                     C.POINTER(C.c_int), C.POINTER(C.c_uint64)]
        lib.ref_cbm_export.argtypes = [vp, _u32p, _u32p, _u64p, _u64p, _u32p, _f32p, C.c_void_p]
        lib.ref_cbm_free.argtypes = [vp]
        lib.ref_count_ops.argtypes = [vp, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        lib.ref_memory_footprint.restype = C.c_uint64
        lib.ref_memory_footprint.argtypes = [vp]
        lib.ref_reconstruct_rows.restype = C.c_uint64
        lib.ref_reconstruct_rows.argtypes = [vp, C.c_void_p, C.c_void_p]
        lib.ref_save_cbm.argtypes = [vp, C.c_char_p]
        lib.ref_load_cbm.restype = vp
        lib.ref_load_cbm.argtypes = [C.c_char_p]
        lib.ref_spmm.argtypes = [vp, _f32p, C.c_uint32, C.c_uint32, _f32p, C.c_int]
        lib.ref_spmv.argtypes = [vp, _f32p, C.c_uint32, _f32p, C.c_int]
        lib.ref_spmm_sequential.argtypes = [vp, _f32p, C.c_uint32, C.c_uint32, _f32p]
        lib.ref_csr_real.restype = vp
        lib.ref_csr_real.argtypes = [vp, C.c_int]
        lib.ref_csr_real_free.argtypes = [vp]
        lib.ref_csr_spmm.argtypes = [vp, _f32p, C.c_uint32, C.c_uint32, _f32p, C.c_int]
        lib.ref_time.restype = C.c_double
        lib.ref_time.argtypes = [C.c_int, vp, _f32p, C.c_uint32, C.c_uint32, C.c_int, C.c_int,
                                 C.c_double, C.POINTER(C.c_int)]
        lib.ref_random_dense.argtypes = [C.c_uint32, C.c_uint32, C.c_double, C.c_double,
                                         C.c_uint64, _f32p]
        lib.ref_gcn_seeded.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, _f32p,
                                       _f32p]
        lib.ref_gcn_forward.argtypes = [vp, _f32p, C.c_uint32, C.c_uint32, _f32p, C.c_uint32,
                                        _f32p, C.c_uint32, _f32p, C.c_int]
        lib.ref_gcn_forward_csr.argtypes = lib.ref_gcn_forward.argtypes
        lib.ref_hw_threads.restype = C.c_int
        _ref = lib
    return _ref


def _err(lib):
    return lib.ref_last_error().decode()


class RefError(Exception):
    pass


def _check(lib, rc):
    if rc == 1:
        raise ValueError(_err(lib))      # std::invalid_argument
    if rc != 0:
        raise RefError(_err(lib))


class RefCsr:
    """Reference CsrBinaryMatrix (csr.hpp:14-40) owned by the reference library."""

    def __init__(self, handle):
        if not handle:
            raise ValueError(_err(ref()))
        self.h = handle

    @classmethod
    def from_arrays(cls, n_rows, n_cols, row_ptr, col_idx):
        lib = ref()
        return cls(lib.ref_csr_from_arrays(n_rows, n_cols,
                                           np.ascontiguousarray(row_ptr, np.uint64),
                                           np.ascontiguousarray(col_idx, np.uint32)))

    @classmethod
    def random_binary(cls, rows, cols, density, seed):
        return cls(ref().ref_gen_random_binary(rows, cols, density, seed))

    @classmethod
    def block_graph(cls, blocks, copies, nnz):
        return cls(ref().ref_gen_block_graph(blocks, copies, nnz))

    @classmethod
    def community_graph(cls, comms, size, base, noise, seed):
        return cls(ref().ref_gen_community_graph(comms, size, base, noise, seed))

    @classmethod
    def citation_graph(cls, nodes, edges, seed):
        return cls(ref().ref_gen_citation_graph(nodes, edges, seed))

    def arrays(self):
        lib = ref()
        r, c, z = C.c_uint32(), C.c_uint32(), C.c_uint64()
        lib.ref_csr_dims(self.h, C.byref(r), C.byref(c), C.byref(z))
        rp = np.zeros(r.value + 1, np.uint64)
        ci = np.zeros(max(1, z.value), np.uint32)
        lib.ref_csr_export(self.h, rp, ci)
        return r.value, c.value, rp, ci[:z.value].copy()

    def __del__(self):
        if getattr(self, "h", None) and _ref is not None:
            _ref.ref_csr_free(self.h)
            self.h = None


class RefCbm:
    """Reference CbmMatrix owned by the reference library."""

    def __init__(self, handle):
        if not handle:
            raise ValueError(_err(ref()))
        self.h = handle

    @classmethod
    def build(cls, csr: RefCsr, alpha=0, threads=1, normalized=False):
        return cls(ref().ref_build_cbm(csr.h, alpha, threads, int(normalized)))

    @classmethod
    def from_arrays(cls, a: RefCbmArrays):
        s = np.ascontiguousarray(a.row_scale, np.float32) if a.normalized else None
        return cls(ref().ref_cbm_from_arrays(
            a.n_rows, a.n_cols, a.alpha, int(a.normalized),
            np.ascontiguousarray(a.parent, np.uint32), np.ascontiguousarray(a.row_ptr, np.uint64),
            np.ascontiguousarray(a.col_idx, np.uint32), np.ascontiguousarray(a.values, np.float32),
            s.ctypes.data if s is not None else None))

    @classmethod
    def load(cls, path):
        return cls(ref().ref_load_cbm(str(path).encode()))

    def save(self, path):
        lib = ref()
        _check(lib, lib.ref_save_cbm(self.h, str(path).encode()))

    def arrays(self) -> RefCbmArrays:
        lib = ref()
        m, n, z, al, nm, nr = (C.c_uint32(), C.c_uint32(), C.c_uint64(), C.c_uint64(),
                               C.c_int(), C.c_uint64())
        lib.ref_cbm_dims(self.h, *(C.byref(v) for v in (m, n, z, al, nm, nr)))
        M, Z = m.value, z.value
        parent = np.zeros(M, np.uint32)
        topo = np.zeros(M, np.uint32)
        bp = np.zeros(nr.value + 1, np.uint64)
        rp = np.zeros(M + 1, np.uint64)
        ci = np.zeros(max(Z, 1), np.uint32)
        va = np.zeros(max(Z, 1), np.float32)
        rs = np.zeros(max(M, 1), np.float32) if nm.value else None
        lib.ref_cbm_export(self.h, parent, topo, bp, rp, ci, va,
                           rs.ctypes.data if rs is not None else None)
        return RefCbmArrays(M, n.value, al.value, bool(nm.value), parent, rp, ci[:Z].copy(),
                            va[:Z].copy(), rs[:M].copy() if rs is not None else None, topo, bp)

    def count_ops(self):
        a, b = C.c_uint64(), C.c_uint64()
        ref().ref_count_ops(self.h, C.byref(a), C.byref(b))
        return a.value, b.value

    def memory_footprint(self):
        return ref().ref_memory_footprint(self.h)

    def dims(self):
        lib = ref()
        m, n, z, al, nm, nr = (C.c_uint32(), C.c_uint32(), C.c_uint64(), C.c_uint64(),
                               C.c_int(), C.c_uint64())
        lib.ref_cbm_dims(self.h, *(C.byref(v) for v in (m, n, z, al, nm, nr)))
        return m.value, n.value, z.value

    def reconstruct_rows(self):
        lib = ref()
        m = self.dims()[0]
        nnz = lib.ref_reconstruct_rows(self.h, None, None)
        rp = np.zeros(m + 1, np.uint64)
        ci = np.zeros(max(1, nnz), np.uint32)
        lib.ref_reconstruct_rows(self.h, rp.ctypes.data, ci.ctypes.data)
        return rp, ci[:nnz].copy()

    def spmm(self, x, threads=1):
        lib = ref()
        x = np.ascontiguousarray(x, np.float32)
        y = np.zeros((self.dims()[0], x.shape[1]), np.float32)
        _check(lib, lib.ref_spmm(self.h, x, x.shape[0], x.shape[1], y, threads))
        return y

    def spmv(self, v, threads=1):
        lib = ref()
        v = np.ascontiguousarray(v, np.float32).reshape(-1, 1)
        y = np.zeros((self.dims()[0], 1), np.float32)
        _check(lib, lib.ref_spmv(self.h, v, v.shape[0], y, threads))
        return y

    def spmm_sequential(self, x):
        lib = ref()
        x = np.ascontiguousarray(x, np.float32)
        y = np.zeros((self.dims()[0], x.shape[1]), np.float32)
        _check(lib, lib.ref_spmm_sequential(self.h, x, x.shape[0], x.shape[1], y))
        return y

    def time_spmm(self, x, threads, runs, min_seconds=0.0, kind=0):
        """Mean seconds per reference spmm_into (kind 0) or spmv_into (kind 2)."""
        lib = ref()
        x = np.ascontiguousarray(x, np.float32)
        done = C.c_int()
        t = lib.ref_time(kind, self.h, x, x.shape[0], x.shape[1], threads, runs, min_seconds,
                         C.byref(done))
        if t < 0:
            raise RefError(_err(lib))
        return t, done.value

    def time_spmv(self, v, threads, runs, min_seconds=0.0):
        return self.time_spmm(v, threads, runs, min_seconds, kind=2)

    def gcn_forward(self, x, w0, w1, threads=1):
        lib = ref()
        x = np.ascontiguousarray(x, np.float32)
        w0 = np.ascontiguousarray(w0, np.float32)
        w1 = np.ascontiguousarray(w1, np.float32)
        out = np.zeros((x.shape[0], w1.shape[1]), np.float32)
        _check(lib, lib.ref_gcn_forward(self.h, x, x.shape[0], x.shape[1], w0, w0.shape[1], w1,
                                        w1.shape[1], out, threads))
        return out

    def __del__(self):
        if getattr(self, "h", None) and _ref is not None:
            _ref.ref_cbm_free(self.h)
            self.h = None


class RefCsrReal:
    """Reference CSR baseline operator: to_real(A) or normalized_adjacency_csr(A)."""

    def __init__(self, csr: RefCsr, normalized: bool):
        lib = ref()
        self.h = lib.ref_csr_real(csr.h, int(normalized))
        if not self.h:
            raise ValueError(_err(lib))

    def spmm(self, x, n_rows, threads=1):
        lib = ref()
        x = np.ascontiguousarray(x, np.float32)
        y = np.zeros((n_rows, x.shape[1]), np.float32)
        _check(lib, lib.ref_csr_spmm(self.h, x, x.shape[0], x.shape[1], y, threads))
        return y

    def time_spmm(self, x, threads, runs, min_seconds=0.0):
        lib = ref()
        x = np.ascontiguousarray(x, np.float32)
        done = C.c_int()
        t = lib.ref_time(1, self.h, x, x.shape[0], x.shape[1], threads, runs, min_seconds,
                         C.byref(done))
        if t < 0:
            raise RefError(_err(lib))
        return t, done.value

    def __del__(self):
        if getattr(self, "h", None) and _ref is not None:
            _ref.ref_csr_real_free(self.h)
            self.h = None


def ref_random_dense(rows, cols, lo, hi, seed):
    out = np.zeros((rows, cols), np.float32)
    ref().ref_random_dense(rows, cols, lo, hi, seed, out)
    return out


def ref_gcn_seeded(f, h, c, seed):
    w0 = np.zeros((f, h), np.float32)
    w1 = np.zeros((h, c), np.float32)
    ref().ref_gcn_seeded(f, h, c, seed, w0, w1)
    return w0, w1
