"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref).

TEST INFRASTRUCTURE ONLY. Run in the build container (needs oracle/_ref, i.e.
/root/reference at build time):  python oracle/make_golden.py

Every fixture stores the input pattern, the reference-built CBM (builder.cpp
output, f32 build), the operand and the reference product (spmm_into /
spmv_into / gcn_forward), so tests can pin both our C restatement and the
GPU path without the reference present. The instances are the reference's
own known-answer and seeded cases (proj/tests/test_kernels.cpp,
proj/tests/acceptance.cpp), regenerated through its generators
(proj/tests/oracles.hpp) and UniformRng streams.
"""
from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests",
                   "golden")


class Rng:
    """UniformRng (prng.hpp) via the restated mt19937_64, for dims draws."""

    def __init__(self, seed):
        import ctypes as C
        self.lib = O.restated()
        self.buf = (C.c_uint64 * 313)()
        self.lib.oracle_rng_seed.argtypes = [C.c_void_p, C.c_uint64]
        self.lib.oracle_rng_bits.argtypes = [C.c_void_p]
        self.lib.oracle_rng_bits.restype = C.c_uint64
        self.lib.oracle_rng_unit.argtypes = [C.c_void_p]
        self.lib.oracle_rng_unit.restype = C.c_double
        self.lib.oracle_rng_seed(self.buf, seed)

    def below(self, n):
        return int(self.lib.oracle_rng_bits(self.buf) % n) if n else 0

    def unit(self):
        return float(self.lib.oracle_rng_unit(self.buf))


def csr_from_rows(n_cols, rows):
    rp = [0]
    ci = []
    for r in rows:
        ci.extend(sorted(r))
        rp.append(len(ci))
    return O.RefCsr.from_arrays(len(rows), n_cols, np.array(rp, np.uint64),
                                np.array(ci, np.uint32))


def pack(name, csr: O.RefCsr, cbm: O.RefCbm, x, y, **extra):
    m, n, rp, ci = csr.arrays()
    a = cbm.arrays()
    d = dict(a_n_rows=m, a_n_cols=n, a_row_ptr=rp, a_col_idx=ci,
             n_rows=a.n_rows, n_cols=a.n_cols, alpha=a.alpha, normalized=int(a.normalized),
             parent=a.parent, topo_order=a.topo_order, branch_ptr=a.branch_ptr,
             row_ptr=a.row_ptr, col_idx=a.col_idx, values=a.values,
             row_scale=a.row_scale if a.normalized else np.zeros(0, np.float32),
             x=x, y=y)
    mult, upd = cbm.count_ops()
    d["ops"] = np.array([mult, upd], np.uint64)
    d.update(extra)
    return name, d


def cases():
    # test_kernels.cpp:45-54 — identical rows, spmv u = (5, 5)
    a = csr_from_rows(3, [[0, 1], [0, 1]])
    c = O.RefCbm.build(a, 0)
    v = np.array([[2.0], [3.0], [5.0]], np.float32)
    yield pack("identical_rows", a, c, v, c.spmv(v), kind=np.array("spmv"))
    # test_kernels.cpp:56-66 — zero matrix and identity pattern
    a = csr_from_rows(3, [[], [], []])
    c = O.RefCbm.build(a, 0)
    v = np.array([[1.0], [2.0], [3.0]], np.float32)
    yield pack("zero", a, c, v, c.spmv(v), kind=np.array("spmv"))
    a = csr_from_rows(3, [[0], [1], [2]])
    c = O.RefCbm.build(a, 0)
    yield pack("identity", a, c, v, c.spmv(v), kind=np.array("spmv"))
    # test_kernels.cpp:68-73 — identity operand densifies A
    a = O.RefCsr.random_binary(12, 12, 0.3, 7)
    c = O.RefCbm.build(a, 0)
    eye = np.eye(12, dtype=np.float32)
    yield pack("identity_operand", a, c, eye, c.spmm(eye), kind=np.array("spmm"))
    # test_kernels.cpp:94-99 — normalized two-node path -> all 0.5
    a = csr_from_rows(2, [[1], [0]])
    c = O.RefCbm.build(a, 0, normalized=True)
    eye = np.eye(2, dtype=np.float32)
    yield pack("two_node_normalized", a, c, eye, c.spmm(eye), kind=np.array("spmm"))
    # test_kernels.cpp:75-92 — 30 random instances x alpha {0,1,2,4} (first 8 kept)
    for seed in range(1, 9):
        dims = Rng(seed * 7919)
        m, n, p = 1 + dims.below(16), 1 + dims.below(16), 1 + dims.below(5)
        a = O.RefCsr.random_binary(m, n, 0.25, seed)
        b = O.ref_random_dense(n, p, -1.0, 1.0, seed + 17)
        for alpha in (0, 1, 2, 4):
            c = O.RefCbm.build(a, alpha)
            yield pack(f"random_s{seed}_a{alpha}", a, c, b, c.spmm(b), kind=np.array("spmm"))
    # test_kernels.cpp:101-114 — normalized random (first 6 seeds) x alpha {0,2,8}
    for seed in range(50, 56):
        dims = Rng(seed)
        n, p = 1 + dims.below(32), 1 + dims.below(6)
        a = O.RefCsr.random_binary(n, n, 0.2, seed)
        b = O.ref_random_dense(n, p, -1.0, 1.0, seed + 3)
        for alpha in (0, 2, 8):
            c = O.RefCbm.build(a, alpha, normalized=True)
            yield pack(f"normalized_s{seed}_a{alpha}", a, c, b, c.spmm(b), kind=np.array("spmm"))
    # acceptance.cpp:198-214 — block graph 100 x 50 x 20 (pattern + CBM only, d = 3)
    a = O.RefCsr.block_graph(100, 50, 20)
    c = O.RefCbm.build(a, 0)
    b = O.ref_random_dense(2000, 3, -1.0, 1.0, 5)
    yield pack("block_graph", a, c, b, c.spmm(b), kind=np.array("spmm"))
    # acceptance.cpp:175-190 — community graph, integer operand (bit-exact gate)
    a = O.RefCsr.community_graph(50, 40, 40, 1, 0xC0FFEE)
    c = O.RefCbm.build(a, 0)
    rng = np.random.default_rng(0xC0FFEE)
    b = rng.integers(-8, 9, size=(2000, 8)).astype(np.float32)
    yield pack("community_int", a, c, b, c.spmm(b), kind=np.array("spmm"))
    cn = O.RefCbm.build(a, 0, normalized=True)
    bn = O.ref_random_dense(2000, 5, -1.0, 1.0, 11)
    yield pack("community_normalized", a, cn, bn, cn.spmm(bn), kind=np.array("spmm"))
    # acceptance.cpp:268-287 — 2-layer GCN on a small normalized graph
    a = O.RefCsr.random_binary(40, 40, 0.15, 0x6D00)
    cn = O.RefCbm.build(a, 2, normalized=True)
    w0, w1 = O.ref_gcn_seeded(24, 16, 7, 0x6E00)
    x = O.ref_random_dense(40, 24, -1.0, 1.0, 0x6F00)
    yield pack("gcn_small", a, cn, x, cn.gcn_forward(x, w0, w1), kind=np.array("gcn"), w0=w0,
               w1=w1)


def main():
    os.makedirs(OUT, exist_ok=True)
    n = 0
    total = 0
    for name, d in cases():
        path = os.path.join(OUT, name + ".npz")
        np.savez_compressed(path, **d)
        total += os.path.getsize(path)
        n += 1
    print(f"wrote {n} fixtures, {total / 1024:.0f} KiB, into {OUT}")


if __name__ == "__main__":
    main()
