"""GPU parity: the sm_100a path (through the C ABI) against the oracle.

Bar (north_star): bit-exact against the reference in the order-faithful mode
for ANY X, and in the default mode for the binary matrix on integer-valued X;
normwise max|G-R|/max|R| <= 1e-5 otherwise (default mode: long rows split,
rows flattened, normalized products fused into one FMA).
"""
import numpy as np
import pytest

import oracle as O
import paper_2409_02208_b200 as P
from helpers import (assert_bitwise, golden_cbm, golden_names, load_golden, normwise_err,
                     oracle_arrays)

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

TOL = 1e-5  # north_star: "within 1e-5 relative (fp32) for Gaussian X", normwise


@pytest.fixture(scope="module")
def dev():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch.device("cuda:0")


def lane_groups(d):
    """Widths the default mode runs with H > 1 lane groups (several deltas per
    warp instruction, summation order changed): 4 <= d <= 64, d % 4 == 0."""
    return 4 <= d <= 64 and d % 4 == 0


def tiled(info, d):
    """The default mode's tiled path (d >= 32) sums staged deltas, then cold
    deltas, then the parent: order changed, integer sums unchanged."""
    return bool(info["tile_active"]) and d >= 32


def gpu_spmm(c, x, dev, **opt):
    opt.setdefault("tile", 0)  # the streaming kernel; tests/test_tile_gpu.py covers tile=1/-1
    d = P.DeviceCbm(c, **opt)
    xt = torch.from_numpy(np.ascontiguousarray(x, np.float32)).to(dev)
    y = d.spmm(xt)
    torch.cuda.synchronize()
    return y.cpu().numpy(), d


# ------------------------------------------------------------- golden pins
@pytest.mark.parametrize("name", golden_names())
@pytest.mark.parametrize("faithful", [True, False])
def test_golden_fixture_bitwise(name, faithful, dev):
    g = load_golden(name)
    c = golden_cbm(g)
    kind = str(g["kind"])
    if kind == "gcn":
        pytest.skip("GCN fixture is exercised by the GCN tests")
    if kind == "spmv":
        d = P.DeviceCbm(c, order_faithful=faithful)
        v = torch.from_numpy(g["x"]).to(dev)
        got = d.spmv(v).cpu().numpy()
        info = d.info()
    else:
        got, d = gpu_spmm(c, g["x"], dev, order_faithful=faithful)
        info = d.info()
    split = info["n_chunk_items"] > 0 or info["n_flattened"] > 0
    split = split or (not faithful and kind != "spmv" and tiled(info, g["x"].shape[1]))
    integer = np.array_equal(g["x"], np.round(g["x"]))
    fused = c.is_normalized and not faithful  # default mode: fma(x, +-s_c, acc)
    grouped = not faithful and kind != "spmv" and lane_groups(g["x"].shape[1])
    if fused or ((split or grouped) and not (integer and not c.is_normalized)):
        # chunked / flattened rows change the summation order, the fused
        # normalized product the rounding: tolerance, not bits
        assert normwise_err(got, g["y"]) <= TOL, name
    else:
        assert_bitwise(got, g["y"], name)


# ------------------------------------------------------------- known answers
def test_known_answers(dev):
    # test_kernels.cpp:45-54
    c = P.build_cbm(P.CsrBinaryMatrix.from_rows(3, [[0, 1], [0, 1]]), 0)
    d = P.DeviceCbm(c)
    u = d.spmv(torch.tensor([[2.0], [3.0], [5.0]], device=dev))
    assert u.cpu().numpy().ravel().tolist() == [5.0, 5.0]
    # :56-66 zero and identity
    zero = P.DeviceCbm(P.build_cbm(P.CsrBinaryMatrix.from_rows(3, [[], [], []]), 0))
    v = torch.tensor([[1.0], [2.0], [3.0]], device=dev)
    assert zero.spmv(v).abs().sum().item() == 0.0
    eye = P.DeviceCbm(P.build_cbm(P.CsrBinaryMatrix.from_rows(3, [[0], [1], [2]]), 0))
    assert torch.equal(eye.spmv(v), v)
    # :68-73 identity operand densifies A
    rp, ci = O.oracle_random_binary(12, 12, 0.3, 7)
    a = P.CsrBinaryMatrix(12, 12, rp, ci)
    got, _ = gpu_spmm(P.build_cbm(a, 0), np.eye(12, dtype=np.float32), dev)
    assert np.array_equal(got, a.dense())
    # :94-99 normalized two-node path
    c2 = P.build_cbm_normalized(P.CsrBinaryMatrix.from_rows(2, [[1], [0]]), 0)
    got, _ = gpu_spmm(c2, np.eye(2, dtype=np.float32), dev)
    assert np.allclose(got, 0.5, rtol=0, atol=1e-7)


def test_shape_errors_mirror_reference(dev):
    # test_kernels.cpp:245-251, kernels.cpp:11-14,107-109
    d = P.DeviceCbm(P.build_cbm(P.CsrBinaryMatrix.from_rows(3, [[0], [1], [2]]), 0))
    with pytest.raises(ValueError, match="spmm: inner dimensions differ"):
        d.spmm(torch.zeros((4, 2), device=dev))
    with pytest.raises(ValueError, match="spmm: output has the wrong shape"):
        d.spmm_into(torch.zeros((3, 2), device=dev), torch.zeros((2, 2), device=dev))
    with pytest.raises(ValueError, match="spmv: operand must be a single column"):
        d.spmv_into(torch.zeros((3, 2), device=dev), torch.zeros((3, 1), device=dev))
    with pytest.raises(ValueError, match="spmv: inner dimensions differ"):
        d.spmv(torch.zeros((4, 1), device=dev))
    # the gather kernels address X rows with a 32-bit byte pitch (checked
    # before any device work, so the buffers are never touched)
    x, y = torch.zeros((3, 2), device=dev), torch.zeros((3, 2), device=dev)
    rc = P._lib.cbm_b200_spmm(d._h, x.data_ptr(), 3, 2, 1 << 30, y.data_ptr(), 3, 2, 2, None)
    assert rc == P.EINVAL and b"below 2^30" in P._lib.cbm_b200_last_error()


# ------------------------------------------------------------- seeded suites
def _suite(normalized, n_cases, seed0):
    rng = np.random.default_rng(seed0)
    for k in range(n_cases):
        n = int(rng.integers(1, 64))
        m = n if normalized else int(rng.integers(1, 64))
        dens = float(rng.uniform(0.05, 0.5))
        rp, ci = O.oracle_random_binary(m, n, dens, seed0 + k)
        a = P.CsrBinaryMatrix(m, n, rp, ci)
        alpha = int(rng.choice([0, 1, 2, 4, 8]))
        c = (P.build_cbm_normalized if normalized else P.build_cbm)(a, alpha)
        d = int(rng.choice([1, 2, 3, 5, 7, 8, 16, 33, 64, 100, 128, 130, 256]))
        x = O.oracle_random_dense(n, d, -1.0, 1.0, seed0 + 1000 + k)
        yield k, c, x


@pytest.mark.parametrize("kernel", ["auto", "scalar"])
@pytest.mark.parametrize("normalized", [False, True])
def test_random_suite_bitwise(normalized, kernel, dev):
    """Reference suites (test_kernels.cpp:75-114 style, all d paths, all kernel
    families): order-faithful is bit-identical; the default mode is
    bit-identical unless it flattened/chunked a row, then within tolerance."""
    for k, c, x in _suite(normalized, 60, 9000 + 100 * normalized):
        want = O.oracle_spmm(oracle_arrays(c), x)
        got, _ = gpu_spmm(c, x, dev, kernel=kernel, order_faithful=True)
        assert_bitwise(got, want, f"case {k} d={x.shape[1]}")
        got, h = gpu_spmm(c, x, dev, kernel=kernel)
        info = h.info()
        # default mode: spmv (d = 1) sums a row's deltas lane-parallel
        if (info["n_flattened"] or info["n_chunk_items"] or normalized or x.shape[1] == 1
                or lane_groups(x.shape[1]) or tiled(info, x.shape[1])):
            assert normwise_err(got, want) <= TOL, f"case {k}"
        else:
            assert_bitwise(got, want, f"default case {k}")


@pytest.mark.parametrize("normalized", [False, True])
def test_flattened_rows(normalized, dev):
    """Rows summed directly instead of through their parent (flatten_gain):
    integer X stays bit-exact for the binary matrix, Gaussian X within 1e-5."""
    a = P.generate_graph("community", [3000, 100, 0.3, 0.002], 23)
    c = (P.build_cbm_normalized if normalized else P.build_cbm)(a, 0, threads=8)
    for gain in (4, 1000):
        for kind in ("int", "normal"):
            x = P.generate_dense(kind, 3000, 128, 24, -8, 8)
            got, h = gpu_spmm(c, x, dev, flatten_gain=gain)
            assert h.info()["n_flattened"] > 0
            want = O.oracle_spmm(oracle_arrays(c), x)
            if kind == "int" and not normalized:
                assert_bitwise(got, want, f"flatten gain={gain}")
            else:
                assert normwise_err(got, want) <= TOL


@pytest.mark.parametrize("kernel", ["auto", "scalar"])
@pytest.mark.parametrize("normalized", [False, True])
def test_split_rows_integer_bitexact_and_gaussian_tolerance(normalized, kernel, dev):
    """Force every long row through the CHUNK path (split_threshold=4, chunk=2)."""
    rng = np.random.default_rng(77)
    for k in range(12):
        n = int(rng.integers(20, 200))
        a = P.generate_graph("community", [n, max(4, n // 5), 0.6, 0.05], 300 + k)
        c = (P.build_cbm_normalized if normalized else P.build_cbm)(a, 0)
        d = int(rng.choice([3, 8, 64, 128, 160]))
        xi = P.generate_dense("int", n, d, 50 + k, -8, 8)
        got, h = gpu_spmm(c, xi, dev, split_threshold=4, chunk=2, kernel=kernel)
        if c.nnz:
            assert h.info()["n_chunk_items"] > 0 or np.diff(c.row_ptr).max() <= 4
        want = O.oracle_spmm(oracle_arrays(c), xi)
        if normalized:
            assert normwise_err(got, want) <= TOL
        else:
            assert_bitwise(got, want, f"split int case {k}")
        xg = P.generate_dense("normal", n, d, 70 + k)
        got, _ = gpu_spmm(c, xg, dev, split_threshold=4, chunk=2, kernel=kernel)
        assert normwise_err(got, O.oracle_spmm(oracle_arrays(c), xg)) <= TOL


def test_column_slab_strides_and_repeat_calls(dev):
    """ldx/ldy > width (a column shard of a wider matrix), repeated calls reuse
    the self-resetting counters and epoch flags."""
    a = P.generate_graph("pa_triangle", [3000, 2, 0.3], 11)
    c = P.build_cbm_normalized(a, 0)
    d = P.DeviceCbm(c, order_faithful=True)
    full = P.generate_dense("normal", 3000, 200, 12)
    xt = torch.from_numpy(full).to(dev)
    want = O.oracle_spmm(oracle_arrays(c), full)
    for c0, w in ((0, 64), (64, 64), (128, 72), (4, 4), (1, 3)):
        y = torch.zeros((3000, 200), device=dev)
        d.spmm_into(xt[:, c0:c0 + w], y[:, c0:c0 + w])
        torch.cuda.synchronize()
        assert_bitwise(y[:, c0:c0 + w].cpu().numpy(), want[:, c0:c0 + w], f"slab {c0}+{w}")
    first = d.spmm(xt).cpu().numpy()
    for _ in range(50):
        again = d.spmm(xt)
    torch.cuda.synchronize()
    assert_bitwise(again.cpu().numpy(), first, "repeat")
    assert_bitwise(first, want, "full")


def test_prescale_modes_identical(dev):
    a = P.generate_graph("community", [2000, 100, 0.5, 0.001], 21)
    c = P.build_cbm_normalized(a, 0)
    x = P.generate_dense("normal", 2000, 128, 22)
    want = O.oracle_spmm(oracle_arrays(c), x)
    for ps in (0, 1, -1):
        got, _ = gpu_spmm(c, x, dev, prescale=ps, order_faithful=True)
        assert_bitwise(got, want, f"prescale={ps}")


def test_host_buffer_entry_point(dev):
    a = P.generate_graph("community", [1024, 64, 0.5, 0.001], 31)
    c = P.build_cbm(a, 0)
    d = P.DeviceCbm(c)
    for width in (64, 7):
        x = P.generate_dense("int", 1024, width, 32, -8, 8)
        assert_bitwise(d.spmm_host(x), O.oracle_spmm(oracle_arrays(c), x), f"host d={width}")


def test_empty_and_degenerate_shapes(dev):
    c = P.build_cbm(P.CsrBinaryMatrix.from_rows(5, [[], [], []]), 0)
    d = P.DeviceCbm(c)
    y = d.spmm(torch.ones((5, 0), device=dev))
    assert y.shape == (3, 0)
    y = d.spmm(torch.ones((5, 4), device=dev))
    assert y.abs().sum().item() == 0.0


# ------------------------------------------------------------- configs
def test_cfg0_full_size_integer_bitexact(dev):
    """cfg[0]: n=4096, 64 communities of 64, p=0.5/0.001, X int in [-8,8], d=64."""
    a = P.generate_graph("community", [4096, 64, 0.5, 0.001], 0xC0F60000)
    c = P.build_cbm(a, 0, threads=8)
    x = P.generate_dense("int", 4096, 64, 0xC0F61000, -8, 8)
    want = O.oracle_spmm(oracle_arrays(c), x)
    for faithful in (True, False):
        for kernel in ("auto", "scalar"):
            got, _ = gpu_spmm(c, x, dev, order_faithful=faithful, kernel=kernel)
            assert_bitwise(got, want, f"cfg0 faithful={faithful} kernel={kernel}")


@pytest.mark.parametrize("kernel", ["auto", "scalar"])
def test_cfg1_full_size_gaussian(kernel, dev):
    """cfg[1]: n=19,717 normalized, X N(0,1), d=512: order-faithful is
    bit-exact, the default split mode within 1e-5 normwise."""
    a = P.generate_graph("pa_triangle", [19717, 2, 0.3], 0xC0F60001)
    c = P.build_cbm_normalized(a, 0, threads=8)
    x = P.generate_dense("normal", 19717, 512, 0xC0F61001)
    want = O.oracle_spmm(oracle_arrays(c), x)
    got, _ = gpu_spmm(c, x, dev, order_faithful=True, kernel=kernel)
    assert_bitwise(got, want, "cfg1 faithful")
    got, _ = gpu_spmm(c, x, dev, kernel=kernel)
    assert normwise_err(got, want) <= TOL


def test_deep_merge_trees(dev):
    """Rows with thousands of deltas split into 2-delta chunks: three levels of
    fan-in-32 MERGE items; integer X stays bit-exact."""
    a = P.generate_graph("community", [3000, 3000, 0.9, 0.0], 41)
    c = P.build_cbm(a, 0, threads=8)
    x = P.generate_dense("int", 3000, 72, 42, -8, 8)
    got, h = gpu_spmm(c, x, dev, split_threshold=4, chunk=2)
    info = h.info()
    assert info["n_chunk_items"] > 1000 and info["max_row_deltas"] > 2000
    assert_bitwise(got, O.oracle_spmm(oracle_arrays(c), x), "deep merge")


@pytest.mark.parametrize("normalized", [False, True])
def test_csr_comparator_operator(normalized, dev):
    """The uncompressed comparator computes the same product (csr_spmm_into,
    kernels.cpp:152): bit-exact for the binary matrix, within tolerance for
    the normalized one (scales applied per column / per row, not fused)."""
    a = P.generate_graph("pa_triangle", [3000, 2, 0.3], 17)
    x = P.generate_dense("normal", 3000, 64, 18)
    got, _ = gpu_spmm(P.csr_operator(a, normalized), x, dev, order_faithful=True)
    c = (P.build_cbm_normalized if normalized else P.build_cbm)(a, 0)
    want = O.oracle_spmm(oracle_arrays(c), x)
    if normalized:
        assert normwise_err(got, want) <= TOL
    else:
        vals = np.ones(a.nnz, np.float32)
        assert_bitwise(got, O.oracle_csr_spmm(a.row_ptr, a.col_idx, vals, x), "csr")


def test_concurrent_streams_share_one_handle(dev):
    """The uploaded operator is shareable: interleaved calls on two streams
    (each with its own workspace) give the same bits as serial calls."""
    a = P.generate_graph("community", [3000, 100, 0.4, 0.002], 61)
    c = P.build_cbm_normalized(a, 0)
    d = P.DeviceCbm(c)
    xa = torch.from_numpy(P.generate_dense("normal", 3000, 96, 62)).to(dev)
    xb = torch.from_numpy(P.generate_dense("normal", 3000, 96, 63)).to(dev)
    want_a, want_b = d.spmm(xa), d.spmm(xb)
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    ya = [torch.empty_like(want_a) for _ in range(20)]
    yb = [torch.empty_like(want_b) for _ in range(20)]
    for i in range(20):
        d.spmm_into(xa, ya[i], s1)
        d.spmm_into(xb, yb[i], s2)
    torch.cuda.synchronize()
    for i in range(20):
        assert torch.equal(ya[i], want_a) and torch.equal(yb[i], want_b), i


@pytest.mark.parametrize("n_handles", [1, 2, 3])
def test_spmm_sharded_host_buffers_bitwise(n_handles, dev):
    """cbm_b200_spmm_sharded: column slabs over several handles (all on
    cuda:0 here; one per device in production) reassemble the single-handle
    result bit for bit."""
    a = P.generate_graph("pa_triangle", [4000, 2, 0.3], 71)
    c = P.build_cbm_normalized(a, 0)
    x = P.generate_dense("normal", 4000, 200, 72)
    want = P.DeviceCbm(c, order_faithful=True).spmm_host(x)
    ops = [P.DeviceCbm(c, device=0, order_faithful=True) for _ in range(n_handles)]
    got = P.spmm_sharded(ops, x)
    assert_bitwise(got, want, f"sharded x{n_handles}")
    # default mode: a slab's kernel variant depends on its width, so the bits
    # may differ from one wide multiply; the tolerance holds
    fast = [P.DeviceCbm(c, device=0) for _ in range(n_handles)]
    assert normwise_err(P.spmm_sharded(fast, x), want) <= TOL
    with pytest.raises(ValueError, match="inner dimensions"):
        P.spmm_sharded(ops, x[:100])
    if n_handles > 1:
        with pytest.raises(ValueError, match="appears twice"):
            P.spmm_sharded([ops[0], ops[0]], x)


@pytest.mark.parametrize("normalized", [False, True])
def test_spmv_lane_parallel(normalized, dev):
    """spmv (d = 1, kernels.cpp:70-103): the lane-per-delta kernel. Order-
    faithful: bit-identical for any v (sequential adds). Default: bit-exact on
    integer v for the binary matrix, 1e-5 normwise otherwise; with long rows
    split into chunks and merge trees too."""
    for kind, params, seed in (("community", [3000, 100, 0.3, 0.002], 101),
                               ("pa_triangle", [4000, 2, 0.3], 102)):
        a = P.generate_graph(kind, params, seed)
        c = (P.build_cbm_normalized if normalized else P.build_cbm)(a, 0)
        arrays = oracle_arrays(c)
        for vkind in ("int", "normal"):
            v = P.generate_dense(vkind, a.n_cols, 1, seed + 1, -8, 8)
            want = O.oracle_spmm(arrays, v)
            vt = torch.from_numpy(v).to(dev)
            got = P.DeviceCbm(c, order_faithful=True).spmv(vt).cpu().numpy()
            assert_bitwise(got, want, f"spmv faithful {kind} {vkind}")
            for opts in ({}, {"split_threshold": 4, "chunk": 2}):
                h = P.DeviceCbm(c, **opts)
                got = h.spmv(vt).cpu().numpy()
                if opts:
                    assert h.info()["n_chunk_items"] > 0
                if vkind == "int" and not normalized:
                    assert_bitwise(got, want, f"spmv default {kind} {opts}")
                else:
                    assert normwise_err(got, want) <= TOL


@pytest.mark.parametrize("d", [1100, 2048])
def test_wide_operands_span_several_slabs(d, dev):
    """d > 512: several 512-column slabs per item (plus a partial one), each
    with its own ready flags; faithful bitwise, default integer bitwise."""
    a = P.generate_graph("community", [1500, 100, 0.4, 0.003], 111)
    c = P.build_cbm(a, 0)
    arrays = oracle_arrays(c)
    xi = P.generate_dense("int", 1500, d, 112, -8, 8)
    xg = P.generate_dense("normal", 1500, d, 113)
    got, _ = gpu_spmm(c, xg, dev, order_faithful=True)
    assert_bitwise(got, O.oracle_spmm(arrays, xg), f"faithful d={d}")
    got, _ = gpu_spmm(c, xi, dev)
    assert_bitwise(got, O.oracle_spmm(arrays, xi), f"default int d={d}")


@pytest.mark.parametrize("sprinkle", [0, 7])
def test_long_runs_of_empty_tickets(sprinkle, dev):
    """Rows equal to their parent have no deltas. Long runs of such tickets
    let the issue cursor run past the staged record window, stall there and
    resume (refilling the copy ring) when the window slides. 400k rows in
    chains of 100: one 20-delta root per chain, every `sprinkle`-th chain row
    one fresh delta."""
    rng = np.random.default_rng(131)
    n, n_cols, chain = 400_000, 6000, 100
    parent = np.empty(n, np.uint32)
    counts = np.zeros(n, np.int64)
    cols = []
    for r0 in range(0, n, chain):
        parent[r0] = 0xFFFFFFFF
        root_cols = np.sort(rng.choice(1000, 20, replace=False)).astype(np.uint32)
        cols.append(root_cols)
        counts[r0] = 20
        nxt = 1000
        for j in range(1, chain):
            parent[r0 + j] = r0 + j - 1
            if sprinkle and j % sprinkle == 0:
                cols.append(np.array([nxt + int(rng.integers(0, 40))], np.uint32))
                nxt += 50
                counts[r0 + j] = 1
    row_ptr = np.zeros(n + 1, np.uint64)
    row_ptr[1:] = np.cumsum(counts)
    col_idx = np.concatenate(cols).astype(np.uint32)
    vals = np.ones(col_idx.shape[0], np.float32)
    c = P.CbmMatrix(n, n_cols, 0, False, parent, row_ptr, col_idx, vals)
    arrays = oracle_arrays(c)
    x = P.generate_dense("int", n_cols, 64, 132, -8, 8)
    want = O.oracle_spmm(arrays, x)
    for faithful in (True, False):
        got, _ = gpu_spmm(c, x, dev, order_faithful=faithful)
        assert_bitwise(got, want, f"empty runs faithful={faithful}")


@pytest.mark.parametrize("normalized", [False, True])
def test_lane_groups_narrow_operands(normalized, dev):
    """Default mode, 4 <= d <= 64: 2, 4, 8 or 16 deltas per warp instruction, each
    lane group summing every H-th delta, combined by a fixed shuffle tree.
    Integer X on the binary matrix stays bit-exact; otherwise 1e-5 normwise;
    long rows chunked and parent chains included."""
    a = P.generate_graph("community", [2500, 100, 0.4, 0.004], 141)
    c = (P.build_cbm_normalized if normalized else P.build_cbm)(a, 0)
    arrays = oracle_arrays(c)
    for d in (4, 8, 12, 16, 20, 32, 36, 64):  # H = 16, 16, 8, 8, 4, 4, 2, 2
        for kind in ("int", "normal"):
            x = P.generate_dense(kind, 2500, d, 142 + d, -8, 8)
            want = O.oracle_spmm(arrays, x)
            for opts in ({}, {"split_threshold": 8, "chunk": 4}):
                got, h = gpu_spmm(c, x, dev, **opts)
                if kind == "int" and not normalized:
                    assert_bitwise(got, want, f"lane groups d={d} {opts}")
                else:
                    assert normwise_err(got, want) <= TOL, (d, kind, opts)


@pytest.mark.parametrize("tile", [0, 1])
@pytest.mark.parametrize("faithful", [False, True])
def test_binary_relu_epilogue(tile, faithful, dev):
    """spmm_ex with CBM_B200_RELU on a BINARY matrix: children must add their
    parent's unclipped row (relu_inplace, dense.cpp:51-54, applies to the
    finished product only)."""
    a = P.generate_graph("community", [2000, 100, 0.5, 0.002], 171)
    c = P.build_cbm(a, 0, threads=8)
    x = P.generate_dense("int", 2000, 96, 172, -8, 8)
    want = O.oracle_spmm(oracle_arrays(c), x)
    want = np.where(want < 0, np.float32(0), want)
    h = P.DeviceCbm(c, tile=tile, order_faithful=faithful)
    y = h.spmm(torch.from_numpy(x).to(dev), relu=True)
    torch.cuda.synchronize()
    assert_bitwise(y.cpu().numpy(), want, f"binary relu tile={tile} faithful={faithful}")


@pytest.mark.parametrize("faithful", [False, True])
@pytest.mark.parametrize("normalized", [False, True])
def test_hub_heavy_clique_overlay(normalized, faithful, dev):
    """cfg[2]-shaped (Zipf clique overlay) at 1/40 scale: hub rows of thousands
    of deltas walk many 32-delta index windows (rotated per ring group; in the
    order-faithful mode unsplit), at every kernel variant's width."""
    a = P.generate_graph("clique_overlay", [6000, 30000, 2, 10, 1.1], 0xC0F60000 + 77)
    c = (P.build_cbm_normalized if normalized else P.build_cbm)(a, 8)
    assert np.diff(c.row_ptr).max() > 256
    arrays = oracle_arrays(c)
    for d in (1, 48, 64, 128, 200, 256, 512):
        kind = "int" if not normalized else "normal"
        x = P.generate_dense(kind, a.n_cols, d, 0xC0F61000 + d, -8, 8)
        want = O.oracle_spmm(arrays, x)
        got, _ = gpu_spmm(c, x, dev, order_faithful=faithful)
        if faithful or not normalized:
            assert_bitwise(got, want, f"clique overlay d={d} faithful={faithful}")
        else:
            assert normwise_err(got, want) <= TOL, d


@pytest.mark.parametrize("tile", [0, -1])
def test_2d_partition_blocks_on_device(tile, dev):
    """bench.py --row-groups: every (row group, column slab) block multiplied
    on the device from its own sub-CBM (sharding.row_partition, cross-group
    parents flattened) reassembles the full 1-GPU multiply exactly (integer X,
    exact in any summation order)."""
    from paper_2409_02208_b200.sharding import all_slabs, row_partition
    a = P.generate_graph("clique_overlay", [6000, 30000, 2, 10, 1.1], 0xC0F60000 + 93)
    c = P.build_cbm(a, 4)
    x = P.generate_dense("int", a.n_cols, 96, 0xC0F61000 + 93, -8, 8)
    want = O.oracle_spmm(oracle_arrays(c), x)
    for groups in (2, 4):
        got = np.full_like(want, np.nan)
        for rows, sub in row_partition(a, c, groups):
            for lo, hi in all_slabs(96, 2):
                y, _ = gpu_spmm(sub, x[:, lo:hi], dev, tile=tile)
                got[rows, lo:hi] = y
        assert_bitwise(got, want, f"{groups} row groups")
