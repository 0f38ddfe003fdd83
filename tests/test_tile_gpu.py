"""GPU parity of the tiled path (DESIGN.md §6 "Tiled path", csrc/tile_kernel.cu).

One CTA per (row block, column slab) sums its rows from an X tile staged in
shared memory. Only the summation order changes (staged deltas, cold deltas,
parent), so the bar is the default mode's: bit-exact for the binary matrix on
integer X, max|G-R|/max|R| <= 1e-5 otherwise (north_star tolerance).
"""
import numpy as np
import pytest

import oracle as O
import paper_2409_02208_b200 as P
from helpers import (assert_bitwise, golden_cbm, golden_names, load_golden, normwise_err,
                     oracle_arrays)

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

TOL = 1e-5


@pytest.fixture(scope="module")
def dev():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch.device("cuda:0")


def run(c, x, dev, **opt):
    opt.setdefault("tile", 1)
    h = P.DeviceCbm(c, **opt)
    xt = torch.from_numpy(np.ascontiguousarray(x, np.float32)).to(dev)
    y = h.spmm(xt)
    torch.cuda.synchronize()
    return y.cpu().numpy(), h


def check(c, x, got, what):
    want = O.oracle_spmm(oracle_arrays(c), x)
    if not c.is_normalized and np.array_equal(x, np.round(x)):
        assert_bitwise(got, want, what)
    else:
        assert normwise_err(got, want) <= TOL, what


@pytest.mark.parametrize("name", golden_names())
def test_golden_fixtures_tiled(name, dev):
    g = load_golden(name)
    if str(g["kind"]) in ("gcn", "spmv"):
        pytest.skip("not an spmm fixture")
    c = golden_cbm(g)
    x = g["x"]
    if x.shape[1] < 32:  # the tiled path serves d >= 32: widen the operand
        x = np.ascontiguousarray(np.tile(x, (1, (32 + x.shape[1] - 1) // x.shape[1])))
    got, h = run(c, x, dev)
    assert h.info()["tile_active"] == 1
    check(c, x, got, name)


@pytest.mark.parametrize("normalized", [False, True])
def test_random_suite_tiled(normalized, dev):
    rng = np.random.default_rng(4242 + normalized)
    for k in range(40):
        n = int(rng.integers(1, 300))
        m = n if normalized else int(rng.integers(1, 300))
        rp, ci = O.oracle_random_binary(m, n, float(rng.uniform(0.02, 0.5)), 500 + k)
        a = P.CsrBinaryMatrix(m, n, rp, ci)
        c = (P.build_cbm_normalized if normalized else P.build_cbm)(a, int(rng.choice([0, 2, 8])))
        d = int(rng.choice([32, 33, 48, 64, 100, 128, 130, 256, 520]))
        opts = dict(tile_rows=int(rng.choice([0, 1, 3, 16, 64])),
                    tile_stage=int(rng.choice([0, 1, 5, 40])),
                    tile_vec=int(rng.choice([0, 1, 2, 4])))
        for kind in ("int", "normal"):
            x = P.generate_dense(kind, n, d, 900 + k, -8, 8)
            got, _ = run(c, x, dev, **opts)
            check(c, x, got, f"case {k} d={d} {opts} {kind}")


@pytest.mark.parametrize("rows,stage", [(0, 0), (8, 0), (37, 3), (512, 1)])
@pytest.mark.parametrize("normalized", [False, True])
def test_community_blocks_cuts_and_cold_deltas(rows, stage, normalized, dev):
    """Trees bigger than the block are cut (cut rows flattened), tiny staging
    capacities push most deltas to the cold path."""
    a = P.generate_graph("community", [3000, 250, 0.5, 0.003], 7)
    c = (P.build_cbm_normalized if normalized else P.build_cbm)(a, 0, threads=8)
    got, h = run(c, P.generate_dense("int", 3000, 96, 8, -8, 8), dev,
                 tile_rows=rows, tile_stage=stage)
    info = h.info()
    assert info["tile_active"] == 1 and info["tile_blocks"] > 0
    if rows and rows < 250:
        assert info["tile_cut_rows"] > 0
    if stage:
        assert info["tile_max_staged"] <= stage
    check(c, P.generate_dense("int", 3000, 96, 8, -8, 8), got, "int")
    xg = P.generate_dense("normal", 3000, 96, 9)
    got, _ = run(c, xg, dev, tile_rows=rows, tile_stage=stage)
    check(c, xg, got, "normal")


def test_cfg0_full_size_tiled_bitexact(dev):
    a = P.generate_graph("community", [4096, 64, 0.5, 0.001], 0xC0F60000)
    c = P.build_cbm(a, 0, threads=8)
    x = P.generate_dense("int", 4096, 64, 0xC0F61000, -8, 8)
    want = O.oracle_spmm(oracle_arrays(c), x)
    for vec in (0, 1, 2):
        got, h = run(c, x, dev, tile_vec=vec)
        assert_bitwise(got, want, f"cfg0 tile_vec={vec}")


def test_auto_mode_picks_tiles_for_communities_only(dev):
    comm = P.build_cbm_normalized(P.generate_graph("community", [6000, 500, 0.8, 1e-4], 3), 0,
                                  threads=8)
    pa = P.build_cbm_normalized(P.generate_graph("pa_triangle", [6000, 2, 0.3], 4), 0)
    assert P.DeviceCbm(comm).info()["tile_active"] == 1
    assert P.DeviceCbm(pa).info()["tile_active"] == 0
    assert P.DeviceCbm(comm, tile=0).info()["tile_active"] == 0
    assert P.DeviceCbm(comm, order_faithful=True).info()["tile_active"] == 0


def test_slabs_relu_strides_and_repeats(dev):
    """Column slabs of a wider X/Y (ldx, ldy > d), the fused ReLU, partial last
    slabs and repeated calls (the interior scratch is rewritten every call)."""
    a = P.generate_graph("community", [2500, 500, 0.6, 0.001], 13)
    c = P.build_cbm_normalized(a, 0, threads=8)
    h = P.DeviceCbm(c, tile=1)
    full = P.generate_dense("normal", 2500, 300, 14)
    xt = torch.from_numpy(full).to(dev)
    want = O.oracle_spmm(oracle_arrays(c), full)
    for c0, w in ((0, 64), (64, 100), (164, 136), (1, 33), (8, 256)):
        y = torch.zeros((2500, 300), device=dev)
        h.spmm_into(xt[:, c0:c0 + w], y[:, c0:c0 + w])
        torch.cuda.synchronize()
        assert normwise_err(y[:, c0:c0 + w].cpu().numpy(), want[:, c0:c0 + w]) <= TOL
    y = torch.empty((2500, 300), device=dev)
    h.spmm_into(xt, y, relu=True)
    first = y.clone()
    for _ in range(20):
        h.spmm_into(xt, y, relu=True)
    torch.cuda.synchronize()
    assert torch.equal(first, y)
    r = np.where(want < 0, np.float32(0), want)
    assert normwise_err(first.cpu().numpy(), r) <= TOL
    assert (first.cpu().numpy() >= 0).all()


def test_empty_rows_and_identity(dev):
    c = P.build_cbm(P.CsrBinaryMatrix.from_rows(40, [[], [3], [], [3, 5], []] * 8), 0)
    x = P.generate_dense("int", 40, 64, 1, -8, 8)
    got, _ = run(c, x, dev)
    check(c, x, got, "empty rows")
    eye = P.build_cbm(P.CsrBinaryMatrix.from_rows(50, [[i] for i in range(50)]), 0)
    x = P.generate_dense("normal", 50, 40, 2)
    got, _ = run(eye, x, dev)
    assert_bitwise(got, x, "identity")


@pytest.mark.parametrize("split", ["1", "7", "100000"])
def test_half_width_units(split, dev, monkeypatch):
    """The last (block, slab) pairs of a launch run as two half-width units
    (shorter last wave); force 1, 7 or all pairs to split."""
    monkeypatch.setenv("CBM_B200_TILE_SPLIT", split)
    a = P.generate_graph("community", [3000, 250, 0.5, 0.003], 7)
    for normalized in (False, True):
        c = (P.build_cbm_normalized if normalized else P.build_cbm)(a, 0, threads=8)
        for d, vec in ((256, 2), (256, 4), (200, 2), (96, 0)):
            x = P.generate_dense("int", 3000, d, 8, -8, 8)
            got, _ = run(c, x, dev, tile_vec=vec)
            check(c, x, got, f"split={split} d={d} vec={vec} norm={normalized}")
