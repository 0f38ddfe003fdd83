"""CBM1 container (io.hpp:44-57, io.cpp:198-382): round trip, interop with the
reference's own save_cbm/load_cbm in both directions, and the reference's
validation errors (test_io.cpp:230-311 style corruptions)."""
import os
import struct

import numpy as np
import pytest

import oracle as O
import paper_2409_02208_b200 as P
from helpers import golden_cbm, golden_names, load_golden, same_cbm


@pytest.mark.parametrize("name", golden_names()[::5])
def test_round_trip_golden(name, tmp_path):
    c = golden_cbm(load_golden(name))
    path = tmp_path / "c.cbm"
    P.save_cbm(c, path)
    back = P.load_cbm(path)
    assert same_cbm(back, c)
    assert back.alpha == c.alpha and back.is_normalized == c.is_normalized
    assert np.array_equal(back.topo_order, c.topo_order)


@pytest.mark.parametrize("normalized", [False, True])
def test_interop_with_reference(normalized, tmp_path):
    if not O.ref_available():
        pytest.skip("compiled reference absent")
    a = O.RefCsr.community_graph(20, 30, 25, 2, 77)
    ref = O.RefCbm.build(a, 2, normalized=normalized)
    p1 = tmp_path / "ref.cbm"
    ref.save(p1)                                   # written by the reference
    ours = P.load_cbm(p1)
    assert same_cbm(ours, ref.arrays())
    p2 = tmp_path / "ours.cbm"
    P.save_cbm(ours, p2)                           # written by us
    assert open(p1, "rb").read() == open(p2, "rb").read()   # byte-identical files
    back = O.RefCbm.load(p2).arrays()              # loaded by the reference
    assert same_cbm(ours, back)


def _good(tmp_path, normalized=True):
    a = P.CsrBinaryMatrix(9, 9, *O.oracle_random_binary(9, 9, 0.4, 3))
    c = (P.build_cbm_normalized if normalized else P.build_cbm)(a, 0)
    path = tmp_path / "g.cbm"
    P.save_cbm(c, path)
    return bytearray(open(path, "rb").read()), c


def _expect(tmp_path, blob, msg):
    path = tmp_path / "bad.cbm"
    open(path, "wb").write(bytes(blob))
    with pytest.raises(P.FormatError, match=msg):
        P.load_cbm(path)


def test_format_errors_mirror_reference(tmp_path):
    blob, c = _good(tmp_path)
    _expect(tmp_path, blob[:3], "truncated container")
    b = bytearray(blob); b[0:4] = b"XBM1"; _expect(tmp_path, b, "bad magic")
    b = bytearray(blob); b[4] = 2; _expect(tmp_path, b, "unsupported container version")
    b = bytearray(blob); b[5] = 3; _expect(tmp_path, b, "unknown flag bits set")
    b = bytearray(blob); b[6] = 1; _expect(tmp_path, b, "reserved header bytes must be zero")
    _expect(tmp_path, blob + b"\0", "payload size mismatch")
    _expect(tmp_path, blob[:-1], "payload size mismatch")
    # a parent pointing at itself -> invalid structure
    b = bytearray(blob); b[40:44] = struct.pack("<I", 0); _expect(tmp_path, b, "invalid container structure")
    # flip a value's sign bit -> still +-s; change magnitude -> disagree with the scales
    m, nnz = c.n_rows, c.nnz
    voff = 40 + 8 * m + 8 * (m + 1) + 4 * nnz
    b = bytearray(blob); b[voff:voff + 8] = struct.pack("<d", 0.123)
    _expect(tmp_path, b, "delta values disagree with the column scales")
    soff = voff + 8 * nnz
    b = bytearray(blob); b[soff:soff + 8] = struct.pack("<d", -1.0)
    _expect(tmp_path, b, "row_scale entries must be positive and finite")


def test_plain_container_value_check(tmp_path):
    blob, c = _good(tmp_path, normalized=False)
    m, nnz = c.n_rows, c.nnz
    voff = 40 + 8 * m + 8 * (m + 1) + 4 * nnz
    b = bytearray(blob); b[voff:voff + 8] = struct.pack("<d", 2.0)
    _expect(tmp_path, b, "delta values must be \\+1 or -1")
    with pytest.raises(P.FormatError, match="cannot open file"):
        P.load_cbm(os.path.join(str(tmp_path), "missing.cbm"))


@pytest.mark.gpu
def test_container_to_device(tmp_path):
    """Ship-pre-compressed path: CBM1 file -> upload -> multiply."""
    import torch
    from helpers import assert_bitwise, oracle_arrays
    a = P.generate_graph("community", [2000, 100, 0.5, 0.002], 9)
    c = P.build_cbm_normalized(a, 0, threads=4)
    path = tmp_path / "c.cbm"
    P.save_cbm(c, path)
    back = P.load_cbm(path)
    x = P.generate_dense("normal", 2000, 96, 10)
    y = P.DeviceCbm(back, order_faithful=True).spmm(torch.from_numpy(x).cuda()).cpu().numpy()
    assert_bitwise(y, O.oracle_spmm(oracle_arrays(c), x), "cbm1 -> device")
