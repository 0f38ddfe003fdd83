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


@pytest.mark.parametrize("normalized", [False, True])
def test_corruptions_report_the_reference_error(normalized, tmp_path):
    """Random byte corruptions (several at once, so several rules can break):
    our mapped parallel loader accepts exactly what the reference's load_cbm
    accepts and reports the same first error (io.cpp:293-382 order)."""
    if not O.ref_available():
        pytest.skip("compiled reference absent")
    a = P.CsrBinaryMatrix(40, 40, *O.oracle_random_binary(40, 40, 0.3, 11))
    c = (P.build_cbm_normalized if normalized else P.build_cbm)(a, 0)
    path = tmp_path / "g.cbm"
    P.save_cbm(c, path)
    good = bytes(open(path, "rb").read())
    rng = np.random.default_rng(7 + normalized)
    seen = set()
    for trial in range(300):
        b = bytearray(good)
        for _ in range(int(rng.integers(1, 4))):
            pos = int(rng.integers(40, len(b)))
            b[pos] = int(rng.integers(0, 256)) if rng.random() < 0.5 else b[pos] ^ (1 << int(rng.integers(0, 8)))
        p = tmp_path / f"t{trial}.cbm"
        open(p, "wb").write(bytes(b))
        try:
            ref = O.RefCbm.load(p)
            ref_err = None
        except Exception as e:  # noqa: BLE001  (the reference's format_error text)
            ref, ref_err = None, str(e)
        try:
            ours = P.load_cbm(p)
            our_err = None
        except P.FormatError as e:
            ours, our_err = None, str(e).split("] ", 1)[-1] if str(e).startswith("[") else str(e)
        if ref_err is None:
            assert our_err is None, (trial, our_err)
            assert same_cbm(ours, ref.arrays())
        else:
            assert our_err is not None and our_err.endswith(ref_err) or ref_err.endswith(our_err), \
                (trial, our_err, ref_err)
            seen.add(ref_err.split(":")[0])
    assert len(seen) >= 3, seen


@pytest.mark.gpu
@pytest.mark.parametrize("normalized", [False, True])
def test_reference_container_straight_to_device(normalized, tmp_path):
    """The reference's own save_cbm -> cbm_b200_upload_cbm1 (mapped, validated,
    uploaded in one call) -> multiply, against the compiled reference's
    spmm_into on the same file and against the oracle."""
    if not O.ref_available():
        pytest.skip("compiled reference absent")
    import torch
    from helpers import assert_bitwise, normwise_err, oracle_arrays
    a = O.RefCsr.community_graph(40, 50, 35, 3, 91)
    ref = O.RefCbm.build(a, 0, threads=4, normalized=normalized)
    path = tmp_path / "ref.cbm"
    ref.save(path)
    n = ref.dims()[1]
    x = (P.generate_dense("int", n, 64, 12, -8, 8) if not normalized
         else P.generate_dense("normal", n, 128, 12))
    want = O.RefCbm.load(path).spmm(x, 4)
    assert_bitwise(O.oracle_spmm(ref.arrays(), x), want, "oracle vs reference")
    for faithful in (True, False):
        op = P.DeviceCbm.from_cbm1(path, device=0, order_faithful=faithful)
        assert (op.n_rows, op.is_normalized) == (ref.dims()[0], normalized)
        got = op.spmm(torch.from_numpy(x).cuda()).cpu().numpy()
        if faithful or not normalized:
            assert_bitwise(got, want, f"cbm1 -> device, faithful={faithful}")
        else:
            assert normwise_err(got, want) <= 1e-5


def test_upload_cbm1_reports_format_errors_without_a_device(tmp_path):
    blob, _ = _good(tmp_path)
    p = tmp_path / "bad.cbm"
    open(p, "wb").write(bytes(blob[:-1]))
    with pytest.raises(P.FormatError, match="payload size mismatch"):
        P.DeviceCbm.from_cbm1(p)
