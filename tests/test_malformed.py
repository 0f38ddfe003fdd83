"""Delta rows that are inconsistent with their parent's row (a minus column the
parent lacks, a plus column it already has). The reference's loader and
constructors accept them (io.cpp:346-380 checks ranges, order and values, not
set consistency) and its multiply computes U = deltas + U_parent
(kernels.cpp:27-53). The device layout must neither overrun a buffer while
flattening such rows (layout.cpp) nor change their values."""
import numpy as np
import pytest

import paper_2409_02208_b200 as P
from helpers import assert_bitwise, oracle_arrays

import oracle as O

V = 0xFFFFFFFF


def malformed():
    # row 0: root +{0..3}; row 1: child of 0 with +{1999} (flattened by the
    # default flatten_gain); row 2: child of 0 with -{10, 11} (not in row 0)
    rows = [([0, 1, 2, 3], [1, 1, 1, 1]), ([1999], [1]), ([10, 11], [-1, -1])]
    parent = np.array([V, 0, 0], np.uint32)
    rp = np.zeros(4, np.uint64)
    ci, vals = [], []
    for i, (c, v) in enumerate(rows):
        ci += c
        vals += v
        rp[i + 1] = len(ci)
    return P.CbmMatrix(3, 2000, 0, False, parent, rp, np.array(ci, np.uint32),
                       np.array(vals, np.float32))


def plus_present():
    # row 1 adds column 2, which row 0 already has (value 2 in the reference)
    parent = np.array([V, 0], np.uint32)
    rp = np.array([0, 3, 5], np.uint64)
    ci = np.array([0, 2, 5, 2, 7], np.uint32)
    vals = np.array([1, 1, 1, 1, 1], np.float32)
    return P.CbmMatrix(2, 8, 0, False, parent, rp, ci, vals)


def test_reference_accepts_inconsistent_rows():
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    c = malformed()
    O.RefCbm.from_arrays(oracle_arrays(c))  # no exception: the reference takes it


def test_upload_of_inconsistent_rows_does_not_overrun_on_the_host():
    # on a CPU-only box the upload plans the layout (where the overrun was),
    # then fails cleanly at the device step; on a GPU box it succeeds
    for c in (malformed(), plus_present()):
        try:
            op = P.DeviceCbm(c)
        except P.CbmError as e:
            assert "CUDA" in str(e) or "device" in str(e).lower() or e.code == 2, str(e)
        else:
            op.close()


@pytest.mark.gpu
@pytest.mark.parametrize("make", [malformed, plus_present])
@pytest.mark.parametrize("tile", [-1, 0])
def test_inconsistent_rows_multiply_like_the_reference(make, tile):
    import torch
    c = make()
    x = P.generate_dense("int", c.n_cols, 64, 5, -8, 8)
    want = O.oracle_spmm(oracle_arrays(c), x)
    for faithful in (False, True):
        op = P.DeviceCbm(c, device=0, order_faithful=faithful, tile=tile)
        got = op.spmm(torch.from_numpy(x).cuda()).cpu().numpy()
        assert_bitwise(got, want, f"{make.__name__} faithful={faithful} tile={tile}")


@pytest.mark.gpu
def test_forced_tiling_refuses_inconsistent_rows():
    with pytest.raises(ValueError, match="inconsistent"):
        P.DeviceCbm(malformed(), device=0, tile=1, tile_rows=64)
