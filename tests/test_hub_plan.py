"""Hub-row panel planner (host only): the panel plus the rest reproduce the
represented matrix; the auto rule declines matrices without hub rows."""
import numpy as np

import paper_2409_02208_b200 as P


def test_plan_counts_partition_the_matrix():
    a = P.generate_graph("clique_overlay", [5000, 15000, 2, 8, 1.1], 51)
    c = P.csr_operator(a)
    s = P.plan_hub(c, 1)
    assert s["active"] and s["rows"] == 128
    lens = np.sort(np.diff(a.row_ptr))[::-1]
    assert s["entries"] == int(lens[:128].sum())
    assert s["rest_deltas"] + s["entries"] == a.nnz
    assert s["chunks"] >= 1 and 1 <= s["pieces"] <= 148


def test_auto_declines_small_and_flat_matrices():
    a = P.generate_graph("clique_overlay", [5000, 15000, 2, 8, 1.1], 51)
    assert not P.plan_hub(P.csr_operator(a), -1)["active"]           # below the size floor
    b = P.generate_graph("community", [40000, 200, 0.15, 1e-5], 52)   # no hub rows
    assert not P.plan_hub(P.csr_operator(b), -1)["active"]


def test_forced_plan_with_compressed_children():
    a = P.generate_graph("clique_overlay", [3000, 9000, 2, 6, 1.1], 53)
    c = P.build_cbm(a, 0, 4)
    s = P.plan_hub(c, 1)
    assert s["active"] and s["rows"] == 128
    lens = np.sort(np.diff(a.row_ptr))[::-1]
    assert s["entries"] == int(lens[:128].sum())   # full rows, whatever their delta form
