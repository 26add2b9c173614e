"""CPU: pin the oracle restatement against fixtures produced by the reference.

The fixtures in tests/golden were produced by running mfglobal 0.1.0 itself
(tests/golden/make_golden.py); this proves the oracle the GPU tests compare
against computes what the reference computes.
"""

import numpy as np
import pytest

from oracle import mfg_oracle as orc


def _om(g, p):
    return orc.from_coo(*g.obs_args(p))


def test_from_coo_matches_reference(golden):
    g = golden("omega.npz")
    for ci in range(4):
        p = f"c{ci}_"
        om = orc.from_coo(int(g[p + "m"]), int(g[p + "n"]), g[p + "in_rows"], g[p + "in_cols"],
                          g[p + "in_vals"])
        assert np.array_equal(om.rows, g[p + "rows"])
        assert np.array_equal(om.cols, g[p + "cols"])
        assert np.array_equal(om.vals, g[p + "vals"])
        assert np.array_equal(om.indptr, g[p + "indptr"])
        t = om.a_csr_t
        assert np.array_equal(t.indptr, g[p + "csc_ptr"])
        assert np.array_equal(t.indices, g[p + "csc_idx"])
        assert np.array_equal(t.data, g[p + "csc_val"])
        # the CSC permutation is the stable argsort of cols
        perm = om.csc_perm()
        assert np.array_equal(om.vals[perm], g[p + "csc_val"])
        assert np.array_equal(om.rows[perm], g[p + "csc_idx"])


def test_from_coo_errors_match_reference(golden):
    g = golden("omega.npz")
    with pytest.raises(orc.OracleDatasetError) as err:
        orc.from_coo(3, 3, [2, 0, 2, 1], [1, 0, 1, 2], [1.0, 2.0, 3.0, 4.0])
    assert str(err.value) == str(g["dup_msg"])
    for bad, args in [("row_range", (2, 2, [0, 2], [0, 0], [1.0, 1.0])),
                      ("col_range", (2, 2, [0, 1], [0, -1], [1.0, 1.0])),
                      ("length", (2, 2, [0, 1], [0], [1.0, 1.0]))]:
        with pytest.raises(orc.OracleDatasetError) as err:
            orc.from_coo(*args)
        assert str(err.value) == str(g["err_" + bad])
    assert np.array_equal(orc.from_coo(3, 4, [], [], []).indptr, g["empty_indptr"])


def test_sweep_matches_reference(golden):
    g = golden("sweep.npz")
    for name in g.names():
        p = name + "_"
        om = _om(g, p)
        r, rh, rtw, sq, w2, h2 = orc.sweep(om, g[p + "w"], g[p + "h"])
        assert np.array_equal(r, g[p + "r"]), name
        assert np.allclose(rh, g[p + "rh"], rtol=0, atol=1e-13), name
        assert np.allclose(rtw, g[p + "rtw"], rtol=0, atol=1e-13), name
        assert sq == pytest.approx(float(g[p + "loss"]), rel=1e-14, abs=1e-300)
        assert w2 + h2 == pytest.approx(float(g[p + "frob"]), rel=1e-14)
        tres = orc.triplet_values(g[p + "tu"], g[p + "ts"], g[p + "tv"], om.rows, om.cols) - om.vals
        assert np.array_equal(tres, g[p + "tres"]), name


def test_bcd_matches_reference(golden):
    g = golden("bcd.npz")
    for name in g.names():
        p = name + "_"
        om = _om(g, p)
        lam = float(g[p + "lam"])
        w1, h1 = orc.bcd_epoch(om, g[p + "w"], g[p + "h"], lam)
        assert np.array_equal(w1, g[p + "w1"]), name
        assert np.array_equal(h1, g[p + "h1"]), name
        assert orc.mf_objective(om, g[p + "w"], g[p + "h"], lam) == float(g[p + "obj0"])
        assert orc.mf_objective(om, w1, h1, lam) == float(g[p + "obj1"])


def test_operator_matches_reference(golden):
    g = golden("operator.npz")
    for name in g.names():
        p = name + "_"
        om = _om(g, p)
        w, h, gv, a = g[p + "w"], g[p + "h"], g[p + "g"], float(g[p + "alpha"])
        assert np.array_equal(orc.shifted_apply(om, w, h, gv, a, g[p + "bn"]), g[p + "apply"])
        assert np.array_equal(orc.shifted_apply_t(om, w, h, gv, a, g[p + "bm"]), g[p + "apply_t"])
        assert np.array_equal(orc.shifted_project_rows(om, w, h, gv, a, g[p + "q"]), g[p + "project"])
        fs = orc.shifted_frob_sq(om, w, h, gv, a)
        assert fs == pytest.approx(float(g[p + "frob_sq"]), rel=1e-13)


def test_dense_kernels_match_reference(golden):
    g = golden("kernels.npz")
    for name in [str(s) for s in g["orth_names"]]:
        q, rank = orc.orthonormalize(g["orth_" + name + "_in"])
        assert rank == int(g["orth_" + name + "_rank"]), name
        assert np.allclose(q @ q.T, g["orth_" + name + "_proj"], atol=1e-12)
    for i in range(int(g["st_count"])):
        sig, kept, lt = orc.soft_threshold(g[f"st{i}_in"], float(g[f"st{i}_beta"]))
        assert np.array_equal(sig, g[f"st{i}_sigma"])
        assert np.array_equal(kept, g[f"st{i}_kept"])
        ref_lt = float(g[f"st{i}_lt"])
        assert (lt is None and np.isnan(ref_lt)) or lt == ref_lt
    for i in range(int(g["svd_count"])):
        _, s, _ = orc.exact_svd_short_fat(g[f"svd{i}_in"])
        assert np.allclose(s, g[f"svd{i}_s"], rtol=1e-12, atol=1e-12)


def test_known_answer_values():
    # r = (1)(1) - 3 = -2  (reference tests/test_data.py:102-106)
    om = orc.from_coo(1, 1, [0], [0], [3.0])
    r = orc.residual(om, np.array([[1.0]]), np.array([[1.0]]))
    assert r.tolist() == [-2.0]
    # scalar normal equation w = 2a/(lam+2) (tests/test_mfsolver.py:107-115)
    w1, _ = orc.bcd_epoch(om, np.array([[10.0]]), np.array([[1.0]]), 0.5)
    assert abs(w1[0, 0] - 2 * 3.0 / 2.5) < 1e-12
