"""Golden vectors produced by the reference itself (tests/golden/make_golden.py).

Every case recreates a fixture of the reference's own tests (file:line in the
comments) and compares against the reference library's recorded output, and —
where the reference test compares against its brute-force oracle — against that
oracle's output too. The same cases run against:

* ``port``  — the C restatement (oracle/), CPU, pins the oracle;
* ``gpu``   — the product's CUDA path through the C-ABI (marked ``gpu``).
"""
import os

import numpy as np
import pytest

from tests.backends import BACKENDS, backend_fixture, golden, names

backend = backend_fixture()


class P:  # duck-typed SgmParams
    def __init__(self, arr):
        self.p1, self.p2, self.paths, self.path_set, self.d_max = (int(v) for v in arr)


class Cal:
    def __init__(self, arr):
        self.focal_px, self.cx, self.cy, self.baseline_m = (float(v) for v in arr[:4])
        self.width, self.height, self.d_max = (int(v) for v in arr[4:])


class F:
    def __init__(self, **kw):
        self.q, self.r, self.p_init, self.disc_thresh = 0.5, 1.0, 4096.0, 2.0
        self.min_range_halfwidth, self.range_use_stddev, self.range_stddev_gain = 2, False, 2.0
        self.__dict__.update(kw)


def test_census_random_patches(backend):
    # test_matching_cost.cpp:48-57
    g = golden("census_rand")
    for t in range(5):
        np.testing.assert_array_equal(backend.census(g[f"{t}__img"]), g[f"{t}__sig"])


def test_ragged_cost_volume(backend):
    # test_matching_cost.cpp:146-161
    g = golden("cost_ragged")
    off, cost = backend.cost_volume(g["left"], g["right"], g["ranges_lo"], g["ranges_hi"])
    np.testing.assert_array_equal(off, g["offsets"])
    np.testing.assert_array_equal(cost, g["cost"])


@pytest.mark.parametrize("group", ["agg_scanline", "agg_full", "agg_ragged"])
def test_aggregation_matches_reference_and_brute_force(backend, group):
    # test_sgm.cpp:232-240, 255-284 (oracle: tests/oracles.hpp:70-144)
    g = golden(group)
    cases = names(g, "cost")
    assert cases
    for pre in cases:
        agg = backend.aggregate(g[pre + "cost"], g[pre + "ranges_lo"], g[pre + "ranges_hi"],
                                P(g[pre + "params"]))
        np.testing.assert_array_equal(agg, g[pre + "agg"])
        np.testing.assert_array_equal(agg, g[pre + "oracle"])
        if pre + "wta_d" in g:
            d, v = backend.wta(agg, g[pre + "ranges_lo"], g[pre + "ranges_hi"])
            np.testing.assert_array_equal(d, g[pre + "wta_d"])
            np.testing.assert_array_equal(v, g[pre + "wta_valid"])


def test_wta_random(backend):
    # test_sgm.cpp:333-343
    g = golden("wta_rand")
    d, v = backend.wta(g["agg"], g["ranges_lo"], g["ranges_hi"])
    np.testing.assert_array_equal(d, g["out_d"])
    np.testing.assert_array_equal(v, g["out_valid"])
    np.testing.assert_array_equal(d, g["oracle_d"])


def test_median_random(backend):
    # test_sgm.cpp:403-416
    g = golden("median_rand")
    for t in range(5):
        d, v = backend.median(g[f"{t}__in_d"], g[f"{t}__in_valid"])
        np.testing.assert_array_equal(d, g[f"{t}__out_d"])
        np.testing.assert_array_equal(v, g[f"{t}__out_valid"])
        np.testing.assert_array_equal(v, g[f"{t}__oracle_valid"])
        np.testing.assert_array_equal(d[v > 0], g[f"{t}__oracle_d"][v > 0])


@pytest.mark.parametrize("group", ["shifted", "shifted12"])
def test_full_range_sgm_on_shifted_pairs(backend, group):
    # test_sgm.cpp:419-432, 446-457
    g = golden(group)
    p = P(g["params"])
    h, w = g["left"].shape
    lo = np.zeros((h, w), np.uint16)
    hi = np.full((h, w), p.d_max - 1, np.uint16)
    d, v = backend.sgm_match(g["left"], g["right"], lo, hi, p)
    np.testing.assert_array_equal(d, g["out_d"])
    np.testing.assert_array_equal(v, g["out_valid"])
    if "median_d" in g:
        md, mv = backend.median(d, v)
        np.testing.assert_array_equal(md, g["median_d"])
        np.testing.assert_array_equal(mv, g["median_valid"])


def test_acceptance_criterion_1(backend):
    # acceptance.cpp:42-90: 50 random 16x8 pairs, random P1/P2/path sets
    g = golden("crit1")
    for t in range(50):
        pre = f"{t}__"
        p = P(g[pre + "params"])
        lo = np.zeros((8, 16), np.uint16)
        hi = np.full((8, 16), 7, np.uint16)
        _, cost = backend.cost_volume(g[pre + "left"], g[pre + "right"], lo, hi)
        np.testing.assert_array_equal(cost, g[pre + "cost"])
        agg = backend.aggregate(cost, lo, hi, p)
        np.testing.assert_array_equal(agg, g[pre + "agg"])
        np.testing.assert_array_equal(agg, g[pre + "oracle"])
        d, v = backend.wta(agg, lo, hi)
        np.testing.assert_array_equal(d, g[pre + "wta_d"])
        np.testing.assert_array_equal(v, g[pre + "wta_valid"])


def test_warp_and_predict(backend):
    # test_geometry.cpp:228-247 (gather oracle tests/oracles.hpp:218-260)
    g = golden("warp")
    for t in range(4):
        pre = f"{t}__"
        cal = Cal(g[pre + "calib"])
        m = g[pre + "motion"]
        R, tr = m[:9].reshape(3, 3), m[9:]
        H = backend.homography(R, tr, cal)
        np.testing.assert_array_equal(H.ravel(), g[pre + "H"])
        od, op, ov, osrc = backend.warp(g[pre + "in_d"], g[pre + "in_p"], g[pre + "in_valid"],
                                        g[pre + "H"].reshape(4, 4), cal.d_max)
        np.testing.assert_array_equal(ov, g[pre + "out_valid"])
        np.testing.assert_array_equal(od, g[pre + "out_d"])
        np.testing.assert_array_equal(op, g[pre + "out_p"])
        np.testing.assert_array_equal(osrc, g[pre + "source_d"])
        np.testing.assert_array_equal(ov, g[pre + "oracle_valid"])
        np.testing.assert_array_equal(od, g[pre + "oracle_d"])
        pd, pp, pv = backend.predict(g[pre + "in_d"], g[pre + "in_p"], g[pre + "in_valid"], R,
                                     tr, cal, F())
        np.testing.assert_array_equal(pv, g[pre + "predict_valid"])
        np.testing.assert_array_equal(pd, g[pre + "predict_d"])
        np.testing.assert_array_equal(pp, g[pre + "predict_p"])


def _check_step(res, g, pre):
    np.testing.assert_array_equal(res["valid"], g[pre + "state_valid"])
    np.testing.assert_array_equal(res["d"], g[pre + "state_d"])
    np.testing.assert_array_equal(res["p"], g[pre + "state_p"])
    np.testing.assert_array_equal(res["export_d"], g[pre + "export_d"])
    np.testing.assert_array_equal(res["export_valid"], g[pre + "export_valid"])
    np.testing.assert_array_equal(res["diff"], g[pre + "diff"])


def test_step_on_empty_state(backend):
    # test_temporal_filter.cpp:317-333
    g = golden("step_empty")
    res = backend.step(None, g["left"], g["right"], np.eye(3), np.zeros(3), Cal(g["calib"]),
                       P(g["params"]), F())
    _check_step(res, g, "")
    np.testing.assert_array_equal(res["export_d"], g["direct_median_d"])
    assert not res["diff"].any()


def test_static_scene_recursion(backend):
    # test_temporal_filter.cpp:335-356 (11 chained steps)
    g = golden("step_static")
    state = None
    for i in range(11):
        res = backend.step(state, g["left"], g["right"], np.eye(3), np.zeros(3),
                           Cal(g["calib"]), P(g["params"]), F())
        _check_step(res, g, f"{i}__")
        state = (res["d"], res["p"], res["valid"])


def test_moving_camera_recursion(backend):
    # harness recursion with the BASELINE penalties/stddev ranges: predict,
    # ranges, reduced SGM and the posterior every frame
    g = golden("step_moving")
    f = F(range_use_stddev=True, range_stddev_gain=3.0)
    cal, p = Cal(g["calib"]), P(g["params"])
    state = None
    for i in range(6):
        pre = f"{i}__"
        m = g[pre + "motion"]
        R, t = m[:9].reshape(3, 3), m[9:]
        res = backend.step(state, g["left"], g["right"], R, t, cal, p, f, debug=True)
        _check_step(res, g, pre)
        np.testing.assert_array_equal(res["pred_valid"], g[pre + "pred_valid"])
        np.testing.assert_array_equal(res["pred_d"], g[pre + "pred_d"])
        np.testing.assert_array_equal(res["pred_p"], g[pre + "pred_p"])
        np.testing.assert_array_equal(res["lo"], g[pre + "ranges_lo"])
        np.testing.assert_array_equal(res["hi"], g[pre + "ranges_hi"])
        np.testing.assert_array_equal(res["meas_d"], g[pre + "meas_d"])
        np.testing.assert_array_equal(res["meas_valid"], g[pre + "meas_valid"])
        state = (res["d"], res["p"], res["valid"])
