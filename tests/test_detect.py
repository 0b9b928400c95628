"""Moving-object box detector (reference
src/motion_detect.cpp): the summed-area table, candidate windows, greedy merge
and end-to-end detection against golden vectors produced by the reference
(tests/golden/make_golden.cpp, det_*), for the oracle (port, CPU) and the
product (gpu). The product's greedy merge is host code (the incremental exact
form), so it is also checked here on the CPU against the reference's own
O(n^3) merge on random box sets. Bit-exact: integer boxes and FP64 scores."""
import dataclasses

import numpy as np
import pytest

from tests.backends import backend_fixture, golden

backend = backend_fixture()


def cfg(**kw):
    from oracle.oracle import DetectConfig
    return dataclasses.replace(DetectConfig(), **kw)


def test_sat_golden(backend):
    """test_motion_detect.cpp:60-69: SAT of a random integer map (seed 61)."""
    g = golden("det_sat")
    np.testing.assert_array_equal(backend.integral_image(g["map"]), g["sat"])


def test_sat_corners(backend):
    """test_motion_detect.cpp:24-37."""
    sat = backend.integral_image(np.ones((4, 5)))
    assert sat[0, 0] == 0.0 and sat[4, 5] == 20.0
    assert (sat[0, :] == 0).all() and (sat[:, 0] == 0).all()
    assert (backend.integral_image(np.zeros((6, 6))) == 0).all()


@pytest.mark.parametrize("name", ["hot", "rand", "flat"])
def test_candidates_golden(backend, name):
    """test_motion_detect.cpp:86-133: emitted windows, order and scores."""
    g = golden("det_cand")
    np.testing.assert_array_equal(backend.candidates(g[name], cfg()), g[name + "_boxes"])


def test_candidates_empty_and_top_third(backend):
    assert len(backend.candidates(np.zeros((120, 120)), cfg())) == 0
    top = np.zeros((120, 120))
    top[0:38, 40:80] = 50.0
    assert len(backend.candidates(top, cfg())) == 0


@pytest.mark.parametrize("seed", [63, 64])
def test_merge_golden(backend, seed):
    """test_motion_detect.cpp:165-195: random box sets."""
    g = golden("det_merge")
    inp = g[f"s{seed}__in"]
    np.testing.assert_array_equal(backend.greedy_merge(inp, cfg()), g[f"s{seed}__out_default"])
    np.testing.assert_array_equal(backend.greedy_merge(inp, cfg(min_box_area=0)),
                                  g[f"s{seed}__out_loose"])


def test_merge_kats(backend):
    """test_motion_detect.cpp:138-163, 196-201."""
    out = backend.greedy_merge([[10, 10, 40, 40, 2.0], [10, 10, 40, 40, 4.0]], cfg())
    assert out.shape == (1, 5) and out[0, 4] == 3.0
    assert len(backend.greedy_merge([[0, 0, 30, 30, 2.0], [60, 60, 90, 90, 2.0]], cfg())) == 2
    out = backend.greedy_merge([[0, 0, 20, 30, 3.0], [10, 0, 30, 30, 3.0], [20, 0, 40, 30, 3.0]],
                               cfg())
    np.testing.assert_array_equal(out, [[0, 0, 40, 30, 3.0]])
    out = backend.greedy_merge([[0, 0, 10, 10, 5.0], [100, 100, 150, 150, 5.0]], cfg())
    np.testing.assert_array_equal(out, [[100, 100, 150, 150, 5.0]])


@pytest.mark.parametrize("name,stop", [("block", 0.12), ("three", 0.2), ("kitti", 0.2)])
def test_detect_golden(backend, name, stop):
    """test_motion_detect.cpp:221-257, plus a KITTI-sized sparse map."""
    g = golden("det_e2e")
    np.testing.assert_array_equal(backend.detect(g[name], cfg(merge_stop_iou=stop)),
                                  g[name + "_boxes"])


def test_detect_kitti_candidates(backend):
    g = golden("det_e2e")
    np.testing.assert_array_equal(backend.candidates(g["kitti"], cfg()), g["kitti_cands"])


@pytest.mark.parametrize("bad", [dict(window_sizes=()), dict(score_thresh=0.0),
                                 dict(merge_stop_iou=1.0), dict(window_sizes=((0, 10),)),
                                 dict(min_box_area=-1)])
def test_config_validation(backend, bad):
    """test_motion_detect.cpp:260-274 (DetectConfig::validate)."""
    with pytest.raises(ValueError, match="DetectConfig"):
        backend.greedy_merge([[0, 0, 10, 10, 1.0]], cfg(**bad))


def test_host_merge_vs_reference_random(reference):
    """The product's incremental merge (host code, no GPU) against the
    reference's exhaustive merge on random sets with many ties and chains."""
    from paper_1809_07986_b200 import tsgm
    for seed in range(40):
        rng = np.random.default_rng(1000 + seed)
        n = int(rng.integers(0, 120))
        grid = int(rng.integers(2, 6))  # coarse coordinates: many equal IoUs
        x0 = rng.integers(0, 16, n) * grid
        y0 = rng.integers(0, 16, n) * grid
        w = rng.integers(2, 10, n) * grid
        h = rng.integers(2, 10, n) * grid
        b = np.stack([x0, y0, x0 + w, y0 + h, rng.uniform(0, 5, n)], 1).astype(float)
        c = cfg(min_box_area=int(rng.integers(0, 500)),
                merge_stop_iou=float(rng.uniform(0.05, 0.7)))
        np.testing.assert_array_equal(tsgm.greedy_merge(b, c), reference.greedy_merge(b, c))
