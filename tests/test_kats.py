"""The reference's hand-constructed known-answer tests, restated against the
oracle (CPU) and the GPU path. Each test cites the reference test it restates
(/root/reference/proj/tests/...). Fixture-seeded (mt19937) cases live in
tests/test_golden.py instead."""
import numpy as np
import pytest

from tests.backends import backend_fixture

backend = backend_fixture()


class P:
    def __init__(self, p1=6, p2=65, paths=8, path_set=0, d_max=128):
        self.p1, self.p2, self.paths, self.path_set, self.d_max = p1, p2, paths, path_set, d_max


class F:
    def __init__(self, **kw):
        self.q, self.r, self.p_init, self.disc_thresh = 0.5, 1.0, 4096.0, 2.0
        self.min_range_halfwidth, self.range_use_stddev, self.range_stddev_gain = 2, False, 2.0
        self.__dict__.update(kw)


class Cal:
    def __init__(self, w, h, d_max, f=200.0, b=0.4):
        self.focal_px, self.cx, self.cy, self.baseline_m = f, w / 2.0, h / 2.0, b
        self.width, self.height, self.d_max = w, h, d_max


def state(w, h):
    return np.zeros((h, w)), np.zeros((h, w)), np.zeros((h, w), np.uint8)


def put(s, x, y, d, p):
    s[0][y, x], s[1][y, x], s[2][y, x] = d, p, 1


# ------------------------------------------------------------ census / cost
def test_census_constant_image_is_zero(backend):
    # test_matching_cost.cpp:10-19
    sig = backend.census(np.full((7, 9), 140, np.uint8))
    assert not sig.any()


def test_census_all_darker_sets_24_bits(backend):
    # test_matching_cost.cpp:21-26
    img = np.full((9, 9), 4, np.uint8)
    img[4, 4] = 5
    assert backend.census(img)[4, 4] == 0x00FFFFFF


def test_census_bit_positions(backend):
    # test_matching_cost.cpp:28-40
    img = np.full((9, 9), 100, np.uint8)
    img[2, 2] = 10
    assert backend.census(img)[4, 4] == 1 << 23
    img[2, 2], img[6, 6] = 100, 10
    assert backend.census(img)[4, 4] == 1
    img[6, 6], img[4, 5] = 100, 10
    assert backend.census(img)[4, 4] == 1 << 11


def test_census_equal_neighbours_and_offsets(backend):
    # test_matching_cost.cpp:42-46, 59-71
    assert backend.census(np.full((9, 9), 77, np.uint8))[4, 4] == 0
    rng = np.random.default_rng(12)
    img = rng.integers(0, 201, (9, 11)).astype(np.uint8)
    np.testing.assert_array_equal(backend.census(img), backend.census(img + 30))


def test_undersized_images_rejected(backend):
    # test_matching_cost.cpp:73-76
    with pytest.raises(ValueError):
        backend.census(np.zeros((9, 4), np.uint8))
    with pytest.raises(ValueError):
        backend.census(np.zeros((4, 9), np.uint8))


def test_cost_volume_full_range_size_and_degenerate(backend):
    # test_matching_cost.cpp:120-144
    rng = np.random.default_rng(15)
    l = rng.integers(0, 256, (7, 10)).astype(np.uint8)
    r = rng.integers(0, 256, (7, 10)).astype(np.uint8)
    off, cost = backend.cost_volume(l, r, np.zeros((7, 10), np.uint16),
                                    np.full((7, 10), 5, np.uint16))
    assert off[-1] == 10 * 7 * 6 and cost.size == 420
    off, cost = backend.cost_volume(l, r, np.full((7, 10), 3, np.uint16),
                                    np.full((7, 10), 3, np.uint16))
    assert cost.size == 70 and (cost <= 24).all()


# ------------------------------------------------------------ aggregation / WTA / median
def test_single_pixel_aggregates_to_paths_times_cost(backend):
    # test_sgm.cpp:35-48
    cost = np.array([7, 0, 24, 3], np.uint8)
    lo, hi = np.zeros((1, 1), np.uint16), np.full((1, 1), 3, np.uint16)
    for paths in (4, 8):
        np.testing.assert_array_equal(backend.aggregate(cost, lo, hi, P(paths=paths)),
                                      paths * cost.astype(np.uint16))


def test_uniform_volume(backend):
    # test_sgm.cpp:60-71
    lo, hi = np.zeros((5, 7), np.uint16), np.full((5, 7), 5, np.uint16)
    agg = backend.aggregate(np.full(5 * 7 * 6, 9, np.uint8), lo, hi, P())
    assert (agg == 72).all()


def test_normalisation_envelope(backend):
    # test_sgm.cpp:104-119
    rng = np.random.default_rng(24)
    a = rng.integers(0, 7, (8, 10))
    b = rng.integers(0, 7, (8, 10))
    lo, hi = np.minimum(a, b).astype(np.uint16), np.maximum(a, b).astype(np.uint16)
    n = int((hi.astype(int) - lo + 1).sum())
    cost = rng.integers(0, 25, n).astype(np.uint8)
    agg = backend.aggregate(cost, lo, hi, P()).astype(int)
    assert (agg >= 8 * cost).all() and (agg <= 8 * (cost.astype(int) + 65)).all()


def test_wta_argmin_ties_and_border(backend):
    # test_sgm.cpp:126-160
    lo, hi = np.full((7, 7), 3, np.uint16), np.full((7, 7), 5, np.uint16)
    agg = np.zeros(49 * 3, np.uint16)
    i = 3 * 7 + 3
    agg[3 * i:3 * i + 3] = [5, 2, 9]
    d, v = backend.wta(agg, lo, hi)
    assert v[3, 3] and d[3, 3] == 4
    lo, hi = np.zeros((7, 7), np.uint16), np.ones((7, 7), np.uint16)
    agg = np.zeros(98, np.uint16)
    agg[2 * i:2 * i + 2] = [2, 2]
    assert backend.wta(agg, lo, hi)[0][3, 3] == 0
    lo, hi = np.zeros((8, 8), np.uint16), np.full((8, 8), 2, np.uint16)
    _, v = backend.wta(np.zeros(64 * 3, np.uint16), lo, hi)
    ys, xs = np.mgrid[0:8, 0:8]
    np.testing.assert_array_equal(v, ((xs >= 2) & (xs < 6) & (ys >= 2) & (ys < 6)).astype(np.uint8))


def test_median_kats(backend):
    # test_sgm.cpp:180-218
    d, v = backend.median(np.full((6, 6), 14, np.int32), np.ones((6, 6), np.uint8))
    corner = np.zeros((6, 6), bool)
    corner[[0, 0, 5, 5], [0, 5, 0, 5]] = True
    np.testing.assert_array_equal(v, (~corner).astype(np.uint8))
    assert (d[v > 0] == 14).all()
    dm = np.full((7, 7), 10, np.int32)
    dm[3, 3] = 100
    assert backend.median(dm, np.ones((7, 7), np.uint8))[0][3, 3] == 10
    dm, vv = np.zeros((5, 5), np.int32), np.zeros((5, 5), np.uint8)
    dm[2, 2], vv[2, 2] = 8, 1
    assert not backend.median(dm, vv)[1].any()
    vv = np.ones((5, 5), np.uint8)
    vv[2, 2] = 0
    d, v = backend.median(np.full((5, 5), 21, np.int32), vv)
    assert v[2, 2] and d[2, 2] == 21


def test_degenerate_single_level_ranges_force_output(backend):
    # test_sgm.cpp:252-262
    rng = np.random.default_rng(29)
    l = rng.integers(0, 256, (12, 20)).astype(np.uint8)
    r = rng.integers(0, 256, (12, 20)).astype(np.uint8)
    d, v = backend.sgm_match(l, r, np.full((12, 20), 6, np.uint16),
                             np.full((12, 20), 6, np.uint16), P(d_max=16))
    assert (d[2:10, 2:18] == 6).all() and v[2:10, 2:18].all()


def test_sgm_params_validation(backend):
    # test_sgm.cpp:276-290 (sgm_match validates its params)
    l = np.zeros((8, 8), np.uint8)
    lo, hi = np.zeros((8, 8), np.uint16), np.full((8, 8), 3, np.uint16)
    for bad in (P(p1=0, d_max=8), P(p1=70, d_max=8), P(paths=6, d_max=8)):
        with pytest.raises(ValueError):
            backend.sgm_match(l, l, lo, hi, bad)
    with pytest.raises(ValueError):  # range outside [0, d_max)
        backend.sgm_match(l, l, lo, np.full((8, 8), 8, np.uint16), P(d_max=8))


# ------------------------------------------------------------ temporal filter
def test_identity_prediction_inflates_variance_by_q(backend):
    # test_temporal_filter.cpp:35-47
    s = state(20, 16)
    s[0][:], s[1][:], s[2][:] = 10.0, 2.0, 1
    d, p, v = backend.predict(*s, np.eye(3), np.zeros(3), Cal(20, 16, 64), F())
    assert v.all() and (d == 10.0).all() and (p == 2.5).all()


def test_prediction_of_invalid_state_stays_invalid(backend):
    # test_temporal_filter.cpp:49-55
    _, _, v = backend.predict(*state(12, 10), np.eye(3), np.zeros(3), Cal(12, 10, 64), F())
    assert not v.any()


def test_forward_motion_grows_disparity_and_variance(backend):
    # test_temporal_filter.cpp:57-73
    s = state(64, 48)
    s[0][:], s[1][:], s[2][:] = 20.0, 2.0, 1
    d, p, v = backend.predict(*s, np.eye(3), np.array([0.0, 0.0, -1.0]), Cal(64, 48, 64), F())
    inner = v[10:38, 10:54] > 0
    assert inner.sum() > 500
    assert (d[10:38, 10:54][inner] > 20.0).all() and (p[10:38, 10:54][inner] > 2.5).all()


def test_discontinuity_rejection(backend):
    # test_temporal_filter.cpp:75-115
    s = state(16, 8)
    s[0][:] = 0.5 * np.arange(16)
    s[1][:], s[2][:] = 1.0, 1
    assert backend.reject(*s, F())[2].all()
    s[0][:] = np.where(np.arange(16) < 8, 10.0, 20.0)
    _, _, v = backend.reject(*s, F())
    np.testing.assert_array_equal(v[0], [0 if x in (7, 8) else 1 for x in range(16)])
    assert not backend.reject(*state(6, 6), F())[2].any()
    s = state(9, 3)
    s[0][:] = np.where(np.arange(9) < 3, 0.0, np.where(np.arange(9) < 6, 10.0, 20.0))
    s[1][:], s[2][:] = 1.0, 1
    _, _, v = backend.reject(*s, F())
    np.testing.assert_array_equal(v[1], [1, 1, 0, 0, 1, 0, 0, 1, 1])


def test_zoom_hole_filling(backend):
    # test_temporal_filter.cpp:117-168
    s = state(5, 5)
    put(s, 1, 2, 10.0, 2.0)
    put(s, 3, 2, 12.0, 4.0)
    d, p, v = backend.fill(*s)
    assert v[2, 2] and d[2, 2] == 11.0 and p[2, 2] == 3.0
    put(s, 2, 1, 20.0, 6.0)
    put(s, 2, 3, 30.0, 8.0)
    d, p, v = backend.fill(*s)
    assert d[2, 2] == 18.0 and p[2, 2] == 5.0
    s = state(5, 5)
    put(s, 1, 2, 10.0, 2.0)
    assert not backend.fill(*s)[2][2, 2]
    s = state(9, 6)
    s[0][:], s[1][:], s[2][:] = 25.0, 1.5, 1
    s[2][:, 4] = 0
    s[0][:, 4] = s[1][:, 4] = 0
    d, p, v = backend.fill(*s)
    assert v[:, 4].all() and (d[:, 4] == 25.0).all() and (p[:, 4] == 1.5).all()
    s = state(10, 6)
    s[0][:], s[1][:], s[2][:] = 25.0, 1.5, 1
    s[2][:, 4:6] = 0
    assert not backend.fill(*s)[2][:, 4:6].any()


def test_search_range_derivation(backend):
    # test_temporal_filter.cpp:170-202
    s = state(8, 4)
    put(s, 0, 0, 40.0, 3.0)
    put(s, 1, 0, 2.0, 5.0)
    put(s, 2, 0, 40.0, 0.1)
    put(s, 3, 0, 126.5, 4.0)
    lo, hi = backend.ranges(*s, Cal(8, 4, 128), F())
    assert (lo[0, 0], hi[0, 0]) == (37, 43)
    assert (lo[0, 1], hi[0, 1]) == (0, 7)
    assert (lo[0, 2], hi[0, 2]) == (38, 42)
    assert hi[0, 3] == 127
    assert (lo[0, 4], hi[0, 4]) == (0, 127)
    t = state(8, 4)
    put(t, 0, 0, 40.0, 9.0)
    lo, hi = backend.ranges(*t, Cal(8, 4, 128), F(range_use_stddev=True, range_stddev_gain=2.0))
    assert (lo[0, 0], hi[0, 0]) == (34, 46)


def test_ranges_nonempty_and_inside(backend):
    # test_temporal_filter.cpp:204-223
    rng = np.random.default_rng(51)
    for _ in range(5):
        s = state(24, 18)
        keep = rng.integers(0, 4, (18, 24)) > 0
        s[0][keep] = rng.uniform(0.5, 63.5, keep.sum())
        s[1][keep] = rng.uniform(0.01, 300.0, keep.sum())
        s[2][keep] = 1
        lo, hi = backend.ranges(*s, Cal(24, 18, 64), F())
        assert (lo <= hi).all() and (hi < 64).all() and (hi.astype(int) - lo + 1 >= 5).all()


def test_measurement_correction(backend):
    # test_temporal_filter.cpp:225-268
    pred = state(3, 3)
    put(pred, 1, 1, 10.0, 1.0)
    md, mv = np.zeros((3, 3), np.int32), np.zeros((3, 3), np.uint8)
    md[1, 1], mv[1, 1] = 14, 1
    d, p, v = backend.correct(*pred, md, mv, F())
    assert d[1, 1] == 12.0 and p[1, 1] == 0.5
    md, mv = np.zeros((3, 3), np.int32), np.zeros((3, 3), np.uint8)
    md[0, 2], mv[0, 2] = 7, 1
    d, p, v = backend.correct(*state(3, 3), md, mv, F())
    assert v[0, 2] and d[0, 2] == 7.0 and p[0, 2] == 1.0
    pred = state(3, 3)
    put(pred, 0, 2, 33.0, 8.0)
    d, p, v = backend.correct(*pred, np.zeros((3, 3), np.int32), np.zeros((3, 3), np.uint8), F())
    assert v[2, 0] and d[2, 0] == 33.0 and p[2, 0] == 8.0
    assert not backend.correct(*state(3, 3), np.zeros((3, 3), np.int32),
                               np.zeros((3, 3), np.uint8), F())[2].any()


def test_kalman_closed_form_100_steps(backend):
    # test_temporal_filter.cpp:293-315 (scalar KF, 1e-12)
    w, h = 12, 10
    md, mv = np.full((h, w), 10, np.int32), np.ones((h, w), np.uint8)
    s = backend.correct(*state(w, h), md, mv, F())
    d_ref, p_ref = 10.0, 1.0
    for _ in range(100):
        s = backend.predict(*s, np.eye(3), np.zeros(3), Cal(w, h, 64), F())
        s = backend.correct(*s, md, mv, F())
        p_ref = p_ref + 0.5
        k = p_ref / (p_ref + 1.0)
        d_ref = d_ref + k * (10.0 - d_ref)
        p_ref = (1.0 - k) * p_ref
        assert abs(s[0][5, 6] - d_ref) <= 1e-12 and abs(s[1][5, 6] - p_ref) <= 1e-12


def test_step_rejects_inconsistent_inputs(backend):
    # test_temporal_filter.cpp:358-368
    cal = Cal(20, 12, 16)
    l = np.zeros((12, 20), np.uint8)
    with pytest.raises(ValueError):
        backend.step(None, l, l, np.eye(3), np.zeros(3), cal, P(d_max=32), F())


# ------------------------------------------------------------ geometry
def test_identity_homography_and_warp(backend):
    # test_geometry.cpp:82-91, 178-190
    cal = Cal(320, 240, 128, f=240.0, b=0.5)
    cal.cx, cal.cy = 160.0, 120.0
    H = backend.homography(np.eye(3), np.zeros(3), cal)
    np.testing.assert_array_equal(H, np.eye(4))
    rng = np.random.default_rng(44)
    s = state(12, 9)
    ys, xs = np.mgrid[0:9, 0:12]
    keep = (xs + ys) % 3 != 0
    s[0][keep], s[1][keep], s[2][keep] = rng.uniform(1, 100, keep.sum()), rng.uniform(1, 100, keep.sum()), 1
    d, p, v, _ = backend.warp(*s, H, 128)
    np.testing.assert_array_equal(v, s[2])
    np.testing.assert_array_equal(d, s[0])
    np.testing.assert_array_equal(p, s[1])


def test_warp_collision_larger_disparity_wins(backend):
    # test_geometry.cpp:191-203
    cal = Cal(320, 240, 128, f=240.0, b=0.5)
    cal.cx, cal.cy = 160.0, 120.0
    H = backend.homography(np.eye(3), np.array([-0.5, 0.0, 0.0]), cal)
    s = state(64, 16)
    put(s, 40, 8, 10.0, 1.0)
    put(s, 60, 8, 30.0, 2.0)
    d, p, v, _ = backend.warp(*s, H, 128)
    assert v[8, 30] and abs(d[8, 30] - 30.0) < 1e-9 and p[8, 30] == 2.0


def test_homography_rejects_degenerate_calibration(backend):
    # test_geometry.cpp:138-145, 147-155
    cal = Cal(320, 240, 128, f=0.0)
    with pytest.raises(ValueError):
        backend.homography(np.eye(3), np.zeros(3), cal)
    cal = Cal(320, 240, 128)
    bad = np.eye(3)
    bad[0, 0] = 2.0
    with pytest.raises(ValueError):
        backend.homography(bad, np.zeros(3), cal)


def test_relative_motion_from_poses(backend):
    # test_geometry.cpp:273-291
    a = np.array([1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0], float)
    b = np.array([1, 0, 0, 1.5, 0, 1, 0, 0, 0, 0, 1, 2.0], float)
    R, t = backend.relative_motion(a, b)
    p = R @ np.array([0.0, 0.0, 10.0]) + t
    np.testing.assert_allclose(p, [-1.5, 0.0, 8.0], atol=1e-12)
    R, t = backend.relative_motion(a, a)
    np.testing.assert_array_equal(R, np.eye(3))
    assert not t.any()
