"""Pins the C oracle to the reference itself: the unmodified reference sources
compiled in place (oracle/_ref/libtsgm_ref.so) and the restatement must agree
bit-for-bit, stage by stage and through step(), on the BASELINE scenes and on
random inputs. CPU only."""
import numpy as np
import pytest

from oracle import Calib, FilterConfig, SgmParams
from paper_1809_07986_b200.scene import SceneConfig, render


@pytest.fixture(scope="module")
def scene():
    cfg = SceneConfig.baseline_config(1, width=400, height=160, focal=240.0, cx=199.5,
                                      cy=79.5, d_max=64, frames=5, seed=4, n_movers=3)
    return cfg, render(cfg)


def test_step_recursion_matches_reference(port, reference, scene):
    cfg, (L, R, P, _) = scene
    calib = Calib(cfg.focal, cfg.cx, cfg.cy, cfg.baseline, cfg.width, cfg.height, cfg.d_max)
    params = SgmParams(10, 120, 8, 0, cfg.d_max)
    filt = FilterConfig(range_use_stddev=True, range_stddev_gain=3.0)
    sa = sb = None
    for k in range(cfg.frames):
        Rm, t = (np.eye(3), np.zeros(3)) if k == 0 else reference.relative_motion(P[k - 1], P[k])
        Rp, tp = (np.eye(3), np.zeros(3)) if k == 0 else port.relative_motion(P[k - 1], P[k])
        np.testing.assert_array_equal(Rm, Rp)
        np.testing.assert_array_equal(t, tp)
        a = port.step(sa, L[k], R[k], Rm, t, calib, params, filt)
        b = reference.step(sb, L[k], R[k], Rm, t, calib, params, filt)
        for key in b:
            np.testing.assert_array_equal(a[key], b[key], err_msg=f"frame {k} {key}")
        sa = (a["d"], a["p"], a["valid"])
        sb = (b["d"], b["p"], b["valid"])


def test_stages_match_reference_on_random_inputs(port, reference):
    rng = np.random.default_rng(99)
    h, w, d = 30, 50, 24
    l = rng.integers(0, 256, (h, w)).astype(np.uint8)
    r = rng.integers(0, 256, (h, w)).astype(np.uint8)
    np.testing.assert_array_equal(port.census(l), reference.census(l))
    a, b = rng.integers(0, d, (h, w)), rng.integers(0, d, (h, w))
    lo, hi = np.minimum(a, b).astype(np.uint16), np.maximum(a, b).astype(np.uint16)
    o1, c1 = port.cost_volume(l, r, lo, hi)
    o2, c2 = reference.cost_volume(l, r, lo, hi)
    np.testing.assert_array_equal(o1, o2)
    np.testing.assert_array_equal(c1, c2)
    for paths, ps in ((8, 0), (4, 0), (4, 1)):
        p = SgmParams(7, 90, paths, ps, d)
        agg = port.aggregate(c1, lo, hi, p)
        np.testing.assert_array_equal(agg, reference.aggregate(c1, lo, hi, p))
        np.testing.assert_array_equal(port.wta(agg, lo, hi)[0], reference.wta(agg, lo, hi)[0])
    # state stages on a random state with a random motion
    sd = rng.uniform(1, d - 1, (h, w))
    sp = rng.uniform(0.1, 20, (h, w))
    sv = (rng.random((h, w)) < 0.8).astype(np.uint8)
    calib = Calib(80.0, 24.5, 14.5, 0.5, w, h, d)
    ang = 0.02
    Rm = np.array([[np.cos(ang), 0, np.sin(ang)], [0, 1, 0], [-np.sin(ang), 0, np.cos(ang)]])
    t = np.array([0.05, -0.01, -0.2])
    np.testing.assert_array_equal(port.homography(Rm, t, calib), reference.homography(Rm, t, calib))
    H = port.homography(Rm, t, calib)
    for x, y in zip(port.warp(sd, sp, sv, H, d), reference.warp(sd, sp, sv, H, d)):
        np.testing.assert_array_equal(x, y)
    f = FilterConfig(range_use_stddev=True, range_stddev_gain=3.0)
    for x, y in zip(port.predict(sd, sp, sv, Rm, t, calib, f),
                    reference.predict(sd, sp, sv, Rm, t, calib, f)):
        np.testing.assert_array_equal(x, y)
    for x, y in zip(port.ranges(sd, sp, sv, calib, f), reference.ranges(sd, sp, sv, calib, f)):
        np.testing.assert_array_equal(x, y)
    md = rng.integers(0, d, (h, w)).astype(np.int32)
    mv = (rng.random((h, w)) < 0.7).astype(np.uint8)
    for x, y in zip(port.correct(sd, sp, sv, md, mv, f), reference.correct(sd, sp, sv, md, mv, f)):
        np.testing.assert_array_equal(x, y)
    np.testing.assert_array_equal(port.diff(sd, sp, sv, md, mv), reference.diff(sd, sp, sv, md, mv))
    m1, m2 = port.median(md, mv), reference.median(md, mv)
    np.testing.assert_array_equal(m1[0], m2[0])
    np.testing.assert_array_equal(m1[1], m2[1])


def test_reference_error_behaviour_matches(port, reference):
    l = np.zeros((12, 20), np.uint8)
    calib = Calib(200.0, 10.0, 6.0, 0.4, 20, 12, 16)
    for impl in (port, reference):
        with pytest.raises(ValueError):
            impl.step(None, l, l, np.eye(3), np.zeros(3), calib, SgmParams(d_max=32), FilterConfig())
        bad = np.eye(3)
        bad[0, 0] = 2.0
        with pytest.raises(ValueError):
            impl.step(None, l, l, bad, np.zeros(3), calib, SgmParams(d_max=16), FilterConfig())
