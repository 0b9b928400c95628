"""Noise calibration on the GPU: the KATs of the reference's
tests/test_noise_calib.cpp (:88-209) retargeted at the product, and the batched
path (more frames than one launch batch) against the oracle port."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1809_07986_b200 import tsgm
from paper_1809_07986_b200.scene import SceneConfig, render
from paper_1809_07986_b200.testing import GpuBackend

pytestmark = pytest.mark.gpu


def _scene(frames, noise_sigma=2.0, **kw):
    base = dict(width=120, height=90, focal=200.0, cx=59.5, cy=44.5, d_max=64, seed=9,
                frames=frames, noise_sigma=noise_sigma)
    base.update(kw)
    cfg = SceneConfig.baseline_config(0, **base)
    left, right, poses, gt = render(cfg, gt=True)
    calib = tsgm.StereoCalib(cfg.focal, cfg.cx, cfg.cy, cfg.baseline, cfg.width, cfg.height,
                             cfg.d_max)
    frames_ = GpuBackend._frames(gt.astype(np.float64), poses, left, right)
    return frames_, calib, cfg


def test_static_camera_zero_process_noise():
    """:88-94: an unmoving camera over a static scene has zero process noise."""
    fr, calib, _ = _scene(3, fwd_m=0.0, yaw_deg=0.0)
    est = tsgm.estimate_process_noise(fr, calib)
    assert est.variance == 0.0
    assert est.samples_used > 0
    assert est.hist.fraction_within_1px() == 1.0


def test_non_overlapping_ground_truth():
    """:121-147: ground truths that never overlap are a runtime error."""
    a = np.zeros((20, 20))
    b = np.zeros((20, 20))
    a[:, 2] = 15.0
    b[:, 17] = 15.0
    pose = np.hstack([np.eye(3), np.zeros((3, 1))])
    fr = [tsgm.SequenceFrame(0, None, None, pose, a), tsgm.SequenceFrame(1, None, None, pose, b)]
    calib = tsgm.StereoCalib(100.0, 9.5, 9.5, 1.0, 20, 20, 64)
    with pytest.raises(RuntimeError, match="no overlapping valid pixels"):
        tsgm.estimate_process_noise(fr, calib)
    with pytest.raises(RuntimeError, match="no overlapping valid pixels"):
        tsgm.accumulate_error_map(fr, calib)


def test_measurement_noise_grows_with_image_noise():
    """:150-158."""
    prev = -1.0
    for sigma in (0.0, 10.0, 25.0):
        fr, _, cfg = _scene(2, noise_sigma=sigma)
        est = tsgm.estimate_measurement_noise(fr, tsgm.SgmParams(d_max=cfg.d_max))
        assert est.variance > prev
        prev = est.variance


def test_measurement_noise_frames_in_isolation():
    """:160-169: swapping the frames leaves the estimate unchanged."""
    fr, _, cfg = _scene(2, noise_sigma=12.0)
    p = tsgm.SgmParams(d_max=cfg.d_max)
    fwd = tsgm.estimate_measurement_noise(fr, p)
    swp = tsgm.estimate_measurement_noise([fr[1], fr[0]], p)
    assert fwd.variance == pytest.approx(swp.variance, rel=1e-12)
    assert fwd.hist.total() == swp.hist.total()
    np.testing.assert_array_equal(fwd.hist.counts, swp.hist.counts)


def test_error_map_adds_up_over_repeated_pairs():
    """:171-191: [s0, s1, s0, s1] accumulates 3x the map of [s0, s1]; errors
    only where the mover went."""
    fr, calib, _ = _scene(2, n_movers=1, n_static=0, fwd_m=0.0, yaw_deg=0.0)
    once = tsgm.accumulate_error_map(fr[:2], calib)
    thrice = tsgm.accumulate_error_map([fr[0], fr[1], fr[0], fr[1]], calib)
    np.testing.assert_allclose(thrice, 3.0 * once, rtol=1e-12, atol=0.0)
    assert once.sum() > 0.0


def test_zero_error_sequence_zero_map():
    """:193-199."""
    fr, calib, _ = _scene(3, fwd_m=0.0, yaw_deg=0.0)
    assert not tsgm.accumulate_error_map(fr, calib).any()


def test_batched_against_port(port):
    """35 frames = five launch batches (8 + 8 + 8 + 8 + 3) of frames: counts,
    tallies and the error map bit-exact vs the port; moments to 1e-9."""
    cfg = SceneConfig.baseline_config(1, width=72, height=48, focal=60.0, cx=35.5, cy=23.5,
                                      d_max=32, seed=4, n_movers=2, frames=35)
    left, right, poses, gt = render(cfg, gt=True)
    gt = gt.astype(np.float64)
    p12 = poses.reshape(-1, 12)
    calib = O.Calib(cfg.focal, cfg.cx, cfg.cy, cfg.baseline, cfg.width, cfg.height, cfg.d_max)
    opts = O.CalibOpts(6.0, 0.5, 0.1)
    sgm = O.SgmParams(10, 120, 8, 0, cfg.d_max)
    gpu = GpuBackend.shared()
    for got, want in ((gpu.process_noise(gt, p12, calib, opts),
                       port.process_noise(gt, p12, calib, opts)),
                      (gpu.measurement_noise(left, right, gt, sgm, opts),
                       port.measurement_noise(left, right, gt, sgm, opts))):
        for k in ("samples_used", "total", "underflow", "overflow"):
            assert got[k] == want[k], k
        np.testing.assert_array_equal(got["counts"], want["counts"])
        np.testing.assert_allclose([got["variance"], got["mean"]], [want["variance"], want["mean"]],
                                   rtol=1e-9)
    np.testing.assert_array_equal(gpu.error_map(gt, p12, calib), port.error_map(gt, p12, calib))
