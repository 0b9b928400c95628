"""Batched detection on the engine's own diff maps:
config-1 scenes with movers, several sequences per launch; each slot's boxes
equal the oracle's detect_moving_objects on the oracle step's diff map."""
import dataclasses

import numpy as np
import pytest

from paper_1809_07986_b200 import tsgm
from paper_1809_07986_b200.scene import SceneConfig, render

pytestmark = pytest.mark.gpu


def test_engine_detect_matches_oracle(port):
    from oracle.oracle import DetectConfig
    cfgs = [SceneConfig.baseline_config(1, width=480, height=180, focal=280.0, cx=239.5,
                                        cy=89.5, d_max=64, seed=s, n_movers=3) for s in (2, 3, 4)]
    calib = tsgm.StereoCalib(280.0, 239.5, 89.5, cfgs[0].baseline, 480, 180, 64)
    params = tsgm.SgmParams(10, 120, 8, 0, 64)
    filt = tsgm.FilterConfig(range_use_stddev=True, range_stddev_gain=3.0)
    seqs = [render(c, 0, 5) for c in cfgs]
    eng = tsgm.Engine(tsgm.EngineConfig(calib, params, filt, max_slots=3, keep_volumes=False))
    states = [None] * 3
    det = DetectConfig(score_thresh=1.0, min_box_area=100)
    total = 0
    for k in range(5):
        mots = [(np.eye(3), np.zeros(3)) if k == 0 else tsgm.relative_motion(P[k - 1], P[k])
                for (_, _, P, _) in seqs]
        eng.step([0, 1, 2], [s[0][k] for s in seqs], [s[1][k] for s in seqs], mots)
        got = eng.detect([0, 1, 2], tsgm.DetectConfig(**dataclasses.asdict(det)))
        for i, (L, R, _, _) in enumerate(seqs):
            ref = port.step(states[i], L[k], R[k], mots[i][0], mots[i][1], calib, params, filt)
            np.testing.assert_array_equal(eng.fetch(i, "diff"), ref["diff"])
            want = port.detect(ref["diff"], det)
            np.testing.assert_array_equal(got[i], want)
            total += len(want)
            states[i] = (ref["d"], ref["p"], ref["valid"])
    assert total > 0  # the movers are found
    eng.close()


def test_random_maps_vs_oracle(port):
    """Dense random maps: many candidates, exact scores and order."""
    from oracle.oracle import DetectConfig
    for seed in range(4):
        rng = np.random.default_rng(seed)
        h, w = int(rng.integers(60, 300)), int(rng.integers(60, 700))
        diff = np.where(rng.random((h, w)) < 0.3, rng.uniform(0, 8, (h, w)), 0.0)
        c = DetectConfig(window_sizes=((12, 9), (20, 20), (33, 17), (50, 75)), score_thresh=1.5)
        np.testing.assert_array_equal(tsgm.integral_image(diff), port.integral_image(diff))
        np.testing.assert_array_equal(tsgm.detect_candidate_windows(diff, c),
                                      port.candidates(diff, c))
