"""KITTI-style outlier count (reference src/eval.cpp:59-93)
against the reference's golden counts (tests/golden/make_golden.cpp,
eval_outliers) and the hand KATs of test_eval.cpp, for the oracle (port, CPU)
and the product (gpu). Exact integer counts."""
import numpy as np
import pytest

from tests.backends import backend_fixture, golden

backend = backend_fixture()


@pytest.mark.parametrize("case", range(4))
@pytest.mark.parametrize("strict", [False, True])
def test_golden(backend, case, strict):
    g = golden("eval_outliers")
    ev, out = backend.count_outliers(g[f"{case}__d"], g[f"{case}__valid"], g[f"{case}__gt"],
                                     strict=strict)
    assert [ev, out] == list(g[f"{case}__counts_strict{int(strict)}"])


def _fixture(n, cases):
    d = np.zeros((1, n), np.int32)
    v = np.zeros((1, n), np.uint8)
    gt = np.zeros((1, n))
    for x, (est, g) in cases.items():
        d[0, x], v[0, x], gt[0, x] = est, 1, g
    return d, v, gt


def test_gates(backend):
    """test_eval.cpp:45-74: absolute AND relative gates, strict density."""
    d, v, gt = _fixture(6, {0: (14, 10.0), 1: (104, 100.0), 2: (10, 10.0), 3: (77, 80.0),
                            4: (10, 20.0)})
    gt[0, 5] = 50.0
    assert backend.count_outliers(d, v, gt) == (5, 2)
    assert backend.count_outliers(d, v, gt, strict=True) == (6, 3)


def test_ten_pixel_percentage(backend):
    """test_eval.cpp:76-89: 50% exactly."""
    d, v, gt = _fixture(10, {0: (14, 10.0), 1: (104, 100.0), 2: (12, 12.0), 3: (6, 2.0),
                             4: (77, 80.0), 5: (36, 40.0), 6: (195, 200.0), 7: (10, 20.0),
                             8: (7, 7.0), 9: (54, 50.5)})
    ev, out = backend.count_outliers(d, v, gt)
    assert 100.0 * out / ev == 50.0


@pytest.mark.gpu
def test_outlier_rate_errors():
    from paper_1809_07986_b200 import tsgm
    d = np.zeros((2, 2), np.int32)
    v = np.ones((2, 2), np.uint8)
    with pytest.raises(RuntimeError, match="no mutually valid"):
        tsgm.outlier_rate(d, v, np.zeros((2, 2)))
    with pytest.raises(ValueError, match="dimension"):
        tsgm.count_outliers(d, v, np.zeros((3, 2)))


@pytest.mark.gpu
def test_engine_batch_vs_oracle(port):
    """Batched on the engine's own export and WTA maps against the synthetic
    ground truth of config-1 scenes."""
    from paper_1809_07986_b200 import tsgm
    from paper_1809_07986_b200.scene import SceneConfig, render
    cfgs = [SceneConfig.baseline_config(1, width=320, height=120, focal=200.0, cx=159.5,
                                        cy=59.5, d_max=64, seed=s, n_movers=2) for s in (1, 2)]
    calib = tsgm.StereoCalib(200.0, 159.5, 59.5, cfgs[0].baseline, 320, 120, 64)
    params = tsgm.SgmParams(10, 120, 8, 0, 64)
    filt = tsgm.FilterConfig(range_use_stddev=True, range_stddev_gain=3.0)
    seqs = [render(c, 0, 3, gt=True) for c in cfgs]
    eng = tsgm.Engine(tsgm.EngineConfig(calib, params, filt, max_slots=2, keep_volumes=False))
    for k in range(3):
        mots = [(np.eye(3), np.zeros(3)) if k == 0 else tsgm.relative_motion(P[k - 1], P[k])
                for (_, _, P, _) in seqs]
        eng.step([0, 1], [s[0][k] for s in seqs], [s[1][k] for s in seqs], mots)
        gts = [s[3][k].astype(np.float64) for s in seqs]
        for what, dk, vk in (("export_d", "export_d", "export_valid"),
                             ("meas_d", "meas_d", "meas_valid")):
            for strict in (False, True):
                ev, out = eng.count_outliers([0, 1], gts, what,
                                             tsgm.OutlierOptions(strict_density=strict))
                for i in range(2):
                    want = port.count_outliers(eng.fetch(i, dk), eng.fetch(i, vk), gts[i],
                                               strict=strict)
                    assert (int(ev[i]), int(out[i])) == want
                    assert ev[i] > 0
    eng.close()
