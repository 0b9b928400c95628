"""GPU parity on the BASELINE scenes: the batched Engine (C-ABI context, several
sequences per launch) against the C oracle, frame by frame, every output and
intermediate, bit-exact (integer stages and the FP64 state alike: the FP64
kernels mirror the reference's operation order without FMA, so the 1e-4
relative gate of north_star is met with zero error)."""
import numpy as np
import pytest

from paper_1809_07986_b200 import tsgm
from paper_1809_07986_b200.scene import SceneConfig, render

pytestmark = pytest.mark.gpu

OUTS = [("d", "state_d"), ("p", "state_p"), ("valid", "state_valid"),
        ("export_d", "export_d"), ("export_valid", "export_valid"), ("diff", "diff"),
        ("pred_d", "pred_d"), ("pred_p", "pred_p"), ("pred_valid", "pred_valid"),
        ("lo", "lo"), ("hi", "hi"), ("meas_d", "meas_d"), ("meas_valid", "meas_valid"),
        ("mask", "mask")]


def run_parity(port, cfgs, frames, params, filt, check_volumes=False, vol_slots=0):
    calib = tsgm.StereoCalib(cfgs[0].focal, cfgs[0].cx, cfgs[0].cy, cfgs[0].baseline,
                             cfgs[0].width, cfgs[0].height, cfgs[0].d_max)
    seqs = [render(c, 0, frames) for c in cfgs]
    eng = tsgm.Engine(tsgm.EngineConfig(calib, params, filt, max_slots=len(cfgs) + 1,
                                        vol_slots=vol_slots))
    if vol_slots:
        assert eng.vol_slots == vol_slots
    # use non-contiguous slots to exercise the slot indirection
    slots = [i + 1 for i in range(len(cfgs))][::-1]
    states = [None] * len(cfgs)
    for k in range(frames):
        motions = []
        for (_, _, poses, _) in seqs:
            motions.append((np.eye(3), np.zeros(3)) if k == 0 else
                           tsgm.relative_motion(poses[k - 1], poses[k]))
        eng.step(slots, [s[0][k] for s in seqs], [s[1][k] for s in seqs], motions)
        for i, (L, R, _, _) in enumerate(seqs):
            ref = port.step(states[i], L[k], R[k], motions[i][0], motions[i][1], calib, params,
                            filt, debug=True)
            for rk, gk in OUTS:
                got = eng.fetch(slots[i], gk)
                assert np.array_equal(got, ref[rk]), f"seq {i} frame {k}: {gk} differs"
            if check_volumes and k < 2:
                off, cost = port.cost_volume(L[k], R[k], ref["lo"], ref["hi"])
                np.testing.assert_array_equal(eng.fetch(slots[i], "offsets"), off)
                np.testing.assert_array_equal(eng.fetch(slots[i], "cost"), cost)
                agg = port.aggregate(cost, ref["lo"], ref["hi"], params)
                np.testing.assert_array_equal(eng.fetch(slots[i], "agg"), agg)
            states[i] = (ref["d"], ref["p"], ref["valid"])
    eng.close()


def test_config0_full_size(port):
    """BASELINE config 0 at full 1242x375 (8 frames, D=128, P1=10, P2=120)."""
    cfg = SceneConfig.baseline_config(0)
    run_parity(port, [cfg], 8, tsgm.SgmParams(10, 120, 8, 0, 128),
               tsgm.FilterConfig(range_use_stddev=True, range_stddev_gain=3.0),
               check_volumes=True)


@pytest.mark.parametrize("vol_slots", [1, 2])
def test_volume_chunks(port, vol_slots):
    """A batch larger than the volume working set runs the matching stages in
    chunks (config 4's memory plan): every output still bit-exact."""
    cfgs = [SceneConfig.baseline_config(1, width=256, height=96, focal=160.0, cx=127.5,
                                        cy=47.5, d_max=48, seed=s, n_movers=2) for s in range(5)]
    run_parity(port, cfgs, 4, tsgm.SgmParams(10, 120, 8, 0, 48),
               tsgm.FilterConfig(range_use_stddev=True, range_stddev_gain=3.0),
               vol_slots=vol_slots)


def test_volume_fetch_needs_last_chunk(port):
    """C/S of a slot are fetchable while its volumes are resident (the last
    chunk); older chunks' volumes were recycled and the fetch says so."""
    cfg = SceneConfig.baseline_config(0, width=128, height=64, focal=100.0, cx=63.5, cy=31.5,
                                      d_max=32, seed=4)
    L, R, _, _ = render(cfg, 0, 1)
    calib = tsgm.StereoCalib(cfg.focal, cfg.cx, cfg.cy, cfg.baseline, 128, 64, 32)
    params, filt = tsgm.SgmParams(10, 120, 8, 0, 32), tsgm.FilterConfig()
    eng = tsgm.Engine(tsgm.EngineConfig(calib, params, filt, max_slots=3, vol_slots=1))
    eye = (np.eye(3), np.zeros(3))
    eng.step([0, 1, 2], [L[0]] * 3, [R[0]] * 3, [eye] * 3)
    ref = port.step(None, L[0], R[0], eye[0], eye[1], calib, params, filt, debug=True)
    _, cost = port.cost_volume(L[0], R[0], ref["lo"], ref["hi"])
    np.testing.assert_array_equal(eng.fetch(2, "cost"), cost)
    with pytest.raises(ValueError, match="not resident"):
        eng.fetch(0, "cost")
    eng.close()


@pytest.mark.parametrize("scan", ["groups32", "groups16", "groups8", "lines"])
def test_config1_movers_batched(port, monkeypatch, scan):
    """Config-1 scenes with movers, 3 sequences batched, reduced size, with
    each aggregation scan kernel."""
    monkeypatch.setenv("TSGM_SCAN_KERNEL", "lines" if scan == "lines" else "groups")
    if scan != "lines":
        monkeypatch.setenv("TSGM_SCAN_SPW", scan[len("groups"):])
    cfgs = [SceneConfig.baseline_config(1, width=320, height=120, focal=200.0, cx=159.5,
                                        cy=59.5, d_max=64, seed=s, n_movers=3) for s in range(3)]
    run_parity(port, cfgs, 10, tsgm.SgmParams(10, 120, 8, 0, 64),
               tsgm.FilterConfig(range_use_stddev=True, range_stddev_gain=3.0))


@pytest.mark.parametrize("paths,path_set", [(4, 0), (4, 1)])
def test_four_path_sets(port, paths, path_set):
    cfg = SceneConfig.baseline_config(0, width=200, height=80, focal=150.0, cx=99.5, cy=39.5,
                                      d_max=48, seed=5)
    run_parity(port, [cfg], 4, tsgm.SgmParams(6, 65, paths, path_set, 48), tsgm.FilterConfig(),
               check_volumes=True)


def test_reset_restarts_full_range(port):
    cfg = SceneConfig.baseline_config(0, width=160, height=64, focal=120.0, cx=79.5, cy=31.5,
                                      d_max=32, seed=9)
    L, R, poses, _ = render(cfg, 0, 2)
    calib = tsgm.StereoCalib(cfg.focal, cfg.cx, cfg.cy, cfg.baseline, cfg.width, cfg.height, 32)
    params, filt = tsgm.SgmParams(10, 120, 8, 0, 32), tsgm.FilterConfig()
    eng = tsgm.Engine(tsgm.EngineConfig(calib, params, filt, max_slots=1))
    eng.step([0], [L[0]], [R[0]], [(np.eye(3), np.zeros(3))])
    eng.step([0], [L[1]], [R[1]], [tsgm.relative_motion(poses[0], poses[1])])
    eng.reset(0)
    eng.step([0], [L[1]], [R[1]], [(np.eye(3), np.zeros(3))])
    ref = port.step(None, L[1], R[1], np.eye(3), np.zeros(3), calib, params, filt)
    np.testing.assert_array_equal(eng.fetch(0, "export_d"), ref["export_d"])
    np.testing.assert_array_equal(eng.fetch(0, "state_p"), ref["p"])
    assert (eng.fetch(0, "hi") == 31).all() and (eng.fetch(0, "lo") == 0).all()
    eng.close()


def test_overlapped_fetch_captures_each_frame(port):
    """fetch_batch copies run on the copy stream while the next frame computes;
    every frame's copies must hold that frame's outputs."""
    cfgs = [SceneConfig.baseline_config(1, width=256, height=96, focal=160.0, cx=127.5, cy=47.5,
                                        d_max=48, seed=s, n_movers=2) for s in (3, 4)]
    calib = tsgm.StereoCalib(160.0, 127.5, 47.5, cfgs[0].baseline, 256, 96, 48)
    params, filt = tsgm.SgmParams(10, 120, 8, 0, 48), tsgm.FilterConfig(range_use_stddev=True,
                                                                        range_stddev_gain=3.0)
    seqs = [render(c, 0, 5) for c in cfgs]
    eng = tsgm.Engine(tsgm.EngineConfig(calib, params, filt, max_slots=2, keep_volumes=False))
    got = []
    for k in range(5):
        mots = [(np.eye(3), np.zeros(3)) if k == 0 else tsgm.relative_motion(P[k - 1], P[k])
                for (_, _, P, _) in seqs]
        eng.step([0, 1], [s[0][k] for s in seqs], [s[1][k] for s in seqs], mots)
        ed = [np.empty((96, 256), np.int32) for _ in range(2)]
        pp = [np.empty((96, 256), np.float64) for _ in range(2)]
        mk = [np.empty((96, 256), np.uint8) for _ in range(2)]
        eng.fetch_batch([0, 1], "export_d", ed)
        eng.fetch_batch([0, 1], "state_p", pp)
        eng.fetch_batch([0, 1], "mask", mk)
        got.append((ed, pp, mk))
    eng.sync()
    for i, (L, R, P, _) in enumerate(seqs):
        state = None
        for k in range(5):
            m = (np.eye(3), np.zeros(3)) if k == 0 else tsgm.relative_motion(P[k - 1], P[k])
            ref = port.step(state, L[k], R[k], m[0], m[1], calib, params, filt, debug=True)
            np.testing.assert_array_equal(got[k][0][i], ref["export_d"])
            np.testing.assert_array_equal(got[k][1][i], ref["p"])
            np.testing.assert_array_equal(got[k][2][i], ref["mask"])
            state = (ref["d"], ref["p"], ref["valid"])
    eng.close()


def test_interleaved_batches(port):
    """Sequences stepping at different rates share one engine: slot 0 every
    call, slot 2 every other call, slot 1 never; the host-image uploads
    alternate staging buffers on their own stream. Each sequence matches the
    oracle run on its own frames."""
    cfgs = [SceneConfig.baseline_config(1, width=192, height=80, focal=120.0, cx=95.5, cy=39.5,
                                        d_max=40, seed=s, n_movers=1) for s in (6, 7)]
    calib = tsgm.StereoCalib(120.0, 95.5, 39.5, cfgs[0].baseline, 192, 80, 40)
    params, filt = tsgm.SgmParams(10, 120, 8, 0, 40), tsgm.FilterConfig(range_use_stddev=True,
                                                                        range_stddev_gain=3.0)
    seqs = [render(c, 0, 6) for c in cfgs]
    eng = tsgm.Engine(tsgm.EngineConfig(calib, params, filt, max_slots=3, keep_volumes=False))
    nxt = [0, 0]
    states = [None, None]

    def mot(i, k):
        P = seqs[i][2]
        return (np.eye(3), np.zeros(3)) if k == 0 else tsgm.relative_motion(P[k - 1], P[k])

    for call in range(6):
        active = [0] + ([1] if call % 2 == 1 else [])
        slots = [0 if i == 0 else 2 for i in active]
        eng.step(slots, [seqs[i][0][nxt[i]] for i in active],
                 [seqs[i][1][nxt[i]] for i in active], [mot(i, nxt[i]) for i in active])
        for i, sl in zip(active, slots):
            k = nxt[i]
            m = mot(i, k)
            ref = port.step(states[i], seqs[i][0][k], seqs[i][1][k], m[0], m[1], calib, params,
                            filt)
            np.testing.assert_array_equal(eng.fetch(sl, "export_d"), ref["export_d"])
            np.testing.assert_array_equal(eng.fetch(sl, "state_p"), ref["p"])
            states[i] = (ref["d"], ref["p"], ref["valid"])
            nxt[i] += 1
    assert not eng.fetch(1, "state_valid").any()
    eng.close()


@pytest.mark.parametrize("half", [2, 4, 8, 16])
def test_config3_fixed_window_sweep(port, half):
    """Config 3: reduced windows of exactly 2h+1 levels (stddev ranges with a
    vanishing gain and min_range_halfwidth = h)."""
    cfg = SceneConfig.baseline_config(3, width=320, height=120, focal=200.0, cx=159.5, cy=59.5,
                                      d_max=128, seed=21)
    run_parity(port, [cfg], 4, tsgm.SgmParams(10, 120, 8, 0, 128),
               tsgm.FilterConfig(range_use_stddev=True, range_stddev_gain=1e-9,
                                 min_range_halfwidth=half), check_volumes=True)


@pytest.mark.parametrize("scan", ["groups32", "groups8", "lines"])
def test_config3_full_range_d256(port, monkeypatch, scan):
    """Config 3's D=256 full-range baseline (p_init >= d_max^2/4)."""
    monkeypatch.setenv("TSGM_SCAN_KERNEL", "lines" if scan == "lines" else "groups")
    if scan != "lines":
        monkeypatch.setenv("TSGM_SCAN_SPW", scan[len("groups"):])
    cfg = SceneConfig.baseline_config(3, width=384, height=96, focal=240.0, cx=191.5, cy=47.5,
                                      d_max=256, seed=22)
    run_parity(port, [cfg], 2, tsgm.SgmParams(10, 120, 8, 0, 256),
               tsgm.FilterConfig(p_init=16384.0, range_use_stddev=True, range_stddev_gain=3.0),
               check_volumes=True)


def test_config4_gain_and_occluders(port):
    """Config 4 at reduced size: per-frame global gain +-10%, occluding movers
    up to 30% of the image, D=256, two sequences batched."""
    cfgs = [SceneConfig.baseline_config(4, width=512, height=256, focal=275.0, cx=255.5,
                                        cy=127.5, seed=s) for s in (1, 2)]
    run_parity(port, cfgs, 4, tsgm.SgmParams(10, 120, 8, 0, 256),
               tsgm.FilterConfig(p_init=16384.0, range_use_stddev=True, range_stddev_gain=3.0))


def test_subpixel_extension(port):
    """A22 extension (opt-in, export only): the f32 parabola refinement of the
    WTA level, bit-exact against the oracle's definition; the integer outputs
    and the Kalman state are unchanged by it."""
    cfg = SceneConfig.baseline_config(1, width=320, height=120, focal=200.0, cx=159.5, cy=59.5,
                                      d_max=64, seed=8, n_movers=2)
    L, R, P, _ = render(cfg, 0, 3)
    calib = tsgm.StereoCalib(cfg.focal, cfg.cx, cfg.cy, cfg.baseline, 320, 120, 64)
    params = tsgm.SgmParams(10, 120, 8, 0, 64)
    filt = tsgm.FilterConfig(range_use_stddev=True, range_stddev_gain=3.0)
    eng = tsgm.Engine(tsgm.EngineConfig(calib, params, filt, max_slots=1, subpixel=True))
    state = None
    for k in range(3):
        m = (np.eye(3), np.zeros(3)) if k == 0 else tsgm.relative_motion(P[k - 1], P[k])
        eng.step([0], [L[k]], [R[k]], [m])
        ref = port.step(state, L[k], R[k], m[0], m[1], calib, params, filt, debug=True)
        np.testing.assert_array_equal(eng.fetch(0, "meas_d"), ref["meas_d"])
        np.testing.assert_array_equal(eng.fetch(0, "state_p"), ref["p"])
        _, cost = port.cost_volume(L[k], R[k], ref["lo"], ref["hi"])
        agg = port.aggregate(cost, ref["lo"], ref["hi"], params)
        want = port.subpixel(agg, ref["lo"], ref["hi"], ref["meas_d"], ref["meas_valid"])
        got = eng.fetch(0, "subpixel")
        np.testing.assert_array_equal(got, want)
        v = ref["meas_valid"] > 0
        assert (np.abs(got[v] - ref["meas_d"][v]) <= 0.5).all()
        state = (ref["d"], ref["p"], ref["valid"])
    eng.close()


@pytest.mark.parametrize("n_seq", [4, 8, 16])
def test_config2_per_gpu_shares(port, n_seq):
    """Config 2 at full size with the per-GPU batch of 16, 8 and 4 sequences
    (the strong-scaling shares of 4 and 8 GPUs and a smaller one), 3 frames:
    every output bit-exact through the default small-batch kernel choices
    (mixed scan kernels: 32-lane or G-lane horizontal groups, 8-scanline
    horizontal warps)."""
    cfgs = [SceneConfig.baseline_config(2, seed=s, n_movers=s % 5, frames=3) for s in range(n_seq)]
    run_parity(port, cfgs, 3, tsgm.SgmParams(10, 120, 8, 0, 128),
               tsgm.FilterConfig(range_use_stddev=True, range_stddev_gain=3.0))
