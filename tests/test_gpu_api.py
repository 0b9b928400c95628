"""Engine API contract on the GPU: argument validation before the C-ABI reads
raw pointers (the reference's step() messages, temporal_filter.cpp:198-204),
volume residency across changing batches, StepResult::timings
(temporal_filter.hpp:57-69, sgm.hpp:59-69) and stream ordering of
tsgm_step_device."""
import numpy as np
import pytest

from paper_1809_07986_b200 import tsgm
from paper_1809_07986_b200.scene import SceneConfig, render

pytestmark = pytest.mark.gpu

W, H, D = 128, 64, 32


def _scene(seed=4, frames=2):
    cfg = SceneConfig.baseline_config(1, width=W, height=H, focal=100.0, cx=63.5, cy=31.5,
                                      d_max=D, seed=seed, n_movers=1, frames=frames)
    calib = tsgm.StereoCalib(cfg.focal, cfg.cx, cfg.cy, cfg.baseline, W, H, D)
    return cfg, calib


def _engine(calib, **kw):
    return tsgm.Engine(tsgm.EngineConfig(calib, tsgm.SgmParams(10, 120, 8, 0, D),
                                         tsgm.FilterConfig(range_use_stddev=True,
                                                           range_stddev_gain=3.0), **kw))


EYE = (np.eye(3), np.zeros(3))


def test_step_rejects_wrong_shapes():
    cfg, calib = _scene()
    L, R, _, _ = render(cfg, 0, 1)
    eng = _engine(calib, max_slots=2)
    with pytest.raises(ValueError, match="left/right dimension mismatch"):
        eng.step([0], [L[0]], [R[0][:, :-1]], [EYE])
    with pytest.raises(ValueError, match="state dimension mismatch"):
        eng.step([0], [L[0][:-1]], [R[0][:-1]], [EYE])
    with pytest.raises(ValueError, match="differ in length"):
        eng.step([0, 1], [L[0]], [R[0]], [EYE])
    with pytest.raises(ValueError, match="state dimension mismatch"):
        eng.set_state(0, np.zeros((H, W - 1)), np.zeros((H, W)), np.zeros((H, W), np.uint8))
    eng.step([0, 1], [L[0], L[0]], [R[0], R[0]], [EYE, EYE])
    small = [np.zeros((H, W), np.int32), np.zeros((H, W - 1), np.int32)]
    with pytest.raises(ValueError, match="too small"):
        eng.fetch_batch([0, 1], "export_d", small)
    with pytest.raises(ValueError, match="one output array per slot"):
        eng.fetch_batch([0, 1], "export_d", small[:1])
    eng.close()


def test_volume_owner_changes_with_the_batch(port):
    """positions past the last chunk must not keep owners from an
    earlier frame. step([0..3]) then step([3..7]) with 4 volume positions: the
    second frame's last chunk is {5, 6, 7}; slot 3's old volume at position 3
    must read as not resident, and slots 5-7 must return this frame's C."""
    cfg, calib = _scene(frames=1)
    L, R, _, _ = render(cfg, 0, 1)
    params = tsgm.SgmParams(10, 120, 8, 0, D)
    filt = tsgm.FilterConfig(range_use_stddev=True, range_stddev_gain=3.0)
    eng = tsgm.Engine(tsgm.EngineConfig(calib, params, filt, max_slots=8, vol_slots=4))
    eng.step([0, 1, 2, 3], [L[0]] * 4, [R[0]] * 4, [EYE] * 4)
    eng.step([3, 4, 5, 6, 7], [L[0]] * 5, [R[0]] * 5, [EYE] * 5)
    with pytest.raises(ValueError, match="not resident"):
        eng.fetch(3, "cost")
    ref = port.step(None, L[0], R[0], EYE[0], EYE[1], calib, params, filt, debug=True)
    _, cost = port.cost_volume(L[0], R[0], ref["lo"], ref["hi"])
    for s in (5, 6, 7):
        np.testing.assert_array_equal(eng.fetch(s, "cost"), cost)
    eng.close()


def test_step_timings_filled():
    cfg, calib = _scene()
    L, R, poses, _ = render(cfg, 0, 2)
    params = tsgm.SgmParams(10, 120, 8, 0, D)
    filt = tsgm.FilterConfig(range_use_stddev=True, range_stddev_gain=3.0)
    r0 = tsgm.step(None, L[0], R[0], EYE[0], EYE[1], calib, params, filt)
    Rm, t = tsgm.relative_motion(poses[0], poses[1])
    r1 = tsgm.step((r0["d"], r0["p"], r0["valid"]), L[1], R[1], Rm, t, calib, params, filt)
    for r in (r0, r1):
        tm = r["timings"]
        assert tm["predict_s"] > 0 and tm["ranges_s"] > 0 and tm["correct_s"] > 0
        assert all(v > 0 for v in tm["sgm"].values()), tm
        assert sum(tm["sgm"].values()) < 1.0
    st = {}
    lo = np.zeros((H, W), np.uint16)
    hi = np.full((H, W), D - 1, np.uint16)
    tsgm.sgm_match(L[0], R[0], lo, hi, params, timings=st)
    assert set(st) == {"census_s", "cost_s", "aggregate_s", "wta_s"}
    assert all(v > 0 for v in st.values())
    eng = _engine(calib, max_slots=2, stage_timings=True)
    eng.step([0, 1], [L[0]] * 2, [R[0]] * 2, [EYE] * 2)
    tm = eng.timings()
    assert tm["predict_s"] > 0 and tm["sgm"]["aggregate_s"] > 0 and tm["sgm"]["wta_s"] > 0
    eng.close()
    eng = _engine(calib, max_slots=1)
    eng.step([0], [L[0]], [R[0]], [EYE])
    with pytest.raises(ValueError, match="TSGM_STAGE_TIMINGS"):
        eng.timings()
    eng.close()


def test_step_device_after_producer_stream(port):
    """Images produced on a torch stream: the step waits for them
    (tsgm_step_device_after) and the caller's stream waits for the census
    before refilling them (tsgm_inputs_consumed)."""
    torch = pytest.importorskip("torch")
    cfg, calib = _scene(frames=2)
    L, R, poses, _ = render(cfg, 0, 2)
    params = tsgm.SgmParams(10, 120, 8, 0, D)
    filt = tsgm.FilterConfig(range_use_stddev=True, range_stddev_gain=3.0)
    eng = _engine(calib, max_slots=1)
    s = torch.cuda.Stream()
    dl = torch.empty((H, W), dtype=torch.uint8, device="cuda")
    dr = torch.empty((H, W), dtype=torch.uint8, device="cuda")
    hl = [torch.from_numpy(x).pin_memory() for x in L]
    hr = [torch.from_numpy(x).pin_memory() for x in R]
    state = None
    for k in range(2):
        Rm, t = EYE if k == 0 else tsgm.relative_motion(poses[k - 1], poses[k])
        with torch.cuda.stream(s):
            if k:
                eng.inputs_consumed(s.cuda_stream)
            dl.copy_(hl[k], non_blocking=True)
            dr.copy_(hr[k], non_blocking=True)
        m = np.concatenate([np.asarray(Rm).ravel(), np.asarray(t).ravel()])[None]
        eng.step_device([0], [dl.data_ptr()], [dr.data_ptr()], m, after_stream=s.cuda_stream)
        ref = port.step(state, L[k], R[k], Rm, t, calib, params, filt)
        np.testing.assert_array_equal(eng.fetch(0, "export_d"), ref["export_d"])
        np.testing.assert_array_equal(eng.fetch(0, "state_p"), ref["p"])
        state = (ref["d"], ref["p"], ref["valid"])
    eng.close()


def test_pipelined_engine_matches_one_context():
    """PipelinedEngine (the batch over several contexts, each with its own
    streams) returns exactly what one context returns: sequences are
    independent (eval.cpp:114-144). 5 sequences over 2 and 3 contexts (uneven
    groups), interleaved slot order, host and batched fetches."""
    frames, S = 3, 5
    scenes = []
    for s in range(S):
        cfg, calib = _scene(seed=10 + s, frames=frames)
        L, R, P, _ = render(cfg)
        scenes.append((L, R, P))
    base = _engine(calib, max_slots=S)
    order = [3, 0, 4, 1, 2]
    for groups in (2, 3):
        pe = tsgm.PipelinedEngine(base.cfg, groups)
        assert len(pe.engines) == groups
        for s in range(S):
            base.reset(s)
            pe.reset(s)
        for k in range(frames):
            mots = [EYE if k == 0 else tsgm.relative_motion(scenes[s][2][k - 1], scenes[s][2][k])
                    for s in order]
            ls, rs = [scenes[s][0][k] for s in order], [scenes[s][1][k] for s in order]
            base.step(order, ls, rs, mots)
            pe.step(order, ls, rs, mots)
            outs = [np.zeros((H, W), np.int32) for _ in order]
            pe.fetch_batch(order, "export_d", outs)
            pe.sync()
            for s, o in zip(order, outs):
                assert np.array_equal(o, base.fetch(s, "export_d"))
                for what in ("state_d", "state_p", "state_valid", "diff", "mask"):
                    assert np.array_equal(pe.fetch(s, what), base.fetch(s, what)), (groups, k, s, what)
                assert pe.cells(s) == base.cells(s)
        assert pe.launches > 0
        pe.close()
    base.close()


@pytest.mark.parametrize("d_max", [32, 64, 128])
def test_full_range_line_groups_match_the_masked_path(monkeypatch, port, d_max):
    """Frame 0 of fresh sequences (every window [0, d_max - 1]) runs rfull_task
    (register line groups, the window compiled in); TSGM_RFULL=0 keeps
    lines_task + scan_pixel_full. Same S, same WTA, both equal to the oracle's
    aggregate_paths (sgm.cpp:39-161)."""
    w, h = 96, 40
    cfg = SceneConfig.baseline_config(1, width=w, height=h, focal=100.0, cx=47.5, cy=19.5,
                                      d_max=d_max, seed=3, n_movers=1, frames=1)
    calib = tsgm.StereoCalib(cfg.focal, cfg.cx, cfg.cy, cfg.baseline, w, h, d_max)
    L, R, _, _ = render(cfg, 0, 1)
    params = tsgm.SgmParams(10, 120, 8, 0, d_max)
    out = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("TSGM_RFULL", mode)
        eng = tsgm.Engine(tsgm.EngineConfig(calib, params, tsgm.FilterConfig(), max_slots=3))
        eng.step([0, 1, 2], [L[0]] * 3, [R[0]] * 3, [EYE] * 3)
        out[mode] = (eng.last_kernels(), eng.fetch(1, "agg"), eng.fetch(1, "meas_d"), eng.fetch(1, "cost"))
        eng.close()
    assert "[rfull]" in out["1"][0] and "[rfull]" not in out["0"][0], (out["1"][0], out["0"][0])
    assert np.array_equal(out["1"][1], out["0"][1]) and np.array_equal(out["1"][2], out["0"][2])
    lo = np.zeros((h, w), np.uint16)
    hi = np.full((h, w), d_max - 1, np.uint16)
    np.testing.assert_array_equal(out["1"][1], port.aggregate(out["1"][3], lo, hi, params))
