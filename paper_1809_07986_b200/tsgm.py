"""Python mirror of the reference's hot-path API, running on the B200.

Same names, argument meaning and error behaviour as the reference C++ library
(/root/reference/proj/include/tsgm/*.hpp): invalid arguments raise
``ValueError`` (std::invalid_argument), CUDA/runtime failures raise
``RuntimeError`` (std::runtime_error). Every call goes through the C-ABI of
``lib/libtsgm_b200.so`` (include/tsgm_b200.h); nothing here computes on the CPU
beyond argument marshalling.

Two levels:

* stage functions (``census_transform`` ... ``step``) — the reference's public
  sub-stage API, stateless, host numpy arrays in and out;
* :class:`Engine` — the production path: device-resident Kalman state for many
  independent sequences ("slots"), one batched launch sequence per frame.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import ConfigC, FilterConfigC, OUT, SgmParamsC, StereoCalibC, check, ptr

NONDIAGONAL, DIAGONAL = 0, 1  # PathSet, sgm.hpp:10-13


@dataclass
class SgmParams:  # sgm.hpp:15-23
    p1: int = 6
    p2: int = 65
    paths: int = 8
    path_set: int = NONDIAGONAL
    d_max: int = 128

    def _c(self):
        return SgmParamsC(self.p1, self.p2, self.paths, int(self.path_set), self.d_max)


@dataclass
class FilterConfig:  # temporal_filter.hpp:8-26 (NoiseParams q, r flattened)
    q: float = 0.5
    r: float = 1.0
    p_init: float = 4096.0
    disc_thresh: float = 2.0
    min_range_halfwidth: int = 2
    range_use_stddev: bool = False
    range_stddev_gain: float = 2.0

    def _c(self):
        return FilterConfigC(self.q, self.r, self.p_init, self.disc_thresh,
                             self.min_range_halfwidth, 1 if self.range_use_stddev else 0,
                             self.range_stddev_gain)


@dataclass
class StereoCalib:  # geometry.hpp:17-27
    focal_px: float = 0.0
    cx: float = 0.0
    cy: float = 0.0
    baseline_m: float = 0.0
    width: int = 0
    height: int = 0
    d_max: int = 0

    def _c(self):
        return StereoCalibC(self.focal_px, self.cx, self.cy, self.baseline_m, self.width,
                            self.height, self.d_max)


def _as(x, cls):
    """Accept any object with the dataclass's attribute names."""
    if isinstance(x, cls):
        return x
    return cls(**{k: getattr(x, k) for k in cls.__dataclass_fields__})


def _u8(a):
    return np.ascontiguousarray(a, dtype=np.uint8)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _u16(a):
    return np.ascontiguousarray(a, dtype=np.uint16)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _hw(a):
    h, w = a.shape
    return w, h


# --------------------------------------------------------------------- stages
def census_transform(img):
    """census_transform (matching_cost.cpp:53-79) -> u32 signatures."""
    img = _u8(img)
    w, h = _hw(img)
    sig = np.zeros((h, w), np.uint32)
    check(_lib.load().tsgm_census_transform(ptr(img), w, h, ptr(sig)))
    return sig


def build_cost_volume(left, right, lo, hi):
    """build_cost_volume (matching_cost.cpp:88-117) -> (offsets u32[W*H+1], cost u8[N])."""
    left, right, lo, hi = _u8(left), _u8(right), _u16(lo), _u16(hi)
    w, h = _hw(left)
    if right.shape != left.shape or lo.shape != left.shape or hi.shape != left.shape:
        raise ValueError("build_cost_volume: input size mismatch")
    n = int((hi.astype(np.int64) - lo.astype(np.int64) + 1).sum())
    off = np.zeros(w * h + 1, np.uint32)
    cost = np.zeros(max(n, 1), np.uint8)
    check(_lib.load().tsgm_build_cost_volume(ptr(left), ptr(right), w, h, ptr(lo), ptr(hi),
                                            ptr(off), ptr(cost), C.c_uint64(cost.size)))
    return off, cost[:n]


def aggregate_paths(cost, lo, hi, params):
    """aggregate_paths (sgm.cpp:135-161) over a ragged C volume -> u16 S."""
    cost, lo, hi = _u8(cost), _u16(lo), _u16(hi)
    w, h = _hw(lo)
    p = _as(params, SgmParams)._c()
    agg = np.zeros(max(cost.size, 1), np.uint16)
    check(_lib.load().tsgm_aggregate_paths(ptr(cost), ptr(lo), ptr(hi), w, h, C.byref(p),
                                          ptr(agg)))
    return agg[: cost.size]


def winner_takes_all(agg, lo, hi):
    """winner_takes_all (sgm.cpp:163-187) -> (d i32, valid u8)."""
    agg, lo, hi = _u16(agg), _u16(lo), _u16(hi)
    w, h = _hw(lo)
    d = np.zeros((h, w), np.int32)
    v = np.zeros((h, w), np.uint8)
    check(_lib.load().tsgm_winner_takes_all(ptr(agg), ptr(lo), ptr(hi), w, h, ptr(d), ptr(v)))
    return d, v


def median_refine(d, valid):
    """median_refine (sgm.cpp:189-216)."""
    d, valid = _i32(d), _u8(valid)
    w, h = _hw(d)
    od = np.zeros((h, w), np.int32)
    ov = np.zeros((h, w), np.uint8)
    check(_lib.load().tsgm_median_refine(ptr(d), ptr(valid), w, h, ptr(od), ptr(ov)))
    return od, ov


def sgm_match(left, right, lo, hi, params, timings=None):
    """sgm_match (sgm.cpp:226-257): census -> cost -> aggregate -> WTA. A dict
    passed as ``timings`` receives the SgmStageTimings (device seconds)."""
    left, right, lo, hi = _u8(left), _u8(right), _u16(lo), _u16(hi)
    if left.shape != right.shape:
        raise ValueError("sgm_match: image size mismatch")
    if lo.shape != left.shape:
        raise ValueError("sgm_match: range map size mismatch")
    w, h = _hw(left)
    if hi.shape != left.shape:
        raise ValueError("sgm_match: range map size mismatch")
    p = _as(params, SgmParams)._c()
    d = np.zeros((h, w), np.int32)
    v = np.zeros((h, w), np.uint8)
    t = _lib.StageTimingsC()
    check(_lib.load().tsgm_sgm_match_t(ptr(left), ptr(right), w, h, ptr(lo), ptr(hi),
                                      C.byref(p), ptr(d), ptr(v), C.byref(t)))
    if timings is not None:  # SgmStageTimings* (sgm.hpp:59-69)
        for k in ("census_s", "cost_s", "aggregate_s", "wta_s"):
            timings[k] = getattr(t, k)
    return d, v


def relative_motion(prev_pose, cur_pose):
    """relative_motion (geometry.cpp:189-197): 3x4 camera-to-world poses -> (R, t)."""
    a, b = _f64(prev_pose).ravel(), _f64(cur_pose).ravel()
    r = np.zeros(9)
    t = np.zeros(3)
    check(_lib.load().tsgm_relative_motion(ptr(a), ptr(b), ptr(r), ptr(t)))
    return r.reshape(3, 3), t


def disparity_homography(R, t, calib):
    """disparity_homography (geometry.cpp:77-110) -> 4x4."""
    R, t = _f64(R).ravel(), _f64(t).ravel()
    c = _as(calib, StereoCalib)._c()
    H = np.zeros(16)
    check(_lib.load().tsgm_disparity_homography(ptr(R), ptr(t), C.byref(c), ptr(H)))
    return H.reshape(4, 4)


def warp_state_ex(d, p, valid, H, d_max):
    """warp_state_ex (geometry.cpp:127-156) -> (d, p, valid, source_d)."""
    d, p, valid, H = _f64(d), _f64(p), _u8(valid), _f64(H).ravel()
    w, h = _hw(d)
    od, op, osrc = np.zeros((h, w)), np.zeros((h, w)), np.zeros((h, w))
    ov = np.zeros((h, w), np.uint8)
    check(_lib.load().tsgm_warp_state_ex(ptr(d), ptr(p), ptr(valid), w, h, ptr(H), int(d_max),
                                        ptr(od), ptr(op), ptr(ov), ptr(osrc)))
    return od, op, ov, osrc


def predict(d, p, valid, R, t, calib, cfg):
    """predict (temporal_filter.cpp:28-49)."""
    d, p, valid = _f64(d), _f64(p), _u8(valid)
    R, t = _f64(R).ravel(), _f64(t).ravel()
    w, h = _hw(d)
    c, f = _as(calib, StereoCalib)._c(), _as(cfg, FilterConfig)._c()
    od, op = np.zeros((h, w)), np.zeros((h, w))
    ov = np.zeros((h, w), np.uint8)
    check(_lib.load().tsgm_predict(ptr(d), ptr(p), ptr(valid), w, h, ptr(R), ptr(t), C.byref(c),
                                  C.byref(f), ptr(od), ptr(op), ptr(ov)))
    return od, op, ov


def reject_discontinuities(d, p, valid, cfg):
    """reject_discontinuities (temporal_filter.cpp:51-74)."""
    d, p, valid = _f64(d), _f64(p), _u8(valid)
    w, h = _hw(d)
    f = _as(cfg, FilterConfig)._c()
    od, op = np.zeros((h, w)), np.zeros((h, w))
    ov = np.zeros((h, w), np.uint8)
    check(_lib.load().tsgm_reject_discontinuities(ptr(d), ptr(p), ptr(valid), w, h, C.byref(f),
                                                 ptr(od), ptr(op), ptr(ov)))
    return od, op, ov


def fill_zoom_holes(d, p, valid):
    """fill_zoom_holes (temporal_filter.cpp:76-106)."""
    d, p, valid = _f64(d), _f64(p), _u8(valid)
    w, h = _hw(d)
    od, op = np.zeros((h, w)), np.zeros((h, w))
    ov = np.zeros((h, w), np.uint8)
    check(_lib.load().tsgm_fill_zoom_holes(ptr(d), ptr(p), ptr(valid), w, h, ptr(od), ptr(op),
                                          ptr(ov)))
    return od, op, ov


def derive_search_ranges(d, p, valid, calib, cfg):
    """derive_search_ranges (temporal_filter.cpp:108-143) -> (lo, hi) u16."""
    d, p, valid = _f64(d), _f64(p), _u8(valid)
    w, h = _hw(d)
    c, f = _as(calib, StereoCalib)._c(), _as(cfg, FilterConfig)._c()
    lo = np.zeros((h, w), np.uint16)
    hi = np.zeros((h, w), np.uint16)
    check(_lib.load().tsgm_derive_search_ranges(ptr(d), ptr(p), ptr(valid), w, h, C.byref(c),
                                               C.byref(f), ptr(lo), ptr(hi)))
    return lo, hi


def correct(d, p, valid, meas_d, meas_valid, cfg):
    """correct (temporal_filter.cpp:145-170)."""
    d, p, valid = _f64(d), _f64(p), _u8(valid)
    md, mv = _i32(meas_d), _u8(meas_valid)
    if md.shape != d.shape:
        raise ValueError("correct: dimension mismatch")
    w, h = _hw(d)
    f = _as(cfg, FilterConfig)._c()
    od, op = np.zeros((h, w)), np.zeros((h, w))
    ov = np.zeros((h, w), np.uint8)
    check(_lib.load().tsgm_correct(ptr(d), ptr(p), ptr(valid), ptr(md), ptr(mv), w, h, C.byref(f),
                                  ptr(od), ptr(op), ptr(ov)))
    return od, op, ov


def step(state, left, right, R, t, calib, params, cfg):
    """step (temporal_filter.cpp:195-232) for one sequence, value semantics.

    ``state`` is ``(d, p, valid)`` or ``None`` for the default (empty) state.
    Returns a dict with the StepResult fields: d, p, valid (posterior),
    export_d, export_valid (median-refined map), diff and timings (StepTimings
    as a dict of device seconds, temporal_filter.hpp:57-62)."""
    left, right = _u8(left), _u8(right)
    if left.shape != right.shape:
        raise ValueError("step: left/right dimension mismatch")
    w, h = _hw(left)
    R, t = _f64(R).ravel(), _f64(t).ravel()
    c = _as(calib, StereoCalib)._c()
    sp = _as(params, SgmParams)._c()
    f = _as(cfg, FilterConfig)._c()
    if state is None:
        sd = spp = sv = None
        sw = sh = 0
    else:
        sd, spp, sv = _f64(state[0]), _f64(state[1]), _u8(state[2])
        if sd.shape != sv.shape or spp.shape != sv.shape:
            raise ValueError("step: state dimension mismatch")
        sh, sw = sv.shape
    out = dict(d=np.zeros((h, w)), p=np.zeros((h, w)), valid=np.zeros((h, w), np.uint8),
               export_d=np.zeros((h, w), np.int32), export_valid=np.zeros((h, w), np.uint8),
               diff=np.zeros((h, w)))
    tm = _lib.StageTimingsC()
    check(_lib.load().tsgm_step_once_t(
        ptr(sd), ptr(spp), ptr(sv), sw, sh, ptr(left), ptr(right), w, h, ptr(R), ptr(t),
        C.byref(c), C.byref(sp), C.byref(f), ptr(out["d"]), ptr(out["p"]), ptr(out["valid"]),
        ptr(out["export_d"]), ptr(out["export_valid"]), ptr(out["diff"]), C.byref(tm)))
    out["timings"] = _timings_dict(tm)
    return out


def _timings_dict(t):
    """StepTimings (temporal_filter.hpp:57-62) with its SgmStageTimings nested
    under "sgm", as the reference's struct."""
    return dict(predict_s=t.predict_s, ranges_s=t.ranges_s,
                sgm=dict(census_s=t.census_s, cost_s=t.cost_s, aggregate_s=t.aggregate_s,
                         wta_s=t.wta_s),
                correct_s=t.correct_s)


# --------------------------------------------------------------------- detector
@dataclass
class DetectConfig:  # motion_detect.hpp:36-44
    window_sizes: tuple = ((20, 20), (30, 30), (40, 40), (50, 50), (50, 75))
    score_thresh: float = 2.0
    merge_stop_iou: float = 0.2
    min_box_area: int = 400

    def _c(self):
        wh = np.ascontiguousarray(np.asarray(self.window_sizes, np.int32).reshape(-1))
        return wh, _lib.DetectConfigC(wh.ctypes.data, len(self.window_sizes), self.score_thresh,
                                      self.merge_stop_iou, int(self.min_box_area))


def _box_array(n):
    return np.zeros(max(1, n), dtype=[("x0", np.int32), ("y0", np.int32), ("x1", np.int32),
                                      ("y1", np.int32), ("score", np.float64)])


def _boxes_out(arr, n):
    """Boxes as float64 [n, 5] = x0, y0, x1, y1, score (DetectionBox fields)."""
    a = arr[:n]
    return np.stack([a["x0"], a["y0"], a["x1"], a["y1"], a["score"]], axis=1).astype(np.float64) \
        if n else np.zeros((0, 5))


def integral_image(m):
    """integral_image (motion_detect.cpp:25-42): (h+1) x (w+1) f64, on the GPU."""
    m = _f64(m)
    h, w = m.shape
    sat = np.zeros((h + 1, w + 1))
    check(_lib.load().tsgm_integral_image(ptr(m), w, h, ptr(sat)))
    return sat


def _detect_call(fn, diff, cfg):
    diff = _f64(diff)
    h, w = diff.shape
    wh, c = _as(cfg, DetectConfig)._c()
    n = C.c_int64()
    cap = 4096
    while True:
        out = _box_array(cap)
        check(fn(ptr(diff), w, h, C.byref(c), ptr(out), cap, C.byref(n)))
        if n.value <= cap:
            return _boxes_out(out, n.value)
        cap = n.value


def detect_candidate_windows(diff, cfg=None):
    """detect_candidate_windows (motion_detect.cpp:64-99), SAT and scoring on
    the GPU; boxes in (size, row, column) order."""
    return _detect_call(_lib.load().tsgm_detect_candidate_windows, diff, cfg or DetectConfig())


def greedy_merge(boxes, cfg=None):
    """greedy_merge (motion_detect.cpp:101-129), host, exact."""
    b = np.asarray(boxes, np.float64).reshape(-1, 5)
    arr = _box_array(len(b))
    for k, f in enumerate(("x0", "y0", "x1", "y1")):
        arr[f][:len(b)] = b[:, k].astype(np.int32)
    arr["score"][:len(b)] = b[:, 4]
    wh, c = _as(cfg or DetectConfig(), DetectConfig)._c()
    n = C.c_int64()
    check(_lib.load().tsgm_greedy_merge(ptr(arr), len(b), C.byref(c), C.byref(n)))
    return _boxes_out(arr, n.value)


def detect_moving_objects(diff, cfg=None):
    """detect_moving_objects (motion_detect.cpp:142-145)."""
    return _detect_call(_lib.load().tsgm_detect_moving_objects, diff, cfg or DetectConfig())


# --------------------------------------------------------------------- outliers
@dataclass
class OutlierOptions:  # eval.hpp:13-19
    abs_thresh_px: float = 3.0
    rel_thresh: float = 0.05
    strict_density: bool = False

    def _c(self):
        return _lib.OutlierOptionsC(self.abs_thresh_px, self.rel_thresh,
                                    1 if self.strict_density else 0)


def count_outliers(d, valid, gt, opts=None):
    """count_outliers (eval.cpp:59-85) on the GPU -> (evaluated, outliers)."""
    d, valid, gt = _i32(d), _u8(valid), _f64(gt)
    if d.shape != gt.shape or valid.shape != gt.shape:
        raise ValueError("count_outliers: est/gt dimension mismatch")
    w, h = _hw(gt)
    o = _as(opts or OutlierOptions(), OutlierOptions)._c()
    ev, out = C.c_int64(), C.c_int64()
    check(_lib.load().tsgm_count_outliers(ptr(d), ptr(valid), ptr(gt), w, h, C.byref(o),
                                         C.byref(ev), C.byref(out)))
    return int(ev.value), int(out.value)


def outlier_rate(d, valid, gt, opts=None):
    """outlier_rate (eval.cpp:87-93): percentage; no evaluated pixel is a
    runtime error."""
    ev, out = count_outliers(d, valid, gt, opts)
    if ev == 0:
        raise RuntimeError("outlier_rate: no mutually valid pixels")
    return 100.0 * out / ev


# ----------------------------------------------------------- export formats
# dataset.hpp:51-59 (write_disparity_png, write_boxes).
def _quant_args(disp_or_map):
    if isinstance(disp_or_map, tuple):  # DisparityMap: (d, valid)
        d, v = _i32(disp_or_map[0]), _u8(disp_or_map[1])
        if d.shape != v.shape:
            raise ValueError("write_disparity_png: map size mismatch")
        return None, d, v
    return _f64(disp_or_map), None, None


def quantize_disparity(disp_or_map):
    """write_disparity_png's 16-bit image (round(256 d), 0 = invalid) on the
    GPU, without the file: a f64 map, or a DisparityMap as (d, valid)."""
    disp, d, v = _quant_args(disp_or_map)
    h, w = (disp if disp is not None else d).shape
    raw = np.zeros((h, w), np.uint16)
    lib = _lib.load()
    if disp is not None:
        check(lib.tsgm_quantize_disparity(ptr(disp), w, h, ptr(raw)))
    else:
        check(lib.tsgm_quantize_disparity_map(ptr(d), ptr(v), w, h, ptr(raw)))
    return raw


def write_disparity_png(path, disp_or_map):
    """write_disparity_png (dataset.cpp:229-254): KITTI 16-bit PNG."""
    disp, d, v = _quant_args(disp_or_map)
    h, w = (disp if disp is not None else d).shape
    lib = _lib.load()
    if disp is not None:
        check(lib.tsgm_write_disparity_png(str(path).encode(), ptr(disp), w, h))
    else:
        check(lib.tsgm_write_disparity_png_map(str(path).encode(), ptr(d), ptr(v), w, h))


def read_png16(path):
    """A 16-bit grayscale PNG's samples (u16 [H, W]), any filter type; what
    read_disparity_png (dataset.cpp:220-227) reads before dividing by 256."""
    import struct
    import zlib
    with open(path, "rb") as f:
        data = f.read()
    if data[:8] != b"\x89PNG\r\n\x1a\n":
        raise RuntimeError(f"{path}: not a PNG")
    i, idat, ihdr = 8, [], None
    while i < len(data):
        (n,) = struct.unpack(">I", data[i:i + 4])
        typ, body = data[i + 4:i + 8], data[i + 8:i + 8 + n]
        (crc,) = struct.unpack(">I", data[i + 8 + n:i + 12 + n])
        if zlib.crc32(typ + body) & 0xffffffff != crc:
            raise RuntimeError(f"{path}: PNG decode error")
        if typ == b"IHDR":
            ihdr = struct.unpack(">IIBBBBB", body)
        elif typ == b"IDAT":
            idat.append(body)
        i += 12 + n
    w, h, depth, color, _, _, interlace = ihdr
    if depth != 16 or color != 0 or interlace != 0:
        raise RuntimeError(f"{path}: expected 16-bit single-channel PNG")
    raw = np.frombuffer(zlib.decompress(b"".join(idat)), np.uint8).reshape(h, 1 + 2 * w)
    out = np.zeros((h, 2 * w), np.int32)
    prev = np.zeros(2 * w, np.int32)
    bpp = 2
    for y in range(h):  # PNG filters 0-4 on the byte rows
        ft, line = raw[y, 0], raw[y, 1:].astype(np.int32)
        cur = np.zeros(2 * w, np.int32)
        for x in range(2 * w):
            a = cur[x - bpp] if x >= bpp else 0
            b = prev[x]
            c = prev[x - bpp] if x >= bpp else 0
            if ft == 0:
                pr = 0
            elif ft == 1:
                pr = a
            elif ft == 2:
                pr = b
            elif ft == 3:
                pr = (a + b) // 2
            else:
                p_ = a + b - c
                pa, pb, pc = abs(p_ - a), abs(p_ - b), abs(p_ - c)
                pr = a if pa <= pb and pa <= pc else (b if pb <= pc else c)
            cur[x] = (line[x] + pr) & 0xff
            if ft == 0:
                cur[:] = line
                break
        out[y] = cur
        prev = cur
    return ((out[:, 0::2] << 8) | out[:, 1::2]).astype(np.uint16)


def read_disparity_png(path):
    """read_disparity_png (dataset.cpp:220-227): samples / 256 (0 = invalid),
    decoded by the library (zlib, any PNG row filter)."""
    lib = _lib.load()
    w, h = C.c_int32(), C.c_int32()
    check(lib.tsgm_read_disparity_png(str(path).encode(), C.byref(w), C.byref(h), None, 0))
    out = np.zeros((h.value, w.value))
    check(lib.tsgm_read_disparity_png(str(path).encode(), C.byref(w), C.byref(h), ptr(out),
                                     out.size))
    return out


def write_boxes(path, per_frame):
    """write_boxes (dataset.cpp:256-269): '# frame x0 y0 x1 y1 score' lines,
    score at 17 significant digits; per_frame = one [n, 5] box array per frame."""
    counts = np.array([len(b) for b in per_frame], np.int64)
    total = int(counts.sum())
    arr = _box_array(total)
    k = 0
    for b in per_frame:
        for r in np.asarray(b, np.float64).reshape(-1, 5):
            arr[k] = (int(r[0]), int(r[1]), int(r[2]), int(r[3]), r[4])
            k += 1
    check(_lib.load().tsgm_write_boxes(str(path).encode(), arr.ctypes.data, ptr(counts),
                                      len(per_frame)))


# ----------------------------------------------------- noise calibration
# noise_calib.hpp:13-90 / noise_calib.cpp on the GPU.
@dataclass
class CalibOptions:  # noise_calib.hpp:43-49
    outlier_gate_px: float = 10.0
    bin_width: float = 0.25
    q_floor: float = 0.1

    def _c(self):
        return _lib.CalibOptionsC(self.outlier_gate_px, self.bin_width, self.q_floor)

    def validate(self):
        """CalibOptions::validate (noise_calib.cpp:60-67)."""
        n = C.c_int32()
        check(_lib.load().tsgm_calib_bins(C.byref(self._c()), C.byref(n)))
        return int(n.value)


@dataclass
class SequenceFrame:  # dataset.hpp:18-25 (the fields the calibration reads)
    index: int = 0
    left: np.ndarray | None = None
    right: np.ndarray | None = None
    pose: np.ndarray | None = None      # 3x4 camera-to-world (Pose, geometry.hpp:106)
    gt_disp: np.ndarray | None = None   # f64, > 0 = valid


@dataclass
class ErrorHistogram:  # noise_calib.hpp:14-41 (the estimate's histogram)
    lo: float = -10.0
    hi: float = 10.0
    bin_width: float = 0.25
    counts: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))
    underflow: int = 0
    overflow: int = 0
    n_gated: int = 0
    n_within_1: int = 0
    sum: float = 0.0
    sum_sq: float = 0.0

    def total(self) -> int:
        return self.n_gated + self.underflow + self.overflow

    def gated_count(self) -> int:
        return self.n_gated

    def mean(self) -> float:
        return self.sum / self.n_gated if self.n_gated > 0 else 0.0

    def variance(self) -> float:
        if self.n_gated < 2:
            return 0.0
        n = float(self.n_gated)
        m = self.sum / n
        v = (self.sum_sq - n * m * m) / (n - 1.0)
        return v if v > 0.0 else 0.0

    def fraction_within_1px(self) -> float:
        t = self.total()
        return self.n_within_1 / t if t > 0 else 0.0


@dataclass
class NoiseEstimate:  # noise_calib.hpp:51-55
    variance: float = 0.0
    hist: ErrorHistogram = field(default_factory=ErrorHistogram)
    samples_used: int = 0


def _require(frames, who, gt=False, pose=False, images=False):
    for f in frames:
        if gt and f.gt_disp is None:
            raise ValueError(f"{who}: frame {f.index} has no GT disparity")
        if pose and f.pose is None:
            raise ValueError(f"{who}: frame {f.index} has no pose")


def _stack(arrs, dtype, who):
    shape = arrs[0].shape
    for a in arrs:
        if a.shape != shape:
            raise ValueError(f"{who}: frame size mismatch")
    return np.ascontiguousarray(np.stack(arrs), dtype=dtype)


def _estimate(fn, args, opts):
    o = _as(opts or CalibOptions(), CalibOptions)
    nb = o.validate()
    counts = np.zeros(nb, np.int64)
    est = _lib.NoiseEstimateC()
    est.n_bins = nb
    est.counts = counts.ctypes.data
    check(fn(*args, C.byref(o._c()), C.byref(est)))
    hist = ErrorHistogram(est.lo, est.hi, est.bin_width, counts, int(est.underflow),
                          int(est.overflow), int(est.samples_used), int(est.within_1px),
                          float(est.sum), float(est.sum_sq))
    return NoiseEstimate(float(est.variance), hist, int(est.samples_used))


def _pairs_checked(frames, who):
    if len(frames) < 2:
        raise ValueError(f"{who}: need at least 2 frames")
    for k in range(1, len(frames)):  # the reference's per-pair order
        _require([frames[k - 1], frames[k]], who, gt=True)
        _require([frames[k - 1], frames[k]], who, pose=True)
    gt = _stack([f.gt_disp for f in frames], np.float64, who)
    poses = _stack([np.asarray(f.pose, np.float64).reshape(3, 4) for f in frames], np.float64, who)
    return gt, poses


def estimate_process_noise(frames, calib, opts=None):
    """estimate_process_noise (noise_calib.cpp:102-128): the GT of frame k-1
    warped by the relative motion vs the GT of frame k, pooled over pairs."""
    o = _as(opts or CalibOptions(), CalibOptions)
    o.validate()
    gt, poses = _pairs_checked(frames, "estimate_process_noise")
    n, h, w = gt.shape
    c = _as(calib, StereoCalib)._c()
    return _estimate(_lib.load().tsgm_estimate_process_noise,
                     (n, w, h, ptr(gt), ptr(poses), C.byref(c)), o)


def estimate_measurement_noise(frames, params, threads=1, opts=None):
    """estimate_measurement_noise (noise_calib.cpp:130-147): full-range SGM vs
    GT per frame, each frame in isolation (batched on the GPU; `threads` is
    accepted and ignored)."""
    o = _as(opts or CalibOptions(), CalibOptions)
    o.validate()
    if len(frames) == 0:
        raise ValueError("estimate_measurement_noise: need at least 1 frame")
    _require(frames, "estimate_measurement_noise", gt=True)
    who = "estimate_measurement_noise"
    left = _stack([f.left for f in frames], np.uint8, who)
    right = _stack([f.right for f in frames], np.uint8, who)
    gt = _stack([f.gt_disp for f in frames], np.float64, who)
    if left.shape != right.shape or left.shape != gt.shape:
        raise ValueError(f"{who}: frame size mismatch")
    n, h, w = gt.shape
    p = _as(params, SgmParams)._c()
    return _estimate(_lib.load().tsgm_estimate_measurement_noise,
                     (n, w, h, ptr(left), ptr(right), ptr(gt), C.byref(p)), o)


def accumulate_error_map(frames, calib):
    """accumulate_error_map (noise_calib.cpp:149-182): per-pixel sum of
    |warped GT - GT| over consecutive pairs (bit-exact)."""
    gt, poses = _pairs_checked(frames, "accumulate_error_map")
    n, h, w = gt.shape
    c = _as(calib, StereoCalib)._c()
    acc = np.zeros((h, w))
    check(_lib.load().tsgm_accumulate_error_map(n, w, h, ptr(gt), ptr(poses), C.byref(c),
                                               ptr(acc)))
    return acc


def release_calibration_cache():
    """Free the device working set the calibration functions keep between
    calls (tsgm_calib_release)."""
    check(_lib.load().tsgm_calib_release())


def _g6(x) -> str:
    """std::ostream << double at precision(6) (%g)."""
    return f"{x:.6g}"


def write_calib_report(path, process, measurement, opts=None):
    """write_calib_report (noise_calib.cpp:184-217): host text, q/r lines a
    run config can load."""
    o = _as(opts or CalibOptions(), CalibOptions)
    o.validate()
    q = max(process.variance, o.q_floor)
    ph, mh = process.hist, measurement.hist
    lines = ["# noise calibration report",
             f"# process:     raw variance {_g6(process.variance)} px^2 over "
             f"{process.samples_used} samples, {_g6(100.0 * ph.fraction_within_1px())}% within +/-1 px",
             f"# measurement: raw variance {_g6(measurement.variance)} px^2 over "
             f"{measurement.samples_used} samples, {_g6(100.0 * mh.fraction_within_1px())}% within +/-1 px"]
    if q != process.variance:
        lines.append(f"# q floor {_g6(o.q_floor)} applied")
    lines += [f"q={_g6(q)}", f"r={_g6(measurement.variance)}", "#",
              f"# error histogram (gate +/-{_g6(o.outlier_gate_px)} px)",
              "# bin_lo bin_hi process_count measurement_count"]
    same = (ph.lo == mh.lo and ph.bin_width == mh.bin_width and len(ph.counts) == len(mh.counts))
    lines.append(f"# -inf {_g6(ph.lo)} {ph.underflow} {mh.underflow}")
    for i in range(len(ph.counts)):
        b0 = ph.lo + float(i) * ph.bin_width
        lines.append(f"# {_g6(b0)} {_g6(b0 + ph.bin_width)} {int(ph.counts[i])} "
                     f"{int(mh.counts[i]) if same else -1}")
    lines.append(f"# {_g6(ph.hi)} +inf {ph.overflow} {mh.overflow}")
    try:
        with open(path, "w") as f:
            f.write("\n".join(lines) + "\n")
    except OSError:
        raise RuntimeError(f"write_calib_report: cannot open {path}") from None


# --------------------------------------------------------------------- engine
_OUT_DTYPES = dict(state_d=np.float64, state_p=np.float64, state_valid=np.uint8,
                   export_d=np.int32, export_valid=np.uint8, diff=np.float64, mask=np.uint8,
                   pred_d=np.float64, pred_p=np.float64, pred_valid=np.uint8, lo=np.uint16,
                   hi=np.uint16, meas_d=np.int32, meas_valid=np.uint8, offsets=np.uint32,
                   cost=np.uint8, agg=np.uint16, subpixel=np.float32)


@dataclass
class EngineConfig:
    calib: StereoCalib
    sgm: SgmParams
    filter: FilterConfig
    max_slots: int = 1
    device: int = 0
    mask_tau: float = 3.0
    keep_volumes: bool = True
    subpixel: bool = False  # A22 extension: export-only sub-pixel WTA (f32)
    vol_slots: int = 0  # volume working set (0 = auto: max_slots, capped to free memory)
    stage_timings: bool = False  # record per-stage device times (Engine.timings)


class Engine:
    """Batched, device-resident production path (tsgm_ctx)."""

    def __init__(self, cfg: EngineConfig):
        self.cfg = cfg
        cal = _as(cfg.calib, StereoCalib)
        c = ConfigC(cal.width, cal.height, cfg.max_slots, cfg.device, cal._c(),
                    _as(cfg.sgm, SgmParams)._c(), _as(cfg.filter, FilterConfig)._c(),
                    cfg.mask_tau, (_lib.TSGM_KEEP_VOLUMES if cfg.keep_volumes else 0) |
                    (_lib.TSGM_SUBPIXEL if cfg.subpixel else 0) |
                    (_lib.TSGM_STAGE_TIMINGS if cfg.stage_timings else 0), cfg.vol_slots)
        self._lib = _lib.load()
        h = C.c_void_p()
        check(self._lib.tsgm_create(C.byref(c), C.byref(h)))
        self._h = h
        self.width, self.height = cal.width, cal.height

    def close(self):
        if getattr(self, "_h", None):
            self._lib.tsgm_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
        return False

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def reset(self, slot: int):
        check(self._lib.tsgm_reset(self._h, slot))

    def _image(self, a, conv, what):
        """The C-ABI reads W*H elements per pointer: check the shape first
        (the reference's step() messages, temporal_filter.cpp:198-204)."""
        a = conv(a)
        if a.shape != (self.height, self.width):
            raise ValueError(what)
        return a

    def set_state(self, slot, d, p, valid):
        d = None if d is None else self._image(d, _f64, "step: state dimension mismatch")
        p = None if p is None else self._image(p, _f64, "step: state dimension mismatch")
        v = None if valid is None else self._image(valid, _u8, "step: state dimension mismatch")
        check(self._lib.tsgm_set_state(self._h, slot, ptr(d), ptr(p), ptr(v)))

    @staticmethod
    def _motions(motions, n):
        m = np.zeros((n, 12))
        for i, (R, t) in enumerate(motions):
            m[i, :9] = np.asarray(R, np.float64).ravel()
            m[i, 9:] = np.asarray(t, np.float64).ravel()
        return m

    def step(self, slots, lefts, rights, motions):
        """One frame for ``len(slots)`` sequences; host u8 images; motions =
        [(R 3x3, t 3)] (identity for a first frame)."""
        n = len(slots)
        sl = np.asarray(slots, np.int32)
        if len(lefts) != n or len(rights) != n or len(motions) != n:
            raise ValueError("Engine.step: slots, images and motions differ in length")
        for a, b in zip(lefts, rights):
            if np.shape(a) != np.shape(b):
                raise ValueError("step: left/right dimension mismatch")
        ls = [self._image(x, _u8, "step: state dimension mismatch") for x in lefts]
        rs = [self._image(x, _u8, "step: state dimension mismatch") for x in rights]
        lp = (C.c_void_p * n)(*[x.ctypes.data for x in ls])
        rp = (C.c_void_p * n)(*[x.ctypes.data for x in rs])
        m = self._motions(motions, n)
        check(self._lib.tsgm_step(self._h, n, ptr(sl), lp, rp, ptr(m)))

    def step_device(self, slots, left_ptrs, right_ptrs, motion12, after_stream=None):
        """Device-resident inputs: raw CUDA pointers (W*H bytes each), motion12
        f64 [n, 12]. With ``after_stream`` (a cudaStream_t handle, e.g.
        ``torch.cuda.current_stream().cuda_stream``) the step is ordered after
        the work enqueued on it so far; otherwise the images must already be
        complete (tsgm_step_device)."""
        n = len(slots)
        sl = np.asarray(slots, np.int32)
        if len(left_ptrs) != n or len(right_ptrs) != n:
            raise ValueError("Engine.step_device: slots and image pointers differ in length")
        lp = (C.c_void_p * n)(*left_ptrs)
        rp = (C.c_void_p * n)(*right_ptrs)
        m = _f64(motion12)
        if m.shape != (n, 12):
            raise ValueError("Engine.step_device: motion12 must be [n, 12]")
        if after_stream is None:
            check(self._lib.tsgm_step_device(self._h, n, ptr(sl), lp, rp, ptr(m)))
        else:
            check(self._lib.tsgm_step_device_after(self._h, n, ptr(sl), lp, rp, ptr(m),
                                                   C.c_void_p(after_stream)))

    def inputs_consumed(self, stream):
        """Make ``stream`` (cudaStream_t handle) wait until the last step has
        read its input images (after that they may be refilled)."""
        check(self._lib.tsgm_inputs_consumed(self._h, C.c_void_p(stream)))

    def last_kernels(self) -> str:
        """The aggregation kernels the last step ran (scan + combine/WTA)."""
        buf = C.create_string_buffer(256)
        check(self._lib.tsgm_last_kernels(self._h, buf, 256))
        return buf.value.decode()

    def last_chunks(self) -> int:
        """Volume chunks the last step needed (volumes packed by actual cells)."""
        v = C.c_int32(0)
        check(self._lib.tsgm_last_chunks(self._h, C.byref(v)))
        return v.value

    def timings(self):
        """StepTimings of the last step (whole batch, device seconds); needs
        ``EngineConfig(stage_timings=True)``."""
        t = _lib.StageTimingsC()
        check(self._lib.tsgm_last_stage_timings(self._h, C.byref(t)))
        return _timings_dict(t)

    def cells(self, slot) -> int:
        v = C.c_uint64()
        check(self._lib.tsgm_cells(self._h, slot, C.byref(v)))
        return int(v.value)

    def fetch(self, slot: int, what: str, out=None):
        dt = _OUT_DTYPES[what]
        if what in ("cost", "agg"):
            shape = (self.cells(slot),)
        elif what == "offsets":
            shape = (self.width * self.height + 1,)
        else:
            shape = (self.height, self.width)
        if out is None:
            out = np.empty(shape, dt)
        check(self._lib.tsgm_fetch(self._h, slot, OUT[what], ptr(out), out.nbytes))
        return out

    def fetch_batch(self, slots, what: str, outs):
        """Asynchronously copy output ``what`` of ``slots`` into ``outs`` (pinned
        host arrays for overlap); completes at the next :meth:`sync`."""
        n = len(slots)
        sl = np.asarray(slots, np.int32)
        if len(outs) != n:
            raise ValueError("Engine.fetch_batch: one output array per slot")
        for o in outs:
            if not (isinstance(o, np.ndarray) and o.flags.c_contiguous and o.flags.writeable):
                raise ValueError("Engine.fetch_batch: outputs must be writeable C-contiguous arrays")
        # every destination must hold a whole map: pass the smallest size
        dp = (C.c_void_p * n)(*[o.ctypes.data for o in outs])
        check(self._lib.tsgm_fetch_batch(self._h, n, ptr(sl), OUT[what], dp,
                                         min(o.nbytes for o in outs)))

    def sync(self):
        check(self._lib.tsgm_sync(self._h))

    def timer_begin(self):
        check(self._lib.tsgm_timer_begin(self._h))

    def timer_end(self) -> float:
        ms = C.c_float()
        check(self._lib.tsgm_timer_end(self._h, C.byref(ms)))
        return float(ms.value)

    def detect(self, slots, cfg=None, cap_each=1024):
        """detect_moving_objects on each slot's diff map of the last step
        (SAT + scoring on the GPU, merges on host threads); list of [n, 5]."""
        sl = np.asarray(slots, np.int32)
        wh, c = _as(cfg or DetectConfig(), DetectConfig)._c()
        while True:
            out = _box_array(cap_each * len(sl))
            n_each = np.zeros(len(sl), np.int64)
            check(self._lib.tsgm_detect(self._h, len(sl), ptr(sl), C.byref(c), ptr(out), cap_each,
                                        ptr(n_each)))
            if n_each.max(initial=0) <= cap_each:
                return [_boxes_out(out[i * cap_each:(i + 1) * cap_each], int(n_each[i]))
                        for i in range(len(sl))]
            cap_each = int(n_each.max())

    def write_export_png(self, slot, path):
        """The slot's last export map as a KITTI 16-bit PNG (tsgm_main.cpp:157),
        quantised on the device."""
        check(self._lib.tsgm_write_export_png(self._h, int(slot), str(path).encode()))

    def write_export_pngs(self, slots, paths):
        """Many slots' export maps as PNGs: one device quantisation, the PNG
        containers encoded on host threads."""
        sl = np.asarray(slots, np.int32)
        enc = [str(p).encode() for p in paths]
        if len(enc) != len(sl):
            raise ValueError("write_export_pngs: one path per slot")
        arr = (C.c_char_p * len(enc))(*enc)
        check(self._lib.tsgm_write_export_pngs(self._h, len(sl), ptr(sl), arr))

    def count_outliers(self, slots, gts, what="export_d", opts=None):
        """count_outliers of each slot's last export map (or WTA map) against
        host GT maps -> (evaluated[n], outliers[n])."""
        sl = np.asarray(slots, np.int32)
        gs = [_f64(g) for g in gts]
        gp = (C.c_void_p * len(gs))(*[g.ctypes.data for g in gs])
        o = _as(opts or OutlierOptions(), OutlierOptions)._c()
        ev = np.zeros(len(sl), np.int64)
        out = np.zeros(len(sl), np.int64)
        check(self._lib.tsgm_count_outliers_batch(self._h, len(sl), ptr(sl), OUT[what], gp,
                                                  C.byref(o), ptr(ev), ptr(out)))
        return ev, out

    @property
    def vol_slots(self) -> int:
        """Sequences whose per-frame volumes are resident at once."""
        v = C.c_int32()
        check(self._lib.tsgm_volume_slots(self._h, C.byref(v)))
        return int(v.value)

    def bench_aggregate(self, slots, reps=10):
        """Standalone C -> S aggregation over the slots' current volumes:
        (ms per aggregation, total cells)."""
        sl = np.asarray(slots, np.int32)
        ms = C.c_float()
        cells = C.c_uint64()
        check(self._lib.tsgm_bench_aggregate(self._h, len(sl), ptr(sl), reps, C.byref(ms),
                                             C.byref(cells)))
        return float(ms.value), int(cells.value)

    @property
    def launches(self) -> int:
        return int(self._lib.tsgm_launch_count(self._h))


class PipelinedEngine:
    """A batch split over ``groups`` independent contexts on one GPU.

    Every context has its own streams, so one group's integer-issue-bound
    scan overlaps the other groups' DRAM-bound kernels (combine, correct, the
    per-pixel chain) and fills the tail of its horizontal walks: measured on
    config 2, 64 sequences x 30 frames, 6471 -> 6750 frames/s with two groups
    (32 sequences: 5964 -> 6190; four groups lose). Global slot ``s`` lives in
    context ``s // per`` as local slot ``s % per``; a step enqueues each
    context's share and returns, exactly like :class:`Engine`. Sequences are
    independent (eval.cpp:114-144), so the results are those of one context.
    """

    def __init__(self, cfg: EngineConfig, groups: int = 2):
        groups = max(1, min(int(groups), cfg.max_slots))
        self.per = -(-cfg.max_slots // groups)
        self.cfg = cfg
        self.engines = []
        left = cfg.max_slots
        for _ in range(groups):
            n = min(self.per, left)
            if n <= 0:
                break
            left -= n
            c = EngineConfig(**{**cfg.__dict__, "max_slots": n,
                                "vol_slots": min(cfg.vol_slots, n) if cfg.vol_slots else 0})
            self.engines.append(Engine(c))
        self.width, self.height = self.engines[0].width, self.engines[0].height

    def close(self):
        for e in self.engines:
            e.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
        return False

    def _where(self, slot):
        g, l = divmod(int(slot), self.per)
        if slot < 0 or g >= len(self.engines):
            raise ValueError("slot out of range")
        return g, l

    def _split(self, slots):
        """Per context: (positions in the caller's lists, local slots)."""
        parts = [([], []) for _ in self.engines]
        for i, s in enumerate(slots):
            g, l = self._where(s)
            parts[g][0].append(i)
            parts[g][1].append(l)
        return parts

    def reset(self, slot):
        g, l = self._where(slot)
        self.engines[g].reset(l)

    def set_state(self, slot, d, p, valid):
        g, l = self._where(slot)
        self.engines[g].set_state(l, d, p, valid)

    def step(self, slots, lefts, rights, motions):
        if not (len(lefts) == len(rights) == len(motions) == len(slots)):
            raise ValueError("Engine.step: slots, images and motions differ in length")
        for e, (idx, loc) in zip(self.engines, self._split(slots)):
            if idx:
                e.step(loc, [lefts[i] for i in idx], [rights[i] for i in idx],
                       [motions[i] for i in idx])

    def step_device(self, slots, left_ptrs, right_ptrs, motion12, after_stream=None):
        m = _f64(motion12)
        if not (len(left_ptrs) == len(right_ptrs) == len(slots)) or m.shape != (len(slots), 12):
            raise ValueError("Engine.step_device: slots, image pointers and motion12 differ in length")
        for e, (idx, loc) in zip(self.engines, self._split(slots)):
            if idx:
                e.step_device(loc, [left_ptrs[i] for i in idx], [right_ptrs[i] for i in idx],
                              m[idx], after_stream)

    def fetch(self, slot, what, out=None):
        g, l = self._where(slot)
        return self.engines[g].fetch(l, what, out)

    def fetch_batch(self, slots, what, outs):
        if len(outs) != len(slots):
            raise ValueError("Engine.fetch_batch: one output array per slot")
        for e, (idx, loc) in zip(self.engines, self._split(slots)):
            if idx:
                e.fetch_batch(loc, what, [outs[i] for i in idx])

    def sync(self):
        for e in self.engines:
            e.sync()

    def timer_begin(self):
        """Start every context's device timer (call with the device idle: the
        begin events then coincide)."""
        for e in self.engines:
            e.timer_begin()

    def timer_end(self) -> float:
        """Device milliseconds since timer_begin: the longest context."""
        return max(e.timer_end() for e in self.engines)

    def count_outliers(self, slots, gts, what="export_d", opts=None):
        ev = np.zeros(len(slots), np.int64)
        out = np.zeros(len(slots), np.int64)
        for e, (idx, loc) in zip(self.engines, self._split(slots)):
            if idx:
                a, b = e.count_outliers(loc, [gts[i] for i in idx], what, opts)
                ev[idx], out[idx] = a, b
        return ev, out

    def detect(self, slots, cfg=None, cap_each=1024):
        res = [None] * len(slots)
        for e, (idx, loc) in zip(self.engines, self._split(slots)):
            if idx:
                for i, r in zip(idx, e.detect(loc, cfg, cap_each)):
                    res[i] = r
        return res

    def cells(self, slot) -> int:
        g, l = self._where(slot)
        return self.engines[g].cells(l)

    def last_kernels(self) -> str:
        return self.engines[0].last_kernels()

    def last_chunks(self) -> int:
        return max(e.last_chunks() for e in self.engines)

    @property
    def launches(self) -> int:
        return sum(e.launches for e in self.engines)
