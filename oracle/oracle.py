"""TEST INFRASTRUCTURE ONLY — ctypes front-end over the two CPU checkers.

``Port`` wraps the C restatement (oracle/tsgm_oracle.c); ``Reference`` wraps
the reference's own sources compiled in place (oracle/Makefile +
oracle/ref_runner.cpp). Both expose the same numpy-level API so a test can run
the same comparison against either. Parameter objects are duck-typed: anything
with the attribute names of ``Calib`` / ``SgmParams`` / ``FilterConfig``
(including the product's own dataclasses) is accepted.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")
PORT_SO = os.path.join(REF_DIR, "liboracle.so")
REF_SO = os.path.join(REF_DIR, "libtsgm_ref.so")
REFERENCE_SRC = "/root/reference/proj"


@dataclass
class Calib:
    focal_px: float = 720.0
    cx: float = 621.0
    cy: float = 187.5
    baseline_m: float = 0.54
    width: int = 1242
    height: int = 375
    d_max: int = 128


@dataclass
class SgmParams:
    p1: int = 6
    p2: int = 65
    paths: int = 8
    path_set: int = 0  # 0 nondiagonal, 1 diagonal (sgm.hpp:10-13)
    d_max: int = 128


@dataclass
class FilterConfig:
    q: float = 0.5
    r: float = 1.0
    p_init: float = 4096.0
    disc_thresh: float = 2.0
    min_range_halfwidth: int = 2
    range_use_stddev: bool = False
    range_stddev_gain: float = 2.0


@dataclass
class CalibOpts:
    """CalibOptions (noise_calib.hpp:43-49)."""
    outlier_gate_px: float = 10.0
    bin_width: float = 0.25
    q_floor: float = 0.1


@dataclass
class DetectConfig:
    """DetectConfig (motion_detect.hpp:36-44)."""
    window_sizes: tuple = ((20, 20), (30, 30), (40, 40), (50, 50), (50, 75))
    score_thresh: float = 2.0
    merge_stop_iou: float = 0.2
    min_box_area: int = 400


def _wh(cfg):
    return np.ascontiguousarray(np.array(cfg.window_sizes, dtype=np.int32).reshape(-1))


def _boxes_arr(boxes):
    """Boxes as float64 [n, 5] = x0, y0, x1, y1, score."""
    return np.ascontiguousarray(np.asarray(boxes, dtype=np.float64).reshape(-1, 5))


def build(reference: bool = True) -> None:
    """Compile the checkers (``make -C oracle``); the reference only when its
    sources are present (this container, not the GPU box)."""
    targets = ["oracle"]
    if reference and os.path.isdir(os.path.join(REFERENCE_SRC, "src")):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _u8(a):
    return np.ascontiguousarray(a, dtype=np.uint8)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _sgm_arr(p):
    return np.array([p.p1, p.p2, p.paths, int(p.path_set), p.d_max], dtype=np.int32)


def _filter_arr(f):
    return np.array([f.q, f.r, f.p_init, f.disc_thresh, f.min_range_halfwidth,
                     1.0 if f.range_use_stddev else 0.0, f.range_stddev_gain], dtype=np.float64)


def offsets_of(lo, hi):
    n = (hi.astype(np.int64) - lo.astype(np.int64) + 1).ravel()
    off = np.zeros(n.size + 1, dtype=np.int64)
    np.cumsum(n, out=off[1:])
    return off.astype(np.uint32) if off[-1] <= 0xFFFFFFFF else off


class _Lib:
    so_path = ""

    def __init__(self):
        if not os.path.exists(self.so_path):
            raise FileNotFoundError(f"{self.so_path} missing: run `make -C oracle`")
        self.lib = C.CDLL(self.so_path)

    def _check(self, rc, errfn):
        if rc == 0:
            return
        msg = errfn().decode()
        if rc == 1:
            raise ValueError(msg)
        raise RuntimeError(msg)


class Reference(_Lib):
    """The reference's own code (oracle/_ref/libtsgm_ref.so)."""

    so_path = REF_SO
    kind = "reference"

    def __init__(self):
        super().__init__()
        self.lib.ref_last_error.restype = C.c_char_p

    def _c(self, rc):
        self._check(rc, self.lib.ref_last_error)

    def census(self, img):
        img = _u8(img)
        h, w = img.shape
        sig = np.zeros((h, w), np.uint32)
        self._c(self.lib.ref_census(_p(img), w, h, _p(sig)))
        return sig

    def cost_volume(self, left, right, lo, hi, threads=1):
        left, right = _u8(left), _u8(right)
        h, w = left.shape
        lo = np.ascontiguousarray(lo, np.uint16)
        hi = np.ascontiguousarray(hi, np.uint16)
        off = offsets_of(lo, hi)
        cap = int(off[-1])
        cost = np.zeros(cap + 1, np.uint8)
        off32 = np.zeros(w * h + 1, np.uint32)
        self._c(self.lib.ref_cost_volume(_p(left), _p(right), w, h, _p(lo), _p(hi), _p(off32),
                                         _p(cost), C.c_uint64(cap + 1), threads))
        return off32, cost[:cap]

    def aggregate(self, cost, lo, hi, params):
        lo = np.ascontiguousarray(lo, np.uint16)
        hi = np.ascontiguousarray(hi, np.uint16)
        h, w = lo.shape
        cost = _u8(cost)
        agg = np.zeros(max(cost.size, 1), np.uint16)
        sp = _sgm_arr(params)
        self._c(self.lib.ref_aggregate(_p(cost), _p(lo), _p(hi), w, h, _p(sp), _p(agg)))
        return agg[: cost.size]

    def wta(self, agg, lo, hi):
        lo = np.ascontiguousarray(lo, np.uint16)
        hi = np.ascontiguousarray(hi, np.uint16)
        h, w = lo.shape
        agg = np.ascontiguousarray(agg, np.uint16)
        d = np.zeros((h, w), np.int32)
        v = np.zeros((h, w), np.uint8)
        self._c(self.lib.ref_wta(_p(agg), _p(lo), _p(hi), w, h, _p(d), _p(v)))
        return d, v

    def median(self, d, valid):
        d = np.ascontiguousarray(d, np.int32)
        valid = _u8(valid)
        h, w = d.shape
        od = np.zeros((h, w), np.int32)
        ov = np.zeros((h, w), np.uint8)
        self._c(self.lib.ref_median(_p(d), _p(valid), w, h, _p(od), _p(ov)))
        return od, ov

    def sgm_match(self, left, right, lo, hi, params, threads=1):
        left, right = _u8(left), _u8(right)
        h, w = left.shape
        lo = np.ascontiguousarray(lo, np.uint16)
        hi = np.ascontiguousarray(hi, np.uint16)
        d = np.zeros((h, w), np.int32)
        v = np.zeros((h, w), np.uint8)
        sp = _sgm_arr(params)
        self._c(self.lib.ref_sgm_match(_p(left), _p(right), w, h, _p(lo), _p(hi), _p(sp),
                                       threads, _p(d), _p(v)))
        return d, v

    def relative_motion(self, prev12, cur12):
        prev12, cur12 = _f64(prev12).ravel(), _f64(cur12).ravel()
        r = np.zeros(9)
        t = np.zeros(3)
        self._c(self.lib.ref_relative_motion(_p(prev12), _p(cur12), _p(r), _p(t)))
        return r.reshape(3, 3), t

    def homography(self, R, t, calib):
        R, t = _f64(R).ravel(), _f64(t).ravel()
        c4 = np.array([calib.focal_px, calib.cx, calib.cy, calib.baseline_m])
        H = np.zeros(16)
        self._c(self.lib.ref_homography(_p(R), _p(t), _p(c4), calib.width, calib.height,
                                        calib.d_max, _p(H)))
        return H.reshape(4, 4)

    def warp(self, d, p, valid, H, d_max):
        d, p, valid, H = _f64(d), _f64(p), _u8(valid), _f64(H).ravel()
        h, w = d.shape
        od, op, osrc = (np.zeros((h, w)) for _ in range(3))
        ov = np.zeros((h, w), np.uint8)
        self._c(self.lib.ref_warp(_p(d), _p(p), _p(valid), w, h, _p(H), d_max, _p(od), _p(op),
                                  _p(ov), _p(osrc)))
        return od, op, ov, osrc

    def predict(self, d, p, valid, R, t, calib, filt):
        d, p, valid = _f64(d), _f64(p), _u8(valid)
        R, t = _f64(R).ravel(), _f64(t).ravel()
        h, w = d.shape
        c4 = np.array([calib.focal_px, calib.cx, calib.cy, calib.baseline_m])
        fa = _filter_arr(filt)
        od, op = np.zeros((h, w)), np.zeros((h, w))
        ov = np.zeros((h, w), np.uint8)
        self._c(self.lib.ref_predict(_p(d), _p(p), _p(valid), w, h, _p(R), _p(t), _p(c4),
                                     calib.d_max, _p(fa), _p(od), _p(op), _p(ov)))
        return od, op, ov

    def reject(self, d, p, valid, filt):
        d, p, valid = _f64(d), _f64(p), _u8(valid)
        h, w = d.shape
        fa = _filter_arr(filt)
        od, op = np.zeros((h, w)), np.zeros((h, w))
        ov = np.zeros((h, w), np.uint8)
        self._c(self.lib.ref_reject(_p(d), _p(p), _p(valid), w, h, _p(fa), _p(od), _p(op),
                                    _p(ov)))
        return od, op, ov

    def fill(self, d, p, valid):
        d, p, valid = _f64(d), _f64(p), _u8(valid)
        h, w = d.shape
        od, op = np.zeros((h, w)), np.zeros((h, w))
        ov = np.zeros((h, w), np.uint8)
        self._c(self.lib.ref_fill(_p(d), _p(p), _p(valid), w, h, _p(od), _p(op), _p(ov)))
        return od, op, ov

    def ranges(self, d, p, valid, calib, filt):
        d, p, valid = _f64(d), _f64(p), _u8(valid)
        h, w = d.shape
        c4 = np.array([calib.focal_px, calib.cx, calib.cy, calib.baseline_m])
        fa = _filter_arr(filt)
        lo = np.zeros((h, w), np.uint16)
        hi = np.zeros((h, w), np.uint16)
        self._c(self.lib.ref_ranges(_p(d), _p(p), _p(valid), w, h, _p(c4), calib.d_max, _p(fa),
                                    _p(lo), _p(hi)))
        return lo, hi

    def correct(self, d, p, valid, md, mv, filt):
        d, p, valid = _f64(d), _f64(p), _u8(valid)
        md, mv = np.ascontiguousarray(md, np.int32), _u8(mv)
        h, w = d.shape
        fa = _filter_arr(filt)
        od, op = np.zeros((h, w)), np.zeros((h, w))
        ov = np.zeros((h, w), np.uint8)
        self._c(self.lib.ref_correct(_p(d), _p(p), _p(valid), _p(md), _p(mv), w, h, _p(fa),
                                     _p(od), _p(op), _p(ov)))
        return od, op, ov

    def diff(self, d, p, valid, md, mv):
        d, p, valid = _f64(d), _f64(p), _u8(valid)
        md, mv = np.ascontiguousarray(md, np.int32), _u8(mv)
        h, w = d.shape
        out = np.zeros((h, w))
        self._c(self.lib.ref_disparity_difference(_p(d), _p(p), _p(valid), _p(md), _p(mv), w, h,
                                                  _p(out)))
        return out

    def step(self, state, left, right, R, t, calib, params, filt, threads=1):
        """tsgm::step. ``state`` = (d, p, valid) or None for the default state."""
        left, right = _u8(left), _u8(right)
        h, w = left.shape
        R, t = _f64(R).ravel(), _f64(t).ravel()
        c4 = np.array([calib.focal_px, calib.cx, calib.cy, calib.baseline_m])
        sp, fa = _sgm_arr(params), _filter_arr(filt)
        if state is None:
            sd = sp_ = sv = None
            sw = sh = 0
        else:
            sd, sp_, sv = _f64(state[0]), _f64(state[1]), _u8(state[2])
            sh, sw = sd.shape
        od, op, diff = np.zeros((h, w)), np.zeros((h, w)), np.zeros((h, w))
        ov = np.zeros((h, w), np.uint8)
        ed = np.zeros((h, w), np.int32)
        ev = np.zeros((h, w), np.uint8)
        self._c(self.lib.ref_step(_p(sd), _p(sp_), _p(sv), sw, sh, _p(left), _p(right), w, h,
                                  _p(R), _p(t), _p(c4), calib.d_max, _p(sp), _p(fa), threads,
                                  _p(od), _p(op), _p(ov), _p(ed), _p(ev), _p(diff)))
        return dict(d=od, p=op, valid=ov, export_d=ed, export_valid=ev, diff=diff)


    # ---- box detector (motion_detect.cpp) ----
    def integral_image(self, m):
        m = _f64(m)
        h, w = m.shape
        sat = np.zeros((h + 1, w + 1))
        self._c(self.lib.ref_integral_image(_p(m), w, h, _p(sat)))
        return sat

    def _detect_args(self, cfg):
        wh = _wh(cfg)
        return wh, [_p(wh), len(cfg.window_sizes), C.c_double(cfg.score_thresh),
                    C.c_double(cfg.merge_stop_iou), C.c_longlong(cfg.min_box_area)]

    def candidates(self, diff, cfg, threads=1):
        diff = _f64(diff)
        h, w = diff.shape
        wh, args = self._detect_args(cfg)
        n = C.c_longlong()
        cap = 1 << 16
        while True:
            out = np.zeros((cap, 5))
            self._c(self.lib.ref_candidates(_p(diff), w, h, *args, threads, _p(out),
                                            C.c_longlong(cap), C.byref(n)))
            if n.value <= cap:
                return out[:n.value]
            cap = n.value

    def greedy_merge(self, boxes, cfg):
        b = _boxes_arr(boxes)
        wh, args = self._detect_args(cfg)
        out = np.zeros_like(b)
        n = C.c_longlong()
        self._c(self.lib.ref_greedy_merge(_p(b), C.c_longlong(len(b)), *args, _p(out),
                                          C.byref(n)))
        return out[:n.value]

    def detect(self, diff, cfg, threads=1):
        return self.greedy_merge(self.candidates(diff, cfg, threads), cfg)


    def count_outliers(self, d, valid, gt, abs_thresh=3.0, rel_thresh=0.05, strict=False):
        d, valid, gt = np.ascontiguousarray(d, np.int32), _u8(valid), _f64(gt)
        h, w = gt.shape
        ev, out = C.c_longlong(), C.c_longlong()
        self._c(self.lib.ref_count_outliers(_p(d), _p(valid), _p(gt), w, h, C.c_double(abs_thresh),
                                            C.c_double(rel_thresh), int(strict), C.byref(ev),
                                            C.byref(out)))
        return ev.value, out.value


class _OrCalib(C.Structure):
    _fields_ = [("focal_px", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("baseline_m", C.c_double), ("width", C.c_int), ("height", C.c_int),
                ("d_max", C.c_int)]


class _OrSgm(C.Structure):
    _fields_ = [("p1", C.c_int), ("p2", C.c_int), ("paths", C.c_int), ("path_set", C.c_int),
                ("d_max", C.c_int)]


class _OrFilter(C.Structure):
    _fields_ = [("q", C.c_double), ("r", C.c_double), ("p_init", C.c_double),
                ("disc_thresh", C.c_double), ("min_range_halfwidth", C.c_int),
                ("range_use_stddev", C.c_int), ("range_stddev_gain", C.c_double)]


class _OrDebug(C.Structure):
    _fields_ = [("pred_d", C.c_void_p), ("pred_p", C.c_void_p), ("pred_v", C.c_void_p),
                ("lo", C.c_void_p), ("hi", C.c_void_p), ("meas_d", C.c_void_p),
                ("meas_v", C.c_void_p), ("mask", C.c_void_p), ("mask_tau", C.c_double)]


def _calib(c):
    return _OrCalib(c.focal_px, c.cx, c.cy, c.baseline_m, c.width, c.height, c.d_max)


def _sgm(p):
    return _OrSgm(p.p1, p.p2, p.paths, int(p.path_set), p.d_max)


def _filt(f):
    return _OrFilter(f.q, f.r, f.p_init, f.disc_thresh, f.min_range_halfwidth,
                     1 if f.range_use_stddev else 0, f.range_stddev_gain)


class Port(_Lib):
    """The C restatement (oracle/_ref/liboracle.so)."""

    so_path = PORT_SO
    kind = "port"

    def __init__(self):
        super().__init__()
        self.lib.or_last_error.restype = C.c_char_p
        self.lib.or_offsets.restype = C.c_int64

    def _c(self, rc):
        self._check(rc, self.lib.or_last_error)

    def census(self, img):
        img = _u8(img)
        h, w = img.shape
        sig = np.zeros((h, w), np.uint32)
        self._c(self.lib.or_census(_p(img), w, h, _p(sig)))
        return sig

    def offsets(self, lo, hi):
        lo = np.ascontiguousarray(lo, np.uint16)
        hi = np.ascontiguousarray(hi, np.uint16)
        off = np.zeros(lo.size + 1, np.uint32)
        n = self.lib.or_offsets(_p(lo), _p(hi), C.c_size_t(lo.size), _p(off))
        if n < 0:
            self._c(1)
        return off

    def cost_volume(self, left, right, lo, hi, threads=1):
        lo = np.ascontiguousarray(lo, np.uint16)
        hi = np.ascontiguousarray(hi, np.uint16)
        h, w = lo.shape
        sl, sr = self.census(left), self.census(right)
        off = self.offsets(lo, hi)
        cost = np.zeros(int(off[-1]) + 1, np.uint8)
        self.lib.or_cost_volume(_p(sl), _p(sr), w, h, _p(lo), _p(off), _p(cost))
        return off, cost[: int(off[-1])]

    def aggregate(self, cost, lo, hi, params):
        lo = np.ascontiguousarray(lo, np.uint16)
        hi = np.ascontiguousarray(hi, np.uint16)
        h, w = lo.shape
        off = self.offsets(lo, hi)
        cost = _u8(cost)
        agg = np.zeros(max(cost.size, 1), np.uint16)
        sp = _sgm(params)
        self._c(self.lib.or_aggregate(_p(cost), _p(lo), _p(off), w, h, C.byref(sp), _p(agg)))
        return agg[: cost.size]

    def aggregate_direction(self, cost, lo, hi, dx, dy, p1, p2):
        lo = np.ascontiguousarray(lo, np.uint16)
        hi = np.ascontiguousarray(hi, np.uint16)
        h, w = lo.shape
        off = self.offsets(lo, hi)
        cost = _u8(cost)
        out = np.zeros(max(cost.size, 1), np.uint16)
        self.lib.or_aggregate_direction(_p(cost), _p(lo), _p(off), w, h, dx, dy, p1, p2, _p(out))
        return out[: cost.size]

    def wta(self, agg, lo, hi):
        lo = np.ascontiguousarray(lo, np.uint16)
        hi = np.ascontiguousarray(hi, np.uint16)
        h, w = lo.shape
        off = self.offsets(lo, hi)
        agg = np.ascontiguousarray(agg, np.uint16)
        d = np.zeros((h, w), np.int32)
        v = np.zeros((h, w), np.uint8)
        self.lib.or_wta(_p(agg), _p(lo), _p(off), w, h, _p(d), _p(v))
        return d, v

    def median(self, d, valid):
        d = np.ascontiguousarray(d, np.int32)
        valid = _u8(valid)
        h, w = d.shape
        od = np.zeros((h, w), np.int32)
        ov = np.zeros((h, w), np.uint8)
        self.lib.or_median(_p(d), _p(valid), w, h, _p(od), _p(ov))
        return od, ov

    def sgm_match(self, left, right, lo, hi, params, threads=1):
        left, right = _u8(left), _u8(right)
        h, w = left.shape
        lo = np.ascontiguousarray(lo, np.uint16)
        hi = np.ascontiguousarray(hi, np.uint16)
        d = np.zeros((h, w), np.int32)
        v = np.zeros((h, w), np.uint8)
        sp = _sgm(params)
        self._c(self.lib.or_sgm_match(_p(left), _p(right), w, h, _p(lo), _p(hi), C.byref(sp),
                                      _p(d), _p(v)))
        return d, v

    def relative_motion(self, prev12, cur12):
        prev12, cur12 = _f64(prev12).ravel(), _f64(cur12).ravel()
        r = np.zeros(9)
        t = np.zeros(3)
        self._c(self.lib.or_relative_motion(_p(prev12), _p(cur12), _p(r), _p(t)))
        return r.reshape(3, 3), t

    def homography(self, R, t, calib):
        R, t = _f64(R).ravel(), _f64(t).ravel()
        H = np.zeros(16)
        c = _calib(calib)
        self._c(self.lib.or_homography(_p(R), _p(t), C.byref(c), _p(H)))
        return H.reshape(4, 4)

    def warp(self, d, p, valid, H, d_max):
        d, p, valid, H = _f64(d), _f64(p), _u8(valid), _f64(H).ravel()
        h, w = d.shape
        od, op, osrc = (np.zeros((h, w)) for _ in range(3))
        ov = np.zeros((h, w), np.uint8)
        self.lib.or_warp(_p(d), _p(p), _p(valid), w, h, _p(H), d_max, _p(od), _p(op), _p(ov),
                         _p(osrc))
        return od, op, ov, osrc

    def predict(self, d, p, valid, R, t, calib, filt):
        d, p, valid = _f64(d), _f64(p), _u8(valid)
        R, t = _f64(R).ravel(), _f64(t).ravel()
        h, w = d.shape
        od, op = np.zeros((h, w)), np.zeros((h, w))
        ov = np.zeros((h, w), np.uint8)
        c, f = _calib(calib), _filt(filt)
        self._c(self.lib.or_predict(_p(d), _p(p), _p(valid), w, h, _p(R), _p(t), C.byref(c),
                                    C.byref(f), _p(od), _p(op), _p(ov)))
        return od, op, ov

    def reject(self, d, p, valid, filt):
        d, p, valid = _f64(d), _f64(p), _u8(valid)
        h, w = d.shape
        od, op = np.zeros((h, w)), np.zeros((h, w))
        ov = np.zeros((h, w), np.uint8)
        self.lib.or_reject(_p(d), _p(p), _p(valid), w, h, C.c_double(filt.disc_thresh), _p(od),
                           _p(op), _p(ov))
        return od, op, ov

    def fill(self, d, p, valid):
        d, p, valid = _f64(d), _f64(p), _u8(valid)
        h, w = d.shape
        od, op = np.zeros((h, w)), np.zeros((h, w))
        ov = np.zeros((h, w), np.uint8)
        self.lib.or_fill(_p(d), _p(p), _p(valid), w, h, _p(od), _p(op), _p(ov))
        return od, op, ov

    def ranges(self, d, p, valid, calib, filt):
        d, p, valid = _f64(d), _f64(p), _u8(valid)
        h, w = d.shape
        lo = np.zeros((h, w), np.uint16)
        hi = np.zeros((h, w), np.uint16)
        f = _filt(filt)
        self.lib.or_ranges(_p(d), _p(p), _p(valid), w, h, calib.d_max, C.byref(f), _p(lo),
                           _p(hi))
        return lo, hi

    def correct(self, d, p, valid, md, mv, filt):
        d, p, valid = _f64(d), _f64(p), _u8(valid)
        md, mv = np.ascontiguousarray(md, np.int32), _u8(mv)
        h, w = d.shape
        od, op = np.zeros((h, w)), np.zeros((h, w))
        ov = np.zeros((h, w), np.uint8)
        self.lib.or_correct(_p(d), _p(p), _p(valid), _p(md), _p(mv), w, h, C.c_double(filt.r),
                            _p(od), _p(op), _p(ov))
        return od, op, ov

    def diff(self, d, p, valid, md, mv):
        d, valid = _f64(d), _u8(valid)
        md, mv = np.ascontiguousarray(md, np.int32), _u8(mv)
        h, w = d.shape
        out = np.zeros((h, w))
        self.lib.or_diff(_p(d), _p(valid), _p(md), _p(mv), w, h, _p(out))
        return out

    def mask(self, d, p, valid, md, mv, r, tau):
        d, p, valid = _f64(d), _f64(p), _u8(valid)
        md, mv = np.ascontiguousarray(md, np.int32), _u8(mv)
        h, w = d.shape
        out = np.zeros((h, w), np.uint8)
        self.lib.or_mask(_p(d), _p(p), _p(valid), _p(md), _p(mv), w, h, C.c_double(r),
                         C.c_double(tau), _p(out))
        return out

    def subpixel(self, agg, lo, hi, d, valid):
        lo = np.ascontiguousarray(lo, np.uint16)
        hi = np.ascontiguousarray(hi, np.uint16)
        hh, w = lo.shape
        off = self.offsets(lo, hi)
        agg = np.ascontiguousarray(agg, np.uint16)
        out = np.zeros((hh, w), np.float32)
        self.lib.or_subpixel(_p(agg), _p(lo), _p(hi), _p(off), _p(np.ascontiguousarray(d, np.int32)),
                             _p(_u8(valid)), w, hh, _p(out))
        return out

    def render(self, d, valid):
        d, valid = _f64(d), _u8(valid)
        h, w = d.shape
        od = np.zeros((h, w), np.int32)
        ov = np.zeros((h, w), np.uint8)
        self.lib.or_render(_p(d), _p(valid), w, h, _p(od), _p(ov))
        return od, ov

    def step(self, state, left, right, R, t, calib, params, filt, threads=1, debug=False,
             mask_tau=3.0):
        """tsgm::step; with ``debug`` also returns pred/ranges/meas/mask."""
        left, right = _u8(left), _u8(right)
        h, w = left.shape
        R, t = _f64(R).ravel(), _f64(t).ravel()
        c, sp, f = _calib(calib), _sgm(params), _filt(filt)
        if state is None:
            sd = sp_ = sv = None
            sw = sh = 0
        else:
            sd, sp_, sv = _f64(state[0]), _f64(state[1]), _u8(state[2])
            sh, sw = sd.shape
        out = dict(d=np.zeros((h, w)), p=np.zeros((h, w)), valid=np.zeros((h, w), np.uint8),
                   export_d=np.zeros((h, w), np.int32),
                   export_valid=np.zeros((h, w), np.uint8), diff=np.zeros((h, w)))
        dbg = None
        if debug:
            out.update(pred_d=np.zeros((h, w)), pred_p=np.zeros((h, w)),
                       pred_valid=np.zeros((h, w), np.uint8), lo=np.zeros((h, w), np.uint16),
                       hi=np.zeros((h, w), np.uint16), meas_d=np.zeros((h, w), np.int32),
                       meas_valid=np.zeros((h, w), np.uint8), mask=np.zeros((h, w), np.uint8))
            dbg = _OrDebug(*(out[k].ctypes.data for k in
                             ("pred_d", "pred_p", "pred_valid", "lo", "hi", "meas_d",
                              "meas_valid", "mask")), mask_tau)
        self._c(self.lib.or_step(_p(sd), _p(sp_), _p(sv), sw, sh, _p(left), _p(right), w, h,
                                 _p(R), _p(t), C.byref(c), C.byref(sp), C.byref(f),
                                 _p(out["d"]), _p(out["p"]), _p(out["valid"]),
                                 _p(out["export_d"]), _p(out["export_valid"]), _p(out["diff"]),
                                 C.byref(dbg) if dbg is not None else None))
        return out



class _OrBox(C.Structure):
    _fields_ = [("x0", C.c_int), ("y0", C.c_int), ("x1", C.c_int), ("y1", C.c_int),
                ("score", C.c_double)]


class _OrDetect(C.Structure):
    _fields_ = [("window_wh", C.c_void_p), ("n_windows", C.c_int), ("score_thresh", C.c_double),
                ("merge_stop_iou", C.c_double), ("min_box_area", C.c_longlong)]


def _port_detect_methods(cls):
    def _dc(self, cfg):
        wh = _wh(cfg)
        return wh, _OrDetect(wh.ctypes.data, len(cfg.window_sizes), cfg.score_thresh,
                             cfg.merge_stop_iou, cfg.min_box_area)

    def integral_image(self, m):
        m = _f64(m)
        h, w = m.shape
        sat = np.zeros((h + 1, w + 1))
        self.lib.or_integral_image(_p(m), w, h, _p(sat))
        return sat

    def candidates(self, diff, cfg, threads=1):
        diff = _f64(diff)
        h, w = diff.shape
        wh, dc = _dc(self, cfg)
        self.lib.or_candidates.restype = C.c_longlong
        cap = 1 << 16
        while True:
            out = (_OrBox * cap)()
            n = self.lib.or_candidates(_p(diff), w, h, C.byref(dc), out, C.c_longlong(cap))
            if n < 0:
                self._c(1)
            if n <= cap:
                return np.array([[b.x0, b.y0, b.x1, b.y1, b.score] for b in out[:n]],
                                dtype=np.float64).reshape(-1, 5)
            cap = n

    def greedy_merge(self, boxes, cfg):
        b = _boxes_arr(boxes)
        wh, dc = _dc(self, cfg)
        self._c(self.lib.or_detect_validate(C.byref(dc)))
        arr = (_OrBox * max(1, len(b)))(*[_OrBox(int(r[0]), int(r[1]), int(r[2]), int(r[3]), r[4])
                                         for r in b])
        self.lib.or_greedy_merge.restype = C.c_longlong
        n = self.lib.or_greedy_merge(arr, C.c_longlong(len(b)), C.byref(dc))
        return np.array([[x.x0, x.y0, x.x1, x.y1, x.score] for x in arr[:n]],
                        dtype=np.float64).reshape(-1, 5)

    def detect(self, diff, cfg, threads=1):
        return greedy_merge(self, candidates(self, diff, cfg), cfg)

    for f in (integral_image, candidates, greedy_merge, detect):
        setattr(cls, f.__name__, f)
    return cls


_port_detect_methods(Port)


def _port_count_outliers(self, d, valid, gt, abs_thresh=3.0, rel_thresh=0.05, strict=False):
    d, valid, gt = np.ascontiguousarray(d, np.int32), _u8(valid), _f64(gt)
    h, w = gt.shape
    ev, out = C.c_longlong(), C.c_longlong()
    self.lib.or_count_outliers(_p(d), _p(valid), _p(gt), w, h, C.c_double(abs_thresh),
                               C.c_double(rel_thresh), int(strict), C.byref(ev), C.byref(out))
    return ev.value, out.value


Port.count_outliers = _port_count_outliers


# ------------------------------------------------ noise calibration (row 4)
# Results of both checkers: dict(variance, mean, within_1px (fraction),
# samples_used, total, underflow, overflow, counts).
def _nbins(opts):
    import math
    return int(math.ceil((2.0 * opts.outlier_gate_px) / opts.bin_width))


def _opts3(opts):
    return np.array([opts.outlier_gate_px, opts.bin_width, opts.q_floor], np.float64)


def _ref_estimate(self, call, opts):
    nb = _nbins(opts)
    mom = np.zeros(3)
    ints = np.zeros(5, np.int64)
    counts = np.zeros(nb, np.int64)
    self._c(call(_p(mom), _p(ints), _p(counts), nb))
    return dict(variance=mom[0], mean=mom[1], within_1px=mom[2], samples_used=int(ints[0]),
                total=int(ints[1]), underflow=int(ints[2]), overflow=int(ints[3]), counts=counts)


def _ref_process_noise(self, gt, poses, calib, opts):
    gt = _f64(gt)
    n, h, w = gt.shape
    poses = None if poses is None else _f64(poses)
    c4 = np.array([calib.focal_px, calib.cx, calib.cy, calib.baseline_m])
    o3 = _opts3(opts)
    return _ref_estimate(self, lambda m, i, cn, nb: self.lib.ref_process_noise(
        n, w, h, _p(gt), _p(poses), _p(c4), calib.width, calib.height, calib.d_max,
        _p(o3), m, i, cn, nb), opts)


def _ref_measurement_noise(self, left, right, gt, params, opts, threads=1):
    left, right, gt = _u8(left), _u8(right), _f64(gt)
    n, h, w = gt.shape
    sp = np.array([params.p1, params.p2, params.paths, params.path_set, params.d_max], np.int32)
    o3 = _opts3(opts)
    return _ref_estimate(self, lambda m, i, cn, nb: self.lib.ref_measurement_noise(
        n, w, h, _p(left), _p(right), _p(gt), _p(sp), threads, _p(o3), m, i, cn, nb), opts)


def _ref_error_map(self, gt, poses, calib):
    gt, poses = _f64(gt), _f64(poses)
    n, h, w = gt.shape
    c4 = np.array([calib.focal_px, calib.cx, calib.cy, calib.baseline_m])
    acc = np.zeros((h, w))
    self._c(self.lib.ref_accumulate_error_map(n, w, h, _p(gt), _p(poses), _p(c4), calib.width,
                                              calib.height, calib.d_max, _p(acc)))
    return acc


def _ref_calib_report(self, path, left, right, gt, poses, calib, params, opts):
    """write_calib_report of the reference's own estimates, run in a separate
    process (oracle/report_driver.c): its iostreams crash inside Python."""
    import tempfile
    left, right, gt, poses = _u8(left), _u8(right), _f64(gt), _f64(poses)
    n, h, w = gt.shape
    hd = np.array([n, w, h, calib.width, calib.height, calib.d_max, params.p1, params.p2,
                   params.paths, params.path_set, params.d_max], np.int32)
    with tempfile.NamedTemporaryFile(suffix=".bin") as f:
        for a in (hd, np.array([calib.focal_px, calib.cx, calib.cy, calib.baseline_m]),
                  _opts3(opts), left, right, gt, poses):
            f.write(np.ascontiguousarray(a).tobytes())
        f.flush()
        r = subprocess.run([os.path.join(REF_DIR, "report_driver"), f.name, str(path)],
                           capture_output=True, text=True)
    if r.returncode == 1:
        raise ValueError(r.stderr.strip())
    if r.returncode != 0:
        raise RuntimeError(r.stderr.strip() or f"report_driver failed ({r.returncode})")


Reference.process_noise = _ref_process_noise
Reference.measurement_noise = _ref_measurement_noise
Reference.error_map = _ref_error_map
Reference.calib_report = _ref_calib_report


def _port_hist(self, es, uses, opts):
    """ErrorHistogram over the (e, use) maps in order (or_error_hist)."""
    nb = _nbins(opts)
    counts = np.zeros(nb, np.int64)
    tal = np.zeros(4, np.int64)
    sums = np.zeros(2)
    for e, u in zip(es, uses):
        e, u = _f64(e), _u8(u)
        self.lib.or_error_hist(_p(e), _p(u), C.c_size_t(e.size), C.c_double(-opts.outlier_gate_px),
                               C.c_double(opts.outlier_gate_px), C.c_double(opts.bin_width),
                               _p(counts), nb, _p(tal), _p(sums))
    gated = int(tal[3])
    total = gated + int(tal[0]) + int(tal[1])
    var = 0.0
    if gated >= 2:  # ErrorHistogram::variance, noise_calib.cpp:45-52
        n = float(gated)
        m = sums[0] / n
        var = max((sums[1] - n * m * m) / (n - 1.0), 0.0)
    return dict(variance=var, mean=sums[0] / gated if gated else 0.0,
                within_1px=int(tal[2]) / total if total else 0.0, samples_used=gated,
                total=total, underflow=int(tal[0]), overflow=int(tal[1]), counts=counts,
                sum=sums[0], sum_sq=sums[1])


def _port_warped_pairs(self, gt, poses, calib):
    """state_from_gt of frame k-1 warped by relative_motion(k-1, k)
    (noise_calib.cpp:71-78, 115-119) -> [(warped d, warped valid, gt k)]."""
    gt, poses = _f64(gt), _f64(poses)
    out = []
    for k in range(1, gt.shape[0]):
        R, t = self.relative_motion(poses[k - 1], poses[k])
        H = self.homography(R, t, calib)
        g = gt[k - 1]
        v = (g > 0.0).astype(np.uint8)
        d = np.where(v == 1, g, 0.0)
        wd, _, wv, _ = self.warp(d, np.zeros_like(d), v, H, calib.d_max)
        out.append((wd, wv, gt[k]))
    return out


def _port_process_noise(self, gt, poses, calib, opts):
    pairs = _port_warped_pairs(self, gt, poses, calib)
    r = _port_hist(self, [wd - g for wd, wv, g in pairs],
                   [(wv == 1) & (g > 0.0) for wd, wv, g in pairs], opts)
    if r["total"] == 0:
        raise RuntimeError("estimate_process_noise: no overlapping valid pixels")
    return r


def _port_measurement_noise(self, left, right, gt, params, opts):
    es, uses = [], []
    for k in range(gt.shape[0]):
        h, w = gt[k].shape
        lo = np.zeros((h, w), np.uint16)
        hi = np.full((h, w), params.d_max - 1, np.uint16)
        d, v = self.sgm_match(left[k], right[k], lo, hi, params)
        es.append(d.astype(np.float64) - gt[k])
        uses.append((v == 1) & (gt[k] > 0.0))
    r = _port_hist(self, es, uses, opts)
    if r["total"] == 0:
        raise RuntimeError("estimate_measurement_noise: no overlapping valid pixels")
    return r


def _port_error_map(self, gt, poses, calib):
    acc = np.zeros(_f64(gt).shape[1:])
    overlap = 0
    for wd, wv, g in _port_warped_pairs(self, gt, poses, calib):
        m = (wv == 1) & (g > 0.0)
        acc[m] += np.abs(wd[m] - g[m])  # per pixel in pair order, as the reference
        overlap += int(m.sum())
    if overlap == 0:
        raise RuntimeError("accumulate_error_map: no overlapping valid pixels")
    return acc


Port.process_noise = _port_process_noise
Port.measurement_noise = _port_measurement_noise
Port.error_map = _port_error_map


# ------------------------------------------------ export formats (row 2)
def quantize_disparity(disp):
    """write_disparity_png's quantisation (dataset.cpp:229-244), numpy
    restatement: d == 0 -> 0; v = std::lround(d * 256.0) (half away from
    zero; NaN/out of range -> LONG_MIN); 0 < v <= 65535 else the reference's
    std::invalid_argument at the first such pixel in raster order."""
    disp = _f64(disp)
    x = disp * 256.0
    t = np.trunc(x)
    with np.errstate(invalid="ignore"):
        t = t + np.where(np.abs(x - t) >= 0.5, np.copysign(1.0, x), 0.0)
        ok_range = (t >= -9.223372036854775808e18) & (t < 9.223372036854775808e18)
    v = np.where(ok_range, t, -9.223372036854775808e18)
    bad = (disp != 0.0) & ((v <= 0) | (v > 65535))
    if bad.any():
        i = int(np.flatnonzero(bad.ravel())[0])
        h, w = disp.shape
        raise ValueError(f"write_disparity_png: disparity {disp.ravel()[i]:f} not encodable at "
                         f"({i % w}, {i // w})")
    return np.where(disp == 0.0, 0, v).astype(np.uint16)


def quantize_disparity_map(d, valid):
    """write_disparity_png(const DisparityMap&) (dataset.cpp:246-254)."""
    return quantize_disparity(np.where(_u8(valid) != 0, np.asarray(d, np.float64), 0.0))


_port = None
_reference = None


def port() -> Port:
    global _port
    if _port is None:
        _port = Port()
    return _port


def reference() -> Reference:
    global _reference
    if _reference is None:
        _reference = Reference()
    return _reference
