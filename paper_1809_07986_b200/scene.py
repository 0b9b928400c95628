"""Seeded synthetic stereo sequences for BASELINE.json configs 0-4.

Thin ctypes front-end over ``csrc/scene.c`` (``libtsgm_scene.so``). The same
frames feed the GPU path and the CPU reference/oracle. Input generation only —
not part of the hot path.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from ._build import lib_path

_lib = None


class _Cfg(C.Structure):
    _fields_ = [("width", C.c_int), ("height", C.c_int), ("d_max", C.c_int),
                ("focal", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("baseline", C.c_double), ("frames", C.c_int), ("seed", C.c_uint64),
                ("n_static", C.c_int), ("n_movers", C.c_int), ("fwd_m", C.c_double),
                ("yaw_deg", C.c_double), ("mover_speed_min", C.c_double),
                ("mover_speed_max", C.c_double), ("gain_jitter", C.c_double),
                ("mover_max_frac", C.c_double), ("noise_sigma", C.c_double)]


def _load():
    global _lib
    if _lib is None:
        path = lib_path("libtsgm_scene.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run __graft_entry__.build()")
        _lib = C.CDLL(path)
    return _lib


@dataclass
class SceneConfig:
    width: int = 1242
    height: int = 375
    d_max: int = 128
    focal: float = 720.0
    cx: float = 621.0
    cy: float = 187.5
    baseline: float = 0.54
    frames: int = 8
    seed: int = 0
    n_static: int = 6
    n_movers: int = 0
    fwd_m: float = 0.8
    yaw_deg: float = 0.5
    mover_speed_min: float = 0.5
    mover_speed_max: float = 1.5
    gain_jitter: float = 0.0
    mover_max_frac: float = 0.0
    noise_sigma: float = 2.0

    @classmethod
    def baseline_config(cls, config: int, **overrides) -> "SceneConfig":
        """BASELINE.json ``configs[config]`` defaults (synthetic KITTI stand-in)."""
        c = _Cfg()
        _load().tsgm_scene_default(C.byref(c), int(config))
        kw = {f: getattr(c, f) for f, _ in _Cfg._fields_}
        kw.update(overrides)
        return cls(**kw)

    def _c(self) -> _Cfg:
        return _Cfg(*(getattr(self, f) for f, _ in _Cfg._fields_))


def render(cfg: SceneConfig, frame_begin: int = 0, frame_end: int | None = None,
           threads: int | None = None, gt: bool = False, out_left=None, out_right=None):
    """Render frames [frame_begin, frame_end). Returns (left, right, poses, gt):
    left/right u8 [F, H, W], poses f64 [frames, 3, 4] (camera-to-world), gt f32
    [F, H, W] or None. ``out_left``/``out_right`` may be preallocated (e.g.
    pinned) contiguous u8 buffers of the right size."""
    if frame_end is None:
        frame_end = cfg.frames
    n = frame_end - frame_begin
    shape = (n, cfg.height, cfg.width)
    left = np.empty(shape, np.uint8) if out_left is None else out_left
    right = np.empty(shape, np.uint8) if out_right is None else out_right
    gtd = np.empty(shape, np.float32) if gt else None
    poses = np.empty((cfg.frames, 3, 4), np.float64)
    threads = threads or os.cpu_count() or 1
    c = cfg._c()
    rc = _load().tsgm_scene_render(
        C.byref(c), frame_begin, frame_end, C.c_void_p(left.ctypes.data),
        C.c_void_p(right.ctypes.data), C.c_void_p(gtd.ctypes.data) if gt else None,
        C.c_void_p(poses.ctypes.data), int(threads))
    if rc != 0:
        raise ValueError("tsgm_scene_render: invalid configuration")
    return left, right, poses, gtd
