"""aggregate_paths on the GPU vs the oracle on adversarial ragged volumes:
random narrow/wide/full windows, large window shifts between neighbours,
odd sizes, d_max not a multiple of 4, every path set, random P1/P2 — for all
three aggregation kernels (scanline groups, line groups, per-direction
scanline). Bit-exact."""
import numpy as np
import pytest

from paper_1809_07986_b200 import tsgm

pytestmark = pytest.mark.gpu


def ragged_ranges(rng, w, h, d_max, p_full=0.2, p_wide=0.05):
    lo = np.zeros((h, w), np.int64)
    hi = np.zeros((h, w), np.int64)
    kind = rng.random((h, w))
    centre = rng.integers(0, d_max, (h, w))
    # smooth-ish centres along rows for realistic small shifts
    centre = np.clip(np.cumsum(rng.integers(-1, 2, (h, w)), axis=1) + centre[:, :1], 0,
                     d_max - 1)
    half = rng.integers(0, 6, (h, w))
    lo[:] = np.clip(centre - half, 0, d_max - 1)
    hi[:] = np.clip(centre + half, 0, d_max - 1)
    full = kind < p_full
    lo[full], hi[full] = 0, d_max - 1
    wide = (kind >= p_full) & (kind < p_full + p_wide)
    a = rng.integers(0, d_max, (h, w))
    b = rng.integers(0, d_max, (h, w))
    lo[wide], hi[wide] = np.minimum(a, b)[wide], np.maximum(a, b)[wide]
    return lo.astype(np.uint16), hi.astype(np.uint16)


CASES = [
    # w, h, d_max, p_full
    (37, 23, 16, 0.2),
    (64, 40, 5, 0.5),
    (61, 29, 130, 0.3),
    (200, 75, 128, 0.21),
    (96, 33, 256, 0.1),
    (130, 41, 200, 0.4),
    (33, 64, 64, 0.9),
]


@pytest.mark.parametrize("kernel", ["groups32", "groups16", "groups8", "groups32h8", "groups32h16",
                                    "groups16h8", "groups32hlines", "groups8hlines", "groups32hlines8", "lines",
                                    "lines16h", "lines32h", "scanline",
                                    "lines@r0", "lines@r2", "lines32h@r0", "lines32h@r2",
                                    "groups32hlines@r0", "groups32hlines8@r0"])
@pytest.mark.parametrize("w,h,d_max,p_full", CASES)
def test_random_ragged_volumes(port, monkeypatch, kernel, w, h, d_max, p_full):
    """groupsN[hM]: the scanline-group kernel with N scanlines per warp (M for
    the horizontal lines) (batched throughput path); lines: the line-group kernel (single sequences,
    full-range frames); scanline: the per-direction fallback; @rN: TSGM_RLINE=N
    (line groups with the path state in shared memory / in registers)."""
    kernel, _, rl = kernel.partition("@r")
    if rl:  # register line groups: 0 = off, 1 = horizontal tasks (default), 2 = every direction
        monkeypatch.setenv("TSGM_RLINE", rl)
    if kernel == "scanline":
        monkeypatch.setenv("TSGM_FORCE_SCANLINE_AGG", "1")
    elif kernel.startswith("lines"):
        monkeypatch.setenv("TSGM_SCAN_KERNEL", "lines")
        if kernel != "lines":  # wider groups for the horizontal lines
            monkeypatch.setenv("TSGM_LINES_H", kernel[len("lines"):-1])
    else:
        monkeypatch.setenv("TSGM_SCAN_KERNEL", "groups")
        spw, _, spwh = kernel[len("groups"):].partition("h")
        if spwh.startswith("lines") and spwh != "lines":  # line-group width
            monkeypatch.setenv("TSGM_MIXED_GH", spwh[len("lines"):])
            spwh = "lines"
        monkeypatch.setenv("TSGM_SCAN_SPW", spw)
        if spwh:  # thinner warps for the horizontal lines
            monkeypatch.setenv("TSGM_SCAN_SPW_H", spwh)
    rng = np.random.default_rng(w * 1000 + h * 7 + d_max)
    lo, hi = ragged_ranges(rng, w, h, d_max, p_full)
    n = int((hi.astype(np.int64) - lo + 1).sum())
    cost = rng.integers(0, 25, n).astype(np.uint8)
    for paths, path_set in ((8, 0), (4, 0), (4, 1)):
        p1 = int(rng.integers(1, 12))
        p2 = p1 + int(rng.integers(0, 120))
        params = tsgm.SgmParams(p1, p2, paths, path_set, d_max)
        got = tsgm.aggregate_paths(cost, lo, hi, params)
        want = port.aggregate(cost, lo, hi, params)
        np.testing.assert_array_equal(got, want)


def test_full_size_realistic(port):
    """1242x375, D=128: 21% full-range windows, narrow ones 7-11 levels."""
    rng = np.random.default_rng(7)
    w, h, d = 1242, 375, 128
    lo, hi = ragged_ranges(rng, w, h, d, p_full=0.21, p_wide=0.0)
    n = int((hi.astype(np.int64) - lo + 1).sum())
    cost = rng.integers(0, 25, n).astype(np.uint8)
    params = tsgm.SgmParams(10, 120, 8, 0, d)
    np.testing.assert_array_equal(tsgm.aggregate_paths(cost, lo, hi, params),
                                  port.aggregate(cost, lo, hi, params))


def test_large_p2_falls_back_to_scanline(port):
    """P2 + 24 > 255 does not fit the u8 line state: the scanline kernel runs."""
    rng = np.random.default_rng(3)
    lo, hi = ragged_ranges(rng, 40, 20, 32)
    n = int((hi.astype(np.int64) - lo + 1).sum())
    cost = rng.integers(0, 25, n).astype(np.uint8)
    params = tsgm.SgmParams(10, 400, 8, 0, 32)
    np.testing.assert_array_equal(tsgm.aggregate_paths(cost, lo, hi, params),
                                  port.aggregate(cost, lo, hi, params))
