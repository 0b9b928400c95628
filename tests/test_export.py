"""Export formats (reference src/dataset.cpp:220-269):
the KITTI 16-bit disparity PNG quantisation and boxes.txt, against the
reference's own outputs (tests/golden/export.npz, made by
tests/golden/make_golden_export.py from dataset.cpp compiled in place with a
recording stand-in for its libpng writer). The numpy restatement (oracle) and
the host writers run on the CPU; the GPU quantisation and the PNG files are
gpu-marked. Bit-exact: the 16-bit samples, the error messages, the text."""
import zlib

import numpy as np
import pytest

from oracle import oracle as O
from tests.backends import golden

F64 = ["f64_0", "f64_1", "f64_2"]
MAPS = ["map_0", "map_1"]
BAD = ["bad_0", "bad_1", "bad_2", "bad_3"]


@pytest.mark.parametrize("case", F64)
def test_oracle_quantize_f64(case):
    g = golden("export")
    np.testing.assert_array_equal(O.quantize_disparity(g[f"{case}__disp"]), g[f"{case}__raw"])


@pytest.mark.parametrize("case", MAPS)
def test_oracle_quantize_map(case):
    g = golden("export")
    np.testing.assert_array_equal(O.quantize_disparity_map(g[f"{case}__d"], g[f"{case}__valid"]),
                                  g[f"{case}__raw"])


@pytest.mark.parametrize("case", BAD)
def test_oracle_not_encodable(case):
    g = golden("export")
    with pytest.raises(ValueError) as e:
        O.quantize_disparity(g[f"{case}__disp"])
    assert str(e.value) == bytes(g[f"{case}__msg"]).decode()


def _per_frame(g):
    flat, counts = g["boxes__flat"], g["boxes__counts"]
    out, k = [], 0
    for n in counts:
        out.append(flat[k:k + n])
        k += n
    return out


def test_write_boxes_text(tmp_path):
    """write_boxes' text, byte for byte (host writer in the product library)."""
    from paper_1809_07986_b200 import tsgm
    g = golden("export")
    path = tmp_path / "boxes.txt"
    tsgm.write_boxes(path, _per_frame(g))
    assert path.read_bytes() == bytes(g["boxes__text"])


def _png(raw, filters):
    """A 16-bit grayscale PNG with the given per-row filter types (encoder for
    the decoder's test)."""
    import struct
    h, w = raw.shape
    b = np.zeros((h, 2 * w), np.int32)
    b[:, 0::2], b[:, 1::2] = raw >> 8, raw & 0xff
    rows, prev = [], np.zeros(2 * w, np.int32)
    for y in range(h):
        ft, cur = filters[y % len(filters)], b[y]
        a = np.concatenate([[0, 0], cur[:-2]])
        c = np.concatenate([[0, 0], prev[:-2]])
        if ft == 0:
            f = cur
        elif ft == 1:
            f = cur - a
        elif ft == 2:
            f = cur - prev
        elif ft == 3:
            f = cur - (a + prev) // 2
        else:
            p = a + prev - c
            pa, pb, pc = np.abs(p - a), np.abs(p - prev), np.abs(p - c)
            f = cur - np.where((pa <= pb) & (pa <= pc), a, np.where(pb <= pc, prev, c))
        rows.append(bytes([ft]) + bytes((f & 0xff).astype(np.uint8)))
        prev = cur

    def chunk(t, d):
        return struct.pack(">I", len(d)) + t + d + struct.pack(">I", zlib.crc32(t + d) & 0xffffffff)
    return (b"\x89PNG\r\n\x1a\n" + chunk(b"IHDR", struct.pack(">IIBBBBB", w, h, 16, 0, 0, 0, 0)) +
            chunk(b"IDAT", zlib.compress(b"".join(rows))) + chunk(b"IEND", b""))


def test_png_reader_all_filters(tmp_path):
    """read_png16 (read_disparity_png's decode) on every PNG filter type."""
    from paper_1809_07986_b200 import tsgm
    raw = golden("export")["f64_1__raw"]
    path = tmp_path / "f.png"
    path.write_bytes(_png(raw, [0, 1, 2, 3, 4]))
    np.testing.assert_array_equal(tsgm.read_png16(path), raw)
    np.testing.assert_array_equal(tsgm.read_disparity_png(path), raw / 256.0)


# ---- the product on the GPU ----
@pytest.mark.gpu
@pytest.mark.parametrize("case", F64 + MAPS)
def test_gpu_quantize_and_png(case, tmp_path):
    from paper_1809_07986_b200 import tsgm
    g = golden("export")
    arg = g[f"{case}__disp"] if case.startswith("f64") else (g[f"{case}__d"], g[f"{case}__valid"])
    np.testing.assert_array_equal(tsgm.quantize_disparity(arg), g[f"{case}__raw"])
    path = tmp_path / "d.png"
    tsgm.write_disparity_png(path, arg)
    np.testing.assert_array_equal(tsgm.read_png16(path), g[f"{case}__raw"])


@pytest.mark.gpu
@pytest.mark.parametrize("case", BAD)
def test_gpu_not_encodable(case, tmp_path):
    from paper_1809_07986_b200 import tsgm
    g = golden("export")
    with pytest.raises(ValueError) as e:
        tsgm.write_disparity_png(tmp_path / "e.png", g[f"{case}__disp"])
    assert str(e.value) == bytes(g[f"{case}__msg"]).decode()
    assert not (tmp_path / "e.png").exists()


@pytest.mark.gpu
def test_gpu_engine_export_png(tmp_path):
    """tsgm_main's per-frame export (tsgm_main.cpp:157) from the device-resident
    export map == write_disparity_png of the fetched map."""
    from paper_1809_07986_b200 import tsgm
    from paper_1809_07986_b200.scene import SceneConfig, render
    cfg = SceneConfig.baseline_config(1, width=320, height=120, focal=200.0, cx=159.5, cy=59.5,
                                      d_max=64, seed=5, n_movers=2, frames=3)
    L, R, P, _ = render(cfg)
    calib = tsgm.StereoCalib(cfg.focal, cfg.cx, cfg.cy, cfg.baseline, cfg.width, cfg.height,
                             cfg.d_max)
    with tsgm.Engine(tsgm.EngineConfig(calib, tsgm.SgmParams(10, 120, 8, 0, 64),
                                       tsgm.FilterConfig(range_use_stddev=True,
                                                         range_stddev_gain=3.0),
                                       max_slots=2)) as eng:
        for k in range(3):
            mot = (np.eye(3), np.zeros(3)) if k == 0 else tsgm.relative_motion(P[k - 1], P[k])
            eng.step([1], [L[k]], [R[k]], [mot])
        eng.write_export_png(1, tmp_path / "e.png")
        eng.write_export_pngs([1, 0], [tmp_path / "b1.png", tmp_path / "b0.png"])
        want = O.quantize_disparity_map(eng.fetch(1, "export_d"), eng.fetch(1, "export_valid"))
    got = tsgm.read_png16(tmp_path / "e.png")
    assert got.any()
    np.testing.assert_array_equal(got, want)
    np.testing.assert_array_equal(tsgm.read_png16(tmp_path / "b1.png"), want)
    assert not tsgm.read_png16(tmp_path / "b0.png").any()  # slot 0 never stepped: all invalid


def test_png_reader_rejects(tmp_path):
    """read_disparity_png's errors (image_io.cpp:25-33, 180-182): a missing
    file, a non-PNG, an 8-bit PNG."""
    import struct
    from paper_1809_07986_b200 import tsgm
    with pytest.raises(RuntimeError, match="cannot open file"):
        tsgm.read_disparity_png(tmp_path / "missing.png")
    (tmp_path / "x.png").write_bytes(b"P5\n2 2\n255\n\x00\x00\x00\x00")
    with pytest.raises(RuntimeError):
        tsgm.read_disparity_png(tmp_path / "x.png")

    def chunk(t, d):
        return struct.pack(">I", len(d)) + t + d + struct.pack(">I", zlib.crc32(t + d) & 0xffffffff)
    png8 = (b"\x89PNG\r\n\x1a\n" + chunk(b"IHDR", struct.pack(">IIBBBBB", 2, 2, 8, 0, 0, 0, 0)) +
            chunk(b"IDAT", zlib.compress(b"\x00\x01\x02\x00\x03\x04")) + chunk(b"IEND", b""))
    (tmp_path / "g8.png").write_bytes(png8)
    with pytest.raises(RuntimeError, match="expected 16-bit single-channel PNG"):
        tsgm.read_disparity_png(tmp_path / "g8.png")


def test_png_reader_checks_crc(tmp_path):
    """A chunk whose CRC-32 does not match fails like libpng's read."""
    from paper_1809_07986_b200 import tsgm
    raw = golden("export")["f64_1__raw"]
    data = bytearray(_png(raw, [0]))
    data[33 + 8] ^= 0x01  # first byte of the IDAT data: its CRC no longer matches
    (tmp_path / "c.png").write_bytes(bytes(data))
    with pytest.raises(RuntimeError, match="PNG decode error"):
        tsgm.read_disparity_png(tmp_path / "c.png")
    with pytest.raises(RuntimeError, match="PNG decode error"):
        tsgm.read_png16(tmp_path / "c.png")
