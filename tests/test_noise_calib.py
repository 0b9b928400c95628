"""Noise calibration (reference src/noise_calib.cpp:102-217)
for the oracle (port, CPU) and the product (gpu) against the reference's own
outputs (tests/golden/noise_calib.npz, tests/golden/make_golden_noise.py) and
the KATs of the reference's tests/test_noise_calib.cpp.

Exactness: histogram counts, tallies and the accumulated error map are
bit-exact; the port also reproduces the reference's raster-order FP64 moments
bit for bit, the GPU reduces them in a fixed tree order (deterministic), so its
variance and mean are checked to 1e-9 relative (the variance
(sum_sq - n m^2) / (n - 1) amplifies the sums' last-bit differences)."""
import numpy as np
import pytest

from oracle import oracle as O
from tests.backends import backend_fixture, golden

backend = backend_fixture()

CASES = ["a", "b"]


def _case(name):
    g = golden("noise_calib")
    c = g[f"{name}_calib"]
    calib = O.Calib(c[0], c[1], c[2], c[3], int(c[4]), int(c[5]), int(c[6]))
    o = g[f"{name}_opts"]
    opts = O.CalibOpts(o[0], o[1], o[2])
    s = g[f"{name}_sgm"]
    sgm = O.SgmParams(*(int(v) for v in s))
    return g, calib, opts, sgm


def _check(backend, got, g, key):
    mom, ints, counts = g[f"{key}_moments"], g[f"{key}_ints"], g[f"{key}_counts"]
    assert [got["samples_used"], got["total"], got["underflow"], got["overflow"]] == list(ints)
    np.testing.assert_array_equal(got["counts"], counts)
    rtol = 0.0 if backend.kind == "port" else 1e-9
    np.testing.assert_allclose([got["variance"], got["mean"]], mom[:2], rtol=rtol, atol=0.0)
    assert got["within_1px"] == mom[2]


@pytest.mark.parametrize("name", CASES)
def test_process_noise_golden(backend, name):
    g, calib, opts, _ = _case(name)
    _check(backend, backend.process_noise(g[f"{name}_gt"], g[f"{name}_poses"], calib, opts), g,
           f"{name}_process")


@pytest.mark.parametrize("name", CASES)
def test_measurement_noise_golden(backend, name):
    g, _, opts, sgm = _case(name)
    got = backend.measurement_noise(g[f"{name}_left"], g[f"{name}_right"], g[f"{name}_gt"], sgm,
                                    opts)
    _check(backend, got, g, f"{name}_meas")


@pytest.mark.parametrize("name", CASES)
def test_error_map_golden(backend, name):
    g, calib, _, _ = _case(name)
    np.testing.assert_array_equal(backend.error_map(g[f"{name}_gt"], g[f"{name}_poses"], calib),
                                  g[f"{name}_error_map"])


def test_reference_reproduces_golden(reference):
    """The fixture generator is the reference itself (skipped without it)."""
    g, calib, opts, sgm = _case("a")
    _check(reference, reference.process_noise(g["a_gt"], g["a_poses"], calib, opts), g,
           "a_process")


# ---- KATs of the reference's tests/test_noise_calib.cpp, on the port's
# histogram restatement (or_error_hist) ----
def _hist(port, samples, lo=-10.0, hi=10.0, bw=0.25):
    import ctypes as C
    e = np.asarray(samples, np.float64)
    u = np.ones(e.size, np.uint8)
    nb = int(np.ceil((hi - lo) / bw))
    counts = np.zeros(nb, np.int64)
    tal = np.zeros(4, np.int64)
    sums = np.zeros(2)
    p = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    port.lib.or_error_hist(p(e), p(u), C.c_size_t(e.size), C.c_double(lo), C.c_double(hi),
                           C.c_double(bw), p(counts), nb, p(tal), p(sums))
    return counts, tal, sums


def test_histogram_bins(port):
    """test_noise_calib.cpp:43-57: samples land in the expected bins."""
    counts, tal, _ = _hist(port, [0.0, 0.1, -10.0, 9.99])
    assert counts[40] == 2 and counts[0] == 1 and counts[79] == 1
    assert tal[3] + tal[0] + tal[1] == 4 and tal[0] == 0 and tal[1] == 0


def test_histogram_gate(port):
    """test_noise_calib.cpp:58-70: out-of-gate samples count but stay out of
    the moments."""
    counts, tal, sums = _hist(port, [1.0, -1.0, 50.0, -12.0])
    under, over, within, gated = (int(v) for v in tal)
    assert gated + under + over == 4 and gated == 2 and over == 1 and under == 1
    assert sums[0] / gated == pytest.approx(0.0)
    n = float(gated)
    m = sums[0] / n
    assert (sums[1] - n * m * m) / (n - 1.0) == pytest.approx(2.0)
    assert within / 4 == pytest.approx(0.5)


def test_histogram_order(port):
    """test_noise_calib.cpp:71-85: insertion order does not matter."""
    rng = np.random.default_rng(91)
    s = rng.normal(0.3, 1.7, 500)
    a = _hist(port, s)
    b = _hist(port, rng.permutation(s))
    np.testing.assert_array_equal(a[0], b[0])
    assert a[2][0] == pytest.approx(b[2][0], rel=1e-12, abs=1e-12)


def test_calib_options_validate():
    """CalibOptions::validate / ErrorHistogram layout (noise_calib.cpp:9-14,
    60-67) through the C-ABI (host-only call)."""
    from paper_1809_07986_b200 import tsgm
    assert tsgm.CalibOptions().validate() == 80
    assert tsgm.CalibOptions(4.0, 0.5, 0.05).validate() == 16
    for bad in (tsgm.CalibOptions(0.0), tsgm.CalibOptions(5.0, 0.0), tsgm.CalibOptions(5.0, 6.0),
                tsgm.CalibOptions(5.0, 0.5, -1.0)):
        with pytest.raises(ValueError, match="CalibOptions"):
            bad.validate()


def test_frame_checks_before_the_device():
    """The reference's input errors (noise_calib.cpp:80-89, 104-114, 133-136)
    are raised by the host mirror before any device work."""
    from paper_1809_07986_b200 import tsgm
    f = tsgm.SequenceFrame(0, None, None, np.zeros((3, 4)), np.ones((8, 8)))
    calib = tsgm.StereoCalib(100.0, 3.5, 3.5, 1.0, 8, 8, 16)
    with pytest.raises(ValueError, match="need at least 2 frames"):
        tsgm.estimate_process_noise([f], calib)
    g = tsgm.SequenceFrame(1, None, None, np.zeros((3, 4)), None)
    with pytest.raises(ValueError, match="frame 1 has no GT disparity"):
        tsgm.estimate_process_noise([f, g], calib)
    g = tsgm.SequenceFrame(1, None, None, None, np.ones((8, 8)))
    with pytest.raises(ValueError, match="frame 1 has no pose"):
        tsgm.accumulate_error_map([f, g], calib)
    with pytest.raises(ValueError, match="need at least 1 frame"):
        tsgm.estimate_measurement_noise([], tsgm.SgmParams(d_max=16))


def test_report_text(tmp_path):
    """write_calib_report (noise_calib.cpp:184-217): the host mirror writes the
    reference's text from the same estimate values."""
    from paper_1809_07986_b200 import tsgm
    g = golden("noise_calib")
    want = bytes(g["a_report"]).decode()
    # rebuild the estimates' reported fields from the reference report itself
    lines = want.splitlines()
    rows = [ln.split() for ln in lines if ln.startswith("# ") and len(ln.split()) == 5
            and ln.split()[1] not in ("bin_lo", "-inf", "q") and ln.split()[2] != "+inf"]
    pc = np.array([int(r[3]) for r in rows], np.int64)
    mc = np.array([int(r[4]) for r in rows], np.int64)
    under = [ln.split() for ln in lines if ln.startswith("# -inf")][0]
    over = [ln.split() for ln in lines if "+inf" in ln][0]

    def est(var_line, counts, u, o):
        t = var_line.split()
        var, n, pct = float(t[4]), int(t[7]), float(t[9].rstrip("%"))
        total = int(counts.sum()) + u + o
        h = tsgm.ErrorHistogram(-10.0, 10.0, 0.25, counts, u, o, n, 0)
        # n_within_1 that prints the same percentage
        h.n_within_1 = int(round(pct / 100.0 * total))
        return tsgm.NoiseEstimate(var, h, n)

    pe = est(lines[1], pc, int(under[3]), int(over[3]))
    me = est(lines[2], mc, int(under[4]), int(over[4]))
    path = tmp_path / "report.txt"
    tsgm.write_calib_report(str(path), pe, me, tsgm.CalibOptions(10.0, 0.25, 0.1))
    assert path.read_text() == want


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_gpu_report_matches_reference(name, tmp_path):
    """Report written from the GPU estimates == the reference's report."""
    from paper_1809_07986_b200 import tsgm
    from paper_1809_07986_b200.testing import GpuBackend
    g, calib, opts, sgm = _case(name)
    fr = GpuBackend._frames(g[f"{name}_gt"], g[f"{name}_poses"], g[f"{name}_left"],
                            g[f"{name}_right"])
    o = tsgm.CalibOptions(opts.outlier_gate_px, opts.bin_width, opts.q_floor)
    pe = tsgm.estimate_process_noise(fr, calib, o)
    me = tsgm.estimate_measurement_noise(fr, sgm, 1, o)
    path = tmp_path / "report.txt"
    tsgm.write_calib_report(str(path), pe, me, o)
    assert path.read_text() == bytes(g[f"{name}_report"]).decode()

