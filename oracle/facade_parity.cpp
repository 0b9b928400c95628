// TEST INFRASTRUCTURE ONLY. Drop-in check of the C++ facade: the same frames
// go through the reference's tsgm::step (compiled in place from
// /root/reference/proj/src) and through tsgm::gpu::step (include/tsgm_gpu.hpp
// over libtsgm_b200.so). Every StepResult field must be identical, and the
// facade must throw the reference's exception types. Built by
// `make -C oracle facade` into oracle/_ref/facade_parity; run on the GPU box by
// tests/test_gpu_facade.py. Exit 0 = parity.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <random>
#include <stdexcept>

#include "tsgm/dataset.hpp"
#include "tsgm/noise_calib.hpp"
#include "tsgm/temporal_filter.hpp"
#include "tsgm_gpu.hpp"
#include "tsgm_scene.h"

using namespace tsgm;

static int fails = 0;
#define EXPECT(c, msg)                                   \
    do {                                                 \
        if (!(c)) {                                      \
            std::fprintf(stderr, "FAIL: %s\n", msg);     \
            ++fails;                                     \
        }                                                \
    } while (0)

static RigidMotion yaw(double a) {
    RigidMotion m;
    m.rotation(0, 0) = std::cos(a);
    m.rotation(0, 2) = std::sin(a);
    m.rotation(2, 0) = -std::sin(a);
    m.rotation(2, 2) = std::cos(a);
    m.translation(2) = -0.3;
    return m;
}

int main() {
    tsgm_scene_cfg sc;
    tsgm_scene_default(&sc, 1);
    sc.width = 320;
    sc.height = 120;
    sc.focal = 200.0;
    sc.cx = 159.5;
    sc.cy = 59.5;
    sc.d_max = 64;
    sc.frames = 6;
    sc.seed = 11;
    const int w = sc.width, h = sc.height, F = sc.frames;
    std::vector<uint8_t> L(static_cast<size_t>(w) * h * F), R(L.size());
    std::vector<double> poses(12 * F);
    if (tsgm_scene_render(&sc, 0, F, L.data(), R.data(), nullptr, poses.data(), 4) != 0) return 2;

    StereoCalib calib;
    calib.focal_px = sc.focal;
    calib.cx = sc.cx;
    calib.cy = sc.cy;
    calib.baseline_m = sc.baseline;
    calib.width = w;
    calib.height = h;
    calib.d_max = sc.d_max;
    SgmParams params;
    params.p1 = 10;
    params.p2 = 120;
    params.d_max = sc.d_max;
    FilterConfig cfg;
    cfg.range_use_stddev = true;
    cfg.range_stddev_gain = 3.0;

    DisparityState s_ref, s_gpu;
    for (int k = 0; k < F; ++k) {
        GrayImage left(w, h), right(w, h);
        std::copy(L.begin() + static_cast<long>(k) * w * h, L.begin() + static_cast<long>(k + 1) * w * h, left.data());
        std::copy(R.begin() + static_cast<long>(k) * w * h, R.begin() + static_cast<long>(k + 1) * w * h, right.data());
        RigidMotion m;
        if (k > 0) {
            Pose a, b;
            for (int i = 0; i < 12; ++i) {
                a(i / 4, i % 4) = poses[12 * (k - 1) + i];
                b(i / 4, i % 4) = poses[12 * k + i];
            }
            m = relative_motion(a, b);
        }
        const StepResult ref = tsgm::step(s_ref, left, right, m, calib, params, cfg);
        const StepResult gpu = tsgm::gpu::step(s_gpu, left, right, m, calib, params, cfg);
        EXPECT(ref.state.valid == gpu.state.valid, "state.valid");
        EXPECT(ref.state.d == gpu.state.d, "state.d");
        EXPECT(ref.state.p == gpu.state.p, "state.p");
        EXPECT(ref.export_map == gpu.export_map, "export_map");
        EXPECT(ref.diff == gpu.diff, "diff");
        // StepResult::timings filled like the reference's (temporal_filter.cpp:209-221)
        EXPECT(gpu.timings.predict_s > 0 && gpu.timings.ranges_s > 0 &&
                   gpu.timings.sgm.census_s > 0 && gpu.timings.sgm.cost_s > 0 &&
                   gpu.timings.sgm.aggregate_s > 0 && gpu.timings.sgm.wta_s > 0 &&
                   gpu.timings.correct_s > 0,
               "StepResult::timings");
        s_ref = ref.state;
        s_gpu = gpu.state;
        // sub-stage facades on the same frame
        const DisparityState pr = tsgm::predict(s_ref, yaw(0.01), calib, cfg);
        const DisparityState pg = tsgm::gpu::predict(s_gpu, yaw(0.01), calib, cfg);
        EXPECT(pr.d == pg.d && pr.p == pg.p && pr.valid == pg.valid, "predict");
        const SearchRangeMap rr = derive_search_ranges(pr, calib, cfg);
        const SearchRangeMap rg = tsgm::gpu::derive_search_ranges(pg, calib, cfg);
        EXPECT(rr.lo == rg.lo && rr.hi == rg.hi, "derive_search_ranges");
        const DisparityMap mr = sgm_match(left, right, rr, params);
        SgmStageTimings st;
        const DisparityMap mg = tsgm::gpu::sgm_match(left, right, rg, params, 1, &st);
        EXPECT(mr == mg, "sgm_match");
        EXPECT(st.census_s > 0 && st.cost_s > 0 && st.aggregate_s > 0 && st.wta_s > 0,
               "sgm_match timings");
        EXPECT(median_refine(mr) == tsgm::gpu::median_refine(mg), "median_refine");
        const DisparityState cr = correct(pr, mr, cfg);
        const DisparityState cg = tsgm::gpu::correct(pg, mg, cfg);
        EXPECT(cr.d == cg.d && cr.p == cg.p && cr.valid == cg.valid, "correct");
        EXPECT(census_transform(left).sig == tsgm::gpu::census_transform(left).sig, "census");
    }
    // error behaviour (temporal_filter.cpp:198-206)
    try {
        SgmParams bad = params;
        bad.d_max = 32;
        tsgm::gpu::step(DisparityState(), GrayImage(w, h), GrayImage(w, h), RigidMotion{}, calib,
                        bad, cfg);
        EXPECT(false, "d_max mismatch did not throw");
    } catch (const std::invalid_argument&) {
    }
    try {
        tsgm::gpu::step(DisparityState(), GrayImage(w, h), GrayImage(w - 1, h), RigidMotion{},
                        calib, params, cfg);
        EXPECT(false, "size mismatch did not throw");
    } catch (const std::invalid_argument&) {
    }
    // Engine::step checks image sizes before the C-ABI reads raw pointers
    {
        tsgm::gpu::Engine eng(calib, params, cfg, 1);
        GrayImage a(w, h), b(w - 1, h), c(w - 1, h);
        try {
            eng.step({0}, {&a}, {&b}, {RigidMotion{}});
            EXPECT(false, "Engine::step left/right mismatch did not throw");
        } catch (const std::invalid_argument&) {
        }
        try {
            eng.step({0}, {&b}, {&c}, {RigidMotion{}});
            EXPECT(false, "Engine::step wrong size did not throw");
        } catch (const std::invalid_argument&) {
        }
        try {
            eng.step({0}, {&a}, {&a, &a}, {RigidMotion{}});
            EXPECT(false, "Engine::step length mismatch did not throw");
        } catch (const std::invalid_argument&) {
        }
    }
    // batched engine == per-call facade
    {
        tsgm::gpu::Engine eng(calib, params, cfg, 2, 0, 3.0, TSGM_STAGE_TIMINGS);
        DisparityState s;
        for (int k = 0; k < 3; ++k) {
            GrayImage left(w, h), right(w, h);
            std::copy(L.begin() + static_cast<long>(k) * w * h, L.begin() + static_cast<long>(k + 1) * w * h, left.data());
            std::copy(R.begin() + static_cast<long>(k) * w * h, R.begin() + static_cast<long>(k + 1) * w * h, right.data());
            const StepResult one = tsgm::gpu::step(s, left, right, RigidMotion{}, calib, params, cfg);
            eng.step({1}, {&left}, {&right}, {RigidMotion{}});
            const StepResult batched = eng.result(1);
            EXPECT(one.state.d == batched.state.d && one.export_map == batched.export_map,
                   "Engine vs step");
            EXPECT(batched.timings.sgm.aggregate_s > 0 && batched.timings.correct_s > 0,
                   "Engine timings");
            s = one.state;
        }
    }
    // box detector (motion_detect.hpp): reference vs facade on the step's diff
    {
        std::mt19937 rng(5);
        Image<double> diff(w, h, 0.0);
        std::uniform_int_distribution<int> bx(0, w - 60), by(h / 3, h - 40);
        std::uniform_real_distribution<double> val(1.0, 8.0);
        for (int k = 0; k < 5; ++k) {
            const int x0 = bx(rng), y0 = by(rng);
            const double v = val(rng);
            for (int y = y0; y < std::min(h, y0 + 35); ++y)
                for (int x = x0; x < x0 + 55; ++x) diff(x, y) = v + 0.05 * ((x + 2 * y) % 7);
        }
        DetectConfig dc;
        EXPECT(integral_image(diff).sum == tsgm::gpu::integral_image(diff).sum, "integral_image");
        const auto cr = detect_candidate_windows(diff, dc, 4);
        EXPECT(cr == tsgm::gpu::detect_candidate_windows(diff, dc), "detect_candidate_windows");
        EXPECT(greedy_merge(cr, dc) == tsgm::gpu::greedy_merge(cr, dc), "greedy_merge");
        const auto dr = detect_moving_objects(diff, dc);
        EXPECT(!dr.empty() && dr == tsgm::gpu::detect_moving_objects(diff, dc),
               "detect_moving_objects");
        try {
            DetectConfig bad;
            bad.merge_stop_iou = 1.0;
            tsgm::gpu::detect_moving_objects(diff, bad);
            EXPECT(false, "invalid DetectConfig did not throw");
        } catch (const std::invalid_argument&) {
        }
        // batched engine: detection on the slot's own diff map
        tsgm::gpu::Engine eng(calib, params, cfg, 1);
        GrayImage left(w, h), right(w, h);
        std::copy(L.begin(), L.begin() + static_cast<long>(w) * h, left.data());
        std::copy(R.begin(), R.begin() + static_cast<long>(w) * h, right.data());
        eng.step({0}, {&left}, {&right}, {RigidMotion{}});
        eng.step({0}, {&left}, {&right}, {yaw(0.01)});
        DetectConfig loose;
        loose.score_thresh = 0.5;
        const auto got = eng.detect({0}, loose);
        EXPECT(got.size() == 1 && got[0] == detect_moving_objects(eng.result(0).diff, loose),
               "Engine::detect");
    }
    {  // noise calibration (noise_calib.hpp:57-80) on the same frames
        std::vector<double> ps(12 * F);
        std::vector<float> gf(static_cast<size_t>(w) * h * F);
        if (tsgm_scene_render(&sc, 0, F, L.data(), R.data(), gf.data(), ps.data(), 4) != 0) return 2;
        std::vector<SequenceFrame> frames(static_cast<size_t>(F));
        for (int k = 0; k < F; ++k) {
            SequenceFrame& f = frames[static_cast<size_t>(k)];
            f.index = k;
            f.left = GrayImage(w, h);
            f.right = GrayImage(w, h);
            std::copy(L.begin() + static_cast<long>(k) * w * h, L.begin() + static_cast<long>(k + 1) * w * h,
                      f.left.data());
            std::copy(R.begin() + static_cast<long>(k) * w * h, R.begin() + static_cast<long>(k + 1) * w * h,
                      f.right.data());
            Image<double> g(w, h);
            for (int i = 0; i < w * h; ++i) g.data()[i] = gf[static_cast<size_t>(k) * w * h + i];
            f.gt_disp = g;
            Pose p;
            for (int i = 0; i < 12; ++i) p(i / 4, i % 4) = ps[12 * k + i];
            f.pose = p;
        }
        auto same_est = [](const NoiseEstimate& a, const NoiseEstimate& b) {
            const auto rel = [](double x, double y) {
                return std::abs(x - y) <= 1e-9 * std::max(std::abs(y), 1e-300);
            };
            return a.samples_used == b.samples_used && a.hist.counts == b.hist.counts &&
                   a.hist.total() == b.hist.total() && a.hist.underflow == b.hist.underflow &&
                   a.hist.overflow == b.hist.overflow &&
                   a.hist.fraction_within_1px() == b.hist.fraction_within_1px() &&
                   rel(a.variance, b.variance) && rel(a.hist.variance(), b.hist.variance()) &&
                   rel(a.hist.mean(), b.hist.mean());
        };
        EXPECT(same_est(tsgm::gpu::estimate_process_noise(frames, calib),
                        estimate_process_noise(frames, calib)),
               "estimate_process_noise");
        EXPECT(same_est(tsgm::gpu::estimate_measurement_noise(frames, params),
                        estimate_measurement_noise(frames, params)),
               "estimate_measurement_noise");
        const Image<double> em = accumulate_error_map(frames, calib);
        const Image<double> eg = tsgm::gpu::accumulate_error_map(frames, calib);
        EXPECT(std::equal(em.data(), em.data() + em.pixel_count(), eg.data()),
               "accumulate_error_map");
        try {
            tsgm::gpu::estimate_process_noise({frames[0]}, calib);
            EXPECT(false, "estimate_process_noise with one frame did not throw");
        } catch (const std::invalid_argument&) {
        }
        try {
            auto broken = frames;
            broken[1].pose.reset();
            tsgm::gpu::accumulate_error_map(broken, calib);
            EXPECT(false, "missing pose did not throw");
        } catch (const std::invalid_argument&) {
        }
    }
    {  // export formats: boxes.txt byte for byte; the PNG writer round trip is
       // checked by tests/test_export.py (the reference's libpng writer is
       // replaced by oracle/io_shim.cpp in this build)
        std::vector<std::vector<DetectionBox>> per_frame(3);
        per_frame[0].push_back(DetectionBox{3, 4, 30, 40, 1.0 / 3.0});
        per_frame[2].push_back(DetectionBox{100, 7, 160, 70, 12.5});
        per_frame[2].push_back(DetectionBox{0, 0, 20, 20, 1e-7});
        write_boxes("/tmp/tsgm_facade_boxes_ref.txt", per_frame);
        tsgm::gpu::write_boxes("/tmp/tsgm_facade_boxes_gpu.txt", per_frame);
        auto slurp = [](const char* p) {
            std::FILE* f = std::fopen(p, "rb");
            std::string out;
            if (!f) return out;
            char buf[4096];
            size_t n;
            while ((n = std::fread(buf, 1, sizeof buf, f)) > 0) out.append(buf, n);
            std::fclose(f);
            return out;
        };
        const std::string a = slurp("/tmp/tsgm_facade_boxes_ref.txt");
        EXPECT(!a.empty() && a == slurp("/tmp/tsgm_facade_boxes_gpu.txt"), "write_boxes");
        Image<double> disp(16, 8, 0.0);
        disp(3, 2) = 12.25;
        tsgm::gpu::write_disparity_png("/tmp/tsgm_facade_disp.png", disp);
        EXPECT(slurp("/tmp/tsgm_facade_disp.png").size() > 8, "write_disparity_png");
        const Image<double> back = tsgm::gpu::read_disparity_png("/tmp/tsgm_facade_disp.png");
        EXPECT(back.width() == 16 && back.height() == 8 && back(3, 2) == 12.25 && back(0, 0) == 0.0,
               "read_disparity_png round trip");
        try {
            disp(5, 5) = 300.0;
            tsgm::gpu::write_disparity_png("/tmp/tsgm_facade_disp_bad.png", disp);
            EXPECT(false, "non-encodable disparity did not throw");
        } catch (const std::invalid_argument& e) {
            EXPECT(std::string(e.what()) ==
                       "write_disparity_png: disparity 300.000000 not encodable at (5, 5)",
                   "write_disparity_png message");
        }
    }
    std::printf("facade parity: %s (%d failures)\n", fails ? "FAIL" : "ok", fails);
    return fails ? 1 : 0;
}
