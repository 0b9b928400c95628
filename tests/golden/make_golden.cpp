// Golden-fixture generator (test infrastructure, run HERE only: it needs
// /root/reference). Recreates the seeded fixtures of the reference's own unit
// tests and acceptance criteria (std::mt19937 + the helpers of
// /root/reference/proj/tests/oracles.hpp) and records the REFERENCE library's
// outputs for them, plus the outputs of the reference's brute-force oracles
// where the test compares against one. Build + run: tests/golden/make_golden.py.
//
// Output: a flat record stream "name\0 dtype\0 ndim shape... bytes" that
// make_golden.py turns into tests/golden/*.npz.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "oracles.hpp"
#include "tsgm/eval.hpp"
#include "tsgm/geometry.hpp"
#include "tsgm/matching_cost.hpp"
#include "tsgm/motion_detect.hpp"
#include "tsgm/sgm.hpp"
#include "tsgm/temporal_filter.hpp"

using namespace tsgm;

static FILE* g_out;

static void put(const std::string& name, const char* dtype, std::vector<long> shape,
                const void* data, size_t bytes) {
    std::fwrite(name.c_str(), 1, name.size() + 1, g_out);
    std::fwrite(dtype, 1, std::strlen(dtype) + 1, g_out);
    int nd = static_cast<int>(shape.size());
    std::fwrite(&nd, 4, 1, g_out);
    for (long s : shape) {
        long long v = s;
        std::fwrite(&v, 8, 1, g_out);
    }
    unsigned long long b = bytes;
    std::fwrite(&b, 8, 1, g_out);
    std::fwrite(data, 1, bytes, g_out);
}

template <typename T>
const char* dt();
template <> const char* dt<uint8_t>() { return "u1"; }
template <> const char* dt<uint16_t>() { return "u2"; }
template <> const char* dt<uint32_t>() { return "u4"; }
template <> const char* dt<int32_t>() { return "i4"; }
template <> const char* dt<double>() { return "f8"; }
template <> const char* dt<int64_t>() { return "i8"; }

template <typename T>
void put_img(const std::string& n, const Image<T>& im) {
    put(n, dt<T>(), {im.height(), im.width()}, im.data(), sizeof(T) * im.pixel_count());
}
template <typename T>
void put_vec(const std::string& n, const std::vector<T>& v) {
    put(n, dt<T>(), {static_cast<long>(v.size())}, v.data(), sizeof(T) * v.size());
}
void put_scalar(const std::string& n, double v) { put(n, "f8", {}, &v, 8); }
void put_params(const std::string& n, const SgmParams& p) {
    std::vector<int32_t> v = {p.p1, p.p2, p.paths, p.path_set == PathSet::diagonal ? 1 : 0, p.d_max};
    put_vec(n, v);
}
void put_state(const std::string& n, const DisparityState& s) {
    put_img(n + "_d", s.d);
    put_img(n + "_p", s.p);
    put_img(n + "_valid", s.valid);
}
void put_dmap(const std::string& n, const DisparityMap& m) {
    put_img(n + "_d", m.d);
    put_img(n + "_valid", m.valid);
}
void put_ranges(const std::string& n, const SearchRangeMap& r) {
    put_img(n + "_lo", r.lo);
    put_img(n + "_hi", r.hi);
}
std::vector<uint16_t> flatten(const oracle::CostGrid& g) {
    std::vector<uint16_t> out;
    for (const auto& px : g)
        for (long long v : px) out.push_back(static_cast<uint16_t>(v));
    return out;
}
void put_motion(const std::string& n, const RigidMotion& m) {
    std::vector<double> v;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) v.push_back(m.rotation(i, j));
    for (int i = 0; i < 3; ++i) v.push_back(m.translation(i));
    put_vec(n, v);
}

MatchingCostVolume random_volume(const SearchRangeMap& ranges, std::mt19937& rng) {
    MatchingCostVolume vol = make_cost_volume<std::uint8_t>(ranges);
    std::uniform_int_distribution<int> dist(0, kMaxMatchingCost);
    for (auto& c : vol.cost) c = static_cast<std::uint8_t>(dist(rng));
    return vol;
}

// Rodrigues rotation (harness-side; the fixture stores the resulting matrix).
Eigen::Matrix3d axis_rot(int axis, double a) {
    Eigen::Matrix3d r = Eigen::Matrix3d::Identity();
    const double c = std::cos(a), s = std::sin(a);
    const int i = (axis + 1) % 3, j = (axis + 2) % 3;
    r(i, i) = c;
    r(i, j) = -s;
    r(j, i) = s;
    r(j, j) = c;
    return r;
}
RigidMotion random_motion(std::mt19937& rng) {
    std::uniform_real_distribution<double> angle(-0.05, 0.05);
    std::uniform_real_distribution<double> shift(-0.3, 0.3);
    RigidMotion m;
    const double ax = angle(rng), ay = angle(rng), az = angle(rng);
    m.rotation = axis_rot(0, ax) * axis_rot(1, ay) * axis_rot(2, az);
    const double tx = shift(rng), ty = shift(rng), tz = shift(rng);
    m.translation = Eigen::Vector3d(tx, ty, tz);
    return m;
}

StereoCalib calib_of(double f, double cx, double cy, double b, int w, int h, int d_max) {
    StereoCalib c;
    c.focal_px = f;
    c.cx = cx;
    c.cy = cy;
    c.baseline_m = b;
    c.width = w;
    c.height = h;
    c.d_max = d_max;
    return c;
}
void put_calib(const std::string& n, const StereoCalib& c) {
    std::vector<double> v = {c.focal_px, c.cx, c.cy, c.baseline_m,
                             double(c.width), double(c.height), double(c.d_max)};
    put_vec(n, v);
}

int main(int argc, char** argv) {
    g_out = std::fopen(argc > 1 ? argv[1] : "golden.bin", "wb");

    // test_matching_cost.cpp:48-57 — census vs naive double loop, seed 11
    {
        std::mt19937 rng(11);
        for (int t = 0; t < 5; ++t) {
            const GrayImage img = oracle::random_gray(9, 9, rng);
            put_img("census_rand/" + std::to_string(t) + "/img", img);
            put_img("census_rand/" + std::to_string(t) + "/sig", census_transform(img).sig);
        }
    }
    // test_matching_cost.cpp:146-161 — ragged volume, seed 17
    {
        std::mt19937 rng(17);
        const GrayImage l = oracle::random_gray(14, 9, rng);
        const GrayImage r = oracle::random_gray(14, 9, rng);
        const SearchRangeMap ranges = oracle::random_ranges(14, 9, 10, rng);
        const MatchingCostVolume vol =
            build_cost_volume(census_transform(l), census_transform(r), ranges);
        put_img("cost_ragged/left", l);
        put_img("cost_ragged/right", r);
        put_ranges("cost_ragged/ranges", ranges);
        put_vec("cost_ragged/offsets", vol.offsets);
        put_vec("cost_ragged/cost", vol.cost);
    }
    // test_sgm.cpp:232-240, 255-284 — aggregation vs brute-force oracle
    {
        std::mt19937 rng(21);
        const SearchRangeMap ranges(5, 1, 0, 3);
        const MatchingCostVolume vol = random_volume(ranges, rng);
        SgmParams p;
        p.paths = 4;
        p.d_max = 4;
        put_ranges("agg_scanline/ranges", ranges);
        put_vec("agg_scanline/cost", vol.cost);
        put_params("agg_scanline/params", p);
        put_vec("agg_scanline/agg", aggregate_paths(vol, p).cost);
        put_vec("agg_scanline/oracle", flatten(oracle::aggregate(vol, p)));
    }
    {
        std::mt19937 rng(22);
        int k = 0;
        for (int trial = 0; trial < 3; ++trial) {
            const SearchRangeMap ranges = SearchRangeMap::full(9, 6, 5);
            const MatchingCostVolume vol = random_volume(ranges, rng);
            for (auto [paths, set] : {std::pair{8, PathSet::nondiagonal},
                                      {4, PathSet::nondiagonal},
                                      {4, PathSet::diagonal}}) {
                SgmParams p;
                p.paths = paths;
                p.path_set = set;
                p.d_max = 5;
                const std::string n = "agg_full/" + std::to_string(k++);
                put_ranges(n + "/ranges", ranges);
                put_vec(n + "/cost", vol.cost);
                put_params(n + "/params", p);
                put_vec(n + "/agg", aggregate_paths(vol, p).cost);
                put_vec(n + "/oracle", flatten(oracle::aggregate(vol, p)));
            }
        }
    }
    {
        std::mt19937 rng(23);
        int k = 0;
        for (int trial = 0; trial < 4; ++trial) {
            const SearchRangeMap ranges = oracle::random_ranges(8, 7, 9, rng);
            const MatchingCostVolume vol = random_volume(ranges, rng);
            SgmParams p;
            p.d_max = 9;
            SgmParams d4 = p;
            d4.paths = 4;
            d4.path_set = PathSet::diagonal;
            for (const SgmParams& pp : {p, d4}) {
                const std::string n = "agg_ragged/" + std::to_string(k++);
                put_ranges(n + "/ranges", ranges);
                put_vec(n + "/cost", vol.cost);
                put_params(n + "/params", pp);
                const AggregatedCostVolume agg = aggregate_paths(vol, pp);
                put_vec(n + "/agg", agg.cost);
                put_vec(n + "/oracle", flatten(oracle::aggregate(vol, pp)));
                put_dmap(n + "/wta", winner_takes_all(agg));
            }
        }
    }
    // test_sgm.cpp:333-343 — WTA vs linear scan, seed 25
    {
        std::mt19937 rng(25);
        const SearchRangeMap ranges = oracle::random_ranges(11, 9, 8, rng);
        AggregatedCostVolume agg = make_cost_volume<std::uint16_t>(ranges);
        std::uniform_int_distribution<int> dist(0, 500);
        for (auto& c : agg.cost) c = static_cast<std::uint16_t>(dist(rng));
        put_ranges("wta_rand/ranges", ranges);
        put_vec("wta_rand/agg", agg.cost);
        put_dmap("wta_rand/out", winner_takes_all(agg));
        put_dmap("wta_rand/oracle", oracle::wta(oracle::grid_from_volume(agg), ranges));
    }
    // test_sgm.cpp:403-416 — median vs sort-based oracle, seed 27
    {
        std::mt19937 rng(27);
        std::uniform_int_distribution<int> dval(0, 60);
        std::uniform_int_distribution<int> dvalid(0, 3);
        for (int t = 0; t < 5; ++t) {
            DisparityMap dm(9, 8);
            for (int y = 0; y < 8; ++y)
                for (int x = 0; x < 9; ++x) {
                    dm.d(x, y) = dval(rng);
                    dm.valid(x, y) = dvalid(rng) > 0 ? 1 : 0;
                }
            const std::string n = "median_rand/" + std::to_string(t);
            put_dmap(n + "/in", dm);
            put_dmap(n + "/out", median_refine(dm));
            put_dmap(n + "/oracle", oracle::median3(dm));
        }
    }
    // test_sgm.cpp:419-432 — shifted pair, seed 28, and :446-457 seed 30
    {
        std::mt19937 rng(28);
        const auto [l, r] = oracle::shifted_pair(40, 20, 5, rng);
        SgmParams p;
        p.d_max = 16;
        put_img("shifted/left", l);
        put_img("shifted/right", r);
        put_params("shifted/params", p);
        put_dmap("shifted/out", sgm_match(l, r, SearchRangeMap::full(40, 20, 16), p));
    }
    {
        std::mt19937 rng(30);
        const auto [l, r] = oracle::shifted_pair(45, 30, 7, rng);
        SgmParams p;
        p.d_max = 12;
        put_img("shifted12/left", l);
        put_img("shifted12/right", r);
        put_params("shifted12/params", p);
        const DisparityMap dm = sgm_match(l, r, SearchRangeMap::full(45, 30, 12), p);
        put_dmap("shifted12/out", dm);
        put_dmap("shifted12/median", median_refine(dm));
    }
    // acceptance.cpp:42-90 (criterion 1) — 50 random 16x8 pairs, seed 101
    {
        std::mt19937 rng(101);
        std::uniform_int_distribution<int> p1_dist(1, 8);
        std::uniform_int_distribution<int> p2_extra(0, 70);
        for (int trial = 0; trial < 50; ++trial) {
            const GrayImage left = oracle::random_gray(16, 8, rng);
            const GrayImage right = oracle::random_gray(16, 8, rng);
            SgmParams p;
            p.d_max = 8;
            p.p1 = p1_dist(rng);
            p.p2 = p.p1 + p2_extra(rng);
            p.paths = trial % 3 == 2 ? 4 : 8;
            p.path_set = trial % 3 == 1 ? PathSet::diagonal : PathSet::nondiagonal;
            const SearchRangeMap ranges = SearchRangeMap::full(16, 8, 8);
            const MatchingCostVolume vol =
                build_cost_volume(census_transform(left), census_transform(right), ranges);
            const AggregatedCostVolume agg = aggregate_paths(vol, p);
            const std::string n = "crit1/" + std::to_string(trial);
            put_img(n + "/left", left);
            put_img(n + "/right", right);
            put_params(n + "/params", p);
            put_vec(n + "/cost", vol.cost);
            put_vec(n + "/agg", agg.cost);
            put_vec(n + "/oracle", flatten(oracle::aggregate(vol, p)));
            put_dmap(n + "/wta", winner_takes_all(agg));
        }
    }
    // test_geometry.cpp:228-247 — warp vs gather oracle, seed 46
    {
        std::mt19937 rng(46);
        const StereoCalib c = calib_of(240.0, 160.0, 120.0, 0.5, 320, 240, 128);
        std::uniform_real_distribution<double> pd(1.0, 120.0);
        std::uniform_real_distribution<double> pp(0.5, 50.0);
        std::uniform_int_distribution<int> keep(0, 4);
        for (int t = 0; t < 4; ++t) {
            DisparityState s(48, 36);
            for (int y = 0; y < 36; ++y)
                for (int x = 0; x < 48; ++x)
                    if (keep(rng) > 0) {
                        const double dv = pd(rng);
                        const double pv = pp(rng);
                        s.set(x, y, dv, pv);
                    }
            const RigidMotion m = random_motion(rng);
            const DispHomography h = disparity_homography(m, c);
            const std::string n = "warp/" + std::to_string(t);
            put_calib(n + "/calib", c);
            put_motion(n + "/motion", m);
            std::vector<double> hv;
            for (int i = 0; i < 4; ++i)
                for (int j = 0; j < 4; ++j) hv.push_back(h.m(i, j));
            put_vec(n + "/H", hv);
            put_state(n + "/in", s);
            const WarpedState ws = warp_state_ex(s, h, c.d_max);
            put_state(n + "/out", ws.state);
            put_img(n + "/source_d", ws.source_d);
            put_state(n + "/oracle", oracle::warp(s, h, c.d_max));
            put_state(n + "/predict", predict(s, m, c, FilterConfig{}));
        }
    }
    // test_temporal_filter.cpp:317-356 — step on empty state; static contraction
    {
        std::mt19937 rng(53);
        const auto [l, r] = oracle::shifted_pair(48, 24, 6, rng);
        const StereoCalib calib = calib_of(200.0, 24.0, 12.0, 0.4, 48, 24, 16);
        SgmParams p;
        p.d_max = 16;
        const StepResult res = step(DisparityState(), l, r, RigidMotion{}, calib, p, FilterConfig{});
        put_img("step_empty/left", l);
        put_img("step_empty/right", r);
        put_calib("step_empty/calib", calib);
        put_params("step_empty/params", p);
        put_state("step_empty/state", res.state);
        put_dmap("step_empty/export", res.export_map);
        put_img("step_empty/diff", res.diff);
        put_dmap("step_empty/direct_median",
                 median_refine(sgm_match(l, r, SearchRangeMap::full(48, 24, 16), p)));
    }
    {
        std::mt19937 rng(54);
        const auto [l, r] = oracle::shifted_pair(48, 24, 6, rng);
        const StereoCalib calib = calib_of(200.0, 24.0, 12.0, 0.4, 48, 24, 16);
        SgmParams p;
        p.d_max = 16;
        put_img("step_static/left", l);
        put_img("step_static/right", r);
        put_calib("step_static/calib", calib);
        put_params("step_static/params", p);
        StepResult res = step(DisparityState(), l, r, RigidMotion{}, calib, p, FilterConfig{});
        for (int i = 0; i <= 10; ++i) {
            const std::string n = "step_static/" + std::to_string(i);
            put_state(n + "/state", res.state);
            put_dmap(n + "/export", res.export_map);
            put_img(n + "/diff", res.diff);
            res = step(res.state, l, r, RigidMotion{}, calib, p, FilterConfig{});
        }
    }
    // moving-camera recursion with the BASELINE parameters on a textured
    // shifted pair (harness-made; exercises predict/ranges/reduced SGM/correct)
    {
        std::mt19937 rng(77);
        const int w = 96, h = 48;
        const auto [l, r] = oracle::shifted_pair(w, h, 9, rng);
        const StereoCalib calib = calib_of(120.0, 47.5, 23.5, 0.54, w, h, 32);
        SgmParams p;
        p.p1 = 10;
        p.p2 = 120;
        p.d_max = 32;
        FilterConfig f;
        f.range_use_stddev = true;
        f.range_stddev_gain = 3.0;
        put_img("step_moving/left", l);
        put_img("step_moving/right", r);
        put_calib("step_moving/calib", calib);
        put_params("step_moving/params", p);
        DisparityState st;
        for (int i = 0; i < 6; ++i) {
            RigidMotion m;
            if (i > 0) {
                m.rotation = axis_rot(1, 0.002 * i);
                m.translation = Eigen::Vector3d(0.01 * i, 0.0, -0.05);
            }
            const std::string n = "step_moving/" + std::to_string(i);
            put_motion(n + "/motion", m);
            const DisparityState prior = st.width() ? st : DisparityState(w, h);
            const DisparityState pred = predict(prior, m, calib, f);
            const SearchRangeMap ranges = derive_search_ranges(pred, calib, f);
            const DisparityMap meas = sgm_match(l, r, ranges, p);
            put_state(n + "/pred", pred);
            put_ranges(n + "/ranges", ranges);
            put_dmap(n + "/meas", meas);
            const StepResult res = step(st, l, r, m, calib, p, f);
            put_state(n + "/state", res.state);
            put_dmap(n + "/export", res.export_map);
            put_img(n + "/diff", res.diff);
            st = res.state;
        }
    }
    // ---- box detector (test_motion_detect.cpp), SURVEY §8(f) row 1 ----
    auto put_boxes = [](const std::string& n, const std::vector<DetectionBox>& v) {
        std::vector<double> f;
        for (const DetectionBox& b : v) {
            f.push_back(b.x0);
            f.push_back(b.y0);
            f.push_back(b.x1);
            f.push_back(b.y1);
            f.push_back(b.score);
        }
        put(n, "f8", {static_cast<long>(v.size()), 5}, f.data(), sizeof(double) * f.size());
    };
    {   // test_motion_detect.cpp:60-69 — SAT of a random integer map, seed 61
        std::mt19937 rng(61);
        Image<double> m(100, 100);
        std::uniform_int_distribution<int> dist(0, 20);
        for (int y = 0; y < 100; ++y)
            for (int x = 0; x < 100; ++x) m(x, y) = dist(rng);
        const SummedAreaTable sat = integral_image(m);
        put_img("det_sat/map", m);
        put("det_sat/sat", "f8", {101, 101}, sat.sum.data(), sizeof(double) * sat.sum.size());
    }
    {   // :86-133 — candidate windows on the test maps
        DetectConfig cfg;
        Image<double> hot(120, 120, 0.0);
        for (int y = 60; y < 100; ++y)
            for (int x = 40; x < 80; ++x) hot(x, y) = 10.0;
        put_img("det_cand/hot", hot);
        put_boxes("det_cand/hot_boxes", detect_candidate_windows(hot, cfg));
        std::mt19937 rng(62);
        Image<double> rnd(150, 150, 0.0);
        std::uniform_real_distribution<double> v(0.0, 6.0);
        for (int y = 0; y < 150; ++y)
            for (int x = 0; x < 150; ++x) rnd(x, y) = v(rng);
        put_img("det_cand/rand", rnd);
        put_boxes("det_cand/rand_boxes", detect_candidate_windows(rnd, cfg));
        Image<double> flat(200, 90, 5.0);
        put_img("det_cand/flat", flat);
        put_boxes("det_cand/flat_boxes", detect_candidate_windows(flat, cfg));
    }
    {   // :165-195 — greedy merging of random box sets, seeds 63 and 64
        for (int seed : {63, 64}) {
            std::mt19937 rng(seed);
            std::uniform_int_distribution<int> c(0, seed == 63 ? 60 : 50);
            std::uniform_int_distribution<int> sz(seed == 63 ? 20 : 21, seed == 63 ? 40 : 35);
            std::vector<DetectionBox> in;
            for (int i = 0; i < (seed == 63 ? 40 : 25); ++i) {
                const int x0 = c(rng), y0 = c(rng);
                in.push_back({x0, y0, x0 + sz(rng), y0 + sz(rng), 1.0});
            }
            DetectConfig loose;
            loose.min_box_area = 0;
            const std::string n = "det_merge/s" + std::to_string(seed);
            put_boxes(n + "/in", in);
            put_boxes(n + "/out_default", greedy_merge(in, DetectConfig{}));
            put_boxes(n + "/out_loose", greedy_merge(in, loose));
        }
    }
    {   // :221-257 — end-to-end detection, plus a KITTI-sized sparse map
        Image<double> blk(160, 160, 0.0);
        for (int y = 90; y < 130; ++y)
            for (int x = 60; x < 100; ++x) blk(x, y) = 3.0;
        DetectConfig cfg;
        cfg.merge_stop_iou = 0.12;
        put_img("det_e2e/block", blk);
        put_boxes("det_e2e/block_boxes", detect_moving_objects(blk, cfg));
        Image<double> three(160, 160, 0.0);
        for (auto [bx, by] : {std::pair{20, 60}, {90, 100}, {40, 120}})
            for (int y = by; y < by + 25; ++y)
                for (int x = bx; x < bx + 25; ++x) three(x, y) = 6.0;
        put_img("det_e2e/three", three);
        put_boxes("det_e2e/three_boxes", detect_moving_objects(three, DetectConfig{}));
        std::mt19937 rng(65);
        Image<double> big(1242, 375, 0.0);
        std::uniform_int_distribution<int> bxd(0, 1100), byd(100, 300), bsz(20, 120);
        std::uniform_real_distribution<double> val(1.0, 9.0);
        for (int k = 0; k < 8; ++k) {
            const int x0 = bxd(rng), y0 = byd(rng), w = bsz(rng), h = bsz(rng) / 2 + 10;
            const double v0 = val(rng);
            for (int y = y0; y < std::min(375, y0 + h); ++y)
                for (int x = x0; x < std::min(1242, x0 + w); ++x) big(x, y) = v0 + 0.01 * ((x * 7 + y * 3) % 11);
        }
        put_img("det_e2e/kitti", big);
        put_boxes("det_e2e/kitti_cands", detect_candidate_windows(big, DetectConfig{}));
        put_boxes("det_e2e/kitti_boxes", detect_moving_objects(big, DetectConfig{}));
    }
    {   // eval.cpp:59-85 / test_eval.cpp — outlier counts on random maps
        std::mt19937 rng(66);
        for (int t = 0; t < 4; ++t) {
            const int w = 40 + 30 * t, h = 20 + 10 * t;
            DisparityMap est(w, h);
            Image<double> gt(w, h, 0.0);
            std::uniform_int_distribution<int> dd(0, 90), vv(0, 4);
            std::uniform_real_distribution<double> gg(-5.0, 90.0);
            for (int y = 0; y < h; ++y)
                for (int x = 0; x < w; ++x) {
                    est.d(x, y) = dd(rng);
                    est.valid(x, y) = vv(rng) != 0;
                    const double g = gg(rng);
                    gt(x, y) = g < 0.0 ? 0.0 : (t == 3 ? std::round(g) : g);
                }
            const std::string n = "eval_outliers/" + std::to_string(t);
            put_img(n + "/d", est.d);
            put_img(n + "/valid", est.valid);
            put_img(n + "/gt", gt);
            for (int strict = 0; strict < 2; ++strict) {
                OutlierOptions o;
                o.strict_density = strict != 0;
                const OutlierStats s = count_outliers(est, gt, o);
                const std::vector<int64_t> c = {s.evaluated, s.outliers};
                put_vec(n + "/counts_strict" + std::to_string(strict), c);
            }
        }
    }
    std::fclose(g_out);
    return 0;
}
