// TEST INFRASTRUCTURE ONLY. C-ABI harness over the UNMODIFIED reference
// sources (compiled in place from /root/reference/proj/src by oracle/Makefile
// into oracle/_ref/libtsgm_ref.so). Only tests/, bench.py's reference arm /
// cpu_baseline leg and __graft_entry__.smoke() load it, always as the checker
// or the CPU baseline, never as the product.
//
// Every entry point returns 0 on success, 1 for std::invalid_argument, 2 for
// any other exception; the message is available from ref_last_error().
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "tsgm/eval.hpp"
#include "tsgm/geometry.hpp"
#include "tsgm/matching_cost.hpp"
#include "tsgm/motion_detect.hpp"
#include "tsgm/sgm.hpp"
#include "tsgm/temporal_filter.hpp"

using namespace tsgm;

namespace {

thread_local std::string g_err;

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

template <typename T>
Image<T> to_image(const T* src, int w, int h) {
    Image<T> img(w, h);
    if (src)
        std::memcpy(img.data(), src, sizeof(T) * static_cast<size_t>(w) * h);
    return img;
}

template <typename T>
void from_image(const Image<T>& img, T* dst) {
    if (dst)
        std::memcpy(dst, img.data(), sizeof(T) * img.pixel_count());
}

DisparityState to_state(const double* d, const double* p, const uint8_t* v, int w, int h) {
    DisparityState s;
    s.d = to_image(d, w, h);
    s.p = to_image(p, w, h);
    s.valid = to_image(v, w, h);
    return s;
}

void from_state(const DisparityState& s, double* d, double* p, uint8_t* v) {
    from_image(s.d, d);
    from_image(s.p, p);
    from_image(s.valid, v);
}

SearchRangeMap to_ranges(const uint16_t* lo, const uint16_t* hi, int w, int h) {
    SearchRangeMap r;
    r.lo = to_image(lo, w, h);
    r.hi = to_image(hi, w, h);
    return r;
}

StereoCalib make_calib(const double* c4, int w, int h, int d_max) {
    StereoCalib c;
    c.focal_px = c4[0];
    c.cx = c4[1];
    c.cy = c4[2];
    c.baseline_m = c4[3];
    c.width = w;
    c.height = h;
    c.d_max = d_max;
    return c;
}

RigidMotion make_motion(const double* r9, const double* t3) {
    RigidMotion m;
    for (int i = 0; i < 3; ++i) {
        for (int j = 0; j < 3; ++j)
            m.rotation(i, j) = r9[i * 3 + j];
        m.translation(i) = t3[i];
    }
    return m;
}

// sgm params: {p1, p2, paths, path_set(0 nondiag, 1 diag), d_max}
SgmParams make_params(const int* sp) {
    SgmParams p;
    p.p1 = sp[0];
    p.p2 = sp[1];
    p.paths = sp[2];
    p.path_set = sp[3] ? PathSet::diagonal : PathSet::nondiagonal;
    p.d_max = sp[4];
    return p;
}

// filter: {q, r, p_init, disc_thresh, min_range_halfwidth, range_use_stddev, gain}
FilterConfig make_filter(const double* fc) {
    FilterConfig f;
    f.noise.q = fc[0];
    f.noise.r = fc[1];
    f.p_init = fc[2];
    f.disc_thresh = fc[3];
    f.min_range_halfwidth = static_cast<int>(fc[4]);
    f.range_use_stddev = fc[5] != 0.0;
    f.range_stddev_gain = fc[6];
    return f;
}

DisparityMap to_dmap(const int32_t* d, const uint8_t* v, int w, int h) {
    DisparityMap m;
    m.d = to_image(d, w, h);
    m.valid = to_image(v, w, h);
    return m;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_census(const uint8_t* img, int w, int h, uint32_t* sig) {
    return guarded([&] { from_image(census_transform(to_image(img, w, h)).sig, sig); });
}

// Ragged cost volume for (left, right, ranges). offsets: w*h+1 u32, cost: cap bytes.
int ref_cost_volume(const uint8_t* left, const uint8_t* right, int w, int h, const uint16_t* lo,
                    const uint16_t* hi, uint32_t* offsets, uint8_t* cost, uint64_t cap,
                    int threads) {
    return guarded([&] {
        const CensusMap cl = census_transform(to_image(left, w, h), threads);
        const CensusMap cr = census_transform(to_image(right, w, h), threads);
        const MatchingCostVolume vol = build_cost_volume(cl, cr, to_ranges(lo, hi, w, h), threads);
        if (vol.cost.size() > cap)
            throw std::runtime_error("ref_cost_volume: capacity too small");
        std::memcpy(offsets, vol.offsets.data(), vol.offsets.size() * 4);
        std::memcpy(cost, vol.cost.data(), vol.cost.size());
    });
}

// aggregate_paths over a caller-provided ragged matching-cost volume.
int ref_aggregate(const uint8_t* cost, const uint16_t* lo, const uint16_t* hi, int w, int h,
                  const int* sgm_params, uint16_t* agg) {
    return guarded([&] {
        MatchingCostVolume vol = make_cost_volume<std::uint8_t>(to_ranges(lo, hi, w, h));
        std::memcpy(vol.cost.data(), cost, vol.cost.size());
        const AggregatedCostVolume a = aggregate_paths(vol, make_params(sgm_params));
        std::memcpy(agg, a.cost.data(), a.cost.size() * 2);
    });
}

int ref_wta(const uint16_t* agg, const uint16_t* lo, const uint16_t* hi, int w, int h,
            int32_t* d, uint8_t* valid) {
    return guarded([&] {
        AggregatedCostVolume a = make_cost_volume<std::uint16_t>(to_ranges(lo, hi, w, h));
        std::memcpy(a.cost.data(), agg, a.cost.size() * 2);
        const DisparityMap dm = winner_takes_all(a);
        from_image(dm.d, d);
        from_image(dm.valid, valid);
    });
}

int ref_median(const int32_t* d, const uint8_t* valid, int w, int h, int32_t* out_d,
               uint8_t* out_valid) {
    return guarded([&] {
        const DisparityMap m = median_refine(to_dmap(d, valid, w, h));
        from_image(m.d, out_d);
        from_image(m.valid, out_valid);
    });
}

int ref_sgm_match(const uint8_t* left, const uint8_t* right, int w, int h, const uint16_t* lo,
                  const uint16_t* hi, const int* sgm_params, int threads, int32_t* d,
                  uint8_t* valid) {
    return guarded([&] {
        const DisparityMap dm = sgm_match(to_image(left, w, h), to_image(right, w, h),
                                          to_ranges(lo, hi, w, h), make_params(sgm_params), threads);
        from_image(dm.d, d);
        from_image(dm.valid, valid);
    });
}

int ref_relative_motion(const double* prev12, const double* cur12, double* r9, double* t3) {
    return guarded([&] {
        Pose a, b;
        for (int i = 0; i < 12; ++i) {
            a(i / 4, i % 4) = prev12[i];
            b(i / 4, i % 4) = cur12[i];
        }
        const RigidMotion m = relative_motion(a, b);
        for (int i = 0; i < 3; ++i) {
            for (int j = 0; j < 3; ++j)
                r9[i * 3 + j] = m.rotation(i, j);
            t3[i] = m.translation(i);
        }
    });
}

int ref_homography(const double* r9, const double* t3, const double* calib4, int w, int h,
                   int d_max, double* h16) {
    return guarded([&] {
        const DispHomography hm =
            disparity_homography(make_motion(r9, t3), make_calib(calib4, w, h, d_max));
        for (int i = 0; i < 4; ++i)
            for (int j = 0; j < 4; ++j)
                h16[i * 4 + j] = hm.m(i, j);
    });
}

int ref_warp(const double* d, const double* p, const uint8_t* valid, int w, int h,
             const double* h16, int d_max, double* od, double* op, uint8_t* ovalid,
             double* osrc) {
    return guarded([&] {
        DispHomography hm;
        for (int i = 0; i < 4; ++i)
            for (int j = 0; j < 4; ++j)
                hm.m(i, j) = h16[i * 4 + j];
        const WarpedState ws = warp_state_ex(to_state(d, p, valid, w, h), hm, d_max);
        from_state(ws.state, od, op, ovalid);
        from_image(ws.source_d, osrc);
    });
}

int ref_predict(const double* d, const double* p, const uint8_t* valid, int w, int h,
                const double* r9, const double* t3, const double* calib4, int d_max,
                const double* filter, double* od, double* op, uint8_t* ovalid) {
    return guarded([&] {
        const DisparityState s = predict(to_state(d, p, valid, w, h), make_motion(r9, t3),
                                         make_calib(calib4, w, h, d_max), make_filter(filter));
        from_state(s, od, op, ovalid);
    });
}

int ref_reject(const double* d, const double* p, const uint8_t* valid, int w, int h,
               const double* filter, double* od, double* op, uint8_t* ovalid) {
    return guarded([&] {
        from_state(reject_discontinuities(to_state(d, p, valid, w, h), make_filter(filter)), od,
                   op, ovalid);
    });
}

int ref_fill(const double* d, const double* p, const uint8_t* valid, int w, int h, double* od,
             double* op, uint8_t* ovalid) {
    return guarded(
        [&] { from_state(fill_zoom_holes(to_state(d, p, valid, w, h)), od, op, ovalid); });
}

int ref_ranges(const double* d, const double* p, const uint8_t* valid, int w, int h,
               const double* calib4, int d_max, const double* filter, uint16_t* lo,
               uint16_t* hi) {
    return guarded([&] {
        const SearchRangeMap r = derive_search_ranges(
            to_state(d, p, valid, w, h), make_calib(calib4, w, h, d_max), make_filter(filter));
        from_image(r.lo, lo);
        from_image(r.hi, hi);
    });
}

int ref_correct(const double* d, const double* p, const uint8_t* valid, const int32_t* md,
                const uint8_t* mvalid, int w, int h, const double* filter, double* od,
                double* op, uint8_t* ovalid) {
    return guarded([&] {
        from_state(correct(to_state(d, p, valid, w, h), to_dmap(md, mvalid, w, h),
                           make_filter(filter)),
                   od, op, ovalid);
    });
}

int ref_disparity_difference(const double* d, const double* p, const uint8_t* valid,
                             const int32_t* md, const uint8_t* mvalid, int w, int h,
                             double* diff) {
    return guarded([&] {
        from_image(disparity_difference(to_state(d, p, valid, w, h), to_dmap(md, mvalid, w, h)),
                   diff);
    });
}

// tsgm::step. state_* may be null together with w_state == 0 for the default
// (empty) state. Outputs: posterior state, export map, diff.
int ref_step(const double* sd, const double* sp, const uint8_t* sv, int state_w, int state_h,
             const uint8_t* left, const uint8_t* right, int w, int h, const double* r9,
             const double* t3, const double* calib4, int calib_d_max, const int* sgm_params,
             const double* filter, int threads, double* od, double* op, uint8_t* ov,
             int32_t* ed, uint8_t* ev, double* diff) {
    return guarded([&] {
        DisparityState st;
        if (state_w > 0 || state_h > 0)
            st = to_state(sd, sp, sv, state_w, state_h);
        const StepResult res =
            step(st, to_image(left, w, h), to_image(right, w, h), make_motion(r9, t3),
                 make_calib(calib4, w, h, calib_d_max), make_params(sgm_params),
                 make_filter(filter), threads);
        from_state(res.state, od, op, ov);
        from_image(res.export_map.d, ed);
        from_image(res.export_map.valid, ev);
        from_image(res.diff, diff);
    });
}

int ref_sgm_validate(const int* sgm_params) {
    return guarded([&] { make_params(sgm_params).validate(); });
}

int ref_filter_validate(const double* filter, int d_max) {
    return guarded([&] { make_filter(filter).validate(d_max); });
}


// ---- box detector (motion_detect.cpp), SURVEY §8(f) row 1. Boxes are
// exchanged as 5 doubles each: x0, y0, x1, y1, score.
}  // extern "C"

namespace {
DetectConfig make_detect(const int* wh, int n_windows, double thresh, double stop_iou,
                         long long min_area) {
    DetectConfig c;
    c.window_sizes.clear();
    for (int i = 0; i < n_windows; ++i) c.window_sizes.emplace_back(wh[2 * i], wh[2 * i + 1]);
    c.score_thresh = thresh;
    c.merge_stop_iou = stop_iou;
    c.min_box_area = min_area;
    return c;
}
long long put_boxes(const std::vector<DetectionBox>& v, double* out, long long cap) {
    for (size_t i = 0; i < v.size() && static_cast<long long>(i) < cap; ++i) {
        out[5 * i + 0] = v[i].x0;
        out[5 * i + 1] = v[i].y0;
        out[5 * i + 2] = v[i].x1;
        out[5 * i + 3] = v[i].y1;
        out[5 * i + 4] = v[i].score;
    }
    return static_cast<long long>(v.size());
}
std::vector<DetectionBox> get_boxes(const double* in, long long n) {
    std::vector<DetectionBox> v(static_cast<size_t>(n));
    for (long long i = 0; i < n; ++i)
        v[i] = DetectionBox{static_cast<int>(in[5 * i]), static_cast<int>(in[5 * i + 1]),
                            static_cast<int>(in[5 * i + 2]), static_cast<int>(in[5 * i + 3]),
                            in[5 * i + 4]};
    return v;
}
}  // namespace

extern "C" {

int ref_integral_image(const double* map, int w, int h, double* sat) {
    return guarded([&] {
        const SummedAreaTable t = integral_image(to_image(map, w, h));
        std::memcpy(sat, t.sum.data(), sizeof(double) * t.sum.size());
    });
}

int ref_candidates(const double* diff, int w, int h, const int* wh, int n_windows, double thresh,
                   double stop_iou, long long min_area, int threads, double* out, long long cap,
                   long long* n_out) {
    return guarded([&] {
        *n_out = put_boxes(detect_candidate_windows(to_image(diff, w, h),
                                                    make_detect(wh, n_windows, thresh, stop_iou,
                                                                min_area),
                                                    threads),
                           out, cap);
    });
}

int ref_greedy_merge(const double* in, long long n, const int* wh, int n_windows, double thresh,
                     double stop_iou, long long min_area, double* out, long long* n_out) {
    return guarded([&] {
        *n_out = put_boxes(greedy_merge(get_boxes(in, n),
                                        make_detect(wh, n_windows, thresh, stop_iou, min_area)),
                           out, n);
    });
}

int ref_detect(const double* diff, int w, int h, const int* wh, int n_windows, double thresh,
               double stop_iou, long long min_area, int threads, double* out, long long cap,
               long long* n_out) {
    return guarded([&] {
        *n_out = put_boxes(detect_moving_objects(to_image(diff, w, h),
                                                 make_detect(wh, n_windows, thresh, stop_iou,
                                                             min_area),
                                                 threads),
                           out, cap);
    });
}

int ref_count_outliers(const int32_t* d, const uint8_t* valid, const double* gt, int w, int h,
                       double abs_thresh, double rel_thresh, int strict, long long* evaluated,
                       long long* outliers) {
    return guarded([&] {
        DisparityMap est;
        est.d = to_image(d, w, h);
        est.valid = to_image(valid, w, h);
        OutlierOptions o;
        o.abs_thresh_px = abs_thresh;
        o.rel_thresh = rel_thresh;
        o.strict_density = strict != 0;
        const OutlierStats s = count_outliers(est, to_image(gt, w, h), o);
        *evaluated = s.evaluated;
        *outliers = s.outliers;
    });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Noise calibration (noise_calib.cpp), SURVEY §8(f) row 4. Frames: n
// contiguous W x H maps; null image / gt / pose arrays leave the optional
// fields empty (for the reference's own "missing GT / pose" errors).
#include "tsgm/noise_calib.hpp"

namespace {

std::vector<SequenceFrame> make_frames(int n, int w, int h, const uint8_t* left,
                                       const uint8_t* right, const double* gt,
                                       const double* poses) {
    const size_t P = static_cast<size_t>(w) * h;
    std::vector<SequenceFrame> frames(static_cast<size_t>(n));
    for (int k = 0; k < n; ++k) {
        SequenceFrame& f = frames[static_cast<size_t>(k)];
        f.index = k;
        if (left) f.left = to_image(left + k * P, w, h);
        if (right) f.right = to_image(right + k * P, w, h);
        if (gt) f.gt_disp = to_image(gt + k * P, w, h);
        if (poses) {
            Pose p;
            for (int i = 0; i < 12; ++i) p(i / 4, i % 4) = poses[12 * k + i];
            f.pose = p;
        }
    }
    return frames;
}

CalibOptions make_opts(const double* o3) {
    CalibOptions o;
    o.outlier_gate_px = o3[0];
    o.bin_width = o3[1];
    o.q_floor = o3[2];
    return o;
}

// moments: variance, mean, fraction within 1 px; ints: samples_used, total,
// underflow, overflow; counts: the bins (up to nbins)
void put_estimate(const NoiseEstimate& e, double* moments, long long* ints, long long* counts,
                  int nbins) {
    moments[0] = e.variance;
    moments[1] = e.hist.mean();
    moments[2] = e.hist.fraction_within_1px();
    ints[0] = e.samples_used;
    ints[1] = e.hist.total();
    ints[2] = e.hist.underflow;
    ints[3] = e.hist.overflow;
    ints[4] = static_cast<long long>(e.hist.counts.size());
    for (size_t i = 0; i < e.hist.counts.size() && static_cast<int>(i) < nbins; ++i)
        counts[i] = e.hist.counts[i];
}

}  // namespace

extern "C" {

int ref_process_noise(int n, int w, int h, const double* gt, const double* poses,
                      const double* calib4, int cw, int ch, int d_max, const double* opts3,
                      double* moments, long long* ints, long long* counts, int nbins) {
    return guarded([&] {
        const NoiseEstimate e = estimate_process_noise(
            make_frames(n, w, h, nullptr, nullptr, gt, poses), make_calib(calib4, cw, ch, d_max),
            make_opts(opts3));
        put_estimate(e, moments, ints, counts, nbins);
    });
}

int ref_measurement_noise(int n, int w, int h, const uint8_t* left, const uint8_t* right,
                          const double* gt, const int* sgm_params, int threads,
                          const double* opts3, double* moments, long long* ints,
                          long long* counts, int nbins) {
    return guarded([&] {
        const NoiseEstimate e =
            estimate_measurement_noise(make_frames(n, w, h, left, right, gt, nullptr),
                                       make_params(sgm_params), threads, make_opts(opts3));
        put_estimate(e, moments, ints, counts, nbins);
    });
}

int ref_accumulate_error_map(int n, int w, int h, const double* gt, const double* poses,
                             const double* calib4, int cw, int ch, int d_max, double* acc) {
    return guarded([&] {
        const Image<double> m = accumulate_error_map(
            make_frames(n, w, h, nullptr, nullptr, gt, poses), make_calib(calib4, cw, ch, d_max));
        from_image(m, acc);
    });
}

// Both estimates by the reference, then its write_calib_report.
int ref_calib_report(const char* path, int n, int w, int h, const uint8_t* left,
                     const uint8_t* right, const double* gt, const double* poses,
                     const double* calib4, int cw, int ch, int d_max, const int* sgm_params,
                     const double* opts3) {
    return guarded([&] {
        const auto frames = make_frames(n, w, h, left, right, gt, poses);
        const CalibOptions o = make_opts(opts3);
        const NoiseEstimate pe = estimate_process_noise(frames, make_calib(calib4, cw, ch, d_max), o);
        const NoiseEstimate me = estimate_measurement_noise(frames, make_params(sgm_params), 1, o);
        write_calib_report(path, pe, me, o);
    });
}

}  // extern "C"
