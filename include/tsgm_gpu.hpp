// tsgm::gpu — header-only C++ facade with the reference's own signatures and
// types, running on the B200 through the C-ABI in tsgm_b200.h.
//
// Drop-in use: a caller of the reference library (/root/reference/proj)
// includes this header next to "tsgm/temporal_filter.hpp" and replaces
//     tsgm::step(state, left, right, motion, calib, params, cfg, threads)
// with
//     tsgm::gpu::step(state, left, right, motion, calib, params, cfg, threads)
// (temporal_filter.hpp:74-76). Results are bit-identical (DESIGN.md,
// "Parity"). Errors are rethrown as the reference's exception types:
// status 1 -> std::invalid_argument, 2 -> std::runtime_error. `threads` is
// accepted and ignored (the GPU grid replaces parallel_rows).
//
// For many sequences use tsgm::gpu::Engine: device-resident state per slot,
// one batched launch sequence per frame.
#pragma once

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "tsgm/dataset.hpp"
#include "tsgm/geometry.hpp"
#include "tsgm/matching_cost.hpp"
#include "tsgm/motion_detect.hpp"
#include "tsgm/noise_calib.hpp"
#include "tsgm/sgm.hpp"
#include "tsgm/temporal_filter.hpp"
#include "tsgm_b200.h"

namespace tsgm {
namespace gpu {

namespace detail {

inline void check(int rc) {
    if (rc == TSGM_OK) return;
    const std::string msg = tsgm_last_error();
    if (rc == TSGM_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

inline tsgm_sgm_params to_c(const SgmParams& p) {
    return tsgm_sgm_params{p.p1, p.p2, p.paths, p.path_set == PathSet::diagonal ? 1 : 0,
                           p.d_max};
}
inline tsgm_filter_config to_c(const FilterConfig& f) {
    return tsgm_filter_config{f.noise.q, f.noise.r, f.p_init, f.disc_thresh,
                              f.min_range_halfwidth, f.range_use_stddev ? 1 : 0,
                              f.range_stddev_gain};
}
inline tsgm_stereo_calib to_c(const StereoCalib& c) {
    return tsgm_stereo_calib{c.focal_px, c.cx, c.cy, c.baseline_m, c.width, c.height, c.d_max};
}
inline void to_timings(const tsgm_stage_timings& t, StepTimings& out) {
    out.predict_s = t.predict_s;
    out.ranges_s = t.ranges_s;
    out.sgm.census_s = t.census_s;
    out.sgm.cost_s = t.cost_s;
    out.sgm.aggregate_s = t.aggregate_s;
    out.sgm.wta_s = t.wta_s;
    out.correct_s = t.correct_s;
}
inline void motion12(const RigidMotion& m, double* r9, double* t3) {
    for (int i = 0; i < 3; ++i) {
        for (int j = 0; j < 3; ++j) r9[i * 3 + j] = m.rotation(i, j);
        t3[i] = m.translation(i);
    }
}

}  // namespace detail

// step (temporal_filter.hpp:74-76, temporal_filter.cpp:195-232)
inline StepResult step(const DisparityState& state, const GrayImage& left,
                       const GrayImage& right, const RigidMotion& motion,
                       const StereoCalib& calib, const SgmParams& params,
                       const FilterConfig& cfg, int threads = 1) {
    (void)threads;
    if (!left.same_size(right)) throw std::invalid_argument("step: left/right dimension mismatch");
    const int w = left.width(), h = left.height();
    double r9[9], t3[3];
    detail::motion12(motion, r9, t3);
    const tsgm_stereo_calib c = detail::to_c(calib);
    const tsgm_sgm_params p = detail::to_c(params);
    const tsgm_filter_config f = detail::to_c(cfg);
    StepResult res;
    res.state = DisparityState(w, h);
    res.export_map = DisparityMap(w, h);
    res.diff = Image<double>(w, h, 0.0);
    // StepResult::timings: per-stage device seconds (tsgm_stage_timings)
    tsgm_stage_timings t{};
    detail::check(tsgm_step_once_t(state.d.data(), state.p.data(), state.valid.data(),
                                   state.width(), state.height(), left.data(), right.data(), w, h,
                                   r9, t3, &c, &p, &f, res.state.d.data(), res.state.p.data(),
                                   res.state.valid.data(), res.export_map.d.data(),
                                   res.export_map.valid.data(), res.diff.data(), &t));
    detail::to_timings(t, res.timings);
    return res;
}

// census_transform (matching_cost.hpp:80)
inline CensusMap census_transform(const GrayImage& img, int threads = 1) {
    (void)threads;
    CensusMap m{Image<std::uint32_t>(img.width(), img.height())};
    detail::check(tsgm_census_transform(img.data(), img.width(), img.height(), m.sig.data()));
    return m;
}

// sgm_match (sgm.hpp:67-69); `timings` gets per-stage device seconds
inline DisparityMap sgm_match(const GrayImage& left, const GrayImage& right,
                              const SearchRangeMap& ranges, const SgmParams& params,
                              int threads = 1, SgmStageTimings* timings = nullptr) {
    (void)threads;
    if (!left.same_size(right)) throw std::invalid_argument("sgm_match: image size mismatch");
    if (!left.same_size(ranges.lo)) throw std::invalid_argument("sgm_match: range map size mismatch");
    DisparityMap dm(left.width(), left.height());
    const tsgm_sgm_params p = detail::to_c(params);
    tsgm_stage_timings t{};
    detail::check(tsgm_sgm_match_t(left.data(), right.data(), left.width(), left.height(),
                                   ranges.lo.data(), ranges.hi.data(), &p, dm.d.data(),
                                   dm.valid.data(), timings ? &t : nullptr));
    if (timings) {
        timings->census_s = t.census_s;
        timings->cost_s = t.cost_s;
        timings->aggregate_s = t.aggregate_s;
        timings->wta_s = t.wta_s;
    }
    return dm;
}

// aggregate_paths (sgm.hpp:47) over a reference MatchingCostVolume
inline AggregatedCostVolume aggregate_paths(const MatchingCostVolume& vol, const SgmParams& params) {
    AggregatedCostVolume agg;
    agg.ranges = vol.ranges;
    agg.offsets = vol.offsets;
    agg.cost.assign(vol.cost.size(), 0);
    const tsgm_sgm_params p = detail::to_c(params);
    detail::check(tsgm_aggregate_paths(vol.cost.data(), vol.ranges.lo.data(),
                                       vol.ranges.hi.data(), vol.width(), vol.height(), &p,
                                       agg.cost.data()));
    return agg;
}

// winner_takes_all (sgm.hpp:52)
inline DisparityMap winner_takes_all(const AggregatedCostVolume& agg, int threads = 1) {
    (void)threads;
    DisparityMap dm(agg.width(), agg.height());
    detail::check(tsgm_winner_takes_all(agg.cost.data(), agg.ranges.lo.data(),
                                        agg.ranges.hi.data(), agg.width(), agg.height(),
                                        dm.d.data(), dm.valid.data()));
    return dm;
}

// median_refine (sgm.hpp:57)
inline DisparityMap median_refine(const DisparityMap& dm, int threads = 1) {
    (void)threads;
    DisparityMap out(dm.width(), dm.height());
    detail::check(tsgm_median_refine(dm.d.data(), dm.valid.data(), dm.width(), dm.height(),
                                     out.d.data(), out.valid.data()));
    return out;
}

// predict (temporal_filter.hpp:32-33)
inline DisparityState predict(const DisparityState& state, const RigidMotion& motion,
                              const StereoCalib& calib, const FilterConfig& cfg) {
    double r9[9], t3[3];
    detail::motion12(motion, r9, t3);
    const tsgm_stereo_calib c = detail::to_c(calib);
    const tsgm_filter_config f = detail::to_c(cfg);
    DisparityState out(state.width(), state.height());
    detail::check(tsgm_predict(state.d.data(), state.p.data(), state.valid.data(), state.width(),
                               state.height(), r9, t3, &c, &f, out.d.data(), out.p.data(),
                               out.valid.data()));
    return out;
}

// derive_search_ranges (temporal_filter.hpp:48-49)
inline SearchRangeMap derive_search_ranges(const DisparityState& state, const StereoCalib& calib,
                                           const FilterConfig& cfg) {
    const tsgm_stereo_calib c = detail::to_c(calib);
    const tsgm_filter_config f = detail::to_c(cfg);
    SearchRangeMap r(state.width(), state.height(), 0, 0);
    detail::check(tsgm_derive_search_ranges(state.d.data(), state.p.data(), state.valid.data(),
                                            state.width(), state.height(), &c, &f, r.lo.data(),
                                            r.hi.data()));
    return r;
}

// correct (temporal_filter.hpp:54-55)
inline DisparityState correct(const DisparityState& pred, const DisparityMap& meas,
                              const FilterConfig& cfg) {
    if (!pred.valid.same_size(meas.valid)) throw std::invalid_argument("correct: dimension mismatch");
    const tsgm_filter_config f = detail::to_c(cfg);
    DisparityState out(pred.width(), pred.height());
    detail::check(tsgm_correct(pred.d.data(), pred.p.data(), pred.valid.data(), meas.d.data(),
                               meas.valid.data(), pred.width(), pred.height(), &f, out.d.data(),
                               out.p.data(), out.valid.data()));
    return out;
}

// ---- box detector (motion_detect.hpp:46-72): SAT + scoring on the GPU,
// greedy merge on the host; results equal the reference's.
namespace detail {
struct DetectC {
    std::vector<std::int32_t> wh;
    tsgm_detect_config c{};
    explicit DetectC(const DetectConfig& cfg) {
        for (const auto& [w, h] : cfg.window_sizes) {
            wh.push_back(w);
            wh.push_back(h);
        }
        c.window_wh = wh.data();
        c.n_windows = static_cast<std::int32_t>(cfg.window_sizes.size());
        c.score_thresh = cfg.score_thresh;
        c.merge_stop_iou = cfg.merge_stop_iou;
        c.min_box_area = cfg.min_box_area;
    }
};
inline std::vector<DetectionBox> to_boxes(const std::vector<tsgm_box>& v, std::int64_t n) {
    std::vector<DetectionBox> out;
    for (std::int64_t i = 0; i < n; ++i)
        out.push_back(DetectionBox{v[i].x0, v[i].y0, v[i].x1, v[i].y1, v[i].score});
    return out;
}
template <typename Fn>
std::vector<DetectionBox> boxes_call(Fn fn) {
    std::vector<tsgm_box> buf(4096);
    std::int64_t n = 0;
    check(fn(buf.data(), static_cast<std::int64_t>(buf.size()), &n));
    if (n > static_cast<std::int64_t>(buf.size())) {
        buf.resize(static_cast<size_t>(n));
        check(fn(buf.data(), n, &n));
    }
    return to_boxes(buf, n);
}
}  // namespace detail

inline SummedAreaTable integral_image(const Image<double>& map) {
    SummedAreaTable sat;
    sat.width = map.width();
    sat.height = map.height();
    sat.sum.assign(static_cast<size_t>(sat.height + 1) * (sat.width + 1), 0.0);
    detail::check(tsgm_integral_image(map.data(), map.width(), map.height(), sat.sum.data()));
    return sat;
}

inline std::vector<DetectionBox> detect_candidate_windows(const Image<double>& diff,
                                                          const DetectConfig& cfg,
                                                          int threads = 1) {
    (void)threads;
    const detail::DetectC c(cfg);
    return detail::boxes_call([&](tsgm_box* out, std::int64_t cap, std::int64_t* n) {
        return tsgm_detect_candidate_windows(diff.data(), diff.width(), diff.height(), &c.c, out,
                                             cap, n);
    });
}

inline std::vector<DetectionBox> greedy_merge(std::vector<DetectionBox> boxes,
                                              const DetectConfig& cfg) {
    const detail::DetectC c(cfg);
    std::vector<tsgm_box> v;
    for (const DetectionBox& b : boxes) v.push_back(tsgm_box{b.x0, b.y0, b.x1, b.y1, b.score});
    std::int64_t n = 0;
    detail::check(tsgm_greedy_merge(v.data(), static_cast<std::int64_t>(v.size()), &c.c, &n));
    return detail::to_boxes(v, n);
}

inline std::vector<DetectionBox> detect_moving_objects(const Image<double>& diff,
                                                       const DetectConfig& cfg, int threads = 1) {
    (void)threads;
    const detail::DetectC c(cfg);
    return detail::boxes_call([&](tsgm_box* out, std::int64_t cap, std::int64_t* n) {
        return tsgm_detect_moving_objects(diff.data(), diff.width(), diff.height(), &c.c, out,
                                          cap, n);
    });
}

// ---- noise calibration (noise_calib.hpp:57-80) on the GPU ----
namespace detail {
// ErrorHistogram keeps its moments private (noise_calib.hpp:35-40); the
// facade fills them through pointers-to-member obtained by explicit template
// instantiation (which is exempt from access checking), so the returned
// NoiseEstimate behaves exactly like the reference's (mean, variance, total,
// fraction_within_1px).
template <typename Tag, typename Tag::type M>
struct HistAccess {
    friend typename Tag::type member(Tag) { return M; }
};
struct HistNGated { using type = long long ErrorHistogram::*; friend type member(HistNGated); };
struct HistNWithin { using type = long long ErrorHistogram::*; friend type member(HistNWithin); };
struct HistSum { using type = double ErrorHistogram::*; friend type member(HistSum); };
struct HistSumSq { using type = double ErrorHistogram::*; friend type member(HistSumSq); };
template struct HistAccess<HistNGated, &ErrorHistogram::n_gated_>;
template struct HistAccess<HistNWithin, &ErrorHistogram::n_within_1_>;
template struct HistAccess<HistSum, &ErrorHistogram::sum_>;
template struct HistAccess<HistSumSq, &ErrorHistogram::sum_sq_>;

inline tsgm_calib_options to_c(const CalibOptions& o) {
    return tsgm_calib_options{o.outlier_gate_px, o.bin_width, o.q_floor};
}

// frames -> contiguous maps (the reference's own missing-field errors first)
struct CalibFrames {
    int n = 0, w = 0, h = 0;
    std::vector<double> gt, poses;
    std::vector<std::uint8_t> left, right;
    CalibFrames(const std::vector<SequenceFrame>& frames, const char* who, bool need_pose,
                bool images) {
        n = static_cast<int>(frames.size());
        for (const SequenceFrame& f : frames) {
            if (!f.gt_disp)
                throw std::invalid_argument(std::string(who) + ": frame " + std::to_string(f.index) +
                                            " has no GT disparity");
            if (need_pose && !f.pose)
                throw std::invalid_argument(std::string(who) + ": frame " + std::to_string(f.index) +
                                            " has no pose");
        }
        if (frames.empty()) return;
        w = frames[0].gt_disp->width();
        h = frames[0].gt_disp->height();
        const size_t P = static_cast<size_t>(w) * h;
        for (const SequenceFrame& f : frames) {
            if (f.gt_disp->width() != w || f.gt_disp->height() != h ||
                (images && (f.left.width() != w || f.left.height() != h ||
                            f.right.width() != w || f.right.height() != h)))
                throw std::invalid_argument(std::string(who) + ": frame size mismatch");
            gt.insert(gt.end(), f.gt_disp->data(), f.gt_disp->data() + P);
            if (images) {
                left.insert(left.end(), f.left.data(), f.left.data() + P);
                right.insert(right.end(), f.right.data(), f.right.data() + P);
            }
            if (need_pose)
                for (int i = 0; i < 12; ++i) poses.push_back((*f.pose)(i / 4, i % 4));
        }
    }
};

template <typename Call>
inline NoiseEstimate estimate(const CalibOptions& opts, Call&& call) {
    const tsgm_calib_options o = to_c(opts);
    std::int32_t nb = 0;
    check(tsgm_calib_bins(&o, &nb));
    std::vector<std::int64_t> counts(static_cast<size_t>(nb));
    tsgm_noise_estimate e{};
    e.n_bins = nb;
    e.counts = counts.data();
    check(call(&o, &e));
    NoiseEstimate out;
    out.variance = e.variance;
    out.samples_used = e.samples_used;
    out.hist = ErrorHistogram(e.lo, e.hi, e.bin_width);
    out.hist.counts.assign(counts.begin(), counts.end());
    out.hist.underflow = e.underflow;
    out.hist.overflow = e.overflow;
    out.hist.*member(HistNGated{}) = e.samples_used;
    out.hist.*member(HistNWithin{}) = e.within_1px;
    out.hist.*member(HistSum{}) = e.sum;
    out.hist.*member(HistSumSq{}) = e.sum_sq;
    return out;
}
}  // namespace detail

inline NoiseEstimate estimate_process_noise(const std::vector<SequenceFrame>& frames,
                                            const StereoCalib& calib,
                                            const CalibOptions& opts = {}) {
    opts.validate();
    if (frames.size() < 2)
        throw std::invalid_argument("estimate_process_noise: need at least 2 frames");
    const detail::CalibFrames f(frames, "estimate_process_noise", true, false);
    const tsgm_stereo_calib c = detail::to_c(calib);
    return detail::estimate(opts, [&](const tsgm_calib_options* o, tsgm_noise_estimate* e) {
        return tsgm_estimate_process_noise(f.n, f.w, f.h, f.gt.data(), f.poses.data(), &c, o, e);
    });
}

inline NoiseEstimate estimate_measurement_noise(const std::vector<SequenceFrame>& frames,
                                                const SgmParams& params, int threads = 1,
                                                const CalibOptions& opts = {}) {
    (void)threads;
    opts.validate();
    if (frames.empty())
        throw std::invalid_argument("estimate_measurement_noise: need at least 1 frame");
    const detail::CalibFrames f(frames, "estimate_measurement_noise", false, true);
    const tsgm_sgm_params p = detail::to_c(params);
    return detail::estimate(opts, [&](const tsgm_calib_options* o, tsgm_noise_estimate* e) {
        return tsgm_estimate_measurement_noise(f.n, f.w, f.h, f.left.data(), f.right.data(),
                                               f.gt.data(), &p, o, e);
    });
}

inline Image<double> accumulate_error_map(const std::vector<SequenceFrame>& frames,
                                          const StereoCalib& calib) {
    if (frames.size() < 2)
        throw std::invalid_argument("accumulate_error_map: need at least 2 frames");
    const detail::CalibFrames f(frames, "accumulate_error_map", true, false);
    const tsgm_stereo_calib c = detail::to_c(calib);
    Image<double> acc(f.w, f.h, 0.0);
    detail::check(tsgm_accumulate_error_map(f.n, f.w, f.h, f.gt.data(), f.poses.data(), &c,
                                            acc.data()));
    return acc;
}

// ---- export formats (dataset.hpp:51-59) ----
// write_disparity_png: quantised on the GPU, 16-bit grayscale PNG on the host
// (not libpng's bytes; the decoded samples are the reference's).
inline void write_disparity_png(const std::string& path, const Image<double>& disp) {
    detail::check(tsgm_write_disparity_png(path.c_str(), disp.data(), disp.width(), disp.height()));
}
inline void write_disparity_png(const std::string& path, const DisparityMap& dm) {
    detail::check(tsgm_write_disparity_png_map(path.c_str(), dm.d.data(), dm.valid.data(),
                                               dm.d.width(), dm.d.height()));
}
inline Image<double> read_disparity_png(const std::string& path) {
    std::int32_t w = 0, h = 0;
    detail::check(tsgm_read_disparity_png(path.c_str(), &w, &h, nullptr, 0));
    Image<double> img(w, h, 0.0);
    detail::check(tsgm_read_disparity_png(path.c_str(), &w, &h, img.data(), img.pixel_count()));
    return img;
}
inline void write_boxes(const std::string& path,
                        const std::vector<std::vector<DetectionBox>>& per_frame) {
    std::vector<tsgm_box> flat;
    std::vector<std::int64_t> counts;
    for (const auto& f : per_frame) {
        counts.push_back(static_cast<std::int64_t>(f.size()));
        for (const DetectionBox& b : f) flat.push_back(tsgm_box{b.x0, b.y0, b.x1, b.y1, b.score});
    }
    detail::check(tsgm_write_boxes(path.c_str(), flat.data(), counts.data(),
                                   static_cast<std::int32_t>(counts.size())));
}

// Batched, device-resident production path.
class Engine {
public:
    Engine(const StereoCalib& calib, const SgmParams& params, const FilterConfig& cfg,
           int max_slots, int device = 0, double mask_tau = 3.0, unsigned flags = 0,
           int vol_slots = 0) {
        tsgm_config c{};
        c.width = calib.width;
        c.height = calib.height;
        c.max_slots = max_slots;
        c.device = device;
        c.calib = detail::to_c(calib);
        c.sgm = detail::to_c(params);
        c.filter = detail::to_c(cfg);
        c.mask_tau = mask_tau;
        c.flags = flags;
        c.vol_slots = vol_slots;
        detail::check(tsgm_create(&c, &ctx_));
        timed_ = (flags & TSGM_STAGE_TIMINGS) != 0;
        w_ = calib.width;
        h_ = calib.height;
    }
    ~Engine() { tsgm_destroy(ctx_); }
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;

    void reset(int slot) { detail::check(tsgm_reset(ctx_, slot)); }

    // One frame for slots[i] with images lefts[i]/rights[i] and motions[i].
    void step(const std::vector<int>& slots, const std::vector<const GrayImage*>& lefts,
              const std::vector<const GrayImage*>& rights,
              const std::vector<RigidMotion>& motions) {
        const int n = static_cast<int>(slots.size());
        // the C-ABI reads W*H bytes per image: check what step() would
        // (temporal_filter.cpp:198-199) before handing over raw pointers
        if (lefts.size() != slots.size() || rights.size() != slots.size() ||
            motions.size() != slots.size())
            throw std::invalid_argument("Engine::step: slots, images and motions differ in length");
        for (int i = 0; i < n; ++i) {
            if (!lefts[i] || !rights[i]) throw std::invalid_argument("Engine::step: null image");
            if (!lefts[i]->same_size(*rights[i]))
                throw std::invalid_argument("step: left/right dimension mismatch");
            if (lefts[i]->width() != w_ || lefts[i]->height() != h_)
                throw std::invalid_argument("step: state dimension mismatch");
        }
        std::vector<const std::uint8_t*> l(n), r(n);
        std::vector<double> m(12 * static_cast<size_t>(n));
        for (int i = 0; i < n; ++i) {
            l[i] = lefts[i]->data();
            r[i] = rights[i]->data();
            detail::motion12(motions[i], &m[12 * i], &m[12 * i + 9]);
        }
        detail::check(tsgm_step(ctx_, n, slots.data(), l.data(), r.data(), m.data()));
    }

    // Per-stage device time of the last step, whole batch (engine created
    // with flags |= TSGM_STAGE_TIMINGS).
    StepTimings timings() const {
        tsgm_stage_timings t{};
        detail::check(tsgm_last_stage_timings(ctx_, &t));
        StepTimings out;
        detail::to_timings(t, out);
        return out;
    }

    // StepResult of a slot's last frame (state, export map, diff; timings of
    // the batch when the engine records them).
    StepResult result(int slot) const {
        StepResult res;
        res.state = DisparityState(w_, h_);
        res.export_map = DisparityMap(w_, h_);
        res.diff = Image<double>(w_, h_, 0.0);
        fetch(slot, TSGM_OUT_STATE_D, res.state.d.data(), 8);
        fetch(slot, TSGM_OUT_STATE_P, res.state.p.data(), 8);
        fetch(slot, TSGM_OUT_STATE_VALID, res.state.valid.data(), 1);
        fetch(slot, TSGM_OUT_EXPORT_D, res.export_map.d.data(), 4);
        fetch(slot, TSGM_OUT_EXPORT_VALID, res.export_map.valid.data(), 1);
        fetch(slot, TSGM_OUT_DIFF, res.diff.data(), 8);
        if (timed_) res.timings = timings();
        return res;
    }

    // detect_moving_objects on the diff maps of the slots' last frame.
    std::vector<std::vector<DetectionBox>> detect(const std::vector<int>& slots,
                                                  const DetectConfig& cfg) const {
        const detail::DetectC c(cfg);
        const int n = static_cast<int>(slots.size());
        std::int64_t cap = 1024;
        std::vector<std::int64_t> cnt(n);
        std::vector<tsgm_box> buf;
        for (;;) {
            buf.assign(static_cast<size_t>(cap) * n, tsgm_box{});
            detail::check(tsgm_detect(ctx_, n, slots.data(), &c.c, buf.data(), cap, cnt.data()));
            std::int64_t mx = 0;
            for (std::int64_t v : cnt) mx = std::max(mx, v);
            if (mx <= cap) break;
            cap = mx;
        }
        std::vector<std::vector<DetectionBox>> out(n);
        for (int i = 0; i < n; ++i)
            out[i] = detail::to_boxes(std::vector<tsgm_box>(buf.begin() + i * cap,
                                                            buf.begin() + i * cap + cnt[i]),
                                      cnt[i]);
        return out;
    }

    // A21 moving-object mask of a slot's last frame.
    Image<std::uint8_t> mask(int slot) const {
        Image<std::uint8_t> m(w_, h_);
        fetch(slot, TSGM_OUT_MASK, m.data(), 1);
        return m;
    }

private:
    void fetch(int slot, int what, void* dst, size_t elem) const {
        detail::check(tsgm_fetch(ctx_, slot, what, dst, elem * static_cast<size_t>(w_) * h_));
    }
    tsgm_ctx* ctx_ = nullptr;
    int w_ = 0, h_ = 0;
    bool timed_ = false;
};

}  // namespace gpu
}  // namespace tsgm
