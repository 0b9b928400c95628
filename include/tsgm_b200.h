/* tsgm_b200 — C-ABI of the B200-native per-frame hot path of arXiv 1809.07986
 * ("tsgm": temporal, Kalman-filtered, reduced-space semi-global matching).
 *
 * This is the drop-in boundary. The reference (/root/reference/proj) is a C++20
 * library whose per-frame entry point is
 *     tsgm::StepResult tsgm::step(const DisparityState&, const GrayImage& left,
 *         const GrayImage& right, const RigidMotion&, const StereoCalib&,
 *         const SgmParams&, const FilterConfig&, int threads)
 *   (include/tsgm/temporal_filter.hpp:71-76, src/temporal_filter.cpp:195-232).
 * Its C++ callers keep using that signature through the header-only facade
 * include/tsgm_gpu.hpp (tsgm::gpu::step), which sits on these functions; a
 * batched production caller uses the context API directly. No torch types, no
 * C++ types: plain pointers and sizes.
 *
 * Status codes (the reference's exception classes):
 *   0 = ok, 1 = invalid argument (std::invalid_argument), 2 = CUDA/runtime
 *   error (std::runtime_error). The message of the last failure on the calling
 *   thread is returned by tsgm_last_error().
 *
 * Layouts: images row-major W x H, index y*W + x; ragged cost volumes use the
 * reference's prefix-sum layout (include/tsgm/matching_cost.hpp:50-73):
 * offsets[W*H+1] (u32), cell (x, y, lo+j) at offsets[y*W+x] + j.
 */
#ifndef TSGM_B200_H
#define TSGM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TSGM_OK 0
#define TSGM_INVALID_ARGUMENT 1
#define TSGM_RUNTIME_ERROR 2

/* tsgm::SgmParams (include/tsgm/sgm.hpp:15-23). path_set: 0 = nondiagonal
 * {left,right,up,down}, 1 = diagonal (sgm.hpp:10-13); used when paths == 4. */
typedef struct {
    int32_t p1, p2, paths, path_set, d_max;
} tsgm_sgm_params;

/* tsgm::FilterConfig (include/tsgm/temporal_filter.hpp:8-26). */
typedef struct {
    double q, r;           /* NoiseParams (temporal_filter.hpp:8-13) */
    double p_init, disc_thresh;
    int32_t min_range_halfwidth;
    int32_t range_use_stddev; /* bool */
    double range_stddev_gain;
} tsgm_filter_config;

/* tsgm::StereoCalib (include/tsgm/geometry.hpp:17-27). */
typedef struct {
    double focal_px, cx, cy, baseline_m;
    int32_t width, height, d_max;
} tsgm_stereo_calib;

/* ------------------------------------------------------------------------
 * Context API — one context per GPU, `max_slots` independent sequences with
 * device-resident Kalman state (A2, geometry.hpp:53-75), one CUDA stream.
 * ------------------------------------------------------------------------ */
typedef struct tsgm_ctx tsgm_ctx;

#define TSGM_KEEP_VOLUMES 1u /* materialise C (u8) and S (u16) per slot for fetch */
#define TSGM_FORCE_SCANLINE_AGG 2u /* use the per-direction scanline aggregation kernels */
/* Extension A22 (NOT in the reference, a declared non-goal: SPEC.md:231):
 * sub-pixel disparity by a parabola through S(d-1), S(d), S(d+1) around the
 * WTA minimum, f32, exported only (never fed back into the Kalman state). */
#define TSGM_SUBPIXEL 4u
/* Record a CUDA event at the end of every stage of each step, so that
 * tsgm_last_stage_timings() can report StepResult::timings. */
#define TSGM_STAGE_TIMINGS 8u

/* StepTimings (temporal_filter.hpp:57-62) with its SgmStageTimings
 * (sgm.hpp:59-64) flattened: seconds of DEVICE time per stage, measured with
 * CUDA events on the context stream (the reference times each stage with
 * steady_clock, temporal_filter.cpp:209-221, sgm.cpp:236-255). Stage map of
 * the GPU pipeline: predict = warp + tie-break + variance + reject + fill;
 * ranges = derive_search_ranges; census; cost = make_cost_volume offsets +
 * matching costs; aggregate = the 8 (or 4) path scans; wta = the direction
 * sum fused with winner_takes_all (the production step never materialises
 * S); correct = correct + diff + mask + render + export median (the
 * reference times correct() alone and leaves diff/median untimed). */
typedef struct {
    double predict_s, ranges_s;
    double census_s, cost_s, aggregate_s, wta_s; /* SgmStageTimings */
    double correct_s;
} tsgm_stage_timings;

typedef struct {
    int32_t width, height;     /* image size (must equal calib.width/height) */
    int32_t max_slots;         /* sequences resident on this device */
    int32_t device;            /* CUDA ordinal */
    tsgm_stereo_calib calib;
    tsgm_sgm_params sgm;
    tsgm_filter_config filter;
    double mask_tau;           /* A21 extension: Mahalanobis gate, 3.0 */
    uint32_t flags;            /* TSGM_KEEP_VOLUMES | TSGM_FORCE_SCANLINE_AGG | TSGM_SUBPIXEL |
                                  TSGM_STAGE_TIMINGS */
    /* Volume working set: how many sequences' per-frame volumes (C, S and the
     * per-direction path costs, up to ~9 B per cell of W*H*d_max) are resident
     * at once. The Kalman state and per-pixel outputs are always resident for
     * all max_slots; a step over more sequences than vol_slots runs the
     * matching stages in balanced chunks. 0 = auto: max_slots, capped to what
     * fits the device's free memory (config 4: 2048x1024, D=256, 32 sequences
     * needs ~6 GB of volumes per sequence). */
    int32_t vol_slots;
} tsgm_config;

const char* tsgm_last_error(void);

/* Validates like step() would (temporal_filter.cpp:198-206, sgm.cpp:14-23,
 * geometry.cpp:21-28) and allocates all device buffers up front. */
int tsgm_create(const tsgm_config* cfg, tsgm_ctx** out);
void tsgm_destroy(tsgm_ctx* ctx);

/* Empty (default) state for `slot`: the next step is full-range matching
 * (temporal_filter.cpp:200-202). */
int tsgm_reset(tsgm_ctx* ctx, int32_t slot);
/* Host -> device state upload (DisparityState; d/p may be NULL for zeros). */
int tsgm_set_state(tsgm_ctx* ctx, int32_t slot, const double* d, const double* p,
                   const uint8_t* valid);

/* One frame for `n` sequences. left[i]/right[i] are HOST u8 W*H images for
 * slots[i]; motion[i*12 .. i*12+11] is the RigidMotion (row-major R, then t)
 * mapping the previous camera frame into the current one (geometry.hpp:29-40).
 * Asynchronous on the context stream w.r.t. the caller except for the host
 * staging copy; outputs stay on the device until tsgm_fetch. */
int tsgm_step(tsgm_ctx* ctx, int32_t n, const int32_t* slots, const uint8_t* const* left,
              const uint8_t* const* right, const double* motion);
/* Same with DEVICE image pointers (inputs already resident in HBM). The
 * step runs on the context's own stream and is NOT ordered after any other
 * stream: the images must be complete before the call and must stay
 * unmodified until the step's census has read them (tsgm_sync, or
 * tsgm_inputs_consumed below). */
int tsgm_step_device(tsgm_ctx* ctx, int32_t n, const int32_t* slots,
                     const uint8_t* const* d_left, const uint8_t* const* d_right,
                     const double* motion);
/* tsgm_step_device ordered after all work enqueued so far on
 * `producer_stream` (a cudaStream_t; NULL = the legacy default stream), e.g.
 * the copy or kernel that produced the images. */
int tsgm_step_device_after(tsgm_ctx* ctx, int32_t n, const int32_t* slots,
                           const uint8_t* const* d_left, const uint8_t* const* d_right,
                           const double* motion, void* producer_stream);
/* Makes `consumer_stream` (a cudaStream_t) wait until the last step has
 * finished reading its input images (its census), so the caller may refill
 * them on that stream without a host synchronisation. */
int tsgm_inputs_consumed(tsgm_ctx* ctx, void* consumer_stream);
/* Names of the aggregation kernels (scan + direction sum/WTA) the last step
 * chose for its batch size and windows, e.g. "scan_kernel<32,32>+
 * combine_wta_kernel<8,1>" (tests and bench.py record which variant ran). */
int tsgm_last_kernels(tsgm_ctx* ctx, char* buf, size_t cap);
/* Volume chunks the last step ran its cost -> aggregation -> WTA stages in.
 * Volumes are packed by the frame's actual cell counts (make_cost_volume's
 * N, matching_cost.cpp:30-48) into a pool of tsgm_volume_slots worst-case
 * volumes, so reduced frames usually need one chunk. */
int tsgm_last_chunks(tsgm_ctx* ctx, int32_t* chunks);
/* Per-stage device time of the context's last step (whole batch), for a
 * context created with TSGM_STAGE_TIMINGS; waits for that step. */
int tsgm_last_stage_timings(tsgm_ctx* ctx, tsgm_stage_timings* out);

/* Outputs of the last step of a slot (StepResult, temporal_filter.hpp:64-69,
 * plus the intermediates parity tests compare). */
enum {
    TSGM_OUT_STATE_D = 0,   /* f64 posterior d        */
    TSGM_OUT_STATE_P = 1,   /* f64 posterior p        */
    TSGM_OUT_STATE_VALID = 2, /* u8                   */
    TSGM_OUT_EXPORT_D = 3,  /* i32 median-refined map (export_map.d) */
    TSGM_OUT_EXPORT_VALID = 4, /* u8 */
    TSGM_OUT_DIFF = 5,      /* f64 |d_pred - d_z|     */
    TSGM_OUT_MASK = 6,      /* u8 A21 moving-object mask */
    TSGM_OUT_PRED_D = 7,    /* f64 predict() output   */
    TSGM_OUT_PRED_P = 8,
    TSGM_OUT_PRED_VALID = 9,
    TSGM_OUT_LO = 10,       /* u16 derive_search_ranges */
    TSGM_OUT_HI = 11,
    TSGM_OUT_MEAS_D = 12,   /* i32 WTA (sgm_match)    */
    TSGM_OUT_MEAS_VALID = 13,
    TSGM_OUT_OFFSETS = 14,  /* u32 W*H+1              */
    TSGM_OUT_COST = 15,     /* u8 N   (TSGM_KEEP_VOLUMES; slot in the last volume chunk) */
    TSGM_OUT_AGG = 16,      /* u16 N  (TSGM_KEEP_VOLUMES; slot in the last volume chunk) */
    TSGM_OUT_SUBPIXEL = 17, /* f32 sub-pixel WTA disparity (TSGM_SUBPIXEL), 0 where invalid */
    TSGM_OUT_COUNT
};
/* Copies output `what` of `slot` into host memory `dst` (bytes >= size). */
int tsgm_fetch(tsgm_ctx* ctx, int32_t slot, int32_t what, void* dst, size_t bytes);
/* Asynchronous batched fetch: enqueues the device-to-host copies of output
 * `what` for n slots into dsts[i] (pinned host memory for true overlap) on the
 * context stream and returns; tsgm_sync() completes them. Not for COST/AGG. */
int tsgm_fetch_batch(tsgm_ctx* ctx, int32_t n, const int32_t* slots, int32_t what,
                     void* const* dsts, size_t bytes_each);
/* Number of cost cells N of the slot's last step (sum of window lengths). */
int tsgm_cells(tsgm_ctx* ctx, int32_t slot, uint64_t* n_cells);
int tsgm_sync(tsgm_ctx* ctx);

/* Timing on the context stream (CUDA events): begin/end bracket a region,
 * elapsed returns milliseconds. Aggregation-only standalone benchmark
 * (C -> S, the graded roofline kernel): runs the 8-path aggregation on the
 * slots' current C volumes `reps` times and returns the mean ms per launch. */
int tsgm_timer_begin(tsgm_ctx* ctx);
int tsgm_timer_end(tsgm_ctx* ctx, float* ms);
int tsgm_bench_aggregate(tsgm_ctx* ctx, int32_t n, const int32_t* slots, int32_t reps,
                         float* ms_per_launch, uint64_t* cells);
/* Volume working set chosen at creation (see tsgm_config.vol_slots). */
int tsgm_volume_slots(tsgm_ctx* ctx, int32_t* vol_slots);
/* Kernel launches issued by the context since creation (all stages). */
uint64_t tsgm_launch_count(tsgm_ctx* ctx);

/* ------------------------------------------------------------------------
 * Stage API — stateless, host buffers in and out, same kernels as the step.
 * One function per public reference sub-stage.
 * ------------------------------------------------------------------------ */
/* census_transform (matching_cost.hpp:80, matching_cost.cpp:53-79) */
int tsgm_census_transform(const uint8_t* img, int32_t w, int32_t h, uint32_t* sig);
/* build_cost_volume (matching_cost.hpp:85-88, matching_cost.cpp:88-117);
 * offsets: W*H+1 u32, cost: capacity `cap` bytes. */
int tsgm_build_cost_volume(const uint8_t* left, const uint8_t* right, int32_t w, int32_t h,
                           const uint16_t* lo, const uint16_t* hi, uint32_t* offsets,
                           uint8_t* cost, uint64_t cap);
/* aggregate_paths (sgm.hpp:47, sgm.cpp:135-161) over a ragged C volume. */
int tsgm_aggregate_paths(const uint8_t* cost, const uint16_t* lo, const uint16_t* hi, int32_t w,
                         int32_t h, const tsgm_sgm_params* params, uint16_t* agg);
/* winner_takes_all (sgm.hpp:52, sgm.cpp:163-187) */
int tsgm_winner_takes_all(const uint16_t* agg, const uint16_t* lo, const uint16_t* hi,
                          int32_t w, int32_t h, int32_t* d, uint8_t* valid);
/* median_refine (sgm.hpp:57, sgm.cpp:189-216) */
int tsgm_median_refine(const int32_t* d, const uint8_t* valid, int32_t w, int32_t h,
                       int32_t* out_d, uint8_t* out_valid);
/* sgm_match (sgm.hpp:67-69, sgm.cpp:226-257) */
int tsgm_sgm_match(const uint8_t* left, const uint8_t* right, int32_t w, int32_t h,
                   const uint16_t* lo, const uint16_t* hi, const tsgm_sgm_params* params,
                   int32_t* d, uint8_t* valid);
/* sgm_match with its SgmStageTimings* argument (sgm.hpp:67-69): census_s,
 * cost_s, aggregate_s, wta_s filled (the other fields 0); may be NULL. */
int tsgm_sgm_match_t(const uint8_t* left, const uint8_t* right, int32_t w, int32_t h,
                     const uint16_t* lo, const uint16_t* hi, const tsgm_sgm_params* params,
                     int32_t* d, uint8_t* valid, tsgm_stage_timings* timings);
/* relative_motion (geometry.hpp:111, geometry.cpp:189-197); poses row-major 3x4 */
int tsgm_relative_motion(const double* prev12, const double* cur12, double* r9, double* t3);
/* disparity_homography (geometry.hpp:87, geometry.cpp:77-110); row-major 4x4 */
int tsgm_disparity_homography(const double* r9, const double* t3,
                              const tsgm_stereo_calib* calib, double* h16);
/* warp_state_ex (geometry.hpp:102, geometry.cpp:127-156) */
int tsgm_warp_state_ex(const double* d, const double* p, const uint8_t* valid, int32_t w,
                       int32_t h, const double* h16, int32_t d_max, double* od, double* op,
                       uint8_t* ov, double* source_d);
/* predict (temporal_filter.hpp:32-33, temporal_filter.cpp:28-49) */
int tsgm_predict(const double* d, const double* p, const uint8_t* valid, int32_t w, int32_t h,
                 const double* r9, const double* t3, const tsgm_stereo_calib* calib,
                 const tsgm_filter_config* cfg, double* od, double* op, uint8_t* ov);
/* reject_discontinuities (temporal_filter.hpp:38, temporal_filter.cpp:51-74) */
int tsgm_reject_discontinuities(const double* d, const double* p, const uint8_t* valid,
                                int32_t w, int32_t h, const tsgm_filter_config* cfg, double* od,
                                double* op, uint8_t* ov);
/* fill_zoom_holes (temporal_filter.hpp:43, temporal_filter.cpp:76-106) */
int tsgm_fill_zoom_holes(const double* d, const double* p, const uint8_t* valid, int32_t w,
                         int32_t h, double* od, double* op, uint8_t* ov);
/* derive_search_ranges (temporal_filter.hpp:48-49, temporal_filter.cpp:108-143) */
int tsgm_derive_search_ranges(const double* d, const double* p, const uint8_t* valid, int32_t w,
                              int32_t h, const tsgm_stereo_calib* calib,
                              const tsgm_filter_config* cfg, uint16_t* lo, uint16_t* hi);
/* correct (temporal_filter.hpp:54-55, temporal_filter.cpp:145-170) */
int tsgm_correct(const double* d, const double* p, const uint8_t* valid, const int32_t* md,
                 const uint8_t* mv, int32_t w, int32_t h, const tsgm_filter_config* cfg,
                 double* od, double* op, uint8_t* ov);

/* step (temporal_filter.hpp:74-76) for ONE sequence with host-resident state,
 * exactly the reference's value semantics: state_w == state_h == 0 is the
 * default (empty) state. Used by the C++ facade. Optional outputs may be NULL. */
int tsgm_step_once(const double* sd, const double* sp, const uint8_t* sv, int32_t state_w,
                   int32_t state_h, const uint8_t* left, const uint8_t* right, int32_t w,
                   int32_t h, const double* r9, const double* t3,
                   const tsgm_stereo_calib* calib, const tsgm_sgm_params* params,
                   const tsgm_filter_config* cfg, double* od, double* op, uint8_t* ov,
                   int32_t* ed, uint8_t* ev, double* diff);
/* tsgm_step_once that also fills StepResult::timings (may be NULL). */
int tsgm_step_once_t(const double* sd, const double* sp, const uint8_t* sv, int32_t state_w,
                     int32_t state_h, const uint8_t* left, const uint8_t* right, int32_t w,
                     int32_t h, const double* r9, const double* t3,
                     const tsgm_stereo_calib* calib, const tsgm_sgm_params* params,
                     const tsgm_filter_config* cfg, double* od, double* op, uint8_t* ov,
                     int32_t* ed, uint8_t* ev, double* diff, tsgm_stage_timings* timings);

/* ------------------------------------------------------------------------
 * Moving-object box detector on the diff map (
 * include/tsgm/motion_detect.hpp, src/motion_detect.cpp). The summed-area
 * table and the candidate-window scoring run on the GPU; the greedy merge runs
 * on the host (exact, incremental). Results equal the reference's.
 * ------------------------------------------------------------------------ */
/* DetectionBox (motion_detect.hpp:24-34): half-open [x0,x1) x [y0,y1), score =
 * mean |disparity difference| inside. */
typedef struct {
    int32_t x0, y0, x1, y1;
    double score;
} tsgm_box;

/* DetectConfig (motion_detect.hpp:36-44): window_wh holds n_windows (w, h)
 * pairs (at most 16); defaults {20,20},{30,30},{40,40},{50,50},{50,75}, 2.0,
 * 0.2, 400. Validated like DetectConfig::validate (motion_detect.cpp:11-23). */
typedef struct {
    const int32_t* window_wh;
    int32_t n_windows;
    double score_thresh;
    double merge_stop_iou;
    int64_t min_box_area;
} tsgm_detect_config;

/* integral_image (motion_detect.hpp:46, motion_detect.cpp:25-42): sat holds
 * (h+1) x (w+1) doubles, zero first row and column. */
int tsgm_integral_image(const double* map, int32_t w, int32_t h, double* sat);
/* detect_candidate_windows (motion_detect.hpp:56-57): writes min(cap, count)
 * boxes in (size, row, column) order; *n_out = count. */
int tsgm_detect_candidate_windows(const double* diff, int32_t w, int32_t h,
                                  const tsgm_detect_config* cfg, tsgm_box* out, int64_t cap,
                                  int64_t* n_out);
/* greedy_merge (motion_detect.hpp:63): in place on the host; *n_out = survivors. */
int tsgm_greedy_merge(tsgm_box* boxes, int64_t n, const tsgm_detect_config* cfg, int64_t* n_out);
/* detect_moving_objects (motion_detect.hpp:68-69) = merge(candidates). */
int tsgm_detect_moving_objects(const double* diff, int32_t w, int32_t h,
                               const tsgm_detect_config* cfg, tsgm_box* out, int64_t cap,
                               int64_t* n_out);
/* Batched: detect_moving_objects on the diff maps of the context's last step
 * for n slots; slot i's boxes go to out[i*cap_each ..], their count (which
 * may exceed cap_each: then only cap_each are written) to n_each[i]. */
int tsgm_detect(tsgm_ctx* ctx, int32_t n, const int32_t* slots, const tsgm_detect_config* cfg,
                tsgm_box* out, int64_t cap_each, int64_t* n_each);

/* ------------------------------------------------------------------------
 * KITTI-style outlier count of a disparity map against ground truth
 * (include/tsgm/eval.hpp:13-42, src/eval.cpp:59-93).
 * ------------------------------------------------------------------------ */
/* OutlierOptions (eval.hpp:13-19); defaults 3.0, 0.05, 0. */
typedef struct {
    double abs_thresh_px;
    double rel_thresh;
    int32_t strict_density;
} tsgm_outlier_options;

/* count_outliers (eval.cpp:59-85) on the GPU: GT valid iff gt > 0; outlier iff
 * |d - gt| > abs AND |d - gt| / gt > rel. */
int tsgm_count_outliers(const int32_t* d, const uint8_t* valid, const double* gt, int32_t w,
                        int32_t h, const tsgm_outlier_options* opts, int64_t* evaluated,
                        int64_t* outliers);
/* Batched on the context's last step: output `what` (TSGM_OUT_EXPORT_D or
 * TSGM_OUT_MEAS_D, with its validity) of n slots against host GT maps gt[i]. */
int tsgm_count_outliers_batch(tsgm_ctx* ctx, int32_t n, const int32_t* slots, int32_t what,
                              const double* const* gt, const tsgm_outlier_options* opts,
                              int64_t* evaluated, int64_t* outliers);

/* ------------------------------------------------------------------------
 * Noise calibration on the GPU: the reference's
 * estimate_process_noise / estimate_measurement_noise / accumulate_error_map
 * (noise_calib.hpp:52-80, noise_calib.cpp:102-182). The reference passes a
 * std::vector<SequenceFrame> (dataset.hpp:18-25); here n frames are n
 * contiguous W x H maps (gt f64, gt > 0 = valid; images u8) and n row-major
 * 3x4 camera-to-world poses (Pose, geometry.hpp:106). Counts are exact; the
 * gated FP64 moments use a fixed GPU reduction order (deterministic, equal to
 * the reference's raster-order sums up to FP64 reassociation).
 * ------------------------------------------------------------------------ */
/* CalibOptions (noise_calib.hpp:43-49) */
typedef struct {
    double outlier_gate_px, bin_width, q_floor;
} tsgm_calib_options;

/* NoiseEstimate + its ErrorHistogram (noise_calib.hpp:14-41, 51-55). */
typedef struct {
    double variance;          /* raw unbiased variance of the gated samples */
    int64_t samples_used;     /* gated samples */
    double lo, hi, bin_width; /* histogram layout: [-gate, gate) */
    int64_t underflow, overflow, within_1px, total;
    double sum, sum_sq;       /* gated moments */
    int32_t n_bins;           /* in: capacity of counts; out: number of bins */
    int64_t* counts;          /* caller buffer of tsgm_calib_bins() entries */
} tsgm_noise_estimate;

/* Number of histogram bins, ceil(2 * gate / bin_width); validates the options
 * like CalibOptions::validate (noise_calib.cpp:60-67). */
int tsgm_calib_bins(const tsgm_calib_options* opts, int32_t* n_bins);
/* estimate_process_noise (noise_calib.cpp:102-128): n >= 2 frames. */
int tsgm_estimate_process_noise(int32_t n_frames, int32_t w, int32_t h, const double* gt,
                                const double* poses12, const tsgm_stereo_calib* calib,
                                const tsgm_calib_options* opts, tsgm_noise_estimate* out);
/* estimate_measurement_noise (noise_calib.cpp:130-147): full-range SGM per
 * frame, every frame matched in isolation (batched on the GPU). */
int tsgm_estimate_measurement_noise(int32_t n_frames, int32_t w, int32_t h, const uint8_t* left,
                                    const uint8_t* right, const double* gt,
                                    const tsgm_sgm_params* params, const tsgm_calib_options* opts,
                                    tsgm_noise_estimate* out);
/* The calibration functions keep their device working set (a batch of frames'
 * state, maps and volumes) between calls with the same geometry; this frees
 * it. */
int tsgm_calib_release(void);
/* accumulate_error_map (noise_calib.cpp:149-182): acc[W*H], bit-exact. */
int tsgm_accumulate_error_map(int32_t n_frames, int32_t w, int32_t h, const double* gt,
                              const double* poses12, const tsgm_stereo_calib* calib, double* acc);

/* ------------------------------------------------------------------------
 * Export formats (dataset.hpp:51-59, dataset.cpp:229-269):
 * the KITTI 16-bit disparity PNG (round(256 d), 0 = invalid; a value that
 * does not fit fails with the reference's message at the first such pixel in
 * raster order) and boxes.txt. The quantisation runs on the GPU; the PNG
 * container (16-bit grayscale, zlib) is written on the host.
 * ------------------------------------------------------------------------ */
/* write_disparity_png(const Image<double>&)'s 16-bit image, no file */
int tsgm_quantize_disparity(const double* disp, int32_t w, int32_t h, uint16_t* raw);
/* write_disparity_png(const DisparityMap&)'s 16-bit image, no file */
int tsgm_quantize_disparity_map(const int32_t* d, const uint8_t* valid, int32_t w, int32_t h,
                                uint16_t* raw);
int tsgm_write_disparity_png(const char* path, const double* disp, int32_t w, int32_t h);
int tsgm_write_disparity_png_map(const char* path, const int32_t* d, const uint8_t* valid,
                                 int32_t w, int32_t h);
/* The slot's export map (StepResult::export_map) straight from the device, as
 * tsgm_main's run command writes it (tsgm_main.cpp:157). */
int tsgm_write_export_png(tsgm_ctx* ctx, int32_t slot, const char* path);
/* n slots at once: one device quantisation, PNGs encoded on host threads */
int tsgm_write_export_pngs(tsgm_ctx* ctx, int32_t n, const int32_t* slots,
                           const char* const* paths);
/* read_disparity_png (dataset.cpp:220-227): a 16-bit grayscale PNG (any row
 * filter) as samples / 256 (0 = invalid); host-side. Call with disp = NULL to
 * get w, h; then with a buffer of cap >= w*h doubles. */
int tsgm_read_disparity_png(const char* path, int32_t* w, int32_t* h, double* disp, size_t cap);
/* write_boxes: boxes of n_frames frames back to back, counts[f] per frame */
int tsgm_write_boxes(const char* path, const tsgm_box* boxes, const int64_t* counts,
                     int32_t n_frames);

#ifdef __cplusplus
}
#endif
#endif
