// Shared device-side definitions for the tsgm sm_100a kernels.
//
// Batched layout in HBM: every per-pixel map is slot-major, [max_slots][W*H]
// (offsets: [max_slots][W*H+1]); ragged cost volumes live in a pool sized by
// the frame's ACTUAL cell counts: position a of a volume chunk starts at cell
// vbase[a] (prefix of the chunk's ncells), and within it cell (x, y, lo+j)
// sits at off[y*W+x] + j exactly as in the reference's CostVolume
// (include/tsgm/matching_cost.hpp:50-73; make_cost_volume sizes by N too,
// matching_cost.cpp:30-48). A launch
// covers `n` active slots; blockIdx.{y,z} selects the active index a, and
// slots[a] the slot. Per-pixel maps are indexed by the slot, volumes by a
// (the volume stages run in chunks of at most vol_slots sequences).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "../../include/tsgm_b200.h"

namespace tsgm {

constexpr int kCensusRadius = 2;  // matching_cost.hpp:11
constexpr int kMaxCost = 24;      // matching_cost.hpp:13

struct Bufs {
    int W, H, P, d_max;
    size_t vol_cap;  // worst-case cells of one sequence's volume (W*H*d_max)
    // cost, agg and pdir are indexed by the position a of the slot in the
    // launch's batch (a volume chunk), not by the slot: only the per-pixel
    // state and outputs are slot-resident. vol_slots = the pool in worst-case
    // sequences; a chunk holds as many sequences as their actual cells fit.
    int vol_slots;
    const unsigned long long* vbase;   // [position] first cell in cost/agg (volume_plan_kernel)
    const unsigned long long* vqbase;  // [position] first quad in each direction's pdir region
    size_t pool_cells;                 // cells of the cost/agg pools
    size_t pool_quads;                 // quads per direction region of pdir
    const int* slots;  // device [n] slot ids of the active batch
    // posterior state (A2)
    double *sd, *sp;
    uint8_t* sv;
    // warp keys (A6) and warp output (pre reject/fill)
    unsigned long long* kd;  // [slot][P] winning d' key (atomicMax)
    ulonglong2* kps;         // [slot][P] (p key, source-d key), lexicographic min (128-bit CAS)
    int* wtgt;               // [slot][P] pass-1 target pixel of each source (-1: dropped)
    unsigned long long* wdk; // [slot][P] pass-1 d' key of each source
    double *wd, *wp, *wsrc;
    uint8_t* wv;
    // prediction (predict() output)
    double *pd, *pp;
    uint8_t* pv;
    // ranges + prefix sums (A10, A11)
    uint16_t *lo, *hi;
    uint32_t* lohi;      // [slot][P] lo | hi << 16 (packed copy for the aggregation)
    uint32_t* off;       // [slot][P+1]
    uint32_t* row_sum;   // [slot][H]
    uint32_t* qoff;      // [slot][P+1] quad-aligned offsets (aggregation partials)
    uint2* tmeta;        // [slot][W][H] column-major {lohi, qoff} (horizontal scanlines)
    uint2* rmeta;        // [slot][H][W] row-major {lohi, qoff} (the other scanlines)
    uint32_t* qrow_sum;  // [slot][H]
    uint2* tsum;         // [slot][H][ceil(W/32)] (cells, quads) of 32-px tile rows -> tile offsets
    unsigned long long* ncells;  // [slot]
    unsigned long long* nquads;  // [slot]
    int* overflow;       // [slot] volume >= 2^32
    // census + volumes (A12-A14)
    uint32_t *sigl, *sigr;
    const uint8_t* const* left;   // device [n] image pointers
    const uint8_t* const* right;
    uint8_t* cost;   // [pool_cells] (position a at vbase[a]): the reference layout, on demand
    uint32_t* costq; // [pool_quads] (position a at vqbase[a]): quad layout, 0xff outside [lo, hi]
    uint16_t* agg;   // [pool_cells] (position a at vbase[a])
    // scanline-group aggregation: per-direction path costs (u8) in the quad
    // layout (qoff), [dir][pool_quads][4] (position a at vqbase[a])
    uint8_t* pdir;
    size_t quad_cap;  // worst-case quads of one sequence
    int max_slots;
    int num_sms;     // of the context's device (kernel-choice thresholds)
    int* work;
    // WTA, render, export (A15, A18, A19)
    int32_t *md, *rd, *ed;
    uint8_t *mv, *rv, *ev;
    // diff, mask (A17, A21); optional sub-pixel WTA (A22 extension)
    double* diff;
    uint8_t* mask;
    float* sub;
    // per active index: 4x4 homography (row-major), A4
    const double* H16;
};

__device__ __forceinline__ int slot_of(const Bufs& b, int a) { return b.slots[a]; }

// Quads ALLOCATED to a window of nq quads in the quad layout (costq, pdir):
// a multiple of kQuadAlign, so every window starts 16-byte aligned and the
// scan moves a narrow window, or a lane's 4 quads of a wide one, as one
// 128-bit access instead of 3-4 32-bit ones (the scan runs at ~74% L1/LSU
// throughput with 4-byte accesses: 945 M L1 tag requests per 0.70 G cells).
constexpr uint32_t kQuadAlign = 4;
__host__ __device__ inline uint32_t alloc_quads(uint32_t nq) {
    return (nq + (kQuadAlign - 1)) & ~(kQuadAlign - 1);
}

// Doubles -> u64 keys whose unsigned order is the numeric order; -0.0 is
// canonicalised to +0.0 so ties behave like the reference's `!=` tests
// (geometry.cpp:116-123).
__device__ __forceinline__ unsigned long long ord_key(double x) {
    unsigned long long u = (x == 0.0) ? 0ull : static_cast<unsigned long long>(__double_as_longlong(x));
    return (u >> 63) ? ~u : (u | (1ull << 63));
}
__device__ __forceinline__ double key_double(unsigned long long k) {
    unsigned long long u = (k >> 63) ? (k & ~(1ull << 63)) : ~k;
    return __longlong_as_double(static_cast<long long>(u));
}

// static_cast<int>(std::lround(x)) as compiled for x86-64 (geometry.cpp:143-144,
// temporal_filter.cpp:263): round half away from zero to long; out-of-range or
// NaN yields LONG_MIN (cvttsd2si); the int cast keeps the low 32 bits.
__device__ __forceinline__ long long x86_lround_long(double x) {
    double t = trunc(x);
    if (fabs(x - t) >= 0.5) t += copysign(1.0, x);
    if (t >= -9223372036854775808.0 && t < 9223372036854775808.0) return static_cast<long long>(t);
    return static_cast<long long>(0x8000000000000000ull);
}
__device__ __forceinline__ int x86_lround_int(double x) {
    const long long v = x86_lround_long(x);
    return static_cast<int>(static_cast<unsigned int>(static_cast<unsigned long long>(v)));
}

// static_cast<int>(double) as compiled for x86-64 (cvttsd2si, 32-bit):
// truncation; out-of-range or NaN yields INT_MIN (temporal_filter.cpp:119-124).
__device__ __forceinline__ int x86_cvtt_int(double x) {
    if (x > -2147483649.0 && x < 2147483648.0) return static_cast<int>(x);
    return static_cast<int>(0x80000000u);
}

// derive_search_ranges for a valid prediction, temporal_filter.cpp:115-137
__device__ __forceinline__ void derive_range(double d, double p, int top, int min_len,
                                             int use_stddev, double gain, int& lo, int& hi) {
    const double half = use_stddev ? gain * sqrt(p) : p;
    lo = x86_cvtt_int(floor(d - half));
    hi = x86_cvtt_int(ceil(d + half));
    lo = max(0, min(top, lo));
    hi = max(0, min(top, hi));
    const int deficit = min_len - (hi - lo + 1);
    if (deficit > 0) {
        lo -= deficit / 2;
        hi += deficit - deficit / 2;
        if (lo < 0) {
            hi = min(top, hi - lo);
            lo = 0;
        }
        if (hi > top) {
            lo = max(0, lo - (hi - top));
            hi = top;
        }
    }
}

__device__ __forceinline__ bool census_defined(int x, int y, int W, int H) {
    return x >= kCensusRadius && x < W - kCensusRadius && y >= kCensusRadius &&
           y < H - kCensusRadius;
}

// ------------------------------------------------------------------ launchers
// (defined in the .cu files; all enqueue on `st` and count launches)
// Stages of StepTimings / SgmStageTimings (temporal_filter.hpp:57-62,
// sgm.hpp:59-64) a launcher may mark the end of (tsgm_stage_timings).
enum Stage { kStPredict = 0, kStRanges, kStCensus, kStCost, kStAggregate, kStWta, kStCorrect,
             kStCount };

struct Launch {
    cudaStream_t st;
    unsigned long long* counter;
    // optional: records a CUDA event marking the end of `stage` on `st`
    void (*mark)(void* arg, int stage) = nullptr;
    void* mark_arg = nullptr;
    void end_stage(int stage) const {
        if (mark) mark(mark_arg, stage);
    }
};

void launch_census(const Bufs& b, int n, Launch L);
// the step's fused chain: forward warp (no pass-1 cache), then the predict
// tile kernel (variance, reject, fill, ranges, tile counts), then offsets +
// scan records + key re-arm
void launch_warp_step(const Bufs& b, int n, int d_max, Launch L);
void launch_predict_tile(const Bufs& b, int n, double q, double disc_thresh, int min_hw,
                         int use_stddev, double gain, Launch L);
void launch_offsets_step(const Bufs& b, int n, Launch L);
void launch_ranges_from_pred(const Bufs& b, int n, int min_hw, int use_stddev, double gain,
                             Launch L);
void launch_ranges_given(const Bufs& b, int n, Launch L);  // lo/hi already set
void launch_offsets(const Bufs& b, int n, Launch L);       // row scan + finalize
void launch_volume_plan(const Bufs& b, int m, Launch L);
void launch_cost(const Bufs& b, int n, Launch L);  // quad layout (costq), the aggregation's input
void launch_cost_ragged(const Bufs& b, int n, Launch L);  // reference layout (cost)
void launch_cost_quads_from_ragged(const Bufs& b, int n, Launch L);
void launch_wta(const Bufs& b, int n, Launch L);
void launch_median(const Bufs& b, int n, const int32_t* in_d, const uint8_t* in_v,
                   int32_t* out_d, uint8_t* out_v, Launch L);

void launch_warp(const Bufs& b, int n, const double* src_d, const double* src_p,
                 const uint8_t* src_v, int d_max, Launch L);
// predict tail: phi/variance (A7) then optionally reject (A8) and fill (A9)
void launch_predict_finalize(const Bufs& b, int n, double q, int apply_phi, Launch L);
void launch_reject_fill(const Bufs& b, int n, const double* in_d, const double* in_p,
                        const uint8_t* in_v, double* out_d, double* out_p, uint8_t* out_v,
                        double disc_thresh, int do_reject, int do_fill, Launch L);
void launch_correct(const Bufs& b, int n, double r, double mask_tau, Launch L);
// correct + render + export median fused (the step's path)
void launch_correct_median(const Bufs& b, int n, double r, double mask_tau, Launch L);

void launch_aggregate(const Bufs& b, int n, int p1, int p2, int paths, int path_set, Launch L);
// Line-sweep aggregation (aggregate_sweep.cu): returns false when the
// configuration does not fit its shared-memory plan (caller falls back).
bool sweep_supported(int W, int H, int d_max, int p2);
const char* last_sweep_variant();  // kernels of the calling thread's last sweep launch
// write_s: store S in the ragged volume; do_wta: fuse winner_takes_all
// (writes md/mv). At least one of the two must be set. full_range: every
// window spans d_max (frames from an empty state): the line-group scan wins.
void launch_aggregate_sweep(const Bufs& b, int n, int p1, int p2, int paths, int path_set,
                            int write_s, int do_wta, Launch L, int subpix = 0,
                            bool full_range = false);

// Noise calibration (noise.cu), SURVEY §8(f) row 4.
struct HistSpec {
    double lo, hi, bw;  // ErrorHistogram(lo, hi, bin_width), noise_calib.cpp:9-14
    int nbins;
};
struct HistAcc {                   // device buffers, zeroed by the caller
    unsigned long long* counts;    // [nbins]
    unsigned long long* tallies;   // underflow, overflow, within 1 px, gated
    double* partial;               // [hist_partial_doubles()]
    double* sums;                  // gated sum, sum of squares (running over batches)
};
size_t hist_partial_doubles();
void launch_gt_state(const Bufs& b, const double* gt, int n, Launch L);
void launch_error_hist_warped(const Bufs& b, const double* gt, int n, const HistSpec& hs,
                              const HistAcc& acc, Launch L);
void launch_error_hist_wta(const Bufs& b, const double* gt, int n, const HistSpec& hs,
                           const HistAcc& acc, Launch L);
void launch_error_map(const Bufs& b, const double* gt, int n, double* acc,
                      unsigned long long* overlap, Launch L);

// Export formats (export.cu): write_disparity_png's
// 16-bit quantisation on the device. disp (f64) or (d, valid) maps at
// base + (slots ? slots[a] : a) * P; raw u16 out at raw + a * P; first_bad[a]
// = the first raster index not encodable (or ~0), zeroed by the launcher.
void launch_quantize_disparity(const double* disp, const int32_t* d, const uint8_t* valid,
                               size_t P, int n, const int* slots, uint16_t* raw,
                               unsigned long long* first_bad, Launch L);
// Host PNG encoder (16-bit grayscale, zlib) and boxes.txt writer.
void write_png16(const std::string& path, const uint16_t* raw, int w, int h);
void read_png16(const std::string& path, std::vector<uint16_t>& raw, int& w, int& h);

// Box detector (detect.cu), SURVEY §8(f) row 1.
constexpr int kMaxDetectWindows = 64;  // kernel-parameter table (1.6 KB); INTEGRATION.md
struct DetectWindows {
    int n;
    int ww[kMaxDetectWindows], wh[kMaxDetectWindows];
    int cols[kMaxDetectWindows], rows[kMaxDetectWindows];  // positions per size
    long long base[kMaxDetectWindows + 1];                  // prefix of positions per size
    int region_top;
    double thresh;
};
// Window positions of the sizes that fit (motion_detect.cpp:68-76).
void detect_windows(const tsgm_detect_config& c, int W, int H, DetectWindows& dw);
// SAT of n maps (map + slots[a] * map_stride, or + a * map_stride when slots
// is null) into sat + a * sat_stride, (H+1) x (W+1) each.
void launch_sat(const double* map, size_t map_stride, double* sat, size_t sat_stride, int W, int H,
                int n, const int* slots, Launch L);
void launch_candidates(const double* sat, size_t sat_stride, int W, const DetectWindows& dw, int n,
                       tsgm_box* out, long long cap, long long* counts, Launch L);
long long greedy_merge_host(tsgm_box* boxes, long long n, const tsgm_detect_config& c);

// Outlier count (detect.cu): n maps, d/valid/gt at
// base + (slots ? slots[a] : a) * P for d/valid and gt + a * P; counts[2a],
// counts[2a+1] = evaluated, outliers (zeroed by the launcher).
void launch_count_outliers(const int32_t* d, const uint8_t* valid, const double* gt, size_t P,
                           int n, const int* slots, double abs_thresh, double rel_thresh,
                           int strict, unsigned long long* counts, Launch L);

}  // namespace tsgm
