// Host runtime behind include/tsgm_b200.h: device-resident per-slot state,
// batched per-frame launch sequence on one stream, the stateless stage API, and
// the host-side FP64 geometry (relative_motion, disparity_homography) in the
// reference's operation order.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"
#include "tsgm_b200.h"

using namespace tsgm;

namespace {

thread_local std::string g_err;

struct invalid_arg : std::runtime_error {
    using std::runtime_error::runtime_error;
};

[[noreturn]] void bad(const char* msg) { throw invalid_arg(msg); }

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}
#define CK(x) cuda_check((x), #x)

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return TSGM_OK;
    } catch (const invalid_arg& e) {
        g_err = e.what();
        return TSGM_INVALID_ARGUMENT;
    } catch (const std::exception& e) {
        g_err = e.what();
        return TSGM_RUNTIME_ERROR;
    }
}

// ------------------------------------------------------------------ geometry
// Sequential-k products without FMA (the host compiler runs with
// -ffp-contract=off): the same order as the oracle restatement
// (oracle/tsgm_oracle.c) and the oracle build's Eigen stand-in.
void mat3_mul(const double* a, const double* b, double* r) {
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            r[i * 3 + j] = (a[i * 3 + 0] * b[0 * 3 + j] + a[i * 3 + 1] * b[1 * 3 + j]) +
                           a[i * 3 + 2] * b[2 * 3 + j];
}
void mat3_vec(const double* a, const double* v, double* r) {
    for (int i = 0; i < 3; ++i) r[i] = (a[i * 3 + 0] * v[0] + a[i * 3 + 1] * v[1]) + a[i * 3 + 2] * v[2];
}
void mat4_mul(const double* a, const double* b, double* r) {
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j)
            r[i * 4 + j] = ((a[i * 4 + 0] * b[0 * 4 + j] + a[i * 4 + 1] * b[1 * 4 + j]) +
                            a[i * 4 + 2] * b[2 * 4 + j]) +
                           a[i * 4 + 3] * b[3 * 4 + j];
}

// RigidMotion::validate, geometry.cpp:30-36
void motion_validate(const double* r) {
    double rt[9], g[9];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) rt[i * 3 + j] = r[j * 3 + i];
    mat3_mul(rt, r, g);
    double mx = 0.0;
    for (int i = 0; i < 9; ++i) {
        const double e = std::fabs(g[i] - ((i % 4) == 0 ? 1.0 : 0.0));
        if (i == 0 || e > mx) mx = e;
    }
    if (!(mx <= 1e-9)) bad("RigidMotion: rotation is not orthonormal");
    const double det = r[0] * (r[4] * r[8] - r[5] * r[7]) - r[3] * (r[1] * r[8] - r[2] * r[7]) +
                       r[6] * (r[1] * r[5] - r[2] * r[4]);
    if (!(std::fabs(det - 1.0) <= 1e-9)) bad("RigidMotion: rotation determinant is not +1");
}

// StereoCalib::validate, geometry.cpp:21-28
void calib_validate(const tsgm_stereo_calib& c) {
    if (!(c.focal_px > 0.0)) bad("StereoCalib: focal_px must be positive");
    if (!(c.baseline_m > 0.0)) bad("StereoCalib: baseline_m must be positive");
    if (!(c.width > 0 && c.height > 0)) bad("StereoCalib: empty image");
    if (!(c.cx >= 0.0 && c.cx < c.width)) bad("StereoCalib: cx outside image");
    if (!(c.cy >= 0.0 && c.cy < c.height)) bad("StereoCalib: cy outside image");
    if (!(c.d_max >= 1)) bad("StereoCalib: d_max must be at least 1");
}

// SgmParams::validate, sgm.cpp:14-23
void sgm_validate(const tsgm_sgm_params& p) {
    if (p.p1 <= 0 || p.p2 < p.p1) bad("SgmParams: require 0 < p1 <= p2");
    if (p.paths != 4 && p.paths != 8) bad("SgmParams: paths must be 4 or 8");
    if (p.d_max < 1 || p.d_max > 65535) bad("SgmParams: d_max out of range");
    if ((kMaxCost + p.p2) * p.paths > 65535) bad("SgmParams: p2 too large for 16-bit accumulation");
}

// disparity_homography, geometry.cpp:77-110 (row-major out)
void homography(const double* r9, const double* t3, const tsgm_stereo_calib& c, double* h16) {
    calib_validate(c);
    motion_validate(r9);
    bool ident = t3[0] == 0.0 && t3[1] == 0.0 && t3[2] == 0.0;
    for (int i = 0; i < 9; ++i) ident = ident && r9[i] == ((i % 4) == 0 ? 1.0 : 0.0);
    std::memset(h16, 0, 16 * sizeof(double));
    if (ident) {
        h16[0] = h16[5] = h16[10] = h16[15] = 1.0;
        return;
    }
    const double f = c.focal_px, b = c.baseline_m;
    double q[16] = {0}, qi[16] = {0}, t[16] = {0}, tmp[16];
    q[0] = 1.0;
    q[3] = -c.cx;
    q[5] = 1.0;
    q[7] = -c.cy;
    q[11] = f;
    q[14] = 1.0 / b;
    qi[0] = 1.0;
    qi[2] = c.cx / f;
    qi[5] = 1.0;
    qi[6] = c.cy / f;
    qi[11] = b;
    qi[14] = 1.0 / f;
    for (int i = 0; i < 3; ++i) {
        for (int j = 0; j < 3; ++j) t[i * 4 + j] = r9[i * 3 + j];
        t[i * 4 + 3] = t3[i];
    }
    t[15] = 1.0;
    mat4_mul(qi, t, tmp);
    mat4_mul(tmp, q, h16);
}

// relative_motion, geometry.cpp:189-197
void relative_motion(const double* prev12, const double* cur12, double* r9, double* t3) {
    double rp[9], rc[9], tp[3], tc[3];
    for (int i = 0; i < 3; ++i) {
        for (int j = 0; j < 3; ++j) {
            rp[i * 3 + j] = prev12[i * 4 + j];
            rc[i * 3 + j] = cur12[i * 4 + j];
        }
        tp[i] = prev12[i * 4 + 3];
        tc[i] = cur12[i * 4 + 3];
    }
    motion_validate(rp);
    motion_validate(rc);
    bool same = true;
    for (int i = 0; i < 12; ++i) same = same && prev12[i] == cur12[i];
    if (same) {
        for (int i = 0; i < 9; ++i) r9[i] = (i % 4) == 0 ? 1.0 : 0.0;
        t3[0] = t3[1] = t3[2] = 0.0;
        return;
    }
    double rct[9], it[3], tmp[3];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) rct[i * 3 + j] = rc[j * 3 + i];
    mat3_vec(rct, tc, tmp);
    for (int i = 0; i < 3; ++i) it[i] = -tmp[i];
    mat3_mul(rct, rp, r9);
    mat3_vec(rct, tp, tmp);
    for (int i = 0; i < 3; ++i) t3[i] = tmp[i] + it[i];
}

}  // namespace

// ====================================================================== context
constexpr int kRing = 8;

struct tsgm_ctx {
    tsgm_config cfg{};
    int W = 0, H = 0, P = 0, d_max = 0, max_slots = 0;
    size_t vol_cap = 0;
    int vol_slots = 0;            // volume pool, in worst-case (full-range) sequences
    std::vector<int> vol_owner;   // slot whose volumes sit at each position (-1: none)
    unsigned long long* d_vb = nullptr;  // [2][max_slots] position bases (volume_plan_kernel)
    std::vector<unsigned long long> h_cells, h_quads;  // readback for chunk planning
    std::vector<int> h_slots;     // host copy of the current batch's slots
    std::vector<char> fresh;      // slot holds the empty state (its next frame is full range)
    int device = 0;
    int num_sms = 148;
    bool use_sweep = false;  // line-sweep aggregation (else per-direction scanline kernel)
    cudaStream_t st = nullptr;
    Bufs b{};
    unsigned long long launches = 0;
    std::vector<void*> allocs;
    // per-step device arrays
    int* d_slots = nullptr;
    const uint8_t** d_left = nullptr;
    const uint8_t** d_right = nullptr;
    double* d_H = nullptr;
    // pinned staging ring
    struct Stage {
        int* slots;
        const uint8_t** left;
        const uint8_t** right;
        double* H;
        cudaEvent_t done;
        bool used;
    } ring[kRing]{};
    int ring_i = 0;
    uint8_t* d_img = nullptr;  // [max_slots][2][P] staging for host-image steps
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    // Host-image steps upload on their own stream into two alternating
    // staging buffers, so frame k+1's images cross PCIe while frame k
    // computes; a buffer is reused once the census that read it has run.
    cudaStream_t up_st = nullptr;
    static constexpr int kImgBufs = 2;
    uint8_t* d_img_up[kImgBufs]{};
    int img_buf = 0;
    int img_pending_free = -1;  // buffer the current step reads (free after census)
    cudaEvent_t ev_img_ready[kImgBufs]{}, ev_img_free[kImgBufs]{};
    bool img_free_recorded[kImgBufs]{};
    // Batched fetches: a device-to-device snapshot on the compute stream, then
    // the device-to-host copy from the snapshot on the copy stream, so the
    // next frame never waits for PCIe; a kind's snapshot is rewritten only
    // after its previous copy-out finished (a frame later).
    cudaStream_t copy_st = nullptr;
    cudaEvent_t ev_frame = nullptr;
    void* snap[TSGM_OUT_COUNT]{};
    cudaEvent_t ev_snap_copied[TSGM_OUT_COUNT]{};
    bool snap_pending[TSGM_OUT_COUNT]{};
    // Outputs written only by the frame's last kernel (correct_median: state,
    // export map, diff, mask) are copied out directly from the live buffers;
    // the next frame's correct_median waits for those copies instead.
    cudaEvent_t ev_direct_copied = nullptr;
    bool direct_pending = false;
    // box detector (tsgm_detect): per-slot SAT, candidate boxes and counts
    double* det_sat = nullptr;
    tsgm_box* det_boxes = nullptr;
    long long* det_counts = nullptr;
    long long det_cap = 0;  // candidate capacity per slot
    // outlier metric (tsgm_count_outliers_batch): uploaded GT maps and counts
    double* eval_gt = nullptr;
    unsigned long long* eval_counts = nullptr;
    // per-stage device times of the last step (StepResult::timings,
    // temporal_filter.hpp:57-69): events recorded at stage ends on `st`
    std::string last_kernels;  // aggregation kernels of the last step's last chunk
    int last_chunks = 0;       // volume chunks of the last step
    int last_c0 = 0;           // batch index of the last chunk's first sequence
    bool last_full = false;    // the last chunk's windows are all full range (every sequence fresh)
    bool stage_timing = false;
    std::vector<cudaEvent_t> tev;
    std::vector<int> tstage;
    int tev_used = 0;
    // tsgm_step_device_after / tsgm_inputs_consumed: the input-release event
    cudaEvent_t ev_inputs = nullptr, ev_consumed = nullptr;
    bool consumed_recorded = false;

    template <typename T>
    T* dalloc(size_t count) {
        void* p = nullptr;
        CK(cudaMalloc(&p, sizeof(T) * std::max<size_t>(count, 1)));
        allocs.push_back(p);
        return static_cast<T*>(p);
    }
    ~tsgm_ctx() {
        if (device >= 0) cudaSetDevice(device);
        if (st) cudaStreamSynchronize(st);
        for (void* p : allocs) cudaFree(p);
        for (auto& r : ring) {
            if (r.slots) cudaFreeHost(r.slots);
            if (r.left) cudaFreeHost(r.left);
            if (r.right) cudaFreeHost(r.right);
            if (r.H) cudaFreeHost(r.H);
            if (r.done) cudaEventDestroy(r.done);
        }
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
        if (copy_st) cudaStreamSynchronize(copy_st);
        if (up_st) cudaStreamSynchronize(up_st);
        if (ev_frame) cudaEventDestroy(ev_frame);
        for (auto e : ev_snap_copied)
            if (e) cudaEventDestroy(e);
        for (auto e : tev) cudaEventDestroy(e);
        if (ev_inputs) cudaEventDestroy(ev_inputs);
        if (ev_consumed) cudaEventDestroy(ev_consumed);
        if (ev_direct_copied) cudaEventDestroy(ev_direct_copied);
        for (int i = 0; i < kImgBufs; ++i) {
            if (ev_img_ready[i]) cudaEventDestroy(ev_img_ready[i]);
            if (ev_img_free[i]) cudaEventDestroy(ev_img_free[i]);
        }
        if (copy_st) cudaStreamDestroy(copy_st);
        if (up_st) cudaStreamDestroy(up_st);
        if (st) cudaStreamDestroy(st);
    }
    // records the end of `stage` (or the step's start, stage < 0)
    void mark(int stage) {
        if (!stage_timing) return;
        if (tev_used == static_cast<int>(tev.size())) {
            cudaEvent_t e = nullptr;
            if (cudaEventCreate(&e) != cudaSuccess) throw std::runtime_error("cudaEventCreate failed");
            tev.push_back(e);
            tstage.push_back(-1);
        }
        if (cudaEventRecord(tev[tev_used], st) != cudaSuccess) throw std::runtime_error("cudaEventRecord failed");
        tstage[tev_used++] = stage;
    }
    static void mark_cb(void* self, int stage) { static_cast<tsgm_ctx*>(self)->mark(stage); }
    Launch L() {
        Launch l{st, &launches};
        if (stage_timing) {
            l.mark = &tsgm_ctx::mark_cb;
            l.mark_arg = this;
        }
        return l;
    }
    // seconds per stage between the recorded marks (waits for the last one)
    void stage_seconds(double* t) {
        for (int k = 0; k < kStCount; ++k) t[k] = 0.0;
        if (tev_used < 2) return;
        if (cudaEventSynchronize(tev[tev_used - 1]) != cudaSuccess)
            throw std::runtime_error("cudaEventSynchronize failed");
        for (int i = 1; i < tev_used; ++i) {
            float ms = 0.f;
            if (cudaEventElapsedTime(&ms, tev[i - 1], tev[i]) != cudaSuccess)
                throw std::runtime_error("cudaEventElapsedTime failed");
            if (tstage[i] >= 0 && tstage[i] < kStCount) t[tstage[i]] += 1e-3 * ms;
        }
    }
};

namespace {

void validate_config(const tsgm_config& c) {
    // step() preconditions, temporal_filter.cpp:198-206 + what sgm_match /
    // census_transform / make_cost_volume would throw on every frame
    if (c.width != c.calib.width || c.height != c.calib.height)
        bad("tsgm_create: image size must equal calib.width x calib.height");
    if (c.sgm.d_max != c.calib.d_max) bad("step: params.d_max disagrees with calibration");
    calib_validate(c.calib);
    sgm_validate(c.sgm);
    if (c.width < 2 * kCensusRadius + 1 || c.height < 2 * kCensusRadius + 1)
        bad("census_transform: image smaller than the 5x5 window");
    const unsigned long long cap = 1ull * c.width * c.height * c.sgm.d_max;
    if (cap > 0xffffffffull) bad("CostVolume: volume exceeds 32-bit addressing");
    if (c.max_slots < 1) bad("tsgm_create: max_slots must be >= 1");
}

// The reference-layout cost pool, allocated on first need (16 bytes of
// padding on both sides: the fallback and stage kernels read aligned words).
void ensure_ragged_cost(tsgm_ctx* ctx) {
    if (!ctx->b.cost) ctx->b.cost = ctx->dalloc<uint8_t>(ctx->b.pool_cells + 32) + 16;
}

void init_ctx(tsgm_ctx* ctx, const tsgm_config& c) {
    ctx->cfg = c;
    ctx->W = c.width;
    ctx->H = c.height;
    ctx->P = c.width * c.height;
    ctx->d_max = c.sgm.d_max;
    ctx->max_slots = c.max_slots;
    ctx->vol_cap = static_cast<size_t>(ctx->P) * ctx->d_max;
    ctx->device = c.device;
    CK(cudaSetDevice(c.device));
    CK(cudaStreamCreateWithFlags(&ctx->st, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&ctx->copy_st, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&ctx->up_st, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&ctx->ev_frame, cudaEventDisableTiming));
    for (auto& e : ctx->ev_snap_copied) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ctx->ev_direct_copied, cudaEventDisableTiming));
    for (int i = 0; i < tsgm_ctx::kImgBufs; ++i) {
        CK(cudaEventCreateWithFlags(&ctx->ev_img_ready[i], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&ctx->ev_img_free[i], cudaEventDisableTiming));
    }
    CK(cudaEventCreate(&ctx->ev0));
    CK(cudaEventCreate(&ctx->ev1));
    CK(cudaEventCreateWithFlags(&ctx->ev_inputs, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ctx->ev_consumed, cudaEventDisableTiming));
    ctx->stage_timing = (c.flags & TSGM_STAGE_TIMINGS) != 0;
    const size_t S = c.max_slots, P = ctx->P;
    Bufs& b = ctx->b;
    b.W = ctx->W;
    b.H = ctx->H;
    b.P = ctx->P;
    b.d_max = ctx->d_max;
    b.vol_cap = ctx->vol_cap;
    b.sd = ctx->dalloc<double>(S * P);
    b.sp = ctx->dalloc<double>(S * P);
    b.sv = ctx->dalloc<uint8_t>(S * P);
    b.kd = ctx->dalloc<unsigned long long>(S * P);
    b.kps = ctx->dalloc<ulonglong2>(S * P);
    b.wtgt = ctx->dalloc<int>(S * P);
    b.wdk = ctx->dalloc<unsigned long long>(S * P);
    b.wd = ctx->dalloc<double>(S * P);
    b.wp = ctx->dalloc<double>(S * P);
    b.wsrc = ctx->dalloc<double>(S * P);
    b.wv = ctx->dalloc<uint8_t>(S * P);
    b.pd = ctx->dalloc<double>(S * P);
    b.pp = ctx->dalloc<double>(S * P);
    b.pv = ctx->dalloc<uint8_t>(S * P);
    b.lo = ctx->dalloc<uint16_t>(S * P);
    b.hi = ctx->dalloc<uint16_t>(S * P);
    b.lohi = ctx->dalloc<uint32_t>(S * P);
    b.off = ctx->dalloc<uint32_t>(S * (P + 1));
    b.row_sum = ctx->dalloc<uint32_t>(S * ctx->H);
    b.qoff = ctx->dalloc<uint32_t>(S * (P + 1));
    b.tmeta = ctx->dalloc<uint2>(S * P);
    b.rmeta = ctx->dalloc<uint2>(S * P);
    b.qrow_sum = ctx->dalloc<uint32_t>(S * ctx->H);
    b.tsum = ctx->dalloc<uint2>(S * ctx->H * static_cast<size_t>((ctx->W + 31) / 32));
    b.nquads = ctx->dalloc<unsigned long long>(S);
    b.ncells = ctx->dalloc<unsigned long long>(S);
    b.overflow = ctx->dalloc<int>(S);
    b.sigl = ctx->dalloc<uint32_t>(S * P);
    b.sigr = ctx->dalloc<uint32_t>(S * P);
    const char* force = std::getenv("TSGM_FORCE_SCANLINE_AGG");
    const bool force_scan = (c.flags & TSGM_FORCE_SCANLINE_AGG) || (force && force[0] == '1');
    ctx->use_sweep = !force_scan &&
                     sweep_supported(ctx->W, ctx->H, ctx->d_max, c.sgm.p2);
    // multiple of 4 quads: the combine reads each direction 16 bytes at a time
    b.quad_cap = (P * static_cast<size_t>(alloc_quads(static_cast<uint32_t>((ctx->d_max - 1) / 4 + 1))) + 3) & ~static_cast<size_t>(3);
    b.max_slots = c.max_slots;
    b.work = ctx->dalloc<int>(1);
    CK(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, c.device));
    b.num_sms = ctx->num_sms;
    b.md = ctx->dalloc<int32_t>(S * P);
    b.rd = ctx->dalloc<int32_t>(S * P);
    b.ed = ctx->dalloc<int32_t>(S * P);
    b.mv = ctx->dalloc<uint8_t>(S * P);
    b.rv = ctx->dalloc<uint8_t>(S * P);
    b.ev = ctx->dalloc<uint8_t>(S * P);
    b.diff = ctx->dalloc<double>(S * P);
    b.mask = ctx->dalloc<uint8_t>(S * P);
    b.sub = (c.flags & TSGM_SUBPIXEL) ? ctx->dalloc<float>(S * P) : nullptr;
    ctx->d_slots = ctx->dalloc<int>(S);
    ctx->d_left = ctx->dalloc<const uint8_t*>(S);
    ctx->d_right = ctx->dalloc<const uint8_t*>(S);
    ctx->d_H = ctx->dalloc<double>(S * 16);
    ctx->d_img = ctx->dalloc<uint8_t>(S * 2 * P);
    for (auto& u : ctx->d_img_up) u = ctx->dalloc<uint8_t>(S * 2 * P);
    // the per-frame volumes last: C (u8), S (u16) and, for the scan
    // aggregation, 8 directions of u8 path costs per cell, for vol_slots
    // sequences at a time (the rest of the batch runs in further chunks)
    // (the reference-layout cost is allocated on demand: fetch, stage API, fallback)
    const size_t vol_bytes = 2 * ctx->vol_cap + 4 * b.quad_cap + (ctx->use_sweep ? 8 * b.quad_cap * 4 : 0);
    int vs = c.vol_slots > 0 ? std::min(c.vol_slots, c.max_slots) : c.max_slots;
    if (c.vol_slots <= 0) {
        size_t free_b = 0, total_b = 0;
        CK(cudaMemGetInfo(&free_b, &total_b));
        // headroom: the runtime, plus fetch_batch snapshots of every per-pixel output
        const size_t reserve = (size_t(1) << 30) + S * P * 16;
        const size_t fit = free_b > reserve ? (free_b - reserve) / vol_bytes : 0;
        vs = static_cast<int>(std::min<size_t>(vs, fit));
        if (vs < 1) throw std::runtime_error("tsgm_create: device memory too small for one frame's volumes");
    }
    ctx->vol_slots = vs;
    ctx->vol_owner.assign(c.max_slots, -1);
    ctx->fresh.assign(c.max_slots, 1);
    b.vol_slots = vs;
    // The pool holds vs worst-case volumes (plus the per-position rounding of
    // volume_plan_kernel); a chunk packs as many sequences as their ACTUAL
    // cells fit (reduced frames need ~10x fewer than P*d_max).
    b.pool_cells = static_cast<size_t>(vs) * ctx->vol_cap + 16 * S;
    b.pool_quads = static_cast<size_t>(vs) * b.quad_cap + 4 * S;
    ctx->d_vb = ctx->dalloc<unsigned long long>(2 * S);
    CK(cudaMemsetAsync(ctx->d_vb, 0, sizeof(unsigned long long) * 2 * S, ctx->st));
    b.vbase = ctx->d_vb;
    b.vqbase = ctx->d_vb + S;
    // 16 bytes of padding on both sides: the sweep reads aligned words around
    // each window
    b.cost = nullptr;
    if (!ctx->use_sweep || c.max_slots == 1) ensure_ragged_cost(ctx);
    // (+64 words: a narrow lane reads up to 3 quads past its window)
    b.costq = ctx->dalloc<uint32_t>(b.pool_quads + 64);
    b.agg = ctx->dalloc<uint16_t>(b.pool_cells);
    if (ctx->use_sweep) b.pdir = ctx->dalloc<uint8_t>(8 * b.pool_quads * 4);
    b.slots = ctx->d_slots;
    b.left = ctx->d_left;
    b.right = ctx->d_right;
    b.H16 = ctx->d_H;
    // empty state everywhere, warp keys armed
    CK(cudaMemsetAsync(b.sd, 0, sizeof(double) * S * P, ctx->st));
    CK(cudaMemsetAsync(b.sp, 0, sizeof(double) * S * P, ctx->st));
    CK(cudaMemsetAsync(b.sv, 0, S * P, ctx->st));
    CK(cudaMemsetAsync(b.kd, 0, sizeof(unsigned long long) * S * P, ctx->st));
    CK(cudaMemsetAsync(b.kps, 0xff, sizeof(ulonglong2) * S * P, ctx->st));
    CK(cudaMemsetAsync(b.ncells, 0, sizeof(unsigned long long) * S, ctx->st));
    for (auto& r : ctx->ring) {
        CK(cudaMallocHost(&r.slots, sizeof(int) * S));
        CK(cudaMallocHost(reinterpret_cast<void**>(&r.left), sizeof(void*) * S));
        CK(cudaMallocHost(reinterpret_cast<void**>(&r.right), sizeof(void*) * S));
        CK(cudaMallocHost(&r.H, sizeof(double) * 16 * S));
        CK(cudaEventCreateWithFlags(&r.done, cudaEventDisableTiming));
        r.used = false;
    }
    CK(cudaStreamSynchronize(ctx->st));
}

// Stage the per-step arrays (slots, image pointers, homographies) and upload.
void upload_step(tsgm_ctx* ctx, int n, const int32_t* slots, const uint8_t* const* dl,
                 const uint8_t* const* dr, const double* H) {
    auto& r = ctx->ring[ctx->ring_i];
    ctx->ring_i = (ctx->ring_i + 1) % kRing;
    if (r.used) CK(cudaEventSynchronize(r.done));
    std::memcpy(r.slots, slots, sizeof(int) * n);
    ctx->h_slots.assign(slots, slots + n);
    std::memcpy(r.left, dl, sizeof(void*) * n);
    std::memcpy(r.right, dr, sizeof(void*) * n);
    std::memcpy(r.H, H, sizeof(double) * 16 * n);
    CK(cudaMemcpyAsync(ctx->d_slots, r.slots, sizeof(int) * n, cudaMemcpyHostToDevice, ctx->st));
    CK(cudaMemcpyAsync(ctx->d_left, r.left, sizeof(void*) * n, cudaMemcpyHostToDevice, ctx->st));
    CK(cudaMemcpyAsync(ctx->d_right, r.right, sizeof(void*) * n, cudaMemcpyHostToDevice, ctx->st));
    CK(cudaMemcpyAsync(ctx->d_H, r.H, sizeof(double) * 16 * n, cudaMemcpyHostToDevice, ctx->st));
    CK(cudaEventRecord(r.done, ctx->st));
    r.used = true;
}

// Before the compute stream overwrites a directly copied output (state,
// export map, diff, mask), its pending copy-out must have finished.
void wait_direct_copies(tsgm_ctx* ctx) {
    if (!ctx->direct_pending) return;
    CK(cudaStreamWaitEvent(ctx->st, ctx->ev_direct_copied, 0));
    ctx->direct_pending = false;
}

void check_slots(tsgm_ctx* ctx, int n, const int32_t* slots) {
    if (n < 1 || n > ctx->max_slots) bad("tsgm_step: n out of range");
    std::vector<char> seen(ctx->max_slots, 0);
    for (int i = 0; i < n; ++i) {
        if (slots[i] < 0 || slots[i] >= ctx->max_slots) bad("tsgm_step: slot out of range");
        if (seen[slots[i]]) bad("tsgm_step: duplicate slot in batch");
        seen[slots[i]] = 1;
    }
}

// aggregate_paths for the active slots: the scanline-group kernel when the
// configuration fits it, else the per-direction scanline kernels. With
// fuse_wta, winner_takes_all is fused into the combine (S is then written
// only if keep_s) and the caller skips launch_wta.
// cost_in_ragged: the matching costs come from a caller (b.cost, reference
// layout) instead of launch_cost (b.costq, quad layout).
bool aggregate(tsgm_ctx* ctx, const Bufs& b, int n, Launch L, bool fuse_wta = false,
               bool keep_s = true, bool full_range = false, bool cost_in_ragged = false) {
    const tsgm_config& c = ctx->cfg;
    if (ctx->use_sweep && sweep_supported(ctx->W, ctx->H, ctx->d_max, c.sgm.p2)) {
        if (cost_in_ragged) launch_cost_quads_from_ragged(b, n, L);
        launch_aggregate_sweep(b, n, c.sgm.p1, c.sgm.p2, c.sgm.paths, c.sgm.path_set,
                               (keep_s || !fuse_wta) ? 1 : 0, fuse_wta ? 1 : 0, L,
                               (fuse_wta && b.sub) ? 1 : 0, full_range);
        ctx->last_kernels = last_sweep_variant();
        return fuse_wta;
    }
    if (b.sub) bad("TSGM_SUBPIXEL needs the scan aggregation (P2 + 24 <= 255, d_max <= 256)");
    // the per-direction fallback reads the reference layout
    if (!cost_in_ragged) launch_cost_ragged(b, n, L);
    launch_aggregate(b, n, c.sgm.p1, c.sgm.p2, c.sgm.paths, c.sgm.path_set, L);
    ctx->last_kernels = "aggregate_kernels(scanline fallback)+wta_kernel";
    return false;
}

// The batch arrays of a volume chunk starting at batch position c0.
Bufs chunk_bufs(const Bufs& b, int c0) {
    Bufs bc = b;
    bc.slots = b.slots + c0;
    bc.left = b.left + c0;
    bc.right = b.right + c0;
    bc.H16 = b.H16 + 16 * static_cast<size_t>(c0);
    return bc;
}

// Volume position of a slot whose volumes are still resident (last chunk).
int vol_pos(tsgm_ctx* ctx, int slot) {
    for (int a = 0; a < static_cast<int>(ctx->vol_owner.size()); ++a)
        if (ctx->vol_owner[a] == slot) return a;
    bad("tsgm_fetch: the volumes of this slot are not resident (not in the last volume chunk)");
}

// Volume chunks of the n active slots (sizes, in batch order). When n
// worst-case volumes fit the pool: one chunk, nothing read back. Otherwise
// this frame's actual sizes (make_cost_volume's N, matching_cost.cpp:30-48,
// from the offsets kernels) are read back and packed: K = the greedy chunk
// count, then K chunks balanced by cells where they fit (else greedy).
std::vector<int> plan_chunks(tsgm_ctx* ctx, int n) {
    if (n <= ctx->vol_slots) return {n};
    const Bufs& b = ctx->b;
    const size_t S = ctx->max_slots;
    ctx->h_cells.resize(S);
    ctx->h_quads.resize(S);
    CK(cudaMemcpyAsync(ctx->h_cells.data(), b.ncells, 8 * S, cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaMemcpyAsync(ctx->h_quads.data(), b.nquads, 8 * S, cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    std::vector<unsigned long long> rc(n), rq(n);
    unsigned long long total = 0;
    for (int i = 0; i < n; ++i) {
        const int s = ctx->h_slots[i];
        rc[i] = (ctx->h_cells[s] + 15) & ~15ull;
        rq[i] = (ctx->h_quads[s] + 3) & ~3ull;
        total += rc[i];
    }
    auto pack = [&](double target) {
        std::vector<int> m;
        unsigned long long c = 0, q = 0, done = 0;
        int cnt = 0;
        for (int i = 0; i < n; ++i) {
            const bool over = c + rc[i] > b.pool_cells || q + rq[i] > b.pool_quads;
            const bool bal = target > 0 && cnt > 0 &&
                             static_cast<double>(done + c + rc[i]) >
                                 target * static_cast<double>(m.size() + 1) * 1.0001;
            if (cnt > 0 && (over || bal)) {
                m.push_back(cnt);
                done += c;
                c = q = 0;
                cnt = 0;
            }
            c += rc[i];
            q += rq[i];
            ++cnt;
        }
        m.push_back(cnt);
        return m;
    };
    const std::vector<int> greedy = pack(0.0);
    if (greedy.size() == 1) return greedy;
    const std::vector<int> bal = pack(static_cast<double>(total) / static_cast<double>(greedy.size()));
    return bal.size() <= greedy.size() ? bal : greedy;
}

// The per-frame pipeline of step() (temporal_filter.cpp:195-232) for n slots.
void run_step(tsgm_ctx* ctx, int n) {
    const Bufs& b = ctx->b;
    const tsgm_config& c = ctx->cfg;
    Launch L = ctx->L();
    ctx->tev_used = 0;
    ctx->mark(-1);
    // predict (A5-A9): the forward warp, then one fused tile kernel for the
    // variance step, reject, fill and derive_search_ranges (A10)
    launch_warp_step(b, n, c.calib.d_max, L);
    ctx->mark(kStPredict);
    launch_predict_tile(b, n, c.filter.q, c.filter.disc_thresh, c.filter.min_range_halfwidth,
                        c.filter.range_use_stddev, c.filter.range_stddev_gain, L);
    ctx->mark(kStRanges);
    // make_cost_volume's offsets (A11) + the scan records; re-arms the keys
    launch_offsets_step(b, n, L);
    ctx->mark(kStCost);
    // sgm_match (A12-A15)
    launch_census(b, n, L);
    ctx->mark(kStCensus);
    // the census is the last reader of the step's images (tsgm_inputs_consumed)
    CK(cudaEventRecord(ctx->ev_consumed, ctx->st));
    ctx->consumed_recorded = true;
    // Release the upload buffer right after the census, its only reader. (The
    // release must come early in the frame: recorded after the cost kernels
    // instead, it measurably serialised the next uploads behind the copy-outs.)
    if (ctx->img_pending_free >= 0) {
        CK(cudaEventRecord(ctx->ev_img_free[ctx->img_pending_free], ctx->st));
        ctx->img_free_recorded[ctx->img_pending_free] = true;
        ctx->img_pending_free = -1;
    }
    // the volume stages in balanced chunks of at most vol_slots sequences;
    // cost, agg and pdir are indexed by the position within the chunk. No
    // position keeps an owner from an earlier frame: a slot's volumes are
    // resident (tsgm_fetch COST/AGG) only if it is in this frame's last chunk.
    std::fill(ctx->vol_owner.begin(), ctx->vol_owner.end(), -1);
    // all-fresh batches are full range (every volume worst case): balanced by count
    bool all_fresh = true;
    for (int i = 0; i < n; ++i) all_fresh = all_fresh && ctx->fresh[ctx->h_slots[i]];
    std::vector<int> sizes;
    if (all_fresh) {
        const int chunks = (n + ctx->vol_slots - 1) / ctx->vol_slots;
        for (int k = 0, c0 = 0; k < chunks; ++k) {
            sizes.push_back((n - c0) / (chunks - k));
            c0 += sizes.back();
        }
    } else {
        sizes = plan_chunks(ctx, n);
    }
    ctx->last_chunks = static_cast<int>(sizes.size());
    for (int k = 0, c0 = 0; k < static_cast<int>(sizes.size()); ++k) {
        const int m = sizes[k];
        const Bufs bc = chunk_bufs(b, c0);
        bool full = true;  // every sequence of the chunk starts empty: full-range windows
        for (int a = 0; a < m; ++a) full = full && ctx->fresh[ctx->h_slots[c0 + a]];
        launch_volume_plan(bc, m, L);
        launch_cost(bc, m, L);
        ctx->mark(kStCost);
        if (!aggregate(ctx, bc, m, L, /*fuse_wta=*/true, (c.flags & TSGM_KEEP_VOLUMES) != 0, full)) {
            ctx->mark(kStAggregate);
            launch_wta(bc, m, L);
            ctx->mark(kStWta);
        }
        for (int a = 0; a < m; ++a) ctx->vol_owner[a] = ctx->h_slots[c0 + a];
        ctx->last_c0 = c0;
        ctx->last_full = full;
        c0 += m;
    }
    // correct + diff + mask + render, then the export median (A16-A19, A21)
    wait_direct_copies(ctx);  // the previous frame's outputs may still be copying out
    launch_correct_median(b, n, c.filter.r, c.mask_tau, L);
    ctx->mark(kStCorrect);
    for (int i = 0; i < n; ++i) ctx->fresh[ctx->h_slots[i]] = 0;
    CK(cudaGetLastError());
    CK(cudaEventRecord(ctx->ev_frame, ctx->st));
}

void step_impl(tsgm_ctx* ctx, int n, const int32_t* slots, const uint8_t* const* dl,
               const uint8_t* const* dr, const double* motion) {
    check_slots(ctx, n, slots);
    std::vector<double> H(16 * static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) homography(motion + 12 * i, motion + 12 * i + 9, ctx->cfg.calib, &H[16 * i]);
    CK(cudaSetDevice(ctx->device));
    upload_step(ctx, n, slots, dl, dr, H.data());
    run_step(ctx, n);
}

struct OutDesc {
    const void* base;
    size_t elem;
    size_t stride;  // elements per slot
};

OutDesc out_desc(tsgm_ctx* ctx, int what) {
    const Bufs& b = ctx->b;
    const size_t P = ctx->P;
    switch (what) {
        case TSGM_OUT_STATE_D: return {b.sd, 8, P};
        case TSGM_OUT_STATE_P: return {b.sp, 8, P};
        case TSGM_OUT_STATE_VALID: return {b.sv, 1, P};
        case TSGM_OUT_EXPORT_D: return {b.ed, 4, P};
        case TSGM_OUT_EXPORT_VALID: return {b.ev, 1, P};
        case TSGM_OUT_DIFF: return {b.diff, 8, P};
        case TSGM_OUT_MASK: return {b.mask, 1, P};
        case TSGM_OUT_PRED_D: return {b.pd, 8, P};
        case TSGM_OUT_PRED_P: return {b.pp, 8, P};
        case TSGM_OUT_PRED_VALID: return {b.pv, 1, P};
        case TSGM_OUT_LO: return {b.lo, 2, P};
        case TSGM_OUT_HI: return {b.hi, 2, P};
        case TSGM_OUT_MEAS_D: return {b.md, 4, P};
        case TSGM_OUT_MEAS_VALID: return {b.mv, 1, P};
        case TSGM_OUT_OFFSETS: return {b.off, 4, P + 1};
        case TSGM_OUT_COST: return {b.cost, 1, ctx->vol_cap};
        case TSGM_OUT_AGG: return {b.agg, 2, ctx->vol_cap};
        case TSGM_OUT_SUBPIXEL:
            if (!b.sub) bad("tsgm_fetch: context created without TSGM_SUBPIXEL");
            return {b.sub, 4, P};
        default: bad("tsgm_fetch: unknown output");
    }
}

unsigned long long cells_of(tsgm_ctx* ctx, int slot) {
    unsigned long long n = 0;
    CK(cudaMemcpyAsync(&n, ctx->b.ncells + slot, sizeof n, cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    return n;
}

// One-slot scratch context for the stateless stage API.
std::unique_ptr<tsgm_ctx> scratch(int w, int h, int d_max) {
    tsgm_config c{};
    c.width = w;
    c.height = h;
    c.max_slots = 1;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    c.device = dev;
    c.calib = tsgm_stereo_calib{1.0, 0.0, 0.0, 1.0, w, h, d_max};
    c.sgm = tsgm_sgm_params{6, 65, 8, 0, d_max};
    c.mask_tau = 3.0;
    auto ctx = std::make_unique<tsgm_ctx>();
    init_ctx(ctx.get(), c);
    const int zero = 0;
    const double I[16] = {1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1};
    const uint8_t* l = ctx->d_img;
    const uint8_t* r = ctx->d_img + ctx->P;
    upload_step(ctx.get(), 1, &zero, &l, &r, I);
    return ctx;
}

template <typename T>
void h2d(tsgm_ctx* ctx, T* dst, const T* src, size_t count) {
    CK(cudaMemcpyAsync(dst, src, sizeof(T) * count, cudaMemcpyHostToDevice, ctx->st));
}
template <typename T>
void d2h(tsgm_ctx* ctx, T* dst, const T* src, size_t count) {
    if (dst) CK(cudaMemcpyAsync(dst, src, sizeof(T) * count, cudaMemcpyDeviceToHost, ctx->st));
}
void sync(tsgm_ctx* ctx) {
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(ctx->st));
    if (ctx->copy_st) CK(cudaStreamSynchronize(ctx->copy_st));
    if (ctx->up_st) CK(cudaStreamSynchronize(ctx->up_st));
}

// Host-side window bookkeeping for caller-provided ranges (make_cost_volume,
// matching_cost.cpp:30-48, with its u64 wrap-around on hi < lo).
unsigned long long ranges_total(const uint16_t* lo, const uint16_t* hi, size_t n, int* max_hi) {
    unsigned long long total = 0;
    int mh = 0;
    for (size_t i = 0; i < n; ++i) {
        total += static_cast<unsigned long long>(hi[i]) - lo[i] + 1;
        mh = std::max<int>(mh, hi[i]);
    }
    if (total > 0xffffffffull) bad("CostVolume: volume exceeds 32-bit addressing");
    *max_hi = mh;
    return total;
}

void fill_timings(const double* t, tsgm_stage_timings* out) {
    out->predict_s = t[kStPredict];
    out->ranges_s = t[kStRanges];
    out->census_s = t[kStCensus];
    out->cost_s = t[kStCost];
    out->aggregate_s = t[kStAggregate];
    out->wta_s = t[kStWta];
    out->correct_s = t[kStCorrect];
}

}  // namespace

// ====================================================================== C-ABI
extern "C" {

const char* tsgm_last_error(void) { return g_err.c_str(); }

int tsgm_create(const tsgm_config* cfg, tsgm_ctx** out) {
    return guarded([&] {
        if (!cfg || !out) bad("tsgm_create: null argument");
        validate_config(*cfg);
        auto ctx = std::make_unique<tsgm_ctx>();
        init_ctx(ctx.get(), *cfg);
        *out = ctx.release();
    });
}

void tsgm_destroy(tsgm_ctx* ctx) { delete ctx; }

int tsgm_reset(tsgm_ctx* ctx, int32_t slot) {
    return guarded([&] {
        if (slot < 0 || slot >= ctx->max_slots) bad("tsgm_reset: slot out of range");
        CK(cudaSetDevice(ctx->device));
        wait_direct_copies(ctx);
        const size_t P = ctx->P;
        CK(cudaMemsetAsync(ctx->b.sd + slot * P, 0, 8 * P, ctx->st));
        CK(cudaMemsetAsync(ctx->b.sp + slot * P, 0, 8 * P, ctx->st));
        CK(cudaMemsetAsync(ctx->b.sv + slot * P, 0, P, ctx->st));
        ctx->fresh[slot] = 1;
    });
}

int tsgm_set_state(tsgm_ctx* ctx, int32_t slot, const double* d, const double* p,
                   const uint8_t* valid) {
    return guarded([&] {
        if (slot < 0 || slot >= ctx->max_slots) bad("tsgm_set_state: slot out of range");
        CK(cudaSetDevice(ctx->device));
        wait_direct_copies(ctx);
        ctx->fresh[slot] = 0;  // a caller state may hold valid pixels: reduced windows
        const size_t P = ctx->P;
        if (d) h2d(ctx, ctx->b.sd + slot * P, d, P);
        else CK(cudaMemsetAsync(ctx->b.sd + slot * P, 0, 8 * P, ctx->st));
        if (p) h2d(ctx, ctx->b.sp + slot * P, p, P);
        else CK(cudaMemsetAsync(ctx->b.sp + slot * P, 0, 8 * P, ctx->st));
        if (valid) h2d(ctx, ctx->b.sv + slot * P, valid, P);
        else CK(cudaMemsetAsync(ctx->b.sv + slot * P, 0, P, ctx->st));
        sync(ctx);
    });
}

int tsgm_step(tsgm_ctx* ctx, int32_t n, const int32_t* slots, const uint8_t* const* left,
              const uint8_t* const* right, const double* motion) {
    return guarded([&] {
        if (!ctx || !slots || !left || !right || !motion) bad("tsgm_step: null argument");
        check_slots(ctx, n, slots);
        CK(cudaSetDevice(ctx->device));
        std::vector<const uint8_t*> dl(n), dr(n);
        const size_t P = ctx->P;
        const int bi = ctx->img_buf;
        ctx->img_buf = (ctx->img_buf + 1) % tsgm_ctx::kImgBufs;
        uint8_t* img = ctx->d_img_up[bi];
        if (ctx->img_free_recorded[bi]) CK(cudaStreamWaitEvent(ctx->up_st, ctx->ev_img_free[bi], 0));
        for (int i = 0; i < n; ++i) {
            uint8_t* base = img + static_cast<size_t>(slots[i]) * 2 * P;
            CK(cudaMemcpyAsync(base, left[i], P, cudaMemcpyHostToDevice, ctx->up_st));
            CK(cudaMemcpyAsync(base + P, right[i], P, cudaMemcpyHostToDevice, ctx->up_st));
            dl[i] = base;
            dr[i] = base + P;
        }
        CK(cudaEventRecord(ctx->ev_img_ready[bi], ctx->up_st));
        CK(cudaStreamWaitEvent(ctx->st, ctx->ev_img_ready[bi], 0));
        ctx->img_pending_free = bi;
        step_impl(ctx, n, slots, dl.data(), dr.data(), motion);
    });
}

int tsgm_step_device(tsgm_ctx* ctx, int32_t n, const int32_t* slots,
                     const uint8_t* const* d_left, const uint8_t* const* d_right,
                     const double* motion) {
    return guarded([&] {
        if (!ctx || !slots || !d_left || !d_right || !motion) bad("tsgm_step_device: null argument");
        step_impl(ctx, n, slots, d_left, d_right, motion);
    });
}

int tsgm_step_device_after(tsgm_ctx* ctx, int32_t n, const int32_t* slots,
                           const uint8_t* const* d_left, const uint8_t* const* d_right,
                           const double* motion, void* producer_stream) {
    return guarded([&] {
        if (!ctx || !slots || !d_left || !d_right || !motion) bad("tsgm_step_device: null argument");
        CK(cudaSetDevice(ctx->device));
        // the step's kernels start only after the work enqueued so far on the
        // producer stream (e.g. the copy or kernel that filled the images)
        CK(cudaEventRecord(ctx->ev_inputs, static_cast<cudaStream_t>(producer_stream)));
        CK(cudaStreamWaitEvent(ctx->st, ctx->ev_inputs, 0));
        step_impl(ctx, n, slots, d_left, d_right, motion);
    });
}

int tsgm_inputs_consumed(tsgm_ctx* ctx, void* consumer_stream) {
    return guarded([&] {
        if (!ctx) bad("tsgm_inputs_consumed: null argument");
        CK(cudaSetDevice(ctx->device));
        if (ctx->consumed_recorded)
            CK(cudaStreamWaitEvent(static_cast<cudaStream_t>(consumer_stream), ctx->ev_consumed, 0));
    });
}

int tsgm_last_chunks(tsgm_ctx* ctx, int32_t* chunks) {
    return guarded([&] {
        if (!ctx || !chunks) bad("tsgm_last_chunks: null argument");
        *chunks = ctx->last_chunks;
    });
}

int tsgm_last_kernels(tsgm_ctx* ctx, char* buf, size_t cap) {
    return guarded([&] {
        if (!ctx || !buf || cap == 0) bad("tsgm_last_kernels: null argument");
        std::snprintf(buf, cap, "%s", ctx->last_kernels.c_str());
    });
}

int tsgm_last_stage_timings(tsgm_ctx* ctx, tsgm_stage_timings* out) {
    return guarded([&] {
        if (!ctx || !out) bad("tsgm_last_stage_timings: null argument");
        if (!ctx->stage_timing) bad("tsgm_last_stage_timings: context created without TSGM_STAGE_TIMINGS");
        CK(cudaSetDevice(ctx->device));
        double t[kStCount];
        ctx->stage_seconds(t);
        fill_timings(t, out);
    });
}

int tsgm_fetch(tsgm_ctx* ctx, int32_t slot, int32_t what, void* dst, size_t bytes) {
    return guarded([&] {
        if (slot < 0 || slot >= ctx->max_slots) bad("tsgm_fetch: slot out of range");
        CK(cudaSetDevice(ctx->device));
        const OutDesc o = out_desc(ctx, what);
        size_t count = o.stride;
        size_t pos = static_cast<size_t>(slot);
        size_t first = pos * o.stride;  // first element
        if (what == TSGM_OUT_COST || what == TSGM_OUT_AGG) {
            count = cells_of(ctx, slot);
            pos = static_cast<size_t>(vol_pos(ctx, slot));
            if (what == TSGM_OUT_COST) {
                // the reference layout from the census of the slot's last step
                ensure_ragged_cost(ctx);
                Bufs one = chunk_bufs(ctx->b, ctx->last_c0 + static_cast<int>(pos));
                one.vbase = ctx->b.vbase + pos;
                one.vqbase = ctx->b.vqbase + pos;
                launch_cost_ragged(one, 1, ctx->L());
            }
            unsigned long long vb = 0;
            CK(cudaMemcpyAsync(&vb, ctx->d_vb + pos, sizeof vb, cudaMemcpyDeviceToHost, ctx->st));
            CK(cudaStreamSynchronize(ctx->st));
            first = static_cast<size_t>(vb);
        }
        if (bytes < count * o.elem) bad("tsgm_fetch: destination too small");
        const void* base = what == TSGM_OUT_COST ? static_cast<const void*>(ctx->b.cost) : o.base;
        const char* src = static_cast<const char*>(base) + first * o.elem;
        CK(cudaMemcpyAsync(dst, src, count * o.elem, cudaMemcpyDeviceToHost, ctx->st));
        sync(ctx);
    });
}

int tsgm_fetch_batch(tsgm_ctx* ctx, int32_t n, const int32_t* slots, int32_t what,
                     void* const* dsts, size_t bytes_each) {
    return guarded([&] {
        if (what == TSGM_OUT_COST || what == TSGM_OUT_AGG) bad("tsgm_fetch_batch: volumes need tsgm_fetch");
        CK(cudaSetDevice(ctx->device));
        const OutDesc o = out_desc(ctx, what);
        if (bytes_each < o.stride * o.elem) bad("tsgm_fetch_batch: destination too small");
        for (int i = 0; i < n; ++i)
            if (slots[i] < 0 || slots[i] >= ctx->max_slots) bad("tsgm_fetch_batch: slot out of range");
        const size_t bytes = o.stride * o.elem;
        const bool direct = what == TSGM_OUT_STATE_D || what == TSGM_OUT_STATE_P ||
                            what == TSGM_OUT_STATE_VALID || what == TSGM_OUT_EXPORT_D ||
                            what == TSGM_OUT_EXPORT_VALID || what == TSGM_OUT_DIFF ||
                            what == TSGM_OUT_MASK;
        if (!direct) {
            if (!ctx->snap[what]) ctx->snap[what] = ctx->dalloc<char>(bytes * ctx->max_slots);
            // the kind's previous copy-out must have left the snapshot
            if (ctx->snap_pending[what]) CK(cudaStreamWaitEvent(ctx->st, ctx->ev_snap_copied[what], 0));
        }
        // runs of consecutive slots with contiguous destinations: one copy each
        std::vector<std::pair<int, int>> runs;  // (first batch index, length)
        for (int i = 0; i < n; ++i) {
            if (!runs.empty()) {
                auto& r = runs.back();
                const int j = r.first + r.second - 1;
                if (slots[i] == slots[j] + 1 &&
                    static_cast<char*>(dsts[i]) == static_cast<char*>(dsts[j]) + bytes) {
                    ++r.second;
                    continue;
                }
            }
            runs.push_back({i, 1});
        }
        const char* src = direct ? static_cast<const char*>(o.base) : static_cast<char*>(ctx->snap[what]);
        if (!direct)
            for (auto& r : runs) {
                const size_t at = static_cast<size_t>(slots[r.first]) * bytes;
                CK(cudaMemcpyAsync(ctx->snap[what] ? static_cast<char*>(ctx->snap[what]) + at : nullptr,
                                   static_cast<const char*>(o.base) + at, bytes * r.second,
                                   cudaMemcpyDeviceToDevice, ctx->st));
            }
        CK(cudaEventRecord(ctx->ev_frame, ctx->st));
        CK(cudaStreamWaitEvent(ctx->copy_st, ctx->ev_frame, 0));
        for (auto& r : runs) {
            const size_t at = static_cast<size_t>(slots[r.first]) * bytes;
            CK(cudaMemcpyAsync(dsts[r.first], src + at, bytes * r.second, cudaMemcpyDeviceToHost,
                               ctx->copy_st));
        }
        if (direct) {
            CK(cudaEventRecord(ctx->ev_direct_copied, ctx->copy_st));
            ctx->direct_pending = true;
        } else {
            CK(cudaEventRecord(ctx->ev_snap_copied[what], ctx->copy_st));
            ctx->snap_pending[what] = true;
        }
    });
}

int tsgm_cells(tsgm_ctx* ctx, int32_t slot, uint64_t* n_cells) {
    return guarded([&] {
        if (slot < 0 || slot >= ctx->max_slots) bad("tsgm_cells: slot out of range");
        CK(cudaSetDevice(ctx->device));
        *n_cells = cells_of(ctx, slot);
    });
}

int tsgm_sync(tsgm_ctx* ctx) {
    return guarded([&] {
        CK(cudaSetDevice(ctx->device));
        sync(ctx);
    });
}

int tsgm_timer_begin(tsgm_ctx* ctx) {
    return guarded([&] { CK(cudaEventRecord(ctx->ev0, ctx->st)); });
}

int tsgm_timer_end(tsgm_ctx* ctx, float* ms) {
    return guarded([&] {
        CK(cudaEventRecord(ctx->ev1, ctx->st));
        CK(cudaEventSynchronize(ctx->ev1));
        CK(cudaEventElapsedTime(ms, ctx->ev0, ctx->ev1));
    });
}

int tsgm_bench_aggregate(tsgm_ctx* ctx, int32_t n, const int32_t* slots, int32_t reps,
                         float* ms_per_launch, uint64_t* cells) {
    return guarded([&] {
        check_slots(ctx, n, slots);
        if (n > static_cast<int>(ctx->vol_owner.size()))
            bad("tsgm_bench_aggregate: more slots than the volume working set");
        for (int i = 0; i < n; ++i)
            if (ctx->vol_owner[i] != slots[i])
                bad("tsgm_bench_aggregate: slots must be the last volume chunk, in step order");
        CK(cudaSetDevice(ctx->device));
        std::vector<const uint8_t*> dl(n, ctx->d_img), dr(n, ctx->d_img);
        std::vector<double> H(16 * static_cast<size_t>(n), 0.0);
        upload_step(ctx, n, slots, dl.data(), dr.data(), H.data());
        Launch L{ctx->st, &ctx->launches};  // (no stage marks)
        // (the same kernel choice as the step that built these volumes)
        const bool full = ctx->last_full;
        aggregate(ctx, ctx->b, n, L, false, true, full);  // warm
        CK(cudaEventRecord(ctx->ev0, ctx->st));
        for (int r = 0; r < reps; ++r) aggregate(ctx, ctx->b, n, L, false, true, full);
        CK(cudaEventRecord(ctx->ev1, ctx->st));
        CK(cudaEventSynchronize(ctx->ev1));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
        *ms_per_launch = ms / std::max(1, reps);
        unsigned long long total = 0;
        for (int i = 0; i < n; ++i) total += cells_of(ctx, slots[i]);
        *cells = total;
    });
}

int tsgm_volume_slots(tsgm_ctx* ctx, int32_t* vol_slots) {
    return guarded([&] {
        if (!ctx || !vol_slots) bad("tsgm_volume_slots: null argument");
        *vol_slots = ctx->vol_slots;
    });
}

uint64_t tsgm_launch_count(tsgm_ctx* ctx) { return ctx ? ctx->launches : 0; }

// ---------------------------------------------------------------- stage API
int tsgm_census_transform(const uint8_t* img, int32_t w, int32_t h, uint32_t* sig) {
    return guarded([&] {
        if (w < 2 * kCensusRadius + 1 || h < 2 * kCensusRadius + 1)
            bad("census_transform: image smaller than the 5x5 window");
        auto ctx = scratch(w, h, 1);
        h2d(ctx.get(), ctx->d_img, img, ctx->P);
        h2d(ctx.get(), ctx->d_img + ctx->P, img, ctx->P);
        launch_census(ctx->b, 1, ctx->L());
        d2h(ctx.get(), sig, ctx->b.sigl, ctx->P);
        sync(ctx.get());
    });
}

int tsgm_build_cost_volume(const uint8_t* left, const uint8_t* right, int32_t w, int32_t h,
                           const uint16_t* lo, const uint16_t* hi, uint32_t* offsets,
                           uint8_t* cost, uint64_t cap) {
    return guarded([&] {
        if (w < 2 * kCensusRadius + 1 || h < 2 * kCensusRadius + 1)
            bad("census_transform: image smaller than the 5x5 window");
        int max_hi = 0;
        const unsigned long long total = ranges_total(lo, hi, static_cast<size_t>(w) * h, &max_hi);
        if (total > cap) bad("tsgm_build_cost_volume: capacity too small");
        auto ctx = scratch(w, h, max_hi + 1);
        tsgm_ctx* c = ctx.get();
        h2d(c, c->d_img, left, c->P);
        h2d(c, c->d_img + c->P, right, c->P);
        h2d(c, c->b.lo, lo, c->P);
        h2d(c, c->b.hi, hi, c->P);
        launch_ranges_given(c->b, 1, c->L());
        launch_offsets(c->b, 1, c->L());
        launch_census(c->b, 1, c->L());
        launch_cost_ragged(c->b, 1, c->L());
        d2h(c, offsets, c->b.off, c->P + 1);
        d2h(c, cost, c->b.cost, total);
        sync(c);
    });
}

int tsgm_aggregate_paths(const uint8_t* cost, const uint16_t* lo, const uint16_t* hi, int32_t w,
                         int32_t h, const tsgm_sgm_params* params, uint16_t* agg) {
    return guarded([&] {
        sgm_validate(*params);
        int max_hi = 0;
        const unsigned long long total = ranges_total(lo, hi, static_cast<size_t>(w) * h, &max_hi);
        auto ctx = scratch(w, h, max_hi + 1);
        tsgm_ctx* c = ctx.get();
        h2d(c, c->b.lo, lo, c->P);
        h2d(c, c->b.hi, hi, c->P);
        h2d(c, c->b.cost, cost, total);
        launch_ranges_given(c->b, 1, c->L());
        launch_offsets(c->b, 1, c->L());
        c->cfg.sgm = *params;
        aggregate(c, c->b, 1, c->L(), false, true, false, /*cost_in_ragged=*/true);
        d2h(c, agg, c->b.agg, total);
        sync(c);
    });
}

int tsgm_winner_takes_all(const uint16_t* agg, const uint16_t* lo, const uint16_t* hi,
                          int32_t w, int32_t h, int32_t* d, uint8_t* valid) {
    return guarded([&] {
        int max_hi = 0;
        const unsigned long long total = ranges_total(lo, hi, static_cast<size_t>(w) * h, &max_hi);
        auto ctx = scratch(w, h, max_hi + 1);
        tsgm_ctx* c = ctx.get();
        h2d(c, c->b.lo, lo, c->P);
        h2d(c, c->b.hi, hi, c->P);
        h2d(c, c->b.agg, agg, total);
        launch_ranges_given(c->b, 1, c->L());
        launch_offsets(c->b, 1, c->L());
        launch_wta(c->b, 1, c->L());
        d2h(c, d, c->b.md, c->P);
        d2h(c, valid, c->b.mv, c->P);
        sync(c);
    });
}

int tsgm_median_refine(const int32_t* d, const uint8_t* valid, int32_t w, int32_t h,
                       int32_t* out_d, uint8_t* out_valid) {
    return guarded([&] {
        auto ctx = scratch(w, h, 1);
        tsgm_ctx* c = ctx.get();
        h2d(c, c->b.rd, d, c->P);
        h2d(c, c->b.rv, valid, c->P);
        launch_median(c->b, 1, c->b.rd, c->b.rv, c->b.ed, c->b.ev, c->L());
        d2h(c, out_d, c->b.ed, c->P);
        d2h(c, out_valid, c->b.ev, c->P);
        sync(c);
    });
}

int tsgm_sgm_match_t(const uint8_t* left, const uint8_t* right, int32_t w, int32_t h,
                     const uint16_t* lo, const uint16_t* hi, const tsgm_sgm_params* params,
                     int32_t* d, uint8_t* valid, tsgm_stage_timings* timings) {
    return guarded([&] {
        // sgm_match, sgm.cpp:229-234: params, then ranges.validate(d_max)
        sgm_validate(*params);
        const size_t P = static_cast<size_t>(w) * h;
        for (size_t i = 0; i < P; ++i)
            if (lo[i] > hi[i] || hi[i] >= params->d_max) bad("SearchRangeMap: range outside [0, d_max)");
        if (w < 2 * kCensusRadius + 1 || h < 2 * kCensusRadius + 1)
            bad("census_transform: image smaller than the 5x5 window");
        auto ctx = scratch(w, h, params->d_max);
        tsgm_ctx* c = ctx.get();
        c->stage_timing = timings != nullptr;
        h2d(c, c->d_img, left, P);
        h2d(c, c->d_img + P, right, P);
        h2d(c, c->b.lo, lo, P);
        h2d(c, c->b.hi, hi, P);
        c->tev_used = 0;
        c->mark(-1);
        // sgm.cpp:236-255: census, cost (make_cost_volume + matching costs),
        // aggregate, WTA
        launch_census(c->b, 1, c->L());
        c->mark(kStCensus);
        launch_ranges_given(c->b, 1, c->L());
        launch_offsets(c->b, 1, c->L());
        launch_cost(c->b, 1, c->L());
        c->mark(kStCost);
        c->cfg.sgm = *params;
        aggregate(c, c->b, 1, c->L());
        launch_wta(c->b, 1, c->L());
        c->mark(kStWta);
        d2h(c, d, c->b.md, P);
        d2h(c, valid, c->b.mv, P);
        sync(c);
        if (timings) {
            double t[kStCount];
            c->stage_seconds(t);
            fill_timings(t, timings);
        }
    });
}

int tsgm_sgm_match(const uint8_t* left, const uint8_t* right, int32_t w, int32_t h,
                   const uint16_t* lo, const uint16_t* hi, const tsgm_sgm_params* params,
                   int32_t* d, uint8_t* valid) {
    return tsgm_sgm_match_t(left, right, w, h, lo, hi, params, d, valid, nullptr);
}

int tsgm_relative_motion(const double* prev12, const double* cur12, double* r9, double* t3) {
    return guarded([&] { relative_motion(prev12, cur12, r9, t3); });
}

int tsgm_disparity_homography(const double* r9, const double* t3,
                              const tsgm_stereo_calib* calib, double* h16) {
    return guarded([&] { homography(r9, t3, *calib, h16); });
}

int tsgm_warp_state_ex(const double* d, const double* p, const uint8_t* valid, int32_t w,
                       int32_t h, const double* h16, int32_t d_max, double* od, double* op,
                       uint8_t* ov, double* source_d) {
    return guarded([&] {
        auto ctx = scratch(w, h, 1);
        tsgm_ctx* c = ctx.get();
        const size_t P = c->P;
        const int zero = 0;
        const uint8_t* img = c->d_img;
        upload_step(c, 1, &zero, &img, &img, h16);
        h2d(c, c->b.sd, d, P);
        h2d(c, c->b.sp, p, P);
        h2d(c, c->b.sv, valid, P);
        launch_warp(c->b, 1, c->b.sd, c->b.sp, c->b.sv, d_max, c->L());
        launch_predict_finalize(c->b, 1, 0.0, 0, c->L());
        d2h(c, od, c->b.wd, P);
        d2h(c, op, c->b.wp, P);
        d2h(c, ov, c->b.wv, P);
        d2h(c, source_d, c->b.wsrc, P);
        sync(c);
    });
}

int tsgm_predict(const double* d, const double* p, const uint8_t* valid, int32_t w, int32_t h,
                 const double* r9, const double* t3, const tsgm_stereo_calib* calib,
                 const tsgm_filter_config* cfg, double* od, double* op, uint8_t* ov) {
    return guarded([&] {
        double H[16];
        homography(r9, t3, *calib, H);
        auto ctx = scratch(w, h, 1);
        tsgm_ctx* c = ctx.get();
        const size_t P = c->P;
        const int zero = 0;
        const uint8_t* img = c->d_img;
        upload_step(c, 1, &zero, &img, &img, H);
        h2d(c, c->b.sd, d, P);
        h2d(c, c->b.sp, p, P);
        h2d(c, c->b.sv, valid, P);
        launch_warp(c->b, 1, c->b.sd, c->b.sp, c->b.sv, calib->d_max, c->L());
        launch_predict_finalize(c->b, 1, cfg->q, 1, c->L());
        launch_reject_fill(c->b, 1, c->b.wd, c->b.wp, c->b.wv, c->b.pd, c->b.pp, c->b.pv,
                           cfg->disc_thresh, 1, 1, c->L());
        d2h(c, od, c->b.pd, P);
        d2h(c, op, c->b.pp, P);
        d2h(c, ov, c->b.pv, P);
        sync(c);
    });
}

static int reject_fill_api(const double* d, const double* p, const uint8_t* valid, int32_t w,
                           int32_t h, double thr, int rej, int fil, double* od, double* op,
                           uint8_t* ov) {
    return guarded([&] {
        auto ctx = scratch(w, h, 1);
        tsgm_ctx* c = ctx.get();
        const size_t P = c->P;
        h2d(c, c->b.wd, d, P);
        h2d(c, c->b.wp, p, P);
        h2d(c, c->b.wv, valid, P);
        launch_reject_fill(c->b, 1, c->b.wd, c->b.wp, c->b.wv, c->b.pd, c->b.pp, c->b.pv, thr, rej,
                           fil, c->L());
        d2h(c, od, c->b.pd, P);
        d2h(c, op, c->b.pp, P);
        d2h(c, ov, c->b.pv, P);
        sync(c);
    });
}

int tsgm_reject_discontinuities(const double* d, const double* p, const uint8_t* valid,
                                int32_t w, int32_t h, const tsgm_filter_config* cfg, double* od,
                                double* op, uint8_t* ov) {
    return reject_fill_api(d, p, valid, w, h, cfg->disc_thresh, 1, 0, od, op, ov);
}

int tsgm_fill_zoom_holes(const double* d, const double* p, const uint8_t* valid, int32_t w,
                         int32_t h, double* od, double* op, uint8_t* ov) {
    return reject_fill_api(d, p, valid, w, h, 0.0, 0, 1, od, op, ov);
}

int tsgm_derive_search_ranges(const double* d, const double* p, const uint8_t* valid, int32_t w,
                              int32_t h, const tsgm_stereo_calib* calib,
                              const tsgm_filter_config* cfg, uint16_t* lo, uint16_t* hi) {
    return guarded([&] {
        auto ctx = scratch(w, h, calib->d_max);
        tsgm_ctx* c = ctx.get();
        const size_t P = c->P;
        h2d(c, c->b.pd, d, P);
        h2d(c, c->b.pp, p, P);
        h2d(c, c->b.pv, valid, P);
        launch_ranges_from_pred(c->b, 1, cfg->min_range_halfwidth, cfg->range_use_stddev,
                                cfg->range_stddev_gain, c->L());
        d2h(c, lo, c->b.lo, P);
        d2h(c, hi, c->b.hi, P);
        sync(c);
    });
}

int tsgm_correct(const double* d, const double* p, const uint8_t* valid, const int32_t* md,
                 const uint8_t* mv, int32_t w, int32_t h, const tsgm_filter_config* cfg,
                 double* od, double* op, uint8_t* ov) {
    return guarded([&] {
        auto ctx = scratch(w, h, 1);
        tsgm_ctx* c = ctx.get();
        const size_t P = c->P;
        h2d(c, c->b.pd, d, P);
        h2d(c, c->b.pp, p, P);
        h2d(c, c->b.pv, valid, P);
        h2d(c, c->b.md, md, P);
        h2d(c, c->b.mv, mv, P);
        launch_correct(c->b, 1, cfg->r, 3.0, c->L());
        d2h(c, od, c->b.sd, P);
        d2h(c, op, c->b.sp, P);
        d2h(c, ov, c->b.sv, P);
        sync(c);
    });
}

int tsgm_step_once(const double* sd, const double* sp, const uint8_t* sv, int32_t state_w,
                   int32_t state_h, const uint8_t* left, const uint8_t* right, int32_t w,
                   int32_t h, const double* r9, const double* t3,
                   const tsgm_stereo_calib* calib, const tsgm_sgm_params* params,
                   const tsgm_filter_config* cfg, double* od, double* op, uint8_t* ov,
                   int32_t* ed, uint8_t* ev, double* diff) {
    return tsgm_step_once_t(sd, sp, sv, state_w, state_h, left, right, w, h, r9, t3, calib, params,
                            cfg, od, op, ov, ed, ev, diff, nullptr);
}

int tsgm_step_once_t(const double* sd, const double* sp, const uint8_t* sv, int32_t state_w,
                     int32_t state_h, const uint8_t* left, const uint8_t* right, int32_t w,
                     int32_t h, const double* r9, const double* t3,
                     const tsgm_stereo_calib* calib, const tsgm_sgm_params* params,
                     const tsgm_filter_config* cfg, double* od, double* op, uint8_t* ov,
                     int32_t* ed, uint8_t* ev, double* diff, tsgm_stage_timings* timings) {
    return guarded([&] {
        // step(), temporal_filter.cpp:198-206
        const bool empty = state_w == 0 && state_h == 0;
        if (!empty && (state_w != w || state_h != h)) bad("step: state dimension mismatch");
        if (params->d_max != calib->d_max) bad("step: params.d_max disagrees with calibration");
        tsgm_config c{};
        c.width = w;
        c.height = h;
        c.max_slots = 1;
        CK(cudaGetDevice(&c.device));
        c.calib = *calib;
        // the reference reads only f/cx/cy/b from calib in step; its size
        // fields are validated by disparity_homography but need not equal the
        // image (geometry.cpp:21-28)
        c.sgm = *params;
        c.filter = *cfg;
        c.mask_tau = 3.0;
        double H[16];
        homography(r9, t3, *calib, H);
        sgm_validate(*params);
        if (w < 2 * kCensusRadius + 1 || h < 2 * kCensusRadius + 1)
            bad("census_transform: image smaller than the 5x5 window");
        if (1ull * w * h * params->d_max > 0xffffffffull)
            bad("CostVolume: volume exceeds 32-bit addressing");
        thread_local std::unique_ptr<tsgm_ctx> cache;
        if (!cache || std::memcmp(&cache->cfg, &c, sizeof c) != 0) {
            cache.reset();
            auto ctx = std::make_unique<tsgm_ctx>();
            init_ctx(ctx.get(), c);
            cache = std::move(ctx);
        }
        tsgm_ctx* x = cache.get();
        const size_t P = x->P;
        x->fresh[0] = (empty || !sv) ? 1 : 0;
        if (empty || !sv) {
            CK(cudaMemsetAsync(x->b.sd, 0, 8 * P, x->st));
            CK(cudaMemsetAsync(x->b.sp, 0, 8 * P, x->st));
            CK(cudaMemsetAsync(x->b.sv, 0, P, x->st));
        } else {
            h2d(x, x->b.sd, sd, P);
            h2d(x, x->b.sp, sp, P);
            h2d(x, x->b.sv, sv, P);
        }
        h2d(x, x->d_img, left, P);
        h2d(x, x->d_img + P, right, P);
        const int zero = 0;
        const uint8_t* l = x->d_img;
        const uint8_t* r = x->d_img + P;
        upload_step(x, 1, &zero, &l, &r, H);
        x->stage_timing = timings != nullptr;
        run_step(x, 1);
        d2h(x, od, x->b.sd, P);
        d2h(x, op, x->b.sp, P);
        d2h(x, ov, x->b.sv, P);
        d2h(x, ed, x->b.ed, P);
        d2h(x, ev, x->b.ev, P);
        d2h(x, diff, x->b.diff, P);
        sync(x);
        if (timings) {
            double t[kStCount];
            x->stage_seconds(t);
            fill_timings(t, timings);
        }
    });
}


// ---------------------------------------------------------------- box detector
}  // extern "C"

namespace {

// DetectConfig::validate (motion_detect.cpp:11-23), same messages.
void detect_validate(const tsgm_detect_config* c) {
    if (!c) bad("DetectConfig: null configuration");
    if (c->n_windows < 1 || !c->window_wh) bad("DetectConfig: no window sizes");
    if (c->n_windows > kMaxDetectWindows) bad("DetectConfig: at most 64 window sizes (GPU limit, INTEGRATION.md)");
    for (int i = 0; i < c->n_windows; ++i)
        if (c->window_wh[2 * i] < 1 || c->window_wh[2 * i + 1] < 1)
            bad("DetectConfig: non-positive window size");
    if (!(c->score_thresh > 0.0)) bad("DetectConfig: score_thresh must be positive");
    if (!(c->merge_stop_iou > 0.0 && c->merge_stop_iou < 1.0))
        bad("DetectConfig: merge_stop_iou must lie in (0, 1)");
    if (c->min_box_area < 0) bad("DetectConfig: negative min_box_area");
}

// Device scratch for the stateless detector calls.
struct DevScratch {
    std::vector<void*> p;
    cudaStream_t st = nullptr;
    unsigned long long launches = 0;
    DevScratch() { CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking)); }
    ~DevScratch() {
        if (st) cudaStreamSynchronize(st);
        for (void* q : p) cudaFree(q);
        if (st) cudaStreamDestroy(st);
    }
    template <typename T>
    T* alloc(size_t n) {
        void* q = nullptr;
        CK(cudaMalloc(&q, sizeof(T) * std::max<size_t>(n, 1)));
        p.push_back(q);
        return static_cast<T*>(q);
    }
    Launch L() { return Launch{st, &launches}; }
};

// SAT + candidates of one host map on the GPU; returns the full count and
// fills `boxes` with all of them.
long long candidates_one(const double* diff, int w, int h, const tsgm_detect_config& c,
                         std::vector<tsgm_box>& boxes) {
    boxes.clear();
    DetectWindows dw;
    detect_windows(c, w, h, dw);
    const long long total = dw.base[dw.n];
    if (total == 0) return 0;
    DevScratch d;
    const size_t P = static_cast<size_t>(w) * h, SP = static_cast<size_t>(w + 1) * (h + 1);
    double* m = d.alloc<double>(P);
    double* sat = d.alloc<double>(SP);
    tsgm_box* out = d.alloc<tsgm_box>(static_cast<size_t>(total));
    long long* cnt = d.alloc<long long>(1);
    CK(cudaMemcpyAsync(m, diff, sizeof(double) * P, cudaMemcpyHostToDevice, d.st));
    launch_sat(m, P, sat, SP, w, h, 1, nullptr, d.L());
    launch_candidates(sat, SP, w, dw, 1, out, total, cnt, d.L());
    CK(cudaGetLastError());
    long long n = 0;
    CK(cudaMemcpyAsync(&n, cnt, sizeof n, cudaMemcpyDeviceToHost, d.st));
    CK(cudaStreamSynchronize(d.st));
    boxes.resize(static_cast<size_t>(n));
    if (n) CK(cudaMemcpy(boxes.data(), out, sizeof(tsgm_box) * n, cudaMemcpyDeviceToHost));
    return n;
}

}  // namespace

extern "C" {

int tsgm_integral_image(const double* map, int32_t w, int32_t h, double* sat) {
    return guarded([&] {
        if (!sat || (w > 0 && h > 0 && !map)) bad("integral_image: null argument");
        if (w < 0 || h < 0) bad("integral_image: negative size");
        const size_t SP = static_cast<size_t>(w + 1) * (h + 1);
        if (w == 0 || h == 0) {
            std::memset(sat, 0, sizeof(double) * SP);
            return;
        }
        DevScratch d;
        const size_t P = static_cast<size_t>(w) * h;
        double* m = d.alloc<double>(P);
        double* s = d.alloc<double>(SP);
        CK(cudaMemcpyAsync(m, map, sizeof(double) * P, cudaMemcpyHostToDevice, d.st));
        launch_sat(m, P, s, SP, w, h, 1, nullptr, d.L());
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(sat, s, sizeof(double) * SP, cudaMemcpyDeviceToHost, d.st));
        CK(cudaStreamSynchronize(d.st));
    });
}

int tsgm_detect_candidate_windows(const double* diff, int32_t w, int32_t h,
                                  const tsgm_detect_config* cfg, tsgm_box* out, int64_t cap,
                                  int64_t* n_out) {
    return guarded([&] {
        detect_validate(cfg);
        if (!n_out || (cap > 0 && !out)) bad("detect_candidate_windows: null argument");
        if (w < 1 || h < 1 || !diff) bad("detect_candidate_windows: empty map");
        std::vector<tsgm_box> boxes;
        const long long n = candidates_one(diff, w, h, *cfg, boxes);
        std::memcpy(out, boxes.data(), sizeof(tsgm_box) * static_cast<size_t>(std::min<long long>(n, cap)));
        *n_out = n;
    });
}

int tsgm_greedy_merge(tsgm_box* boxes, int64_t n, const tsgm_detect_config* cfg, int64_t* n_out) {
    return guarded([&] {
        detect_validate(cfg);
        if (!n_out || (n > 0 && !boxes) || n < 0) bad("greedy_merge: bad arguments");
        *n_out = greedy_merge_host(boxes, n, *cfg);
    });
}

int tsgm_detect_moving_objects(const double* diff, int32_t w, int32_t h,
                               const tsgm_detect_config* cfg, tsgm_box* out, int64_t cap,
                               int64_t* n_out) {
    return guarded([&] {
        detect_validate(cfg);
        if (!n_out || (cap > 0 && !out)) bad("detect_moving_objects: null argument");
        if (w < 1 || h < 1 || !diff) bad("detect_moving_objects: empty map");
        std::vector<tsgm_box> boxes;
        const long long n = candidates_one(diff, w, h, *cfg, boxes);
        const long long m = greedy_merge_host(boxes.data(), n, *cfg);
        std::memcpy(out, boxes.data(), sizeof(tsgm_box) * static_cast<size_t>(std::min<long long>(m, cap)));
        *n_out = m;
    });
}

int tsgm_detect(tsgm_ctx* ctx, int32_t n, const int32_t* slots, const tsgm_detect_config* cfg,
                tsgm_box* out, int64_t cap_each, int64_t* n_each) {
    return guarded([&] {
        detect_validate(cfg);
        if (!ctx || !slots || !n_each || (cap_each > 0 && !out)) bad("tsgm_detect: null argument");
        check_slots(ctx, n, slots);
        CK(cudaSetDevice(ctx->device));
        DetectWindows dw;
        detect_windows(*cfg, ctx->W, ctx->H, dw);
        const long long total = dw.base[dw.n];
        if (total == 0) {
            for (int i = 0; i < n; ++i) n_each[i] = 0;
            return;
        }
        const size_t SP = static_cast<size_t>(ctx->W + 1) * (ctx->H + 1);
        if (!ctx->det_sat) {
            ctx->det_sat = ctx->dalloc<double>(SP * ctx->max_slots);
            ctx->det_counts = ctx->dalloc<long long>(ctx->max_slots);
        }
        if (total > ctx->det_cap) {
            if (ctx->det_boxes) {
                CK(cudaStreamSynchronize(ctx->st));
                CK(cudaFree(ctx->det_boxes));
                ctx->allocs.erase(std::find(ctx->allocs.begin(), ctx->allocs.end(),
                                            static_cast<void*>(ctx->det_boxes)));
            }
            ctx->det_boxes = ctx->dalloc<tsgm_box>(static_cast<size_t>(total) * ctx->max_slots);
            ctx->det_cap = total;
        }
        // this call's slot list (it may differ from the last step's)
        std::vector<const uint8_t*> dl(n, ctx->d_img), dr(n, ctx->d_img);
        std::vector<double> Hm(16 * static_cast<size_t>(n), 0.0);
        upload_step(ctx, n, slots, dl.data(), dr.data(), Hm.data());
        Launch L = ctx->L();
        launch_sat(ctx->b.diff, ctx->P, ctx->det_sat, SP, ctx->W, ctx->H, n, ctx->d_slots, L);
        launch_candidates(ctx->det_sat, SP, ctx->W, dw, n, ctx->det_boxes, ctx->det_cap,
                          ctx->det_counts, L);
        CK(cudaGetLastError());
        std::vector<long long> cnt(n);
        CK(cudaMemcpyAsync(cnt.data(), ctx->det_counts, sizeof(long long) * n,
                           cudaMemcpyDeviceToHost, ctx->st));
        CK(cudaStreamSynchronize(ctx->st));
        std::vector<std::vector<tsgm_box>> boxes(n);
        for (int i = 0; i < n; ++i) {
            boxes[i].resize(static_cast<size_t>(cnt[i]));
            if (cnt[i])
                CK(cudaMemcpyAsync(boxes[i].data(), ctx->det_boxes + static_cast<size_t>(i) * ctx->det_cap,
                                   sizeof(tsgm_box) * cnt[i], cudaMemcpyDeviceToHost, ctx->st));
        }
        CK(cudaStreamSynchronize(ctx->st));
        // host merges, one sequence per worker thread
        const int nt = std::max(1, std::min<int>(n, static_cast<int>(std::thread::hardware_concurrency())));
        std::vector<std::thread> pool;
        std::vector<long long> kept(n, 0);
        for (int t = 0; t < nt; ++t)
            pool.emplace_back([&, t] {
                for (int i = t; i < n; i += nt)
                    kept[i] = greedy_merge_host(boxes[i].data(), cnt[i], *cfg);
            });
        for (auto& th : pool) th.join();
        for (int i = 0; i < n; ++i) {
            n_each[i] = kept[i];
            std::memcpy(out + static_cast<size_t>(i) * cap_each, boxes[i].data(),
                        sizeof(tsgm_box) * static_cast<size_t>(std::min<long long>(kept[i], cap_each)));
        }
    });
}

// ---------------------------------------------------------------- outliers
}  // extern "C"

namespace {
void outlier_validate(const tsgm_outlier_options* o) {
    if (!o) bad("count_outliers: null options");
}
}  // namespace

extern "C" {

int tsgm_count_outliers(const int32_t* d, const uint8_t* valid, const double* gt, int32_t w,
                        int32_t h, const tsgm_outlier_options* opts, int64_t* evaluated,
                        int64_t* outliers) {
    return guarded([&] {
        outlier_validate(opts);
        if (!evaluated || !outliers || w < 0 || h < 0) bad("count_outliers: bad arguments");
        const size_t P = static_cast<size_t>(w) * h;
        if (P == 0) {
            *evaluated = *outliers = 0;
            return;
        }
        if (!d || !valid || !gt) bad("count_outliers: null argument");
        DevScratch s;
        int32_t* dd = s.alloc<int32_t>(P);
        uint8_t* dv = s.alloc<uint8_t>(P);
        double* dg = s.alloc<double>(P);
        unsigned long long* cnt = s.alloc<unsigned long long>(2);
        CK(cudaMemcpyAsync(dd, d, 4 * P, cudaMemcpyHostToDevice, s.st));
        CK(cudaMemcpyAsync(dv, valid, P, cudaMemcpyHostToDevice, s.st));
        CK(cudaMemcpyAsync(dg, gt, 8 * P, cudaMemcpyHostToDevice, s.st));
        launch_count_outliers(dd, dv, dg, P, 1, nullptr, opts->abs_thresh_px, opts->rel_thresh,
                              opts->strict_density, cnt, s.L());
        CK(cudaGetLastError());
        unsigned long long h2[2];
        CK(cudaMemcpyAsync(h2, cnt, sizeof h2, cudaMemcpyDeviceToHost, s.st));
        CK(cudaStreamSynchronize(s.st));
        *evaluated = static_cast<int64_t>(h2[0]);
        *outliers = static_cast<int64_t>(h2[1]);
    });
}

int tsgm_count_outliers_batch(tsgm_ctx* ctx, int32_t n, const int32_t* slots, int32_t what,
                              const double* const* gt, const tsgm_outlier_options* opts,
                              int64_t* evaluated, int64_t* outliers) {
    return guarded([&] {
        outlier_validate(opts);
        if (!ctx || !slots || !gt || !evaluated || !outliers) bad("count_outliers_batch: null argument");
        if (what != TSGM_OUT_EXPORT_D && what != TSGM_OUT_MEAS_D)
            bad("count_outliers_batch: what must be TSGM_OUT_EXPORT_D or TSGM_OUT_MEAS_D");
        check_slots(ctx, n, slots);
        CK(cudaSetDevice(ctx->device));
        const size_t P = ctx->P;
        if (!ctx->eval_gt) {
            ctx->eval_gt = ctx->dalloc<double>(P * ctx->max_slots);
            ctx->eval_counts = ctx->dalloc<unsigned long long>(2 * static_cast<size_t>(ctx->max_slots));
        }
        for (int i = 0; i < n; ++i) {
            if (!gt[i]) bad("count_outliers_batch: null GT map");
            CK(cudaMemcpyAsync(ctx->eval_gt + i * P, gt[i], 8 * P, cudaMemcpyHostToDevice, ctx->st));
        }
        std::vector<const uint8_t*> dl(n, ctx->d_img), dr(n, ctx->d_img);
        std::vector<double> Hm(16 * static_cast<size_t>(n), 0.0);
        upload_step(ctx, n, slots, dl.data(), dr.data(), Hm.data());
        const Bufs& b = ctx->b;
        launch_count_outliers(what == TSGM_OUT_EXPORT_D ? b.ed : b.md,
                              what == TSGM_OUT_EXPORT_D ? b.ev : b.mv, ctx->eval_gt, P, n,
                              ctx->d_slots, opts->abs_thresh_px, opts->rel_thresh,
                              opts->strict_density, ctx->eval_counts, ctx->L());
        CK(cudaGetLastError());
        std::vector<unsigned long long> c(2 * static_cast<size_t>(n));
        CK(cudaMemcpyAsync(c.data(), ctx->eval_counts, sizeof(unsigned long long) * 2 * n,
                           cudaMemcpyDeviceToHost, ctx->st));
        CK(cudaStreamSynchronize(ctx->st));
        for (int i = 0; i < n; ++i) {
            evaluated[i] = static_cast<int64_t>(c[2 * i]);
            outliers[i] = static_cast<int64_t>(c[2 * i + 1]);
        }
    });
}

}  // extern "C"

// ---------------------------------------------------------------- noise calibration
// SURVEY §8(f) row 4 (noise_calib.cpp:102-182): the warp and full-range SGM
// kernels of the step, batched over frames, plus the histogram / error-map
// kernels of noise.cu.
namespace {

void calib_options_validate(const tsgm_calib_options* o) {  // noise_calib.cpp:60-67
    if (!o) bad("CalibOptions: null options");
    if (!(o->outlier_gate_px > 0.0)) bad("CalibOptions: outlier_gate_px must be positive");
    if (!(o->bin_width > 0.0) || o->bin_width > o->outlier_gate_px) bad("CalibOptions: bad bin_width");
    if (!(o->q_floor >= 0.0)) bad("CalibOptions: negative q_floor");
}

HistSpec hist_spec(const tsgm_calib_options* o) {  // ErrorHistogram(-gate, gate, bw), :9-14
    HistSpec hs{};
    hs.lo = -o->outlier_gate_px;
    hs.hi = o->outlier_gate_px;
    hs.bw = o->bin_width;
    if (!(hs.hi > hs.lo) || !(hs.bw > 0.0)) bad("ErrorHistogram: bad bin layout");
    const double nb = std::ceil((hs.hi - hs.lo) / hs.bw);
    if (!(nb >= 1.0 && nb <= double(1 << 26))) bad("ErrorHistogram: bad bin layout");
    hs.nbins = static_cast<int>(nb);
    return hs;
}

constexpr int kNoiseBatch = 8;  // frames (or frame pairs) per batched launch (memory: ~8 volumes)

// A context for the calibration stages: images, state and per-pixel buffers
// for `slots` frames; volumes only when sgm is given (measurement noise).
std::unique_ptr<tsgm_ctx> noise_ctx(int w, int h, int slots, const tsgm_sgm_params* sgm) {
    tsgm_config c{};
    c.width = w;
    c.height = h;
    c.max_slots = slots;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    c.device = dev;
    const int dv = sgm ? sgm->d_max : 1;
    c.calib = tsgm_stereo_calib{1.0, 0.0, 0.0, 1.0, w, h, dv};
    c.sgm = sgm ? *sgm : tsgm_sgm_params{6, 65, 8, 0, dv};
    c.mask_tau = 3.0;
    c.vol_slots = sgm ? 0 : 1;
    auto ctx = std::make_unique<tsgm_ctx>();
    init_ctx(ctx.get(), c);
    return ctx;
}

// The calibration functions are stateless like the reference's, but their
// working set (a batch of frames' state, maps and, for the measurement noise,
// volumes: GBs) is kept between calls with the same geometry — allocating it
// per call cost more than the calibration itself. One cache entry per kind
// (0: warped ground-truth pairs, 1: full-range matching), guarded by a mutex
// (concurrent calls serialise); tsgm_calib_release() frees them.
struct CalibCache {
    std::unique_ptr<tsgm_ctx> ctx;
    int dev = -1, w = 0, h = 0, slots = 0;
    tsgm_sgm_params sgm{};
    double* dgt = nullptr;             // (slots + 1) * P ground truth staging
    double* dacc = nullptr;            // P, error map
    unsigned long long* dsmall = nullptr;  // error-map overlap; histogram tallies
    double* dsums = nullptr;           // 2 + partials
    unsigned long long* dcounts = nullptr;
    int counts_cap = 0;
};
std::mutex g_calib_mu;
// never destroyed: at process exit the CUDA runtime may already be gone
CalibCache* const g_calib = new CalibCache[2];

CalibCache& calib_cache(int kind, int w, int h, int slots, const tsgm_sgm_params* sgm) {
    CalibCache& c = g_calib[kind];
    int dev = 0;
    CK(cudaGetDevice(&dev));
    const bool same = c.ctx && c.dev == dev && c.w == w && c.h == h && c.slots == slots &&
                      (!sgm || std::memcmp(&c.sgm, sgm, sizeof *sgm) == 0);
    if (!same) {
        c = CalibCache{};
        c.ctx = noise_ctx(w, h, slots, sgm);
        c.dev = dev;
        c.w = w;
        c.h = h;
        c.slots = slots;
        if (sgm) c.sgm = *sgm;
        const size_t P = static_cast<size_t>(w) * h;
        c.dgt = c.ctx->dalloc<double>((slots + 1) * P);
        if (kind == 0) c.dacc = c.ctx->dalloc<double>(P);
        c.dsmall = c.ctx->dalloc<unsigned long long>(8);
        c.dsums = c.ctx->dalloc<double>(2 + hist_partial_doubles());
    }
    return c;
}

// Run fn under the cache lock; any failure drops the entry (its device state
// may be half-written).
template <typename Fn>
void with_calib_cache(int kind, Fn&& fn) {
    std::lock_guard<std::mutex> lk(g_calib_mu);
    try {
        fn();
    } catch (...) {
        g_calib[kind] = CalibCache{};
        throw;
    }
}

struct NoiseAccum {
    HistSpec hs;
    HistAcc acc;
    tsgm_ctx* ctx;
    NoiseAccum(CalibCache& c, const HistSpec& h) : hs(h), ctx(c.ctx.get()) {
        if (c.counts_cap < h.nbins) {  // grows only (a cached context's allocation)
            c.dcounts = ctx->dalloc<unsigned long long>(h.nbins);
            c.counts_cap = h.nbins;
        }
        acc.counts = c.dcounts;
        acc.tallies = c.dsmall;
        acc.sums = c.dsums;
        acc.partial = c.dsums + 2;
        CK(cudaMemsetAsync(acc.counts, 0, sizeof(unsigned long long) * h.nbins, ctx->st));
        CK(cudaMemsetAsync(acc.tallies, 0, sizeof(unsigned long long) * 4, ctx->st));
        CK(cudaMemsetAsync(acc.sums, 0, sizeof(double) * 2, ctx->st));
    }
    // NoiseEstimate (noise_calib.cpp:91-99: finish) from the device tallies
    void finish(tsgm_noise_estimate* out, const char* who) {
        std::vector<unsigned long long> counts(hs.nbins);
        unsigned long long tal[4];
        double sums[2];
        CK(cudaMemcpyAsync(counts.data(), acc.counts, sizeof(unsigned long long) * hs.nbins,
                           cudaMemcpyDeviceToHost, ctx->st));
        CK(cudaMemcpyAsync(tal, acc.tallies, sizeof tal, cudaMemcpyDeviceToHost, ctx->st));
        CK(cudaMemcpyAsync(sums, acc.sums, sizeof sums, cudaMemcpyDeviceToHost, ctx->st));
        CK(cudaStreamSynchronize(ctx->st));
        CK(cudaGetLastError());
        const long long gated = static_cast<long long>(tal[3]);
        const long long total = gated + static_cast<long long>(tal[0] + tal[1]);
        if (total == 0) throw std::runtime_error(std::string(who) + ": no overlapping valid pixels");
        double var = 0.0;  // ErrorHistogram::variance, noise_calib.cpp:45-52
        if (gated >= 2) {
            const double n = static_cast<double>(gated);
            const double m = sums[0] / n;
            const double v = (sums[1] - n * m * m) / (n - 1.0);
            var = v > 0.0 ? v : 0.0;
        }
        out->variance = var;
        out->samples_used = gated;
        out->lo = hs.lo;
        out->hi = hs.hi;
        out->bin_width = hs.bw;
        out->underflow = static_cast<int64_t>(tal[0]);
        out->overflow = static_cast<int64_t>(tal[1]);
        out->within_1px = static_cast<int64_t>(tal[2]);
        out->total = total;
        out->sum = sums[0];
        out->sum_sq = sums[1];
        if (out->counts)
            for (int k = 0; k < hs.nbins; ++k) out->counts[k] = static_cast<int64_t>(counts[k]);
        out->n_bins = hs.nbins;
    }
};

// Frame pairs (k, k+1), k = 0 .. n-2, in batches: slot i holds state_from_gt
// of frame k0+i warped by relative_motion(pose k0+i, pose k0+i+1)
// (noise_calib.cpp:115-119); fn(cache, gt of frames k0+1 .., m) consumes them.
template <typename Begin, typename Fn, typename End>
void warp_gt_pairs(int n, int w, int h, const double* gt, const double* poses,
                   const tsgm_stereo_calib& calib, Begin&& begin, Fn&& fn, End&& end) {
    const size_t P = static_cast<size_t>(w) * h;
    const int pairs = n - 1;
    // validate every pair's motion + homography first (what the reference's
    // loop would throw on)
    std::vector<double> H(16 * static_cast<size_t>(pairs));
    for (int k = 0; k < pairs; ++k) {
        double r9[9], t3[3];
        relative_motion(poses + 12 * k, poses + 12 * (k + 1), r9, t3);
        homography(r9, t3, calib, &H[16 * static_cast<size_t>(k)]);
    }
    with_calib_cache(0, [&] {
        const int B = std::min(pairs, kNoiseBatch);
        CalibCache& cc = calib_cache(0, w, h, kNoiseBatch, nullptr);
        tsgm_ctx* c = cc.ctx.get();
        std::vector<int> slots(B);
        for (int i = 0; i < B; ++i) slots[i] = i;
        std::vector<const uint8_t*> img(B, c->d_img);
        begin(cc);
        for (int k0 = 0; k0 < pairs; k0 += B) {
            const int m = std::min(B, pairs - k0);
            h2d(c, cc.dgt, gt + static_cast<size_t>(k0) * P, (m + 1) * P);
            upload_step(c, m, slots.data(), img.data(), img.data(), &H[16 * static_cast<size_t>(k0)]);
            Launch L = c->L();
            launch_gt_state(c->b, cc.dgt, m, L);
            launch_warp(c->b, m, c->b.sd, c->b.sp, c->b.sv, calib.d_max, L);
            launch_predict_finalize(c->b, m, 0.0, 0, L);
            fn(cc, cc.dgt + P, m);
            CK(cudaStreamSynchronize(c->st));  // dgt is overwritten by the next batch
        }
        end(cc);
    });
}

}  // namespace

extern "C" {

int tsgm_calib_bins(const tsgm_calib_options* opts, int32_t* n_bins) {
    return guarded([&] {
        calib_options_validate(opts);
        if (!n_bins) bad("tsgm_calib_bins: null argument");
        *n_bins = hist_spec(opts).nbins;
    });
}

int tsgm_estimate_process_noise(int32_t n_frames, int32_t w, int32_t h, const double* gt,
                                const double* poses12, const tsgm_stereo_calib* calib,
                                const tsgm_calib_options* opts, tsgm_noise_estimate* out) {
    return guarded([&] {
        calib_options_validate(opts);
        if (n_frames < 2) bad("estimate_process_noise: need at least 2 frames");
        if (!gt || !poses12 || !calib || !out || w < 0 || h < 0)
            bad("estimate_process_noise: null argument");
        const HistSpec hs = hist_spec(opts);
        if (out->counts && out->n_bins < hs.nbins) bad("estimate_process_noise: counts buffer too small");
        if (static_cast<size_t>(w) * h == 0) {  // no pixels: nothing can overlap
            for (int k = 0; k + 1 < n_frames; ++k) {
                double r9[9], t3[3], H[16];
                relative_motion(poses12 + 12 * k, poses12 + 12 * (k + 1), r9, t3);
                homography(r9, t3, *calib, H);
            }
            throw std::runtime_error("estimate_process_noise: no overlapping valid pixels");
        }
        std::unique_ptr<NoiseAccum> acc;
        warp_gt_pairs(
            n_frames, w, h, gt, poses12, *calib,
            [&](CalibCache& cc) { acc = std::make_unique<NoiseAccum>(cc, hs); },
            [&](CalibCache& cc, const double* tgt, int m) {
                launch_error_hist_warped(cc.ctx->b, tgt, m, hs, acc->acc, cc.ctx->L());
            },
            [&](CalibCache&) { acc->finish(out, "estimate_process_noise"); });
    });
}

int tsgm_accumulate_error_map(int32_t n_frames, int32_t w, int32_t h, const double* gt,
                              const double* poses12, const tsgm_stereo_calib* calib, double* acc) {
    return guarded([&] {
        if (n_frames < 2) bad("accumulate_error_map: need at least 2 frames");
        if (!gt || !poses12 || !calib || !acc || w < 0 || h < 0)
            bad("accumulate_error_map: null argument");
        const size_t P = static_cast<size_t>(w) * h;
        if (P == 0) {
            for (int k = 0; k + 1 < n_frames; ++k) {
                double r9[9], t3[3], H[16];
                relative_motion(poses12 + 12 * k, poses12 + 12 * (k + 1), r9, t3);
                homography(r9, t3, *calib, H);
            }
            throw std::runtime_error("accumulate_error_map: no overlapping valid pixels");
        }
        warp_gt_pairs(
            n_frames, w, h, gt, poses12, *calib,
            [&](CalibCache& cc) {
                CK(cudaMemsetAsync(cc.dacc, 0, sizeof(double) * P, cc.ctx->st));
                CK(cudaMemsetAsync(cc.dsmall, 0, sizeof(unsigned long long), cc.ctx->st));
            },
            [&](CalibCache& cc, const double* tgt, int m) {
                launch_error_map(cc.ctx->b, tgt, m, cc.dacc, cc.dsmall, cc.ctx->L());
            },
            [&](CalibCache& cc) {
                tsgm_ctx* c = cc.ctx.get();
                unsigned long long ov = 0;
                CK(cudaMemcpyAsync(&ov, cc.dsmall, sizeof ov, cudaMemcpyDeviceToHost, c->st));
                d2h(c, acc, cc.dacc, P);
                sync(c);
                if (ov == 0) throw std::runtime_error("accumulate_error_map: no overlapping valid pixels");
            });
    });
}

int tsgm_estimate_measurement_noise(int32_t n_frames, int32_t w, int32_t h, const uint8_t* left,
                                    const uint8_t* right, const double* gt,
                                    const tsgm_sgm_params* params, const tsgm_calib_options* opts,
                                    tsgm_noise_estimate* out) {
    return guarded([&] {
        calib_options_validate(opts);
        if (n_frames < 1) bad("estimate_measurement_noise: need at least 1 frame");
        if (!left || !right || !gt || !params || !out || w < 0 || h < 0)
            bad("estimate_measurement_noise: null argument");
        sgm_validate(*params);
        const HistSpec hs = hist_spec(opts);
        if (out->counts && out->n_bins < hs.nbins)
            bad("estimate_measurement_noise: counts buffer too small");
        // sgm_match on full ranges (noise_calib.cpp:138-140): census, then the volume size
        if (w < 2 * kCensusRadius + 1 || h < 2 * kCensusRadius + 1)
            bad("census_transform: image smaller than the 5x5 window");
        if (1ull * w * h * params->d_max > 0xffffffffull)
            bad("CostVolume: volume exceeds 32-bit addressing");
        const size_t P = static_cast<size_t>(w) * h;
        std::lock_guard<std::mutex> lk(g_calib_mu);
        try {
            const int B = std::min<int>(n_frames, kNoiseBatch);
            CalibCache& cc = calib_cache(1, w, h, kNoiseBatch, params);
            tsgm_ctx* c = cc.ctx.get();
            NoiseAccum acc(cc, hs);
            double* dgt = cc.dgt;
            std::vector<int> slots(B);
            std::vector<const uint8_t*> dl(B), dr(B);
            for (int i = 0; i < B; ++i) {
                slots[i] = i;
                dl[i] = c->d_img + 2 * static_cast<size_t>(i) * P;
                dr[i] = dl[i] + P;
            }
            const std::vector<uint16_t> lo(P, 0), hi(P, static_cast<uint16_t>(params->d_max - 1));
            std::vector<double> I(16 * static_cast<size_t>(B), 0.0);
            for (int i = 0; i < B; ++i)
                for (int j = 0; j < 4; ++j) I[16 * i + 5 * j] = 1.0;
            for (int k0 = 0; k0 < n_frames; k0 += B) {
                const int m = std::min(B, n_frames - k0);
                for (int i = 0; i < m; ++i) {
                    h2d(c, const_cast<uint8_t*>(dl[i]), left + static_cast<size_t>(k0 + i) * P, P);
                    h2d(c, const_cast<uint8_t*>(dr[i]), right + static_cast<size_t>(k0 + i) * P, P);
                    h2d(c, c->b.lo + static_cast<size_t>(i) * P, lo.data(), P);
                    h2d(c, c->b.hi + static_cast<size_t>(i) * P, hi.data(), P);
                }
                h2d(c, dgt, gt + static_cast<size_t>(k0) * P, m * P);
                upload_step(c, m, slots.data(), dl.data(), dr.data(), I.data());
                Launch L = c->L();
                const Bufs& b = c->b;
                launch_ranges_given(b, m, L);
                launch_offsets(b, m, L);
                launch_census(b, m, L);
                const int chunks = (m + c->vol_slots - 1) / c->vol_slots;
                for (int k = 0, c0 = 0; k < chunks; ++k) {
                    const int mc = (m - c0) / (chunks - k);
                    const Bufs bc = chunk_bufs(b, c0);
                    launch_volume_plan(bc, mc, L);
                    launch_cost(bc, mc, L);
                    if (!aggregate(c, bc, mc, L, /*fuse_wta=*/true, /*keep_s=*/false, /*full_range=*/true))
                        launch_wta(bc, mc, L);
                    c0 += mc;
                }
                launch_error_hist_wta(b, dgt, m, hs, acc.acc, L);
                CK(cudaStreamSynchronize(c->st));  // staging buffers are reused by the next batch
            }
            acc.finish(out, "estimate_measurement_noise");
        } catch (...) {
            g_calib[1] = CalibCache{};
            throw;
        }
    });
}

int tsgm_calib_release(void) {
    return guarded([&] {
        std::lock_guard<std::mutex> lk(g_calib_mu);
        for (int k = 0; k < 2; ++k) g_calib[k] = CalibCache{};
    });
}

}  // extern "C"

// ---------------------------------------------------------------- export formats
// SURVEY §8(f) row 2 (dataset.cpp:229-269): device quantisation (export.cu)
// + host PNG / boxes.txt writers.
namespace {

std::string std_to_string(double v) {  // std::to_string(double): "%f"
    char buf[512];
    std::snprintf(buf, sizeof buf, "%f", v);
    return buf;
}

// write_disparity_png's quantisation of one host map (disp, or d + valid)
void quantize_host(const double* disp, const int32_t* d, const uint8_t* valid, int w, int h,
                   uint16_t* raw) {
    if (w < 0 || h < 0 || !raw || (!disp && (!d || !valid))) bad("write_disparity_png: bad arguments");
    const size_t P = static_cast<size_t>(w) * h;
    if (P == 0) return;
    DevScratch s;
    const double* ddisp = nullptr;
    const int32_t* dd = nullptr;
    const uint8_t* dv = nullptr;
    if (disp) {
        double* t = s.alloc<double>(P);
        CK(cudaMemcpyAsync(t, disp, 8 * P, cudaMemcpyHostToDevice, s.st));
        ddisp = t;
    } else {
        int32_t* t = s.alloc<int32_t>(P);
        uint8_t* u = s.alloc<uint8_t>(P);
        CK(cudaMemcpyAsync(t, d, 4 * P, cudaMemcpyHostToDevice, s.st));
        CK(cudaMemcpyAsync(u, valid, P, cudaMemcpyHostToDevice, s.st));
        dd = t;
        dv = u;
    }
    uint16_t* draw = s.alloc<uint16_t>(P);
    unsigned long long* fb = s.alloc<unsigned long long>(1);
    launch_quantize_disparity(ddisp, dd, dv, P, 1, nullptr, draw, fb, s.L());
    CK(cudaGetLastError());
    unsigned long long first = 0;
    CK(cudaMemcpyAsync(raw, draw, 2 * P, cudaMemcpyDeviceToHost, s.st));
    CK(cudaMemcpyAsync(&first, fb, sizeof first, cudaMemcpyDeviceToHost, s.st));
    CK(cudaStreamSynchronize(s.st));
    if (first != ~0ull) {
        const double v = disp ? disp[first] : static_cast<double>(d[first]);
        const std::string msg = "write_disparity_png: disparity " + std_to_string(v) +
                                " not encodable at (" + std::to_string(first % w) + ", " +
                                std::to_string(first / w) + ")";
        bad(msg.c_str());
    }
}

void write_png_checked(const char* path, const uint16_t* raw, int w, int h) {
    if (!path) bad("write_disparity_png: null path");
    if (w <= 0 || h <= 0) throw std::runtime_error(std::string(path) + ": PNG encode error");
    write_png16(path, raw, w, h);
}

}  // namespace

extern "C" {

int tsgm_quantize_disparity(const double* disp, int32_t w, int32_t h, uint16_t* raw) {
    return guarded([&] {
        if (!disp) bad("write_disparity_png: null map");
        quantize_host(disp, nullptr, nullptr, w, h, raw);
    });
}

int tsgm_quantize_disparity_map(const int32_t* d, const uint8_t* valid, int32_t w, int32_t h,
                                uint16_t* raw) {
    return guarded([&] {
        if (!d || !valid) bad("write_disparity_png: null map");
        quantize_host(nullptr, d, valid, w, h, raw);
    });
}

int tsgm_write_disparity_png(const char* path, const double* disp, int32_t w, int32_t h) {
    return guarded([&] {
        if (!disp) bad("write_disparity_png: null map");
        std::vector<uint16_t> raw(static_cast<size_t>(std::max(0, w)) * std::max(0, h));
        quantize_host(disp, nullptr, nullptr, w, h, raw.data());
        write_png_checked(path, raw.data(), w, h);
    });
}

int tsgm_write_disparity_png_map(const char* path, const int32_t* d, const uint8_t* valid,
                                 int32_t w, int32_t h) {
    return guarded([&] {
        if (!d || !valid) bad("write_disparity_png: null map");
        std::vector<uint16_t> raw(static_cast<size_t>(std::max(0, w)) * std::max(0, h));
        quantize_host(nullptr, d, valid, w, h, raw.data());
        write_png_checked(path, raw.data(), w, h);
    });
}

int tsgm_write_export_pngs(tsgm_ctx* ctx, int32_t n, const int32_t* slots,
                           const char* const* paths) {
    return guarded([&] {
        if (!ctx || !slots || !paths) bad("tsgm_write_export_png: null argument");
        if (n < 1 || n > ctx->max_slots) bad("tsgm_write_export_png: n out of range");
        for (int i = 0; i < n; ++i) {
            if (slots[i] < 0 || slots[i] >= ctx->max_slots) bad("tsgm_write_export_png: slot out of range");
            if (!paths[i]) bad("tsgm_write_export_png: null path");
        }
        CK(cudaSetDevice(ctx->device));
        const size_t P = ctx->P;
        DevScratch s;
        CK(cudaStreamWaitEvent(s.st, ctx->ev_frame, 0));  // the slots' last step
        uint16_t* draw = s.alloc<uint16_t>(P * n);
        unsigned long long* fb = s.alloc<unsigned long long>(n);
        int* dslots = s.alloc<int>(n);
        CK(cudaMemcpyAsync(dslots, slots, sizeof(int) * n, cudaMemcpyHostToDevice, s.st));
        launch_quantize_disparity(nullptr, ctx->b.ed, ctx->b.ev, P, n, dslots, draw, fb, s.L());
        CK(cudaGetLastError());
        uint16_t* raw = nullptr;
        CK(cudaMallocHost(&raw, 2 * P * n));
        std::unique_ptr<uint16_t, cudaError_t (*)(void*)> raw_guard(raw, &cudaFreeHost);
        std::vector<unsigned long long> first(n);
        CK(cudaMemcpyAsync(raw, draw, 2 * P * n, cudaMemcpyDeviceToHost, s.st));
        CK(cudaMemcpyAsync(first.data(), fb, sizeof(unsigned long long) * n, cudaMemcpyDeviceToHost,
                           s.st));
        CK(cudaStreamSynchronize(s.st));
        // slot by slot like the reference's write_disparity_png calls: the
        // files of the slots before the first non-encodable map are written,
        // then that map's error is raised (dataset.cpp:229-254)
        int n_ok = n;
        for (int i = 0; i < n; ++i)
            if (first[i] != ~0ull) {
                n_ok = i;
                break;
            }
        // PNG containers on host worker threads (zlib is the only host work)
        const int nt = std::max(1, std::min<int>(std::max(n_ok, 1),
                                                 static_cast<int>(std::thread::hardware_concurrency())));
        std::vector<std::string> errs(nt);
        std::vector<int> err_at(nt, n);
        std::vector<std::thread> pool;
        for (int t = 0; t < nt; ++t)
            pool.emplace_back([&, t] {
                for (int i = t; i < n_ok; i += nt) {
                    try {
                        write_png_checked(paths[i], raw + P * i, ctx->W, ctx->H);
                    } catch (const std::exception& e) {
                        if (i < err_at[t]) {
                            err_at[t] = i;
                            errs[t] = e.what();
                        }
                    }
                }
            });
        for (auto& th : pool) th.join();
        int t_err = -1;  // the first failing slot in batch order
        for (int t = 0; t < nt; ++t)
            if (!errs[t].empty() && (t_err < 0 || err_at[t] < err_at[t_err])) t_err = t;
        if (t_err >= 0) throw std::runtime_error(errs[t_err]);
        if (n_ok < n) {
            const int i = n_ok;
            int32_t v = 0;
            CK(cudaMemcpy(&v, ctx->b.ed + static_cast<size_t>(slots[i]) * P + first[i], 4,
                          cudaMemcpyDeviceToHost));
            const std::string msg = "write_disparity_png: disparity " +
                                    std_to_string(static_cast<double>(v)) + " not encodable at (" +
                                    std::to_string(first[i] % ctx->W) + ", " +
                                    std::to_string(first[i] / ctx->W) + ")";
            bad(msg.c_str());
        }
    });
}

int tsgm_write_export_png(tsgm_ctx* ctx, int32_t slot, const char* path) {
    return tsgm_write_export_pngs(ctx, 1, &slot, &path);
}

int tsgm_read_disparity_png(const char* path, int32_t* w, int32_t* h, double* disp, size_t cap) {
    return guarded([&] {
        if (!path || !w || !h) bad("read_disparity_png: null argument");
        std::vector<uint16_t> raw;
        int ww = 0, hh = 0;
        read_png16(path, raw, ww, hh);
        *w = ww;
        *h = hh;
        if (disp) {
            if (cap < raw.size()) bad("read_disparity_png: buffer too small");
            for (size_t i = 0; i < raw.size(); ++i) disp[i] = raw[i] / 256.0;  // dataset.cpp:224-225
        }
    });
}

int tsgm_write_boxes(const char* path, const tsgm_box* boxes, const int64_t* counts,
                     int32_t n_frames) {
    return guarded([&] {
        if (!path || n_frames < 0 || (n_frames > 0 && !counts)) bad("write_boxes: bad arguments");
        std::unique_ptr<FILE, int (*)(FILE*)> f(std::fopen(path, "w"), &std::fclose);
        if (!f) throw std::runtime_error(std::string("write_boxes: cannot open ") + path);
        bool ok = std::fputs("# frame x0 y0 x1 y1 score\n", f.get()) >= 0;
        int64_t k = 0;
        for (int32_t fr = 0; fr < n_frames; ++fr)
            for (int64_t i = 0; i < counts[fr]; ++i, ++k) {
                const tsgm_box& b = boxes[k];
                ok = ok && std::fprintf(f.get(), "%d %d %d %d %d %.17g\n", fr, b.x0, b.y0, b.x1,
                                        b.y1, b.score) > 0;
            }
        if (!ok || std::fflush(f.get()) != 0)
            throw std::runtime_error(std::string("write_boxes: write failed for ") + path);
    });
}

}  // extern "C"
