// FP64 Kalman-state kernels: ego-motion forward warp with the reference's
// lexicographic collision rule, prediction variance, discontinuity rejection,
// zoom-hole fill, correction, diff, mask and integer rendering (SURVEY.md
// §8(a) rows A5-A9, A16-A18, A21). Compiled with -fmad=false and written in
// the reference's operation order, so results are bit-identical to the x86-64
// reference build (which has no FMA).
#include "common.cuh"

namespace tsgm {

// ---------------------------------------------------------------- warp (A5, A6)
// warp_state_ex, geometry.cpp:127-156. A colliding target keeps the
// lexicographic maximum of (d' up, p down, source d down) (replaces(),
// geometry.cpp:116-123). Pass 1 maps every source once (DispHomography::apply
// and the target rounding), caches (target, d' key) and atomicMax-es the d'
// key; pass 2, for sources whose d' equals the winner, takes the
// lexicographic minimum of (p key, source-d key) with a 128-bit CAS loop.
// Keys are order-preserving u64 images of the doubles, so the result is exact
// and independent of thread order.
struct Mapped {
    int t;  // target pixel index, -1 if dropped
    double dp;
};

__device__ __forceinline__ Mapped map_source(const double* H, int x, int y, double ds, int W,
                                             int Hh, int d_max) {
    Mapped m{-1, 0.0};
    const double xd = static_cast<double>(x), yd = static_cast<double>(y);
    double v[4];
#pragma unroll
    for (int r = 0; r < 4; ++r)  // DispHomography::apply, geometry.cpp:56-61
        v[r] = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(H[r * 4 + 0], xd), __dmul_rn(H[r * 4 + 1], yd)),
                                   __dmul_rn(H[r * 4 + 2], ds)),
                         __dmul_rn(H[r * 4 + 3], 1.0));
    if (!(v[3] > 1e-12)) return m;
    const double mx = v[0] / v[3], my = v[1] / v[3], dp = v[2] / v[3];
    if (!(dp > 0.0) || !(dp < static_cast<double>(d_max))) return m;
    const int tx = x86_lround_int(mx), ty = x86_lround_int(my);
    if (tx < 0 || tx >= W || ty < 0 || ty >= Hh) return m;
    m.t = ty * W + tx;
    m.dp = dp;
    return m;
}

// kCache: pass 1 stores each source's (target, d' key) for pass 2 (stage
// API); the step recomputes the mapping in pass 2 instead (a few FP64 ops
// per source against 24 B/px of cache traffic).
template <bool kCache>
__global__ void warp_map_kernel(Bufs b, const double* src_d, const uint8_t* src_v, int d_max) {
    const int a = blockIdx.y, s = slot_of(b, a);
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= b.P) return;
    const size_t base = static_cast<size_t>(s) * b.P;
    int tgt = -1;
    unsigned long long kd = 0ull;
    if (src_v[base + i]) {
        const Mapped m = map_source(b.H16 + 16 * a, i % b.W, i / b.W, src_d[base + i], b.W, b.H,
                                    d_max);
        if (m.t >= 0) {
            tgt = m.t;
            kd = ord_key(m.dp);
            atomicMax(&b.kd[base + m.t], kd);
        }
    }
    if (kCache) {
        b.wtgt[base + i] = tgt;
        b.wdk[base + i] = kd;
    }
}

__device__ __forceinline__ ulonglong2 cas128(ulonglong2* addr, ulonglong2 cmp, ulonglong2 val) {
    ulonglong2 old;
    asm volatile(
        "{\n\t.reg .b128 d, c, v;\n\t"
        "mov.b128 c, {%2, %3};\n\t"
        "mov.b128 v, {%4, %5};\n\t"
        "atom.global.cas.b128 d, [%6], c, v;\n\t"
        "mov.b128 {%0, %1}, d;\n\t}"
        : "=l"(old.x), "=l"(old.y)
        : "l"(cmp.x), "l"(cmp.y), "l"(val.x), "l"(val.y), "l"(addr)
        : "memory");
    return old;
}

__device__ __forceinline__ bool lex_less(ulonglong2 a, ulonglong2 b) {
    return a.x < b.x || (a.x == b.x && a.y < b.y);
}

template <bool kCached>
__global__ void warp_tiebreak_kernel(Bufs b, const double* src_d, const double* src_p,
                                     const uint8_t* src_v, int d_max) {
    const int a = blockIdx.y, s = slot_of(b, a);
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= b.P) return;
    const size_t base = static_cast<size_t>(s) * b.P;
    int tgt;
    unsigned long long dk;
    if (kCached) {
        tgt = b.wtgt[base + i];
        if (tgt < 0) return;
        dk = b.wdk[base + i];
    } else {  // the same mapping as pass 1 (deterministic: same ops, same inputs)
        if (!src_v[base + i]) return;
        const Mapped m = map_source(b.H16 + 16 * a, i % b.W, i / b.W, src_d[base + i], b.W, b.H,
                                    d_max);
        if (m.t < 0) return;
        tgt = m.t;
        dk = ord_key(m.dp);
    }
    const size_t t = base + tgt;
    if (b.kd[t] != dk) return;
    const ulonglong2 mine = make_ulonglong2(ord_key(src_p[base + i]), ord_key(src_d[base + i]));
    ulonglong2* addr = b.kps + t;
    // start from the armed value: only the CAS reads the pair atomically (a
    // plain 16-byte load may tear and hide a smaller pair)
    ulonglong2 cur = make_ulonglong2(~0ull, ~0ull);
    while (lex_less(mine, cur)) {
        const ulonglong2 prev = cas128(addr, cur, mine);
        if (prev.x == cur.x && prev.y == cur.y) break;
        cur = prev;
    }
}

void launch_warp(const Bufs& b, int n, const double* src_d, const double* src_p,
                 const uint8_t* src_v, int d_max, Launch L) {
    dim3 grid((b.P + 255) / 256, n);
    warp_map_kernel<true><<<grid, 256, 0, L.st>>>(b, src_d, src_v, d_max);
    warp_tiebreak_kernel<true><<<grid, 256, 0, L.st>>>(b, src_d, src_p, src_v, d_max);
    *L.counter += 2;
}

// (measured: recomputing the mapping in pass 2 instead of the 12 B/px cache
// doubled the tie-break kernel, 0.35 -> 0.70 ms for 64 sequences: FP64
// divisions cost more than the cache traffic)
void launch_warp_step(const Bufs& b, int n, int d_max, Launch L) {
    launch_warp(b, n, b.sd, b.sp, b.sv, d_max, L);
}

// Decode the winners (warp_state_ex output) and apply predict's variance step,
// temporal_filter.cpp:35-47: invalidate if the source disparity is not
// positive, phi = d'/d_src, p = (phi*phi)*p + q. Also re-arms the keys for the
// next frame (kd = 0, (kp, ks) = ~0).
__global__ void predict_finalize_kernel(Bufs b, double q, int apply_phi) {
    const int a = blockIdx.y, s = slot_of(b, a);
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= b.P) return;
    const size_t t = static_cast<size_t>(s) * b.P + i;
    const unsigned long long kd = b.kd[t];
    double d = 0.0, p = 0.0, src = 0.0;
    uint8_t v = 0;
    if (kd != 0ull) {
        const ulonglong2 k2 = b.kps[t];
        d = key_double(kd);
        p = key_double(k2.x);
        src = key_double(k2.y);
        v = 1;
        if (apply_phi) {
            if (!(src > 0.0)) {
                d = p = 0.0;
                v = 0;
            } else {
                const double phi = d / src;
                p = __dadd_rn(__dmul_rn(__dmul_rn(phi, phi), p), q);
            }
        }
        b.kps[t] = make_ulonglong2(~0ull, ~0ull);
    }
    b.wd[t] = d;
    b.wp[t] = p;
    b.wv[t] = v;
    // source_d is an output of warp_state_ex only (the stage API, apply_phi = 0)
    if (!apply_phi) b.wsrc[t] = kd != 0ull ? src : 0.0;
    if (kd != 0ull) b.kd[t] = 0ull;  // untouched keys are still armed
}

void launch_predict_finalize(const Bufs& b, int n, double q, int apply_phi, Launch L) {
    predict_finalize_kernel<<<dim3((b.P + 255) / 256, n), 256, 0, L.st>>>(b, q, apply_phi);
    ++*L.counter;
}

// ---------------------------------------------------------------- reject + fill (A8, A9)
// reject_discontinuities (temporal_filter.cpp:51-74) decided on its input,
// then fill_zoom_holes (:76-106) decided on reject's output, fused: a pixel's
// fill needs reject's verdict at its 4 neighbours (radius-2 dependence).
// Tiled: the (32+4) x (8+4) input tile is staged in shared memory, the
// rejection verdict is computed once for the (32+2) x (8+2) ring the fill
// needs, then the 32 x 8 outputs.
constexpr int kRfW = 32, kRfH = 8;

__global__ void reject_fill_kernel(Bufs b, const double* in_d, const double* in_p,
                                   const uint8_t* in_v, double* out_d, double* out_p,
                                   uint8_t* out_v, double thr, int do_reject, int do_fill) {
    __shared__ double td[kRfH + 4][kRfW + 4];
    __shared__ double tp[kRfH + 4][kRfW + 4];
    __shared__ uint8_t tv[kRfH + 4][kRfW + 4];
    __shared__ uint8_t rv[kRfH + 2][kRfW + 2];  // validity after rejection
    const int a = blockIdx.z, s = slot_of(b, a);
    const size_t base = static_cast<size_t>(s) * b.P;
    const int W = b.W, H = b.H;
    const int x0 = blockIdx.x * kRfW - 2, y0 = blockIdx.y * kRfH - 2;
    const int tid = threadIdx.y * kRfW + threadIdx.x;
    for (int k = tid; k < (kRfH + 4) * (kRfW + 4); k += kRfW * kRfH) {
        const int ty = k / (kRfW + 4), tx = k % (kRfW + 4);
        const int gx = x0 + tx, gy = y0 + ty;
        const bool in = gx >= 0 && gx < W && gy >= 0 && gy < H;
        const size_t g = base + static_cast<size_t>(in ? gy : 0) * W + (in ? gx : 0);
        td[ty][tx] = in ? in_d[g] : 0.0;
        tp[ty][tx] = in ? in_p[g] : 0.0;
        tv[ty][tx] = in ? in_v[g] : 0;
    }
    __syncthreads();
    // verdicts for the ring: tile coords (ty, tx) in [1, kRfH+3) x [1, kRfW+3)
    for (int k = tid; k < (kRfH + 2) * (kRfW + 2); k += kRfW * kRfH) {
        const int ry = k / (kRfW + 2), rx = k % (kRfW + 2);
        const int ty = ry + 1, tx = rx + 1;
        const int gx = x0 + tx, gy = y0 + ty;
        bool v = tv[ty][tx] != 0;
        if (v && do_reject) {
            // neighbour order (1,0), (-1,0), (0,1), (0,-1) as kDx/kDy at :52-53
            const double di = td[ty][tx];
            if (gx + 1 < W && tv[ty][tx + 1] && fabs(di - td[ty][tx + 1]) > thr) v = false;
            else if (gx - 1 >= 0 && tv[ty][tx - 1] && fabs(di - td[ty][tx - 1]) > thr) v = false;
            else if (gy + 1 < H && tv[ty + 1][tx] && fabs(di - td[ty + 1][tx]) > thr) v = false;
            else if (gy - 1 >= 0 && tv[ty - 1][tx] && fabs(di - td[ty - 1][tx]) > thr) v = false;
        }
        rv[ry][rx] = v;
    }
    __syncthreads();
    const int x = blockIdx.x * kRfW + threadIdx.x, y = blockIdx.y * kRfH + threadIdx.y;
    if (x >= W || y >= H) return;
    const int tx = threadIdx.x + 2, ty = threadIdx.y + 2, rx = threadIdx.x + 1, ry = threadIdx.y + 1;
    double od = td[ty][tx], op = tp[ty][tx];
    uint8_t ov = tv[ty][tx];
    if (ov && !rv[ry][rx]) {
        od = op = 0.0;  // DisparityState::invalidate, geometry.hpp:70-74
        ov = 0;
    }
    if (do_fill && !ov) {
        const bool horiz = x - 1 >= 0 && x + 1 < W && rv[ry][rx - 1] && rv[ry][rx + 1];
        const bool vert = y - 1 >= 0 && y + 1 < H && rv[ry - 1][rx] && rv[ry + 1][rx];
        if (horiz || vert) {
            double ds = 0.0, ps = 0.0;
            int nn = 0;
            if (horiz) {
                ds = __dadd_rn(ds, __dadd_rn(td[ty][tx - 1], td[ty][tx + 1]));
                ps = __dadd_rn(ps, __dadd_rn(tp[ty][tx - 1], tp[ty][tx + 1]));
                nn += 2;
            }
            if (vert) {
                ds = __dadd_rn(ds, __dadd_rn(td[ty - 1][tx], td[ty + 1][tx]));
                ps = __dadd_rn(ps, __dadd_rn(tp[ty - 1][tx], tp[ty + 1][tx]));
                nn += 2;
            }
            od = ds / nn;
            op = ps / nn;
            ov = 1;
        }
    }
    const size_t g = base + static_cast<size_t>(y) * W + x;
    out_d[g] = od;
    out_p[g] = op;
    out_v[g] = ov;
}

void launch_reject_fill(const Bufs& b, int n, const double* in_d, const double* in_p,
                        const uint8_t* in_v, double* out_d, double* out_p, uint8_t* out_v,
                        double disc_thresh, int do_reject, int do_fill, Launch L) {
    dim3 grid((b.W + kRfW - 1) / kRfW, (b.H + kRfH - 1) / kRfH, n);
    reject_fill_kernel<<<grid, dim3(kRfW, kRfH), 0, L.st>>>(b, in_d, in_p, in_v, out_d, out_p,
                                                           out_v, disc_thresh, do_reject, do_fill);
    ++*L.counter;
}


// ---------------------------------------------------------------- fused predict tile (A6-A10)
// The step's per-pixel chain after the forward warp, one 32x8 tile per CTA:
// decode the warp winners (warp_state_ex output, geometry.cpp:127-156) and
// apply predict's variance step (temporal_filter.cpp:35-47) for the tile and
// its 2-px halo, reject_discontinuities on the 1-px ring (:51-74, decided on
// its input), fill_zoom_holes on the tile (:76-106, decided on reject's
// output), then derive_search_ranges (:108-143). Writes the prediction
// (pd/pp/pv), the windows (lo, hi, packed lohi) and each tile row's window
// and quad counts (tsum) for make_cost_volume's prefix sum
// (matching_cost.cpp:30-48). Halo values are recomputed from the same keys
// with the same operations as the neighbouring tiles, so they agree bit for
// bit. The keys stay untouched (other tiles read them as halo); the offsets
// kernel re-arms them.
constexpr int kPtW = 32, kPtH = 8;

__global__ void __launch_bounds__(kPtW * kPtH, 5) predict_tile_kernel(Bufs b, double q, double thr,
                                                                   int min_hw, int use_stddev,
                                                                   double gain) {
    __shared__ double td[kPtH + 4][kPtW + 4];
    __shared__ double tp[kPtH + 4][kPtW + 4];
    __shared__ uint8_t tv[kPtH + 4][kPtW + 4];
    __shared__ uint8_t rv[kPtH + 2][kPtW + 2];
    const int a = blockIdx.z, s = slot_of(b, a);
    const size_t base = static_cast<size_t>(s) * b.P;
    const int W = b.W, H = b.H;
    const int x0 = blockIdx.x * kPtW - 2, y0 = blockIdx.y * kPtH - 2;
    const int tid = threadIdx.y * kPtW + threadIdx.x;
    constexpr int kHalo = (kPtH + 4) * (kPtW + 4), kT = kPtW * kPtH;
    static_assert(kHalo <= 2 * kT, "two halo pixels per thread");
    // both halo pixels' keys loaded up front (the pair unconditionally: most
    // pixels hold a prediction, and the dependent load would cost a round trip)
    unsigned long long kd[2];
    ulonglong2 k2[2];
    bool in[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        const int k = tid + u * kT;
        const int ty = k / (kPtW + 4), tx = k % (kPtW + 4);
        const int gx = x0 + tx, gy = y0 + ty;
        in[u] = k < kHalo && gx >= 0 && gx < W && gy >= 0 && gy < H;
        const size_t t = base + (in[u] ? static_cast<size_t>(gy) * W + gx : 0);
        kd[u] = in[u] ? b.kd[t] : 0ull;
        k2[u] = in[u] ? b.kps[t] : make_ulonglong2(0ull, 0ull);
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        const int k = tid + u * kT;
        if (k >= kHalo) break;
        const int ty = k / (kPtW + 4), tx = k % (kPtW + 4);
        double d = 0.0, p = 0.0;
        uint8_t v = 0;
        if (kd[u] != 0ull) {
            const double src = key_double(k2[u].y);
            if (src > 0.0) {  // predict: invalidate unless the source d > 0
                d = key_double(kd[u]);
                const double phi = d / src;
                p = __dadd_rn(__dmul_rn(__dmul_rn(phi, phi), key_double(k2[u].x)), q);
                v = 1;
            }
        }
        td[ty][tx] = d;
        tp[ty][tx] = p;
        tv[ty][tx] = v;
    }
    __syncthreads();
    for (int k = tid; k < (kPtH + 2) * (kPtW + 2); k += kPtW * kPtH) {
        const int ry = k / (kPtW + 2), rx = k % (kPtW + 2);
        const int ty = ry + 1, tx = rx + 1;
        const int gx = x0 + tx, gy = y0 + ty;
        bool v = tv[ty][tx] != 0;
        if (v) {  // neighbour order (1,0), (-1,0), (0,1), (0,-1) as kDx/kDy at :52-53
            const double di = td[ty][tx];
            if (gx + 1 < W && tv[ty][tx + 1] && fabs(di - td[ty][tx + 1]) > thr) v = false;
            else if (gx - 1 >= 0 && tv[ty][tx - 1] && fabs(di - td[ty][tx - 1]) > thr) v = false;
            else if (gy + 1 < H && tv[ty + 1][tx] && fabs(di - td[ty + 1][tx]) > thr) v = false;
            else if (gy - 1 >= 0 && tv[ty - 1][tx] && fabs(di - td[ty - 1][tx]) > thr) v = false;
        }
        rv[ry][rx] = v;
    }
    __syncthreads();
    const int x = blockIdx.x * kPtW + threadIdx.x, y = blockIdx.y * kPtH + threadIdx.y;
    const bool inb = x < W && y < H;
    uint32_t cells = 0u, quads = 0u;
    if (inb) {
        const int tx = threadIdx.x + 2, ty = threadIdx.y + 2, rx = threadIdx.x + 1, ry = threadIdx.y + 1;
        double od = td[ty][tx], op = tp[ty][tx];
        uint8_t ov = tv[ty][tx];
        if (ov && !rv[ry][rx]) {
            od = op = 0.0;  // DisparityState::invalidate, geometry.hpp:70-74
            ov = 0;
        }
        if (!ov) {
            const bool horiz = x - 1 >= 0 && x + 1 < W && rv[ry][rx - 1] && rv[ry][rx + 1];
            const bool vert = y - 1 >= 0 && y + 1 < H && rv[ry - 1][rx] && rv[ry + 1][rx];
            if (horiz || vert) {
                double ds = 0.0, ps = 0.0;
                int nn = 0;
                if (horiz) {
                    ds = __dadd_rn(ds, __dadd_rn(td[ty][tx - 1], td[ty][tx + 1]));
                    ps = __dadd_rn(ps, __dadd_rn(tp[ty][tx - 1], tp[ty][tx + 1]));
                    nn += 2;
                }
                if (vert) {
                    ds = __dadd_rn(ds, __dadd_rn(td[ty - 1][tx], td[ty + 1][tx]));
                    ps = __dadd_rn(ps, __dadd_rn(tp[ty - 1][tx], tp[ty + 1][tx]));
                    nn += 2;
                }
                // (nn is 2 or 4: the division is the exact scaling by 1/nn)
                const double inv = nn == 2 ? 0.5 : 0.25;
                od = __dmul_rn(ds, inv);
                op = __dmul_rn(ps, inv);
                ov = 1;
            }
        }
        const size_t g = base + static_cast<size_t>(y) * W + x;
        b.pd[g] = od;
        b.pp[g] = op;
        b.pv[g] = ov;
        const int top = b.d_max - 1;
        int lo = 0, hi = top;
        if (ov) derive_range(od, op, top, 2 * min_hw + 1, use_stddev, gain, lo, hi);
        b.lo[g] = static_cast<uint16_t>(lo);
        b.hi[g] = static_cast<uint16_t>(hi);
        b.lohi[g] = static_cast<uint32_t>(lo) | (static_cast<uint32_t>(hi) << 16);
        cells = static_cast<uint32_t>(hi - lo + 1);
        quads = alloc_quads(static_cast<uint32_t>((hi >> 2) - (lo >> 2) + 1));
    }
    // this tile row's counts (one warp = one row of 32 pixels)
    cells = __reduce_add_sync(0xffffffffu, cells);
    quads = __reduce_add_sync(0xffffffffu, quads);
    if (threadIdx.x == 0 && y < H) {
        const int tiles_x = (W + kPtW - 1) / kPtW;
        b.tsum[(static_cast<size_t>(s) * H + y) * tiles_x + blockIdx.x] = make_uint2(cells, quads);
    }
}

void launch_predict_tile(const Bufs& b, int n, double q, double disc_thresh, int min_hw,
                         int use_stddev, double gain, Launch L) {
    dim3 grid((b.W + kPtW - 1) / kPtW, (b.H + kPtH - 1) / kPtH, n);
    predict_tile_kernel<<<grid, dim3(kPtW, kPtH), 0, L.st>>>(b, q, disc_thresh, min_hw, use_stddev,
                                                             gain);
    ++*L.counter;
}

// ---------------------------------------------------------------- correct (A16-A18, A21)
// correct (temporal_filter.cpp:145-170), the diff map (:223-229), the
// Mahalanobis mask extension (A21) and render_integer (:178-191), fused.
struct Corrected {
    double d, p, diff;
    uint8_t v, mask;
};

__device__ __forceinline__ Corrected correct_px(const Bufs& b, size_t t, double r, double tau) {
    const bool hp = b.pv[t] != 0, hm = b.mv[t] != 0;
    const double pdv = b.pd[t], ppv = b.pp[t];
    const double dz = static_cast<double>(b.md[t]);
    double d = 0.0, p = 0.0;
    uint8_t v = 0;
    if (hp && hm) {
        const double k = ppv / __dadd_rn(ppv, r);
        d = __dadd_rn(pdv, __dmul_rn(k, __dsub_rn(dz, pdv)));
        const double omk = __dsub_rn(1.0, k);
        p = __dadd_rn(__dmul_rn(__dmul_rn(omk, omk), ppv), __dmul_rn(__dmul_rn(k, k), r));
        v = 1;
    } else if (hm) {
        d = dz;
        p = r;
        v = 1;
    } else if (hp) {
        d = pdv;
        p = ppv;
        v = 1;
    }
    uint8_t mk = 0;
    if (hp && hm) {
        const double e = __dsub_rn(dz, pdv);
        mk = __dmul_rn(e, e) > __dmul_rn(__dmul_rn(tau, tau), __dadd_rn(ppv, r)) ? 1 : 0;
    }
    return Corrected{d, p, (hp && hm) ? fabs(__dsub_rn(pdv, dz)) : 0.0, v, mk};
}

__device__ __forceinline__ void store_corrected(const Bufs& b, size_t t, const Corrected& c) {
    b.sd[t] = c.d;
    b.sp[t] = c.p;
    b.sv[t] = c.v;
    b.diff[t] = c.diff;
    b.mask[t] = c.mask;
}

__global__ void correct_kernel(Bufs b, double r, double tau) {
    const int a = blockIdx.y, s = slot_of(b, a);
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= b.P) return;
    const size_t t = static_cast<size_t>(s) * b.P + i;
    const Corrected c = correct_px(b, t, r, tau);
    store_corrected(b, t, c);
    b.rd[t] = c.v ? x86_lround_int(c.d) : 0;
    b.rv[t] = c.v;
}

void launch_correct(const Bufs& b, int n, double r, double mask_tau, Launch L) {
    correct_kernel<<<dim3((b.P + 255) / 256, n), 256, 0, L.st>>>(b, r, mask_tau);
    ++*L.counter;
}

// correct + render_integer + median_refine fused for the step (A16-A19, A21):
// a 32x8 tile computes correct and render for its 34x10 footprint (the 1-px
// halo recomputed from the same inputs), writes the state, diff and mask of
// its own pixels, and takes the 3x3 lower median of the rendered map from
// shared memory (median_kernel's keys: INT32_MAX for invalid or missing) —
// the rendered map never goes to HBM.
constexpr int kCmW = 32, kCmH = 8;

__device__ __forceinline__ void cm_swap(int32_t& a, int32_t& b) {
    const int32_t lo = min(a, b), hi = max(a, b);
    a = lo;
    b = hi;
}

__global__ void __launch_bounds__(kCmW * kCmH) correct_median_kernel(Bufs b, double r, double tau) {
    __shared__ int32_t key[kCmH + 2][kCmW + 2];
    __shared__ uint8_t okv[kCmH + 2][kCmW + 2];
    const int a = blockIdx.z, s = slot_of(b, a);
    const size_t base = static_cast<size_t>(s) * b.P;
    const int W = b.W, H = b.H;
    const int x0 = blockIdx.x * kCmW - 1, y0 = blockIdx.y * kCmH - 1;
    for (int k = threadIdx.y * kCmW + threadIdx.x; k < (kCmH + 2) * (kCmW + 2); k += kCmW * kCmH) {
        const int ty = k / (kCmW + 2), tx = k % (kCmW + 2);
        const int gx = x0 + tx, gy = y0 + ty;
        int32_t kv = INT32_MAX;
        uint8_t ov = 0;
        if (gx >= 0 && gx < W && gy >= 0 && gy < H) {
            const size_t t = base + static_cast<size_t>(gy) * W + gx;
            const Corrected c = correct_px(b, t, r, tau);
            if (ty >= 1 && ty <= kCmH && tx >= 1 && tx <= kCmW) store_corrected(b, t, c);
            if (c.v) {
                kv = x86_lround_int(c.d);  // render_integer, temporal_filter.cpp:178-191
                ov = 1;
            }
        }
        key[ty][tx] = kv;
        okv[ty][tx] = ov;
    }
    __syncthreads();
    const int x = blockIdx.x * kCmW + threadIdx.x, y = blockIdx.y * kCmH + threadIdx.y;
    if (x >= W || y >= H) return;
    int32_t v[9];
    int nv = 0;
#pragma unroll
    for (int dy = 0; dy < 3; ++dy)
#pragma unroll
        for (int dx = 0; dx < 3; ++dx) {
            v[dy * 3 + dx] = key[threadIdx.y + dy][threadIdx.x + dx];
            nv += okv[threadIdx.y + dy][threadIdx.x + dx];
        }
    const size_t i = base + static_cast<size_t>(y) * W + x;
    if (nv < 5) {  // median_refine: valid iff at least 5 valid neighbours (sgm.cpp:189-216)
        b.ed[i] = 0;
        b.ev[i] = 0;
        return;
    }
    cm_swap(v[0], v[3]); cm_swap(v[1], v[7]); cm_swap(v[2], v[5]); cm_swap(v[4], v[8]);
    cm_swap(v[0], v[7]); cm_swap(v[2], v[4]); cm_swap(v[3], v[8]); cm_swap(v[5], v[6]);
    cm_swap(v[0], v[2]); cm_swap(v[1], v[3]); cm_swap(v[4], v[5]); cm_swap(v[7], v[8]);
    cm_swap(v[1], v[4]); cm_swap(v[3], v[6]); cm_swap(v[5], v[7]);
    cm_swap(v[0], v[1]); cm_swap(v[2], v[4]); cm_swap(v[3], v[5]); cm_swap(v[6], v[8]);
    cm_swap(v[2], v[3]); cm_swap(v[4], v[5]); cm_swap(v[6], v[7]);
    cm_swap(v[1], v[2]); cm_swap(v[3], v[4]); cm_swap(v[5], v[6]);
    const int k = (nv - 1) / 2;
    b.ed[i] = k == 2 ? v[2] : (k == 3 ? v[3] : v[4]);
    b.ev[i] = 1;
}

void launch_correct_median(const Bufs& b, int n, double r, double mask_tau, Launch L) {
    dim3 grid((b.W + kCmW - 1) / kCmW, (b.H + kCmH - 1) / kCmH, n);
    correct_median_kernel<<<grid, dim3(kCmW, kCmH), 0, L.st>>>(b, r, mask_tau);
    ++*L.counter;
}

}  // namespace tsgm
