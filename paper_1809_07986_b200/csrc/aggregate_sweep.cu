// Scanline-group 8-path aggregation over ragged windows (aggregate_paths,
// sgm.cpp:39-161 / SURVEY.md §8(a) row A14), the fast path.
//
// Work unit: ONE WARP = 32 scanlines of one direction of one sequence, lane j
// walking scanline j pixel by pixel. Scanlines of a direction never interact,
// so warps need no synchronisation at all. Lines are parameterised so that at
// every step the 32 lanes sit on adjacent pixels of one row (vertical and
// diagonal directions: x = c + sl*y, sweeping y) or of one column
// (horizontal: sweeping x), which keeps the metadata and cost loads
// coalesced. A pixel whose window spans <= 4 aligned quads of levels is
// computed by its own lane (Q = 2..4 consecutive quads, the warp's widest);
// wider windows are computed cooperatively by groups of G = 2, 4, 8 or 16
// lanes x 4 quads (5-8, 9-16, 17-32, 33-64 quads), 32/G windows per pass. Arithmetic
// is u16x2 SIMD (VIADDMNMX / VIMNMX .U16x2), two levels per instruction.
//
// State. Each scanline keeps its last pixel's normalised path cost
//   M(d) = min(L(d) - min_k L(k), P2)
// in shared memory at ABSOLUTE level d (u8), so the recursion (sgm.cpp:100-126)
//   L(d) = C(d) + min(M(d), min(M(d-1), M(d+1)) + P1)
// needs no window bookkeeping: predecessor levels outside its quad range read
// as P2 — exactly the reference's q_min + P2 cap after normalisation — and
// with no predecessor (first pixel of the scanline) M reads as 0, giving
// L = C (sgm.cpp:93-99).
//
// Output. Each direction writes its path costs (u8: L <= 24 + P2 <= 255) in a
// quad-aligned copy of the ragged layout (qoff); the combine kernel adds the 4
// or 8 directions into S in the reference's layout. u16 sums never overflow
// (SgmParams::validate, sgm.cpp:21-22), so the grouping is exact.
//
// Layout. Every window is allocated a multiple of 4 quads (alloc_quads,
// common.cuh), so it starts 16-byte aligned: a narrow window, and a lane's 4
// quads of a full-range window, move as ONE 128-bit load (costs) and ONE
// 128-bit store (path costs). The scan is co-limited by integer issue and by
// the L1/LSU pipe; 4-byte accesses cost it 3x the L1 tag requests.
//
// Small batches. Line groups (a fixed group of G lanes per scanline) give
// more, shorter tasks when few sequences fill the GPU: lines_task keeps the
// state in shared memory like scan_task; rline_task keeps it in registers
// (lanes over absolute levels) and is used for the horizontal walks.
#include "common.cuh"

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>
#include <algorithm>

namespace tsgm {

#ifndef SCAN_WARPS
#define SCAN_WARPS 2
#endif
constexpr int kScanWarps = SCAN_WARPS;  // warps per CTA (one task each)

// slot: quads -1 .. ceil(D/4) (the ends are only ever read masked)
#ifndef SCAN_SLOT_ODD
#define SCAN_SLOT_ODD 1
#endif
__host__ __device__ inline int scan_slot_bytes(int d_max) {
    const int w = (d_max + 3) / 4 + 2;
    // (an odd word stride spreads the 32 scanlines' slots over the banks)
    return 4 * (SCAN_SLOT_ODD ? (w | 1) : w);
}
// shared bytes per warp: 32 scanline slots, 32 quad ranges, 16 group sources
__host__ __device__ inline int scan_warp_bytes(int d_max, int spw = 32) {
    return spw * (scan_slot_bytes(d_max) + 4) + 64;
}

bool sweep_supported(int W, int H, int d_max, int p2) {
    // u8 path costs need 24 + P2 <= 255; a window is <= 16 lanes x 4 quads
    (void)W;
    (void)H;
    return kMaxCost + p2 <= 255 && (d_max + 3) / 4 <= 64;
}

struct ScanParams {
    int p1, p2;
    int ndir;
    int dx[8], dy[8];        // predecessor offsets of the active directions
    int task_off[9];         // prefix of warp tasks per direction (per slot)
    int nlead;               // leading directions ordered direction-major (the horizontals)
    int n;                   // active slots
    int full_ok;             // ceil(d_max/4) is a power of two >= 8: full windows take scan_pixel_full
    uint32_t full_lohi;      // lohi of a full-range window: 0 | (d_max - 1) << 16
    uint32_t full_rng;       // quad range of a full-range window: 0 | (qmax - 1) << 16
    int warp_bytes;          // shared bytes per warp (scan_kernel)
    int rline;               // line groups with register state: 1 = horizontal tasks, 2 = every direction
    int all_full;            // every window of the launch is [0, d_max - 1] and d_max = 16 G: rfull_task
    // non-lead tasks split by length (plan_task_order): per slot, n_long tasks
    // whose 32 lines all cross the whole image (direction i: groups long_g0[i]
    // .. of long_off[i+1] - long_off[i] tasks), then n_short tasks of the
    // shorter diagonal lines near the image corners, longest first
    int n_long, n_short;
    int long_off[9], long_g0[8];
    uint8_t short_d[256], short_g[256];
};

// Task order (blockIdx order ~ dispatch order): the first nlead directions
// (the W-step horizontal walks, the kernel's longest tasks) direction-major
// over all slots, so they start first; then the other directions
// SEQUENCE-major, so one sequence's downward (and upward) scans are resident
// together and sweep the same cost / record rows at the same time: those rows
// are read from L2 instead of DRAM by all but the first of them. The diagonal
// tasks near the image corners (lines shorter than the image height) come
// LAST, over all slots, longest first: the kernel's final wave then drains
// through short tasks instead of full-length ones.
__device__ __forceinline__ void decode_task(const ScanParams& sp, int task, int& d, int& a, int& g) {
    const int lead = sp.task_off[sp.nlead] * sp.n;
    if (task < lead) {
        d = 0;
        while (task >= sp.task_off[d + 1] * sp.n) ++d;
        const int r = task - sp.task_off[d] * sp.n;
        const int groups = sp.task_off[d + 1] - sp.task_off[d];
        a = r / groups;
        g = r % groups;
    } else if (sp.n_long > 0) {
        const int t = task - lead;
        if (t < sp.n_long * sp.n) {
            a = t / sp.n_long;
            const int r = t % sp.n_long;
            d = sp.nlead;
            while (r >= sp.long_off[d + 1]) ++d;
            g = sp.long_g0[d] + r - sp.long_off[d];
        } else {
            const int u = t - sp.n_long * sp.n;
            const int si = u / sp.n;
            a = u % sp.n;
            d = sp.short_d[si];
            g = sp.short_g[si];
        }
    } else {
        const int per = sp.task_off[sp.ndir] - sp.task_off[sp.nlead];  // tasks per slot
        const int t = task - lead;
        a = t / per;
        const int r = t % per + sp.task_off[sp.nlead];
        d = sp.nlead;
        while (r >= sp.task_off[d + 1]) ++d;
        g = r - sp.task_off[d];
    }
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t s) {
    return __byte_perm(a, b, s);
}
// PRMT with the selector nibbles' msb honoured (sign replication of the
// selected byte); __byte_perm uses only the low 3 bits of each nibble.
__device__ __forceinline__ uint32_t prmt_sx(uint32_t a, uint32_t s) {
    uint32_t d;
    asm("prmt.b32 %0, %1, 0, %2;" : "=r"(d) : "r"(a), "r"(s));
    return d;
}
// Cost of a level outside the window: L = C + min(...) stays < 2^16 and
// L - min L >= kPoisonQ - 255 > P2, so it never wins a min and normalises to P2.
constexpr uint32_t kPoisonQ = 0x3fff3fffu;
// Quad range of a scanline with no predecessor yet (task start; a scanline's
// active pixels are contiguous, so this is the only case): no quad falls in
// it, and the out-of-range words read 0 instead of P2 (sgm.cpp:93-99: L = C).
constexpr uint32_t kNoPred = 0x7fff7fffu;

__device__ __forceinline__ uint32_t mad_u32(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

// shared-window byte address -> shared pointer: plain (non-asm) accesses let
// the compiler fold constant offsets into LDS/STS immediates
__device__ __forceinline__ volatile uint32_t* sptr(uint32_t addr) {
    return reinterpret_cast<volatile uint32_t*>(__cvta_shared_to_generic(addr));
}
__device__ __forceinline__ uint32_t lds32(uint32_t addr) { return *sptr(addr); }
__device__ __forceinline__ void sts32(uint32_t addr, uint32_t v) { *sptr(addr) = v; }
__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.cta.shared.u32 %0, [%1];"
                 : "=r"(v)
                 : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(p)))
                 : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
    asm volatile("st.release.cta.shared.u32 [%0], %1;" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(p))),
                 "r"(v)
                 : "memory");
}

// min over the G lanes of a group; all 32 lanes must call it.
template <int G>
__device__ __forceinline__ uint32_t group_min(uint32_t v) {
    if constexpr (G == 1) {
        return v;
    } else if constexpr (G == 32) {
        return __reduce_min_sync(0xffffffffu, v);
    } else {
#pragma unroll
        for (int o = 1; o < G; o <<= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
        return v;
    }
}

// lohi = lo | hi << 16, qo = the window's first quad in the quad layout (the
// 8-byte scan record written by the offsets kernel).
struct PixMeta {
    uint32_t lohi, qo;
};
// quads of the window
__device__ __forceinline__ uint32_t quads_of(uint32_t lohi) {
    return (lohi >> 18) - ((lohi & 0xffffu) >> 2) + 1u;
}

// One pixel, processed by a group of G lanes; lane lg owns the Q consecutive
// quads [lg*Q, lg*Q + Q) of the window. All lanes of the warp call it (pix =
// false: no pixel for this group; everything masked, nothing stored). `sb` /
// `rp` are the shared addresses of the scanline's slot and quad range.
// kPre: the window's cost words were loaded a step early (pre[0..Q-1], from
// costq + qo + min(k0, nq - 1), see lines_task).
// kV128 (G = 1): the window's 4 allocated quads leave as one 128-bit store.
template <int G, int Q, bool kPre = false, bool kV128 = false>
__device__ __forceinline__ void scan_pixel(bool pix, const PixMeta& pm,
                                           uint32_t sb, uint32_t rp, const uint32_t* costq,
                                           uint32_t* out, uint32_t P1x2, uint32_t P2x2,
                                           uint32_t P2x4, const uint32_t* pre = nullptr) {
    const int lg = static_cast<int>(threadIdx.x & (G - 1));
    const int lo = static_cast<int>(pm.lohi & 0xffffu), hi = static_cast<int>(pm.lohi >> 16);
    const int q0 = lo >> 2, q1 = hi >> 2, nq = q1 - q0 + 1;
    const int k0 = lg * Q;                  // first window quad of this lane
    const int a0 = q0 + min(k0, nq - 1);    // absolute quad (clamped into the window)

    uint32_t CA[Q], CB[Q], LA[Q], LB[Q];
    bool act[Q];
    {
        // matching costs of window quads a0 - q0 .. a0 - q0 + Q - 1 in the quad
        // layout (launch_cost): a level outside [lo, hi] inside the window's
        // quads holds 0xff, whose sign-replicated u16 0xffff masks to the
        // poison 0x3fff; quads past the window (and lanes without a pixel) are
        // poisoned whole. Poisoned levels lose every min and normalise to P2.
        const uint32_t* cw = costq + pm.qo + static_cast<uint32_t>(a0 - q0);
#pragma unroll
        for (int t = 0; t < Q; ++t) {
            act[t] = pix && k0 + t < nq;
            const uint32_t c = kPre ? pre[t] : __ldg(cw + t);
            const uint32_t am = act[t] ? 0xffffffffu : 0u;
            // kPoisonQ & (x | ~am): x masked to 14 bits, or the poison when inactive
            CA[t] = kPoisonQ & (prmt_sx(c, 0x9180u) | ~am);
            CB[t] = kPoisonQ & (prmt_sx(c, 0xb3a2u) | ~am);
        }
    }
    // predecessor words of quads a0-1 .. a0+Q (quad x at sb + 4 + 4x)
    const uint32_t prng = lds32(rp);
    // no predecessor: every word reads 0 (an empty range no quad falls in)
    const int pq0 = static_cast<int>(prng & 0xffffu);
    const uint32_t span = (prng >> 16) - static_cast<uint32_t>(pq0);
    const uint32_t fill = prng == kNoPred ? 0u : P2x4;
    uint32_t w[Q + 2];
#pragma unroll
    for (int u = 0; u < Q + 2; ++u) {
        const uint32_t raw = lds32(sb + 4u * static_cast<uint32_t>(a0 + u));
        w[u] = static_cast<uint32_t>(a0 - 1 + u - pq0) <= span ? raw : fill;
    }
    // levels outside the window carry a poisoned cost (kPoison): they lose every
    // min and normalise to exactly P2 below, so no masking is needed
    uint32_t mn = 0xffffffffu;
    uint32_t mma = prmt(w[0], prmt(w[1], 0u, 0x4140u), 0x5453u);  // M(d0-1), M(d0)
#pragma unroll
    for (int t = 0; t < Q; ++t) {
        const uint32_t e0 = prmt(w[t + 1], 0u, 0x4140u);   // M(d0),   M(d0+1)
        const uint32_t e1 = prmt(w[t + 1], 0u, 0x4342u);   // M(d0+2), M(d0+3)
        const uint32_t mpa = prmt(w[t + 1], 0u, 0x4241u);  // M(d0+1), M(d0+2)
        const uint32_t mpb = prmt(e1, w[t + 2], 0x1432u);  // M(d0+3), M(d0+4)
        // u16 lanes never carry here, so the adds go to the FMA pipe (IMAD)
        LA[t] = mad_u32(__viaddmin_u16x2(__vminu2(mma, mpa), P1x2, e0), 1u, CA[t]);
        LB[t] = mad_u32(__viaddmin_u16x2(__vminu2(mpa, mpb), P1x2, e1), 1u, CB[t]);
        mn = __vimin3_u16x2(mn, LA[t], LB[t]);
        mma = mpb;
    }
    const uint32_t m = group_min<G>(min(mn & 0xffffu, mn >> 16));
    const uint32_t neg = ((0x10000u - m) & 0xffffu) * 0x10001u;
    if (G > 1) __syncwarp();  // the group's reads of this slot are done
    if constexpr (G == 1 && kV128) {
        // the 4 allocated quads in one 128-bit store (the words past the
        // window's last quad are padding nobody reads)
        if (pix) {
            uint32_t o4[4] = {0u, 0u, 0u, 0u};
#pragma unroll
            for (int t = 0; t < Q; ++t) o4[t] = prmt(LA[t], LB[t], 0x6420u);
            *reinterpret_cast<uint4*>(out + pm.qo) = make_uint4(o4[0], o4[1], o4[2], o4[3]);
        }
    }
#pragma unroll
    for (int t = 0; t < Q; ++t) {
        if (!act[t]) continue;
        const uint32_t ma = __viaddmin_u16x2(LA[t], neg, P2x2);
        const uint32_t mb = __viaddmin_u16x2(LB[t], neg, P2x2);
        sts32(sb + 4u + 4u * static_cast<uint32_t>(a0 + t), prmt(ma, mb, 0x6420u));
        if constexpr (!(G == 1 && kV128)) (out + pm.qo + k0)[t] = prmt(LA[t], LB[t], 0x6420u);
    }
    if (pix && lg == 0) sts32(rp, static_cast<uint32_t>(q0) | (static_cast<uint32_t>(q1) << 16));
}

// scan_pixel for a full-range window [0, d_max-1] with 4G = ceil(d_max/4)
// quads (every lane's 16 levels valid): no masks, no poison, and when the
// predecessor's window was full range as well its words are used unchecked —
// the slot's guard words (quads -1 and qmax) hold P2, which is what the masked
// path reads there. Same arithmetic as scan_pixel<G, Q>.
template <int G, int Q = 4, bool kPre = false>
__device__ __forceinline__ void scan_pixel_full(bool pix, const PixMeta& pm,
                                                uint32_t sb, uint32_t rp, const uint32_t* costq,
                                                uint32_t* out, uint32_t P1x2, uint32_t P2x2,
                                                uint32_t P2x4, uint32_t full_rng,
                                                const uint32_t* pre = nullptr) {
    const int lg = static_cast<int>(threadIdx.x & (G - 1));
    const int a0 = lg * Q;
    uint32_t CA[Q], CB[Q], LA[Q], LB[Q];
    {
        // (a group without a pixel reads the volume's first window instead: in
        // bounds); a full window's quads hold no pad bytes
        const uint32_t* cw = costq + (pix ? pm.qo : 0u) + a0;
        uint32_t cc[Q];
        if constexpr (Q % 4 == 0 && !kPre) {
            // the lane's quads as 128-bit loads (16-byte aligned windows)
#pragma unroll
            for (int t = 0; t < Q; t += 4) {
                const uint4 v = __ldg(reinterpret_cast<const uint4*>(cw + t));
                cc[t] = v.x; cc[t + 1] = v.y; cc[t + 2] = v.z; cc[t + 3] = v.w;
            }
        } else {
#pragma unroll
            for (int t = 0; t < Q; ++t) cc[t] = kPre ? pre[t] : __ldg(cw + t);
        }
#pragma unroll
        for (int t = 0; t < Q; ++t) {
            CA[t] = prmt(cc[t], 0u, 0x4140u);
            CB[t] = prmt(cc[t], 0u, 0x4342u);
        }
    }
    // (a group without a pixel stays on the unchecked path: nothing is stored)
    const uint32_t prng = pix ? lds32(rp) : full_rng;
    uint32_t w[Q + 2];
#pragma unroll
    for (int u = 0; u < Q + 2; ++u) w[u] = lds32(sb + 4u * static_cast<uint32_t>(a0 + u));
    if (prng != full_rng) {
        const int pq0 = static_cast<int>(prng & 0xffffu);
        const uint32_t span = (prng >> 16) - static_cast<uint32_t>(pq0);
        const uint32_t fill = prng == kNoPred ? 0u : P2x4;
#pragma unroll
        for (int u = 0; u < Q + 2; ++u) {
            const bool in = static_cast<uint32_t>(a0 - 1 + u - pq0) <= span;
            w[u] = in ? w[u] : fill;
        }
    }
    uint32_t mn = 0xffffffffu;
    uint32_t mma = prmt(w[0], prmt(w[1], 0u, 0x4140u), 0x5453u);
#pragma unroll
    for (int t = 0; t < Q; ++t) {
        const uint32_t e0 = prmt(w[t + 1], 0u, 0x4140u);
        const uint32_t e1 = prmt(w[t + 1], 0u, 0x4342u);
        const uint32_t mpa = prmt(w[t + 1], 0u, 0x4241u);
        const uint32_t mpb = prmt(e1, w[t + 2], 0x1432u);
        LA[t] = mad_u32(__viaddmin_u16x2(__vminu2(mma, mpa), P1x2, e0), 1u, CA[t]);
        LB[t] = mad_u32(__viaddmin_u16x2(__vminu2(mpa, mpb), P1x2, e1), 1u, CB[t]);
        mn = __vimin3_u16x2(mn, LA[t], LB[t]);
        mma = mpb;
    }
    const uint32_t m = group_min<G>(min(mn & 0xffffu, mn >> 16));
    const uint32_t neg = ((0x10000u - m) & 0xffffu) * 0x10001u;
    if (G > 1) __syncwarp();
    if (pix) {
        uint32_t o[Q];
#pragma unroll
        for (int t = 0; t < Q; ++t) {
            const uint32_t ma = __viaddmin_u16x2(LA[t], neg, P2x2);
            const uint32_t mb = __viaddmin_u16x2(LB[t], neg, P2x2);
            sts32(sb + 4u + 4u * static_cast<uint32_t>(a0 + t), prmt(ma, mb, 0x6420u));
            o[t] = prmt(LA[t], LB[t], 0x6420u);
        }
        if constexpr (Q % 4 == 0) {
#pragma unroll
            for (int t = 0; t < Q; t += 4)
                *reinterpret_cast<uint4*>(out + pm.qo + a0 + t) = make_uint4(o[t], o[t + 1], o[t + 2], o[t + 3]);
        } else {
#pragma unroll
            for (int t = 0; t < Q; ++t) (out + pm.qo + a0)[t] = o[t];
        }
        if (lg == 0) sts32(rp, full_rng);
    }
}

// SPW = scanlines per warp (32, 16 or 8): a narrow window (<= 4 quads) is
// computed by GN = 32/SPW lanes x QN = 4/GN quads of its scanline's group;
// fewer scanlines per warp give proportionally more warps for small batches.
// One warp task: SPW scanlines (g-th group) of direction d of batch position
// a; wbase = the warp's shared-memory area.
// kQ8: full-range windows as G x 8 quads (half the passes; the small-batch
// mixed kernel, where each pass's latency chain is on the critical path)
// instead of 2G x 4 (large batches, where the extra live registers cost)
template <int SPW, bool kQ8 = false>
__device__ __forceinline__ void scan_task(const Bufs& b, const ScanParams& sp, int d, int a, int g,
                                          uint32_t wbase) {
    constexpr int GN = 32 / SPW, QN = 4 / GN;
    const int lane = static_cast<int>(threadIdx.x & 31);
    const int s = slot_of(b, a);
    const int W = b.W, H = b.H;
    const int dx = sp.dx[d], dy = sp.dy[d];
    const int SB = scan_slot_bytes(b.d_max);
    const int gs = lane / GN, lgs = lane % GN;  // the lane's scanline in the warp, rank in its group
    const uint32_t my_sb = wbase + static_cast<uint32_t>(gs) * SB;
    const uint32_t rbase = wbase + static_cast<uint32_t>(SPW * SB);
    const uint32_t my_rp = rbase + 4u * static_cast<uint32_t>(gs);
    const uint32_t srcbase = rbase + 4u * SPW;  // 16 group source lanes
    const uint32_t P1x2 = static_cast<uint32_t>(sp.p1) * 0x10001u;
    const uint32_t P2x2 = static_cast<uint32_t>(sp.p2) * 0x10001u;
    const uint32_t P2x4 = static_cast<uint32_t>(sp.p2) * 0x01010101u;
    if (lgs == 0) {  // guard words of the scanline's slot: quads -1 and qmax read as P2
        const int qmax = (b.d_max + 3) / 4;
        sts32(my_sb, P2x4);
        sts32(my_sb + 4u + 4u * static_cast<uint32_t>(qmax), P2x4);
        sts32(my_rp, kNoPred);
    }
    __syncwarp();

    const uint32_t* costq = b.costq + b.vqbase[a];
    uint32_t* out = reinterpret_cast<uint32_t*>(
        b.pdir + (static_cast<size_t>(d) * b.pool_quads + b.vqbase[a]) * 4);

    // line geometry: horizontal directions sweep x with lane = row; the others
    // sweep y with lane = line c, pixel x = c + sl*y (sl = dx*dy)
    const bool horiz = dy == 0;
    const int nsteps = horiz ? W : H;
    const int sl = dx * dy;
    const int c = (horiz ? 0 : (sl == 1 ? -(H - 1) : 0)) + SPW * g + gs;

    // p: the metadata index of step k (column-major for horizontal lines)
    auto pixel_at = [&](int k, int& p) -> bool {
        if (horiz) {
            const int x = dx < 0 ? k : W - 1 - k;
            p = x * H + c;
            return c < H;
        }
        const int y = dy < 0 ? k : H - 1 - k;
        const int x = c + sl * y;
        p = y * W + x;
        return x >= 0 && x < W;
    };
    const uint2* tmeta = b.tmeta + static_cast<size_t>(s) * b.P;
    const uint2* rmeta = b.rmeta + static_cast<size_t>(s) * b.P;
    auto load_meta = [&](int p, PixMeta& m) {
        // horizontal: lanes = consecutive rows (the column-major copy), else
        // adjacent pixels of a row: one coalesced 8-byte record each
        const uint2 v = __ldg((horiz ? tmeta : rmeta) + p);
        m.lohi = v.x;
        m.qo = v.y;
    };

    // metadata two steps ahead, costs of the next step prefetched into L1
    int p_tmp = 0;
    bool act1 = pixel_at(0, p_tmp);
    PixMeta m1{0u, 0u};
    if (act1) load_meta(p_tmp, m1);
    bool act2 = nsteps > 1 && pixel_at(1, p_tmp);
    PixMeta m2{0u, 0u};
    if (act2) load_meta(p_tmp, m2);
    for (int k = 0; k < nsteps; ++k) {
        const bool active = act1;
        const PixMeta mc = m1;
        // (32 scanlines per warp) the lane's own window — its 4 allocated
        // quads, 16-byte aligned — loaded here, a whole bookkeeping section
        // (~110 instructions) before the narrow pass uses it: the first use
        // of these words held 18% of the kernel's stall samples
        uint32_t cpre[4] = {0u, 0u, 0u, 0u};
        if constexpr (SPW == 32) {
            const uint4 v = __ldg(reinterpret_cast<const uint4*>(costq + mc.qo));
            cpre[0] = v.x; cpre[1] = v.y; cpre[2] = v.z; cpre[3] = v.w;
        }
        act1 = act2;
        m1 = m2;
#ifndef SCAN_PREFETCH
#define SCAN_PREFETCH 1
#endif
        if (SCAN_PREFETCH == 1 && act1 && lgs == 0) {  // step k+1's window towards L1 (its metadata arrived a step ago)
            const int nb = 4 * static_cast<int>(quads_of(m1.lohi));  // the window's bytes (quad layout)
            const char* c0 = reinterpret_cast<const char*>(costq + m1.qo);
            // straight-line (windows are <= 64 quads, sweep_supported): 0.8%
            // faster than the loop
            asm volatile("prefetch.global.L1 [%0];" ::"l"(c0));
            if (nb + 4 > 128) asm volatile("prefetch.global.L1 [%0];" ::"l"(c0 + 128));
            if (nb + 4 > 256) asm volatile("prefetch.global.L1 [%0];" ::"l"(c0 + 256));
        }
        // SCAN_PREFETCH 2: prefetches issued a pass, not a step, before their
        // use (a step is ~6000 cycles under load and the L1 turns over in less):
        // this step's WIDE window here (used after the narrow pass), the next
        // step's narrow window after this step's narrow pass
        if (SCAN_PREFETCH == 2 && active && lgs == 0 && quads_of(mc.lohi) > 4u) {
            const int nb = 4 * static_cast<int>(quads_of(mc.lohi));
            const char* c0 = reinterpret_cast<const char*>(costq + mc.qo);
            asm volatile("prefetch.global.L1 [%0];" ::"l"(c0));
            asm volatile("prefetch.global.L1 [%0];" ::"l"(c0 + 124));
            if (nb > 128) asm volatile("prefetch.global.L1 [%0];" ::"l"(c0 + 252));
        }
        act2 = k + 2 < nsteps && pixel_at(k + 2, p_tmp);
        if (act2) load_meta(p_tmp, m2);
        // the step's window classes in ONE warp reduction: bits 1..4 = narrow
        // windows of that many quads, 8 = full range, 9 = other wide windows
        const int nq = static_cast<int>(quads_of(mc.lohi));
        const bool narrow = active && nq <= 4;
        const bool owner = active && lgs == 0;
        const bool fullw = sp.full_ok && mc.lohi == sp.full_lohi;
        const bool part = owner && !fullw && nq > 4;
        const uint32_t cls = __reduce_or_sync(
            0xffffffffu, (narrow ? 1u << nq : 0u) | (owner && fullw ? 0x100u : 0u) | (part ? 0x200u : 0u));
        if (cls == 0u) continue;  // no pixel on any of the warp's scanlines
        if (SPW == 32) {
            // windows of <= 4 quads: the lane itself, Q = the warp's widest such window
            if (cls & 0x10u)
                scan_pixel<1, 4, true, true>(narrow, mc, my_sb, my_rp, costq, out, P1x2, P2x2, P2x4, cpre);
            else if (cls & 0x8u)
                scan_pixel<1, 3, true, true>(narrow, mc, my_sb, my_rp, costq, out, P1x2, P2x2, P2x4, cpre);
            else if (cls & 0x6u)
                scan_pixel<1, 2, true, true>(narrow, mc, my_sb, my_rp, costq, out, P1x2, P2x2, P2x4, cpre);
        } else if (cls & 0x1eu) {
            // windows of <= 4 quads: the scanline's GN lanes x QN quads
            scan_pixel<GN, QN>(narrow, mc, my_sb, my_rp, costq, out, P1x2, P2x2, P2x4);
        }
        if (SCAN_PREFETCH == 2 && act1 && lgs == 0 && quads_of(m1.lohi) <= 4u) {
            const char* c0 = reinterpret_cast<const char*>(costq + m1.qo);
            asm volatile("prefetch.global.L1 [%0];" ::"l"(c0));
            asm volatile("prefetch.global.L1 [%0];" ::"l"(c0 + 12));  // (a window across two lines)
        }
        // wider windows: groups of G lanes x 4 quads, 32/G windows per pass;
        // a window's owner is the first lane of its scanline's group
        const auto wide = [&](auto gtag, auto qtag, unsigned bw, bool full) {
            constexpr int G = decltype(gtag)::value;
            constexpr int QQ = decltype(qtag)::value;  // quads per lane (full windows)
            constexpr int PER = 32 / G;
            const int gi = lane / G;
            while (bw) {
                int src, cnt;
                if constexpr (PER <= 4) {
                    // the pass's windows = the lowest PER set bits of bw; group
                    // gi takes the gi-th of them (warp-uniform bit arithmetic:
                    // no shared-memory table, vote or barrier on the chain)
                    unsigned nxt = bw, bsel = 0u;
#pragma unroll
                    for (int j = 0; j < PER; ++j) {
                        if (j == gi) bsel = nxt;
                        nxt &= nxt - 1u;
                    }
                    cnt = bsel != 0u ? PER : 0;  // (gi < cnt <=> the group has a window)
                    src = bsel != 0u ? __ffs(bsel) - 1 : lane;
                    bw = nxt;
                } else {
                    const bool mine = (bw >> lane) & 1u;
                    const int rank = __popc(bw & ((1u << lane) - 1u));
                    const bool go = mine && rank < PER;
                    if (go) sts32(srcbase + 4u * static_cast<uint32_t>(rank), static_cast<uint32_t>(lane));
                    const unsigned done = __ballot_sync(0xffffffffu, go);
                    cnt = __popc(done);
                    src = gi < cnt ? static_cast<int>(lds32(srcbase + 4u * static_cast<uint32_t>(gi))) : lane;
                    __syncwarp();
                    bw &= ~done;
                }
                PixMeta pw;
                pw.lohi = full ? sp.full_lohi : __shfl_sync(0xffffffffu, mc.lohi, src);
                pw.qo = __shfl_sync(0xffffffffu, mc.qo, src);
                const uint32_t sline = static_cast<uint32_t>(src / GN);
                if (full)
                    scan_pixel_full<G, QQ>(gi < cnt, pw, wbase + sline * SB, rbase + 4u * sline,
                                           costq, out, P1x2, P2x2, P2x4, sp.full_rng);
                else
                    scan_pixel<G, 4>(gi < cnt, pw, wbase + sline * SB, rbase + 4u * sline, costq,
                                     out, P1x2, P2x2, P2x4);
            }
        };
        // the four partial-wide classes only when the step has such a window
        // (rare: 5+ quads, not full range) (aggregation 8.10 -> 7.84 ms)
        if (cls & 0x200u) {
            const unsigned b2 = __ballot_sync(0xffffffffu, part && nq <= 8);
            if (b2) wide(std::integral_constant<int, 2>{}, std::integral_constant<int, 4>{}, b2, false);
            const unsigned b4 = __ballot_sync(0xffffffffu, part && nq > 8 && nq <= 16);
            if (b4) wide(std::integral_constant<int, 4>{}, std::integral_constant<int, 4>{}, b4, false);
            const unsigned b8 = __ballot_sync(0xffffffffu, part && nq > 16 && nq <= 32);
            if (b8) wide(std::integral_constant<int, 8>{}, std::integral_constant<int, 4>{}, b8, false);
            const unsigned b16 = __ballot_sync(0xffffffffu, part && nq > 32);
            if (b16) wide(std::integral_constant<int, 16>{}, std::integral_constant<int, 4>{}, b16, false);
        }
        // full-range windows (when their class covers them exactly) take the
        // unmasked pass
        if (cls & 0x100u) {
            const unsigned bf = __ballot_sync(0xffffffffu, owner && fullw);
            // G lanes x Q quads = the window's quads; with kQ8, Q = 8 where
            // the group source table allows (G >= 2): half the passes, the
            // per-pass dispatch, min and shared-memory overhead spread over 32
            // levels per lane. Measured (frames/s): 8 sequences 4101 -> 4266,
            // 64 sequences 6480 -> 6432 (64 registers, so not there).
            constexpr bool FULL_Q4 = !kQ8;
            using I2 = std::integral_constant<int, 2>;
            using I4 = std::integral_constant<int, 4>;
            using I8 = std::integral_constant<int, 8>;
            using I16 = std::integral_constant<int, 16>;
            switch (sp.full_ok) {  // quads of the full window
                case 8: wide(I2{}, I4{}, bf, true); break;
                case 16: if (FULL_Q4) wide(I4{}, I4{}, bf, true); else wide(I2{}, I8{}, bf, true); break;
                case 32: if (FULL_Q4) wide(I8{}, I4{}, bf, true); else wide(I4{}, I8{}, bf, true); break;
                default: if (FULL_Q4) wide(I16{}, I4{}, bf, true); else wide(I8{}, I8{}, bf, true); break;
            }
        }
    }
}

// SPWH / SPWV scanlines per warp for the horizontal / the other directions:
// horizontal lines walk W steps (the kernel's critical path at small batches),
// so they may take thinner warps than the H-step vertical and diagonal lines.
// Tasks are direction-major over all slots (the long horizontal ones start
// first); sp.task_off counts each direction's tasks with its own SPW.
#ifndef SCAN_MINB
#define SCAN_MINB 16
#endif
#ifndef SCAN_Q8
#define SCAN_Q8 false  // (scan_kernel: 2G x 4-quad full-range passes, see scan_task)
#endif
template <int SPWH, int SPWV>
__global__ void __launch_bounds__(32 * kScanWarps, SCAN_MINB) scan_kernel(Bufs b, ScanParams sp) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int warp = static_cast<int>(threadIdx.x >> 5);
    const int task = blockIdx.x * kScanWarps + warp;
    if (task >= sp.task_off[sp.ndir] * sp.n) return;
    int d, a, g;
    decode_task(sp, task, d, a, g);
    const uint32_t wbase = static_cast<uint32_t>(__cvta_generic_to_shared(smem)) +
                           static_cast<uint32_t>(warp) * static_cast<uint32_t>(sp.warp_bytes);
    if (SPWH == SPWV || sp.dy[d] != 0)  // (one body when both widths agree)
        scan_task<SPWV, SCAN_Q8>(b, sp, d, a, g, wbase);
    else
        scan_task<SPWH, SCAN_Q8>(b, sp, d, a, g, wbase);
}


// Line-group variant for small batches (latency): a warp owns 32/G
// scanlines, each with a fixed group of G lanes x 4 quads (every window fits,
// G = the smallest power of two with 4G >= ceil(d_max/4)), one scan_pixel per
// step. ~8x more warps than scan_kernel, no per-step window classes: for one
// or a few sequences the GPU is otherwise nearly idle (scan_kernel has 306
// warp tasks per sequence).
template <int G, int Q = 4>
__device__ __forceinline__ void lines_task(const Bufs& b, const ScanParams& sp, int d, int a, int g,
                                           uint32_t wbase) {
    constexpr int LPW = 32 / G;  // scanlines per warp
    const int lane = static_cast<int>(threadIdx.x & 31);
    const int gi = lane / G;
    const int s = slot_of(b, a);
    const int W = b.W, H = b.H;
    const int dx = sp.dx[d], dy = sp.dy[d];
    const int SB = scan_slot_bytes(b.d_max);
    const uint32_t my_sb = wbase + static_cast<uint32_t>(gi) * SB;
    const uint32_t my_rp = wbase + static_cast<uint32_t>(LPW * SB) + 4u * static_cast<uint32_t>(gi);
    const uint32_t P1x2 = static_cast<uint32_t>(sp.p1) * 0x10001u;
    const uint32_t P2x2 = static_cast<uint32_t>(sp.p2) * 0x10001u;
    const uint32_t P2x4 = static_cast<uint32_t>(sp.p2) * 0x01010101u;
    if ((lane & (G - 1)) == 0) {  // guard words of the scanline's slot, no predecessor yet
        const int qmax = (b.d_max + 3) / 4;
        sts32(my_sb, P2x4);
        sts32(my_sb + 4u + 4u * static_cast<uint32_t>(qmax), P2x4);
        sts32(my_rp, kNoPred);
    }
    __syncwarp();
    const uint32_t* costq = b.costq + b.vqbase[a];
    uint32_t* out = reinterpret_cast<uint32_t*>(
        b.pdir + (static_cast<size_t>(d) * b.pool_quads + b.vqbase[a]) * 4);
    const bool horiz = dy == 0;
    const int nsteps = horiz ? W : H;
    const int sl = dx * dy;
    const int c = (horiz ? 0 : (sl == 1 ? -(H - 1) : 0)) + LPW * g + gi;
    const uint2* meta = (horiz ? b.tmeta : b.rmeta) + static_cast<size_t>(s) * b.P;
    auto pixel_at = [&](int k, int& p) -> bool {
        if (horiz) {
            const int x = dx < 0 ? k : W - 1 - k;
            p = x * H + c;
            return c < H;
        }
        const int y = dy < 0 ? k : H - 1 - k;
        const int x = c + sl * y;
        p = y * W + x;
        return x >= 0 && x < W;
    };
    auto load_meta = [&](int p, PixMeta& m) {
        const uint2 v = __ldg(meta + p);
        m.lohi = v.x;
        m.qo = v.y;
    };
    int p_tmp = 0;
    bool act1 = pixel_at(0, p_tmp);
    PixMeta m1{0u, 0u};
    if (act1) load_meta(p_tmp, m1);
    bool act2 = nsteps > 1 && pixel_at(1, p_tmp);
    PixMeta m2{0u, 0u};
    if (act2) load_meta(p_tmp, m2);
    const int lg = lane & (G - 1);
    // the lane's Q cost words of the NEXT step's window, loaded a step early
    // (a line-group walk is latency-bound: the cost load was its top stall);
    // the same words for the masked and the full-range pass: window quads
    // min(k0, nq - 1) .. + Q - 1 (zeros without a pixel)
    uint32_t cn[Q];
    auto preload = [&](bool act, const PixMeta& m) {
        const uint32_t nqn = quads_of(m.lohi);
        const uint32_t k0 = static_cast<uint32_t>(lg * Q);
        const uint32_t* cw = costq + m.qo + (k0 < nqn ? k0 : nqn - 1u);
        if (Q == 4 && act && k0 + 4u <= nqn) {
            // (the lane's 4 quads lie inside a 16-byte aligned window: one load)
            const uint4 v = __ldg(reinterpret_cast<const uint4*>(cw));
            cn[0] = v.x; cn[1] = v.y; cn[2 % Q] = v.z; cn[3 % Q] = v.w;
        } else {
#pragma unroll
            for (int t = 0; t < Q; ++t) cn[t] = act ? __ldg(cw + t) : 0u;
        }
    };
    preload(act1, m1);
    for (int k = 0; k < nsteps; ++k) {
        const bool active = act1;
        const PixMeta mc = m1;
        uint32_t cc[Q];
#pragma unroll
        for (int t = 0; t < Q; ++t) cc[t] = cn[t];
        act1 = act2;
        m1 = m2;
        preload(act1, m1);
        act2 = k + 2 < nsteps && pixel_at(k + 2, p_tmp);
        if (act2) load_meta(p_tmp, m2);
        if (__ballot_sync(0xffffffffu, active) == 0u) continue;
        // the unmasked pass when every active scanline of the warp has a full
        // window of the class size (frames from an empty state)
        const bool fullw = sp.full_ok == Q * G && mc.lohi == sp.full_lohi;
        if (__all_sync(0xffffffffu, fullw || !active))
            scan_pixel_full<G, Q, true>(active, mc, my_sb, my_rp, costq, out, P1x2, P2x2, P2x4,
                                        sp.full_rng, cc);
        else
            scan_pixel<G, Q, true>(active, mc, my_sb, my_rp, costq, out, P1x2, P2x2, P2x4, cc);
    }
}

// Line groups with LANES OVER LEVELS and the path state in REGISTERS: a warp
// owns 32/G scanlines of one direction, each a group of G lanes; lane lg of a
// group owns the absolute quads [lg*Q, lg*Q + Q) (G*Q >= qmax: the line
// groups' G x 4, or 32 x 1 (D <= 128) / 32 x 2 (D <= 256) — one scanline per
// warp, the shortest step, for the W-step horizontal walks that are the
// scan's critical path at small batches). A step has no shared memory, no
// quad-range bookkeeping and a short dependent chain: two neighbour shuffles,
// the min-plus update of the lane's own quads, one REDUX (G = 32) or log2 G
// shuffles for the pixel's minimum — ~75 instructions per step for 32 x 1 and
// ~130 for 8 x 4 (4 scanlines), against ~100 and ~260 in lines_task. Same
// arithmetic and masking as scan_pixel: a level of a quad outside the
// predecessor's quad range reads P2 (the register holds P2 there), every
// level reads 0 at the scanline's first pixel, pad levels are poisoned by
// their cost bytes 0xff. Records come from the row-major copy, RING steps
// ahead, and the cost words PF steps ahead: no load is on the chain.
// Records come from the row-major copy, RING steps ahead, and the cost words
// PF steps ahead, in register rings. (Measured and dropped: the same pipeline
// with cp.async into shared-memory rings — 100 instead of 86 instructions per
// step for 32 x 1, and these walks are issue-bound even for one sequence: 1
// sequence 1700 -> 1620 frames/s, 4 sequences 2790 -> 2400.)
template <int G, int Q>
__device__ __forceinline__ void rline_task(const Bufs& b, const ScanParams& sp, int d, int a, int g) {
    constexpr int PF = Q >= 4 ? 2 : 4, RING = 2 * PF, LPW = 32 / G;
    const int lane = static_cast<int>(threadIdx.x & 31);
    const int lg = lane & (G - 1);
    const int W = b.W, H = b.H;
    const int dx = sp.dx[d], dy = sp.dy[d];
    const bool horiz = dy == 0;
    const int nsteps = horiz ? W : H;
    const int sl = dx * dy;
    // scanline c: a row (horizontal), else the line x = c + sl*y (lines_task's numbering)
    const int c = (horiz ? 0 : (sl == 1 ? -(H - 1) : 0)) + LPW * g + lane / G;
    const int s = slot_of(b, a);
    const uint2* meta = b.rmeta + static_cast<size_t>(s) * b.P;
    const uint32_t* costq = b.costq + b.vqbase[a];
    uint32_t* out = reinterpret_cast<uint32_t*>(
        b.pdir + (static_cast<size_t>(d) * b.pool_quads + b.vqbase[a]) * 4);
    const uint32_t P1x2 = static_cast<uint32_t>(sp.p1) * 0x10001u;
    const uint32_t P2x2 = static_cast<uint32_t>(sp.p2) * 0x10001u;
    const int ql = lg * Q;  // the lane's first absolute quad

    // the line's records are a linear walk through the row-major copy: step k
    // at i0 + k*di, for the steps [ka, kb) on which the line has a pixel;
    // elsewhere {~0, 0} (a window no quad falls in)
    int i0, di, ka = 0, kb = nsteps;
    if (horiz) {
        i0 = c * W + (dx < 0 ? 0 : W - 1);
        di = dx < 0 ? 1 : -1;
        if (c >= H) kb = 0;
    } else {
        const int y0 = dy < 0 ? 0 : H - 1, dyy = dy < 0 ? 1 : -1;
        i0 = y0 * W + c + sl * y0;
        di = dyy * (W + sl);
        // x(k) = c + sl*(y0 + k*dyy) in [0, W)
        if (sl == 0) {
            if (c < 0 || c >= W) kb = 0;
        } else {
            const int x0 = c + sl * y0, dxx = sl * dyy;  // x(k) = x0 + k*dxx
            if (dxx > 0) {
                ka = max(0, -x0);
                kb = min(nsteps, W - x0);
            } else {
                ka = max(0, x0 - (W - 1));
                kb = min(nsteps, x0 + 1);
            }
        }
    }
    const uint2* mp = meta + i0;
    auto rec_at = [&](int k) -> uint2 {
        if (k < ka || k >= kb) return make_uint2(0xffffffffu, 0u);
        return __ldg(mp + k * di);
    };
    // the lane's cost words of a window (zeros outside it)
    auto cost_of = [&](const uint2& r, uint32_t (&cw)[Q]) {
        const int q0 = static_cast<int>((r.x & 0xffffu) >> 2), q1 = static_cast<int>(r.x >> 18);
        const uint32_t i = r.y + static_cast<uint32_t>(ql - q0);  // (used only where q >= q0)
#pragma unroll
        for (int t = 0; t < Q; ++t) {
            const int q = ql + t;
            cw[t] = (q >= q0 && q <= q1) ? __ldg(costq + (i + t)) : 0u;
        }
    };
    uint2 rec[RING];
    uint32_t cst[PF][Q];
#pragma unroll
    for (int j = 0; j < RING; ++j) rec[j] = rec_at(j);
#pragma unroll
    for (int j = 0; j < PF; ++j) cost_of(rec[j], cst[j]);
    uint32_t MA[Q], MB[Q];  // M(4q), M(4q+1) | M(4q+2), M(4q+3) as u16x2
#pragma unroll
    for (int t = 0; t < Q; ++t) MA[t] = MB[t] = 0u;

    for (int k0 = 0; k0 < nsteps; k0 += RING) {
#pragma unroll
        for (int j = 0; j < RING; ++j) {
            const int k = k0 + j;
            if (k >= nsteps) break;
            const uint2 r = rec[j];
            uint32_t cw[Q];
#pragma unroll
            for (int t = 0; t < Q; ++t) cw[t] = cst[j % PF][t];
            // refill the rings: step k + PF's cost words, step k + RING's record
            cost_of(rec[(j + PF) % RING], cst[j % PF]);
            rec[j] = rec_at(k + RING);

            const int q0 = static_cast<int>((r.x & 0xffffu) >> 2), q1 = static_cast<int>(r.x >> 18);
            const bool act = r.x != 0xffffffffu;
            // neighbour levels across the group's lanes; the ends of the level axis read P2
            uint32_t left = P2x2, right = P2x2;
            if constexpr (G > 1) {
                const uint32_t l = __shfl_up_sync(0xffffffffu, MB[Q - 1], 1, G);
                const uint32_t rr = __shfl_down_sync(0xffffffffu, MA[0], 1, G);
                if (lg != 0) left = l;
                if (lg != G - 1) right = rr;
            }
            uint32_t LA[Q], LB[Q];
            bool in[Q];
            uint32_t mn = 0xffffffffu;
#pragma unroll
            for (int t = 0; t < Q; ++t) {
                const int q = ql + t;
                in[t] = q >= q0 && q <= q1;  // (never where the line has no pixel)
                const uint32_t CA = kPoisonQ & prmt_sx(cw[t], 0x9180u);
                const uint32_t CB = kPoisonQ & prmt_sx(cw[t], 0xb3a2u);
                const uint32_t lw = t == 0 ? left : MB[t > 0 ? t - 1 : 0];
                const uint32_t rw = t == Q - 1 ? right : MA[t < Q - 1 ? t + 1 : 0];
                const uint32_t mma = prmt(lw, MA[t], 0x5432u);     // M(d0-1), M(d0)
                const uint32_t mpa = prmt(MA[t], MB[t], 0x5432u);  // M(d0+1), M(d0+2)
                const uint32_t mpb = prmt(MB[t], rw, 0x5432u);     // M(d0+3), M(d0+4)
                LA[t] = mad_u32(__viaddmin_u16x2(__vminu2(mma, mpa), P1x2, MA[t]), 1u, CA);
                LB[t] = mad_u32(__viaddmin_u16x2(__vminu2(mpa, mpb), P1x2, MB[t]), 1u, CB);
                if (in[t]) mn = __vimin3_u16x2(mn, LA[t], LB[t]);
            }
            const uint32_t m = group_min<G>(min(mn & 0xffffu, mn >> 16));
            const uint32_t neg = ((0x10000u - m) & 0xffffu) * 0x10001u;
            if (act) {
#pragma unroll
                for (int t = 0; t < Q; ++t) {
                    MA[t] = in[t] ? __viaddmin_u16x2(LA[t], neg, P2x2) : P2x2;
                    MB[t] = in[t] ? __viaddmin_u16x2(LB[t], neg, P2x2) : P2x2;
                    if (in[t]) out[r.y + static_cast<uint32_t>(ql - q0) + t] = prmt(LA[t], LB[t], 0x6420u);
                }
            }
        }
    }
}

// rline_task for a batch whose windows are ALL full range [0, d_max - 1] with
// d_max = 16 G (frames from the empty state: frame 0 of every sequence,
// config 3's full-range setting, the noise calibration): nothing is read per
// pixel but its costs. Pixel p's window is the G 16-byte words p*G .. p*G+G-1
// of the quad layout (every window holds 4G quads, so qoff[p] = 4G*p), lane
// lg of the scanline's group loads word p*G + lg, updates its 16 levels (no
// pads, no range tests, no records), and stores word p*G + lg of the
// direction's path costs. ~90 instructions per step of 32/G scanlines
// against ~200 in lines_task + scan_pixel_full.
template <int G>
__device__ __forceinline__ void rfull_task(const Bufs& b, const ScanParams& sp, int d, int a, int g) {
    constexpr int Q = 4, PF = 2, LPW = 32 / G;
    const int lane = static_cast<int>(threadIdx.x & 31);
    const int lg = lane & (G - 1);
    const int W = b.W, H = b.H;
    const int dx = sp.dx[d], dy = sp.dy[d];
    const bool horiz = dy == 0;
    const int nsteps = horiz ? W : H;
    const int sl = dx * dy;
    const int c = (horiz ? 0 : (sl == 1 ? -(H - 1) : 0)) + LPW * g + lane / G;
    const uint4* cost4 = reinterpret_cast<const uint4*>(b.costq + b.vqbase[a]) + lg;
    uint4* out4 = reinterpret_cast<uint4*>(
        b.pdir + (static_cast<size_t>(d) * b.pool_quads + b.vqbase[a]) * 4) + lg;
    const uint32_t P1x2 = static_cast<uint32_t>(sp.p1) * 0x10001u;
    const uint32_t P2x2 = static_cast<uint32_t>(sp.p2) * 0x10001u;
    // the line's pixels: step k at pixel i0 + k*di for k in [ka, kb)
    int i0, di, ka = 0, kb = nsteps;
    if (horiz) {
        i0 = c * W + (dx < 0 ? 0 : W - 1);
        di = dx < 0 ? 1 : -1;
        if (c >= H) kb = 0;
    } else {
        const int y0 = dy < 0 ? 0 : H - 1, dyy = dy < 0 ? 1 : -1;
        i0 = y0 * W + c + sl * y0;
        di = dyy * (W + sl);
        if (sl == 0) {
            if (c < 0 || c >= W) kb = 0;
        } else {
            const int x0 = c + sl * y0, dxx = sl * dyy;  // x(k) = x0 + k*dxx in [0, W)
            if (dxx > 0) {
                ka = max(0, -x0);
                kb = min(nsteps, W - x0);
            } else {
                ka = max(0, x0 - (W - 1));
                kb = min(nsteps, x0 + 1);
            }
        }
    }
    auto cost_at = [&](int k) -> uint4 {
        if (k < ka || k >= kb) return make_uint4(0u, 0u, 0u, 0u);
        return __ldg(cost4 + static_cast<long long>(i0 + k * di) * G);
    };
    uint4 ring[PF];
#pragma unroll
    for (int j = 0; j < PF; ++j) ring[j] = cost_at(ka + j);
    uint32_t MA[Q], MB[Q];
#pragma unroll
    for (int t = 0; t < Q; ++t) MA[t] = MB[t] = 0u;
    // (every group walks its own [ka, kb): the warp runs the longest walk)
    const int span = kb - ka;
    int maxspan = span;
#pragma unroll
    for (int o = G; o < 32; o <<= 1) maxspan = max(maxspan, __shfl_xor_sync(0xffffffffu, maxspan, o));
    for (int j0 = 0; j0 < maxspan; j0 += PF) {
#pragma unroll
        for (int jj = 0; jj < PF; ++jj) {
            const int j = j0 + jj;
            if (j >= maxspan) break;
            const bool act = j < span;
            const uint4 cv = ring[jj];
            ring[jj] = (j + PF < span) ? cost_at(ka + j + PF) : make_uint4(0u, 0u, 0u, 0u);
            const uint32_t cw[Q] = {cv.x, cv.y, cv.z, cv.w};
            uint32_t left = P2x2, right = P2x2;
            {
                const uint32_t l = __shfl_up_sync(0xffffffffu, MB[Q - 1], 1, G);
                const uint32_t rr = __shfl_down_sync(0xffffffffu, MA[0], 1, G);
                if (lg != 0) left = l;
                if (lg != G - 1) right = rr;
            }
            uint32_t LA[Q], LB[Q];
            uint32_t mn = 0xffffffffu;
#pragma unroll
            for (int t = 0; t < Q; ++t) {
                const uint32_t CA = prmt(cw[t], 0u, 0x4140u);
                const uint32_t CB = prmt(cw[t], 0u, 0x4342u);
                const uint32_t lw = t == 0 ? left : MB[t > 0 ? t - 1 : 0];
                const uint32_t rw = t == Q - 1 ? right : MA[t < Q - 1 ? t + 1 : 0];
                const uint32_t mma = prmt(lw, MA[t], 0x5432u);
                const uint32_t mpa = prmt(MA[t], MB[t], 0x5432u);
                const uint32_t mpb = prmt(MB[t], rw, 0x5432u);
                LA[t] = mad_u32(__viaddmin_u16x2(__vminu2(mma, mpa), P1x2, MA[t]), 1u, CA);
                LB[t] = mad_u32(__viaddmin_u16x2(__vminu2(mpa, mpb), P1x2, MB[t]), 1u, CB);
                mn = __vimin3_u16x2(mn, LA[t], LB[t]);
            }
            const uint32_t m = group_min<G>(min(mn & 0xffffu, mn >> 16));
            const uint32_t neg = ((0x10000u - m) & 0xffffu) * 0x10001u;
            if (act) {
#pragma unroll
                for (int t = 0; t < Q; ++t) {
                    MA[t] = __viaddmin_u16x2(LA[t], neg, P2x2);
                    MB[t] = __viaddmin_u16x2(LB[t], neg, P2x2);
                }
                out4[static_cast<long long>(i0 + (ka + j) * di) * G] =
                    make_uint4(prmt(LA[0], LB[0], 0x6420u), prmt(LA[1], LB[1], 0x6420u),
                               prmt(LA[2], LB[2], 0x6420u), prmt(LA[3], LB[3], 0x6420u));
            }
        }
    }
}

__host__ __device__ inline int lines_warp_bytes(int d_max, int G) {
    return (32 / G) * (scan_slot_bytes(d_max) + 4);
}

template <int G>
__global__ void __launch_bounds__(32 * kScanWarps) scan_lines_kernel(Bufs b, ScanParams sp) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int warp = static_cast<int>(threadIdx.x >> 5);
    const int task = blockIdx.x * kScanWarps + warp;
    if (task >= sp.task_off[sp.ndir] * sp.n) return;
    int d, a, g;
    decode_task(sp, task, d, a, g);
    const uint32_t wbase = static_cast<uint32_t>(__cvta_generic_to_shared(smem)) +
                           static_cast<uint32_t>(warp) * static_cast<uint32_t>(sp.warp_bytes);
    if (G >= 2 && sp.all_full) rfull_task<(G >= 2 ? G : 2)>(b, sp, d, a, g);
    else if (sp.rline >= (sp.dy[d] == 0 ? 1 : 2)) rline_task<G, 4>(b, sp, d, a, g);
    else lines_task<G>(b, sp, d, a, g, wbase);
}

// Line groups everywhere, the horizontal lines with wider groups (GH lanes x
// QH quads): the W-step horizontal walk is a chain of dependent
// instructions, so fewer instructions per step (fewer quads per lane) make it
// shorter. For one or two sequences.
template <int G, int GH, int QH>
__global__ void __launch_bounds__(32 * kScanWarps) scan_lines_mixed_kernel(Bufs b, ScanParams sp) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int warp = static_cast<int>(threadIdx.x >> 5);
    const int task = blockIdx.x * kScanWarps + warp;
    if (task >= sp.task_off[sp.ndir] * sp.n) return;
    int d, a, g;
    decode_task(sp, task, d, a, g);
    const uint32_t wbase = static_cast<uint32_t>(__cvta_generic_to_shared(smem)) +
                           static_cast<uint32_t>(warp) * static_cast<uint32_t>(sp.warp_bytes);
    if (sp.dy[d] == 0) {
        if (sp.rline >= 1) rline_task<GH, QH>(b, sp, d, a, g);
        else lines_task<GH, QH>(b, sp, d, a, g, wbase);
    } else {
        if (sp.all_full) rfull_task<G>(b, sp, d, a, g);
        else if (sp.rline >= 2) rline_task<G, 4>(b, sp, d, a, g);
        else lines_task<G, 4>(b, sp, d, a, g, wbase);
    }
}

// Mixed: horizontal lines as line groups (G lanes x 4 quads per scanline,
// one scan_pixel per step: the fewest instructions per step, i.e. the
// shortest W-step walk), the other directions as SPWV-scanline groups.
template <int GH, int QH, int SPWV>
// (G-lane groups: 12 CTAs per SM = 80 registers, no spills: 8 sequences
// 3264 -> 3483 frames/s; 32-lane groups keep 16: 4 sequences 2447 vs 2099)
__global__ void __launch_bounds__(32 * kScanWarps, (GH == 32 && QH == 1) ? 16 : 12) scan_mixed_kernel(Bufs b, ScanParams sp) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int warp = static_cast<int>(threadIdx.x >> 5);
    const int task = blockIdx.x * kScanWarps + warp;
    if (task >= sp.task_off[sp.ndir] * sp.n) return;
    int d, a, g;
    decode_task(sp, task, d, a, g);
    const uint32_t wbase = static_cast<uint32_t>(__cvta_generic_to_shared(smem)) +
                           static_cast<uint32_t>(warp) * static_cast<uint32_t>(sp.warp_bytes);
    if (sp.dy[d] == 0) {
        if (sp.rline >= 1) rline_task<GH, QH>(b, sp, d, a, g);
        else lines_task<GH, QH>(b, sp, d, a, g, wbase);
    } else {
        scan_task<SPWV, true>(b, sp, d, a, g, wbase);
    }
}


// Fused combine + winner_takes_all (sgm.cpp:163-187) for the production step,
// also the standalone combine (S only). ONE WARP per 32-pixel chunk of a row,
// independent of every other warp (no block barriers): a shared-memory owner
// map gives each quad of the chunk its pixel; lanes stride the chunk's quads,
// two at a time, with every direction's u32 path-cost word loaded up front
// (coalesced), u16x2 sums, S stored when requested and the quad's first
// (S, level) minimum folded into its pixel's minimum with a shared-memory
// atomicMin (the key (S << 16 | level) makes the minimum the first argmin);
// then lane = pixel writes the WTA result.
constexpr int kCwWarps = 2;
#ifndef CW_LEAN_MINB
#define CW_LEAN_MINB 24  // 40 registers (24 B spilled): 48 resident warps, 1.38 -> 1.23 ms (64 sequences)
#endif
#ifndef CW_FULL_MINB
#define CW_FULL_MINB 20  // standalone C->S: 7.53 -> 7.46 ms (64 sequences)
#endif

// per-warp shared bytes: qo[33], lh[32], cl[32] (u32), own[32*qmax] (u8),
// best[32] (u32), qsum[32*qmax] (uint2, sub-pixel only)
__host__ __device__ inline size_t cw_warp_bytes(int d_max, int subpix) {
    const size_t qm = alloc_quads(static_cast<uint32_t>((d_max - 1) / 4 + 1));  // allocated quads per pixel
    size_t bytes = 4 * 100 + 32 * qm;       // qo, lh, cl + own
    bytes = (bytes + 7) & ~static_cast<size_t>(7);
    bytes += 4 * 32;                         // best
    if (subpix) bytes += 8 * 32 * qm;        // qsum (8-byte aligned)
    return bytes;
}

// Sub-pixel extension (A22, not in the reference): parabola vertex through
// S(d-1), S(d), S(d+1) of the WTA level d when both neighbours are in the
// window and the curvature is positive; else d. f32, IEEE ops in this order.
__device__ __forceinline__ float subpixel_of(int d, int sm1, int s0, int sp1, bool have) {
    const int den = sm1 - 2 * s0 + sp1;
    if (!have || den <= 0) return static_cast<float>(d);
    const float off = __fdiv_rn(static_cast<float>(sm1 - sp1), __fmul_rn(2.0f, static_cast<float>(den)));
    return __fadd_rn(static_cast<float>(d), off);
}

// kLean: the production step's variant (WTA only: no S, no sub-pixel) —
// compiled without those paths it needs fewer registers and runs more warps.
template <int NDIR, bool kLean>
__global__ void __launch_bounds__(32 * kCwWarps, kLean ? CW_LEAN_MINB : CW_FULL_MINB)
    combine_wta_kernel(Bufs b, int n, int write_s_in, int do_wta_in, int subpix_in) {
    const int write_s = kLean ? 0 : write_s_in, do_wta = kLean ? 1 : do_wta_in;
    const int subpix = kLean ? 0 : subpix_in;
    extern __shared__ __align__(16) uint8_t cwm[];
    const int W = b.W, H = b.H;
    const int qmax = static_cast<int>(alloc_quads(static_cast<uint32_t>((b.d_max - 1) / 4 + 1)));
    const int lane = static_cast<int>(threadIdx.x & 31), wib = static_cast<int>(threadIdx.x >> 5);
    const int chunks = (W + 31) / 32;
    const long long task = static_cast<long long>(blockIdx.x) * kCwWarps + wib;
    if (task >= static_cast<long long>(chunks) * H * n) return;
    const int a = static_cast<int>(task / (static_cast<long long>(chunks) * H));
    const int rem = static_cast<int>(task % (static_cast<long long>(chunks) * H));
    const int y = rem / chunks, x0 = (rem % chunks) * 32;
    const int s = slot_of(b, a);
    uint8_t* wsm = cwm + static_cast<size_t>(wib) * cw_warp_bytes(b.d_max, subpix);
    uint32_t* qo = reinterpret_cast<uint32_t*>(wsm);  // 33 chunk-relative quad offsets
    uint32_t* lh = qo + 36;                             // lo | hi << 16
    uint32_t* cl = lh + 32;                             // cell offsets
    uint8_t* own = reinterpret_cast<uint8_t*>(cl + 32); // pixel of each quad
    uint32_t* best_s = reinterpret_cast<uint32_t*>(
        (reinterpret_cast<uintptr_t>(own + 32 * qmax) + 7) & ~static_cast<uintptr_t>(7));
    uint2* qsum = reinterpret_cast<uint2*>(best_s + 32);  // 8-byte aligned

    const int np = min(32, W - x0);
    const size_t pbase = static_cast<size_t>(s) * b.P + static_cast<size_t>(y) * W + x0;
    const size_t obase = static_cast<size_t>(s) * (b.P + 1) + static_cast<size_t>(y) * W + x0;
    const size_t dstride = b.pool_quads;
    const uint32_t* pd = reinterpret_cast<const uint32_t*>(b.pdir) + b.vqbase[a];
    uint16_t* agg = b.agg + b.vbase[a];

    uint32_t my_q = 0, my_lh = 0;
    if (lane < np) {
        my_q = __ldg(b.qoff + obase + lane);
        my_lh = __ldg(b.lohi + pbase + lane);
        cl[lane] = __ldg(b.off + obase + lane);
    }
    best_s[lane] = 0xffffffffu;
    const uint32_t qbase = __shfl_sync(0xffffffffu, my_q, 0);
    // the pixel's allocated quads (alloc_quads: pad quads hold no level of
    // [lo, hi] and fall out in finish())
    const int my_nq = lane < np ? static_cast<int>(alloc_quads((my_lh >> 18) - ((my_lh & 0xffffu) >> 2) + 1u)) : 0;
    const uint32_t rq = my_q - qbase;
    if (lane < np) {
        qo[lane] = rq;
        lh[lane] = my_lh;
        for (int k = 0; k < my_nq; ++k) own[rq + k] = static_cast<uint8_t>(lane);
    }
    const uint32_t nq = __shfl_sync(0xffffffffu, rq + static_cast<uint32_t>(my_nq), np - 1);
    __syncwarp();

    auto finish = [&](uint32_t q, const uint32_t (&w)[NDIR]) {
        uint32_t se = 0u, so = 0u;
#pragma unroll
        for (int d = 0; d < NDIR; ++d) {
            se += __byte_perm(w[d], 0u, 0x4240u);  // levels 0, 2 (u16 lanes never carry)
            so += __byte_perm(w[d], 0u, 0x4341u);  // levels 1, 3
        }
        const int l = own[q];
        const uint32_t plh = lh[l];
        const int lo = static_cast<int>(plh & 0xffffu), hi = static_cast<int>(plh >> 16);
        const int k = static_cast<int>(q - qo[l]);
        const int d0 = 4 * ((lo >> 2) + k);
        const uint32_t v[4] = {se & 0xffffu, so & 0xffffu, se >> 16, so >> 16};
        uint32_t best = 0xffffffffu;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int lv = d0 + u;
            const bool ok = lv >= lo && lv <= hi;
            if (write_s && ok) agg[cl[l] + (lv - lo)] = static_cast<uint16_t>(v[u]);
            best = min(best, ok ? ((v[u] << 16) | static_cast<uint32_t>(lv)) : 0xffffffffu);
        }
        atomicMin(best_s + l, best);
        if (subpix)
            qsum[l * qmax + k] = make_uint2((se & 0xffffu) | (so << 16), (se >> 16) | (so & 0xffff0000u));
    };
    uint32_t q = static_cast<uint32_t>(lane);
    for (; !kLean && q + 32 < nq; q += 64) {
        uint32_t w0[NDIR], w1[NDIR];
#pragma unroll
        for (int d = 0; d < NDIR; ++d) {
            w0[d] = __ldg(pd + d * dstride + qbase + q);
            w1[d] = __ldg(pd + d * dstride + qbase + q + 32);
        }
        finish(q, w0);
        finish(q + 32, w1);
    }
    if (kLean) {
        // two consecutive quads per lane and iteration, every direction's
        // 8-byte pair loaded up front (more bytes in flight per warp); the
        // pairs are 2-quad aligned in the partial buffers, so a quad on each
        // side may belong to the neighbouring chunks and is skipped
        const uint32_t qa = qbase & ~1u;
        const uint32_t span = qbase - qa + nq;
        for (uint32_t g = 2u * static_cast<uint32_t>(lane); g < span; g += 64u) {
            uint2 w2[NDIR];
#pragma unroll
            for (int d = 0; d < NDIR; ++d)
                w2[d] = __ldg(reinterpret_cast<const uint2*>(pd + d * dstride + qa + g));
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const uint32_t qq = qa + g + static_cast<uint32_t>(j) - qbase;  // chunk-relative
                if (qq < nq) {
                    uint32_t w0[NDIR];
#pragma unroll
                    for (int d = 0; d < NDIR; ++d) w0[d] = j == 0 ? w2[d].x : w2[d].y;
                    finish(qq, w0);
                }
            }
        }
    } else {
        for (; q < nq; q += 32) {
            uint32_t w0[NDIR];
#pragma unroll
            for (int d = 0; d < NDIR; ++d) w0[d] = __ldg(pd + d * dstride + qbase + q);
            finish(q, w0);
        }
    }
    __syncwarp();
    if (do_wta && lane < np) {
        const uint32_t best = best_s[lane];
        const int x = x0 + lane;
        const bool def = x >= kCensusRadius && x < W - kCensusRadius &&
                         y >= kCensusRadius && y < H - kCensusRadius;
        b.md[pbase + lane] = def ? static_cast<int32_t>(best & 0xffffu) : 0;
        b.mv[pbase + lane] = def ? 1 : 0;
        if (subpix) {
            const int lo = static_cast<int>(my_lh & 0xffffu), hi = static_cast<int>(my_lh >> 16);
            const int d = static_cast<int>(best & 0xffffu);
            auto s_at = [&](int lv) -> int {
                const uint2 qq = qsum[lane * qmax + (lv >> 2) - (lo >> 2)];
                const uint32_t wv = (lv & 2) ? qq.y : qq.x;
                return static_cast<int>((lv & 1) ? (wv >> 16) : (wv & 0xffffu));
            };
            const bool have = d - 1 >= lo && d + 1 <= hi;
            const float sp = subpixel_of(d, have ? s_at(d - 1) : 0, static_cast<int>(best >> 16),
                                         have ? s_at(d + 1) : 0, have);
            b.sub[pbase + lane] = def ? sp : 0.0f;
        }
    }
}

// name of the scan + combine kernels the last launch on this thread chose
// (tsgm_last_kernels: tests and the bench assert which variant they measured)
thread_local char g_variant[128];
const char* last_sweep_variant() { return g_variant; }

// Split the non-lead tasks of a slot into long ones (every line crosses the
// whole image) and short ones (decode_task); per[i] = lines per task of
// direction i. Leaves n_long = 0 (one sequence-major list) when the short
// list does not fit its table or nothing is long.
static void plan_task_order(ScanParams& sp, int W, int H, const int* per) {
    sp.n_long = sp.n_short = 0;
    const char* fo = std::getenv("TSGM_SCAN_ORDER");
    if (fo && std::strcmp(fo, "flat") == 0) return;
    struct Short { int len, d, g; };
    std::vector<Short> shorts;
    int nl = 0;
    for (int i = 0; i < sp.ndir; ++i) sp.long_off[i] = 0, sp.long_g0[i] = 0;
    for (int i = sp.nlead; i < sp.ndir; ++i) {
        sp.long_off[i] = nl;
        const int groups = sp.task_off[i + 1] - sp.task_off[i];
        const int sl = sp.dx[i] * sp.dy[i];
        if (sp.dy[i] == 0) return;  // (a horizontal direction outside the lead: keep one list)
        if (sl == 0) {  // vertical: every line is H pixels
            sp.long_g0[i] = 0;
            nl += groups;
            continue;
        }
        const int cstart = sl == 1 ? -(H - 1) : 0;
        const int lo = sl == 1 ? 0 : H - 1, hi = sl == 1 ? W - H : W - 1;  // full-length lines
        auto line_len = [&](int c) {
            const int a = sl == 1 ? std::max(0, -c) : std::max(0, c - (W - 1));
            const int z = sl == 1 ? std::min(H - 1, W - 1 - c) : std::min(H - 1, c);
            return std::max(0, z - a + 1);
        };
        int g0 = -1, cnt = 0;
        for (int g = 0; g < groups; ++g) {
            const int c0 = cstart + per[i] * g, c1 = c0 + per[i] - 1;
            if (c0 >= lo && c1 <= hi) {
                if (g0 < 0) g0 = g;
                ++cnt;
            } else {
                int len = 0;
                for (int c = c0; c <= c1; ++c) len = std::max(len, line_len(c));
                shorts.push_back({len, i, g});
            }
        }
        sp.long_g0[i] = std::max(g0, 0);
        nl += cnt;
    }
    sp.long_off[sp.ndir] = nl;
    if (nl == 0 || shorts.size() > 256 || shorts.empty()) return;
    for (const Short& t : shorts)
        if (t.g > 255) return;
    std::stable_sort(shorts.begin(), shorts.end(), [](const Short& x, const Short& y) { return x.len > y.len; });
    for (size_t k = 0; k < shorts.size(); ++k) {
        sp.short_d[k] = static_cast<uint8_t>(shorts[k].d);
        sp.short_g[k] = static_cast<uint8_t>(shorts[k].g);
    }
    sp.n_long = nl;
    sp.n_short = static_cast<int>(shorts.size());
}

void launch_aggregate_sweep(const Bufs& b, int n, int p1, int p2, int paths, int path_set,
                            int write_s, int do_wta, Launch L, int subpix, bool full_range) {
    ScanParams sp{};
    sp.p1 = p1;
    sp.p2 = p2;
    sp.n = n;
    // direction sets of aggregate_paths (sgm.cpp:142-156)
    static const int nondiag[4][2] = {{-1, 0}, {1, 0}, {0, -1}, {0, 1}};
    static const int diag[4][2] = {{-1, -1}, {1, -1}, {1, 1}, {-1, 1}};
    int k = 0;
    if (paths == 8 || path_set == 0)
        for (int i = 0; i < 4; ++i, ++k) { sp.dx[k] = nondiag[i][0]; sp.dy[k] = nondiag[i][1]; }
    if (paths == 8 || path_set == 1)
        for (int i = 0; i < 4; ++i, ++k) { sp.dx[k] = diag[i][0]; sp.dy[k] = diag[i][1]; }
    sp.ndir = k;
    // TSGM_SCAN_DIRS=<bitmask over the directions above> (profiling only:
    // time direction classes separately; the result is then not S)
    if (const char* fd = std::getenv("TSGM_SCAN_DIRS")) {
        const int mask = std::atoi(fd);
        int m = 0;
        for (int i = 0; i < k; ++i)
            if (mask >> i & 1) {
                sp.dx[m] = sp.dx[i];
                sp.dy[m] = sp.dy[i];
                ++m;
            }
        sp.ndir = k = m;
    }
    // task order (decode_task): the leading horizontal directions direction-
    // major, the rest sequence-major (TSGM_SCAN_ORDER=dir: all direction-major)
    {
        int nl = 0;
        while (nl < k && sp.dy[nl] == 0) ++nl;
        const char* fo = std::getenv("TSGM_SCAN_ORDER");
        sp.nlead = (fo && std::strcmp(fo, "dir") == 0) ? k : (fo && std::strcmp(fo, "seq") == 0) ? 0 : nl;
    }
    {
        const int qm = (b.d_max + 3) / 4;
        const bool pow2 = (qm & (qm - 1)) == 0;
        sp.full_ok = (b.d_max % 4 == 0 && pow2 && qm >= 8 && qm <= 64) ? qm : 0;
        sp.full_lohi = static_cast<uint32_t>(b.d_max - 1) << 16;
        sp.full_rng = static_cast<uint32_t>(qm - 1) << 16;
    }
    sp.task_off[0] = 0;
    for (int i = 0; i < k; ++i) {
        const int lines = sp.dy[i] == 0 ? b.H : b.W + (sp.dx[i] != 0 ? b.H - 1 : 0);
        sp.task_off[i + 1] = sp.task_off[i] + (lines + 31) / 32;
    }
    {
        const char* fr = std::getenv("TSGM_RLINE");
        sp.rline = fr ? std::atoi(fr) : 1;
        // TSGM_RFULL=0 keeps full-range launches on lines_task (tests compare both)
        const char* ff = std::getenv("TSGM_RFULL");
        sp.all_full = (full_range && sp.full_ok && !(ff && std::atoi(ff) == 0)) ? 1 : 0;
    }
    // one sequence or full-range frames: the line-group kernel; else
    // the scanline-group kernel (below ~12 sequences with line-group
    // horizontal tasks: 4 sequences 2153 -> 2246 frames/s, 1 sequence equal).
    // TSGM_SCAN_KERNEL=lines|groups forces one (tests).
    const int qmax = (b.d_max + 3) / 4;
    int G = 1;
    while (4 * G < qmax) G <<= 1;
    int batched_warps = 0;
    for (int i = 0; i < k; ++i) {
        const int lines = sp.dy[i] == 0 ? b.H : b.W + (sp.dx[i] != 0 ? b.H - 1 : 0);
        batched_warps += (lines + 31) / 32;
    }
    batched_warps *= n;
    const int sms = b.num_sms > 0 ? b.num_sms : 148;  // thresholds measured on a 148-SM B200
    const char* force = std::getenv("TSGM_SCAN_KERNEL");
    const bool lines_mode =
        force ? std::strcmp(force, "lines") == 0 : (full_range || batched_warps < sms * 3);
    if (lines_mode) {
        const int lpw = 32 / G;
        // horizontal lines with GH-lane groups (TSGM_LINES_H=8|16|32; G = 8 or 16 only)
        const char* flh = std::getenv("TSGM_LINES_H");
        // (1 sequence: 845 -> 1138 frames/s; not for large full-range batches,
        // where the 4x warps only add instructions: 64 sequences' frame 0
        // 21.1 -> 22.9 ms)
        int gh = flh ? std::atoi(flh) : (batched_warps < sms * 9 ? 32 : G);
        if ((G != 8 && G != 16) || gh <= G || (gh != 16 && gh != 32)) gh = G;
        // (all windows full range: rfull_task for every direction beats 32-lane
        // horizontal groups at any batch: 1 sequence 1135 -> 1351 frames/s, 4: 2213 -> 2561)
        if (sp.all_full && !flh) gh = G;
        sp.task_off[0] = 0;
        for (int i = 0; i < k; ++i) {
            const int lines = sp.dy[i] == 0 ? b.H : b.W + (sp.dx[i] != 0 ? b.H - 1 : 0);
            const int per = sp.dy[i] == 0 ? 32 / gh : lpw;
            sp.task_off[i + 1] = sp.task_off[i] + (lines + per - 1) / per;
        }
        const int tasks = sp.task_off[k] * n;
        sp.warp_bytes = lines_warp_bytes(b.d_max, G);
        const size_t smem = static_cast<size_t>(kScanWarps) * sp.warp_bytes;
        const unsigned grid = static_cast<unsigned>((tasks + kScanWarps - 1) / kScanWarps);
        if (gh != G)
            std::snprintf(g_variant, sizeof g_variant, "scan_lines_mixed_kernel<%d,%d,%d>", G, gh,
                          4 * G / gh);
        else
            std::snprintf(g_variant, sizeof g_variant, "scan_lines_kernel<%d>", G);
        if (sp.all_full) {  // (every window full range: rfull_task)
            const size_t used = std::strlen(g_variant);
            std::snprintf(g_variant + used, sizeof g_variant - used, "[rfull]");
        }
        if (gh != G) {
            auto kern = G == 8 ? (gh == 16 ? scan_lines_mixed_kernel<8, 16, 2>
                                           : scan_lines_mixed_kernel<8, 32, 1>)
                               : scan_lines_mixed_kernel<16, 32, 2>;
            kern<<<grid, 32 * kScanWarps, smem, L.st>>>(b, sp);
        } else switch (G) {
            case 1: scan_lines_kernel<1><<<grid, 32 * kScanWarps, smem, L.st>>>(b, sp); break;
            case 2: scan_lines_kernel<2><<<grid, 32 * kScanWarps, smem, L.st>>>(b, sp); break;
            case 4: scan_lines_kernel<4><<<grid, 32 * kScanWarps, smem, L.st>>>(b, sp); break;
            case 8: scan_lines_kernel<8><<<grid, 32 * kScanWarps, smem, L.st>>>(b, sp); break;
            default: scan_lines_kernel<16><<<grid, 32 * kScanWarps, smem, L.st>>>(b, sp); break;
        }
    } else {
        // scanlines per warp. Thinner warps cost instructions (a narrow window
        // is then split over 32/SPW lanes) but shorten each step; only the
        // horizontal lines, which walk W steps, need that while the batch is
        // small: their walk is the kernel's critical path. Measured on config 2
        // (frames/s): 16 sequences 3424 (8/8) -> 3904 (32, horizontal 8),
        // 32 sequences 4464 (16/16) -> 4590, 8 sequences 2694 -> 2711, 64
        // unchanged with 32/32. TSGM_SCAN_SPW / TSGM_SCAN_SPW_H override.
        // Tall images (long vertical walks too: config 4's 2048x1024 chunks of
        // 16 sequences) keep one width for every direction, from the batch
        // size: 16/16 522-534 frames/s there vs 502 (32, horizontal 16) and
        // 485 (32, horizontal 8).
        const bool tall = b.H >= 768;
        const char* fspw = std::getenv("TSGM_SCAN_SPW");
        int spw = fspw ? std::atoi(fspw)
                       : !tall ? 32 : batched_warps < sms * 40 ? 8 : batched_warps < sms * 80 ? 16 : 32;
        if (spw != 8 && spw != 16) spw = 32;
        // TSGM_SCAN_SPW_H=lines: horizontal lines as line groups (G = 8 or 16)
        // (default up to 16 sequences: 8 sequences 2712 -> 3268 frames/s; with
        // register line groups 12 sequences 4337 -> 4759, 16 equal)
        const char* fspwh = std::getenv("TSGM_SCAN_SPW_H");
        const bool hlines = (fspwh ? std::strcmp(fspwh, "lines") == 0
                                   : !fspw && !tall && batched_warps < sms * 34) &&
                            (G == 8 || G == 16);
        // the line groups' width: G lanes x 4 quads, or 32 lanes x 4G/32 quads
        // (fewer instructions per step, 4x the warps): 32 up to ~4 sequences
        // (4: 2255 -> 2318 frames/s; 8: 3244 -> 2613); TSGM_MIXED_GH=8|32
        const char* fmg = std::getenv("TSGM_MIXED_GH");
        // (with register line groups, frames/s: 2 sequences 2101 (line-group
        // kernel) -> 2615 (this kernel, 32-lane groups; G-lane groups 2454);
        // 3: 3157 (32) -> 3230 (G); 4: 3351 (32) -> 3621 (G))
        const int mgh = fmg ? std::atoi(fmg) : (batched_warps < sms * 5 ? 32 : 8);
        // (16 lanes x 2 quads for D = 128: two rows per warp, between the two)
        const int hg = mgh == 32 ? 32 : (mgh == 16 && G == 8) ? 16 : G;
        // (round 2, frames/s: 32 sequences 5759 (8) -> 5948 (16); 16 sequences
        // 5005 (8) vs 4234 (16); 64 equal for 16 and 32)
        int spwh = fspwh ? std::atoi(fspwh)
                         : (fspw || tall) ? spw
                                          : (batched_warps < sms * 50 ? 8 : batched_warps < sms * 80 ? 16 : 32);
        if (spwh != 8 && spwh != 16) spwh = 32;
        if (spwh > spw) spwh = spw;
        sp.task_off[0] = 0;
        for (int i = 0; i < k; ++i) {
            const int lines = sp.dy[i] == 0 ? b.H : b.W + (sp.dx[i] != 0 ? b.H - 1 : 0);
            const int per = sp.dy[i] == 0 ? (hlines ? 32 / hg : spwh) : spw;
            sp.task_off[i + 1] = sp.task_off[i] + (lines + per - 1) / per;
        }
        {
            int per[8];
            for (int i = 0; i < k; ++i) per[i] = sp.dy[i] == 0 ? (hlines ? 32 / hg : spwh) : spw;
            plan_task_order(sp, b.W, b.H, per);
        }
        sp.warp_bytes = std::max(scan_warp_bytes(b.d_max, std::max(spw, spwh)),
                                 hlines ? lines_warp_bytes(b.d_max, hg) : 0);
        const int tasks = sp.task_off[k] * n;
        const size_t smem = static_cast<size_t>(kScanWarps) * sp.warp_bytes;
        const unsigned grid = static_cast<unsigned>((tasks + kScanWarps - 1) / kScanWarps);
        auto kern = scan_kernel<32, 32>;
        if (hlines)
            std::snprintf(g_variant, sizeof g_variant, "scan_mixed_kernel<%d,%d,%d>", hg,
                          4 * G / hg, spw);
        else
            std::snprintf(g_variant, sizeof g_variant, "scan_kernel<%d,%d>",
                          spw == 8 ? 8 : spwh, spw);
        if (hlines) {
            if (hg == 32)
                kern = G == 8 ? (spw == 8 ? scan_mixed_kernel<32, 1, 8> : spw == 16 ? scan_mixed_kernel<32, 1, 16>
                                                                         : scan_mixed_kernel<32, 1, 32>)
                              : (spw == 8 ? scan_mixed_kernel<32, 2, 8> : spw == 16 ? scan_mixed_kernel<32, 2, 16>
                                                                         : scan_mixed_kernel<32, 2, 32>);
            else if (hg == 16 && G == 8)
                kern = spw == 8 ? scan_mixed_kernel<16, 2, 8> : spw == 16 ? scan_mixed_kernel<16, 2, 16>
                                                                : scan_mixed_kernel<16, 2, 32>;
            else if (G == 8)
                kern = spw == 8 ? scan_mixed_kernel<8, 4, 8> : spw == 16 ? scan_mixed_kernel<8, 4, 16>
                                                               : scan_mixed_kernel<8, 4, 32>;
            else
                kern = spw == 8 ? scan_mixed_kernel<16, 4, 8> : spw == 16 ? scan_mixed_kernel<16, 4, 16>
                                                                : scan_mixed_kernel<16, 4, 32>;
        } else if (spw == 8) kern = scan_kernel<8, 8>;
        else if (spw == 16) kern = spwh == 8 ? scan_kernel<8, 16> : scan_kernel<16, 16>;
        else if (spwh == 8) kern = scan_kernel<8, 32>;
        else if (spwh == 16) kern = scan_kernel<16, 32>;
        kern<<<grid, 32 * kScanWarps, smem, L.st>>>(b, sp);
    }
    L.end_stage(kStAggregate);
    const size_t cwsmem = kCwWarps * cw_warp_bytes(b.d_max, subpix);
    const bool lean = !write_s && do_wta && !subpix;
    auto kern = k == 8 ? (lean ? combine_wta_kernel<8, true> : combine_wta_kernel<8, false>)
                       : (lean ? combine_wta_kernel<4, true> : combine_wta_kernel<4, false>);
    {
        const size_t used = std::strlen(g_variant);
        std::snprintf(g_variant + used, sizeof g_variant - used, "+combine_wta_kernel<%d,%d>", k,
                      lean ? 1 : 0);
    }
    static size_t cw_set[4] = {48 * 1024, 48 * 1024, 48 * 1024, 48 * 1024};  // opt in once per variant
    const int vi = (k == 8 ? 2 : 0) + (lean ? 1 : 0);
    if (cwsmem > cw_set[vi]) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(cwsmem));
        cw_set[vi] = cwsmem;
    }
    const long long warps = static_cast<long long>((b.W + 31) / 32) * b.H * n;
    kern<<<static_cast<unsigned>((warps + kCwWarps - 1) / kCwWarps), 32 * kCwWarps, cwsmem, L.st>>>(
        b, n, write_s, do_wta, subpix);
    *L.counter += 2;
    // the direction sum is fused with winner_takes_all (when do_wta)
    L.end_stage(do_wta ? kStWta : kStAggregate);
}

}  // namespace tsgm
