// Line-sweep 8-path aggregation over ragged windows (aggregate_paths,
// sgm.cpp:39-161 / SURVEY.md §8(a) row A14), the fast path.
//
// Decomposition. The 8 directions are grouped into 4 ROLES, each a sweep over
// LINES in which every direction's predecessor lies in the previous line:
//   A: columns x = 0..W-1,   directions (-1,0), (-1,-1), (-1,+1)
//   B: columns x = W-1..0,   directions (+1,0), (+1,-1), (+1,+1)
//   C: rows    y = 0..H-1,   direction  (0,-1)
//   D: rows    y = H-1..0,   direction  (0,+1)
// (4-path sets keep the subset). Within a line all pixels are independent.
// One persistent CTA per (slot, role); warp w OWNS a fixed contiguous block of
// line positions and walks the lines; the only cross-warp dependencies are the
// diagonal predecessors at block boundaries, handled with per-warp
// acquire/release line counters (no CTA barriers). Windows are split into
// aligned quads of 4 levels; a window of <= 4 quads is one lane (4 consecutive
// quads), a wider one is 8 lanes x 4 consecutive quads (4 pixels per warp).
// Arithmetic is u16x2 SIMD (VIADDMNMX / VIMNMX .U16x2), two levels per
// instruction.
//
// State. Per direction, each pixel's normalised path cost
//   M(d) = min(L(d) - min_k L(k), P2)
// lives in shared memory in an ABSOLUTE-level slot (level d at byte 4 + d, u8),
// and the recursion (sgm.cpp:100-126) is
//   L(d) = C(d) + min(M_q(d), min(M_q(d-1), M_q(d+1)) + P1)
// where predecessor levels outside its window read as P2 — exactly the
// reference's q_min + P2 cap after normalisation. The reader masks words
// outside the predecessor's quad range (kept per slot), so slots never need
// clearing. Slots are SHEARED: direction (dl, di) stores line l, position i at
// slot (i + di*l) mod len, so a pixel reads and rewrites the slot its
// predecessor wrote (one buffer per direction, one reader per slot per line).
//
// Output. Each role writes its partial sum per quad (A/B: u16, C/D: u8 since a
// single path cost <= 24 + P2 <= 255) in the quad layout qoff; the combine
// kernel adds the partials into S in the reference's ragged layout. Sums of
// u16 values never overflow (SgmParams::validate, sgm.cpp:21-22), so the
// grouping is exact.
#include "common.cuh"

namespace tsgm {

constexpr int kSweepThreads = 512;
constexpr int kSweepWarps = kSweepThreads / 32;
constexpr int kChunks = 4;  // line length <= kSweepWarps * 32 * kChunks = 2048

// slot: quads -1 .. ceil(D/4) (the ends are only ever read masked)
__host__ __device__ inline int sweep_slot_bytes(int d_max) { return 4 * ((d_max + 3) / 4 + 2); }

struct SweepPlan {
    size_t buf, rng, flags, total;
};

__host__ __device__ inline SweepPlan sweep_plan(int W, int H, int d_max) {
    SweepPlan p;
    const size_t sb = sweep_slot_bytes(d_max);
    const size_t slots = (3 * static_cast<size_t>(H) > static_cast<size_t>(W)) ? 3 * static_cast<size_t>(H) : W;
    p.buf = slots * sb;
    p.rng = slots * 4;
    p.flags = 16 * 4;
    p.total = p.buf + p.rng + p.flags;
    return p;
}

bool sweep_supported(int W, int H, int d_max, int p2) {
    // u8 path costs need 24 + P2 <= 255; a wide window is <= 8 x 4 quads
    const int lmax = W > H ? W : H;
    return kMaxCost + p2 <= 255 && (d_max + 3) / 4 <= 32 &&
           lmax <= kSweepWarps * 32 * kChunks && sweep_plan(W, H, d_max).total <= 227 * 1024;
}

struct SweepParams {
    int p1, p2;
    int roles;    // bit 0 A, 1 B, 2 C, 3 D
    int ndir_ab;  // directions in the column roles
    int di_ab[3];
    int n;        // active slots
};

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t s) {
    return __byte_perm(a, b, s);
}
__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ void sts32(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
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
    if (G == 1) return v;
    if (G == 32) return __reduce_min_sync(0xffffffffu, v);
#pragma unroll
    for (int o = 1; o < G; o <<= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

struct PixMeta {
    uint32_t lohi, cell, qo;
};

// One pixel, processed by a group of G lanes; lane lg owns the Q consecutive
// quads [lg*Q, lg*Q + Q) of the window. All lanes of the warp call it (i < 0:
// no pixel for this group; everything masked, nothing stored).
template <int G, int Q>
__device__ __forceinline__ void sweep_pixel(int i, const PixMeta& pm, int l, int len, int ndir,
                                            int di0, int di1, int di2, int sb0, int sb1, int sb2,
                                            uint32_t mbuf, int SB, uint32_t rng,
                                            const uint8_t* cost, void* out, bool out_u16,
                                            uint32_t P1x2, uint32_t P2x2, uint32_t P2x4) {
    const int lg = static_cast<int>(threadIdx.x & (G - 1));
    const bool px = i >= 0;
    const int ii = px ? i : 0;
    const int lo = static_cast<int>(pm.lohi & 0xffffu), hi = static_cast<int>(pm.lohi >> 16);
    const int q0 = lo >> 2, q1 = hi >> 2, nq = q1 - q0 + 1;
    const uint32_t qrange = static_cast<uint32_t>(q0) | (static_cast<uint32_t>(q1) << 16);
    const int k0 = lg * Q;                  // first window quad of this lane
    const int kc = min(k0, nq - 1);         // clamped (inactive lanes read the window)
    const int a0 = q0 + kc;                 // absolute quad of the lane's first quad

    // matching costs: levels 4*a0 .. 4*a0 + 4Q - 1 (bytes outside the window masked)
    uint32_t CA[Q], CB[Q], ivA[Q], ivB[Q], sA[Q], sB[Q], LA[Q], LB[Q];
    bool act[Q];
    {
        const uintptr_t addr = reinterpret_cast<uintptr_t>(cost) + pm.cell + (4 * a0 - lo);
        const uint32_t* aw = reinterpret_cast<const uint32_t*>(addr & ~static_cast<uintptr_t>(3));
        const uint32_t sh = 8u * static_cast<uint32_t>(addr & 3);
        uint32_t c[Q + 1];
#pragma unroll
        for (int t = 0; t <= Q; ++t) c[t] = __ldg(aw + t);
#pragma unroll
        for (int t = 0; t < Q; ++t) {
            const uint32_t cq = __funnelshift_r(c[t], c[t + 1], sh);
            CA[t] = prmt(cq, 0u, 0x4140u);
            CB[t] = prmt(cq, 0u, 0x4342u);
            act[t] = px && k0 + t < nq;
            const int d0 = 4 * (a0 + t);
            const uint32_t bad0 = (d0 < lo) ? 0x0000ffffu : 0u;
            const uint32_t bad1 = (d0 + 1 < lo || d0 + 1 > hi) ? 0xffff0000u : 0u;
            const uint32_t bad2 = (d0 + 2 < lo || d0 + 2 > hi) ? 0x0000ffffu : 0u;
            const uint32_t bad3 = (d0 + 3 > hi) ? 0xffff0000u : 0u;
            ivA[t] = act[t] ? (bad0 | bad1) : 0xffffffffu;
            ivB[t] = act[t] ? (bad2 | bad3) : 0xffffffffu;
            sA[t] = sB[t] = 0u;
        }
    }

    for (int j = 0; j < ndir; ++j) {
        const int dj = j == 0 ? di0 : (j == 1 ? di1 : di2);
        const int sbj = j == 0 ? sb0 : (j == 1 ? sb1 : sb2);
        const bool has_pred = l > 0 && static_cast<unsigned>(ii + dj) < static_cast<unsigned>(len);
        int sidx = ii + sbj;
        if (sidx >= len) sidx -= len;
        const uint32_t slot = static_cast<uint32_t>(j * len + sidx);
        const uint32_t sb = mbuf + slot * static_cast<uint32_t>(SB);
        const uint32_t rp = rng + 4u * slot;
        // predecessor words for quads a0-1 .. a0+Q (word of quad x at sb + 4 + 4x);
        // outside the predecessor's quad range they read as P2, with no
        // predecessor (image edge) as 0, which gives L = C (sgm.cpp:93-99)
        const uint32_t prng = lds32(rp);
        const int pq0 = static_cast<int>(prng & 0xffffu);
        const uint32_t span = (prng >> 16) - static_cast<uint32_t>(pq0);
        uint32_t w[Q + 2];
#pragma unroll
        for (int u = 0; u < Q + 2; ++u) {
            const uint32_t raw = lds32(sb + 4u * static_cast<uint32_t>(a0 + u));
            const bool in = static_cast<uint32_t>(a0 - 1 + u - pq0) <= span;
            w[u] = has_pred ? (in ? raw : P2x4) : 0u;
        }
        uint32_t mn = 0xffffffffu;
        uint32_t mma = prmt(w[0] >> 24, prmt(w[1], 0u, 0x4140u), 0x5410u);  // M(d0-1), M(d0)
#pragma unroll
        for (int t = 0; t < Q; ++t) {
            const uint32_t e0 = prmt(w[t + 1], 0u, 0x4140u);   // M(d0),   M(d0+1)
            const uint32_t e1 = prmt(w[t + 1], 0u, 0x4342u);   // M(d0+2), M(d0+3)
            const uint32_t mpa = prmt(w[t + 1], 0u, 0x4241u);  // M(d0+1), M(d0+2)
            const uint32_t mpb = prmt(e1, w[t + 2] & 0xffu, 0x5432u);  // M(d0+3), M(d0+4)
            LA[t] = __vadd2(__viaddmin_u16x2(__vminu2(mma, mpa), P1x2, e0), CA[t]);
            LB[t] = __vadd2(__viaddmin_u16x2(__vminu2(mpa, mpb), P1x2, e1), CB[t]);
            mn = __vminu2(mn, __vminu2(LA[t] | ivA[t], LB[t] | ivB[t]));
            mma = mpb;
        }
        const uint32_t m = group_min<G>(min(mn & 0xffffu, mn >> 16));
        const uint32_t neg = ((0x10000u - m) & 0xffffu) * 0x10001u;
        if (G > 1) __syncwarp();  // neighbours' reads of this lane's quads are done
#pragma unroll
        for (int t = 0; t < Q; ++t) {
            const uint32_t ma = __vmaxu2(__viaddmin_u16x2(LA[t], neg, P2x2), ivA[t] & P2x2);
            const uint32_t mb = __vmaxu2(__viaddmin_u16x2(LB[t], neg, P2x2), ivB[t] & P2x2);
            if (act[t]) sts32(sb + 4u + 4u * static_cast<uint32_t>(a0 + t), prmt(ma, mb, 0x6420u));
            sA[t] = __vadd2(sA[t], LA[t]);
            sB[t] = __vadd2(sB[t], LB[t]);
        }
        if (px && lg == 0) sts32(rp, qrange);
    }
#pragma unroll
    for (int t = 0; t < Q; ++t) {
        if (!act[t]) continue;
        const uint32_t qi = pm.qo + static_cast<uint32_t>(k0 + t);
        if (out_u16)
            reinterpret_cast<uint2*>(out)[qi] = make_uint2(sA[t], sB[t]);
        else
            reinterpret_cast<uint32_t*>(out)[qi] = prmt(sA[t], sB[t], 0x6420u);
    }
}

// Per-slot views of one role's line geometry and metadata sources.
struct RoleView {
    bool cols;
    int len, nlines, sign;
    const uint16_t *lo, *hi;
    const uint32_t *off, *qoff;
    const uint32_t *t_lohi, *t_cell, *t_qoff;  // column-major copies (cols)
    int W;
    __device__ __forceinline__ int line_coord(int l) const { return sign > 0 ? l : nlines - 1 - l; }
    // metadata of pixel i of line l (processing order)
    __device__ __forceinline__ void load(int l, int i, uint32_t& lohi, uint32_t& cell,
                                         uint32_t& qo) const {
        const int lc = line_coord(l);
        if (cols) {
            const size_t p = static_cast<size_t>(lc) * len + i;
            lohi = t_lohi[p];
            cell = t_cell[p];
            qo = t_qoff[p];
        } else {
            const size_t p = static_cast<size_t>(lc) * W + i;
            lohi = static_cast<uint32_t>(lo[p]) | (static_cast<uint32_t>(hi[p]) << 16);
            cell = off[p];
            qo = qoff[p];
        }
    }
};

// Column-major copies of (lo|hi<<16, cell offset, quad offset) for the column
// sweeps, via 32x32 shared-memory tiles (coalesced both ways).
__global__ void sweep_meta_kernel(Bufs b) {
    __shared__ uint32_t t0[32][33], t1[32][33], t2[32][33];
    const int a = blockIdx.z, s = slot_of(b, a);
    const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 32;
    const size_t P = b.P;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int x = x0 + threadIdx.x, y = y0 + r;
        if (x < b.W && y < b.H) {
            const size_t p = static_cast<size_t>(s) * P + static_cast<size_t>(y) * b.W + x;
            const size_t po = static_cast<size_t>(s) * (P + 1) + static_cast<size_t>(y) * b.W + x;
            t0[r][threadIdx.x] = static_cast<uint32_t>(b.lo[p]) | (static_cast<uint32_t>(b.hi[p]) << 16);
            t1[r][threadIdx.x] = b.off[po];
            t2[r][threadIdx.x] = b.qoff[po];
        }
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int y = y0 + threadIdx.x, x = x0 + r;
        if (x < b.W && y < b.H) {
            const size_t q = static_cast<size_t>(s) * P + static_cast<size_t>(x) * b.H + y;
            b.mt_lohi[q] = t0[threadIdx.x][r];
            b.mt_cell[q] = t1[threadIdx.x][r];
            b.mt_qoff[q] = t2[threadIdx.x][r];
        }
    }
}

__global__ void __launch_bounds__(kSweepThreads, 1) sweep_kernel(Bufs b, SweepParams sp) {
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ int item_s;
    const SweepPlan plan = sweep_plan(b.W, b.H, b.d_max);
    const int SB = sweep_slot_bytes(b.d_max);
    const uint32_t mbuf = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    const uint32_t rng = mbuf + static_cast<uint32_t>(plan.buf);
    int* done = reinterpret_cast<int*>(smem + plan.buf + plan.rng);
    const int warp = static_cast<int>(threadIdx.x >> 5), lane = static_cast<int>(threadIdx.x & 31);
    const uint32_t P1x2 = static_cast<uint32_t>(sp.p1) * 0x10001u;
    const uint32_t P2x2 = static_cast<uint32_t>(sp.p2) * 0x10001u;
    const uint32_t P2x4 = static_cast<uint32_t>(sp.p2) * 0x01010101u;
    const int n_ab = __popc(sp.roles & 3) * sp.n, n_cd = __popc(sp.roles & 12) * sp.n;

    for (;;) {
        if (threadIdx.x == 0) item_s = atomicAdd(b.work, 1);
        if (threadIdx.x < kSweepWarps) done[threadIdx.x] = 0;
        __syncthreads();
        const int item = item_s;
        __syncthreads();
        if (item >= n_ab + n_cd) break;
        // decode (column roles first: they carry 3 directions)
        int role, a;
        if (item < n_ab) {
            const int per = __popc(sp.roles & 3);
            a = item / per;
            const int r = item % per;
            role = (sp.roles & 1) ? r : 1;
        } else {
            const int it = item - n_ab, per = __popc(sp.roles & 12);
            a = it / per;
            const int r = it % per;
            role = (sp.roles & 4) ? 2 + r : 3;
        }
        const int s = slot_of(b, a);
        RoleView rv;
        rv.cols = role < 2;
        rv.sign = (role == 0 || role == 2) ? 1 : -1;
        rv.len = rv.cols ? b.H : b.W;
        rv.nlines = rv.cols ? b.W : b.H;
        rv.W = b.W;
        rv.lo = b.lo + static_cast<size_t>(s) * b.P;
        rv.hi = b.hi + static_cast<size_t>(s) * b.P;
        rv.off = b.off + static_cast<size_t>(s) * (b.P + 1);
        rv.qoff = b.qoff + static_cast<size_t>(s) * (b.P + 1);
        rv.t_lohi = b.mt_lohi + static_cast<size_t>(s) * b.P;
        rv.t_cell = b.mt_cell + static_cast<size_t>(s) * b.P;
        rv.t_qoff = b.mt_qoff + static_cast<size_t>(s) * b.P;
        const int len = rv.len, nlines = rv.nlines;
        const int ndir = rv.cols ? sp.ndir_ab : 1;
        const int di0 = rv.cols ? sp.di_ab[0] : 0, di1 = sp.di_ab[1], di2 = sp.di_ab[2];
        const bool cross = rv.cols && (ndir > 1 || di0 != 0);  // diagonal dependencies
        const uint8_t* cost = b.cost + static_cast<size_t>(s) * b.vol_cap;
        void* out;
        switch (role) {
            case 0: out = b.pA + static_cast<size_t>(s) * b.quad_cap * 4; break;
            case 1: out = b.pB + static_cast<size_t>(s) * b.quad_cap * 4; break;
            case 2: out = b.pC + static_cast<size_t>(s) * b.quad_cap * 4; break;
            default: out = b.pD + static_cast<size_t>(s) * b.quad_cap * 4; break;
        }
        const bool out_u16 = rv.cols;
        // this warp's block of line positions
        const int blk0 = warp * len / kSweepWarps, blk1 = (warp + 1) * len / kSweepWarps;
        const int nch = (blk1 - blk0 + 31) >> 5;

        PixMeta cur[kChunks], nxt[kChunks];
#pragma unroll
        for (int c = 0; c < kChunks; ++c) {
            const int i = blk0 + 32 * c + lane;
            cur[c] = PixMeta{0u, 0u, 0u};
            if (c < nch && i < blk1) rv.load(0, i, cur[c].lohi, cur[c].cell, cur[c].qo);
        }
        for (int l = 0; l < nlines; ++l) {
            // metadata of the next line (consumed next iteration)
#pragma unroll
            for (int c = 0; c < kChunks; ++c) {
                const int i = blk0 + 32 * c + lane;
                nxt[c] = PixMeta{0u, 0u, 0u};
                if (l + 1 < nlines && c < nch && i < blk1)
                    rv.load(l + 1, i, nxt[c].lohi, nxt[c].cell, nxt[c].qo);
            }
            // the neighbours' boundary pixels of line l-1 must be written
            if (cross && l > 0) {
                if (lane == 0) {
                    while ((warp > 0 && ld_acquire(&done[warp - 1]) < l) ||
                           (warp + 1 < kSweepWarps && ld_acquire(&done[warp + 1]) < l))
                        __nanosleep(32);
                }
                __syncwarp();
            }
            auto sbase = [&](int dj) {
                int v = (dj * l) % len;
                return v < 0 ? v + len : v;
            };
            const int sb0 = sbase(di0), sb1 = sbase(di1), sb2 = sbase(di2);
#pragma unroll
            for (int c = 0; c < kChunks; ++c) {
                if (c >= nch) break;
                const int i = blk0 + 32 * c + lane;
                const bool valid = i < blk1;
                const int nq = static_cast<int>(cur[c].lohi >> 18) -
                               static_cast<int>((cur[c].lohi & 0xffffu) >> 2) + 1;
                const bool narrow = valid && nq <= 4;
                // windows of <= 4 quads: one lane each
                sweep_pixel<1, 4>(narrow ? i : -1, cur[c], l, len, ndir, di0, di1, di2, sb0, sb1,
                                  sb2, mbuf, SB, rng, cost, out, out_u16, P1x2, P2x2, P2x4);
                // wider windows: 8 lanes x 4 quads, 4 pixels per pass
                unsigned bw = __ballot_sync(0xffffffffu, valid && !narrow);
                while (bw) {
                    const int g = lane >> 3;
                    const int cntw = __popc(bw);
                    const int src = g < cntw ? static_cast<int>(__fns(bw, 0, g + 1)) : 0;
                    PixMeta pmw;
                    pmw.lohi = __shfl_sync(0xffffffffu, cur[c].lohi, src);
                    pmw.cell = __shfl_sync(0xffffffffu, cur[c].cell, src);
                    pmw.qo = __shfl_sync(0xffffffffu, cur[c].qo, src);
                    const int iw = __shfl_sync(0xffffffffu, i, src);
                    sweep_pixel<8, 4>(g < cntw ? iw : -1, pmw, l, len, ndir, di0, di1, di2, sb0,
                                      sb1, sb2, mbuf, SB, rng, cost, out, out_u16, P1x2, P2x2,
                                      P2x4);
                    // drop the (up to) 4 pixels just done
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if (bw) bw &= bw - 1;
                }
            }
            if (cross) {
                __syncwarp();
                if (lane == 0) st_release(&done[warp], l + 1);
            }
            // pull line l+1's matching costs towards L2
#pragma unroll
            for (int c = 0; c < kChunks; ++c) {
                const int i = blk0 + 32 * c + lane;
                if (l + 1 < nlines && c < nch && i < blk1) {
                    const int lo = static_cast<int>(nxt[c].lohi & 0xffffu);
                    const int n = static_cast<int>(nxt[c].lohi >> 16) - lo + 1;
                    const uint8_t* c0 = cost + nxt[c].cell;
                    for (int o = 0; o < n + 4; o += 128)
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(c0 + o));
                }
                cur[c] = nxt[c];
            }
        }
        __syncthreads();
    }
}

// S = sum of the role partials, written in the reference's ragged layout. One
// CTA per (row, slot); threads over the row's cells (coalesced S stores).
__global__ void sweep_combine_kernel(Bufs b, int roles) {
    extern __shared__ uint32_t sm[];
    const int a = blockIdx.y, s = slot_of(b, a), y = blockIdx.x, W = b.W;
    uint32_t* o = sm;              // W+1 in-row cell offsets
    uint32_t* qo = o + W + 1;      // W quad offsets
    uint16_t* lo = reinterpret_cast<uint16_t*>(qo + W);
    const size_t pbase = static_cast<size_t>(s) * b.P + static_cast<size_t>(y) * W;
    const uint32_t* off = b.off + static_cast<size_t>(s) * (b.P + 1) + static_cast<size_t>(y) * W;
    const uint32_t* qoff = b.qoff + static_cast<size_t>(s) * (b.P + 1) + static_cast<size_t>(y) * W;
    const uint32_t row0 = off[0];
    for (int x = threadIdx.x; x < W; x += blockDim.x) {
        o[x] = off[x] - row0;
        qo[x] = qoff[x];
        lo[x] = b.lo[pbase + x];
    }
    if (threadIdx.x == 0) o[W] = off[W] - row0;
    __syncthreads();
    const uint32_t n = o[W];
    const size_t qb = static_cast<size_t>(s) * b.quad_cap * 4;
    const uint16_t* pA = b.pA + qb;
    const uint16_t* pB = b.pB + qb;
    const uint8_t* pC = b.pC + qb;
    const uint8_t* pD = b.pD + qb;
    uint16_t* agg = b.agg + static_cast<size_t>(s) * b.vol_cap + row0;
    for (uint32_t c = threadIdx.x; c < n; c += blockDim.x) {
        int l = 0, r = W;
        while (r - l > 1) {
            const int m = (l + r) >> 1;
            if (o[m] <= c) l = m; else r = m;
        }
        const int lv = lo[l] + static_cast<int>(c - o[l]);
        const size_t e = 4 * (static_cast<size_t>(qo[l]) + (lv >> 2) - (lo[l] >> 2)) + (lv & 3);
        uint32_t v = 0;
        if (roles & 1) v += pA[e];
        if (roles & 2) v += pB[e];
        if (roles & 4) v += pC[e];
        if (roles & 8) v += pD[e];
        agg[c] = static_cast<uint16_t>(v);
    }
}

void launch_aggregate_sweep(const Bufs& b, int n, int p1, int p2, int paths, int path_set,
                            int num_sms, Launch L) {
    SweepParams sp{};
    sp.p1 = p1;
    sp.p2 = p2;
    sp.n = n;
    const bool nondiag = paths == 8 || path_set == 0;
    const bool diag = paths == 8 || path_set == 1;
    int k = 0;
    if (nondiag) sp.di_ab[k++] = 0;
    if (diag) {
        sp.di_ab[k++] = -1;
        sp.di_ab[k++] = 1;
    }
    sp.ndir_ab = k;
    sp.roles = 3 | (nondiag ? 12 : 0);
    const SweepPlan plan = sweep_plan(b.W, b.H, b.d_max);
    const int items = (__builtin_popcount(sp.roles & 3) + __builtin_popcount(sp.roles & 12)) * n;
    const int grid = items < num_sms ? items : num_sms;
    cudaMemsetAsync(b.work, 0, sizeof(int), L.st);
    sweep_meta_kernel<<<dim3((b.W + 31) / 32, (b.H + 31) / 32, n), dim3(32, 8), 0, L.st>>>(b);
    cudaFuncSetAttribute(sweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(plan.total));
    sweep_kernel<<<grid, kSweepThreads, plan.total, L.st>>>(b, sp);
    const size_t csmem = sizeof(uint32_t) * (2 * b.W + 1) + sizeof(uint16_t) * b.W;
    sweep_combine_kernel<<<dim3(b.H, n), 512, csmem, L.st>>>(b, sp.roles);
    *L.counter += 3;
}

}  // namespace tsgm
