// Line-sweep 8-path aggregation over ragged windows (aggregate_paths,
// sgm.cpp:39-161 / SURVEY.md §8(a) row A14), the fast path.
//
// Decomposition. The 8 directions are grouped into 4 ROLES, each a sweep over
// LINES in which every direction's predecessor lies in the previous line:
//   A: columns x = 0..W-1,   directions (-1,0), (-1,-1), (-1,+1)
//   B: columns x = W-1..0,   directions (+1,0), (+1,-1), (+1,+1)
//   C: rows    y = 0..H-1,   direction  (0,-1)
//   D: rows    y = H-1..0,   direction  (0,+1)
// (4-path sets keep the subset). Within a line all pixels are independent, so
// a CTA processes a line FLAT: every pixel's window is split into aligned
// quads of 4 levels; pixels of <= 4 quads run as 4-lane groups (8 pixels per
// warp), wider ones as a whole warp. Arithmetic is u16x2 SIMD (VIADDMNMX /
// VIMNMX .U16x2), two levels per instruction.
//
// State. Per direction, each pixel's normalised path cost
//   M(d) = min(L(d) - min_k L(k), P2)      (P2 for levels outside the window)
// lives in shared memory in an ABSOLUTE-level slot (level d at byte 4 + d), so
// the recursion (sgm.cpp:100-126) becomes, with no bounds checks,
//   L(d) = C(d) + min(M_q(d), min(M_q(d-1), M_q(d+1)) + P1)
// (absent predecessor levels read as P2, which is exactly the reference's
// q_min + P2 cap after normalisation). Slots are SHEARED: direction (dl, di)
// stores pixel i of line l at slot (i + di*l) mod len, so a pixel reads and
// rewrites the same slot its predecessor wrote: one buffer per direction, one
// barrier per line. Levels that leave a slot's window are reset to P2 (the
// slot's quad range is tracked), keeping "outside the window == P2" invariant.
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

__host__ __device__ inline int sweep_slot_bytes(int d_max) { return 4 * ((d_max + 3) / 4 + 3); }

struct SweepPlan {
    size_t buf, rng, meta, lists, total;
};

constexpr int kMetaPerThread = 4;  // line length <= kSweepThreads * 4 = 2048

__host__ __device__ inline SweepPlan sweep_plan(int W, int H, int d_max) {
    SweepPlan p;
    const size_t sb = sweep_slot_bytes(d_max);
    const size_t slots = (3 * static_cast<size_t>(H) > static_cast<size_t>(W)) ? 3 * static_cast<size_t>(H) : W;
    const size_t lmax = W > H ? W : H;
    p.buf = slots * sb;
    p.rng = slots * 4;
    p.meta = 2 * 3 * lmax * 4;  // two lines in flight: lohi, cell, qoff
    p.lists = ((2 * lmax * 2) + 15) & ~static_cast<size_t>(15);
    p.total = p.buf + p.rng + p.meta + p.lists;
    return p;
}

bool sweep_supported(int W, int H, int d_max, int p2) {
    // u8 path costs need 24 + P2 <= 255; quads per lane <= 2 (d_max <= 256)
    const int lmax = W > H ? W : H;
    return kMaxCost + p2 <= 255 && d_max <= 256 && lmax <= kSweepThreads * kMetaPerThread &&
           sweep_plan(W, H, d_max).total <= 227 * 1024;
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

// Line metadata of one line (three u32 arrays in shared memory).
struct LineMeta {
    uint32_t* lohi;
    uint32_t* cell;
    uint32_t* qoff;
};

// Matching costs of one pixel's quads for one lane, fetched ahead of use.
template <int Q>
struct CostRegs {
    uint32_t w0[Q], w1[Q], sh[Q];
};

// Every lane of the warp calls this (inactive lanes: i < 0 or quad beyond the
// window) so that the group reductions can use full-warp shuffles; addresses
// are clamped into the window, results of inactive lanes are masked later.
template <int G, int Q>
__device__ __forceinline__ void fetch_costs(int i, const LineMeta& m, const uint8_t* cost,
                                            CostRegs<Q>& r) {
    const int lg = threadIdx.x & (G - 1);
    const uint32_t lohi = i >= 0 ? m.lohi[i] : 0u;
    const int lo = static_cast<int>(lohi & 0xffffu), hi = static_cast<int>(lohi >> 16);
    const int q0 = lo >> 2, nq = (hi >> 2) - q0 + 1;
    const uint32_t cell = i >= 0 ? m.cell[i] : 0u;
#pragma unroll
    for (int t = 0; t < Q; ++t) {
        const int k = min(lg + t * G, nq - 1);
        const uintptr_t addr = reinterpret_cast<uintptr_t>(cost) + cell + (4 * (q0 + k) - lo);
        const uint32_t* aw = reinterpret_cast<const uint32_t*>(addr & ~static_cast<uintptr_t>(3));
        r.w0[t] = __ldg(aw);
        r.w1[t] = __ldg(aw + 1);
        r.sh[t] = 8u * static_cast<uint32_t>(addr & 3);
    }
}

// min over the G lanes of a group; all 32 lanes must call it.
template <int G>
__device__ __forceinline__ uint32_t group_min(uint32_t v) {
    if (G == 32) return __reduce_min_sync(0xffffffffu, v);
#pragma unroll
    for (int o = 1; o < G; o <<= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ void sts32(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

// One pixel of a line, processed by a group of G lanes, each lane holding Q
// quads (quad k = lg + t*G). All lanes of the warp call it; a group with
// i < 0 has no pixel (everything masked, nothing stored). `mbuf` / `rng` are
// 32-bit shared-memory addresses.
template <int G, int Q>
__device__ __forceinline__ void sweep_pixel(int i, int l, int len, int ndir, int di0, int di1,
                                            int di2, int sb0, int sb1, int sb2, uint32_t mbuf,
                                            int SB, uint32_t rng, const LineMeta& meta,
                                            const CostRegs<Q>& cr, void* out, bool out_u16,
                                            uint32_t P1x2, uint32_t P2x2, uint32_t P2x4) {
    const int lane = threadIdx.x & 31;
    const int lg = lane & (G - 1);
    const bool px = i >= 0;
    const int ii = px ? i : 0;
    const uint32_t lohi = px ? meta.lohi[ii] : 0u;
    const int lo = static_cast<int>(lohi & 0xffffu), hi = static_cast<int>(lohi >> 16);
    const int q0 = lo >> 2, q1 = hi >> 2, nq = q1 - q0 + 1;
    const uint32_t qrange = static_cast<uint32_t>(q0) | (static_cast<uint32_t>(q1) << 16);

    bool act[Q];
    uint32_t dq[Q];  // byte offset of the lane's quad in a slot (clamped into the window)
    uint32_t CA[Q], CB[Q], ivA[Q], ivB[Q], sA[Q], sB[Q], LA[Q], LB[Q];
#pragma unroll
    for (int t = 0; t < Q; ++t) {
        const int k = lg + t * G;
        act[t] = px && k < nq;
        const int d0 = 4 * (q0 + min(k, nq - 1));
        dq[t] = static_cast<uint32_t>(d0);
        sA[t] = sB[t] = 0u;
        const uint32_t cq = __funnelshift_r(cr.w0[t], cr.w1[t], cr.sh[t]);
        CA[t] = prmt(cq, 0u, 0x4140u);
        CB[t] = prmt(cq, 0u, 0x4342u);
        const uint32_t bad0 = (d0 < lo) ? 0x0000ffffu : 0u;
        const uint32_t bad1 = (d0 + 1 < lo || d0 + 1 > hi) ? 0xffff0000u : 0u;
        const uint32_t bad2 = (d0 + 2 < lo || d0 + 2 > hi) ? 0x0000ffffu : 0u;
        const uint32_t bad3 = (d0 + 3 > hi) ? 0xffff0000u : 0u;
        ivA[t] = act[t] ? (bad0 | bad1) : 0xffffffffu;
        ivB[t] = act[t] ? (bad2 | bad3) : 0xffffffffu;
    }

    for (int j = 0; j < ndir; ++j) {
        const int dj = j == 0 ? di0 : (j == 1 ? di1 : di2);
        const int sbj = j == 0 ? sb0 : (j == 1 ? sb1 : sb2);
        const bool has_pred = l > 0 && static_cast<unsigned>(ii + dj) < static_cast<unsigned>(len);
        int sidx = ii + sbj;
        if (sidx >= len) sidx -= len;
        const uint32_t slot = static_cast<uint32_t>(j * len + sidx);
        const uint32_t sb = mbuf + slot * static_cast<uint32_t>(SB);
        uint32_t mn = 0xffffffffu;
#pragma unroll
        for (int t = 0; t < Q; ++t) {
            // no predecessor (image edge): M == 0 gives L = C (sgm.cpp:93-99)
            uint32_t w0 = 0u, w1 = 0u, w2 = 0u;
            if (has_pred) {
                w0 = lds32(sb + dq[t]);
                w1 = lds32(sb + dq[t] + 4);
                w2 = lds32(sb + dq[t] + 8);
            }
            const uint32_t e0 = prmt(w1, 0u, 0x4140u);  // M(d0),   M(d0+1)
            const uint32_t e1 = prmt(w1, 0u, 0x4342u);  // M(d0+2), M(d0+3)
            const uint32_t mpa = prmt(w1, 0u, 0x4241u); // M(d0+1), M(d0+2)
            const uint32_t mma = prmt(w0 >> 24, e0, 0x5410u);  // M(d0-1), M(d0)
            const uint32_t mpb = prmt(e1, w2 & 0xffu, 0x5432u); // M(d0+3), M(d0+4)
            LA[t] = __vadd2(__viaddmin_u16x2(__vminu2(mma, mpa), P1x2, e0), CA[t]);
            LB[t] = __vadd2(__viaddmin_u16x2(__vminu2(mpa, mpb), P1x2, e1), CB[t]);
            mn = __vminu2(mn, __vminu2(LA[t] | ivA[t], LB[t] | ivB[t]));
        }
        const uint32_t m = group_min<G>(min(mn & 0xffffu, mn >> 16));
        const uint32_t neg = ((0x10000u - m) & 0xffffu) * 0x10001u;
        // reset levels the slot held but this window does not cover
        const uint32_t rp = rng + 4u * slot;
        const uint32_t old = lds32(rp);
        __syncwarp();
#pragma unroll
        for (int t = 0; t < Q; ++t) {
            const uint32_t ma = __vmaxu2(__viaddmin_u16x2(LA[t], neg, P2x2), ivA[t] & P2x2);
            const uint32_t mb = __vmaxu2(__viaddmin_u16x2(LB[t], neg, P2x2), ivB[t] & P2x2);
            if (act[t]) sts32(sb + 4 + dq[t], prmt(ma, mb, 0x6420u));
            sA[t] = __vadd2(sA[t], LA[t]);
            sB[t] = __vadd2(sB[t], LB[t]);
        }
        if (px && old != qrange) {
            const int oq0 = static_cast<int>(old & 0xffffu), oq1 = static_cast<int>(old >> 16);
            for (int q = oq0 + lg; q <= oq1; q += G)
                if (q < q0 || q > q1) sts32(sb + 4 + 4 * q, P2x4);
            if (lg == 0) sts32(rp, qrange);
        }
    }
    const uint32_t qo = px ? meta.qoff[ii] : 0u;
#pragma unroll
    for (int t = 0; t < Q; ++t) {
        if (!act[t]) continue;
        const uint32_t qi = qo + lg + t * G;
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

template <int GW, int QW>
__global__ void __launch_bounds__(kSweepThreads, 1) sweep_kernel(Bufs b, SweepParams sp) {
    constexpr int kWidePerWarp = 32 / GW;
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ int cnt[2][2];
    __shared__ int item_s;
    const SweepPlan plan = sweep_plan(b.W, b.H, b.d_max);
    const int SB = sweep_slot_bytes(b.d_max);
    const int lmax = b.W > b.H ? b.W : b.H;
    uint8_t* mbuf = smem;
    uint32_t* rng = reinterpret_cast<uint32_t*>(smem + plan.buf);
    const uint32_t mbuf_s = static_cast<uint32_t>(__cvta_generic_to_shared(mbuf));
    const uint32_t rng_s = static_cast<uint32_t>(__cvta_generic_to_shared(rng));
    uint32_t* mbase = reinterpret_cast<uint32_t*>(smem + plan.buf + plan.rng);
    auto meta_set = [&](int k) {
        LineMeta m;
        m.lohi = mbase + (3 * k + 0) * lmax;
        m.cell = mbase + (3 * k + 1) * lmax;
        m.qoff = mbase + (3 * k + 2) * lmax;
        return m;
    };
    uint16_t* l_narrow = reinterpret_cast<uint16_t*>(mbase + 6 * lmax);
    uint16_t* l_wide = l_narrow + lmax;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t P1x2 = static_cast<uint32_t>(sp.p1) * 0x10001u;
    const uint32_t P2x2 = static_cast<uint32_t>(sp.p2) * 0x10001u;
    const uint32_t P2x4 = static_cast<uint32_t>(sp.p2) * 0x01010101u;
    const int n_ab = __popc(sp.roles & 3) * sp.n, n_cd = __popc(sp.roles & 12) * sp.n;

    for (;;) {
        if (threadIdx.x == 0) item_s = atomicAdd(b.work, 1);
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
        const uint8_t* cost = b.cost + static_cast<size_t>(s) * b.vol_cap;
        void* out;
        switch (role) {
            case 0: out = b.pA + static_cast<size_t>(s) * b.quad_cap * 4; break;
            case 1: out = b.pB + static_cast<size_t>(s) * b.quad_cap * 4; break;
            case 2: out = b.pC + static_cast<size_t>(s) * b.quad_cap * 4; break;
            default: out = b.pD + static_cast<size_t>(s) * b.quad_cap * 4; break;
        }
        const bool out_u16 = rv.cols;

        // all slots start as "absent" (P2) with an empty quad range
        {
            uint4* mw = reinterpret_cast<uint4*>(mbuf);
            const size_t vecs = static_cast<size_t>(ndir) * len * SB / 16;
            const uint4 fill = make_uint4(P2x4, P2x4, P2x4, P2x4);
            for (size_t w = threadIdx.x; w < vecs; w += kSweepThreads) mw[w] = fill;
            uint32_t* mt = reinterpret_cast<uint32_t*>(mbuf);
            for (size_t w = vecs * 4 + threadIdx.x; w < static_cast<size_t>(ndir) * len * SB / 4;
                 w += kSweepThreads)
                mt[w] = P2x4;
            for (int w = threadIdx.x; w < ndir * len; w += kSweepThreads) rng[w] = 0x0000ffffu;
        }
        // metadata of lines 0 and 1
        for (int k = 0; k < 2 && k < nlines; ++k) {
            const LineMeta m = meta_set(k);
            for (int i = threadIdx.x; i < len; i += kSweepThreads)
                rv.load(k, i, m.lohi[i], m.cell[i], m.qoff[i]);
        }
        if (threadIdx.x == 0) cnt[0][0] = cnt[0][1] = cnt[1][0] = cnt[1][1] = 0;
        __syncthreads();

        // classify line `l` (metadata in `m`) into the narrow / wide lists
        auto classify = [&](const LineMeta& m, int* c) {
            for (int base = 0; base < len; base += kSweepThreads) {
                const int i = base + threadIdx.x;
                bool narrow = false, wide = false;
                if (i < len) {
                    const uint32_t lohi = m.lohi[i];
                    const int nq = static_cast<int>(lohi >> 18) - static_cast<int>((lohi & 0xffffu) >> 2) + 1;
                    narrow = nq <= 4;
                    wide = !narrow;
                }
                const unsigned bn = __ballot_sync(0xffffffffu, narrow);
                const unsigned bw = __ballot_sync(0xffffffffu, wide);
                int basen = 0, basew = 0;
                if (lane == 0) {
                    if (bn) basen = atomicAdd(&c[0], __popc(bn));
                    if (bw) basew = atomicAdd(&c[1], __popc(bw));
                }
                basen = __shfl_sync(0xffffffffu, basen, 0);
                basew = __shfl_sync(0xffffffffu, basew, 0);
                const unsigned lt = (1u << lane) - 1u;
                if (narrow) l_narrow[basen + __popc(bn & lt)] = static_cast<uint16_t>(i);
                if (wide) l_wide[basew + __popc(bw & lt)] = static_cast<uint16_t>(i);
            }
        };
        classify(meta_set(0), cnt[0]);
        __syncthreads();

        for (int l = 0; l < nlines; ++l) {
            const LineMeta cur = meta_set(l & 1);
            const LineMeta nxt = meta_set((l + 1) & 1);
            // (a) metadata of line l+2 into registers (stored after this line)
            uint32_t r_lohi[kMetaPerThread], r_cell[kMetaPerThread], r_qoff[kMetaPerThread];
            const bool have2 = l + 2 < nlines;
#pragma unroll
            for (int k = 0; k < kMetaPerThread; ++k) {
                const int i = threadIdx.x + k * kSweepThreads;
                if (have2 && i < len) rv.load(l + 2, i, r_lohi[k], r_cell[k], r_qoff[k]);
            }
            // (b) pull line l+1's matching costs towards L2
            if (l + 1 < nlines) {
                for (int i = threadIdx.x; i < len; i += kSweepThreads) {
                    const uint32_t lohi = nxt.lohi[i];
                    const int n = static_cast<int>(lohi >> 16) - static_cast<int>(lohi & 0xffffu) + 1;
                    const uint8_t* c0 = cost + nxt.cell[i];
                    for (int o = 0; o < n + 4; o += 128)
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(c0 + o));
                }
            }
            // (c) this line's pixels, next unit's costs fetched ahead
            int* c_cur = &cnt[0][0] + 2 * (l & 1);
            int* c_nxt = &cnt[0][0] + 2 * ((l + 1) & 1);
            const int n_narrow = c_cur[0], n_wide = c_cur[1];
            if (threadIdx.x == 0) c_nxt[0] = c_nxt[1] = 0;
            const int u_narrow = (n_narrow + 7) >> 3;
            const int u_wide = (n_wide + kWidePerWarp - 1) / kWidePerWarp;
            const int total = u_narrow + u_wide;
            // sheared slot bases of this line, (dj * l) mod len per direction
            auto sbase = [&](int dj) {
                int v = (dj * l) % len;
                return v < 0 ? v + len : v;
            };
            const int sb0 = sbase(di0), sb1 = sbase(di1), sb2 = sbase(di2);
            // pixel of this lane's group in unit uu (-1: none)
            auto unit_pixel = [&](int uu) -> int {
                if (uu < u_narrow) {
                    const int e = uu * 8 + (lane >> 2);
                    return e < n_narrow ? static_cast<int>(l_narrow[e]) : -1;
                }
                const int e = (uu - u_narrow) * kWidePerWarp + lane / GW;
                return e < n_wide ? static_cast<int>(l_wide[e]) : -1;
            };
            int u = warp;
            CostRegs<QW> cr_cur, cr_nxt;
            auto fetch_unit = [&](int uu, CostRegs<QW>& r) {
                if (uu < u_narrow) {
                    CostRegs<1> r1;
                    fetch_costs<4, 1>(unit_pixel(uu), cur, cost, r1);
                    r.w0[0] = r1.w0[0];
                    r.w1[0] = r1.w1[0];
                    r.sh[0] = r1.sh[0];
                } else {
                    fetch_costs<GW, QW>(unit_pixel(uu), cur, cost, r);
                }
            };
            if (u < total) fetch_unit(u, cr_cur);
            while (u < total) {
                const int un = u + kSweepWarps;
                if (un < total) fetch_unit(un, cr_nxt);
                if (u < u_narrow) {
                    CostRegs<1> r1;
                    r1.w0[0] = cr_cur.w0[0];
                    r1.w1[0] = cr_cur.w1[0];
                    r1.sh[0] = cr_cur.sh[0];
                    sweep_pixel<4, 1>(unit_pixel(u), l, len, ndir, di0, di1, di2, sb0, sb1, sb2,
                                      mbuf_s, SB, rng_s, cur, r1, out, out_u16, P1x2, P2x2, P2x4);
                } else {
                    sweep_pixel<GW, QW>(unit_pixel(u), l, len, ndir, di0, di1, di2, sb0, sb1, sb2,
                                        mbuf_s, SB, rng_s, cur, cr_cur, out, out_u16, P1x2, P2x2,
                                        P2x4);
                }
                cr_cur = cr_nxt;
                u = un;
            }
            __syncthreads();
            // line l's metadata slot now takes line l+2; classify line l+1
#pragma unroll
            for (int k = 0; k < kMetaPerThread; ++k) {
                const int i = threadIdx.x + k * kSweepThreads;
                if (have2 && i < len) {
                    cur.lohi[i] = r_lohi[k];
                    cur.cell[i] = r_cell[k];
                    cur.qoff[i] = r_qoff[k];
                }
            }
            if (l + 1 < nlines) classify(nxt, c_nxt);
            __syncthreads();
        }
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
    // wide windows: groups of 8 lanes x 4 quads (<= 128 levels, 4 pixels per
    // warp) or 16 lanes x 4 quads (<= 256 levels)
    if ((b.d_max + 3) / 4 <= 32) {
        cudaFuncSetAttribute(sweep_kernel<8, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(plan.total));
        sweep_kernel<8, 4><<<grid, kSweepThreads, plan.total, L.st>>>(b, sp);
    } else {
        cudaFuncSetAttribute(sweep_kernel<16, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(plan.total));
        sweep_kernel<16, 4><<<grid, kSweepThreads, plan.total, L.st>>>(b, sp);
    }
    const size_t csmem = sizeof(uint32_t) * (2 * b.W + 1) + sizeof(uint16_t) * b.W;
    sweep_combine_kernel<<<dim3(b.H, n), 512, csmem, L.st>>>(b, sp.roles);
    *L.counter += 3;
}

}  // namespace tsgm
