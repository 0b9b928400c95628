// Census, search ranges + prefix sums, ragged matching cost, WTA and median:
// the per-pixel integer stages of sgm_match and step (SURVEY.md §8(a) rows
// A10-A13, A15, A19). All results are bit-exact restatements of the cited
// reference lines.
#include "common.cuh"

namespace tsgm {

// ---------------------------------------------------------------- census (A12)
// census_transform, matching_cost.cpp:53-79, four horizontally adjacent
// pixels per thread in byte-SIMD (SWAR) form: the 5x5 neighbour bytes of the
// four pixels are 4-byte funnel shifts of the tile's row words, one strict
// unsigned compare against the four centres yields the four census bits in
// the bytes' MSBs (3 logic/add ops), and three accumulators collect 8 bits
// per byte lane each (the signature's bytes), assembled per pixel at the end.
// Bit order as the reference: raster order, first compare in bit 23. A CTA
// covers 128 x 8 pixels; the 136 x 12 byte tile (2-px halo, word aligned) is
// staged in shared memory.
constexpr int kCsW = 128, kCsH = 8, kCsPitch = kCsW + 8;

__device__ __forceinline__ uint32_t lt_msb(uint32_t x, uint32_t c_lo7, uint32_t c) {
    // per byte: MSB set iff x < c (unsigned): borrow-free subtract on the low
    // 7 bits, then the top bits decide (checked on all 65536 byte pairs)
    const uint32_t d = (x | 0x80808080u) - c_lo7;
    return (~x & c) | (~(x ^ c) & ~d);
}

__global__ void __launch_bounds__(256) census_kernel(Bufs b) {
    __shared__ __align__(16) uint8_t tile[kCsH + 4][kCsPitch];
    const int a = blockIdx.z >> 1, which = blockIdx.z & 1;
    const int s = slot_of(b, a);
    const uint8_t* img = which ? b.right[a] : b.left[a];
    uint32_t* sig = (which ? b.sigr : b.sigl) + static_cast<size_t>(s) * b.P;
    const int x0 = blockIdx.x * kCsW, y0 = blockIdx.y * kCsH;
    // the tile as 32-bit words (rows are not word-aligned in the image when W
    // % 4 != 0: two aligned loads and a funnel shift per word); CTAs whose
    // halo (plus the 3 bytes a misaligned last word may touch) leaves the
    // image row take the bytewise path
    const int gx0 = x0 - 4;
    if (gx0 >= 0 && gx0 + kCsPitch + 4 <= b.W) {
        for (int ty = threadIdx.y; ty < kCsH + 4; ty += kCsH) {
            const int gy = y0 - 2 + ty;
            uint32_t* trow = reinterpret_cast<uint32_t*>(&tile[ty][0]);
            if (gy < 0 || gy >= b.H) {
                for (int w = threadIdx.x; w < kCsPitch / 4; w += 32) trow[w] = 0u;
                continue;
            }
            const uintptr_t A = reinterpret_cast<uintptr_t>(img + static_cast<size_t>(gy) * b.W + gx0);
            const uint32_t* aw = reinterpret_cast<const uint32_t*>(A & ~static_cast<uintptr_t>(3));
            const uint32_t sh = 8u * static_cast<uint32_t>(A & 3);
            for (int w = threadIdx.x; w < kCsPitch / 4; w += 32) {
                const uint32_t lo = __ldg(aw + w), hi = sh ? __ldg(aw + w + 1) : 0u;
                trow[w] = __funnelshift_r(lo, hi, sh);
            }
        }
    } else {
        for (int ty = threadIdx.y; ty < kCsH + 4; ty += kCsH)
            for (int tx = threadIdx.x; tx < kCsPitch; tx += 32) {
                const int gx = gx0 + tx, gy = y0 - 2 + ty;
                tile[ty][tx] = (gx >= 0 && gx < b.W && gy >= 0 && gy < b.H) ? img[gy * b.W + gx] : 0;
            }
    }
    __syncthreads();
    const int xg = x0 + 4 * static_cast<int>(threadIdx.x), y = y0 + static_cast<int>(threadIdx.y);
    if (xg >= b.W || y >= b.H) return;
    uint32_t nb[5][5];  // neighbour words: [dy][dx] = bytes of x+dx-2 for the four pixels
#pragma unroll
    for (int dy = 0; dy < 5; ++dy) {
        const uint32_t* row = reinterpret_cast<const uint32_t*>(&tile[threadIdx.y + dy][0]);
        const uint32_t A = row[threadIdx.x], B = row[threadIdx.x + 1], C = row[threadIdx.x + 2];
        nb[dy][0] = __funnelshift_r(A, B, 16);
        nb[dy][1] = __funnelshift_r(A, B, 24);
        nb[dy][2] = B;
        nb[dy][3] = __funnelshift_r(B, C, 8);
        nb[dy][4] = __funnelshift_r(B, C, 16);
    }
    const uint32_t c = nb[2][2], c_lo7 = c & 0x7f7f7f7fu;
    uint32_t acc[3] = {0u, 0u, 0u};  // signature bits 16-23, 8-15, 0-7
    // compare k (raster order, centre skipped) lands in bit 23 - k: insert
    // each byte lane's 8 bits from the last compare of its group to the first
#pragma unroll
    for (int k = 23; k >= 0; --k) {
        const int pos = k < 12 ? k : k + 1;  // skip the centre (position 12)
        const uint32_t t = lt_msb(nb[pos / 5][pos % 5], c_lo7, c);
        uint32_t& r = acc[k >> 3];
        r = ((r >> 1) & 0x7f7f7f7fu) | (t & 0x80808080u);
    }
    uint32_t* out = sig + static_cast<size_t>(y) * b.W + xg;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int x = xg + i;
        if (x >= b.W) break;
        uint32_t v = __byte_perm(acc[2], acc[1], static_cast<uint32_t>(i | ((i + 4) << 4)));  // bits 0-15
        v = __byte_perm(v, acc[0], static_cast<uint32_t>(0x10 | (i + 4) << 8)) & 0x00ffffffu;
        out[i] = census_defined(x, y, b.W, b.H) ? v : 0u;
    }
}

void launch_census(const Bufs& b, int n, Launch L) {
    dim3 grid((b.W + kCsW - 1) / kCsW, (b.H + kCsH - 1) / kCsH, 2 * n);
    census_kernel<<<grid, dim3(32, kCsH), 0, L.st>>>(b);
    ++*L.counter;
}

// ---------------------------------------------------------------- ranges (A10, A11)
// derive_search_ranges, temporal_filter.cpp:108-143, fused with the in-row
// part of make_cost_volume's exclusive scan (matching_cost.cpp:30-48).
// One CTA per (row, active slot); row totals go to row_sum.
constexpr int kRowThreads = 256;

// Block-wide exclusive scan of one u32 per thread; returns the block total.
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t& excl) {
    __shared__ uint32_t warp_tot[kRowThreads / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) warp_tot[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        uint32_t w = lane < kRowThreads / 32 ? warp_tot[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += t;
        }
        if (lane < kRowThreads / 32) warp_tot[lane] = w;  // inclusive
    }
    __syncthreads();
    const uint32_t before = wid ? warp_tot[wid - 1] : 0;
    excl = before + incl - v;
    const uint32_t total = warp_tot[kRowThreads / 32 - 1];
    __syncthreads();
    return total;
}

// Quads of a window: aligned groups of 4 levels covering [lo, hi]; the
// aggregation partials use a quad-aligned copy of the ragged layout.
// (the layout allocates alloc_quads() of them: 16-byte aligned windows)
__device__ __forceinline__ uint32_t quads_of(int lo, int hi) {
    return alloc_quads(static_cast<uint32_t>((hi >> 2) - (lo >> 2) + 1));
}

template <bool kDerive>
__global__ void ranges_kernel(Bufs b, int min_hw, int use_stddev, double gain) {
    const int a = blockIdx.y, s = slot_of(b, a), y = blockIdx.x;
    const size_t base = static_cast<size_t>(s) * b.P + static_cast<size_t>(y) * b.W;
    const int per = (b.W + kRowThreads - 1) / kRowThreads;
    const int x0 = threadIdx.x * per;
    const int top = b.d_max - 1, min_len = 2 * min_hw + 1;
    uint32_t sum = 0, qsum = 0;
    for (int k = 0; k < per; ++k) {
        const int x = x0 + k;
        if (x >= b.W) break;
        int lo, hi;
        if (kDerive) {
            lo = 0;
            hi = top;
            if (b.pv[base + x]) derive_range(b.pd[base + x], b.pp[base + x], top, min_len,
                                             use_stddev, gain, lo, hi);
            b.lo[base + x] = static_cast<uint16_t>(lo);
            b.hi[base + x] = static_cast<uint16_t>(hi);
        } else {
            lo = b.lo[base + x];
            hi = b.hi[base + x];
        }
        sum += static_cast<uint32_t>(hi - lo + 1);
        qsum += quads_of(lo, hi);
    }
    uint32_t excl, qexcl;
    const uint32_t total = block_exclusive_scan(sum, excl);
    const uint32_t qtotal = block_exclusive_scan(qsum, qexcl);
    const size_t orow = static_cast<size_t>(s) * (b.P + 1) + static_cast<size_t>(y) * b.W;
    uint32_t* off = b.off + orow;
    uint32_t* qoff = b.qoff + orow;
    uint32_t run = excl, qrun = qexcl;
    for (int k = 0; k < per; ++k) {
        const int x = x0 + k;
        if (x >= b.W) break;
        off[x] = run;  // in-row exclusive; rebased by offsets_finalize
        qoff[x] = qrun;
        const int lo = b.lo[base + x], hi = b.hi[base + x];
        b.lohi[base + x] = static_cast<uint32_t>(lo) | (static_cast<uint32_t>(hi) << 16);
        run += static_cast<uint32_t>(hi - lo + 1);
        qrun += quads_of(lo, hi);
    }
    if (threadIdx.x == 0) {
        b.row_sum[static_cast<size_t>(s) * b.H + y] = total;
        b.qrow_sum[static_cast<size_t>(s) * b.H + y] = qtotal;
    }
}

void launch_ranges_from_pred(const Bufs& b, int n, int min_hw, int use_stddev, double gain,
                             Launch L) {
    ranges_kernel<true><<<dim3(b.H, n), kRowThreads, 0, L.st>>>(b, min_hw, use_stddev, gain);
    ++*L.counter;
}
void launch_ranges_given(const Bufs& b, int n, Launch L) {
    ranges_kernel<false><<<dim3(b.H, n), kRowThreads, 0, L.st>>>(b, 0, 0, 0.0);
    ++*L.counter;
}

// Per slot: exclusive scan of the row totals in u64 (overflow -> flag, the
// reference throws at matching_cost.cpp:43-44), for the cell offsets (y = 0)
// and the quad offsets (y = 1); then rebase every offset.
__global__ void row_scan_kernel(Bufs b) {
    const int a = blockIdx.x, s = slot_of(b, a), which = blockIdx.y;
    __shared__ unsigned long long carry;
    __shared__ unsigned long long part[1024];
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    uint32_t* rs = (which ? b.qrow_sum : b.row_sum) + static_cast<size_t>(s) * b.H;
    for (int base = 0; base < b.H; base += 1024) {
        const int y = base + threadIdx.x;
        const unsigned long long v = y < b.H ? rs[y] : 0ull;
        part[threadIdx.x] = v;
        __syncthreads();
        for (int o = 1; o < 1024; o <<= 1) {  // Hillis-Steele, H is small
            const unsigned long long t = threadIdx.x >= o ? part[threadIdx.x - o] : 0ull;
            __syncthreads();
            part[threadIdx.x] += t;
            __syncthreads();
        }
        const unsigned long long incl = part[threadIdx.x] + carry;
        __syncthreads();
        if (y < b.H) {
            const unsigned long long excl = incl - v;
            rs[y] = excl > 0xffffffffull ? 0xffffffffu : static_cast<uint32_t>(excl);
        }
        if (threadIdx.x == 1023) carry = incl;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const size_t last = static_cast<size_t>(s) * (b.P + 1) + b.P;
        if (which == 0) {
            b.ncells[s] = carry;
            b.overflow[s] = carry > 0xffffffffull ? 1 : 0;
            b.off[last] = static_cast<uint32_t>(carry);
        } else {
            b.nquads[s] = carry;
            b.qoff[last] = static_cast<uint32_t>(carry);
        }
    }
}

// Adds the row bases to the in-row offsets, and writes the packed records
// {lohi, qoff} the scan kernel loads with one 8-byte access: row-major
// (lanes = adjacent pixels of a row) and column-major (horizontal scanlines,
// lanes = consecutive rows). 32x32 tiles through shared memory.
__global__ void offsets_finalize_kernel(Bufs b) {
    __shared__ uint2 tile[32][33];
    const int a = blockIdx.z, s = slot_of(b, a);
    const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 32;
    const int tx = threadIdx.x, ty = threadIdx.y;
    const size_t obase = static_cast<size_t>(s) * (b.P + 1), pbase = static_cast<size_t>(s) * b.P;
    for (int j = ty; j < 32; j += 8) {
        const int y = y0 + j, x = x0 + tx;
        if (y < b.H && x < b.W) {
            const uint32_t rb = b.row_sum[static_cast<size_t>(s) * b.H + y];
            const uint32_t qb = b.qrow_sum[static_cast<size_t>(s) * b.H + y];
            const size_t o = obase + static_cast<size_t>(y) * b.W + x;
            const uint32_t off = b.off[o] + rb, qo = b.qoff[o] + qb;
            b.off[o] = off;
            b.qoff[o] = qo;
            const uint32_t lh = b.lohi[pbase + static_cast<size_t>(y) * b.W + x];
            const uint2 rec = make_uint2(lh, qo);
            b.rmeta[pbase + static_cast<size_t>(y) * b.W + x] = rec;
            tile[j][tx] = rec;
        }
    }
    __syncthreads();
    for (int j = ty; j < 32; j += 8) {
        const int x = x0 + j, y = y0 + tx;
        if (y < b.H && x < b.W) b.tmeta[pbase + static_cast<size_t>(x) * b.H + y] = tile[tx][j];
    }
}

void launch_offsets(const Bufs& b, int n, Launch L) {
    row_scan_kernel<<<dim3(n, 2), 1024, 0, L.st>>>(b);
    offsets_finalize_kernel<<<dim3((b.W + 31) / 32, (b.H + 31) / 32, n), dim3(32, 8), 0, L.st>>>(b);
    *L.counter += 2;
}

// The step's offsets from predict_tile_kernel's per-tile row counts (tsum,
// [slot][H][tiles_x] of (cells, quads) over 32-pixel tile rows).
// tile_scan_kernel: per slot, the row totals' exclusive scan in u64 (the
// reference throws for N >= 2^32, matching_cost.cpp:43-44: validate_config
// bounds W*H*d_max below that), then each tile row's exclusive offset in
// place. One CTA per (slot, cells|quads).
__global__ void tile_scan_kernel(Bufs b) {
    const int a = blockIdx.x, s = slot_of(b, a), which = blockIdx.y;
    const int tiles_x = (b.W + 31) / 32;
    __shared__ unsigned long long carry;
    __shared__ unsigned long long part[1024];
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    uint32_t* ts = reinterpret_cast<uint32_t*>(b.tsum + static_cast<size_t>(s) * b.H * tiles_x) + which;
    for (int base = 0; base < b.H; base += 1024) {
        const int y = base + threadIdx.x;
        unsigned long long v = 0ull;
        if (y < b.H)
            for (int t = 0; t < tiles_x; ++t) v += ts[2 * (static_cast<size_t>(y) * tiles_x + t)];
        part[threadIdx.x] = v;
        __syncthreads();
        for (int o = 1; o < 1024; o <<= 1) {  // Hillis-Steele, H is small
            const unsigned long long t = threadIdx.x >= o ? part[threadIdx.x - o] : 0ull;
            __syncthreads();
            part[threadIdx.x] += t;
            __syncthreads();
        }
        const unsigned long long incl = part[threadIdx.x] + carry;
        __syncthreads();
        if (y < b.H) {
            unsigned long long run = incl - v;
            for (int t = 0; t < tiles_x; ++t) {
                uint32_t* e = ts + 2 * (static_cast<size_t>(y) * tiles_x + t);
                const uint32_t c = *e;
                *e = static_cast<uint32_t>(run);
                run += c;
            }
        }
        if (threadIdx.x == 1023) carry = incl;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const size_t last = static_cast<size_t>(s) * (b.P + 1) + b.P;
        if (which == 0) {
            b.ncells[s] = carry;
            b.overflow[s] = carry > 0xffffffffull ? 1 : 0;
            b.off[last] = static_cast<uint32_t>(carry);
        } else {
            b.nquads[s] = carry;
            b.qoff[last] = static_cast<uint32_t>(carry);
        }
    }
}

// Cell and quad offsets of every pixel (tile offset + in-tile exclusive warp
// scan), the packed scan records (rmeta row-major, tmeta column-major via a
// 32x32 shared-memory transpose) and, for the step, the warp keys re-armed
// for the next frame (kd = 0, (kp, ks) = ~0: nothing reads them after the
// predict tile kernel).
__global__ void offsets_tile_kernel(Bufs b, int arm_keys) {
    __shared__ uint2 tile[32][33];
    const int a = blockIdx.z, s = slot_of(b, a);
    const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 32;
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int tiles_x = (b.W + 31) / 32;
    const size_t obase = static_cast<size_t>(s) * (b.P + 1), pbase = static_cast<size_t>(s) * b.P;
    for (int j = ty; j < 32; j += 8) {  // (uniform per warp: a warp is one tile row)
        const int y = y0 + j, x = x0 + tx;
        const bool in = y < b.H && x < b.W;
        const size_t g = pbase + static_cast<size_t>(y) * b.W + x;
        const uint32_t lh = in ? b.lohi[g] : 0u;
        const uint32_t nc = in ? (lh >> 16) - (lh & 0xffffu) + 1u : 0u;
        const uint32_t nq = in ? alloc_quads((lh >> 18) - ((lh & 0xffffu) >> 2) + 1u) : 0u;
        uint32_t ic = nc, iq = nq;  // inclusive warp scans
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t c = __shfl_up_sync(0xffffffffu, ic, o);
            const uint32_t qq = __shfl_up_sync(0xffffffffu, iq, o);
            if (tx >= o) {
                ic += c;
                iq += qq;
            }
        }
        if (in) {
            const uint2 tb = b.tsum[(static_cast<size_t>(s) * b.H + y) * tiles_x + blockIdx.x];
            const uint32_t off = tb.x + ic - nc, qo = tb.y + iq - nq;
            const size_t o = obase + static_cast<size_t>(y) * b.W + x;
            b.off[o] = off;
            b.qoff[o] = qo;
            const uint2 rec = make_uint2(lh, qo);
            b.rmeta[g] = rec;
            tile[j][tx] = rec;
            if (arm_keys) {
                b.kd[g] = 0ull;
                b.kps[g] = make_ulonglong2(~0ull, ~0ull);
            }
        }
    }
    __syncthreads();
    for (int j = ty; j < 32; j += 8) {
        const int x = x0 + j, y = y0 + tx;
        if (y < b.H && x < b.W) b.tmeta[pbase + static_cast<size_t>(x) * b.H + y] = tile[tx][j];
    }
}

void launch_offsets_step(const Bufs& b, int n, Launch L) {
    tile_scan_kernel<<<dim3(n, 2), 1024, 0, L.st>>>(b);
    offsets_tile_kernel<<<dim3((b.W + 31) / 32, (b.H + 31) / 32, n), dim3(32, 8), 0, L.st>>>(b, 1);
    *L.counter += 2;
}

// ---------------------------------------------------------------- cost (A13)
// (Tried: computing each chunk into a shared-memory staging buffer and
// writing it out with 16-byte stores: 0.85 -> 1.14 ms for 64 sequences'
// reduced frames; the byte stores below are not the limiter.)
// build_cost_volume, matching_cost.cpp:88-117. One CTA per (row, slot); the
// row's census signatures are staged in shared memory. Warps take 32-pixel
// chunks: a window of <= 16 levels is written by its own lane, a wider window
// by the whole warp (lanes across its levels, coalesced byte stores).
__device__ __forceinline__ uint8_t cell_cost(const uint32_t* sl, const uint32_t* sr, int x, int d,
                                             int W, bool row_def) {
    const int xr = x - d;
    const bool ok = row_def && x >= kCensusRadius && x < W - kCensusRadius &&
                    xr >= kCensusRadius && xr < W - kCensusRadius;
    return ok ? static_cast<uint8_t>(__popc(sl[x] ^ sr[xr])) : static_cast<uint8_t>(kMaxCost);
}

__global__ void __launch_bounds__(512) cost_kernel(Bufs b) {
    extern __shared__ uint32_t sm[];
    const int a = blockIdx.y, s = slot_of(b, a), y = blockIdx.x;
    const int W = b.W;
    uint32_t* sl = sm;
    uint32_t* sr = sl + W;
    const size_t pbase = static_cast<size_t>(s) * b.P + static_cast<size_t>(y) * W;
    const uint32_t* off = b.off + static_cast<size_t>(s) * (b.P + 1) + static_cast<size_t>(y) * W;
    for (int x = threadIdx.x; x < W; x += blockDim.x) {
        sl[x] = b.sigl[pbase + x];
        sr[x] = b.sigr[pbase + x];
    }
    __syncthreads();
    uint8_t* base = b.cost + b.vbase[a];
    const bool row_def = y >= kCensusRadius && y < b.H - kCensusRadius;
    const int warp = static_cast<int>(threadIdx.x >> 5), lane = static_cast<int>(threadIdx.x & 31);
    const int nwarps = static_cast<int>(blockDim.x >> 5);
    for (int x0 = warp * 32; x0 < W; x0 += 32 * nwarps) {
        const int x = x0 + lane;
        const bool active = x < W;
        const uint32_t lh = active ? b.lohi[pbase + x] : 0u;
        const uint32_t o = active ? off[x] : 0u;
        const int lo = static_cast<int>(lh & 0xffffu), n = static_cast<int>(lh >> 16) - lo + 1;
        const bool narrow = active && n <= 16;
        if (narrow) {
            uint8_t* dst = base + o;
            for (int j = 0; j < n; ++j) dst[j] = cell_cost(sl, sr, x, lo + j, W, row_def);
        }
        unsigned bw = __ballot_sync(0xffffffffu, active && !narrow);
        while (bw) {
            const int src = __ffs(bw) - 1;
            bw &= bw - 1;
            const int xw = x0 + src;
            const int lo_w = __shfl_sync(0xffffffffu, lo, src);
            const int n_w = __shfl_sync(0xffffffffu, n, src);
            const uint32_t o_w = __shfl_sync(0xffffffffu, o, src);
            // aligned 32-bit words over the window's bytes, one per lane and
            // iteration; only the two end words (shared with the neighbouring
            // windows) are written bytewise
            const bool xdef = row_def && xw >= kCensusRadius && xw < W - kCensusRadius;
            const uint32_t slx = sl[xw];
            const uintptr_t A0 = reinterpret_cast<uintptr_t>(base + o_w);
            const uintptr_t W0 = A0 & ~static_cast<uintptr_t>(3);
            const int head = static_cast<int>(A0 - W0);  // window bytes start inside word 0
            const int nwords = (head + n_w + 3) >> 2;
            for (int wi = lane; wi < nwords; wi += 32) {
                const int j0 = 4 * wi - head;  // window level index of the word's byte 0
                uint32_t word = 0u;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int xr = xw - (lo_w + j0 + k);
                    const bool ok = xdef && xr >= kCensusRadius && xr < W - kCensusRadius;
                    const uint32_t v = ok ? static_cast<uint32_t>(__popc(slx ^ sr[ok ? xr : 0]))
                                          : static_cast<uint32_t>(kMaxCost);
                    word |= v << (8 * k);
                }
                uint8_t* wp = reinterpret_cast<uint8_t*>(W0) + 4 * wi;
                if (j0 >= 0 && j0 + 4 <= n_w) {
                    *reinterpret_cast<uint32_t*>(wp) = word;
                } else {
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if (j0 + k >= 0 && j0 + k < n_w) wp[k] = static_cast<uint8_t>(word >> (8 * k));
                }
            }
        }
    }
}

// The aggregation's cost input (build_cost_volume,
// matching_cost.cpp:88-117) in the QUAD layout of the path-cost partials:
// pixel i's levels 4*(lo/4) .. 4*(hi/4)+3 as u32 words at qoff[i], levels
// outside [lo, hi] as 0xff (valid costs are <= 24), so the scan reads aligned
// words and poisons out-of-window levels from the byte itself. The
// reference's ragged layout (cost_kernel) is produced only where a caller
// asks for it (tsgm_fetch COST, build_cost_volume, the fallback aggregation).
// One CTA per (row, position); census rows staged in shared memory; a window
// of <= 4 quads is written by its own lane, wider ones by the warp (lanes
// across quads, coalesced 32-bit stores).
// Costs of levels d0 .. d0+3 at pixel x (24 where a census pixel is undefined).
__device__ __forceinline__ uint32_t quad_raw(uint32_t slx, const uint32_t* sr, int x, int d0, int W,
                                             bool xdef) {
    if (xdef && x - d0 - 3 >= kCensusRadius && x - d0 < W - kCensusRadius) {
        // both census pixels defined for all four levels (all but the image
        // borders): four popcounts packed by IMAD
        const uint32_t* r = sr + (x - d0 - 3);  // levels d0+3 .. d0 at r[0..3]
        const uint32_t c3 = __popc(slx ^ r[0]), c2 = __popc(slx ^ r[1]);
        const uint32_t c1 = __popc(slx ^ r[2]), c0 = __popc(slx ^ r[3]);
        return c0 + (c1 << 8) + (c2 << 16) + (c3 << 24);
    }
    uint32_t word = 0u;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int xr = x - d0 - u;
        const bool ok = xdef && xr >= kCensusRadius && xr < W - kCensusRadius;
        const uint32_t c = ok ? static_cast<uint32_t>(__popc(slx ^ sr[ok ? xr : 0]))
                              : static_cast<uint32_t>(kMaxCost);
        word |= c << (8 * u);
    }
    return word;
}

// Pad bytes (0xff) of the levels d0 .. d0+3 outside [lo, hi]: only a window's
// first and last quads have any.
__device__ __forceinline__ uint32_t quad_pad(int d0, int lo, int hi) {
    const int lr = min(max(lo - d0, 0), 4), hr = min(max(hi - d0 + 1, 0), 4);
    return ~(__funnelshift_lc(0u, 0xffffffffu, 8 * lr) & ~__funnelshift_lc(0u, 0xffffffffu, 8 * hr));
}

__global__ void __launch_bounds__(256) cost_quad_kernel(Bufs b) {
    extern __shared__ uint32_t sm[];
    const int a = blockIdx.y, s = slot_of(b, a), y = blockIdx.x;
    const int W = b.W;
    uint32_t* sl = sm;
    uint32_t* sr = sl + W;
    const size_t pbase = static_cast<size_t>(s) * b.P + static_cast<size_t>(y) * W;
    const uint32_t* qoff = b.qoff + static_cast<size_t>(s) * (b.P + 1) + static_cast<size_t>(y) * W;
    for (int x = threadIdx.x; x < W; x += blockDim.x) {
        sl[x] = b.sigl[pbase + x];
        sr[x] = b.sigr[pbase + x];
    }
    __syncthreads();
    uint32_t* cq = b.costq + b.vqbase[a];
    const bool row_def = y >= kCensusRadius && y < b.H - kCensusRadius;
    const int warp = static_cast<int>(threadIdx.x >> 5), lane = static_cast<int>(threadIdx.x & 31);
    const int nwarps = static_cast<int>(blockDim.x >> 5);
    for (int x0 = warp * 32; x0 < W; x0 += 32 * nwarps) {
        const int x = x0 + lane;
        const bool active = x < W;
        const uint32_t lh = active ? __ldg(b.lohi + pbase + x) : 0u;
        const uint32_t qo = active ? __ldg(qoff + x) : 0u;
        const int lo = static_cast<int>(lh & 0xffffu), hi = static_cast<int>(lh >> 16);
        const int q0 = lo >> 2, nq = (hi >> 2) - q0 + 1;
        const bool xdef = row_def && x >= kCensusRadius && x < W - kCensusRadius;
        const bool narrow = active && nq <= 4;
        if (narrow) {
            const uint32_t slx = sl[x];
            for (int t = 0; t < nq; ++t) {
                const int d0 = 4 * (q0 + t);
                const uint32_t w = quad_raw(slx, sr, x, d0, W, xdef);
                cq[qo + t] = (t == 0 || t == nq - 1) ? w | quad_pad(d0, lo, hi) : w;
            }
        }
        unsigned bw = __ballot_sync(0xffffffffu, active && !narrow);
        while (bw) {
            const int src = __ffs(bw) - 1;
            bw &= bw - 1;
            const int xw = x0 + src;
            const int lo_w = __shfl_sync(0xffffffffu, lo, src);
            const int hi_w = __shfl_sync(0xffffffffu, hi, src);
            const uint32_t qo_w = __shfl_sync(0xffffffffu, qo, src);
            const bool xdef_w = __shfl_sync(0xffffffffu, xdef, src);
            const int q0w = lo_w >> 2, nqw = (hi_w >> 2) - q0w + 1;
            const uint32_t slx = sl[xw];
            for (int t = lane; t < nqw; t += 32) {
                const int d0 = 4 * (q0w + t);
                const uint32_t w = quad_raw(slx, sr, xw, d0, W, xdef_w);
                cq[qo_w + t] = (t == 0 || t == nqw - 1) ? w | quad_pad(d0, lo_w, hi_w) : w;
            }
        }
    }
}

// Ragged (reference layout) -> quad layout, for a caller-provided cost volume
// (tsgm_aggregate_paths). One thread per pixel.
__global__ void quads_from_ragged_kernel(Bufs b) {
    const int a = blockIdx.y, s = slot_of(b, a);
    const uint8_t* cost = b.cost + b.vbase[a];
    uint32_t* cq = b.costq + b.vqbase[a];
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < b.P; i += gridDim.x * blockDim.x) {
        const uint32_t lh = b.lohi[static_cast<size_t>(s) * b.P + i];
        const int lo = static_cast<int>(lh & 0xffffu), hi = static_cast<int>(lh >> 16);
        const uint32_t o = b.off[static_cast<size_t>(s) * (b.P + 1) + i];
        const uint32_t qo = b.qoff[static_cast<size_t>(s) * (b.P + 1) + i];
        const int q0 = lo >> 2, nq = (hi >> 2) - q0 + 1;
        for (int t = 0; t < nq; ++t) {
            uint32_t word = 0u;
            for (int u = 0; u < 4; ++u) {
                const int d = 4 * (q0 + t) + u;
                word |= (d >= lo && d <= hi ? static_cast<uint32_t>(cost[o + (d - lo)]) : 0xffu) << (8 * u);
            }
            cq[qo + t] = word;
        }
    }
}

// Volume plan of a chunk of m positions: position a
// starts at the prefix of the chunk's ACTUAL cell and quad counts (the N of
// make_cost_volume, matching_cost.cpp:30-48), rounded up to 16 cells / 4
// quads, instead of a worst-case P*d_max stride. One warp, u64 warp scans.
__global__ void volume_plan_kernel(Bufs b, int m, unsigned long long* vb) {
    const int lane = static_cast<int>(threadIdx.x);
    unsigned long long cc = 0, cq = 0;  // carries
    for (int a0 = 0; a0 < m; a0 += 32) {
        const int a = a0 + lane;
        unsigned long long c = 0, q = 0;
        if (a < m) {
            const int s = b.slots[a];
            c = (b.ncells[s] + 15ull) & ~15ull;
            q = (b.nquads[s] + 3ull) & ~3ull;
        }
        unsigned long long ic = c, iq = q;  // inclusive scans
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long tc = __shfl_up_sync(0xffffffffu, ic, o);
            const unsigned long long tq = __shfl_up_sync(0xffffffffu, iq, o);
            if (lane >= o) {
                ic += tc;
                iq += tq;
            }
        }
        if (a < m) {
            vb[a] = cc + ic - c;
            vb[b.max_slots + a] = cq + iq - q;
        }
        cc += __shfl_sync(0xffffffffu, ic, 31);
        cq += __shfl_sync(0xffffffffu, iq, 31);
    }
}

void launch_volume_plan(const Bufs& b, int m, Launch L) {
    volume_plan_kernel<<<1, 32, 0, L.st>>>(b, m, const_cast<unsigned long long*>(b.vbase));
    ++*L.counter;
}

void launch_cost(const Bufs& b, int n, Launch L) {
    const size_t smem = sizeof(uint32_t) * 2 * b.W;
    cost_quad_kernel<<<dim3(b.H, n), 256, smem, L.st>>>(b);
    ++*L.counter;
}

void launch_cost_ragged(const Bufs& b, int n, Launch L) {
    const size_t smem = sizeof(uint32_t) * 2 * b.W;
    cost_kernel<<<dim3(b.H, n), 512, smem, L.st>>>(b);
    ++*L.counter;
}

void launch_cost_quads_from_ragged(const Bufs& b, int n, Launch L) {
    quads_from_ragged_kernel<<<dim3((b.P + 255) / 256 < 1024 ? (b.P + 255) / 256 : 1024, n), 256, 0, L.st>>>(b);
    ++*L.counter;
}

// ---------------------------------------------------------------- WTA (A15)
// winner_takes_all, sgm.cpp:163-187: first minimum of S over the window,
// 2-px census border invalid. One warp per pixel group: lanes stride the
// window, then a (value, index) warp argmin keeps the first minimum.
__global__ void wta_kernel(Bufs b) {
    const int a = blockIdx.y, s = slot_of(b, a);
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    const uint32_t* off = b.off + static_cast<size_t>(s) * (b.P + 1);
    const uint16_t* agg = b.agg + b.vbase[a];
    for (int i = warp; i < b.P; i += nwarps) {
        const int x = i % b.W, y = i / b.W;
        const size_t pi = static_cast<size_t>(s) * b.P + i;
        if (!census_defined(x, y, b.W, b.H)) {
            if (lane == 0) {
                b.md[pi] = 0;
                b.mv[pi] = 0;
            }
            continue;
        }
        const uint32_t o0 = off[i], n = off[i + 1] - o0;
        uint32_t best = 0xffffffffu;  // (value << 16) | index: min keeps first index
        for (uint32_t j = lane; j < n; j += 32) {
            const uint32_t key = (static_cast<uint32_t>(agg[o0 + j]) << 16) | j;
            best = min(best, key);
        }
        best = __reduce_min_sync(0xffffffffu, best);
        if (lane == 0) {
            b.md[pi] = static_cast<int32_t>(b.lo[pi]) + static_cast<int32_t>(best & 0xffffu);
            b.mv[pi] = 1;
        }
    }
}

void launch_wta(const Bufs& b, int n, Launch L) {
    const int blocks = (b.P + 7) / 8 < 2048 ? (b.P + 7) / 8 : 2048;
    wta_kernel<<<dim3(blocks, n), 256, 0, L.st>>>(b);
    ++*L.counter;
}

// ---------------------------------------------------------------- median (A19)
// median_refine, sgm.cpp:189-216: lower median of the valid 3x3 neighbours,
// valid iff at least 5. One thread per pixel of a 32x8 tile; keys (d, or
// INT32_MAX for an invalid or missing neighbour) and validity staged in shared
// memory with a 1-px halo. Invalid keys sort after every valid value (ties
// with a valid INT32_MAX leave the k-th smallest unchanged), so element
// (n-1)/2 of the sorted 9 is the lower median of the n valid ones.
constexpr int kMdW = 32, kMdH = 8;

__device__ __forceinline__ void cswap(int32_t& a, int32_t& b) {
    const int32_t lo = min(a, b), hi = max(a, b);
    a = lo;
    b = hi;
}

__global__ void median_kernel(Bufs b, const int32_t* in_d, const uint8_t* in_v, int32_t* out_d,
                              uint8_t* out_v) {
    __shared__ int32_t key[kMdH + 2][kMdW + 2];
    __shared__ uint8_t ok[kMdH + 2][kMdW + 2];
    const int a = blockIdx.z, s = slot_of(b, a);
    const size_t base = static_cast<size_t>(s) * b.P;
    const int x0 = blockIdx.x * kMdW - 1, y0 = blockIdx.y * kMdH - 1;
    for (int t = threadIdx.y * kMdW + threadIdx.x; t < (kMdH + 2) * (kMdW + 2); t += kMdW * kMdH) {
        const int ty = t / (kMdW + 2), tx = t % (kMdW + 2);
        const int gx = x0 + tx, gy = y0 + ty;
        const bool in = gx >= 0 && gx < b.W && gy >= 0 && gy < b.H;
        const size_t j = base + static_cast<size_t>(in ? gy : 0) * b.W + (in ? gx : 0);
        const bool v = in && in_v[j];
        key[ty][tx] = v ? in_d[j] : INT32_MAX;
        ok[ty][tx] = v ? 1 : 0;
    }
    __syncthreads();
    const int x = blockIdx.x * kMdW + threadIdx.x, y = blockIdx.y * kMdH + threadIdx.y;
    if (x >= b.W || y >= b.H) return;
    int32_t v[9];
    int n = 0;
#pragma unroll
    for (int dy = 0; dy < 3; ++dy)
#pragma unroll
        for (int dx = 0; dx < 3; ++dx) {
            v[dy * 3 + dx] = key[threadIdx.y + dy][threadIdx.x + dx];
            n += ok[threadIdx.y + dy][threadIdx.x + dx];
        }
    const size_t i = base + static_cast<size_t>(y) * b.W + x;
    if (n < 5) {
        out_d[i] = 0;
        out_v[i] = 0;
        return;
    }
    // 9-element sorting network (25 compare-exchanges; the ones that cannot
    // reach elements 2..4 are dead code)
    cswap(v[0], v[3]); cswap(v[1], v[7]); cswap(v[2], v[5]); cswap(v[4], v[8]);
    cswap(v[0], v[7]); cswap(v[2], v[4]); cswap(v[3], v[8]); cswap(v[5], v[6]);
    cswap(v[0], v[2]); cswap(v[1], v[3]); cswap(v[4], v[5]); cswap(v[7], v[8]);
    cswap(v[1], v[4]); cswap(v[3], v[6]); cswap(v[5], v[7]);
    cswap(v[0], v[1]); cswap(v[2], v[4]); cswap(v[3], v[5]); cswap(v[6], v[8]);
    cswap(v[2], v[3]); cswap(v[4], v[5]); cswap(v[6], v[7]);
    cswap(v[1], v[2]); cswap(v[3], v[4]); cswap(v[5], v[6]);
    const int k = (n - 1) / 2;  // 2, 3 or 4
    out_d[i] = k == 2 ? v[2] : (k == 3 ? v[3] : v[4]);
    out_v[i] = 1;
}

void launch_median(const Bufs& b, int n, const int32_t* in_d, const uint8_t* in_v,
                   int32_t* out_d, uint8_t* out_v, Launch L) {
    dim3 grid((b.W + kMdW - 1) / kMdW, (b.H + kMdH - 1) / kMdH, n);
    median_kernel<<<grid, dim3(kMdW, kMdH), 0, L.st>>>(b, in_d, in_v, out_d, out_v);
    ++*L.counter;
}

}  // namespace tsgm
