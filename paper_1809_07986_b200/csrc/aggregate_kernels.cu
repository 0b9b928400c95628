// Semi-global path aggregation over ragged per-pixel disparity windows
// (aggregate_paths, sgm.cpp:39-161).
//
// Per direction r with predecessor q = p + (dx, dy):
//   L_r(p, d) = C(p, d)                                   at the image edge
//   L_r(p, d) = C(p, d) + min(Lq(d), Lq(d+-1) + P1, min_q + P2) - min_q
// over the levels the predecessor's window holds (sgm.cpp:93-126). S is the
// u16 sum over the 4 or 8 directions; u16 never overflows (SgmParams::validate
// bounds (24 + P2) * paths, sgm.cpp:21-22) so direction order is irrelevant.
#include "common.cuh"

namespace tsgm {

// ---------------------------------------------------------------- v1: scanline warps
// One warp per scanline, lanes across the pixel's disparity window; the
// predecessor's path costs live in a per-warp shared buffer, min via
// __reduce_min_sync. One launch per direction, S accumulated in place.
constexpr int kAggWarps = 4;

__device__ __forceinline__ int num_lines(int W, int H, int dx, int dy) {
    if (dy == 0) return H;
    if (dx == 0) return W;
    return W + H - 1;
}

__device__ __forceinline__ void line_start(int line, int W, int H, int dx, int dy, int& x, int& y) {
    if (dy == 0) {
        y = line;
        x = dx < 0 ? 0 : W - 1;
    } else if (dx == 0) {
        x = line;
        y = dy < 0 ? 0 : H - 1;
    } else if (line < W) {
        x = line;
        y = dy < 0 ? 0 : H - 1;
    } else {
        const int k = line - W + 1;
        x = dx < 0 ? 0 : W - 1;
        y = dy < 0 ? k : H - 1 - k;
    }
}

__global__ void __launch_bounds__(32 * kAggWarps)
aggregate_dir_kernel(Bufs b, int dx, int dy, int p1, int p2, int first) {
    extern __shared__ uint16_t lbuf[];  // [warps][2][d_max]
    const int a = blockIdx.y, s = slot_of(b, a);
    const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int line = blockIdx.x * kAggWarps + wib;
    const int W = b.W, H = b.H;
    if (line >= num_lines(W, H, dx, dy)) return;
    uint16_t* bufA = lbuf + static_cast<size_t>(wib) * 2 * b.d_max;
    uint16_t* bufB = bufA + b.d_max;
    const uint32_t* off = b.off + static_cast<size_t>(s) * (b.P + 1);
    const uint16_t* lo = b.lo + static_cast<size_t>(s) * b.P;
    const uint8_t* cost = b.cost + b.vbase[a];
    uint16_t* agg = b.agg + b.vbase[a];

    int x, y;
    line_start(line, W, H, dx, dy, x, y);
    int q_lo = 0, q_n = 0, q_min = 0;
    bool edge = true;
    uint16_t* lq = bufA;
    uint16_t* lc = bufB;
    while (x >= 0 && x < W && y >= 0 && y < H) {
        const int i = y * W + x;
        const uint32_t o = off[i];
        const int n = static_cast<int>(off[i + 1] - o);
        const int lo_i = lo[i];
        int mn = 0x7fffffff;
        if (edge) {
            for (int j = lane; j < n; j += 32) {
                const int l = cost[o + j];
                lc[j] = static_cast<uint16_t>(l);
                agg[o + j] = static_cast<uint16_t>((first ? 0 : agg[o + j]) + l);
                mn = min(mn, l);
            }
        } else {
            const int shift = lo_i - q_lo;
            const int cap = q_min + p2;
            for (int j = lane; j < n; j += 32) {
                const int k = j + shift;
                int best = cap;
                if (k >= 0 && k < q_n) best = min(best, static_cast<int>(lq[k]));
                if (k - 1 >= 0 && k - 1 < q_n) best = min(best, lq[k - 1] + p1);
                if (k + 1 >= 0 && k + 1 < q_n) best = min(best, lq[k + 1] + p1);
                const int l = cost[o + j] + best - q_min;
                lc[j] = static_cast<uint16_t>(l);
                agg[o + j] = static_cast<uint16_t>((first ? 0 : agg[o + j]) + l);
                mn = min(mn, l);
            }
        }
        q_min = static_cast<int>(__reduce_min_sync(0xffffffffu, static_cast<unsigned>(mn)));
        __syncwarp();
        q_lo = lo_i;
        q_n = n;
        edge = false;
        uint16_t* t = lq;
        lq = lc;
        lc = t;
        x -= dx;
        y -= dy;
    }
}

void launch_aggregate(const Bufs& b, int n, int p1, int p2, int paths, int path_set, Launch L) {
    static const int nondiag[4][2] = {{-1, 0}, {0, -1}, {1, 0}, {0, 1}};
    static const int diag[4][2] = {{-1, -1}, {1, -1}, {1, 1}, {-1, 1}};
    const size_t smem = sizeof(uint16_t) * 2 * b.d_max * kAggWarps;
    int first = 1;
    for (int set = 0; set < 2; ++set) {
        const bool use = paths == 8 || path_set == set;
        if (!use) continue;
        for (int k = 0; k < 4; ++k) {
            const int dx = set == 0 ? nondiag[k][0] : diag[k][0];
            const int dy = set == 0 ? nondiag[k][1] : diag[k][1];
            const int lines = dy == 0 ? b.H : (dx == 0 ? b.W : b.W + b.H - 1);
            aggregate_dir_kernel<<<dim3((lines + kAggWarps - 1) / kAggWarps, n), 32 * kAggWarps,
                                   smem, L.st>>>(b, dx, dy, p1, p2, first);
            ++*L.counter;
            first = 0;
        }
    }
}

}  // namespace tsgm
