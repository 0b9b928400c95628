// Moving-object box detector on the diff map (
// reference src/motion_detect.cpp). GPU: the summed-area table and the
// candidate-window scoring with an order-preserving compaction; host: the
// greedy merge, exact but incremental.
//
// Exactness. integral_image (motion_detect.cpp:25-42) accumulates each row
// left to right (row_acc += v) and adds the row above: S[y+1][x+1] =
// S[y][x+1] + R_y[x]. The GPU computes R_y[x] with the same sequential row
// order (one thread per row over shared-memory tiles), then walks each column
// top to bottom (one thread per column), which is the same two-operand FP64
// sum per element. box_sum evaluates ((a - b) - c) + d like :48-49, the mean
// divides by the area as a double like :85, and candidates are emitted in
// (window size, row, column) order like :89-96.
#include <algorithm>
#include <cstring>
#include <thread>
#include <vector>

#include "common.cuh"

namespace tsgm {

// ---------------------------------------------------------------- SAT
// Row pass: one warp per 32 rows; tiles of 32x32 staged in shared memory so
// the loads and stores are coalesced while each lane accumulates its own row
// in order. Writes R_y[x] into S[y+1][x+1].
__global__ void sat_rows_kernel(const double* __restrict__ map, size_t map_stride,
                                double* __restrict__ sat, size_t sat_stride, int W, int H,
                                const int* slots) {
    __shared__ double tile[32][33];
    const int a = blockIdx.y, s = slots ? slots[a] : a;
    const double* m = map + static_cast<size_t>(s) * map_stride;
    double* S = sat + static_cast<size_t>(a) * sat_stride;
    const int lane = threadIdx.x, y0 = blockIdx.x * 32;
    const size_t SW = static_cast<size_t>(W) + 1;
    double acc = 0.0;
    for (int x0 = 0; x0 < W; x0 += 32) {
        for (int r = 0; r < 32; ++r) {
            const int y = y0 + r, x = x0 + lane;
            tile[r][lane] = (y < H && x < W) ? m[static_cast<size_t>(y) * W + x] : 0.0;
        }
        __syncwarp();
        const int n = min(32, W - x0);
        for (int c = 0; c < n; ++c) {  // lane = row: sequential along the row
            acc = __dadd_rn(acc, tile[lane][c]);
            tile[lane][c] = acc;
        }
        __syncwarp();
        for (int r = 0; r < 32; ++r) {
            const int y = y0 + r, x = x0 + lane;
            if (y < H && x < W) S[static_cast<size_t>(y + 1) * SW + x + 1] = tile[r][lane];
        }
        __syncwarp();
    }
}

// Column pass: S[y+1][x+1] = S[y][x+1] + R_y[x], top to bottom; also the zero
// first row and column.
__global__ void sat_cols_kernel(double* __restrict__ sat, size_t sat_stride, int W, int H) {
    const int a = blockIdx.y;
    double* S = sat + static_cast<size_t>(a) * sat_stride;
    const size_t SW = static_cast<size_t>(W) + 1;
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x > W) return;
    S[x] = 0.0;
    if (x == 0) {
        for (int y = 1; y <= H; ++y) S[static_cast<size_t>(y) * SW] = 0.0;
        return;
    }
    double above = 0.0;
    for (int y = 1; y <= H; ++y) {
        double* p = S + static_cast<size_t>(y) * SW + x;
        above = __dadd_rn(above, *p);
        *p = above;
    }
}

// ---------------------------------------------------------------- candidates

__device__ __forceinline__ bool window_at(const double* S, size_t SW, const DetectWindows& dw,
                                          long long pos, tsgm_box& box) {
    int k = 0;
    while (pos >= dw.base[k + 1]) ++k;
    const long long r = pos - dw.base[k];
    const int row = static_cast<int>(r / dw.cols[k]), col = static_cast<int>(r % dw.cols[k]);
    const int sx = max(1, dw.ww[k] / 4), sy = max(1, dw.wh[k] / 4);
    const int x0 = col * sx, y0 = dw.region_top + row * sy;
    const int x1 = x0 + dw.ww[k], y1 = y0 + dw.wh[k];
    const double sum = __dadd_rn(__dsub_rn(__dsub_rn(S[static_cast<size_t>(y1) * SW + x1],
                                                     S[static_cast<size_t>(y0) * SW + x1]),
                                           S[static_cast<size_t>(y1) * SW + x0]),
                                 S[static_cast<size_t>(y0) * SW + x0]);
    const double area = static_cast<double>(static_cast<long long>(x1 - x0) * (y1 - y0));
    const double mean = sum / area;
    box = tsgm_box{x0, y0, x1, y1, mean};
    return mean > dw.thresh;
}

constexpr int kCandThreads = 1024;

// One CTA per sequence: each thread scores a contiguous run of positions,
// a block scan turns the counts into output offsets, and the run is scored
// again and written in order.
__global__ void __launch_bounds__(kCandThreads) candidates_kernel(const double* __restrict__ sat,
                                                                  size_t sat_stride, int W,
                                                                  DetectWindows dw,
                                                                  tsgm_box* out, long long cap,
                                                                  long long* counts) {
    __shared__ long long part[kCandThreads / 32];
    const int a = blockIdx.x;
    const double* S = sat + static_cast<size_t>(a) * sat_stride;
    const size_t SW = static_cast<size_t>(W) + 1;
    const long long total = dw.base[dw.n];
    const long long per = (total + kCandThreads - 1) / kCandThreads;
    const long long p0 = min(total, per * threadIdx.x), p1 = min(total, p0 + per);
    long long cnt = 0;
    tsgm_box bx;
    for (long long p = p0; p < p1; ++p) cnt += window_at(S, SW, dw, p, bx) ? 1 : 0;
    // block exclusive scan of cnt
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    long long v = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const long long t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    if (lane == 31) part[wid] = v;
    __syncthreads();
    if (wid == 0) {
        long long w = part[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long t = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += t;
        }
        part[lane] = w;
    }
    __syncthreads();
    long long at = v - cnt + (wid > 0 ? part[wid - 1] : 0);
    if (threadIdx.x == kCandThreads - 1) counts[a] = at + cnt;
    tsgm_box* o = out + static_cast<size_t>(a) * cap;
    for (long long p = p0; p < p1 && cnt > 0; ++p)
        if (window_at(S, SW, dw, p, bx)) {
            if (at < cap) o[at] = bx;
            ++at;
        }
}

// ---------------------------------------------------------------- host side
namespace {

long long area_of(const tsgm_box& b) { return static_cast<long long>(b.x1 - b.x0) * (b.y1 - b.y0); }

// iou, motion_detect.cpp:52-62
double iou_of(const tsgm_box& a, const tsgm_box& b) {
    const int ix0 = std::max(a.x0, b.x0), iy0 = std::max(a.y0, b.y0);
    const int ix1 = std::min(a.x1, b.x1), iy1 = std::min(a.y1, b.y1);
    if (ix0 >= ix1 || iy0 >= iy1) return 0.0;
    const double inter = static_cast<double>(ix1 - ix0) * (iy1 - iy0);
    const double uni = static_cast<double>(area_of(a)) + static_cast<double>(area_of(b)) - inter;
    return inter / uni;
}

}  // namespace

void detect_windows(const tsgm_detect_config& c, int W, int H, DetectWindows& dw) {
    dw = DetectWindows{};
    dw.region_top = H / 3;  // motion_detect.cpp:69
    dw.thresh = c.score_thresh;
    dw.base[0] = 0;
    for (int i = 0; i < c.n_windows; ++i) {
        const int ww = c.window_wh[2 * i], wh = c.window_wh[2 * i + 1];
        if (ww > W || dw.region_top + wh > H) continue;  // :73-74
        const int sx = std::max(1, ww / 4), sy = std::max(1, wh / 4);
        dw.ww[dw.n] = ww;
        dw.wh[dw.n] = wh;
        dw.rows[dw.n] = (H - wh - dw.region_top) / sy + 1;
        dw.cols[dw.n] = (W - ww) / sx + 1;
        dw.base[dw.n + 1] = dw.base[dw.n] + static_cast<long long>(dw.rows[dw.n]) * dw.cols[dw.n];
        ++dw.n;
    }
    for (int k = dw.n + 1; k <= kMaxDetectWindows; ++k) dw.base[k] = dw.base[dw.n];
}

void launch_sat(const double* map, size_t map_stride, double* sat, size_t sat_stride, int W, int H,
                int n, const int* slots, Launch L) {
    sat_rows_kernel<<<dim3((H + 31) / 32, n), 32, 0, L.st>>>(map, map_stride, sat, sat_stride, W, H,
                                                             slots);
    sat_cols_kernel<<<dim3((W + 1 + 255) / 256, n), 256, 0, L.st>>>(sat, sat_stride, W, H);
    *L.counter += 2;
}

void launch_candidates(const double* sat, size_t sat_stride, int W, const DetectWindows& dw, int n,
                       tsgm_box* out, long long cap, long long* counts, Launch L) {
    candidates_kernel<<<n, kCandThreads, 0, L.st>>>(sat, sat_stride, W, dw, out, cap, counts);
    ++*L.counter;
}

// greedy_merge (motion_detect.cpp:101-129), exact and incremental. The
// reference rescans all pairs per merge and takes the first pair (in list
// order) of maximal IoU > 0. Here every live row i keeps its best (value,
// first j) over live j > i; the global choice is the first row of maximal
// value, i.e. the same pair. A merge changes box bi and removes bj, so only
// row bi, rows whose best was bi or bj, and the entries (k, bi) of earlier
// rows can change; list order of the survivors is untouched by erase().
long long greedy_merge_host(tsgm_box* boxes, long long n, const tsgm_detect_config& c) {
    std::vector<char> alive(static_cast<size_t>(n), 1);
    std::vector<double> bv(static_cast<size_t>(n), 0.0);
    std::vector<long long> bj(static_cast<size_t>(n), -1);
    auto recompute = [&](long long i) {
        double best = 0.0;
        long long j_best = -1;
        for (long long j = i + 1; j < n; ++j)
            if (alive[j]) {
                const double v = iou_of(boxes[i], boxes[j]);
                if (v > best) {
                    best = v;
                    j_best = j;
                }
            }
        bv[i] = best;
        bj[i] = j_best;
    };
    for (long long i = 0; i < n; ++i) recompute(i);
    long long live = n;
    while (live > 1) {
        double best = 0.0;
        long long bi = -1;
        for (long long i = 0; i < n; ++i)
            if (alive[i] && bv[i] > best) {
                best = bv[i];
                bi = i;
            }
        if (bi < 0 || best < c.merge_stop_iou) break;  // best = 0 with no pair also stops
        const long long j = bj[bi];
        tsgm_box& a = boxes[bi];
        const tsgm_box& b = boxes[j];
        const double aa = static_cast<double>(area_of(a)), ab = static_cast<double>(area_of(b));
        a.score = (a.score * aa + b.score * ab) / (aa + ab);
        a.x0 = std::min(a.x0, b.x0);
        a.y0 = std::min(a.y0, b.y0);
        a.x1 = std::max(a.x1, b.x1);
        a.y1 = std::max(a.y1, b.y1);
        alive[j] = 0;
        --live;
        for (long long k = 0; k < n; ++k) {
            if (!alive[k] || k == bi) continue;
            if (bj[k] == j || bj[k] == bi) {
                recompute(k);
            } else if (k < bi) {
                const double v = iou_of(boxes[k], a);
                if (v > bv[k] || (v == bv[k] && v > 0.0 && bi < bj[k])) {
                    bv[k] = v;
                    bj[k] = bi;
                }
            }
        }
        recompute(bi);
    }
    long long m = 0;
    for (long long i = 0; i < n; ++i)
        if (alive[i] && area_of(boxes[i]) >= c.min_box_area) boxes[m++] = boxes[i];
    return m;
}

}  // namespace tsgm
