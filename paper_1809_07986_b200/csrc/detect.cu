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


// IoU as the exact fraction inter / union (both integers, union < 2^53): the
// reference's double division rounds it correctly, and distinct fractions with
// denominators below 2^26 differ by more than an ulp, so comparing fractions
// by cross-multiplication orders (and ties) pairs exactly like comparing the
// reference's doubles. Only a row's winner is divided.
struct Frac {
    long long num = 0, den = 1;
};
Frac iou_frac(const tsgm_box& a, const tsgm_box& b) {
    const int ix0 = std::max(a.x0, b.x0), iy0 = std::max(a.y0, b.y0);
    const int ix1 = std::min(a.x1, b.x1), iy1 = std::min(a.y1, b.y1);
    if (ix0 >= ix1 || iy0 >= iy1) return Frac{};
    const long long inter = static_cast<long long>(ix1 - ix0) * (iy1 - iy0);
    return Frac{inter, area_of(a) + area_of(b) - inter};
}
int frac_cmp(const Frac& a, const Frac& b) {
    const __int128 l = static_cast<__int128>(a.num) * b.den, r = static_cast<__int128>(b.num) * a.den;
    return l < r ? -1 : (l > r ? 1 : 0);
}
double frac_value(const Frac& f) {  // = iou(), motion_detect.cpp:52-62, in double
    return f.num ? static_cast<double>(f.num) / static_cast<double>(f.den) : 0.0;
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
// value (a segment tree over rows), i.e. the same pair. Only overlapping boxes
// can have IoU > 0, so each row scans a neighbour list (built with a uniform
// grid and extended when a merged box grows). A merge changes box bi and
// removes bj: rows whose partner was bi or bj are rescanned, earlier rows
// overlapping the new bi compare against it, and row bi is rescanned; list
// order of the survivors is untouched by erase().
namespace {

bool overlaps(const tsgm_box& a, const tsgm_box& b) {
    return std::max(a.x0, b.x0) < std::min(a.x1, b.x1) && std::max(a.y0, b.y0) < std::min(a.y1, b.y1);
}

struct BestTree {  // max value, then smallest row index
    int n = 1;
    std::vector<double> v;
    std::vector<int> id;
    explicit BestTree(int rows) {
        while (n < rows) n <<= 1;
        v.assign(2 * n, -1.0);
        id.assign(2 * n, -1);
    }
    void set(int i, double val) {
        int k = i + n;
        v[k] = val;
        id[k] = val > 0.0 ? i : -1;
        for (k >>= 1; k >= 1; k >>= 1) {
            const int l = 2 * k, r = 2 * k + 1;
            const bool left = v[l] >= v[r];  // ties: the left (smaller index) wins
            v[k] = left ? v[l] : v[r];
            id[k] = left ? id[l] : id[r];
        }
    }
};

}  // namespace

long long greedy_merge_host(tsgm_box* boxes, long long n_ll, const tsgm_detect_config& c) {
    const int n = static_cast<int>(n_ll);
    if (n <= 1) {
        long long m = 0;
        for (int i = 0; i < n; ++i)
            if (area_of(boxes[i]) >= c.min_box_area) boxes[m++] = boxes[i];
        return m;
    }
    // uniform grid over the boxes' extent for the neighbour lists
    int gx0 = boxes[0].x0, gy0 = boxes[0].y0, gx1 = boxes[0].x1, gy1 = boxes[0].y1;
    for (int i = 1; i < n; ++i) {
        gx0 = std::min(gx0, boxes[i].x0);
        gy0 = std::min(gy0, boxes[i].y0);
        gx1 = std::max(gx1, boxes[i].x1);
        gy1 = std::max(gy1, boxes[i].y1);
    }
    const int cell = 32;
    const int gw = (gx1 - gx0) / cell + 1, gh = (gy1 - gy0) / cell + 1;
    std::vector<std::vector<int>> grid(static_cast<size_t>(gw) * gh);
    auto cells = [&](const tsgm_box& b, auto&& fn) {
        const int cx0 = (b.x0 - gx0) / cell, cx1 = (std::max(b.x1 - 1, b.x0) - gx0) / cell;
        const int cy0 = (b.y0 - gy0) / cell, cy1 = (std::max(b.y1 - 1, b.y0) - gy0) / cell;
        for (int cy = std::max(0, cy0); cy <= std::min(gh - 1, cy1); ++cy)
            for (int cx = std::max(0, cx0); cx <= std::min(gw - 1, cx1); ++cx) fn(cy * gw + cx);
    };
    for (int i = 0; i < n; ++i) cells(boxes[i], [&](int g) { grid[g].push_back(i); });
    std::vector<char> alive(n, 1);
    std::vector<int> stamp(n, -1);
    int now = 0;
    auto cell_inside = [&](int g, const tsgm_box& b) {  // cell g entirely within box b
        const int cx = g % gw, cy = g / gw;
        const int x0 = gx0 + cx * cell, y0 = gy0 + cy * cell;
        return b.x0 <= x0 && x0 + cell <= b.x1 && b.y0 <= y0 && y0 + cell <= b.y1;
    };
    // adjacency: every overlapping pair once (lists hold live overlapping boxes)
    std::vector<std::vector<int>> adj(n);
    for (int i = 0; i < n; ++i) {
        ++now;
        cells(boxes[i], [&](int g) {
            for (int j : grid[g])
                if (j > i && stamp[j] != now) {
                    stamp[j] = now;
                    if (overlaps(boxes[i], boxes[j])) {
                        adj[i].push_back(j);
                        adj[j].push_back(i);
                    }
                }
        });
    }
    // live boxes overlapping the merged box `self` (grown from old_a and
    // old_b): the parts' neighbours, plus a grid scan of the cells not inside
    // either part (a box meeting a cell inside a part overlaps that part, so
    // it is already in the part's list)
    auto merged_neighbours = [&](int self, int other, const tsgm_box& old_a, const tsgm_box& old_b,
                                 std::vector<int>& out) {
        out.clear();
        ++now;
        stamp[self] = now;
        stamp[other] = now;
        for (const std::vector<int>* l : {&adj[self], &adj[other]})
            for (int j : *l)
                if (alive[j] && stamp[j] != now) {
                    stamp[j] = now;
                    if (overlaps(boxes[self], boxes[j])) out.push_back(j);
                }
        cells(boxes[self], [&](int g) {
            if (cell_inside(g, old_a) || cell_inside(g, old_b)) return;
            std::vector<int>& cl = grid[g];
            size_t w = 0;
            for (size_t t = 0; t < cl.size(); ++t) {
                const int j = cl[t];
                if (!alive[j]) continue;  // drop merged-away boxes from the cell
                cl[w++] = j;
                if (stamp[j] != now) {
                    stamp[j] = now;
                    if (overlaps(boxes[self], boxes[j])) out.push_back(j);
                }
            }
            cl.resize(w);
        });
    };
    std::vector<double> bv(n, 0.0);
    std::vector<Frac> bf(n);
    std::vector<int> bj(n, -1);
    BestTree tree(n);
    auto rescan = [&](int i) {
        Frac best;
        int jb = -1;
        std::vector<int>& a = adj[i];
        size_t w = 0;
        ++now;
        for (size_t t = 0; t < a.size(); ++t) {
            const int j = a[t];
            if (!alive[j] || stamp[j] == now) continue;  // prune dead and duplicate entries
            stamp[j] = now;
            a[w++] = j;
            if (j <= i) continue;
            const Frac v = iou_frac(boxes[i], boxes[j]);
            if (v.num == 0) continue;
            const int cmp = jb < 0 ? 1 : frac_cmp(v, best);
            if (cmp > 0 || (cmp == 0 && j < jb)) {
                best = v;
                jb = j;
            }
        }
        a.resize(w);
        bf[i] = best;
        bv[i] = jb >= 0 ? frac_value(best) : 0.0;
        bj[i] = jb;
        tree.set(i, bv[i]);
    };
    for (int i = 0; i < n; ++i) rescan(i);
    std::vector<int> touched, fresh;
    int live = n;
    while (live > 1) {
        const int bi = tree.id[1];
        if (bi < 0 || tree.v[1] < c.merge_stop_iou) break;  // no pair with IoU > 0 also stops
        const int j = bj[bi];
        tsgm_box& a = boxes[bi];
        const tsgm_box b = boxes[j];
        const tsgm_box old_a = a;
        const double aa = static_cast<double>(area_of(a)), ab = static_cast<double>(area_of(b));
        a.score = (a.score * aa + b.score * ab) / (aa + ab);
        a.x0 = std::min(a.x0, b.x0);
        a.y0 = std::min(a.y0, b.y0);
        a.x1 = std::max(a.x1, b.x1);
        a.y1 = std::max(a.y1, b.y1);
        alive[j] = 0;
        --live;
        tree.set(j, 0.0);
        // rows that may change: neighbours of the old bi / bj and of the new bi
        touched.clear();
        for (int k : adj[bi]) touched.push_back(k);
        for (int k : adj[j]) touched.push_back(k);
        {  // a box only grows: register bi in the cells outside its old extent
            const int ox0 = (old_a.x0 - gx0) / cell, ox1 = (std::max(old_a.x1 - 1, old_a.x0) - gx0) / cell;
            const int oy0 = (old_a.y0 - gy0) / cell, oy1 = (std::max(old_a.y1 - 1, old_a.y0) - gy0) / cell;
            cells(a, [&](int g) {
                const int cx = g % gw, cy = g / gw;
                if (cx < ox0 || cx > ox1 || cy < oy0 || cy > oy1) grid[g].push_back(bi);
            });
        }
        merged_neighbours(bi, j, old_a, b, fresh);
        for (int k : fresh) {
            touched.push_back(k);
            adj[k].push_back(bi);
        }
        adj[bi] = fresh;
        ++now;
        const int mark = now;
        for (int k : touched) {
            if (!alive[k] || k == bi || stamp[k] == mark) continue;
            stamp[k] = mark;
            if (bj[k] == j || bj[k] == bi) {
                rescan(k);
                ++now;  // rescan used its own stamp; keep this pass's marks distinct
                // (re-mark k so a later duplicate entry is skipped)
                stamp[k] = mark;
            } else if (k < bi && overlaps(boxes[k], a)) {
                const Frac v = iou_frac(boxes[k], a);
                const int cmp = bj[k] < 0 ? 1 : frac_cmp(v, bf[k]);
                if (cmp > 0 || (cmp == 0 && bi < bj[k])) {
                    bf[k] = v;
                    bv[k] = frac_value(v);
                    bj[k] = bi;
                    tree.set(k, bv[k]);
                }
            }
        }
        rescan(bi);
    }
    long long m = 0;
    for (int i = 0; i < n; ++i)
        if (alive[i] && area_of(boxes[i]) >= c.min_box_area) boxes[m++] = boxes[i];
    return m;
}

// ---------------------------------------------------------------- outliers
// count_outliers (eval.cpp:59-85): the same per-pixel FP64 test, integer
// counts reduced per block and added atomically (exact, order-free).
__global__ void count_outliers_kernel(const int32_t* __restrict__ d, const uint8_t* __restrict__ valid,
                                      const double* __restrict__ gt, size_t P, const int* slots,
                                      double abs_thresh, double rel_thresh, int strict,
                                      unsigned long long* counts) {
    const int a = blockIdx.y, s = slots ? slots[a] : a;
    const size_t base = static_cast<size_t>(s) * P, gbase = static_cast<size_t>(a) * P;
    unsigned long long ev = 0, out = 0;
    for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < P;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const double g = gt[gbase + i];
        if (!(g > 0.0)) continue;
        if (!valid[base + i]) {
            if (strict) {
                ++ev;
                ++out;
            }
            continue;
        }
        ++ev;
        const double e = fabs(__dsub_rn(static_cast<double>(d[base + i]), g));
        if (e > abs_thresh && e / g > rel_thresh) ++out;
    }
    for (int o = 16; o > 0; o >>= 1) {
        ev += __shfl_down_sync(0xffffffffu, ev, o);
        out += __shfl_down_sync(0xffffffffu, out, o);
    }
    if ((threadIdx.x & 31) == 0 && (ev || out)) {
        atomicAdd(counts + 2 * a, ev);
        atomicAdd(counts + 2 * a + 1, out);
    }
}

void launch_count_outliers(const int32_t* d, const uint8_t* valid, const double* gt, size_t P,
                           int n, const int* slots, double abs_thresh, double rel_thresh,
                           int strict, unsigned long long* counts, Launch L) {
    cudaMemsetAsync(counts, 0, sizeof(unsigned long long) * 2 * n, L.st);
    const unsigned blocks = static_cast<unsigned>(std::min<size_t>((P + 255) / 256, 148 * 4));
    count_outliers_kernel<<<dim3(blocks, n), 256, 0, L.st>>>(d, valid, gt, P, slots, abs_thresh,
                                                             rel_thresh, strict, counts);
    ++*L.counter;
}

}  // namespace tsgm
