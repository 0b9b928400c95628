/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference hot path.
 * See tsgm_oracle.h for the contract. Compiled with -ffp-contract=off so no
 * FMA is formed: the x86-64 reference build has none either (no -march in
 * /root/reference/proj/CMakeLists.txt:16). All file:line citations are into
 * /root/reference/proj. */
#include "tsgm_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static char g_err[256];
const char* or_last_error(void) { return g_err; }

static int fail(const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return 1;
}

#define CENSUS_R 2
#define MAX_COST 24

/* ---------------------------------------------------------------- params */

/* SgmParams::validate, src/sgm.cpp:14-23 */
int or_sgm_validate(const or_sgm_params* p) {
    if (p->p1 <= 0 || p->p2 < p->p1) return fail("SgmParams: require 0 < p1 <= p2");
    if (p->paths != 4 && p->paths != 8) return fail("SgmParams: paths must be 4 or 8");
    if (p->d_max < 1 || p->d_max > 65535) return fail("SgmParams: d_max out of range");
    if ((MAX_COST + p->p2) * p->paths > 65535)
        return fail("SgmParams: p2 too large for 16-bit accumulation");
    return 0;
}

/* FilterConfig::validate, src/temporal_filter.cpp:16-26 */
int or_filter_validate(const or_filter* f, int d_max) {
    if (!(f->q > 0.0) || !(f->r > 0.0)) return fail("NoiseParams: q and r must be positive");
    if (f->p_init < (double)d_max * d_max / 4.0)
        return fail("FilterConfig: p_init does not cover the disparity space");
    if (f->disc_thresh < 1.0) return fail("FilterConfig: disc_thresh must be at least 1");
    if (f->min_range_halfwidth < 0) return fail("FilterConfig: negative min_range_halfwidth");
    if (f->range_use_stddev && !(f->range_stddev_gain > 0.0))
        return fail("FilterConfig: range_stddev_gain must be positive");
    return 0;
}

/* ---------------------------------------------------------------- census / cost */

/* census_transform, src/matching_cost.cpp:53-79: 5x5 window, raster order,
 * bit 23 = (-2,-2), strict "darker than centre"; 2-px border signature 0. */
int or_census(const uint8_t* img, int w, int h, uint32_t* sig) {
    if (w < 2 * CENSUS_R + 1 || h < 2 * CENSUS_R + 1)
        return fail("census_transform: image smaller than the 5x5 window");
    memset(sig, 0, sizeof(uint32_t) * (size_t)w * h);
    for (int y = CENSUS_R; y < h - CENSUS_R; ++y)
        for (int x = CENSUS_R; x < w - CENSUS_R; ++x) {
            const uint8_t c = img[(size_t)y * w + x];
            uint32_t s = 0;
            for (int dy = -CENSUS_R; dy <= CENSUS_R; ++dy)
                for (int dx = -CENSUS_R; dx <= CENSUS_R; ++dx) {
                    if (dx == 0 && dy == 0) continue;
                    s = (s << 1) | (img[(size_t)(y + dy) * w + x + dx] < c ? 1u : 0u);
                }
            sig[(size_t)y * w + x] = s;
        }
    return 0;
}

/* make_cost_volume offsets, src/matching_cost.cpp:30-48 */
int64_t or_offsets(const uint16_t* lo, const uint16_t* hi, size_t n, uint32_t* offsets) {
    uint64_t total = 0;
    for (size_t i = 0; i < n; ++i) {
        offsets[i] = (uint32_t)total;
        total += (uint64_t)hi[i] - lo[i] + 1;
    }
    if (total > 0xffffffffull) {
        fail("CostVolume: volume exceeds 32-bit addressing");
        return -1;
    }
    offsets[n] = (uint32_t)total;
    return (int64_t)total;
}

static int census_defined(int x, int y, int w, int h) {
    return x >= CENSUS_R && x < w - CENSUS_R && y >= CENSUS_R && y < h - CENSUS_R;
}

/* build_cost_volume / matching_cost, src/matching_cost.cpp:81-117:
 * C = popcount(sigL(x,y) ^ sigR(x-d,y)), 24 when either side is undefined or
 * x-d < 0. */
void or_cost_volume(const uint32_t* sig_l, const uint32_t* sig_r, int w, int h,
                    const uint16_t* lo, const uint32_t* offsets, uint8_t* cost) {
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            const size_t i = (size_t)y * w + x;
            const uint32_t n = offsets[i + 1] - offsets[i];
            uint8_t* out = cost + offsets[i];
            for (uint32_t j = 0; j < n; ++j) {
                const int xr = x - ((int)lo[i] + (int)j);
                if (!census_defined(x, y, w, h) || xr < 0 || !census_defined(xr, y, w, h))
                    out[j] = MAX_COST;
                else
                    out[j] = (uint8_t)__builtin_popcount(sig_l[i] ^ sig_r[(size_t)y * w + xr]);
            }
        }
}

/* ---------------------------------------------------------------- aggregation */

/* One path direction of Eq. 1 with the reference's ragged-range rules
 * (src/sgm.cpp:93-126; textbook form tests/oracles.hpp:70-118). (dx, dy) is
 * the predecessor offset. L = C at the image edge; otherwise
 *   best = min(qmin + P2, Lq[d], Lq[d-1] + P1, Lq[d+1] + P1) over levels the
 *   predecessor's window holds, L = C + best - qmin. */
void or_aggregate_direction(const uint8_t* cost, const uint16_t* lo, const uint32_t* offsets,
                            int w, int h, int dx, int dy, int p1, int p2, uint16_t* dir) {
    int32_t* qmin_map = (int32_t*)malloc(sizeof(int32_t) * (size_t)w * h);
    const int ys = dy > 0 ? -1 : 1, y0 = dy > 0 ? h - 1 : 0, y1 = dy > 0 ? -1 : h;
    const int xs = dx > 0 ? -1 : 1, x0 = dx > 0 ? w - 1 : 0, x1 = dx > 0 ? -1 : w;
    for (int y = y0; y != y1; y += ys)
        for (int x = x0; x != x1; x += xs) {
            const size_t i = (size_t)y * w + x;
            const int n = (int)(offsets[i + 1] - offsets[i]);
            const uint8_t* c = cost + offsets[i];
            uint16_t* out = dir + offsets[i];
            int32_t mn = 0x7fffffff;
            const int qx = x + dx, qy = y + dy;
            if (qx < 0 || qx >= w || qy < 0 || qy >= h) {
                for (int j = 0; j < n; ++j) {
                    out[j] = c[j];
                    if (c[j] < mn) mn = c[j];
                }
            } else {
                const size_t q = (size_t)qy * w + qx;
                const uint16_t* lq = dir + offsets[q];
                const int qn = (int)(offsets[q + 1] - offsets[q]);
                const int qmin = qmin_map[q];
                const int shift = (int)lo[i] - (int)lo[q];
                for (int j = 0; j < n; ++j) {
                    const int k = j + shift; /* predecessor index of the same level */
                    int best = qmin + p2;
                    if (k >= 0 && k < qn && lq[k] < best) best = lq[k];
                    if (k - 1 >= 0 && k - 1 < qn && lq[k - 1] + p1 < best) best = lq[k - 1] + p1;
                    if (k + 1 >= 0 && k + 1 < qn && lq[k + 1] + p1 < best) best = lq[k + 1] + p1;
                    const int l = c[j] + best - qmin;
                    out[j] = (uint16_t)l;
                    if (l < mn) mn = l;
                }
            }
            qmin_map[i] = mn;
        }
    free(qmin_map);
}

/* aggregate_paths, src/sgm.cpp:135-161: direction sets and the u16 sum. */
int or_aggregate(const uint8_t* cost, const uint16_t* lo, const uint32_t* offsets, int w, int h,
                 const or_sgm_params* p, uint16_t* agg) {
    if (or_sgm_validate(p)) return 1;
    static const int nondiag[4][2] = {{-1, 0}, {0, -1}, {1, 0}, {0, 1}};
    static const int diag[4][2] = {{-1, -1}, {1, -1}, {1, 1}, {-1, 1}};
    const size_t n = offsets[(size_t)w * h];
    uint16_t* dir = (uint16_t*)malloc(sizeof(uint16_t) * (n ? n : 1));
    memset(agg, 0, sizeof(uint16_t) * n);
    const int use_nd = p->paths == 8 || p->path_set == 0;
    const int use_d = p->paths == 8 || p->path_set == 1;
    for (int set = 0; set < 2; ++set) {
        if ((set == 0 && !use_nd) || (set == 1 && !use_d)) continue;
        for (int k = 0; k < 4; ++k) {
            const int* o = set == 0 ? nondiag[k] : diag[k];
            or_aggregate_direction(cost, lo, offsets, w, h, o[0], o[1], p->p1, p->p2, dir);
            for (size_t c = 0; c < n; ++c) agg[c] = (uint16_t)(agg[c] + dir[c]);
        }
    }
    free(dir);
    return 0;
}

/* winner_takes_all, src/sgm.cpp:163-187: first minimum, 2-px border invalid. */
void or_wta(const uint16_t* agg, const uint16_t* lo, const uint32_t* offsets, int w, int h,
            int32_t* d, uint8_t* valid) {
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            const size_t i = (size_t)y * w + x;
            d[i] = 0;
            valid[i] = 0;
            if (!census_defined(x, y, w, h)) continue;
            const uint16_t* s = agg + offsets[i];
            const int n = (int)(offsets[i + 1] - offsets[i]);
            int best = 0;
            for (int j = 1; j < n; ++j)
                if (s[j] < s[best]) best = j;
            d[i] = lo[i] + best;
            valid[i] = 1;
        }
}

/* median_refine, src/sgm.cpp:189-216: lower median of the valid 3x3
 * neighbours, valid iff at least 5 of them. */
void or_median(const int32_t* d, const uint8_t* valid, int w, int h, int32_t* out_d,
               uint8_t* out_valid) {
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            int32_t v[9];
            int n = 0;
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    const int nx = x + dx, ny = y + dy;
                    if (nx < 0 || nx >= w || ny < 0 || ny >= h || !valid[(size_t)ny * w + nx])
                        continue;
                    /* insertion sort as we go */
                    int32_t val = d[(size_t)ny * w + nx];
                    int k = n++;
                    while (k > 0 && v[k - 1] > val) {
                        v[k] = v[k - 1];
                        --k;
                    }
                    v[k] = val;
                }
            const size_t i = (size_t)y * w + x;
            if (n < 5) {
                out_d[i] = 0;
                out_valid[i] = 0;
            } else {
                out_d[i] = v[(n - 1) / 2];
                out_valid[i] = 1;
            }
        }
}

/* sgm_match, src/sgm.cpp:226-257 (validation at :229-234, ranges.validate at
 * src/matching_cost.cpp:14-25). */
int or_sgm_match(const uint8_t* left, const uint8_t* right, int w, int h, const uint16_t* lo,
                 const uint16_t* hi, const or_sgm_params* p, int32_t* d, uint8_t* valid) {
    if (or_sgm_validate(p)) return 1;
    const size_t np = (size_t)w * h;
    for (size_t i = 0; i < np; ++i)
        if (lo[i] > hi[i] || hi[i] >= p->d_max)
            return fail("SearchRangeMap: range outside [0, d_max)");
    if (w < 2 * CENSUS_R + 1 || h < 2 * CENSUS_R + 1)
        return fail("census_transform: image smaller than the 5x5 window");
    uint32_t* sl = (uint32_t*)malloc(4 * np);
    uint32_t* sr = (uint32_t*)malloc(4 * np);
    uint32_t* off = (uint32_t*)malloc(4 * (np + 1));
    or_census(left, w, h, sl);
    or_census(right, w, h, sr);
    const int64_t n = or_offsets(lo, hi, np, off);
    if (n < 0) {
        free(sl); free(sr); free(off);
        return 1;
    }
    uint8_t* cost = (uint8_t*)malloc((size_t)n + 1);
    uint16_t* agg = (uint16_t*)malloc(2 * (size_t)n + 2);
    or_cost_volume(sl, sr, w, h, lo, off, cost);
    or_aggregate(cost, lo, off, w, h, p, agg);
    or_wta(agg, lo, off, w, h, d, valid);
    free(sl); free(sr); free(off); free(cost); free(agg);
    return 0;
}

/* ---------------------------------------------------------------- geometry */

/* Fixed sequential-k products: the order the oracle build's Eigen stand-in
 * uses (oracle/eigen_shim/Eigen/Dense). Row-major here. */
static void mat3_mul(const double* a, const double* b, double* r) {
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            r[i * 3 + j] = (a[i * 3 + 0] * b[0 * 3 + j] + a[i * 3 + 1] * b[1 * 3 + j]) +
                           a[i * 3 + 2] * b[2 * 3 + j];
}
static void mat3_vec(const double* a, const double* v, double* r) {
    for (int i = 0; i < 3; ++i)
        r[i] = (a[i * 3 + 0] * v[0] + a[i * 3 + 1] * v[1]) + a[i * 3 + 2] * v[2];
}
static void mat4_mul(const double* a, const double* b, double* r) {
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j)
            r[i * 4 + j] = ((a[i * 4 + 0] * b[0 * 4 + j] + a[i * 4 + 1] * b[1 * 4 + j]) +
                            a[i * 4 + 2] * b[2 * 4 + j]) +
                           a[i * 4 + 3] * b[3 * 4 + j];
}

/* RigidMotion::validate, src/geometry.cpp:30-36 */
static int motion_validate(const double* r) {
    double rt[9], g[9];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) rt[i * 3 + j] = r[j * 3 + i];
    mat3_mul(rt, r, g);
    double mx = 0.0;
    for (int i = 0; i < 9; ++i) {
        const double e = fabs(g[i] - ((i % 4) == 0 ? 1.0 : 0.0));
        if (i == 0 || e > mx) mx = e;
    }
    if (!(mx <= 1e-9)) return fail("RigidMotion: rotation is not orthonormal");
    const double det = r[0] * (r[4] * r[8] - r[5] * r[7]) - r[3] * (r[1] * r[8] - r[2] * r[7]) +
                       r[6] * (r[1] * r[5] - r[2] * r[4]);
    if (!(fabs(det - 1.0) <= 1e-9)) return fail("RigidMotion: rotation determinant is not +1");
    return 0;
}

/* StereoCalib::validate, src/geometry.cpp:21-28 */
static int calib_validate(const or_calib* c) {
    if (!(c->focal_px > 0.0)) return fail("StereoCalib: focal_px must be positive");
    if (!(c->baseline_m > 0.0)) return fail("StereoCalib: baseline_m must be positive");
    if (!(c->width > 0 && c->height > 0)) return fail("StereoCalib: empty image");
    if (!(c->cx >= 0.0 && c->cx < c->width)) return fail("StereoCalib: cx outside image");
    if (!(c->cy >= 0.0 && c->cy < c->height)) return fail("StereoCalib: cy outside image");
    if (!(c->d_max >= 1)) return fail("StereoCalib: d_max must be at least 1");
    return 0;
}

/* relative_motion, src/geometry.cpp:189-197: cur_to_world^-1 after prev_to_world,
 * exact identity for repeated poses. Poses are row-major 3x4 [R|t]. */
int or_relative_motion(const double* prev12, const double* cur12, double* r9, double* t3) {
    double rp[9], rc[9], tp[3], tc[3];
    for (int i = 0; i < 3; ++i) {
        for (int j = 0; j < 3; ++j) {
            rp[i * 3 + j] = prev12[i * 4 + j];
            rc[i * 3 + j] = cur12[i * 4 + j];
        }
        tp[i] = prev12[i * 4 + 3];
        tc[i] = cur12[i * 4 + 3];
    }
    if (motion_validate(rp) || motion_validate(rc)) return 1;
    int same = 1;
    for (int i = 0; i < 12; ++i) same &= prev12[i] == cur12[i];
    if (same) {
        for (int i = 0; i < 9; ++i) r9[i] = (i % 4) == 0 ? 1.0 : 0.0;
        t3[0] = t3[1] = t3[2] = 0.0;
        return 0;
    }
    double rct[9], it[3], tmp[3];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) rct[i * 3 + j] = rc[j * 3 + i];
    mat3_vec(rct, tc, tmp); /* inverse(): t = -(R^T t) (geometry.cpp:42-47) */
    for (int i = 0; i < 3; ++i) it[i] = -tmp[i];
    mat3_mul(rct, rp, r9); /* after(): R = R2 R1, t = R2 t1 + t2 (:49-54) */
    mat3_vec(rct, tp, tmp);
    for (int i = 0; i < 3; ++i) t3[i] = tmp[i] + it[i];
    return 0;
}

/* disparity_homography, src/geometry.cpp:77-110: H = Qinv * T * Q, evaluated
 * left to right; exact identity motion short-circuits to I. Row-major h16. */
int or_homography(const double* r9, const double* t3, const or_calib* c, double* h16) {
    if (calib_validate(c) || motion_validate(r9)) return 1;
    int ident = t3[0] == 0.0 && t3[1] == 0.0 && t3[2] == 0.0;
    for (int i = 0; i < 9; ++i) ident &= r9[i] == ((i % 4) == 0 ? 1.0 : 0.0);
    memset(h16, 0, 16 * sizeof(double));
    if (ident) {
        h16[0] = h16[5] = h16[10] = h16[15] = 1.0;
        return 0;
    }
    const double f = c->focal_px, b = c->baseline_m;
    double q[16] = {0}, qi[16] = {0}, t[16] = {0}, tmp[16];
    q[0 * 4 + 0] = 1.0;
    q[0 * 4 + 3] = -c->cx;
    q[1 * 4 + 1] = 1.0;
    q[1 * 4 + 3] = -c->cy;
    q[2 * 4 + 3] = f;
    q[3 * 4 + 2] = 1.0 / b;
    qi[0 * 4 + 0] = 1.0;
    qi[0 * 4 + 2] = c->cx / f;
    qi[1 * 4 + 1] = 1.0;
    qi[1 * 4 + 2] = c->cy / f;
    qi[2 * 4 + 3] = b;
    qi[3 * 4 + 2] = 1.0 / f;
    for (int i = 0; i < 3; ++i) {
        for (int j = 0; j < 3; ++j) t[i * 4 + j] = r9[i * 3 + j];
        t[i * 4 + 3] = t3[i];
    }
    t[15] = 1.0;
    mat4_mul(qi, t, tmp);
    mat4_mul(tmp, q, h16);
    return 0;
}

/* lexicographic collision order, src/geometry.cpp:116-123 */
static int replaces(double dn, double pn, double sn, double d0, double p0, double s0) {
    if (dn != d0) return dn > d0;
    if (pn != p0) return pn < p0;
    return sn < s0;
}

/* warp_state_ex, src/geometry.cpp:127-156 (DispHomography::apply :56-61). */
void or_warp(const double* d, const double* p, const uint8_t* valid, int w, int h,
             const double* H, int d_max, double* od, double* op, uint8_t* ov, double* osrc) {
    const size_t np = (size_t)w * h;
    memset(od, 0, 8 * np);
    memset(op, 0, 8 * np);
    memset(ov, 0, np);
    memset(osrc, 0, 8 * np);
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            const size_t i = (size_t)y * w + x;
            if (!valid[i]) continue;
            const double ds = d[i], xd = (double)x, yd = (double)y;
            double v[4];
            for (int r = 0; r < 4; ++r)
                v[r] = ((H[r * 4 + 0] * xd + H[r * 4 + 1] * yd) + H[r * 4 + 2] * ds) +
                       H[r * 4 + 3] * 1.0;
            if (!(v[3] > 1e-12)) continue;
            const double mx = v[0] / v[3], my = v[1] / v[3], dp = v[2] / v[3];
            if (!(dp > 0.0) || !(dp < (double)d_max)) continue;
            const int tx = (int)lround(mx);
            const int ty = (int)lround(my);
            if (tx < 0 || tx >= w || ty < 0 || ty >= h) continue;
            const size_t t = (size_t)ty * w + tx;
            const double ps = p[i];
            if (ov[t] && !replaces(dp, ps, ds, od[t], op[t], osrc[t])) continue;
            od[t] = dp;
            op[t] = ps;
            ov[t] = 1;
            osrc[t] = ds;
        }
}

/* reject_discontinuities, src/temporal_filter.cpp:51-74 */
void or_reject(const double* d, const double* p, const uint8_t* valid, int w, int h,
               double disc_thresh, double* od, double* op, uint8_t* ov) {
    static const int kdx[4] = {1, -1, 0, 0}, kdy[4] = {0, 0, 1, -1};
    const size_t np = (size_t)w * h;
    memmove(od, d, 8 * np);
    memmove(op, p, 8 * np);
    memmove(ov, valid, np);
    /* decisions against the input: inputs may alias outputs, so stage them */
    double* din = (double*)malloc(8 * np);
    uint8_t* vin = (uint8_t*)malloc(np);
    memcpy(din, od, 8 * np);
    memcpy(vin, ov, np);
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            const size_t i = (size_t)y * w + x;
            if (!vin[i]) continue;
            for (int n = 0; n < 4; ++n) {
                const int nx = x + kdx[n], ny = y + kdy[n];
                if (nx < 0 || nx >= w || ny < 0 || ny >= h) continue;
                const size_t j = (size_t)ny * w + nx;
                if (!vin[j]) continue;
                if (fabs(din[i] - din[j]) > disc_thresh) {
                    od[i] = 0.0;
                    op[i] = 0.0;
                    ov[i] = 0;
                    break;
                }
            }
        }
    free(din);
    free(vin);
}

/* fill_zoom_holes, src/temporal_filter.cpp:76-106 */
void or_fill(const double* d, const double* p, const uint8_t* valid, int w, int h, double* od,
             double* op, uint8_t* ov) {
    const size_t np = (size_t)w * h;
    double* din = (double*)malloc(8 * np);
    double* pin = (double*)malloc(8 * np);
    uint8_t* vin = (uint8_t*)malloc(np);
    memcpy(din, d, 8 * np);
    memcpy(pin, p, 8 * np);
    memcpy(vin, valid, np);
    memmove(od, din, 8 * np);
    memmove(op, pin, 8 * np);
    memmove(ov, vin, np);
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            const size_t i = (size_t)y * w + x;
            if (vin[i]) continue;
            const int horiz = x - 1 >= 0 && x + 1 < w && vin[i - 1] && vin[i + 1];
            const int vert = y - 1 >= 0 && y + 1 < h && vin[i - w] && vin[i + w];
            if (!horiz && !vert) continue;
            double ds = 0.0, ps = 0.0;
            int n = 0;
            if (horiz) {
                ds += din[i - 1] + din[i + 1];
                ps += pin[i - 1] + pin[i + 1];
                n += 2;
            }
            if (vert) {
                ds += din[i - w] + din[i + w];
                ps += pin[i - w] + pin[i + w];
                n += 2;
            }
            od[i] = ds / n;
            op[i] = ps / n;
            ov[i] = 1;
        }
    free(din);
    free(pin);
    free(vin);
}

/* predict, src/temporal_filter.cpp:28-49: warp, phi = d'/d_src,
 * p' = (phi*phi)*p + q, then reject and fill. */
int or_predict(const double* d, const double* p, const uint8_t* valid, int w, int h,
               const double* r9, const double* t3, const or_calib* c, const or_filter* f,
               double* od, double* op, uint8_t* ov) {
    double H[16];
    if (or_homography(r9, t3, c, H)) return 1;
    const size_t np = (size_t)w * h;
    double* src = (double*)malloc(8 * np);
    or_warp(d, p, valid, w, h, H, c->d_max, od, op, ov, src);
    for (size_t i = 0; i < np; ++i) {
        if (!ov[i]) continue;
        if (!(src[i] > 0.0)) {
            od[i] = op[i] = 0.0;
            ov[i] = 0;
            continue;
        }
        const double phi = od[i] / src[i];
        op[i] = phi * phi * op[i] + f->q;
    }
    free(src);
    or_reject(od, op, ov, w, h, f->disc_thresh, od, op, ov);
    or_fill(od, op, ov, w, h, od, op, ov);
    return 0;
}

/* derive_search_ranges, src/temporal_filter.cpp:108-143 */
void or_ranges(const double* d, const double* p, const uint8_t* valid, int w, int h, int d_max,
               const or_filter* f, uint16_t* lo_out, uint16_t* hi_out) {
    const int top = d_max - 1;
    const int min_len = 2 * f->min_range_halfwidth + 1;
    const size_t np = (size_t)w * h;
    for (size_t i = 0; i < np; ++i) {
        lo_out[i] = 0;
        hi_out[i] = (uint16_t)top;
        if (!valid[i]) continue;
        const double half = f->range_use_stddev ? f->range_stddev_gain * sqrt(p[i]) : p[i];
        int lo = (int)floor(d[i] - half);
        int hi = (int)ceil(d[i] + half);
        lo = lo < top ? lo : top;
        lo = lo > 0 ? lo : 0;
        hi = hi < top ? hi : top;
        hi = hi > 0 ? hi : 0;
        const int deficit = min_len - (hi - lo + 1);
        if (deficit > 0) {
            lo -= deficit / 2;
            hi += deficit - deficit / 2;
            if (lo < 0) {
                hi = (hi - lo) < top ? (hi - lo) : top;
                lo = 0;
            }
            if (hi > top) {
                lo = (lo - (hi - top)) > 0 ? (lo - (hi - top)) : 0;
                hi = top;
            }
        }
        lo_out[i] = (uint16_t)lo;
        hi_out[i] = (uint16_t)hi;
    }
}

/* correct, src/temporal_filter.cpp:145-170 (Joseph-form variance) */
void or_correct(const double* d, const double* p, const uint8_t* valid, const int32_t* md,
                const uint8_t* mv, int w, int h, double r, double* od, double* op, uint8_t* ov) {
    const size_t np = (size_t)w * h;
    for (size_t i = 0; i < np; ++i) {
        const int hp = valid[i] != 0, hm = mv[i] != 0;
        double dd = 0.0, pp = 0.0;
        uint8_t vv = 0;
        if (hp && hm) {
            const double pv = p[i];
            const double k = pv / (pv + r);
            dd = d[i] + k * ((double)md[i] - d[i]);
            pp = (1.0 - k) * (1.0 - k) * pv + k * k * r;
            vv = 1;
        } else if (hm) {
            dd = (double)md[i];
            pp = r;
            vv = 1;
        } else if (hp) {
            dd = d[i];
            pp = p[i];
            vv = 1;
        }
        od[i] = dd;
        op[i] = pp;
        ov[i] = vv;
    }
}

/* step's diff loop, src/temporal_filter.cpp:223-229 (== disparity_difference,
 * src/motion_detect.cpp:131-140) */
void or_diff(const double* pd, const uint8_t* pv, const int32_t* md, const uint8_t* mv, int w,
             int h, double* diff) {
    const size_t np = (size_t)w * h;
    for (size_t i = 0; i < np; ++i)
        diff[i] = (pv[i] && mv[i]) ? fabs(pd[i] - (double)md[i]) : 0.0;
}

/* Extension A21: moving iff both valid and
 * (dz - d_pred)^2 > (tau*tau) * (p_pred + r). */
void or_mask(const double* pd, const double* pp, const uint8_t* pv, const int32_t* md,
             const uint8_t* mv, int w, int h, double r, double tau, uint8_t* mask) {
    const size_t np = (size_t)w * h;
    for (size_t i = 0; i < np; ++i) {
        mask[i] = 0;
        if (!(pv[i] && mv[i])) continue;
        const double e = (double)md[i] - pd[i];
        mask[i] = (e * e > (tau * tau) * (pp[i] + r)) ? 1 : 0;
    }
}

/* render_integer, src/temporal_filter.cpp:178-191 */
void or_render(const double* d, const uint8_t* valid, int w, int h, int32_t* od, uint8_t* ov) {
    const size_t np = (size_t)w * h;
    for (size_t i = 0; i < np; ++i) {
        od[i] = valid[i] ? (int32_t)lround(d[i]) : 0;
        ov[i] = valid[i] ? 1 : 0;
    }
}

/* Extension A22 (tsgm_oracle.h). */
void or_subpixel(const uint16_t* agg, const uint16_t* lo, const uint16_t* hi,
                 const uint32_t* offsets, const int32_t* d, const uint8_t* valid, int w, int h,
                 float* out) {
    const size_t np = (size_t)w * h;
    for (size_t i = 0; i < np; ++i) {
        out[i] = 0.0f;
        if (!valid[i]) continue;
        const int dd = d[i], l = lo[i], u = hi[i];
        const uint16_t* s = agg + offsets[i];
        if (dd - 1 < l || dd + 1 > u) {
            out[i] = (float)dd;
            continue;
        }
        const int sm1 = s[dd - 1 - l], s0 = s[dd - l], sp1 = s[dd + 1 - l];
        const int den = sm1 - 2 * s0 + sp1;
        if (den <= 0) {
            out[i] = (float)dd;
            continue;
        }
        const float off = (float)(sm1 - sp1) / (2.0f * (float)den);
        out[i] = (float)dd + off;
    }
}

/* step, src/temporal_filter.cpp:195-232 */
int or_step(const double* sd, const double* sp, const uint8_t* sv, int state_w, int state_h,
            const uint8_t* left, const uint8_t* right, int w, int h, const double* r9,
            const double* t3, const or_calib* calib, const or_sgm_params* params,
            const or_filter* f, double* od, double* op, uint8_t* ov, int32_t* ed, uint8_t* ev,
            double* diff, or_step_debug* dbg) {
    const size_t np = (size_t)w * h;
    int empty = state_w == 0 && state_h == 0;
    if (!empty && (state_w != w || state_h != h))
        return fail("step: state dimension mismatch");
    if (params->d_max != calib->d_max)
        return fail("step: params.d_max disagrees with calibration");
    double* zd = NULL;
    double* zp = NULL;
    uint8_t* zv = NULL;
    if (empty) {
        zd = (double*)calloc(np, 8);
        zp = (double*)calloc(np, 8);
        zv = (uint8_t*)calloc(np, 1);
        sd = zd;
        sp = zp;
        sv = zv;
    }
    double* pd = (double*)malloc(8 * np);
    double* pp = (double*)malloc(8 * np);
    uint8_t* pv = (uint8_t*)malloc(np);
    uint16_t* lo = (uint16_t*)malloc(2 * np);
    uint16_t* hi = (uint16_t*)malloc(2 * np);
    int32_t* md = (int32_t*)malloc(4 * np);
    uint8_t* mv = (uint8_t*)malloc(np);
    int32_t* rd = (int32_t*)malloc(4 * np);
    uint8_t* rv = (uint8_t*)malloc(np);
    int rc = or_predict(sd, sp, sv, w, h, r9, t3, calib, f, pd, pp, pv);
    if (!rc) {
        or_ranges(pd, pp, pv, w, h, calib->d_max, f, lo, hi);
        rc = or_sgm_match(left, right, w, h, lo, hi, params, md, mv);
    }
    if (!rc) {
        or_correct(pd, pp, pv, md, mv, w, h, f->r, od, op, ov);
        or_diff(pd, pv, md, mv, w, h, diff);
        or_render(od, ov, w, h, rd, rv);
        or_median(rd, rv, w, h, ed, ev);
        if (dbg) {
            if (dbg->pred_d) memcpy(dbg->pred_d, pd, 8 * np);
            if (dbg->pred_p) memcpy(dbg->pred_p, pp, 8 * np);
            if (dbg->pred_v) memcpy(dbg->pred_v, pv, np);
            if (dbg->lo) memcpy(dbg->lo, lo, 2 * np);
            if (dbg->hi) memcpy(dbg->hi, hi, 2 * np);
            if (dbg->meas_d) memcpy(dbg->meas_d, md, 4 * np);
            if (dbg->meas_v) memcpy(dbg->meas_v, mv, np);
            if (dbg->mask) or_mask(pd, pp, pv, md, mv, w, h, f->r, dbg->mask_tau, dbg->mask);
        }
    }
    free(pd); free(pp); free(pv); free(lo); free(hi); free(md); free(mv); free(rd); free(rv);
    free(zd); free(zp); free(zv);
    return rc;
}


/* ======================================================= box detector (§8(f) row 1) */
int or_detect_validate(const or_detect_cfg* c) {
    /* DetectConfig::validate, motion_detect.cpp:11-23 */
    if (c->n_windows < 1) return fail("DetectConfig: no window sizes");
    for (int i = 0; i < c->n_windows; ++i)
        if (c->window_wh[2 * i] < 1 || c->window_wh[2 * i + 1] < 1)
            return fail("DetectConfig: non-positive window size");
    if (!(c->score_thresh > 0.0)) return fail("DetectConfig: score_thresh must be positive");
    if (!(c->merge_stop_iou > 0.0 && c->merge_stop_iou < 1.0))
        return fail("DetectConfig: merge_stop_iou must lie in (0, 1)");
    if (c->min_box_area < 0) return fail("DetectConfig: negative min_box_area");
    return 0;
}

void or_integral_image(const double* map, int w, int h, double* sat) {
    /* integral_image, motion_detect.cpp:25-42: row accumulator left to right,
     * cur = above + row_acc */
    const size_t sw = (size_t)w + 1;
    for (size_t i = 0; i < sw; ++i) sat[i] = 0.0;
    for (int y = 0; y < h; ++y) {
        double acc = 0.0;
        double* cur = sat + (size_t)(y + 1) * sw;
        const double* above = sat + (size_t)y * sw;
        cur[0] = 0.0;
        for (int x = 0; x < w; ++x) {
            acc += map[(size_t)y * w + x];
            cur[x + 1] = above[x + 1] + acc;
        }
    }
}

static double sat_at(const double* sat, int w, int row, int col) {
    return sat[(size_t)row * ((size_t)w + 1) + col];
}

int or_box_sum(const double* sat, int w, int h, const or_box* b, double* out) {
    /* box_sum, motion_detect.cpp:44-50: ((a - b) - c) + d */
    if (b->x0 < 0 || b->y0 < 0 || b->x1 > w || b->y1 > h || b->x0 >= b->x1 || b->y0 >= b->y1)
        return fail("box_sum: box out of bounds");
    *out = sat_at(sat, w, b->y1, b->x1) - sat_at(sat, w, b->y0, b->x1) -
           sat_at(sat, w, b->y1, b->x0) + sat_at(sat, w, b->y0, b->x0);
    return 0;
}

static long long box_area(const or_box* b) { return (long long)(b->x1 - b->x0) * (b->y1 - b->y0); }

double or_iou(const or_box* a, const or_box* b) {
    /* iou, motion_detect.cpp:52-62 */
    const int ix0 = a->x0 > b->x0 ? a->x0 : b->x0;
    const int iy0 = a->y0 > b->y0 ? a->y0 : b->y0;
    const int ix1 = a->x1 < b->x1 ? a->x1 : b->x1;
    const int iy1 = a->y1 < b->y1 ? a->y1 : b->y1;
    if (ix0 >= ix1 || iy0 >= iy1) return 0.0;
    const double inter = (double)(ix1 - ix0) * (iy1 - iy0);
    const double uni = (double)box_area(a) + (double)box_area(b) - inter;
    return inter / uni;
}

long long or_candidates(const double* diff, int w, int h, const or_detect_cfg* c, or_box* out,
                        long long cap) {
    /* detect_candidate_windows, motion_detect.cpp:64-99: sizes in order, rows
     * top to bottom, columns left to right */
    if (or_detect_validate(c)) return -1;
    double* sat = (double*)malloc(sizeof(double) * ((size_t)w + 1) * ((size_t)h + 1));
    or_integral_image(diff, w, h, sat);
    const int region_top = h / 3;
    long long n = 0;
    for (int k = 0; k < c->n_windows; ++k) {
        const int ww = c->window_wh[2 * k], wh = c->window_wh[2 * k + 1];
        if (ww > w || region_top + wh > h) continue;
        const int sx = ww / 4 > 1 ? ww / 4 : 1, sy = wh / 4 > 1 ? wh / 4 : 1;
        const int n_rows = (h - wh - region_top) / sy + 1;
        for (int row = 0; row < n_rows; ++row) {
            const int y0 = region_top + row * sy;
            for (int x0 = 0; x0 + ww <= w; x0 += sx) {
                or_box b = {x0, y0, x0 + ww, y0 + wh, 0.0};
                double sum;
                or_box_sum(sat, w, h, &b, &sum);
                const double mean = sum / (double)box_area(&b);
                if (mean > c->score_thresh) {
                    b.score = mean;
                    if (n < cap) out[n] = b;
                    ++n;
                }
            }
        }
    }
    free(sat);
    return n;
}

long long or_greedy_merge(or_box* boxes, long long n, const or_detect_cfg* c) {
    /* greedy_merge, motion_detect.cpp:101-129: the best pair (first on ties)
     * by exhaustive search, merged into the earlier box; then the area filter */
    while (n > 1) {
        double best = 0.0;
        long long bi = 0, bj = 0;
        for (long long i = 0; i + 1 < n; ++i)
            for (long long j = i + 1; j < n; ++j) {
                const double v = or_iou(&boxes[i], &boxes[j]);
                if (v > best) {
                    best = v;
                    bi = i;
                    bj = j;
                }
            }
        if (best < c->merge_stop_iou) break;
        or_box* a = &boxes[bi];
        const or_box* b = &boxes[bj];
        const double aa = (double)box_area(a), ab = (double)box_area(b);
        a->score = (a->score * aa + b->score * ab) / (aa + ab);
        if (b->x0 < a->x0) a->x0 = b->x0;
        if (b->y0 < a->y0) a->y0 = b->y0;
        if (b->x1 > a->x1) a->x1 = b->x1;
        if (b->y1 > a->y1) a->y1 = b->y1;
        memmove(&boxes[bj], &boxes[bj + 1], sizeof(or_box) * (size_t)(n - bj - 1));
        --n;
    }
    long long m = 0;
    for (long long i = 0; i < n; ++i)
        if (box_area(&boxes[i]) >= c->min_box_area) boxes[m++] = boxes[i];
    return m;
}


/* ======================================================= outlier metric (§8(f) row 3) */
void or_count_outliers(const int32_t* d, const uint8_t* valid, const double* gt, int w, int h,
                       double abs_thresh, double rel_thresh, int strict_density,
                       long long* evaluated, long long* outliers) {
    /* count_outliers, eval.cpp:59-85: GT valid iff gt > 0; an estimate is an
     * outlier iff |e| > abs AND |e| / gt > rel; strict density counts missing
     * estimates as evaluated outliers */
    long long ev = 0, out = 0;
    for (size_t i = 0; i < (size_t)w * h; ++i) {
        const double g = gt[i];
        if (!(g > 0.0)) continue;
        if (!valid[i]) {
            if (strict_density) { ++ev; ++out; }
            continue;
        }
        ++ev;
        const double e = fabs((double)d[i] - g);
        if (e > abs_thresh && e / g > rel_thresh) ++out;
    }
    *evaluated = ev;
    *outliers = out;
}

void or_error_hist(const double* e, const uint8_t* use, size_t n, double lo, double hi,
                   double bw, long long* counts, int nbins, long long* tallies, double* sums) {
    /* ErrorHistogram::add, noise_calib.cpp:16-33, samples in the reference's
     * order (frames in order, each row-major) */
    for (size_t i = 0; i < n; ++i) {
        if (!use[i]) continue;
        const double v = e[i];
        if (fabs(v) <= 1.0) ++tallies[2];
        if (v < lo) { ++tallies[0]; continue; }
        if (v >= hi) { ++tallies[1]; continue; }
        size_t bin = (size_t)((v - lo) / bw);
        if (bin >= (size_t)nbins) bin = (size_t)nbins - 1;
        ++counts[bin];
        ++tallies[3];
        sums[0] += v;
        sums[1] += v * v;
    }
}
