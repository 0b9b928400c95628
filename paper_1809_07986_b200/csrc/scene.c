/* Seeded synthetic stereo sequences standing in for KITTI raw (not in this
 * image): the BASELINE.json configs 0-4. Host C, multi-threaded; used by
 * bench.py and the tests to feed the SAME frames to the GPU path and to the
 * CPU reference/oracle. It is input generation, not part of the hot path.
 *
 * World: X right, Y down, Z forward (camera convention of geometry.hpp:14-16).
 * Scene = ground plane (Y = cam_height) + far wall + N fronto-parallel
 * rectangles standing on the ground, some of them moving. Both cameras are
 * ray-cast against the same world-anchored, band-limited 4-octave value noise
 * (octaves finer than the pixel footprint are faded out, as a lens would), so
 * right(x - d) == left(x) on every surface up to sampling; additive Gaussian
 * noise sigma (default 2) and an optional per-frame gain are applied per image.
 * Poses: camera-to-world [R|t] per frame (KITTI odometry convention, as read
 * by load_poses, geometry.cpp:162-187): forward fwd_m along the heading and
 * yaw_deg about Y per frame. */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../../include/tsgm_scene.h"

#define MAX_RECTS 64

typedef struct {
    double x0, x1, y0, y1, z; /* world extent at frame 0 */
    double vx, vz;            /* per-frame velocity (movers) */
    double cell;              /* base texture cell, metres */
    uint32_t tex_id;
} rect_t;

typedef struct {
    tsgm_scene_cfg cfg;
    rect_t rects[MAX_RECTS];
    int n_rects;
    double wall_z, cam_height;
    double* poses; /* frames x 12 */
    double* gains; /* frames x 2 */
} scene_t;

static uint64_t splitmix(uint64_t* s) {
    uint64_t z = (*s += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
static double urand(uint64_t* s) { return (double)(splitmix(s) >> 11) * (1.0 / 9007199254740992.0); }
static double urange(uint64_t* s, double a, double b) { return a + (b - a) * urand(s); }

static uint32_t hash3(int32_t i, int32_t j, uint32_t k) {
    uint32_t h = (uint32_t)i * 0x8da6b343u ^ (uint32_t)j * 0xd8163841u ^ k * 0xcb1ab31fu;
    h ^= h >> 13;
    h *= 0x5bd1e995u;
    h ^= h >> 15;
    return h;
}
static double lattice(int32_t i, int32_t j, uint32_t k) { return (hash3(i, j, k) & 0xffffff) / 16777215.0; }
static double smooth(double t) { return t * t * (3.0 - 2.0 * t); }

static double value_noise(double u, double v, uint32_t k) {
    const double fu = floor(u), fv = floor(v);
    const int32_t i = (int32_t)fu, j = (int32_t)fv;
    const double a = smooth(u - fu), b = smooth(v - fv);
    const double v00 = lattice(i, j, k), v10 = lattice(i + 1, j, k);
    const double v01 = lattice(i, j + 1, k), v11 = lattice(i + 1, j + 1, k);
    return (v00 + (v10 - v00) * a) + ((v01 + (v11 - v01) * a) - (v00 + (v10 - v00) * a)) * b;
}

/* 4 octaves, each faded out when its cell is below ~1.5 pixel footprints. */
static double texture(double u, double v, double cell, double footprint, uint32_t id) {
    double sum = 0.0, norm = 0.0, amp = 1.0;
    for (int o = 0; o < 4; ++o) {
        const double c = cell / (double)(1 << o);
        double fade = (c / footprint - 1.5) / 1.5;
        fade = fade < 0.0 ? 0.0 : (fade > 1.0 ? 1.0 : fade);
        sum += amp * fade * (value_noise(u / c, v / c, id * 8u + (uint32_t)o) - 0.5);
        norm += amp;
        amp *= 0.6;
    }
    return sum / norm; /* roughly in [-0.5, 0.5] */
}

static void make_poses(scene_t* s) {
    const tsgm_scene_cfg* c = &s->cfg;
    double px = 0.0, pz = 0.0, yaw = 0.0;
    const double dyaw = c->yaw_deg * M_PI / 180.0;
    for (int k = 0; k < c->frames; ++k) {
        double* P = s->poses + 12 * k;
        const double cy = cos(yaw), sy = sin(yaw);
        /* rotation about Y: camera-to-world */
        P[0] = cy;  P[1] = 0.0; P[2] = sy;  P[3] = px;
        P[4] = 0.0; P[5] = 1.0; P[6] = 0.0; P[7] = 0.0;
        P[8] = -sy; P[9] = 0.0; P[10] = cy; P[11] = pz;
        px += sy * c->fwd_m;
        pz += cy * c->fwd_m;
        yaw += dyaw;
    }
}

static void make_scene(scene_t* s) {
    const tsgm_scene_cfg* c = &s->cfg;
    uint64_t rng = c->seed * 0x2545f4914f6cdd1dull + 12345u;
    const double fb = c->focal * c->baseline;
    s->cam_height = 1.65;
    s->wall_z = fb / 5.0; /* background disparity 5 at frame 0 */
    s->n_rects = 0;
    const int total = c->n_static + c->n_movers;
    /* The camera advances fwd_m per frame; every object is placed so that its
     * disparity on the LAST frame lies in [10, 0.75 d_max] (never closer than
     * the matcher can see), which puts frame-0 disparities at 5 and up. */
    const double travel = c->fwd_m * (c->frames - 1);
    for (int r = 0; r < total && r < MAX_RECTS; ++r) {
        rect_t* R = &s->rects[s->n_rects++];
        const int mover = r >= c->n_static;
        const double d_final = urange(&rng, 10.0, 0.75 * c->d_max);
        double z = travel + fb / d_final;
        if (z > s->wall_z - 1.0) z = s->wall_z - 1.0;
        const double disp = fb / z;
        (void)disp;
        /* keep it on screen at frame 0: pick its image-space centre column */
        const double xc_px = urange(&rng, 0.1 * c->width, 0.9 * c->width);
        const double xc = (xc_px - c->cx) * z / c->focal;
        double wm, hm;
        if (mover && c->mover_max_frac > 0.0) {
            /* occluders covering up to mover_max_frac of the image */
            const double frac = urange(&rng, 0.3, 1.0) * c->mover_max_frac;
            const double wpx = sqrt(frac) * c->width * 0.8, hpx = sqrt(frac) * c->height * 1.2;
            wm = wpx * z / c->focal;
            hm = hpx * z / c->focal;
        } else {
            wm = urange(&rng, 1.0, 6.0);
            hm = urange(&rng, 1.0, 4.0);
        }
        R->x0 = xc - 0.5 * wm;
        R->x1 = xc + 0.5 * wm;
        R->y1 = s->cam_height;
        R->y0 = s->cam_height - hm;
        R->z = z;
        R->cell = 10.0 * z / c->focal; /* ~10 px base cell at frame 0 */
        R->tex_id = 16u + (uint32_t)r + (uint32_t)(c->seed * 131u);
        R->vx = R->vz = 0.0;
        if (mover) {
            /* lateral translation, random side, up to ~20 deg off the X axis */
            const double speed = urange(&rng, c->mover_speed_min, c->mover_speed_max);
            const double ang = urange(&rng, -0.35, 0.35) + (urand(&rng) < 0.5 ? M_PI : 0.0);
            R->vx = speed * cos(ang);
            R->vz = speed * sin(ang);
            /* keep the final-frame depth where it was planned */
            R->z -= R->vz * (c->frames - 1);
            if (R->z > s->wall_z - 1.0) R->z = s->wall_z - 1.0;
        }
    }
    for (int k = 0; k < c->frames; ++k) {
        const double g = c->gain_jitter > 0.0 ? urange(&rng, 1.0 - c->gain_jitter, 1.0 + c->gain_jitter) : 1.0;
        s->gains[2 * k] = g;
        s->gains[2 * k + 1] = g;
    }
}

/* Cast one ray; returns intensity in [0,1] and camera depth. */
static double shade(const scene_t* s, int k, double ox, double oy, double oz, double dx, double dy,
                    double dz, double* depth) {
    const tsgm_scene_cfg* c = &s->cfg;
    double best_t = 1e30, val = 0.5;
    /* far wall (world Z = wall_z) */
    if (dz > 1e-9) {
        const double t = (s->wall_z - oz) / dz;
        if (t > 0.0 && t < best_t) {
            best_t = t;
            const double X = ox + t * dx, Y = oy + t * dy;
            val = 0.5 + texture(X, Y, 10.0 * s->wall_z / c->focal, t / c->focal, 7u + (uint32_t)c->seed * 977u);
        }
    }
    /* ground (world Y = cam_height) */
    if (dy > 1e-9) {
        const double t = (s->cam_height - oy) / dy;
        if (t > 0.0 && t < best_t) {
            best_t = t;
            const double X = ox + t * dx, Z = oz + t * dz;
            /* the ground is seen at a grazing angle: footprint ~ t^2/(f*h) */
            const double fp = t * t / (c->focal * s->cam_height);
            val = 0.5 + 0.9 * texture(X, Z, 1.2, fp > t / c->focal ? fp : t / c->focal, 3u + (uint32_t)c->seed * 613u);
        }
    }
    for (int r = 0; r < s->n_rects; ++r) {
        const rect_t* R = &s->rects[r];
        const double rz = R->z + k * R->vz, sx = k * R->vx;
        if (!(dz > 1e-9)) continue;
        const double t = (rz - oz) / dz;
        if (!(t > 0.0 && t < best_t)) continue;
        const double X = ox + t * dx - sx, Y = oy + t * dy;
        if (X < R->x0 || X > R->x1 || Y < R->y0 || Y > R->y1) continue;
        best_t = t;
        val = 0.5 + texture(X - R->x0, Y, R->cell, t / c->focal, R->tex_id);
    }
    *depth = best_t; /* == camera Z for unit-z camera rays */
    return val;
}

typedef struct {
    const scene_t* s;
    int frame_begin, frame_end;
    uint8_t *left, *right;
    float* gt;
    int row_begin, row_end;
} job_t;

static double gauss(uint64_t* st) {
    double u1 = urand(st), u2 = urand(st);
    if (u1 < 1e-300) u1 = 1e-300;
    return sqrt(-2.0 * log(u1)) * cos(2.0 * M_PI * u2);
}

static void* render_rows(void* arg) {
    job_t* j = (job_t*)arg;
    const scene_t* s = j->s;
    const tsgm_scene_cfg* c = &s->cfg;
    const int w = c->width, h = c->height;
    for (int k = j->frame_begin; k < j->frame_end; ++k) {
        const double* P = s->poses + 12 * k;
        const size_t base = (size_t)(k - j->frame_begin) * w * h;
        for (int y = j->row_begin; y < j->row_end; ++y) {
            uint64_t st = c->seed * 0x9e3779b97f4a7c15ull ^ ((uint64_t)k << 40) ^ ((uint64_t)y << 20) ^ 0xabcdefull;
            for (int x = 0; x < w; ++x) {
                const double rx = (x - c->cx) / c->focal, ry = (y - c->cy) / c->focal;
                const double dx = P[0] * rx + P[1] * ry + P[2];
                const double dy = P[4] * rx + P[5] * ry + P[6];
                const double dz = P[8] * rx + P[9] * ry + P[10];
                for (int cam = 0; cam < 2; ++cam) {
                    /* right camera sits +baseline along the camera X axis */
                    const double off = cam ? c->baseline : 0.0;
                    const double ox = P[3] + P[0] * off, oy = P[7] + P[4] * off, oz = P[11] + P[8] * off;
                    double depth;
                    const double v = shade(s, k, ox, oy, oz, dx, dy, dz, &depth);
                    double I = (30.0 + 195.0 * v) * s->gains[2 * k + cam] + c->noise_sigma * gauss(&st);
                    I = I < 0.0 ? 0.0 : (I > 255.0 ? 255.0 : I);
                    const uint8_t u = (uint8_t)(I + 0.5);
                    if (cam == 0) {
                        j->left[base + (size_t)y * w + x] = u;
                        if (j->gt) j->gt[base + (size_t)y * w + x] = (float)(c->focal * c->baseline / depth);
                    } else {
                        j->right[base + (size_t)y * w + x] = u;
                    }
                }
            }
        }
    }
    return NULL;
}

void tsgm_scene_default(tsgm_scene_cfg* c, int config) {
    memset(c, 0, sizeof *c);
    c->width = 1242;
    c->height = 375;
    c->d_max = 128;
    c->focal = 720.0;
    c->cx = 621.0;
    c->cy = 187.5;
    c->baseline = 0.54;
    c->frames = 8;
    c->seed = 0;
    c->n_static = 6;
    c->n_movers = 0;
    c->fwd_m = 0.8;
    c->yaw_deg = 0.5;
    c->mover_speed_min = 0.5;
    c->mover_speed_max = 1.5;
    c->noise_sigma = 2.0;
    switch (config) {
        case 1:
        case 3:
            c->frames = 30;
            c->n_movers = config == 1 ? 3 : 0;
            break;
        case 2:
            c->frames = 30;
            c->n_movers = 2; /* bench overrides per seed: 0-4 */
            break;
        case 4:
            c->width = 2048;
            c->height = 1024;
            c->d_max = 256;
            c->focal = 1100.0;
            c->cx = 1023.5;
            c->cy = 511.5;
            c->baseline = 0.54;
            c->frames = 20;
            c->n_movers = 3;
            c->gain_jitter = 0.10;
            c->mover_max_frac = 0.30;
            break;
        default:
            break;
    }
}

int tsgm_scene_render(const tsgm_scene_cfg* cfg, int frame_begin, int frame_end, uint8_t* left,
                      uint8_t* right, float* gt_disp, double* poses12, int threads) {
    if (!cfg || cfg->width < 5 || cfg->height < 5 || cfg->frames < 1 || frame_begin < 0 ||
        frame_end > cfg->frames || frame_begin > frame_end || cfg->n_static + cfg->n_movers > MAX_RECTS)
        return 1;
    scene_t s;
    s.cfg = *cfg;
    s.poses = (double*)malloc(sizeof(double) * 12 * cfg->frames);
    s.gains = (double*)malloc(sizeof(double) * 2 * cfg->frames);
    make_poses(&s);
    make_scene(&s);
    if (poses12) memcpy(poses12, s.poses, sizeof(double) * 12 * cfg->frames);
    if (left && right && frame_end > frame_begin) {
        if (threads < 1) threads = 1;
        if (threads > cfg->height) threads = cfg->height;
        pthread_t* tid = (pthread_t*)malloc(sizeof(pthread_t) * threads);
        job_t* jobs = (job_t*)malloc(sizeof(job_t) * threads);
        const int chunk = (cfg->height + threads - 1) / threads;
        for (int t = 0; t < threads; ++t) {
            jobs[t] = (job_t){&s, frame_begin, frame_end, left, right, gt_disp, t * chunk,
                              (t + 1) * chunk < cfg->height ? (t + 1) * chunk : cfg->height};
            pthread_create(&tid[t], NULL, render_rows, &jobs[t]);
        }
        for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
        free(tid);
        free(jobs);
    }
    free(s.poses);
    free(s.gains);
    return 0;
}
