/* Synthetic stereo sequence generator (input generation for tests/bench; not
 * part of the hot path). See paper_1809_07986_b200/csrc/scene.c. */
#ifndef TSGM_SCENE_H
#define TSGM_SCENE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int width, height, d_max;
    double focal, cx, cy, baseline;
    int frames;
    uint64_t seed;
    int n_static, n_movers;
    double fwd_m, yaw_deg;
    double mover_speed_min, mover_speed_max;
    double gain_jitter;     /* per-frame global gain in [1-g, 1+g] */
    double mover_max_frac;  /* >0: movers are occluders covering up to this image fraction */
    double noise_sigma;
} tsgm_scene_cfg;

/* Fill *cfg with BASELINE.json config `config` (0-4) defaults. */
void tsgm_scene_default(tsgm_scene_cfg* cfg, int config);

/* Render frames [frame_begin, frame_end) into left/right (frame-major u8,
 * W*H each); gt_disp (optional, f32) receives the true left disparity;
 * poses12 (optional) receives all cfg->frames camera-to-world 3x4 poses.
 * Returns 0, or 1 on invalid arguments. Deterministic in cfg (any thread count). */
int tsgm_scene_render(const tsgm_scene_cfg* cfg, int frame_begin, int frame_end, uint8_t* left,
                      uint8_t* right, float* gt_disp, double* poses12, int threads);

#ifdef __cplusplus
}
#endif
#endif
