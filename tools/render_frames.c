/* render_frames — writes seeded synthetic stereo sequences to a raw file.
 *
 * Input generation for the reference arm of bench.py (--impl reference): the
 * reference process must not map any library of the product package, so the
 * frames come from this separate, non-Python process (built from the same
 * scene.c as paper_1809_07986_b200/lib/libtsgm_scene.so, so the frames are the
 * ones the GPU arm renders).
 *
 *   render_frames <config> <seed_begin> <seed_end> <frames> <out>
 *
 * For each seed s in [seed_begin, seed_end): BASELINE config <config> with
 * seed s and (s % 5) movers (bench.py's config-2 convention), <frames> frames.
 * Output per seed: left u8 [frames][H][W], right u8 [frames][H][W], poses f64
 * [frames][12] (camera-to-world 3x4, row-major). Exit 0 on success. */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <unistd.h>

#include "tsgm_scene.h"

int main(int argc, char** argv) {
    if (argc != 6) {
        fprintf(stderr, "usage: %s config seed_begin seed_end frames out\n", argv[0]);
        return 2;
    }
    const int config = atoi(argv[1]);
    const long s0 = atol(argv[2]), s1 = atol(argv[3]);
    const int frames = atoi(argv[4]);
    FILE* f = fopen(argv[5], "wb");
    if (!f || frames < 1 || s1 < s0) {
        fprintf(stderr, "render_frames: bad arguments\n");
        return 2;
    }
    long threads = sysconf(_SC_NPROCESSORS_ONLN);
    if (threads < 1) threads = 1;
    for (long s = s0; s < s1; ++s) {
        tsgm_scene_cfg c;
        tsgm_scene_default(&c, config);
        c.seed = (uint64_t)s;
        c.n_movers = (int)(s % 5);
        c.frames = frames;
        const size_t P = (size_t)c.width * c.height;
        uint8_t* l = malloc(P * frames);
        uint8_t* r = malloc(P * frames);
        double* poses = malloc(sizeof(double) * 12 * frames);
        if (!l || !r || !poses) return 3;
        if (tsgm_scene_render(&c, 0, frames, l, r, NULL, poses, (int)threads) != 0) return 4;
        if (fwrite(l, 1, P * frames, f) != P * frames || fwrite(r, 1, P * frames, f) != P * frames ||
            fwrite(poses, sizeof(double), 12 * (size_t)frames, f) != 12 * (size_t)frames)
            return 5;
        free(l);
        free(r);
        free(poses);
    }
    return fclose(f) == 0 ? 0 : 5;
}
