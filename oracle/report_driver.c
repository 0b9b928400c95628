/* TEST INFRASTRUCTURE ONLY: runs the reference's write_calib_report
 * (through ref_calib_report, oracle/ref_runner.cpp) in its own process — the
 * reference's iostreams crash when libtsgm_ref.so is loaded into Python.
 * Usage: report_driver <inputs.bin> <report.txt>; inputs.bin holds
 * int32 n, w, h, cw, ch, d_max, sgm[5]; f64 calib4[4], opts3[3]; then
 * u8 left[n*w*h], u8 right[n*w*h], f64 gt[n*w*h], f64 poses[12*n]. */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

int ref_calib_report(const char* path, int n, int w, int h, const uint8_t* left,
                     const uint8_t* right, const double* gt, const double* poses,
                     const double* calib4, int cw, int ch, int d_max, const int* sgm_params,
                     const double* opts3);
const char* ref_last_error(void);

int main(int argc, char** argv) {
    if (argc != 3) return 2;
    FILE* f = fopen(argv[1], "rb");
    if (!f) return 2;
    int32_t hd[11];
    double c4[4], o3[3];
    if (fread(hd, 4, 11, f) != 11 || fread(c4, 8, 4, f) != 4 || fread(o3, 8, 3, f) != 3) return 2;
    const size_t P = (size_t)hd[0] * hd[1] * hd[2];
    uint8_t* l = malloc(P);
    uint8_t* r = malloc(P);
    double* g = malloc(8 * P);
    double* ps = malloc(8 * 12 * (size_t)hd[0]);
    if (fread(l, 1, P, f) != P || fread(r, 1, P, f) != P || fread(g, 8, P, f) != P ||
        fread(ps, 8, 12 * (size_t)hd[0], f) != 12 * (size_t)hd[0])
        return 2;
    fclose(f);
    const int rc = ref_calib_report(argv[2], hd[0], hd[1], hd[2], l, r, g, ps, c4, hd[3], hd[4],
                                    hd[5], hd + 6, o3);
    if (rc) fprintf(stderr, "%s\n", ref_last_error());
    return rc;
}
