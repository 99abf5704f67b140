/*
 * glu_oracle.h -- CPU ORACLE for the Guided Linear Upsampling hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This header and glu_oracle.c restate, in plain
 * C (IEEE double, -ffp-contract=off), the reference algorithm of
 * /root/reference/proj/src/{grid,upsample,jointopt}.cpp so that the CUDA
 * product path can be checked bit for bit.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load it; the product library never links
 * or calls it.
 *
 * Parity of this restatement is PINNED two ways (see tests/test_oracle.py):
 *   1. against golden vectors produced by the reference library itself,
 *      compiled from /root/reference sources into oracle/_ref/ by
 *      oracle/Makefile (tests/golden/make_golden.py), and
 *   2. against the known-answer values of the reference unit tests
 *      (proj/tests/unit/{upsample,jointopt,grid}_test.cpp).
 */
#ifndef GLU_ORACLE_H
#define GLU_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* 12-byte record, same layout as glu::PixelParams (params.hpp:42-46). */
typedef struct {
    uint32_t a;
    uint32_t b;
    float w;
} glu_o_params;

enum { GLU_O_FAST = 0, GLU_O_EXACT = 1, GLU_O_GNU = 2 };

/* Scalar helpers (upsample.cpp:158-176). Colours are 3 floats. */
double glu_o_weight_exact(const float* ip, const float* ia, const float* ib, double eps);
double glu_o_weight_fast(const float* ip, const float* ia, const float* ib, double eps);
double glu_o_pair_objective(const float* ip, const float* ia, const float* ib, double w,
                            double eps);
/* Candidate list: n entries of (index, rgb).  Returns 0, or -1 if n == 0. */
int glu_o_optimize_pixel(const float* ip, const uint32_t* idx, const float* rgb, size_t n,
                         double eps, int mode, glu_o_params* out);

/* grid.cpp:8-23 ceil-div geometry; returns 0 or -1 on invalid arguments. */
int glu_o_grid_dims(int W, int H, int s, int* lowW, int* lowH);
/* grid.cpp:41-52: centre-pixel point sampling.  low: lowW*lowH*3 floats. */
int glu_o_grid_downsample(const float* high, int W, int H, int s, float* low);

/* upsample.cpp:194-216 for every HR pixel (S = window side, odd >= 3). */
int glu_o_optimize_field(const float* high, int W, int H, const float* low, int s, int S,
                         double eps, int mode, glu_o_params* out);
/* upsample.cpp:218-233: the listed pixels only, in list order, in place. */
int glu_o_optimize_pixels(const float* high, int W, int H, const float* low, int s, int S,
                          double eps, int mode, const uint32_t* pixels, size_t n,
                          glu_o_params* field);
/* upsample.cpp:235-252 + upsample.hpp:54-65; channels 3 (reference) or 1
 * (single-channel extension, same per-channel expression). */
int glu_o_apply_field(const glu_o_params* field, int W, int H, const float* lowT, int lowW,
                      int lowH, int channels, int clampOutput, float* out);
/* upsample.cpp:254-267 + upsample.hpp:67-74. */
void glu_o_error_map(const float* high, const float* recon, size_t npx, float* e);

/* jointopt.cpp:9-46.  Writes mask (W*H bytes), and components in CSR form:
 * comp_off[0..ncomp], comp_px[0..comp_off[ncomp]).  Capacities: W*H+1 and W*H.
 * Returns the component count, or -1 on an empty map. */
long glu_o_find_large_error(const float* e, int W, int H, float threshold, uint8_t* mask,
                            uint32_t* comp_off, uint32_t* comp_px);

/* jointopt.cpp:114-180.  Returns 1 accepted, 0 rejected, -1 invalid. */
int glu_o_trial_update_component(const float* high, int W, int H, float* low, int s, int S,
                                 double eps, int mode, int literal, glu_o_params* field,
                                 float* errors, const uint32_t* comp, size_t n);

/* jointopt.cpp:182-206.  Outputs low (lowW*lowH*3), field, errors (W*H) and
 * counters {iterations, accepted, rejected}. */
int glu_o_joint_optimize(const float* high, int W, int H, int s, int S, float threshold,
                         int maxIterations, double eps, int mode, int literal, float* low,
                         glu_o_params* field, float* errors, int* counters);

#ifdef __cplusplus
}
#endif

#endif
