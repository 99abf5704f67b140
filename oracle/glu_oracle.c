/*
 * glu_oracle.c -- CPU ORACLE (test infrastructure only; see glu_oracle.h).
 *
 * Plain C restatement of the reference hot path.  Every function cites the
 * reference file:line it follows.  Build with -ffp-contract=off (the reference
 * does, proj/CMakeLists.txt:15-18): each double expression below is evaluated
 * in exactly the reference's operation order, so results are bit-identical.
 */
#include "glu_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---- per-pixel maths (upsample.cpp:28-42) ---------------------------------- */

/* dist(p, q): upsample.cpp:28-33 */
static double o_dist(const float* p, const float* q) {
    const double d0 = (double)p[0] - (double)q[0];
    const double d1 = (double)p[1] - (double)q[1];
    const double d2 = (double)p[2] - (double)q[2];
    return sqrt(d0 * d0 + d1 * d1 + d2 * d2);
}

/* objective(ip, ia, ib, w, eps): upsample.cpp:35-42 */
static double o_objective(const float* ip, const float* ia, const float* ib, double w,
                          double eps) {
    double r = 0;
    for (int c = 0; c < 3; ++c) {
        const double v = w * (double)ia[c] + (1.0 - w) * (double)ib[c] - (double)ip[c];
        r += v * v;
    }
    return r + eps * w * w;
}

/* weight_exact: upsample.cpp:158-167 */
double glu_o_weight_exact(const float* ip, const float* ia, const float* ib, double eps) {
    double num = 0, den = 0;
    for (int c = 0; c < 3; ++c) {
        const double pb = (double)ip[c] - (double)ib[c];
        const double ab = (double)ia[c] - (double)ib[c];
        num += pb * ab;
        den += ab * ab;
    }
    return num / (den + eps);
}

/* weight_fast: upsample.cpp:169-172 */
double glu_o_weight_fast(const float* ip, const float* ia, const float* ib, double eps) {
    const double db = o_dist(ip, ib);
    return db / (o_dist(ip, ia) + db + eps);
}

/* pair_objective: upsample.cpp:174-176 */
double glu_o_pair_objective(const float* ip, const float* ia, const float* ib, double w,
                            double eps) {
    return o_objective(ip, ia, ib, w, eps);
}

/* pixelFast: upsample.cpp:49-71.  a = first strict argmin of distance; b =
 * first strict argmin of the objective with w_j = d_j / (d_a + d_j + eps). */
static glu_o_params o_pixel_fast(const float* ip, const uint32_t* idx, const float* rgb,
                                 size_t n, double eps, double* scratch) {
    size_t ai = 0;
    for (size_t i = 0; i < n; ++i) {
        scratch[i] = o_dist(ip, rgb + 3 * i);
        if (scratch[i] < scratch[ai]) ai = i;
    }
    const float* ia = rgb + 3 * ai;
    const double da = scratch[ai];
    size_t bi = 0;
    double bestW = 0, bestObj = 0;
    int first = 1;
    for (size_t j = 0; j < n; ++j) {
        const double w = scratch[j] / (da + scratch[j] + eps);
        const double obj = o_objective(ip, ia, rgb + 3 * j, w, eps);
        if (first || obj < bestObj) {
            first = 0;
            bestObj = obj;
            bestW = w;
            bi = j;
        }
    }
    glu_o_params r = {idx[ai], idx[bi], (float)bestW};
    return r;
}

/* pixelExact: upsample.cpp:73-91.  Unordered pairs i <= j, lexicographic. */
static glu_o_params o_pixel_exact(const float* ip, const uint32_t* idx, const float* rgb,
                                  size_t n, double eps) {
    size_t ai = 0, bi = 0;
    double bestW = 0, bestObj = 0;
    int first = 1;
    for (size_t i = 0; i < n; ++i) {
        for (size_t j = i; j < n; ++j) {
            const double w = glu_o_weight_exact(ip, rgb + 3 * i, rgb + 3 * j, eps);
            const double obj = o_objective(ip, rgb + 3 * i, rgb + 3 * j, w, eps);
            if (first || obj < bestObj) {
                first = 0;
                bestObj = obj;
                bestW = w;
                ai = i;
                bi = j;
            }
        }
    }
    glu_o_params r = {idx[ai], idx[bi], (float)bestW};
    return r;
}

/* pixelGnu: upsample.cpp:93-104 */
static glu_o_params o_pixel_gnu(const float* ip, const uint32_t* idx, const float* rgb,
                                size_t n) {
    size_t ai = 0;
    double best = o_dist(ip, rgb);
    for (size_t i = 1; i < n; ++i) {
        const double d = o_dist(ip, rgb + 3 * i);
        if (d < best) {
            best = d;
            ai = i;
        }
    }
    glu_o_params r = {idx[ai], idx[ai], 1.0f};
    return r;
}

static glu_o_params o_dispatch(const float* ip, const uint32_t* idx, const float* rgb,
                               size_t n, double eps, int mode, double* scratch) {
    switch (mode) {
        case GLU_O_EXACT: return o_pixel_exact(ip, idx, rgb, n, eps);
        case GLU_O_GNU: return o_pixel_gnu(ip, idx, rgb, n);
        default: return o_pixel_fast(ip, idx, rgb, n, eps, scratch);
    }
}

int glu_o_optimize_pixel(const float* ip, const uint32_t* idx, const float* rgb, size_t n,
                         double eps, int mode, glu_o_params* out) {
    if (n == 0) return -1; /* requireCandidates, upsample.cpp:44-46 */
    double* scratch = (double*)malloc(n * sizeof(double));
    *out = o_dispatch(ip, idx, rgb, n, eps, mode, scratch);
    free(scratch);
    return 0;
}

/* ---- grid geometry (grid.cpp:8-52) ---------------------------------------- */

int glu_o_grid_dims(int W, int H, int s, int* lowW, int* lowH) {
    if (W <= 0 || H <= 0 || s < 2 || s >= (W < H ? W : H)) return -1; /* grid.cpp:9-14 */
    *lowW = (W + s - 1) / s;
    *lowH = (H + s - 1) / s;
    return 0;
}

int glu_o_grid_downsample(const float* high, int W, int H, int s, float* low) {
    int lw, lh;
    if (glu_o_grid_dims(W, H, s, &lw, &lh)) return -1;
    const int off = s / 2;
    for (int cy = 0; cy < lh; ++cy)
        for (int cx = 0; cx < lw; ++cx) {
            int x = cx * s + off, y = cy * s + off; /* sampleCoord, grid.cpp:25-28 */
            if (x > W - 1) x = W - 1;
            if (y > H - 1) y = H - 1;
            memcpy(low + 3 * ((size_t)cy * lw + cx), high + 3 * ((size_t)y * W + x),
                   3 * sizeof(float));
        }
    return 0;
}

/* gatherWindow + windowBounds (upsample.cpp:136-145, grid.cpp:30-39):
 * cells of the truncated SxS window, cy outer, cx inner. */
static size_t o_gather(const float* low, int lw, int lh, int cx, int cy, int S, uint32_t* idx,
                       float* rgb) {
    const int h = S / 2;
    const int x0 = cx - h < 0 ? 0 : cx - h, y0 = cy - h < 0 ? 0 : cy - h;
    const int x1 = cx + h > lw - 1 ? lw - 1 : cx + h, y1 = cy + h > lh - 1 ? lh - 1 : cy + h;
    size_t n = 0;
    for (int y = y0; y <= y1; ++y)
        for (int x = x0; x <= x1; ++x) {
            idx[n] = (uint32_t)y * (uint32_t)lw + (uint32_t)x;
            memcpy(rgb + 3 * n, low + 3 * (size_t)idx[n], 3 * sizeof(float));
            ++n;
        }
    return n;
}

static int o_check(int W, int H, int s, int S, double eps) {
    int lw, lh;
    if (S < 3 || S % 2 == 0 || !(eps > 0)) return -1; /* GluConfig::validate, params.hpp:30-38 */
    return glu_o_grid_dims(W, H, s, &lw, &lh);
}

/* optimize_field: upsample.cpp:194-216 */
int glu_o_optimize_field(const float* high, int W, int H, const float* low, int s, int S,
                         double eps, int mode, glu_o_params* out) {
    if (o_check(W, H, s, S, eps)) return -1;
    const int lw = (W + s - 1) / s, lh = (H + s - 1) / s;
    const size_t cap = (size_t)S * S;
    uint32_t* idx = (uint32_t*)malloc(cap * sizeof(uint32_t));
    float* rgb = (float*)malloc(cap * 3 * sizeof(float));
    double* scratch = (double*)malloc(cap * sizeof(double));
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            const size_t n = o_gather(low, lw, lh, x / s, y / s, S, idx, rgb);
            out[(size_t)y * W + x] =
                o_dispatch(high + 3 * ((size_t)y * W + x), idx, rgb, n, eps, mode, scratch);
        }
    free(idx);
    free(rgb);
    free(scratch);
    return 0;
}

/* optimize_pixels: upsample.cpp:218-233 */
int glu_o_optimize_pixels(const float* high, int W, int H, const float* low, int s, int S,
                          double eps, int mode, const uint32_t* pixels, size_t n,
                          glu_o_params* field) {
    if (o_check(W, H, s, S, eps)) return -1;
    const int lw = (W + s - 1) / s, lh = (H + s - 1) / s;
    const size_t cap = (size_t)S * S;
    uint32_t* idx = (uint32_t*)malloc(cap * sizeof(uint32_t));
    float* rgb = (float*)malloc(cap * 3 * sizeof(float));
    double* scratch = (double*)malloc(cap * sizeof(double));
    for (size_t k = 0; k < n; ++k) {
        const uint32_t p = pixels[k];
        const int x = (int)(p % (uint32_t)W), y = (int)(p / (uint32_t)W);
        const size_t m = o_gather(low, lw, lh, x / s, y / s, S, idx, rgb);
        field[p] = o_dispatch(high + 3 * (size_t)p, idx, rgb, m, eps, mode, scratch);
    }
    free(idx);
    free(rgb);
    free(scratch);
    return 0;
}

/* reconstruct_pixel: upsample.hpp:54-65 (float maths, no contraction). */
static void o_reconstruct(const glu_o_params* pp, const float* lowT, int channels, int clamp,
                          float* o) {
    const float* la = lowT + (size_t)channels * pp->a;
    const float* lb = lowT + (size_t)channels * pp->b;
    for (int c = 0; c < channels; ++c) {
        float v = pp->w * la[c] + (1.0f - pp->w) * lb[c];
        if (clamp) v = v < 0.0f ? 0.0f : (v > 1.0f ? 1.0f : v);
        o[c] = v;
    }
}

/* apply_field: upsample.cpp:235-252 */
int glu_o_apply_field(const glu_o_params* field, int W, int H, const float* lowT, int lowW,
                      int lowH, int channels, int clampOutput, float* out) {
    (void)lowH;
    (void)lowW;
    if (channels != 1 && channels != 3) return -1;
    const size_t npx = (size_t)W * H;
    for (size_t p = 0; p < npx; ++p)
        o_reconstruct(field + p, lowT, channels, clampOutput, out + (size_t)channels * p);
    return 0;
}

/* pixel_error: upsample.hpp:67-74 */
static float o_pixel_error(const float* t, const float* r) {
    double s = 0;
    for (int c = 0; c < 3; ++c) {
        const double d = (double)t[c] - (double)r[c];
        s += d * d;
    }
    return (float)sqrt(s);
}

/* error_map: upsample.cpp:254-267 */
void glu_o_error_map(const float* high, const float* recon, size_t npx, float* e) {
    for (size_t p = 0; p < npx; ++p) e[p] = o_pixel_error(high + 3 * p, recon + 3 * p);
}

/* ---- joint optimisation (jointopt.cpp) ------------------------------------- */

static int cmp_u32(const void* a, const void* b) {
    const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return x < y ? -1 : (x > y);
}

static int cmp_u64(const void* a, const void* b) {
    const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
    return x < y ? -1 : (x > y);
}

/* find_large_error: jointopt.cpp:9-46.  Strict '>' mask, iterative DFS over
 * 4-neighbours (left, right, up, down pushed in that order), components in
 * raster order of their first pixel, each pixel list sorted ascending. */
long glu_o_find_large_error(const float* e, int W, int H, float threshold, uint8_t* mask,
                            uint32_t* comp_off, uint32_t* comp_px) {
    if (W <= 0 || H <= 0) return -1;
    const size_t npx = (size_t)W * H;
    for (size_t i = 0; i < npx; ++i) mask[i] = e[i] > threshold;
    uint8_t* seen = (uint8_t*)calloc(npx, 1);
    uint32_t* stack = (uint32_t*)malloc(npx * sizeof(uint32_t));
    size_t top = 0, used = 0;
    long ncomp = 0;
    comp_off[0] = 0;
    for (size_t start = 0; start < npx; ++start) {
        if (!mask[start] || seen[start]) continue;
        const size_t begin = used;
        stack[top++] = (uint32_t)start;
        seen[start] = 1;
        while (top) {
            const uint32_t p = stack[--top];
            comp_px[used++] = p;
            const int x = (int)(p % (uint32_t)W), y = (int)(p / (uint32_t)W);
            const int nb[4][2] = {{x - 1, y}, {x + 1, y}, {x, y - 1}, {x, y + 1}};
            for (int k = 0; k < 4; ++k) {
                if (nb[k][0] < 0 || nb[k][0] >= W || nb[k][1] < 0 || nb[k][1] >= H) continue;
                const uint32_t q = (uint32_t)nb[k][1] * (uint32_t)W + (uint32_t)nb[k][0];
                if (mask[q] && !seen[q]) {
                    seen[q] = 1;
                    stack[top++] = q;
                }
            }
        }
        qsort(comp_px + begin, used - begin, sizeof(uint32_t), cmp_u32);
        comp_off[++ncomp] = (uint32_t)used;
    }
    free(seen);
    free(stack);
    return ncomp;
}

/* trial_update_component: jointopt.cpp:114-180, with groupByOwnerCell
 * (56-72) and affectedPixels (76-110). */
int glu_o_trial_update_component(const float* high, int W, int H, float* low, int s, int S,
                                 double eps, int mode, int literal, glu_o_params* field,
                                 float* errors, const uint32_t* comp, size_t n) {
    if (o_check(W, H, s, S, eps) || n == 0) return -1;
    const int lw = (W + s - 1) / s, lh = (H + s - 1) / s;
    const int h = S / 2;

    /* groupByOwnerCell: sort (cell, pixel) pairs. */
    uint64_t* pairs = (uint64_t*)malloc(n * sizeof(uint64_t));
    for (size_t k = 0; k < n; ++k) {
        const uint32_t p = comp[k];
        const uint32_t cell =
            (p / (uint32_t)W / (uint32_t)s) * (uint32_t)lw + (p % (uint32_t)W) / (uint32_t)s;
        pairs[k] = ((uint64_t)cell << 32) | p;
    }
    qsort(pairs, n, sizeof(uint64_t), cmp_u64);
    uint32_t* gcell = (uint32_t*)malloc(n * sizeof(uint32_t));
    size_t ng = 0;
    float* oldColors = (float*)malloc(n * 3 * sizeof(float));
    /* Replace each cell by its worst pixel (first strict argmax, 130-142). */
    for (size_t k = 0; k < n;) {
        const uint32_t cell = (uint32_t)(pairs[k] >> 32);
        uint32_t best = (uint32_t)pairs[k];
        size_t m = k;
        for (; m < n && (uint32_t)(pairs[m] >> 32) == cell; ++m) {
            const uint32_t p = (uint32_t)pairs[m];
            if (errors[p] > errors[best]) best = p;
        }
        gcell[ng] = cell;
        memcpy(oldColors + 3 * ng, low + 3 * (size_t)cell, 3 * sizeof(float));
        memcpy(low + 3 * (size_t)cell, high + 3 * (size_t)best, 3 * sizeof(float));
        ++ng;
        k = m;
    }

    /* Affected set. */
    uint32_t* affected;
    size_t na = 0;
    if (literal) {
        affected = (uint32_t*)malloc(n * sizeof(uint32_t));
        memcpy(affected, comp, n * sizeof(uint32_t));
        na = n;
    } else {
        int bx0 = lw, by0 = lh, bx1 = -1, by1 = -1;
        for (size_t g = 0; g < ng; ++g) {
            const int cx = (int)(gcell[g] % (uint32_t)lw), cy = (int)(gcell[g] / (uint32_t)lw);
            if (cx < bx0) bx0 = cx;
            if (cy < by0) by0 = cy;
            if (cx > bx1) bx1 = cx;
            if (cy > by1) by1 = cy;
        }
        bx0 = bx0 - h < 0 ? 0 : bx0 - h;
        by0 = by0 - h < 0 ? 0 : by0 - h;
        bx1 = bx1 + h > lw - 1 ? lw - 1 : bx1 + h;
        by1 = by1 + h > lh - 1 ? lh - 1 : by1 + h;
        const int bw = bx1 - bx0 + 1, bh = by1 - by0 + 1;
        uint8_t* marked = (uint8_t*)calloc((size_t)bw * bh, 1);
        size_t nmarked = 0;
        for (size_t g = 0; g < ng; ++g) {
            const int cx = (int)(gcell[g] % (uint32_t)lw), cy = (int)(gcell[g] / (uint32_t)lw);
            for (int y = (by0 > cy - h ? by0 : cy - h); y <= (by1 < cy + h ? by1 : cy + h); ++y)
                for (int x = (bx0 > cx - h ? bx0 : cx - h); x <= (bx1 < cx + h ? bx1 : cx + h);
                     ++x) {
                    uint8_t* mk = &marked[(size_t)(y - by0) * bw + (x - bx0)];
                    nmarked += !*mk;
                    *mk = 1;
                }
        }
        affected = (uint32_t*)malloc(nmarked * (size_t)s * s * sizeof(uint32_t));
        for (int y = by0; y <= by1; ++y)
            for (int x = bx0; x <= bx1; ++x) {
                if (!marked[(size_t)(y - by0) * bw + (x - bx0)]) continue;
                /* footprint, grid.cpp:67-79 */
                const int px0 = x * s, py0 = y * s;
                const int px1 = px0 + s < W ? px0 + s : W, py1 = py0 + s < H ? py0 + s : H;
                for (int py = py0; py < py1; ++py)
                    for (int px = px0; px < px1; ++px)
                        affected[na++] = (uint32_t)py * (uint32_t)W + (uint32_t)px;
            }
        free(marked);
    }

    /* Backup and e0 (150-157). */
    glu_o_params* oldParams = (glu_o_params*)malloc((na ? na : 1) * sizeof(glu_o_params));
    float* oldE = (float*)malloc((na ? na : 1) * sizeof(float));
    double e0 = 0;
    for (size_t i = 0; i < na; ++i) {
        oldParams[i] = field[affected[i]];
        oldE[i] = errors[affected[i]];
        e0 += oldE[i];
    }
    /* Re-solve (159) and re-score (160-165). */
    glu_o_optimize_pixels(high, W, H, low, s, S, eps, mode, affected, na, field);
    double e1 = 0;
    for (size_t i = 0; i < na; ++i) {
        const uint32_t p = affected[i];
        float r[3];
        o_reconstruct(&field[p], low, 3, 1, r);
        const float e = o_pixel_error(high + 3 * (size_t)p, r);
        errors[p] = e;
        e1 += e;
    }
    int accepted = e1 <= e0; /* 167 */
    if (!accepted) {         /* bitwise rollback, 169-179 */
        for (size_t i = 0; i < na; ++i) {
            field[affected[i]] = oldParams[i];
            errors[affected[i]] = oldE[i];
        }
        for (size_t g = 0; g < ng; ++g)
            memcpy(low + 3 * (size_t)gcell[g], oldColors + 3 * g, 3 * sizeof(float));
    }
    free(pairs);
    free(gcell);
    free(oldColors);
    free(affected);
    free(oldParams);
    free(oldE);
    return accepted;
}

/* joint_optimize: jointopt.cpp:182-206 */
int glu_o_joint_optimize(const float* high, int W, int H, int s, int S, float threshold,
                         int maxIterations, double eps, int mode, int literal, float* low,
                         glu_o_params* field, float* errors, int* counters) {
    if (o_check(W, H, s, S, eps) || !(threshold >= 0) || maxIterations < 0) return -1;
    const int lw = (W + s - 1) / s, lh = (H + s - 1) / s;
    const size_t npx = (size_t)W * H;
    glu_o_grid_downsample(high, W, H, s, low);
    glu_o_optimize_field(high, W, H, low, s, S, eps, mode, field);
    float* recon = (float*)malloc(npx * 3 * sizeof(float));
    glu_o_apply_field(field, W, H, low, lw, lh, 3, 1, recon);
    glu_o_error_map(high, recon, npx, errors);
    free(recon);

    uint8_t* mask = (uint8_t*)malloc(npx);
    uint32_t* off = (uint32_t*)malloc((npx + 1) * sizeof(uint32_t));
    uint32_t* px = (uint32_t*)malloc(npx * sizeof(uint32_t));
    int iters = 0, acc = 0, rej = 0;
    for (int it = 0; it < maxIterations; ++it) {
        const long nc = glu_o_find_large_error(errors, W, H, threshold, mask, off, px);
        if (nc <= 0) break;
        ++iters;
        int sweepAcc = 0;
        for (long c = 0; c < nc; ++c) {
            const int r = glu_o_trial_update_component(high, W, H, low, s, S, eps, mode, literal,
                                                       field, errors, px + off[c],
                                                       off[c + 1] - off[c]);
            if (r == 1) {
                ++acc;
                ++sweepAcc;
            } else {
                ++rej;
            }
        }
        if (sweepAcc == 0) break;
    }
    free(mask);
    free(off);
    free(px);
    counters[0] = iters;
    counters[1] = acc;
    counters[2] = rej;
    return 0;
}
