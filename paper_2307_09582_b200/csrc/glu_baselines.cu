// glu_baselines.cu -- the reference's comparison upsamplers on device buffers
// (proj/src/baseline.cpp:30-129): joint bilateral,
// nearest and bilinear upsampling.  One thread per HR pixel; the LR images are
// tiny and stay in L1/L2.  Nearest is a copy and bilinear is the reference's
// double expression without contraction, both bit-exact; JBU's weights use
// CUDA's double exp (<= 1 ulp from glibc's), so its float outputs agree with
// the reference to within a float rounding step.
#include <cuda_runtime.h>

#include <cmath>

#include "glu_internal.h"

namespace glu_cu {

namespace {

// lowPos (baseline.cpp:24-25): continuous LR position, block-centre convention
__device__ __forceinline__ double low_pos(int x, int s) { return (x + 0.5) / s - 0.5; }

__global__ void k_nearest(const float* __restrict__ low, int W, int H, int s, int lw,
                          float* __restrict__ out) {
    const size_t p = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= size_t(W) * H) return;
    const int x = int(p % W), y = int(p / W);
    const float* src = low + 3 * (size_t(y / s) * lw + x / s);
    out[3 * p] = src[0];
    out[3 * p + 1] = src[1];
    out[3 * p + 2] = src[2];
}

__global__ void k_bilinear(const float* __restrict__ low, int W, int H, int s, int lw, int lh,
                           float* __restrict__ out) {
    const size_t p = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= size_t(W) * H) return;
    const int x = int(p % W), y = int(p / W);
    const double py = low_pos(y, s), px = low_pos(x, s);
    const int fy = int(floor(py)), fx = int(floor(px));
    const double ty = py - fy, tx = px - fx;
    const int y0 = min(max(fy, 0), lh - 1), y1 = min(max(fy + 1, 0), lh - 1);
    const int x0 = min(max(fx, 0), lw - 1), x1 = min(max(fx + 1, 0), lw - 1);
    for (int c = 0; c < 3; ++c) {
        const double top = (1 - tx) * double(low[3 * (size_t(y0) * lw + x0) + c]) +
                           tx * double(low[3 * (size_t(y0) * lw + x1) + c]);
        const double bot = (1 - tx) * double(low[3 * (size_t(y1) * lw + x0) + c]) +
                           tx * double(low[3 * (size_t(y1) * lw + x1) + c]);
        out[3 * p + c] = float((1 - ty) * top + ty * bot);
    }
}

// jbu_upsample (baseline.cpp:30-85)
__global__ void k_jbu(const float* __restrict__ gh, const float* __restrict__ gl,
                      const float* __restrict__ tl, int W, int H, int s, int lw, int lh,
                      int half, double invD, double invR, float* __restrict__ out) {
    const size_t p = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= size_t(W) * H) return;
    const int x = int(p % W), y = int(p / W);
    const double py = low_pos(y, s), px = low_pos(x, s);
    const int cy = y / s, cx = x / s;
    const float ip[3] = {gh[3 * p], gh[3 * p + 1], gh[3 * p + 2]};
    double acc0 = 0, acc1 = 0, acc2 = 0, wsum = 0;
    for (int gy = cy - half; gy <= cy + half; ++gy) {
        if (gy < 0 || gy >= lh) continue;
        for (int gx = cx - half; gx <= cx + half; ++gx) {
            if (gx < 0 || gx >= lw) continue;
            const double dx = px - gx, dy = py - gy;
            const float* g = gl + 3 * (size_t(gy) * lw + gx);
            double r2 = 0;
            for (int c = 0; c < 3; ++c) {
                const double d = double(ip[c]) - double(g[c]);
                r2 += d * d;
            }
            const double w = exp(-(dx * dx + dy * dy) * invD) * exp(-r2 * invR);
            const float* t = tl + 3 * (size_t(gy) * lw + gx);
            acc0 += w * double(t[0]);
            acc1 += w * double(t[1]);
            acc2 += w * double(t[2]);
            wsum += w;
        }
    }
    if (wsum > 0) {
        out[3 * p] = float(acc0 / wsum);
        out[3 * p + 1] = float(acc1 / wsum);
        out[3 * p + 2] = float(acc2 / wsum);
    } else {
        const float* t = tl + 3 * (size_t(cy) * lw + cx);
        out[3 * p] = t[0];
        out[3 * p + 1] = t[1];
        out[3 * p + 2] = t[2];
    }
}

int check_grid_local(const glu_grid* g) {
    if (!g || g->highW <= 0 || g->highH <= 0 || g->scale < 2 ||
        g->lowW != (g->highW + g->scale - 1) / g->scale ||
        g->lowH != (g->highH + g->scale - 1) / g->scale) {
        set_error("invalid grid");
        return GLU_EINVAL;
    }
    return GLU_OK;
}

unsigned blocks_of(const glu_grid* g) {
    return unsigned((size_t(g->highW) * g->highH + 255) / 256);
}

}  // namespace

}  // namespace glu_cu

using namespace glu_cu;

extern "C" {

int glu_cu_nearest_upsample(glu_ctx* ctx, const float* low, const glu_grid* g, float* out) {
    if (!ctx) {
        set_error("ctx must not be null");
        return GLU_EINVAL;
    }
    if (int rc = check_grid_local(g)) return rc;
    k_nearest<<<blocks_of(g), 256, 0, ctx->stream>>>(low, g->highW, g->highH, g->scale, g->lowW,
                                                     out);
    ++ctx->launches;
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? GLU_OK : fail_cuda(e, "nearest_upsample");
}

int glu_cu_bilinear_upsample(glu_ctx* ctx, const float* low, const glu_grid* g, float* out) {
    if (!ctx) {
        set_error("ctx must not be null");
        return GLU_EINVAL;
    }
    if (int rc = check_grid_local(g)) return rc;
    k_bilinear<<<blocks_of(g), 256, 0, ctx->stream>>>(low, g->highW, g->highH, g->scale,
                                                      g->lowW, g->lowH, out);
    ++ctx->launches;
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? GLU_OK : fail_cuda(e, "bilinear_upsample");
}

int glu_cu_jbu_upsample(glu_ctx* ctx, const float* guideHigh, const float* guideLow,
                        const float* targetLow, const glu_grid* g, int window, double sigmaD,
                        double sigmaR, float* out) {
    if (!ctx) {
        set_error("ctx must not be null");
        return GLU_EINVAL;
    }
    if (window < 1 || window % 2 == 0) {
        set_error("JbuParams: window must be odd and >= 1");
        return GLU_EINVAL;
    }
    if (!(sigmaD > 0) || !(sigmaR > 0)) {
        set_error("JbuParams: sigmas must be > 0");
        return GLU_EINVAL;
    }
    if (int rc = check_grid_local(g)) return rc;
    const double invD = 1.0 / (2 * sigmaD * sigmaD), invR = 1.0 / (2 * sigmaR * sigmaR);
    k_jbu<<<blocks_of(g), 256, 0, ctx->stream>>>(guideHigh, guideLow, targetLow, g->highW,
                                                 g->highH, g->scale, g->lowW, g->lowH,
                                                 window / 2, invD, invR, out);
    ++ctx->launches;
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? GLU_OK : fail_cuda(e, "jbu_upsample");
}

}  // extern "C"
