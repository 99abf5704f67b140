// glu_solve32.cu -- fp32 filter + fp64 verify solve (Fast and GNU modes).
//
// The reference selects (a, b) with double-precision distances and objectives
// (upsample.cpp:28-71, 93-104).  This kernel runs the same selection in fp32
// (FFMA / MUFU) together with a rigorous bound on the fp32 rounding error of
// every compared quantity.  A pixel whose winner is separated from every
// candidate of a different colour by more than the bound is provably the
// reference's choice (candidates of identical colour evaluate identically in
// any precision, and the first-index tie-break keeps the earliest of them).
// Otherwise the pixel is queued in shared memory and re-solved at the end of
// the CTA with the reference's exact double-precision expressions
// (glu_math.cuh), one pixel per thread, so the rare fallbacks do not diverge
// the main pass.  The stored weight is always recomputed in double in the
// reference's operation order, so params are bit-identical.
//
// Error bounds (u = 2^-24, derivation in DESIGN.md "fp32 filter"):
//   stage A  q_j = |I_j - I_p|^2:            |q32 - q| <= 6u q
//   stage B  obj_j = |v|^2 + eps w^2 with v = e_j + w (e_a - e_j):
//            |obj32 - obj| <= u (56 sqrt(obj) s + 10 obj + 28 eps), s = d_a + d_j
// The kernel applies 2-4x those constants.
#include <cuda_runtime.h>

#include "glu_internal.h"
#include "glu_math.cuh"

namespace glu_cu {

namespace {

constexpr int kTX = 32, kTY = 8, kThreads = kTX * kTY;
constexpr float kU = 5.9604645e-08f;  // 2^-24
constexpr float kCA = 32.0f;          // stage A relative margin (in u)
constexpr float kC1 = 128.0f, kC2 = 32.0f, kC3 = 64.0f;

struct Tile4 {
    const float4* tile;
    int ncx, nwx, tx0, ty0;
    __device__ __forceinline__ const float* operator[](int i) const {
        const int r = i / nwx, q = i - r * nwx;
        return reinterpret_cast<const float*>(tile + (ty0 + r) * ncx + tx0 + q);
    }
};

__device__ __forceinline__ bool same_rgb(float4 a, float4 b) {
    return a.x == b.x && a.y == b.y && a.z == b.z;
}

__device__ __forceinline__ float fast_sqrt(float q) {
    return q * rsqrtf(fmaxf(q, 1e-37f));  // q = 0 -> 0
}

// Exact reference weight for the chosen pair (upsample.cpp:28-33, 61).
__device__ __forceinline__ float weight64(const float* ip, float4 ca, float4 cb, double eps) {
    const float a3[3] = {ca.x, ca.y, ca.z}, b3[3] = {cb.x, cb.y, cb.z};
    const double da = dist64(ip, a3), db = dist64(ip, b3);
    return float(db / (da + db + eps));
}

template <int S, int MODE>
__global__ void __launch_bounds__(kThreads) k_solve32(SolveArgs a, int forceFallback) {
    constexpr int N = S * S;
    constexpr int h = S / 2;
    extern __shared__ float4 tile[];
    __shared__ int fbList[kThreads];
    __shared__ int fbCount;

    const int x0 = blockIdx.x * kTX, y0 = blockIdx.y * kTY;
    const int cx0 = max(0, x0 / a.s - h), cy0 = max(0, y0 / a.s - h);
    const int cx1 = min(a.lw - 1, min(x0 + kTX - 1, a.W - 1) / a.s + h);
    const int cy1 = min(a.lh - 1, min(y0 + kTY - 1, a.H - 1) / a.s + h);
    const int ncx = cx1 - cx0 + 1, ncy = cy1 - cy0 + 1;
    if (threadIdx.x == 0) fbCount = 0;
    for (int i = threadIdx.x; i < ncx * ncy; i += kThreads) {
        const int ty = i / ncx, tx = i - ty * ncx;
        const float* src = a.low + 3 * (size_t(cy0 + ty) * a.lw + cx0 + tx);
        tile[i] = make_float4(__ldg(src), __ldg(src + 1), __ldg(src + 2), 0.0f);
    }
    __syncthreads();

    const int x = x0 + (threadIdx.x % kTX), y = y0 + (threadIdx.x / kTX);
    const bool live = x < a.W && y < a.H;
    const size_t p = size_t(y) * a.W + x;
    const int cx = x / a.s, cy = y / a.s;
    const int wx0 = max(0, cx - h), wy0 = max(0, cy - h);
    const int nwx = min(a.lw - 1, cx + h) - wx0 + 1, nwy = min(a.lh - 1, cy + h) - wy0 + 1;
    const float4* win = tile + (wy0 - cy0) * ncx + (wx0 - cx0);

    if (live) {
        const float ip[3] = {__ldg(a.high + 3 * p), __ldg(a.high + 3 * p + 1),
                             __ldg(a.high + 3 * p + 2)};
        // ---- stage A: a = first argmin |I_j - I_p| (compared as squares) ----
        float q[N];
        float qa = __int_as_float(0x7f800000), qmax = 0.0f;
        int ja = 0;
#pragma unroll
        for (int r = 0; r < S; ++r)
#pragma unroll
            for (int c = 0; c < S; ++c) {
                const int j = r * S + c;
                q[j] = __int_as_float(0x7f800000);
                if (r < nwy && c < nwx) {
                    const float4 v = win[r * ncx + c];
                    const float e0 = v.x - ip[0], e1 = v.y - ip[1], e2 = v.z - ip[2];
                    const float qq = __fmaf_rn(e2, e2, __fmaf_rn(e1, e1, __fmul_rn(e0, e0)));
                    q[j] = qq;
                    if (qq < qa) {
                        qa = qq;
                        ja = j;
                    }
                    qmax = fmaxf(qmax, qq);
                }
            }
        const float4 ca = win[(ja / S) * ncx + (ja % S)];
        const float ea0 = ca.x - ip[0], ea1 = ca.y - ip[1], ea2 = ca.z - ip[2];
        bool ok = !forceFallback;
        if (qa < 1e-27f && !(ea0 == 0.0f && ea1 == 0.0f && ea2 == 0.0f)) ok = false;
        {
            const float lim = __fmaf_rn(qa, kCA * kU, qa) + 1e-36f;
#pragma unroll
            for (int j = 0; j < N; ++j)
                if (j != ja && q[j] <= lim && !same_rgb(win[(j / S) * ncx + (j % S)], ca))
                    ok = false;
        }
        int jb = ja;
        float w = 1.0f;
        if (MODE == GLU_MODE_FAST && ok) {
            // ---- stage B: b = first argmin of the objective at w_j ----------
            const float da = fast_sqrt(qa);
            const float eps = float(a.eps);
            float obj[N];
            float best = __int_as_float(0x7f800000);
#pragma unroll
            for (int r = 0; r < S; ++r)
#pragma unroll
                for (int c = 0; c < S; ++c) {
                    const int j = r * S + c;
                    obj[j] = __int_as_float(0x7f800000);
                    if (r < nwy && c < nwx) {
                        const float4 v = win[r * ncx + c];
                        const float e0 = v.x - ip[0], e1 = v.y - ip[1], e2 = v.z - ip[2];
                        const float dj = fast_sqrt(q[j]);
                        const float wj = __fdividef(dj, da + dj + eps);
                        const float v0 = __fmaf_rn(wj, ea0 - e0, e0);
                        const float v1 = __fmaf_rn(wj, ea1 - e1, e1);
                        const float v2 = __fmaf_rn(wj, ea2 - e2, e2);
                        const float o = __fmaf_rn(eps * wj, wj,
                                                  __fmaf_rn(v2, v2, __fmaf_rn(v1, v1, v0 * v0)));
                        obj[j] = o;
                        if (o < best) {
                            best = o;
                            jb = j;
                        }
                    }
                }
            const float4 cb = win[(jb / S) * ncx + (jb % S)];
            if (best == 0.0f) {
                // exact zero: only an exact colour match (w = 0, v = 0) gets there
                ok = cb.x == ip[0] && cb.y == ip[1] && cb.z == ip[2];
            } else {
                const float smax = da + fast_sqrt(qmax);
                const float rt = rsqrtf(best), st = best * rt;
                const float mb = kU * (kC1 * st * smax + kC2 * best + kC3 * eps);
                const float alpha = 1.0f - kU * (0.5f * kC1 * smax * rt + kC2);
                const float rhs = best + mb + kU * (0.5f * kC1 * smax * st + kC3 * eps);
#pragma unroll
                for (int j = 0; j < N; ++j)
                    if (j != jb && obj[j] * alpha <= rhs &&
                        !same_rgb(win[(j / S) * ncx + (j % S)], cb))
                        ok = false;
            }
            if (ok) w = weight64(ip, ca, cb, a.eps);
        }
        if (ok) {
            const uint32_t ia = uint32_t(wy0 + ja / S) * uint32_t(a.lw) + uint32_t(wx0 + ja % S);
            const uint32_t ib = uint32_t(wy0 + jb / S) * uint32_t(a.lw) + uint32_t(wx0 + jb % S);
            if (a.params) {
                unsigned* o = reinterpret_cast<unsigned*>(a.params + p);
                o[0] = ia;
                o[1] = ib;
                o[2] = __float_as_uint(w);
            }
            if (a.lowT) {
                const int C = a.channels;
                for (int k = 0; k < C; ++k)
                    a.out[C * p + k] = lerp_clamp(w, __ldg(a.lowT + size_t(C) * ia + k),
                                                  __ldg(a.lowT + size_t(C) * ib + k),
                                                  a.clamp != 0);
            }
        } else {
            fbList[atomicAdd(&fbCount, 1)] = threadIdx.x;
        }
    }
    __syncthreads();
    // ---- exact double-precision re-solve of the uncertain pixels ---------------
    const int nfb = fbCount;
    for (int i = threadIdx.x; i < nfb; i += kThreads) {
        const int t = fbList[i];
        const int fx = x0 + (t % kTX), fy = y0 + (t / kTX);
        const size_t fp = size_t(fy) * a.W + fx;
        const int fcx = fx / a.s, fcy = fy / a.s;
        const int fwx0 = max(0, fcx - h), fwy0 = max(0, fcy - h);
        const int fnwx = min(a.lw - 1, fcx + h) - fwx0 + 1;
        const int fnwy = min(a.lh - 1, fcy + h) - fwy0 + 1;
        const float ip[3] = {a.high[3 * fp], a.high[3 * fp + 1], a.high[3 * fp + 2]};
        Tile4 tw{tile, ncx, fnwx, fwx0 - cx0, fwy0 - cy0};
        const Pick pk = MODE == GLU_MODE_GNU ? pick_gnu64(ip, tw, fnwx * fnwy)
                                             : pick_fast64(ip, tw, fnwx * fnwy, a.eps);
        const int ar = pk.ai / fnwx, br = pk.bi / fnwx;
        const uint32_t ia = uint32_t(fwy0 + ar) * uint32_t(a.lw) + uint32_t(fwx0 + pk.ai - ar * fnwx);
        const uint32_t ib = uint32_t(fwy0 + br) * uint32_t(a.lw) + uint32_t(fwx0 + pk.bi - br * fnwx);
        const float w = float(pk.w);
        if (a.params) {
            unsigned* o = reinterpret_cast<unsigned*>(a.params + fp);
            o[0] = ia;
            o[1] = ib;
            o[2] = __float_as_uint(w);
        }
        if (a.lowT) {
            const int C = a.channels;
            for (int k = 0; k < C; ++k)
                a.out[C * fp + k] = lerp_clamp(w, a.lowT[size_t(C) * ia + k],
                                               a.lowT[size_t(C) * ib + k], a.clamp != 0);
        }
    }
    if (threadIdx.x == 0 && nfb > 0 && a.fallbacks) atomicAdd(a.fallbacks, (unsigned long long)nfb);
}

template <int S, int MODE>
cudaError_t launch_t(glu_ctx* ctx, const SolveArgs& a, int force) {
    const int h = S / 2;
    const int ncx = (kTX - 1) / a.s + 2 + 2 * h, ncy = (kTY - 1) / a.s + 2 + 2 * h;
    const size_t smem = size_t(ncx) * ncy * sizeof(float4);
    if (smem > 40 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k_solve32<S, MODE>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             int(smem) + 4096);
        if (e != cudaSuccess) return e;
    }
    dim3 grid((a.W + kTX - 1) / kTX, (a.H + kTY - 1) / kTY);
    k_solve32<S, MODE><<<grid, kThreads, smem, ctx->stream>>>(a, force);
    ++ctx->launches;
    return cudaGetLastError();
}

}  // namespace

bool solve32_supported(int mode, int S) {
    return (mode == GLU_MODE_FAST || mode == GLU_MODE_GNU) && (S == 3 || S == 5);
}

cudaError_t launch_solve32(glu_ctx* ctx, const SolveArgs& a, int forceFallback) {
    if (a.mode == GLU_MODE_GNU)
        return a.S == 3 ? launch_t<3, GLU_MODE_GNU>(ctx, a, forceFallback)
                        : launch_t<5, GLU_MODE_GNU>(ctx, a, forceFallback);
    return a.S == 3 ? launch_t<3, GLU_MODE_FAST>(ctx, a, forceFallback)
                    : launch_t<5, GLU_MODE_FAST>(ctx, a, forceFallback);
}

}  // namespace glu_cu
