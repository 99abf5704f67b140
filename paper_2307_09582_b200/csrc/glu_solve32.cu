// glu_solve32.cu -- fp32 filter + fp64 verify solve (Fast and GNU modes).
//
// The reference selects (a, b) with double-precision distances and objectives
// (upsample.cpp:28-71, 93-104).  This kernel runs the same selection in fp32
// (FFMA / MUFU) together with a rigorous bound on the fp32 rounding error of
// every compared quantity.  A pixel whose winner is separated from every
// candidate of a different colour by more than the bound is provably the
// reference's choice (candidates of identical colour evaluate identically in
// any precision, and the first-index tie-break keeps the earliest of them).
// Otherwise the pixel takes the reference's exact double-precision path
// (glu_math.cuh) in place; such pixels are rare (~0.05% on the BASELINE
// scenes), so the divergence costs nothing measurable.  The stored weight is
// always recomputed in double in the reference's operation order, so params
// are bit-identical.
//
// Layout: the LR image is first packed (k_pack_low) into float4 cells with a
// border of h = S/2 cells holding +inf on every side.  Out-of-grid candidates
// then have inf distances and NaN objectives, which never win or tie, so every
// window is a full S x S block read with LDG.128 at compile-time offsets (the
// packed LR image is small and L1/L2-resident; neighbouring pixels share
// cells).  No shared memory, no barriers: every warp is independent.  Each
// stage tracks the best and the second-best value in the same pass; only when
// the second is inside the error bound of the best does a (rare) scan check
// whether the close candidates have the winner's exact colour.
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

constexpr int kThreads = 128;
#ifndef GLU_SOLVE_MIN_BLOCKS
#define GLU_SOLVE_MIN_BLOCKS 8
#endif
constexpr float kU = 5.9604645e-08f;  // 2^-24
constexpr float kCA = 32.0f;          // stage A relative margin (in u)
constexpr float kC1 = 128.0f, kC2 = 32.0f, kC3 = 64.0f;
constexpr float kInf = __builtin_huge_valf();

__device__ __forceinline__ bool same_rgb(float4 a, float4 b) {
    return a.x == b.x && a.y == b.y && a.z == b.z;
}

// MUFU approximations (rel. error <= 2^-22.9); arguments are kept normal by
// the callers, so flush-to-zero never applies.
__device__ __forceinline__ float rsqrt_approx(float x) {
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
// MUFU.SQRT: sqrt(0) = 0, sqrt(inf) = inf (the sentinel's weight is then NaN).
__device__ __forceinline__ float fast_sqrt(float q) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(q));
    return r;
}

// Exact reference weight for the chosen pair (upsample.cpp:28-33, 61).
__device__ __forceinline__ float weight64(const float* ip, float4 ca, float4 cb, double eps) {
    const float a3[3] = {ca.x, ca.y, ca.z}, b3[3] = {cb.x, cb.y, cb.z};
    bool ok = false;
    const float w = weight_fast_verified(ip, a3, b3, eps, &ok);
    if (ok) return w;
    const double da = dist64(ip, a3), db = dist64(ip, b3);
    return float(db / (da + db + eps));
}

__device__ __forceinline__ int div_s(int v, const SolveArgs& a) {
    return a.sdiv ? int(__umulhi(unsigned(v), a.sdiv)) : v / a.s;
}

// Candidate (r, c) of the window whose top-left is `win` (packed pitch `pw`).
template <int S>
__device__ __forceinline__ float4 cand(const float4* win, int pw, int j) {
    return __ldg(win + (j / S) * pw + (j % S));
}

// The truncated window of the packed image as the reference's raster list.
struct PackedWindow {
    const float4* win;  // packed cell of (x0, y0)
    int pw, nwx;
    __device__ __forceinline__ const float* operator[](int i) const {
        const int r = i / nwx, q = i - r * nwx;
        return reinterpret_cast<const float*>(win + r * pw + q);
    }
};

// Also raises *nanFlag when the LR image holds a NaN: the reference's scans
// treat NaN candidates by index order (every comparison is false), which the
// filter does not model, so such a solve runs entirely on the exact path.
__global__ void k_pack_low(const float* __restrict__ low, int lw, int lh, int h,
                           float4* __restrict__ packed, unsigned* nanFlag) {
    const int pw = lw + 2 * h, ph = lh + 2 * h;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= pw * ph) return;
    const int y = i / pw - h, x = i % pw - h;
    float4 v = make_float4(kInf, kInf, kInf, 0.0f);
    if (x >= 0 && y >= 0 && x < lw && y < lh) {
        const float* s = low + 3 * (size_t(y) * lw + x);
        // .w: the cell's largest |channel| (k_solve32f's rounding floor)
        v = make_float4(s[0], s[1], s[2], fmaxf(fabsf(s[0]), fmaxf(fabsf(s[1]), fabsf(s[2]))));
        if (v.x != v.x || v.y != v.y || v.z != v.z) atomicOr(nanFlag, 1u);
    }
    packed[i] = v;
}

template <int S, int MODE>
__global__ void __launch_bounds__(kThreads, GLU_SOLVE_MIN_BLOCKS)
    k_solve32(SolveArgs a, const float4* packed, int forceFallback, const unsigned* nanFlag) {
    forceFallback |= int(__ldg(nanFlag));
    constexpr int N = S * S;
    constexpr int h = S / 2;
    constexpr int NE = S == 3 ? N : 1;  // S = 3 keeps e_j in registers; S = 5 reloads
    const int pw = a.lw + 2 * h;
    // 32 x 4 pixel tiles: a warp covers 32 consecutive pixels of one row
    const int x = blockIdx.x * 32 + (threadIdx.x & 31);
    const int y = blockIdx.y * (kThreads / 32) + (threadIdx.x >> 5);
    if (x >= a.W || y >= a.H) return;
    const size_t p = size_t(y) * a.W + x;
    const int cx = div_s(x, a), cy = div_s(y, a);
    // packed cell (cx - h, cy - h) is at padded (cx, cy)
    const float4* win = packed + size_t(cy) * pw + cx;

    const float ip0 = __ldg(a.high + 3 * p), ip1 = __ldg(a.high + 3 * p + 1),
                ip2 = __ldg(a.high + 3 * p + 2);
    // ---- stage A: a = first argmin |I_j - I_p| (compared as squares) --------
    float q[N], e0[NE], e1[NE], e2[NE];
    float m1 = kInf, m2 = kInf;
    int ja = 0;
#pragma unroll
    for (int j = 0; j < N; ++j) {
        const float4 v = cand<S>(win, pw, j);
        const float d0 = v.x - ip0, d1 = v.y - ip1, d2 = v.z - ip2;
        if (NE == N) {
            e0[j % NE] = d0;
            e1[j % NE] = d1;
            e2[j % NE] = d2;
        }
        const float qq = __fmaf_rn(d2, d2, __fmaf_rn(d1, d1, __fmul_rn(d0, d0)));
        q[j] = qq;
        const bool lt = qq < m1;
        m2 = lt ? m1 : fminf(m2, qq);
        m1 = lt ? qq : m1;
        ja = lt ? j : ja;
    }
    const float4 ca = cand<S>(win, pw, ja);
    const float ea0 = ca.x - ip0, ea1 = ca.y - ip1, ea2 = ca.z - ip2;
    const bool exactA = ca.x == ip0 && ca.y == ip1 && ca.z == ip2;
    // NaN inputs and underflow-sized distances go to the exact path.
    bool ok = !forceFallback && m1 < kInf && ip0 == ip0 && ip1 == ip1 && ip2 == ip2 &&
              (m1 >= 1e-27f || exactA);
    if (ok && m2 <= __fmaf_rn(m1, kCA * kU, m1) + 1e-36f) {
        const float lim = __fmaf_rn(m1, kCA * kU, m1) + 1e-36f;
        for (int j = 0; j < N; ++j)
            if (j != ja && !(q[j] > lim) && !same_rgb(cand<S>(win, pw, j), ca)) ok = false;
    }
    int jb = ja;
    float w = 1.0f;
    bool wExact = false;  // w already settled in double (close-set path)
    if (MODE == GLU_MODE_FAST && ok) {
        // ---- stage B: b = first argmin of the objective at w_j --------------
        const float da = fast_sqrt(m1);
        const float eps = a.epsf;
        float b1 = kInf, b2 = kInf, dmax = 0.0f;
#pragma unroll
        for (int j = 0; j < N; ++j) {
            float d0, d1, d2;
            if (NE == N) {
                d0 = e0[j % NE];
                d1 = e1[j % NE];
                d2 = e2[j % NE];
            } else {
                const float4 v = cand<S>(win, pw, j);
                d0 = v.x - ip0;
                d1 = v.y - ip1;
                d2 = v.z - ip2;
            }
            const float dj = fast_sqrt(q[j]);
            const float wj = dj * rcp_approx((da + dj) + eps);
            // outside the grid dj = inf and wj = inf * 0 = NaN, which fmaxf ignores
            dmax = fmaxf(dmax, __fmaf_rn(wj, 0.0f, dj));
            const float v0 = __fmaf_rn(wj, ea0 - d0, d0);
            const float v1 = __fmaf_rn(wj, ea1 - d1, d1);
            const float v2 = __fmaf_rn(wj, ea2 - d2, d2);
            const float o =
                __fmaf_rn(eps * wj, wj, __fmaf_rn(v2, v2, __fmaf_rn(v1, v1, v0 * v0)));
            const bool lt = o < b1;
            b2 = lt ? b1 : fminf(b2, o);
            b1 = lt ? o : b1;
            jb = lt ? j : jb;
        }
        const float4 cb = cand<S>(win, pw, jb);
        if (b1 == 0.0f) {
            // exact zero: only an exact colour match (w = 0, v = 0) gets there
            ok = cb.x == ip0 && cb.y == ip1 && cb.z == ip2;
        } else {
            const float smax = da + dmax;
            const float bb = fmaxf(b1, 1e-30f);
            const float rt = rsqrt_approx(bb), st = bb * rt;
            const float mb = kU * (kC1 * st * smax + kC2 * b1 + kC3 * eps);
            // near(o): o (1 - u(C1 smax / (2 sqrt b1) + C2)) <= b1 + mb + u(C1 smax sqrt(b1)/2 + C3 eps)
            const float alpha = 1.0f - kU * (0.5f * kC1 * smax * rt + kC2);
            const float rhs = b1 + mb + kU * (0.5f * kC1 * smax * st + kC3 * eps);
            if (b2 * alpha <= rhs || alpha <= 0.0f) {
                // rare: recompute the objectives; the close set (candidates
                // within the bound of the best) holds the reference's first
                // argmin.  All of the winner's colour: done; else settle the
                // set in double, in index order (off-grid members: exact path).
                unsigned close = 1u << jb;
                bool mixed = false;
                for (int j = 0; j < N; ++j) {
                    if (j == jb) continue;
                    const float4 v = cand<S>(win, pw, j);
                    const float d0 = v.x - ip0, d1 = v.y - ip1, d2 = v.z - ip2;
                    const float dj = fast_sqrt(q[j]);
                    const float wj = dj * rcp_approx((da + dj) + eps);
                    const float v0 = __fmaf_rn(wj, ea0 - d0, d0);
                    const float v1 = __fmaf_rn(wj, ea1 - d1, d1);
                    const float v2 = __fmaf_rn(wj, ea2 - d2, d2);
                    const float o = __fmaf_rn(eps * wj, wj,
                                              __fmaf_rn(v2, v2, __fmaf_rn(v1, v1, v0 * v0)));
                    if (o * alpha <= rhs || alpha <= 0.0f) {
                        if (!(q[j] < kInf)) ok = false;
                        close |= 1u << j;
                        mixed |= !same_rgb(v, cb);
                    }
                }
                if (ok && mixed) {
                    const float ip[3] = {ip0, ip1, ip2};
                    const float a3[3] = {ca.x, ca.y, ca.z};
                    const double dA = dist64(ip, a3);
                    double best = 0, bw = 0;
                    int bj = -1;
                    for (int j = 0; j < N; ++j) {
                        if (!(close >> j & 1u)) continue;
                        const float4 v = cand<S>(win, pw, j);
                        const float cj[3] = {v.x, v.y, v.z};
                        const double dj = dist64(ip, cj);
                        const double wj = dj / (dA + dj + a.eps);
                        const double o = objective64(ip, a3, cj, wj, a.eps);
                        if (bj < 0 || o < best) {
                            best = o;
                            bw = wj;
                            bj = j;
                        }
                    }
                    jb = bj;
                    w = float(bw);
                    wExact = true;
                    if (a.fallbacks) atomicAdd(a.fallbacks + 1, 1ull);
                }
            }
        }
        if (ok && !wExact) {
            const float ip[3] = {ip0, ip1, ip2};
            w = weight64(ip, ca, cb, a.eps);
        }
    }
    uint32_t ia, ib;
    if (ok) {
        ia = uint32_t(cy - h + ja / S) * uint32_t(a.lw) + uint32_t(cx - h + ja % S);
        ib = uint32_t(cy - h + jb / S) * uint32_t(a.lw) + uint32_t(cx - h + jb % S);
    } else {
        // ---- exact double-precision path (upsample.cpp:49-71, 93-104) -------
        const int wx0 = max(0, cx - h), wy0 = max(0, cy - h);
        const int nwx = min(a.lw - 1, cx + h) - wx0 + 1;
        const int nwy = min(a.lh - 1, cy + h) - wy0 + 1;
        const float ip[3] = {ip0, ip1, ip2};
        PackedWindow pwin{packed + size_t(wy0 + h) * pw + (wx0 + h), pw, nwx};
        const Pick pk = MODE == GLU_MODE_GNU ? pick_gnu64(ip, pwin, nwx * nwy)
                                             : pick_fast64(ip, pwin, nwx * nwy, a.eps);
        const int ar = pk.ai / nwx, br = pk.bi / nwx;
        ia = uint32_t(wy0 + ar) * uint32_t(a.lw) + uint32_t(wx0 + pk.ai - ar * nwx);
        ib = uint32_t(wy0 + br) * uint32_t(a.lw) + uint32_t(wx0 + pk.bi - br * nwx);
        w = float(pk.w);
        if (a.fallbacks) atomicAdd(a.fallbacks, 1ull);
    }
    if (a.params) {
        unsigned* o = reinterpret_cast<unsigned*>(a.params + p);
        o[0] = ia + a.idxBase;
        o[1] = ib + a.idxBase;
        o[2] = __float_as_uint(w);
    }
    if (a.lowT) {
        const bool clamp = a.clamp != 0;
        if (a.channels == 1) {  // the video path's matte target
            a.out[p] = lerp_clamp(w, __ldg(a.lowT + ia), __ldg(a.lowT + ib), clamp);
        } else {
#pragma unroll
            for (int k = 0; k < 3; ++k)
                a.out[3 * p + k] = lerp_clamp(w, __ldg(a.lowT + 3 * size_t(ia) + k),
                                              __ldg(a.lowT + 3 * size_t(ib) + k), clamp);
        }
    }
    if (a.errOut) {  // pixel_error of the clamped self reconstruction (jointopt.cpp:190)
        float r[3];
#pragma unroll
        for (int k = 0; k < 3; ++k)
            r[k] = lerp_clamp(w, __ldg(a.low + 3 * size_t(ia) + k), __ldg(a.low + 3 * size_t(ib) + k),
                              true);
        const float ipx[3] = {ip0, ip1, ip2};
        a.errOut[p] = pixel_error(ipx, r);
    }
}

template <int S, int MODE>
cudaError_t launch_t(glu_ctx* ctx, const SolveArgs& a, const float4* packed, int force,
                     const unsigned* nanFlag) {
    dim3 grid((a.W + 31) / 32, (a.H + kThreads / 32 - 1) / (kThreads / 32));
    k_solve32<S, MODE><<<grid, kThreads, 0, ctx->stream>>>(a, packed, force, nanFlag);
    ++ctx->launches;
    return cudaGetLastError();
}

}  // namespace

bool solve32_supported(int mode, int S, int s) {
    return ((mode == GLU_MODE_FAST || mode == GLU_MODE_GNU) && (S == 3 || S == 5)) ||
           solve32x_supported(mode, S, s);
}

namespace {

SolveArgs prepared(const SolveArgs& a0) {
    SolveArgs a = a0;
    // x / s as a multiply-high: exact for x, s < 2^16 with m = ceil(2^32 / s).
    a.sdiv = (a.W < 65536 && a.H < 65536)
                 ? unsigned((0x100000000ull + unsigned(a.s) - 1) / unsigned(a.s))
                 : 0u;
    a.epsf = float(a.eps);
    return a;
}

cudaError_t dispatch(glu_ctx* ctx, const SolveArgs& a, const float4* packed, int forceFallback,
                     const unsigned* nanFlag) {
    if (a.mode == GLU_MODE_EXACT) return launch_solve32x(ctx, a, packed, forceFallback, nanFlag);
#ifndef GLU_SOLVE_F
#define GLU_SOLVE_F 1
#endif
    if (GLU_SOLVE_F && solve32f_supported(a.mode, a.S))  // Fast / GNU, S = 3
        return launch_solve32f(ctx, a, packed, forceFallback, nanFlag);
    if (a.mode == GLU_MODE_GNU)
        return a.S == 3 ? launch_t<3, GLU_MODE_GNU>(ctx, a, packed, forceFallback, nanFlag)
                        : launch_t<5, GLU_MODE_GNU>(ctx, a, packed, forceFallback, nanFlag);
    return a.S == 3 ? launch_t<3, GLU_MODE_FAST>(ctx, a, packed, forceFallback, nanFlag)
                    : launch_t<5, GLU_MODE_FAST>(ctx, a, packed, forceFallback, nanFlag);
}

// Per-frame preparation in one launch: grid_downsample (grid.cpp:41-52) into
// `low`, the packed / inf-bordered LR the solve reads, and optionally the 1-ch
// matte target (k_op_matte's expression); raises *nanFlag like k_pack_low.
__global__ void k_frame_prep(const float* __restrict__ high, int W, int H, int s, int lw,
                             int lh, int h, float* __restrict__ low, float4* __restrict__ packed,
                             float* __restrict__ matte, unsigned* nanFlag) {
    const int pw = lw + 2 * h, ph = lh + 2 * h;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= pw * ph) return;
    const int cy = i / pw - h, cx = i % pw - h;
    float4 v = make_float4(kInf, kInf, kInf, 0.0f);
    if (cx >= 0 && cy >= 0 && cx < lw && cy < lh) {
        const int x = min(cx * s + s / 2, W - 1), y = min(cy * s + s / 2, H - 1);
        const float* src = high + 3 * (size_t(y) * W + x);
        v = make_float4(src[0], src[1], src[2],
                        fmaxf(fabsf(src[0]), fmaxf(fabsf(src[1]), fabsf(src[2]))));
        const size_t c = size_t(cy) * lw + cx;
        low[3 * c] = v.x;
        low[3 * c + 1] = v.y;
        low[3 * c + 2] = v.z;
        if (matte) {
            const double Y = 0.299 * v.x + 0.587 * v.y + 0.114 * v.z;
            matte[c] = float(1.0 / (1.0 + exp(-10.0 * (Y - 0.5))));
        }
        if (v.x != v.x || v.y != v.y || v.z != v.z) atomicOr(nanFlag, 1u);
    }
    packed[i] = v;
}

// k_frame_prep over a batch of frames: frame blockIdx.y; its buffers live in
// one set per frame (low at +0, matte at +offMatte, packed at +offPacked).
__global__ void k_frame_prep_batch(const float* __restrict__ high, size_t highStride, int W, int H,
                                   int s, int lw, int lh, int h, char* base, size_t set,
                                   size_t offMatte, size_t offPacked, unsigned* flags) {
    const int f = blockIdx.y;
    char* b = base + size_t(f) * set;
    const int pw = lw + 2 * h, ph = lh + 2 * h;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= pw * ph) return;
    const float* hf = high + size_t(f) * highStride;
    float* low = reinterpret_cast<float*>(b);
    float* matte = reinterpret_cast<float*>(b + offMatte);
    float4* packed = reinterpret_cast<float4*>(b + offPacked);
    const int cy = i / pw - h, cx = i % pw - h;
    float4 v = make_float4(kInf, kInf, kInf, 0.0f);
    if (cx >= 0 && cy >= 0 && cx < lw && cy < lh) {
        const int x = min(cx * s + s / 2, W - 1), y = min(cy * s + s / 2, H - 1);
        const float* src = hf + 3 * (size_t(y) * W + x);
        v = make_float4(src[0], src[1], src[2],
                        fmaxf(fabsf(src[0]), fmaxf(fabsf(src[1]), fabsf(src[2]))));
        const size_t c = size_t(cy) * lw + cx;
        low[3 * c] = v.x;
        low[3 * c + 1] = v.y;
        low[3 * c + 2] = v.z;
        const double Y = 0.299 * v.x + 0.587 * v.y + 0.114 * v.z;
        matte[c] = float(1.0 / (1.0 + exp(-10.0 * (Y - 0.5))));
        if (v.x != v.x || v.y != v.y || v.z != v.z) atomicOr(flags + f, 1u);
    }
    packed[i] = v;
}

}  // namespace

cudaError_t launch_frame_prep_batch(glu_ctx* ctx, cudaStream_t st, const SolveArgs& a0,
                                    const FrameBatch& fb, char* base, size_t set,
                                    size_t offMatte, size_t offPacked, unsigned* flags) {
    const SolveArgs a = prepared(a0);
    const int h = a.S / 2;
    const size_t cells = size_t(a.lw + 2 * h) * (a.lh + 2 * h);
    cudaError_t e = cudaMemsetAsync(flags, 0, sizeof(unsigned) * size_t(fb.frames), st);
    if (e != cudaSuccess) return e;
    k_frame_prep_batch<<<dim3(unsigned((cells + 255) / 256), unsigned(fb.frames)), 256, 0, st>>>(
        a.high, fb.high, a.W, a.H, a.s, a.lw, a.lh, h, base, set, offMatte, offPacked, flags);
    ++ctx->launches;
    return cudaGetLastError();
}

cudaError_t launch_solve32(glu_ctx* ctx, const SolveArgs& a0, int forceFallback) {
    const SolveArgs a = prepared(a0);
    const int h = a.S / 2;
    const size_t cells = size_t(a.lw + 2 * h) * (a.lh + 2 * h);
    float4* packed = static_cast<float4*>(scratch(ctx, S_PACKED, cells * sizeof(float4)));
    if (!packed) return cudaErrorMemoryAllocation;
    unsigned* nanFlag = reinterpret_cast<unsigned*>(ctx->d_counters + 3);
    cudaError_t e = cudaMemsetAsync(nanFlag, 0, sizeof(unsigned), ctx->stream);
    if (e != cudaSuccess) return e;
    k_pack_low<<<unsigned((cells + 255) / 256), 256, 0, ctx->stream>>>(a.low, a.lw, a.lh, h,
                                                                        packed, nanFlag);
    ++ctx->launches;
    return dispatch(ctx, a, packed, forceFallback, nanFlag);
}

cudaError_t launch_frame_prep(glu_ctx* ctx, cudaStream_t st, const SolveArgs& a0, float* low,
                              float* matte, float4* packed, unsigned* nanFlag) {
    const SolveArgs a = prepared(a0);
    const int h = a.S / 2;
    const size_t cells = size_t(a.lw + 2 * h) * (a.lh + 2 * h);
    cudaError_t e = cudaMemsetAsync(nanFlag, 0, sizeof(unsigned), st);
    if (e != cudaSuccess) return e;
    k_frame_prep<<<unsigned((cells + 255) / 256), 256, 0, st>>>(a.high, a.W, a.H, a.s, a.lw, a.lh,
                                                                 h, low, packed, matte, nanFlag);
    ++ctx->launches;
    return cudaGetLastError();
}

cudaError_t launch_prepped_solve32(glu_ctx* ctx, const SolveArgs& a0, const float4* packed,
                                   int forceFallback, const unsigned* nanFlag) {
    return dispatch(ctx, prepared(a0), packed, forceFallback, nanFlag);
}

cudaError_t launch_prepped_solve32f_batch(glu_ctx* ctx, const SolveArgs& a0, const float4* packed,
                                          int forceFallback, const unsigned* flags,
                                          const FrameBatch& fb) {
    const SolveArgs a = prepared(a0);
    if (a.mode == GLU_MODE_EXACT) return launch_solve32x(ctx, a, packed, forceFallback, flags, fb);
    return launch_solve32f(ctx, a, packed, forceFallback, flags, fb);
}

cudaError_t launch_frame_solve32(glu_ctx* ctx, const SolveArgs& a0, float* low, float* matte,
                                 int forceFallback) {
    const SolveArgs a = prepared(a0);
    const int h = a.S / 2;
    const size_t cells = size_t(a.lw + 2 * h) * (a.lh + 2 * h);
    float4* packed = static_cast<float4*>(scratch(ctx, S_PACKED, cells * sizeof(float4)));
    if (!packed) return cudaErrorMemoryAllocation;
    unsigned* nanFlag = reinterpret_cast<unsigned*>(ctx->d_counters + 3);
    cudaError_t e = cudaMemsetAsync(nanFlag, 0, sizeof(unsigned), ctx->stream);
    if (e != cudaSuccess) return e;
    k_frame_prep<<<unsigned((cells + 255) / 256), 256, 0, ctx->stream>>>(
        a.high, a.W, a.H, a.s, a.lw, a.lh, h, low, packed, matte, nanFlag);
    ++ctx->launches;
    return dispatch(ctx, a, packed, forceFallback, nanFlag);
}

}  // namespace glu_cu
