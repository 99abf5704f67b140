// glu_math.cuh -- per-pixel selection maths, bit-compatible with the reference.
//
// The reference evaluates every selection quantity in IEEE double with FP
// contraction disabled (proj/CMakeLists.txt:15-18; upsample.cpp:28-42,
// 49-104, 158-176).  These functions restate those expressions in the same
// operation order.  The whole library is compiled with -fmad=false, so no
// double (or float) expression here is contracted into an FMA; the fp32 search
// kernels request FMAs explicitly with __fmaf_rn where the maths is only a
// filter.  Division and sqrt are the IEEE round-to-nearest operators, so the
// results are bit-identical to the x86-64 SSE2 reference.
#pragma once

#include <stdint.h>

#include "glu_cuda.h"

#if defined(__CUDACC__)
#define GLU_HD __host__ __device__ __forceinline__
#else
#define GLU_HD inline
#include <cmath>
#endif

namespace glu_cu {

GLU_HD double dsqrt(double x) { return sqrt(x); }

// dist(p, q): upsample.cpp:28-33.
GLU_HD double dist64(const float* p, const float* q) {
    const double d0 = double(p[0]) - double(q[0]);
    const double d1 = double(p[1]) - double(q[1]);
    const double d2 = double(p[2]) - double(q[2]);
    return dsqrt(d0 * d0 + d1 * d1 + d2 * d2);
}

// Squared distance before the sqrt (same sums as dist64).
GLU_HD double dist2_64(const float* p, const float* q) {
    const double d0 = double(p[0]) - double(q[0]);
    const double d1 = double(p[1]) - double(q[1]);
    const double d2 = double(p[2]) - double(q[2]);
    return d0 * d0 + d1 * d1 + d2 * d2;
}

// objective(ip, ia, ib, w, eps): upsample.cpp:35-42.
GLU_HD double objective64(const float* ip, const float* ia, const float* ib, double w,
                          double eps) {
    double r = 0;
    for (int c = 0; c < 3; ++c) {
        const double v = w * double(ia[c]) + (1.0 - w) * double(ib[c]) - double(ip[c]);
        r += v * v;
    }
    return r + eps * w * w;
}

// weight_exact: upsample.cpp:158-167.
GLU_HD double weight_exact64(const float* ip, const float* ia, const float* ib, double eps) {
    double num = 0, den = 0;
    for (int c = 0; c < 3; ++c) {
        const double pb = double(ip[c]) - double(ib[c]);
        const double ab = double(ia[c]) - double(ib[c]);
        num += pb * ab;
        den += ab * ab;
    }
    return num / (den + eps);
}

// (float)weight_exact64 with a zero numerator short-cut: num = +-0 (an exact
// colour match I_b = I_p, e.g. every LR sample pixel) gives +-0 / (den + eps)
// = num, bit for bit, without the IEEE division's special-case path.
GLU_HD float weight_exact64_f(const float* ip, const float* ia, const float* ib, double eps) {
    double num = 0, den = 0;
    for (int c = 0; c < 3; ++c) {
        const double pb = double(ip[c]) - double(ib[c]);
        const double ab = double(ia[c]) - double(ib[c]);
        num += pb * ab;
        den += ab * ab;
    }
    return float(num == 0.0 ? num : num / (den + eps));
}

// weight_fast: upsample.cpp:169-172.
GLU_HD double weight_fast64(const float* ip, const float* ia, const float* ib, double eps) {
    const double db = dist64(ip, ib);
    return db / (dist64(ip, ia) + db + eps);
}

#if defined(__CUDACC__)
// float(weight_fast64(ip, ia, ib, eps)) without the IEEE sqrt / division
// sequences (their special-case branches and slow paths are ~15 % of the
// fp32 solve kernel's instructions).  The squared distances are the
// reference's exact double sums; sqrt and the quotient come from the MUFU
// double approximations refined by Newton / FMA residual steps, each within
// 2 ulp of the correctly rounded value, so the double weight is within
// 12 ulp of the reference's (da, db <= da + db, three more roundings).  The
// float rounding of the reference's weight is therefore known unless the
// estimate lies within 32 ulp of a float rounding midpoint: then *ok = false
// and the caller evaluates weight_fast64 (probability ~2^-24 per pixel).
__device__ __forceinline__ double sqrt_refined(double s) {
    double r;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(s));
    const double hs = 0.5 * s;
    r = r * __fma_rn(-(hs * r), r, 1.5);
    r = r * __fma_rn(-(hs * r), r, 1.5);
    const double y = s * r;
    const double z = __fma_rn(__fma_rn(-y, y, s), 0.5 * r, y);
    return s > 0.0 ? z : 0.0;
}

__device__ __forceinline__ float weight_fast_verified(const float* ip, const float* ia,
                                                      const float* ib, double eps, bool* ok) {
    const double da = sqrt_refined(dist2_64(ip, ia));
    const double db = sqrt_refined(dist2_64(ip, ib));
    const double den = (da + db) + eps;
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(den));
    r = __fma_rn(r, __fma_rn(-den, r, 1.0), r);
    r = __fma_rn(r, __fma_rn(-den, r, 1.0), r);
    const double q0 = db * r;
    const double wt = __fma_rn(__fma_rn(-den, q0, db), r, q0);
    if (db == 0.0) {  // 0 / den: exactly 0 on both sides
        *ok = true;
        return 0.0f;
    }
    // the float rounding is settled when both ends of [wt (1 - 2^-48),
    // wt (1 + 2^-48)] round alike (RN is monotone; see weight_fast_lean)
    const float lo = __double2float_rn(__fma_rn(wt, -0x1.0p-48, wt));
    const float hi = __double2float_rn(__fma_rn(wt, 0x1.0p-48, wt));
    *ok = lo == hi && wt > 0x1.0p-100;
    return lo;
}
// (float) of the reference's weight d_b / (d_a + d_b + eps) (upsample.cpp:61)
// from a double estimate good to ~2^-42 (relative): the squared distances
// with DFMA, sqrt and the quotient from the MUFU double approximations (~2^-23)
// with one Newton step each (~2^-45).  Its float rounding is the reference's
// unless the estimate lies within 2^-36 of a float rounding midpoint (a 64x
// margin on the error): then *ok = false and the caller takes the IEEE
// evaluation (~2^-12 of pixels).  d_b = 0 gives exactly 0 on both sides.
__device__ __forceinline__ float weight_fast_lean(float ip0, float ip1, float ip2, float4 ca,
                                                  float4 cb, double eps, bool* ok) {
    const double p0 = ip0, p1 = ip1, p2 = ip2;
    const double a0 = p0 - double(ca.x), a1 = p1 - double(ca.y), a2 = p2 - double(ca.z);
    const double b0 = p0 - double(cb.x), b1 = p1 - double(cb.y), b2 = p2 - double(cb.z);
    const double sa = __fma_rn(a2, a2, __fma_rn(a1, a1, a0 * a0));
    const double sb = __fma_rn(b2, b2, __fma_rn(b1, b1, b0 * b0));
    if (sb == 0.0) {
        *ok = true;
        return 0.0f;
    }
    auto root = [](double x) {  // x > 0
        double r;
        asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
        const double y = x * r;
        return __fma_rn(__fma_rn(-y, y, x), 0.5 * r, y);
    };
    const double da = sa > 0.0 ? root(sa) : 0.0;
    const double db = root(sb);
    const double den = (da + db) + eps;
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(den));
    r = __fma_rn(r, __fma_rn(-den, r, 1.0), r);
    const double wt = db * r;
    // Every value within 2^-36 wt of the estimate has the same float rounding
    // iff the interval's ends do (RN is monotone); that rounding is then the
    // reference's.  (Replaced a midpoint-distance test: 13 -> 6 instructions,
    // k_solve32f 0.1444 -> 0.1402 ms per fused 4K frame.)
    const float lo = __double2float_rn(__fma_rn(wt, -0x1.0p-36, wt));
    const float hi = __double2float_rn(__fma_rn(wt, 0x1.0p-36, wt));
    *ok = lo == hi && wt > 0x1.0p-100;
    return lo;
}

#endif

// Candidate access: any type whose operator[](i) returns candidate i's colour
// (3 floats); candidates are indexed in the reference's raster list order.
struct StridedCands {
    const float* rgb;
    int stride;
    GLU_HD const float* operator[](int i) const { return rgb + i * stride; }
};

struct Pick {
    int ai, bi;
    double w;
};

// pixelFast: upsample.cpp:49-71.  Distances are recomputed in the second loop
// instead of kept in a scratch array; the value is bitwise the same.
template <class Cands>
GLU_HD Pick pick_fast64(const float* ip, Cands c, int n, double eps) {
    int ai = 0;
    double da = dist64(ip, c[0]);
    for (int i = 1; i < n; ++i) {
        const double d = dist64(ip, c[i]);
        if (d < da) {
            da = d;
            ai = i;
        }
    }
    const float* ia = c[ai];
    int bi = 0;
    double bestW = 0, bestObj = 0;
    for (int j = 0; j < n; ++j) {
        const double dj = dist64(ip, c[j]);
        const double w = dj / (da + dj + eps);
        const double obj = objective64(ip, ia, c[j], w, eps);
        if (j == 0 || obj < bestObj) {
            bestObj = obj;
            bestW = w;
            bi = j;
        }
    }
    return {ai, bi, bestW};
}

// pixelExact: upsample.cpp:73-91 (pairs i <= j, lexicographic, first argmin).
template <class Cands>
GLU_HD Pick pick_exact64(const float* ip, Cands c, int n, double eps) {
    Pick best{0, 0, 0.0};
    double bestObj = 0;
    bool first = true;
    for (int i = 0; i < n; ++i) {
        for (int j = i; j < n; ++j) {
            const double w = weight_exact64(ip, c[i], c[j], eps);
            const double obj = objective64(ip, c[i], c[j], w, eps);
            if (first || obj < bestObj) {
                first = false;
                bestObj = obj;
                best = {i, j, w};
            }
        }
    }
    return best;
}

// pixelGnu: upsample.cpp:93-104.
template <class Cands>
GLU_HD Pick pick_gnu64(const float* ip, Cands c, int n) {
    int ai = 0;
    double best = dist64(ip, c[0]);
    for (int i = 1; i < n; ++i) {
        const double d = dist64(ip, c[i]);
        if (d < best) {
            best = d;
            ai = i;
        }
    }
    return {ai, ai, 1.0};
}

template <class Cands>
GLU_HD Pick pick64(int mode, const float* ip, Cands c, int n, double eps) {
    if (mode == GLU_MODE_EXACT) return pick_exact64(ip, c, n, eps);
    if (mode == GLU_MODE_GNU) return pick_gnu64(ip, c, n);
    return pick_fast64(ip, c, n, eps);
}

// NaN results with the reference host's bits.  x86-64 SSE returns the first
// NaN operand of an operation (quieted), or the default NaN (sign set,
// 0xffc00000 as a float) when an invalid operation has no NaN operand; the GPU
// returns a canonical 0x7fffffff instead.  The reference's compiled loops
// evaluate reconstruct_pixel as (la * w) + (lb * (1 - w)) and pixel_error as
// s + (t - r)^2, channel by channel (objdump of apply_field / error_map in
// the reference build), so the first NaN in that order is the result.  Only
// reached when the result is NaN.
#ifdef __CUDA_ARCH__
__device__ __forceinline__ float quiet_nan_of(float x) {
    return __uint_as_float(__float_as_uint(x) | 0x00400000u);
}
__device__ __noinline__ float host_nan_lerp(float w, float la, float lb) {
    if (la != la) return quiet_nan_of(la);
    if (w != w) return quiet_nan_of(w);
    if (lb != lb) return quiet_nan_of(lb);
    return __uint_as_float(0xffc00000u);  // 0 * inf or inf - inf
}
__device__ __noinline__ float host_nan_error(const float* t, const float* r) {
    for (int c = 0; c < 3; ++c) {
        if (t[c] != t[c]) return quiet_nan_of(t[c]);
        if (r[c] != r[c]) return quiet_nan_of(r[c]);
        if (t[c] == r[c] && (t[c] - t[c]) != 0.0f) return __uint_as_float(0xffc00000u);  // inf - inf
    }
    return __uint_as_float(0xffc00000u);
}
#endif

// reconstruct_pixel, one channel (upsample.hpp:54-65): float maths, no FMA.
GLU_HD float lerp_clamp(float w, float la, float lb, bool clampOutput) {
    float v = w * la + (1.0f - w) * lb;
#ifdef __CUDA_ARCH__
    // a NaN passes the reference's clamp unchanged; returned before it, since
    // nvcc lowers the clamp to a NaN-canonicalising FMNMX
    if (v != v) return host_nan_lerp(w, la, lb);
#endif
    if (clampOutput) v = v < 0.0f ? 0.0f : (v > 1.0f ? 1.0f : v);
    return v;
}

// pixel_error (upsample.hpp:67-74).
GLU_HD float pixel_error(const float* t, const float* r) {
    double s = 0;
    for (int c = 0; c < 3; ++c) {
        const double d = double(t[c]) - double(r[c]);
        s += d * d;
    }
    float e = float(dsqrt(s));
#ifdef __CUDA_ARCH__
    if (e != e) e = host_nan_error(t, r);
#endif
    return e;
}

}  // namespace glu_cu
