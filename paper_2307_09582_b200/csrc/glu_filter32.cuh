// glu_filter32.cuh -- the fp32 filter + fp64 verify selection for ONE pixel
// (Fast / GNU, S = 3) on a candidate array, used where the LR image changes
// between calls (the joint loop's trial re-solves, glu_joint.cu).  Same maths,
// bounds and acceptance rules as k_solve32 (glu_solve32.cu);
// candidates outside the grid are passed as +inf and never win or tie.
#pragma once

#include "glu_math.cuh"

namespace glu_cu {

struct Filter32Result {
    bool ok;     // false: take the exact double-precision path
    int why;     // which rule sent the pixel to the exact path (diagnostics)
    int ja, jb;  // slot (r * 3 + c) of a and b in the 3 x 3 window
    float w;
};

__device__ __forceinline__ float f32_sqrt_approx(float q) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(q));
    return r;
}
__device__ __forceinline__ float f32_rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float f32_rsqrt_approx(float x) {
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

__device__ inline Filter32Result filter32_pixel(const float4 (&c)[9], const float* ip,
                                                float epsf, double eps, bool gnu) {
    constexpr float kU = 5.9604645e-08f, kCA = 32.0f, kC1 = 128.0f, kC2 = 32.0f, kC3 = 64.0f;
    constexpr float kInf = __builtin_huge_valf();
    const float ip0 = ip[0], ip1 = ip[1], ip2 = ip[2];
    float q[9], e0[9], e1[9], e2[9];
    float m1 = kInf, m2 = kInf;
    int ja = 0;
#pragma unroll
    for (int j = 0; j < 9; ++j) {
        e0[j] = c[j].x - ip0;
        e1[j] = c[j].y - ip1;
        e2[j] = c[j].z - ip2;
        const float qq = __fmaf_rn(e2[j], e2[j], __fmaf_rn(e1[j], e1[j], __fmul_rn(e0[j], e0[j])));
        q[j] = qq;
        const bool lt = qq < m1;
        m2 = lt ? m1 : fminf(m2, qq);
        m1 = lt ? qq : m1;
        ja = lt ? j : ja;
    }
    Filter32Result r{false, 1, ja, ja, 1.0f};
    // a NaN candidate must take the reference's exact scan (comparisons with
    // NaN keep the earlier index there, e.g. a NaN first candidate stays a)
#pragma unroll
    for (int j = 0; j < 9; ++j)
        if (q[j] != q[j]) return r;
    float4 ca = c[0];
#pragma unroll
    for (int j = 1; j < 9; ++j)
        if (j == ja) ca = c[j];
    const bool exactA = ca.x == ip0 && ca.y == ip1 && ca.z == ip2;
    r.why = 2;
    if (!(m1 < kInf) || ip0 != ip0 || ip1 != ip1 || ip2 != ip2 || !(m1 >= 1e-27f || exactA))
        return r;
    r.why = 3;
    const float lim = __fmaf_rn(m1, kCA * kU, m1) + 1e-36f;
    if (m2 <= lim) {
#pragma unroll
        for (int j = 0; j < 9; ++j)
            if (j != ja && q[j] <= lim &&
                !(c[j].x == ca.x && c[j].y == ca.y && c[j].z == ca.z))
                return r;
    }
    if (gnu) {
        r.ok = true;
        return r;
    }
    const float ea0 = ca.x - ip0, ea1 = ca.y - ip1, ea2 = ca.z - ip2;
    const float da = f32_sqrt_approx(m1);
    float b1 = kInf, b2 = kInf, dmax = 0.0f;
    int jb = ja;
    float obj[9];
#pragma unroll
    for (int j = 0; j < 9; ++j) {
        const float dj = f32_sqrt_approx(q[j]);
        const float wj = dj * f32_rcp_approx((da + dj) + epsf);
        dmax = fmaxf(dmax, __fmaf_rn(wj, 0.0f, dj));
        const float v0 = __fmaf_rn(wj, ea0 - e0[j], e0[j]);
        const float v1 = __fmaf_rn(wj, ea1 - e1[j], e1[j]);
        const float v2 = __fmaf_rn(wj, ea2 - e2[j], e2[j]);
        const float o = __fmaf_rn(epsf * wj, wj, __fmaf_rn(v2, v2, __fmaf_rn(v1, v1, v0 * v0)));
        obj[j] = o;
        const bool lt = o < b1;
        b2 = lt ? b1 : fminf(b2, o);
        b1 = lt ? o : b1;
        jb = lt ? j : jb;
    }
    float4 cb = c[0];
#pragma unroll
    for (int j = 1; j < 9; ++j)
        if (j == jb) cb = c[j];
    r.why = 4;
    if (b1 == 0.0f) {
        if (!(cb.x == ip0 && cb.y == ip1 && cb.z == ip2)) return r;
    } else {
        r.why = 5;
        const float smax = da + dmax;
        const float bb = fmaxf(b1, 1e-30f);
        const float rt = f32_rsqrt_approx(bb), st = bb * rt;
        const float mb = kU * (kC1 * st * smax + kC2 * b1 + kC3 * epsf);
        const float alpha = 1.0f - kU * (0.5f * kC1 * smax * rt + kC2);
        const float rhs = b1 + mb + kU * (0.5f * kC1 * smax * st + kC3 * epsf);
        if (b2 * alpha <= rhs || alpha <= 0.0f) {
            // Close call.  Every candidate outside the close set has a larger
            // double objective than jb, so the reference's first argmin lies in
            // the set: evaluate just those in double, in index order.
            unsigned close = 0;
#pragma unroll
            for (int j = 0; j < 9; ++j)
                if (j == jb || obj[j] * alpha <= rhs || alpha <= 0.0f) {
                    if (!(q[j] < kInf)) return r;  // off-grid slot: exact path
                    close |= 1u << j;
                }
            const float a3[3] = {ca.x, ca.y, ca.z};
            const double dA = dist64(ip, a3);
            double best = 0, bw = 0;
            int bj = -1;
            for (int j = 0; j < 9; ++j) {
                if (!(close >> j & 1u)) continue;
                const float cj[3] = {c[j].x, c[j].y, c[j].z};
                const double dj = dist64(ip, cj);
                const double w = dj / (dA + dj + eps);
                const double o = objective64(ip, a3, cj, w, eps);
                if (bj < 0 || o < best) {
                    best = o;
                    bw = w;
                    bj = j;
                }
            }
            r.ok = true;
            r.jb = bj;
            r.w = float(bw);
            r.why = 6;
            return r;
        }
    }
    const float a3[3] = {ca.x, ca.y, ca.z}, b3[3] = {cb.x, cb.y, cb.z};
    bool wok = false;
    r.w = weight_fast_verified(ip, a3, b3, eps, &wok);
    if (!wok) {
        const double dA = dist64(ip, a3), dB = dist64(ip, b3);
        r.w = float(dB / (dA + dB + eps));
    }
    r.ok = true;
    r.jb = jb;
    return r;
}

}  // namespace glu_cu
