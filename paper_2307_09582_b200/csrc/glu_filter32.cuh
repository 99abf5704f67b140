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

// Exact mode (S = 3) for ONE pixel on a candidate array: the selection of
// k_solve32x (glu_solve32x.cu) with D' = D / sqrt(den)
// formed per pair instead of read from a per-cell table.  Pairs (i <= j) are
// scanned j-outer; exact zeros and close calls recover the reference's
// lexicographic first; mixed close sets are settled in double; NaN, off-grid
// close members and underflow-sized distances take the exact path (ok false).
// ja / jb are the slots of the pair (i, j), w the stored weight.
__device__ inline Filter32Result filter32x_pixel(const float4 (&c)[9], const float* ip, float epsf,
                                                 double eps) {
    constexpr float kU = 5.9604645e-08f, kE = 64.0f * kU;
    constexpr float kInf = __builtin_huge_valf();
    const float ip0 = ip[0], ip1 = ip[1], ip2 = ip[2];
    Filter32Result r{false, 1, 0, 0, 0.0f};
    // c[k] for a run-time k without indexing the array (which would move it to
    // local memory for the whole function)
    auto at = [&](int k) {
        float4 v = c[0];
#pragma unroll
        for (int m = 1; m < 9; ++m)
            if (m == k) v = c[m];
        return v;
    };
    auto dprime = [&](const float4& vi, const float4& vj, float& d0, float& d1, float& d2) {
        d0 = vi.x - vj.x;
        d1 = vi.y - vj.y;
        d2 = vi.z - vj.z;
        const float den = __fmaf_rn(d2, d2, __fmaf_rn(d1, d1, __fmaf_rn(d0, d0, epsf)));
        const float rr = f32_rsqrt_approx(den);
        d0 *= rr;
        d1 *= rr;
        d2 *= rr;
    };
    auto qof = [&](const float4& v, float& e0, float& e1, float& e2) {
        e0 = v.x - ip0;
        e1 = v.y - ip1;
        e2 = v.z - ip2;
        return __fmaf_rn(e2, e2, __fmaf_rn(e1, e1, __fmul_rn(e0, e0)));
    };
    float qmin = kInf, b1 = kInf, m2 = kInf, bme = kInf;
    int bk = 0;
    bool nan = false;
#pragma unroll
    for (int j = 0; j < 9; ++j) {
        float e0, e1, e2;
        const float qj = qof(c[j], e0, e1, e2);
        nan |= qj != qj;
        const float qej = __fmaf_rn(kE, qj, 1e-36f);
        qmin = fminf(qmin, qj);
#pragma unroll
        for (int i = 0; i < j; ++i) {
            float d0, d1, d2;
            dprime(c[i], c[j], d0, d1, d2);
            const float dn = __fmaf_rn(e0, d0, __fmaf_rn(e1, d1, e2 * d2));
            const float o = __fmaf_rn(-dn, dn, qj);
            const float tt = o - qej;
            const bool lt = o < b1;
            m2 = fminf(m2, lt ? bme : tt);
            bme = lt ? tt : bme;
            b1 = lt ? o : b1;
            bk = lt ? (i << 4 | j) : bk;
        }
        const float tt = qj - qej;  // (j, j): w = 0
        const bool lt = qj < b1;
        m2 = fminf(m2, lt ? bme : tt);
        bme = lt ? tt : bme;
        b1 = lt ? qj : b1;
        bk = lt ? (j << 4 | j) : bk;
    }
    if (nan || !(b1 < kInf) || ip0 != ip0 || ip1 != ip1 || ip2 != ip2 ||
        !(qmin >= 1e-27f || qmin == 0.0f))
        return r;
    int bi = bk >> 4, bj = bk & 15;
    float4 ci = c[0], cj = c[0];
#pragma unroll
    for (int k = 1; k < 9; ++k) {
        if (k == bi) ci = c[k];
        if (k == bj) cj = c[k];
    }
    const float eb = __fmaf_rn(kE, __fmaf_rn(cj.z - ip2, cj.z - ip2,
                                             __fmaf_rn(cj.y - ip1, cj.y - ip1,
                                                       __fmul_rn(cj.x - ip0, cj.x - ip0))),
                               1e-36f);
    // an exact-zero distance must be a true colour match (no underflow)
    if (qmin == 0.0f) {
#pragma unroll
        for (int k = 0; k < 9; ++k) {
            float e0, e1, e2;
            if (qof(c[k], e0, e1, e2) == 0.0f && !(e0 == 0.0f && e1 == 0.0f && e2 == 0.0f))
                return r;
        }
    }
    bool wSet = false;
    float wv = 0.0f;
    if (b1 == 0.0f && cj.x == ip0 && cj.y == ip1 && cj.z == ip2) {
        // exact zeros: the lexicographically first is (first in-grid slot, first
        // exact colour match)
        int i0 = -1, j0 = -1;
#pragma unroll
        for (int k = 0; k < 9; ++k) {
            float e0, e1, e2;
            const float qk = qof(c[k], e0, e1, e2);
            if (i0 < 0 && qk < kInf) i0 = k;
            if (j0 < 0 && qk == 0.0f) j0 = k;
        }
        bi = i0;
        bj = j0;
#pragma unroll
        for (int k = 0; k < 9; ++k) {
            if (k == bi) ci = c[k];
            if (k == bj) cj = c[k];
        }
    } else if (m2 <= b1 + eb) {
        // close call: lexicographic re-check of the close pairs
        unsigned long long close = 0;
        bool mixed = false;
        int fi = -1, fj = -1, k = 0;
        for (int i = 0; i < 9; ++i) {
            const float4 vi = at(i);
            for (int j = i; j < 9; ++j, ++k) {
                const float4 vj = at(j);
                float e0, e1, e2;
                const float qj = qof(vj, e0, e1, e2);
                float o = qj;
                if (j != i) {
                    float d0, d1, d2;
                    dprime(vi, vj, d0, d1, d2);
                    const float dn = __fmaf_rn(e0, d0, __fmaf_rn(e1, d1, e2 * d2));
                    o = __fmaf_rn(-dn, dn, qj);
                }
                const bool best = i == bi && j == bj;
                if (!best && (!(o <= kInf) || !(o - __fmaf_rn(kE, qj, 1e-36f) <= b1 + eb)))
                    continue;
                if (!(vi.x < kInf && qj < kInf)) return r;  // off-grid member
                close |= 1ull << k;
                const bool same = vi.x == ci.x && vi.y == ci.y && vi.z == ci.z &&
                                  vj.x == cj.x && vj.y == cj.y && vj.z == cj.z;
                mixed |= !same;
                if (same && fi < 0) {
                    fi = i;
                    fj = j;
                }
            }
        }
        if (!mixed) {
            bi = fi;  // identical colours: identical objective and weight
            bj = fj;
        } else {
            double best = 0, bw = 0;
            int ni = -1, nj = -1, i = 0, j = 0;
            for (int kk = 0; kk < 45; ++kk) {
                if (close >> kk & 1ull) {
                    const float4 vi = at(i), vj = at(j);
                    const float a3[3] = {vi.x, vi.y, vi.z}, b3[3] = {vj.x, vj.y, vj.z};
                    const double wd = weight_exact64(ip, a3, b3, eps);
                    const double o = objective64(ip, a3, b3, wd, eps);
                    if (ni < 0 || o < best) {
                        best = o;
                        bw = wd;
                        ni = i;
                        nj = j;
                    }
                }
                if (++j == 9) j = ++i;
            }
            bi = ni;
            bj = nj;
            wSet = true;
            wv = float(bw);
        }
    }
    if (!wSet) {
        const float a3[3] = {ci.x, ci.y, ci.z}, b3[3] = {cj.x, cj.y, cj.z};
        wv = weight_exact64_f(ip, a3, b3, eps);
    }
    r.ok = true;
    r.ja = bi;
    r.jb = bj;
    r.w = wv;
    return r;
}

}  // namespace glu_cu
