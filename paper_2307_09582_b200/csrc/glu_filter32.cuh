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

// A candidate's largest |channel| (carried in the .w of staged colours: the
// keyed Fast filter's bound on the reference's double rounding).
__device__ __forceinline__ float max_abs3(float x, float y, float z) {
    return fmaxf(fabsf(x), fmaxf(fabsf(y), fabsf(z)));
}

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
    bool wok = false;
    r.w = weight_fast_lean(ip0, ip1, ip2, ca, cb, eps, &wok);
    if (!wok) {
        const float a3[3] = {ca.x, ca.y, ca.z}, b3[3] = {cb.x, cb.y, cb.z};
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
// scanned j-outer, each reduced to one key (the fp32 objective lowered by its
// bound, row i in the low 4 mantissa bits); the smallest key K1 and the
// second smallest K2 decide the pick unless K2 is within the winner's bound.
// Exact colour matches pick (first in-grid slot, first match); close calls
// re-derive the keys, take the first of an all-same-colour close set or
// settle it in double in lexicographic order; NaN, off-grid close members and
// underflow-sized distances take the exact path (ok false).  ja / jb are the
// slots of the pair (i, j), w the stored weight.
__device__ __forceinline__ float f32x_pack(float t, int i, unsigned mask) {
    unsigned r;
    asm("lop3.b32 %0, %1, %2, %3, 0xEC;" : "=r"(r) : "r"(__float_as_uint(t)), "r"(unsigned(i)),
        "r"(mask));
    return __uint_as_float(r);
}

__device__ __forceinline__ void f32x_track(float& K1, float& K2, float k) {
    K2 = fmaxf(fminf(K2, k), K1);
    K1 = fminf(K1, k);
}

__device__ __forceinline__ void f32x_track2(float& K1, float& K2, float a, float b) {
    float mx;
    asm("max.NaN.f32 %0, %1, %2;" : "=f"(mx) : "f"(a), "f"(b));
    K2 = fmaxf(fminf(fminf(K2, a), b), fminf(K1, mx));
    K1 = fminf(fminf(K1, a), b);
}

// Fast mode for ONE pixel with k_solve32f's closed-form keyed stage B
// (glu_solve32f.cu): stage A as filter32_pixel; stage B
// keys = (B d_j c_j + (A - G) q_j) / s_j^2 with the index in the low 4 bits,
// decided by K1 / K2 unless K2 is within the winner's upper bound K1 + 2 G q_b
// / s_b^2 + F.  F = 2^-44 (M^2 + eps) needs M, the largest |channel| of the
// pixel and its window: the callers pass each in-grid candidate's largest
// |channel| in c[k].w (0 for off-grid slots).
__device__ __forceinline__ float f32k_key(float e0, float e1, float e2, float qj, float b0, float b1,
                                          float b2, float at, float Ap, int j, unsigned mask) {
    const float bc = __fmaf_rn(e2, b2, __fmaf_rn(e1, b1, __fmul_rn(e0, b0)));
    const float dj = f32_sqrt_approx(qj);
    const float nl = __fmaf_rn(dj, bc, __fmul_rn(Ap, qj));
    const float sj = __fadd_rn(at, dj);
    const float t = __fmul_rn(nl, f32_rcp_approx(__fmul_rn(sj, sj)));
    unsigned r;
    asm("lop3.b32 %0, %1, %2, %3, 0xEC;" : "=r"(r) : "r"(__float_as_uint(t)), "r"(unsigned(j)),
        "r"(mask));
    return __uint_as_float(r);
}

__device__ inline Filter32Result filter32k_pixel(const float4 (&c)[9], const float* ip, float epsf,
                                                 double eps) {
    constexpr float kU = 5.9604645e-08f, kCA = 32.0f, kG = 96.0f * kU, kF = 5.684342e-14f;
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
#pragma unroll
    for (int j = 0; j < 9; ++j)
        if (q[j] != q[j]) return r;  // NaN candidate: the reference's exact scan
    float4 ca = c[0];
    float mw = c[0].w;
#pragma unroll
    for (int j = 1; j < 9; ++j) {
        if (j == ja) ca = c[j];
        mw = fmaxf(mw, c[j].w);
    }
    const bool exactA = ca.x == ip0 && ca.y == ip1 && ca.z == ip2;
    r.why = 2;
    if (!(m1 < kInf) || ip0 != ip0 || ip1 != ip1 || ip2 != ip2 || !(m1 >= 1e-27f || exactA))
        return r;
    r.why = 3;
    const float limA = __fmaf_rn(m1, kCA * kU, m1) + 1e-36f;
    if (m2 <= limA) {
#pragma unroll
        for (int j = 0; j < 9; ++j)
            if (j != ja && q[j] <= limA &&
                !(c[j].x == ca.x && c[j].y == ca.y && c[j].z == ca.z))
                return r;
    }
    int jb = ja;
    if (!exactA) {  // exact match I_a == I_p: b = a (the first exact zero), w = 0
        const float ea0 = ca.x - ip0, ea1 = ca.y - ip1, ea2 = ca.z - ip2;
        const float da = f32_sqrt_approx(m1);
        const float at = da + epsf;
        const float A = __fadd_rn(__fmaf_rn(at, at, m1), epsf);
        const float B = at + at;
        const float G = kG * __fmaf_rn(B, da, A);
        const float Ap = A - G;
        const float b0 = B * ea0, b1 = B * ea1, b2 = B * ea2;
        const unsigned kmask = 0xfffffff0u | (__float_as_uint(epsf) >> 31);  // opaque: a register
        float K1 = kInf, K2 = kInf, pend = 0.0f;
#pragma unroll
        for (int j = 0; j < 9; ++j) {
            const float key = f32k_key(e0[j], e1[j], e2[j], q[j], b0, b1, b2, at, Ap, j, kmask);
            if (j & 1)
                f32x_track2(K1, K2, pend, key);
            else if (j == 8)
                f32x_track(K1, K2, key);
            else
                pend = key;
        }
        r.why = 4;
        if (!(K1 < kInf)) return r;
        jb = int(__float_as_uint(K1) & 15u);
        float qb = q[0];
        float4 cb = c[0];
#pragma unroll
        for (int j = 1; j < 9; ++j)
            if (j == jb) {
                qb = q[j];
                cb = c[j];
            }
        const float sb = __fadd_rn(at, f32_sqrt_approx(qb));
        const float m = fmaxf(mw, fmaxf(fabsf(ip0), fmaxf(fabsf(ip1), fabsf(ip2))));
        // keys overflow beyond 2^29 (k_solve32f's kMaxMag): exact path
        if (!(m < 536870912.0f)) return r;
        const float F = kF * __fmaf_rn(m, m, epsf);
        const float lim = K1 + __fmaf_rn(2.0f * G * qb, f32_rcp_approx(__fmul_rn(sb, sb)), F);
        if (K2 <= lim) {
            // close call: the candidates whose key is within lim hold the
            // reference's first argmin; all of the winner's colour: the first
            // of them, else settled in double in index order
            unsigned close = 0;
            bool mixed = false;
#pragma unroll
            for (int j = 0; j < 9; ++j) {
                const float key = f32k_key(e0[j], e1[j], e2[j], q[j], b0, b1, b2, at, Ap, j, kmask);
                if (key <= lim) {
                    r.why = 5;
                    if (!(q[j] < kInf)) return r;  // off-grid member: exact path
                    close |= 1u << j;
                    mixed |= !(c[j].x == cb.x && c[j].y == cb.y && c[j].z == cb.z);
                }
            }
            if (!mixed) {
                jb = __ffs(close) - 1;
            } else {
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
    }
    float4 cb = c[0];
#pragma unroll
    for (int j = 1; j < 9; ++j)
        if (j == jb) cb = c[j];
    bool wok = false;
    r.w = weight_fast_lean(ip0, ip1, ip2, ca, cb, eps, &wok);
    if (!wok) {
        const float a3[3] = {ca.x, ca.y, ca.z}, b3[3] = {cb.x, cb.y, cb.z};
        const double dA = dist64(ip, a3), dB = dist64(ip, b3);
        r.w = float(dB / (dA + dB + eps));
    }
    r.ok = true;
    r.jb = jb;
    return r;
}

// ---- Fast / GNU, S = 3, reading the window from shared memory -----------------
//
// The trial re-solve's variant of k_solve32f's per-pixel solve (glu_solve32f.cu,
// DESIGN.md section 3): the 3 x 3 window is read in place from the trial's
// staged LR window (top-left cell `wv`, row pitch `pitch`; off-grid cells +inf,
// .w = the cell's largest |channel|) instead of being copied into a register
// array, so a, b and the winners' colours are single shared-memory loads (the
// array version selected them with chains of FSELs).  Stage A: packed keys
// (q_j with the index in the low 4 mantissa bits) and the exact 32u near-tie
// check; stage B (Fast): the closed-form keys of k_solve32f; the weight by
// weight_fast_lean.  `ok` false: the caller takes the exact double path.

__device__ __forceinline__ int f32s_off(int j, int pitch) {
    const int r = (j * 11) >> 5;  // j / 3 for j < 9
    return r * pitch + (j - 3 * r);
}

__device__ __forceinline__ float f32s_q(float4 v, float ip0, float ip1, float ip2) {
    const float d0 = v.x - ip0, d1 = v.y - ip1, d2 = v.z - ip2;
    return __fmaf_rn(d2, d2, __fmaf_rn(d1, d1, __fmul_rn(d0, d0)));
}

__device__ __forceinline__ float f32s_max_nan(float a, float b) {  // NaN if either is NaN
    float r;
    asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    return r;
}

// The stage-B key of candidate v (k_solve32f's fast_key): the packed
// (B d_j c_j + (A - G) q_j) / s_j^2, (b0, b1, b2) = B e_a.
__device__ __forceinline__ float f32s_key(float4 v, float ip0, float ip1, float ip2, float b0,
                                          float b1, float b2, float at, float Ap, int j,
                                          unsigned mask) {
    const float e0 = v.x - ip0, e1 = v.y - ip1, e2 = v.z - ip2;
    const float qj = __fmaf_rn(e2, e2, __fmaf_rn(e1, e1, __fmul_rn(e0, e0)));
    const float bc = __fmaf_rn(e2, b2, __fmaf_rn(e1, b1, __fmul_rn(e0, b0)));
    const float dj = f32_sqrt_approx(qj);
    const float nl = __fmaf_rn(dj, bc, __fmul_rn(Ap, qj));
    const float sj = __fadd_rn(at, dj);
    const float t = __fmul_rn(nl, f32_rcp_approx(__fmul_rn(sj, sj)));
    unsigned r;
    asm("lop3.b32 %0, %1, %2, %3, 0xEC;" : "=r"(r) : "r"(__float_as_uint(t)), "r"(unsigned(j)),
        "r"(mask));
    return __uint_as_float(r);
}

// Stage-B close call (k_solve32f's resolve_close_fast): the candidates whose
// key is within lim hold the reference's first argmin; all of the winner's
// colour: the first of them, else settled in double in index order.  Returns
// jb, or -1 (an off-grid member: the exact path), and the weight in *w when
// settled in double (*wSet).
__device__ __noinline__ int f32s_close(const float4* wv, int pitch, float ip0, float ip1, float ip2,
                                       float at, float b0, float b1, float b2, float Ap, float lim,
                                       unsigned kmask, int ja, int jb, double eps, float* w,
                                       bool* wSet) {
    const float4 ca = wv[f32s_off(ja, pitch)], cb = wv[f32s_off(jb, pitch)];
    unsigned close = 0;
    bool mixed = false;
#pragma unroll
    for (int j = 0; j < 9; ++j) {
        const float4 v = wv[f32s_off(j, pitch)];
        if (f32s_key(v, ip0, ip1, ip2, b0, b1, b2, at, Ap, j, kmask) <= lim) {
            if (!(f32s_q(v, ip0, ip1, ip2) < __builtin_huge_valf())) return -1;
            close |= 1u << j;
            mixed |= !(v.x == cb.x && v.y == cb.y && v.z == cb.z);
        }
    }
    *wSet = false;
    if (!mixed) return __ffs(close) - 1;  // identical colours: identical objectives
    const float ip[3] = {ip0, ip1, ip2};
    const float a3[3] = {ca.x, ca.y, ca.z};
    const double dA = dist64(ip, a3);
    double best = 0, bw = 0;
    int bj = -1;
    for (unsigned m = close; m; m &= m - 1) {
        const int j = __ffs(m) - 1;
        const float4 v = wv[f32s_off(j, pitch)];
        const float cj[3] = {v.x, v.y, v.z};
        const double dj = dist64(ip, cj);
        const double wj = dj / (dA + dj + eps);
        const double o = objective64(ip, a3, cj, wj, eps);
        if (bj < 0 || o < best) {
            best = o;
            bw = wj;
            bj = j;
        }
    }
    *w = float(bw);
    *wSet = true;
    return bj;
}

__device__ __noinline__ float f32s_weight_ieee(float ip0, float ip1, float ip2, float4 ca,
                                               float4 cb, double eps) {
    const float ip[3] = {ip0, ip1, ip2};
    const float a3[3] = {ca.x, ca.y, ca.z}, b3[3] = {cb.x, cb.y, cb.z};
    const double dA = dist64(ip, a3), dB = dist64(ip, b3);
    return float(dB / (dA + dB + eps));
}

// A trial's re-solve of a pixel whose a and b (slots sa, sb of its 3 x 3 window
// `wv`) are not among the replaced cells (bits of `msk`): only the replaced
// candidates changed, so the reference's new pick is the old one iff none of
// them now beats it -- every replaced candidate strictly farther than a in
// double (stage A; a tie in distance could move a to an earlier index) and,
// in Fast mode unless I_a == I_p (b = a then), every replaced candidate's
// objective strictly above b's (stage B: keys are lower bounds of the
// reference's objectives, key_b + 2 G q_b / s_b^2 + F an upper bound of b's,
// DESIGN.md section 3).  true: a, b and w are the reference's new ones, and
// with a's and b's colours unchanged so is the error.  false: solve in full.
template <bool GNU>
__device__ __forceinline__ bool f32s_unchanged(const float4* wv, int pitch, const float* ip, int sa,
                                               int sb, uint32_t msk, float epsf) {
    constexpr float kU = 5.9604645e-08f, kCA = 32.0f, kG = 96.0f * kU, kF = 5.684342e-14f;
    constexpr float kInf = __builtin_huge_valf();
    constexpr float kMaxMag = 536870912.0f;  // 2^29 (k_solve32f)
    const float ip0 = ip[0], ip1 = ip[1], ip2 = ip[2];
    const float4 ca = wv[f32s_off(sa, pitch)];
    const float qa = f32s_q(ca, ip0, ip1, ip2);
    const bool exactA = ca.x == ip0 && ca.y == ip1 && ca.z == ip2;
    if (!(qa >= 1e-27f || exactA)) return false;  // NaN, underflow-sized distances
    const float thr = __fmaf_rn(qa, kCA * kU, qa) + 1e-36f;
    float m = fmaxf(fmaxf(ca.w, fabsf(ip0)), fmaxf(fabsf(ip1), fabsf(ip2)));
    for (uint32_t r = msk; r; r &= r - 1) {
        const float4 v = wv[f32s_off(__ffs(r) - 1, pitch)];
        if (!(f32s_q(v, ip0, ip1, ip2) > thr)) return false;
        m = fmaxf(m, v.w);
    }
    if (GNU || exactA) return true;
    const float4 cb = wv[f32s_off(sb, pitch)];
    m = fmaxf(m, cb.w);
    if (!(m < kMaxMag)) return false;
    const unsigned kmask = 0xfffffff0u | (__float_as_uint(epsf) >> 31);  // opaque: a register
    const float da = f32_sqrt_approx(qa);
    const float at = da + epsf;
    const float A = __fadd_rn(__fmaf_rn(at, at, qa), epsf);
    const float B = at + at;
    const float G = kG * __fmaf_rn(B, da, A);
    const float Ap = A - G;
    const float b0 = B * (ca.x - ip0), b1 = B * (ca.y - ip1), b2 = B * (ca.z - ip2);
    const float kb = f32s_key(cb, ip0, ip1, ip2, b0, b1, b2, at, Ap, sb, kmask);
    if (!(kb < kInf)) return false;
    const float qb = f32s_q(cb, ip0, ip1, ip2);
    const float sbb = __fadd_rn(at, f32_sqrt_approx(qb));
    const float F = kF * __fmaf_rn(m, m, epsf);
    const float lim = kb + __fmaf_rn(2.0f * G * qb, f32_rcp_approx(__fmul_rn(sbb, sbb)), F);
    for (uint32_t r = msk; r; r &= r - 1) {
        const int j = __ffs(r) - 1;
        if (!(f32s_key(wv[f32s_off(j, pitch)], ip0, ip1, ip2, b0, b1, b2, at, Ap, j, kmask) > lim))
            return false;
    }
    return true;
}

template <bool GNU>
__device__ __forceinline__ Filter32Result filter32_smem(const float4* wv, int pitch,
                                                        const float* ip, float epsf, double eps) {
    constexpr float kU = 5.9604645e-08f, kCA = 32.0f, kG = 96.0f * kU, kF = 5.684342e-14f;
    constexpr float kInf = __builtin_huge_valf();
    constexpr float kMaxMag = 536870912.0f;  // 2^29 (k_solve32f)
    const float ip0 = ip[0], ip1 = ip[1], ip2 = ip[2];
    const unsigned kmask = 0xfffffff0u | (__float_as_uint(epsf) >> 31);  // opaque: a register
    Filter32Result r{false, 2, 0, 0, 1.0f};
    // ---- stage A ----
    float K1a = kInf, K2a = kInf, pa = 0.0f, nanq = 0.0f, mw = 0.0f;
#pragma unroll
    for (int j = 0; j < 9; ++j) {
        const float4 v = wv[f32s_off(j, pitch)];
        const float qq = f32s_q(v, ip0, ip1, ip2);
        nanq = f32s_max_nan(nanq, qq);
        mw = fmaxf(mw, v.w);
        unsigned kb;
        asm("lop3.b32 %0, %1, %2, %3, 0xEC;" : "=r"(kb) : "r"(__float_as_uint(qq)), "r"(unsigned(j)),
            "r"(kmask));
        const float key = __uint_as_float(kb);
        if (j & 1)
            f32x_track2(K1a, K2a, pa, key);
        else if (j == 8)
            f32x_track(K1a, K2a, key);
        else
            pa = key;
    }
    const int ja = int(__float_as_uint(K1a) & 15u);
    const float4 ca = wv[f32s_off(ja, pitch)];
    const float m1 = f32s_q(ca, ip0, ip1, ip2);
    const bool exactA = ca.x == ip0 && ca.y == ip1 && ca.z == ip2;
    // NaN colours (a NaN guide channel makes every key NaN: K1a stays +inf),
    // underflow-sized distances: the exact path
    if (nanq != nanq || !(K1a < kInf) || !(m1 >= 1e-27f || exactA)) return r;
    r.why = 3;
    // any other candidate within (1 + 32u) q_a has a key within K1a (1 + 128u)
    if (K2a <= __fmaf_rn(K1a, 128.0f * kU, K1a) + 2e-36f) {
        const float lim = __fmaf_rn(m1, kCA * kU, m1) + 1e-36f;
#pragma unroll 1
        for (int j = 0; j < 9; ++j) {
            const float4 v = wv[f32s_off(j, pitch)];
            if (j != ja && !(f32s_q(v, ip0, ip1, ip2) > lim) &&
                !(v.x == ca.x && v.y == ca.y && v.z == ca.z))
                return r;
        }
    }
    r.ja = ja;
    if (GNU) {  // b = a, w = 1 (upsample.cpp:93-104)
        r.ok = true;
        r.jb = ja;
        r.w = 1.0f;
        return r;
    }
    int jb = ja;
    if (!exactA) {  // exact match I_a == I_p: b = a (the first exact zero), w = 0
        const float eps32 = epsf;
        const float da = f32_sqrt_approx(m1);
        const float at = da + eps32;
        const float A = __fadd_rn(__fmaf_rn(at, at, m1), eps32);
        const float B = at + at;
        const float G = kG * __fmaf_rn(B, da, A);
        const float Ap = A - G;
        const float b0 = B * (ca.x - ip0), b1 = B * (ca.y - ip1), b2 = B * (ca.z - ip2);
        float K1 = kInf, K2 = kInf, pend = 0.0f;
#pragma unroll
        for (int j = 0; j < 9; ++j) {
            const float key =
                f32s_key(wv[f32s_off(j, pitch)], ip0, ip1, ip2, b0, b1, b2, at, Ap, j, kmask);
            if (j & 1)
                f32x_track2(K1, K2, pend, key);
            else if (j == 8)
                f32x_track(K1, K2, key);
            else
                pend = key;
        }
        jb = int(__float_as_uint(K1) & 15u);
        const float4 cb = wv[f32s_off(jb, pitch)];
        const float qb = f32s_q(cb, ip0, ip1, ip2);
        const float sb = __fadd_rn(at, f32_sqrt_approx(qb));
        const float m = fmaxf(mw, fmaxf(fabsf(ip0), fmaxf(fabsf(ip1), fabsf(ip2))));
        const float F = kF * __fmaf_rn(m, m, eps32);
        const float lim = K1 + __fmaf_rn(2.0f * G * qb, f32_rcp_approx(__fmul_rn(sb, sb)), F);
        r.why = 4;
        if (!(K1 < kInf) || !(m < kMaxMag)) return r;
        if (K2 <= lim) {
            float wc = 0.0f;
            bool wSet = false;
            jb = f32s_close(wv, pitch, ip0, ip1, ip2, at, b0, b1, b2, Ap, lim, kmask, ja, jb, eps,
                            &wc, &wSet);
            r.why = 5;
            if (jb < 0) return r;
            if (wSet) {
                r.ok = true;
                r.why = 6;
                r.jb = jb;
                r.w = wc;
                return r;
            }
        }
    }
    const float4 cb = wv[f32s_off(jb, pitch)];
    bool wok = false;
    r.w = weight_fast_lean(ip0, ip1, ip2, ca, cb, eps, &wok);
    if (!wok) r.w = f32s_weight_ieee(ip0, ip1, ip2, ca, cb, eps);
    r.ok = true;
    r.jb = jb;
    return r;
}

__device__ inline Filter32Result filter32x_pixel(const float4 (&c)[9], const float* ip, float epsf,
                                                 double eps) {
    constexpr float kU = 5.9604645e-08f, kE = 64.0f * kU, kOneMinusE = 1.0f - kE;
    constexpr float kT = 136.0f * kU;
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
    auto qof = [&](const float4& v, float& e0, float& e1, float& e2) {
        e0 = v.x - ip0;
        e1 = v.y - ip1;
        e2 = v.z - ip2;
        return __fmaf_rn(e2, e2, __fmaf_rn(e1, e1, __fmul_rn(e0, e0)));
    };
    // key of pair (i, j), i < j (the same instruction sequence in the scan and
    // the close-call re-check)
    auto pair_t = [&](const float4& vi, const float4& vj, float e0, float e1, float e2,
                      float qm) {
        const float d0 = vi.x - vj.x, d1 = vi.y - vj.y, d2 = vi.z - vj.z;
        const float den = __fmaf_rn(d2, d2, __fmaf_rn(d1, d1, __fmaf_rn(d0, d0, epsf)));
        const float rr = f32_rsqrt_approx(den);
        const float dn = __fmaf_rn(e0, d0 * rr, __fmaf_rn(e1, d1 * rr, e2 * (d2 * rr)));
        return __fmaf_rn(-dn, dn, qm);
    };
    const unsigned kmask = 0xfffffff0u | (__float_as_uint(epsf) >> 31);  // opaque: a register
    float qmin = kInf, K1 = kInf, K2 = kInf;
    int bj = 0;
    bool nan = false;
#pragma unroll
    for (int j = 0; j < 9; ++j) {
        float e0, e1, e2;
        const float qj = qof(c[j], e0, e1, e2);
        nan |= qj != qj;
        qmin = fminf(qmin, qj);
        const float qm = __fmaf_rn(qj, kOneMinusE, -1e-36f);
        const float k1in = K1;
        float pend = 0.0f;
#pragma unroll
        for (int i = 0; i < j; ++i) {
            const float key = f32x_pack(pair_t(c[i], c[j], e0, e1, e2, qm), i, kmask);
            if (i & 1)
                f32x_track2(K1, K2, pend, key);
            else
                pend = key;
        }
        const float kd = f32x_pack(qm, j, kmask);  // (j, j): w = 0
        if (j & 1)
            f32x_track2(K1, K2, pend, kd);
        else
            f32x_track(K1, K2, kd);
        bj = K1 != k1in ? j : bj;
    }
    if (nan || !(K1 < kInf) || ip0 != ip0 || ip1 != ip1 || ip2 != ip2 ||
        !(qmin >= 1e-27f || qmin == 0.0f))
        return r;
    int bi = int(__float_as_uint(K1) & 15u);
    bool wSet = false;
    float wv = 0.0f;
    if (qmin == 0.0f) {
        // exact colour match: (first in-grid slot, first exact match); a zero
        // distance without a match (underflow) takes the exact path
        int i0 = -1, j0 = -1;
#pragma unroll
        for (int k = 8; k >= 0; --k) {
            float e0, e1, e2;
            if (qof(c[k], e0, e1, e2) < kInf) i0 = k;
            if (c[k].x == ip0 && c[k].y == ip1 && c[k].z == ip2) j0 = k;
        }
        if (j0 < 0 || i0 < 0) return r;
        bi = i0;
        bj = j0;
    } else {
        float e0, e1, e2;
        const float qb = qof(at(bj), e0, e1, e2);
        const float lim = K1 + __fmaf_rn(kT, qb, 2e-36f);
        if (K2 <= lim) {
            // close call: the pairs whose key is within lim (bit k =
            // lexicographic pair k) hold the reference's first argmin
            unsigned long long close = 0;
#pragma unroll
            for (int j = 0; j < 9; ++j) {
                const float qj = qof(c[j], e0, e1, e2);
                const float qm = __fmaf_rn(qj, kOneMinusE, -1e-36f);
#pragma unroll
                for (int i = 0; i <= j; ++i) {
                    const float key = i < j ? f32x_pack(pair_t(c[i], c[j], e0, e1, e2, qm), i, kmask)
                                            : f32x_pack(qm, j, kmask);
                    if (key <= lim) close |= 1ull << (i * 9 - i * (i - 1) / 2 + (j - i));
                }
            }
            const float4 ci = at(bi), cj = at(bj);
            bool mixed = false;
            int fi = -1, fj = -1;
            for (unsigned long long m = close; m; m &= m - 1) {
                const int k = __ffsll(static_cast<long long>(m)) - 1;
                const int i = (k >= 9) + (k >= 17) + (k >= 24) + (k >= 30) + (k >= 35) +
                              (k >= 39) + (k >= 42) + (k >= 44);
                const int j = k - (i * 9 - i * (i - 1) / 2) + i;
                const float4 vi = at(i), vj = at(j);
                if (!(vi.x < kInf && vj.x < kInf)) return r;  // off-grid member
                const bool same = vi.x == ci.x && vi.y == ci.y && vi.z == ci.z &&
                                  vj.x == cj.x && vj.y == cj.y && vj.z == cj.z;
                mixed |= !same;
                if (same && fi < 0) {
                    fi = i;
                    fj = j;
                }
            }
            if (!mixed) {
                bi = fi;  // identical colours: identical objective and weight
                bj = fj;
            } else {
                double best = 0, bw = 0;
                int ni = -1, nj = -1;
                for (unsigned long long m = close; m; m &= m - 1) {
                    const int k = __ffsll(static_cast<long long>(m)) - 1;
                    const int i = (k >= 9) + (k >= 17) + (k >= 24) + (k >= 30) + (k >= 35) +
                                  (k >= 39) + (k >= 42) + (k >= 44);
                    const int j = k - (i * 9 - i * (i - 1) / 2) + i;
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
                bi = ni;
                bj = nj;
                wSet = true;
                wv = float(bw);
            }
        }
    }
    if (!wSet) {
        const float4 ci = at(bi), cj = at(bj);
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
