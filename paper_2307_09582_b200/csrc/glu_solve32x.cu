// glu_solve32x.cu -- fp32 filter + fp64 verify solve for Exact mode (S = 3).
//
// The reference's pixelExact (upsample.cpp:73-91) scans the 45 unordered pairs
// (i <= j, lexicographic) of the window with the closed-form weight
// w = (Ip - Ij).(Ii - Ij) / (|Ii - Ij|^2 + eps) (158-167) and keeps the first
// argmin of |w Ii + (1 - w) Ij - Ip|^2 + eps w^2, all in double.
//
// At its own optimum the objective has the closed form
//     obj_ij = |e_j|^2 - num^2 / den,   e = I - I_p, num = -e_j.D, D = I_i - I_j,
//                                       den = |D|^2 + eps,
// (and obj_ii = |e_i|^2 exactly, since w = 0).  D and 1/den depend only on the
// owner cell's window, so each CTA tabulates them once per owner cell in
// shared memory; a pixel then spends ~10 FP32 instructions per pair.  The
// fp32 error of obj_ij is below 17 u |e_j|^2 (u = 2^-24); the
// kernel uses 64 u q_max as a uniform bound, re-checks close calls with the
// per-pair bound, and sends the remaining ties between differently coloured
// pairs to the reference's exact double-precision path.  The stored weight is
// recomputed in double in the reference's order.
#include <cuda_runtime.h>

#include "glu_internal.h"
#include "glu_math.cuh"

namespace glu_cu {

namespace {

constexpr int kTX = 32, kTY = 8, kThreads = kTX * kTY;
constexpr int kPairs = 36;       // i < j over 9 candidates
constexpr int kCellStride = 37;  // float4 per owner cell (592 B: bank-spread)
constexpr int kMaxCells = 48;    // (31/3 + 2) x (7/3 + 2) owner cells for s >= 3
constexpr int kMaxWinCells = 96;  // their candidate cells: (ncw + 2) x (nch + 2) <= 14 x 6
constexpr float kU = 5.9604645e-08f;
constexpr float kCE = 64.0f;  // objective error bound, in u * |e_j|^2
constexpr float kInf = __builtin_huge_valf();

__device__ __forceinline__ float rsqrt_approx(float x) {
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

__device__ __forceinline__ int div_s(int v, const SolveArgs& a) {
    return a.sdiv ? int(__umulhi(unsigned(v), a.sdiv)) : v / a.s;
}

__device__ __forceinline__ bool same_rgb(float4 a, float4 b) {
    return a.x == b.x && a.y == b.y && a.z == b.z;
}

struct PackedWindow {
    const float4* win;
    int pw, nwx;
    __device__ __forceinline__ const float* operator[](int i) const {
        const int r = i / nwx, q = i - r * nwx;
        return reinterpret_cast<const float*>(win + r * pw + q);
    }
};

#ifndef GLU_X_MIN_BLOCKS
#define GLU_X_MIN_BLOCKS 6  // 40 registers: 48 warps per SM
#endif
__global__ void __launch_bounds__(kThreads, GLU_X_MIN_BLOCKS) k_solve32x(SolveArgs a, const float4* packed,
                                                          int forceFallback,
                                                          const unsigned* nanFlag) {
    forceFallback |= int(__ldg(nanFlag));
    __shared__ float4 table[kMaxCells * kCellStride];
    __shared__ float4 wcells[kMaxWinCells];  // the tile's candidate cells (owner cells +- 1)
    const int pw = a.lw + 2;  // h = 1
    const int x0 = blockIdx.x * kTX, y0 = blockIdx.y * kTY;
    const int ocx0 = div_s(x0, a), ocy0 = div_s(y0, a);
    const int ncw = div_s(min(x0 + kTX - 1, a.W - 1), a) - ocx0 + 1;
    const int nch = div_s(min(y0 + kTY - 1, a.H - 1), a) - ocy0 + 1;
    const float eps = a.epsf;
    const int cw = ncw + 2;
    for (int k = threadIdx.x; k < cw * (nch + 2); k += kThreads)
        wcells[k] = __ldg(packed + size_t(ocy0 + k / cw) * pw + (ocx0 + k % cw));
    __syncthreads();
    // thread t builds pair pr = t % 36 for cells t / 36, t / 36 + 7, ... (the
    // pair decode is paid once per thread)
    const int pr = int(threadIdx.x) % kPairs;
    const int ti = (pr >= 8) + (pr >= 15) + (pr >= 21) + (pr >= 26) + (pr >= 30) + (pr >= 33) +
                   (pr >= 35);
    const int tj = pr - (ti * 8 - ti * (ti - 1) / 2) + ti + 1;
    const int oi = (ti / 3) * cw + ti % 3, oj = (tj / 3) * cw + tj % 3;
    constexpr int kCellStep = kThreads / kPairs;  // 7 cells per pass; threads 252.. idle
    for (int cell = int(threadIdx.x) / kPairs; cell < ncw * nch && threadIdx.x < kCellStep * kPairs;
         cell += kCellStep) {
        const int ly = cell / ncw, lx = cell - ly * ncw;
        const float4* w = wcells + ly * cw + lx;
        const float4 ci = w[oi], cj = w[oj];
        const float d0 = ci.x - cj.x, d1 = ci.y - cj.y, d2 = ci.z - cj.z;
        const float den = __fmaf_rn(d2, d2, __fmaf_rn(d1, d1, __fmaf_rn(d0, d0, eps)));
        // D' = D / sqrt(den): then obj_ij = q_j - (e_j . D')^2
        const float r = rsqrt_approx(den);
        table[cell * kCellStride + pr] = make_float4(d0 * r, d1 * r, d2 * r, 0.0f);
    }
    __syncthreads();

    const int x = x0 + (threadIdx.x % kTX), y = y0 + (threadIdx.x / kTX);
    if (x >= a.W || y >= a.H) return;
    const size_t p = size_t(y) * a.W + x;
    const int cx = div_s(x, a), cy = div_s(y, a);
    const float4* win = packed + size_t(cy) * pw + cx;
    // the same window in shared memory: candidate j is swin[(j / 3) * cw + j % 3]
    const float4* swin = wcells + (cy - ocy0) * cw + (cx - ocx0);
    const float4* tab = table + ((cy - ocy0) * ncw + (cx - ocx0)) * kCellStride;
    const float ip0 = __ldg(a.high + 3 * p), ip1 = __ldg(a.high + 3 * p + 1),
                ip2 = __ldg(a.high + 3 * p + 2);

    // j-outer scan: pair (i, j) needs only e_j = I_j - I_p and q_j = |e_j|^2
    // (D'_ij = D_ij / sqrt(den) comes from the cell's table: obj = q_j -
    // (e_j . D')^2), so nothing per candidate stays live across the scan.  Track the strict argmin b1 (pair bk =
    // i << 4 | j) and, for the close-call test, t = o - E per pair (E = kCE u
    // q_j + 1e-36, its error bound): m2 = min of t over the pairs that are not
    // the current best, bme = the best pair's t.  This order is not the
    // reference's lexicographic (i <= j) order, so among exactly tied pairs
    // the lexicographic first is recovered below (exact zeros directly, other
    // ties in the re-check of close calls).
    constexpr float kE = kCE * kU;
    float qmin = kInf, b1 = kInf, m2 = kInf, bme = kInf;
    int bk = 0, i0 = -1, j0 = -1;
#pragma unroll
    for (int j = 0; j < 9; ++j) {
        const float4 v = swin[(j / 3) * cw + j % 3];
        const float e0 = v.x - ip0, e1 = v.y - ip1, e2 = v.z - ip2;
        const float qj = __fmaf_rn(e2, e2, __fmaf_rn(e1, e1, __fmul_rn(e0, e0)));
        const float qej = __fmaf_rn(kE, qj, 1e-36f);
        qmin = fminf(qmin, qj);
        i0 = (i0 < 0 && qj < kInf) ? j : i0;    // first in-grid candidate
        j0 = (j0 < 0 && qj == 0.0f) ? j : j0;  // first exact colour match
#pragma unroll
        for (int i = 0; i < j; ++i) {
            const float4 d = tab[i * 8 - i * (i - 1) / 2 + (j - i - 1)];
            const float dn = __fmaf_rn(e0, d.x, __fmaf_rn(e1, d.y, e2 * d.z));
            const float o = __fmaf_rn(-dn, dn, qj);
            const float tt = o - qej;
            const bool lt = o < b1;
            m2 = fminf(m2, lt ? bme : tt);
            bme = lt ? tt : bme;
            b1 = lt ? o : b1;
            bk = lt ? (i << 4 | j) : bk;
        }
        {
            const float o = qj;  // (j, j): w = 0
            const float tt = o - qej;
            const bool lt = o < b1;
            m2 = fminf(m2, lt ? bme : tt);
            bme = lt ? tt : bme;
            b1 = lt ? o : b1;
            bk = lt ? (j << 4 | j) : bk;
        }
    }
    int bi = bk >> 4, bj = bk & 15;
    float4 ci = swin[(bi / 3) * cw + bi % 3], cj = swin[(bj / 3) * cw + bj % 3];
    // the best pair's bound E_best (the same q_bj as in the scan)
    const float eb0 = cj.x - ip0, eb1 = cj.y - ip1, eb2 = cj.z - ip2;
    const float eb = __fmaf_rn(kE, __fmaf_rn(eb2, eb2, __fmaf_rn(eb1, eb1, __fmul_rn(eb0, eb0))),
                               1e-36f);
    bool ok = !forceFallback && b1 < kInf && ip0 == ip0 && ip1 == ip1 && ip2 == ip2 &&
              (qmin >= 1e-27f || qmin == 0.0f);
    // An exact zero with I_bj == I_p is exact in double too (w = 0, v = 0);
    // every true zero is a pair (i, j) with e_j = 0, which evaluates to exactly
    // 0 in fp32, so the reference's pick is the lexicographically first: (i0,
    // j0), i0 the first in-grid candidate, j0 the first exact colour match.
    // (Every LR sample pixel lands here.)
    const bool exactZero = b1 == 0.0f && cj.x == ip0 && cj.y == ip1 && cj.z == ip2;
    if (exactZero && j0 >= 0) {
        bi = i0;
        bj = j0;
        ci = swin[(bi / 3) * cw + bi % 3];
        cj = swin[(bj / 3) * cw + bj % 3];
    }
    bool wSet = false;  // w settled in double over the close set
    float wClose = 0.0f;
    if (ok && !exactZero && m2 <= b1 + eb) {
#ifdef GLU_X_COUNT_RECHECK
        if (a.fallbacks) atomicAdd(a.fallbacks + 1, 1ull);
#endif
        // rare: per-pair bounds, in lexicographic order.  The close pairs
        // (bit k = lexicographic pair k, the winner included) hold the
        // reference's first argmin: if they all carry the winner's colour
        // tuple, the first of them is the pick; otherwise they are evaluated in
        // double, in lexicographic order.
        unsigned long long close = 0;
        bool mixed = false;
        int fi = -1, fj = -1, k = 0;
#pragma unroll 1
        for (int i = 0; i < 9; ++i) {
            const float4 vi = swin[(i / 3) * cw + i % 3];
            const bool ini = vi.x < kInf;  // the +inf sentinel marks off-grid cells
#pragma unroll 1
            for (int j = i; j < 9; ++j, ++k) {
                const float4 vj = swin[(j / 3) * cw + j % 3];
                const float e0 = vj.x - ip0, e1 = vj.y - ip1, e2 = vj.z - ip2;
                const float qj = __fmaf_rn(e2, e2, __fmaf_rn(e1, e1, __fmul_rn(e0, e0)));
                float o = qj;
                if (j != i) {
                    const float4 d = tab[i * 8 - i * (i - 1) / 2 + (j - i - 1)];
                    const float dn = __fmaf_rn(e0, d.x, __fmaf_rn(e1, d.y, e2 * d.z));
                    o = __fmaf_rn(-dn, dn, qj);
                }
                const bool best = i == bi && j == bj;
                if (!best && (!(o <= kInf) || !(o - __fmaf_rn(kE, qj, 1e-36f) <= b1 + eb)))
                    continue;  // not close (NaN: outside the grid)
                if (!(ini && qj < kInf)) ok = false;  // off-grid member
                close |= 1ull << k;
                const bool same = same_rgb(vi, ci) && same_rgb(vj, cj);
                mixed |= !same;
                if (same && fi < 0) {
                    fi = i;
                    fj = j;
                }
            }
        }
        if (ok && !mixed) {
            bi = fi;  // identical colours: identical objectives and weight
            bj = fj;
        } else if (ok && mixed) {
            const float ip[3] = {ip0, ip1, ip2};
            double best = 0, bw = 0;
            int ni = -1, nj = -1;
            int i = 0, j = 0;
#pragma unroll 1
            for (int kk = 0; kk < 45; ++kk) {
                if (close >> kk & 1ull) {
                    const float4 vi = swin[(i / 3) * cw + i % 3];
                    const float4 vj = swin[(j / 3) * cw + j % 3];
                    const float a3[3] = {vi.x, vi.y, vi.z}, b3[3] = {vj.x, vj.y, vj.z};
                    const double wv = weight_exact64(ip, a3, b3, a.eps);
                    const double o = objective64(ip, a3, b3, wv, a.eps);
                    if (ni < 0 || o < best) {
                        best = o;
                        bw = wv;
                        ni = i;
                        nj = j;
                    }
                }
                if (++j == 9) j = ++i;
            }
            bi = ni;
            bj = nj;
            wClose = float(bw);
            wSet = true;
            if (a.fallbacks) atomicAdd(a.fallbacks + 1, 1ull);
        }
    }
    // stage-A style guard: an exact-zero distance must be a true colour match
    if (ok && qmin == 0.0f) {
#pragma unroll 1
        for (int k = 0; k < 9; ++k) {
            const float4 v = swin[(k / 3) * cw + k % 3];
            const float e0 = v.x - ip0, e1 = v.y - ip1, e2 = v.z - ip2;
            const float qk = __fmaf_rn(e2, e2, __fmaf_rn(e1, e1, __fmul_rn(e0, e0)));
            if (qk == 0.0f && !(e0 == 0.0f && e1 == 0.0f && e2 == 0.0f)) ok = false;
        }
    }
    uint32_t ia, ib;
    float w;
    if (ok) {
        ia = uint32_t(cy - 1 + bi / 3) * uint32_t(a.lw) + uint32_t(cx - 1 + bi % 3);
        ib = uint32_t(cy - 1 + bj / 3) * uint32_t(a.lw) + uint32_t(cx - 1 + bj % 3);
        const float ip[3] = {ip0, ip1, ip2};
        const float a3[3] = {ci.x, ci.y, ci.z}, b3[3] = {cj.x, cj.y, cj.z};
        w = wSet ? wClose : weight_exact64_f(ip, a3, b3, a.eps);
    } else {
        const int wx0 = max(0, cx - 1), wy0 = max(0, cy - 1);
        const int nwx = min(a.lw - 1, cx + 1) - wx0 + 1;
        const int nwy = min(a.lh - 1, cy + 1) - wy0 + 1;
        const float ip[3] = {ip0, ip1, ip2};
        PackedWindow pwin{packed + size_t(wy0 + 1) * pw + (wx0 + 1), pw, nwx};
        const Pick pk = pick_exact64(ip, pwin, nwx * nwy, a.eps);
        const int ar = pk.ai / nwx, br = pk.bi / nwx;
        ia = uint32_t(wy0 + ar) * uint32_t(a.lw) + uint32_t(wx0 + pk.ai - ar * nwx);
        ib = uint32_t(wy0 + br) * uint32_t(a.lw) + uint32_t(wx0 + pk.bi - br * nwx);
        w = float(pk.w);
        if (a.fallbacks) atomicAdd(a.fallbacks, 1ull);
    }
    if (a.params) {
        unsigned* o = reinterpret_cast<unsigned*>(a.params + p);
        o[0] = ia;
        o[1] = ib;
        o[2] = __float_as_uint(w);
    }
    if (a.lowT) {
        const bool clamp = a.clamp != 0;
        if (a.channels == 1) {
            a.out[p] = lerp_clamp(w, __ldg(a.lowT + ia), __ldg(a.lowT + ib), clamp);
        } else {
#pragma unroll
            for (int k = 0; k < 3; ++k)
                a.out[3 * p + k] = lerp_clamp(w, __ldg(a.lowT + 3 * size_t(ia) + k),
                                              __ldg(a.lowT + 3 * size_t(ib) + k), clamp);
        }
    }    if (a.errOut) {  // pixel_error of the clamped self reconstruction (jointopt.cpp:190)
        float r[3];
#pragma unroll
        for (int k = 0; k < 3; ++k)
            r[k] = lerp_clamp(w, __ldg(a.low + 3 * size_t(ia) + k), __ldg(a.low + 3 * size_t(ib) + k),
                              true);
        const float ipx[3] = {ip0, ip1, ip2};
        a.errOut[p] = pixel_error(ipx, r);
    }
}

}  // namespace

bool solve32x_supported(int mode, int S, int s) {
    return mode == GLU_MODE_EXACT && S == 3 && s >= 3;
}

cudaError_t launch_solve32x(glu_ctx* ctx, const SolveArgs& a, const float4* packed,
                            int forceFallback, const unsigned* nanFlag) {
    dim3 grid((a.W + kTX - 1) / kTX, (a.H + kTY - 1) / kTY);
    k_solve32x<<<grid, kThreads, 0, ctx->stream>>>(a, packed, forceFallback, nanFlag);
    ++ctx->launches;
    return cudaGetLastError();
}

}  // namespace glu_cu
