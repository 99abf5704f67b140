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

#include <cassert>

#include "glu_internal.h"
#include "glu_math.cuh"

namespace glu_cu {

namespace {

#ifndef GLU_X_TY
#define GLU_X_TY 4  // warps per CTA (8: 0.7 % slower)
#endif
constexpr int kTX = 32, kTY = GLU_X_TY, kThreads = kTX * kTY;
constexpr int kPairs = 36;       // i < j over 9 candidates
constexpr int kCellStride = 37;  // float4 per owner cell (592 B: bank-spread)
constexpr int kMaxRows = 8;               // pixels per thread (rows y, y + kTY, ...): 1..8
constexpr int kSmemCap = 40 * 1024;       // per CTA, so that GLU_X_MIN_BLOCKS CTAs fit
constexpr float kStageCost = 0.3f;        // a tile's staging, in units of one row of pixels
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

// A pair's key: t with its low 4 mantissa bits replaced by the row index i
// (the perturbation is below 15 ulp; NaN stays NaN).  `mask` = 0xfffffff0 is
// held in a register so that (t & mask) | i is one LOP3 with i as immediate.
__device__ __forceinline__ float pack_key(float t, int i, unsigned mask) {
    unsigned r;
    asm("lop3.b32 %0, %1, %2, %3, 0xEC;" : "=r"(r) : "r"(__float_as_uint(t)), "r"(unsigned(i)),
        "r"(mask));
    return __uint_as_float(r);
}

// Smallest (K1) and second smallest (K2) key so far; a NaN key changes
// neither (fminf / fmaxf return the other operand).
__device__ __forceinline__ void track_key(float& K1, float& K2, float k) {
    K2 = fmaxf(fminf(K2, k), K1);
    K1 = fminf(K1, k);
}

__device__ __forceinline__ float fmax_nan(float a, float b) {  // NaN if either is NaN
    float r;
    asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    return r;
}

// Two keys at once (5 instructions, three-input min): the second smallest of
// {K1 <= K2, a, b} is max(min(K2, a, b), min(K1, max(a, b))); with max
// propagating NaN a NaN key drops out (the one-key update for the other).
__device__ __forceinline__ void track_key2(float& K1, float& K2, float a, float b) {
    K2 = fmaxf(fminf(fminf(K2, a), b), fminf(K1, fmax_nan(a, b)));
    K1 = fminf(fminf(K1, a), b);
}

// Lexicographic pair k (i <= j over 9 candidates: rows start at 0, 9, 17,
// 24, 30, 35, 39, 42, 44) -> (i, j).
__device__ __forceinline__ void lex_pair(int k, int& i, int& j) {
    i = (k >= 9) + (k >= 17) + (k >= 24) + (k >= 30) + (k >= 35) + (k >= 39) + (k >= 42) +
        (k >= 44);
    j = k - (i * 9 - i * (i - 1) / 2) + i;
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
#define GLU_X_MIN_BLOCKS 8  // 64 registers: 32 warps per SM (8 CTAs of 4 warps)
#endif

// Offset of window candidate j (row j / 3, column j % 3) in a staged window
// of pitch cw; (j * 11) >> 5 == j / 3 for j < 9.
__device__ __forceinline__ int woff(int j, int cw) {
    const int r = (j * 11) >> 5;
    return r * cw + (j - 3 * r);
}

// The close-call resolution (rare: a few pixels in 10^4; kept out of line so
// that it does not add register pressure to the scan).  Returns the pick
// (ok = false: an off-grid close pair, the pixel takes the double path).
struct ClosePick {
    int bi, bj;
    float w;
    bool ok, wSet;
};

__device__ __noinline__ ClosePick resolve_close(const float4* swin, const float4* tab, int cw,
                                                float ip0, float ip1, float ip2, float lim,
                                                unsigned kmask, int bi, int bj, double eps,
                                                unsigned long long* counters) {
    constexpr float kOneMinusE = 1.0f - kCE * kU;
    const float4 ci = swin[woff(bi, cw)], cj = swin[woff(bj, cw)];
    bool ok = true, wSet = false;
    float wClose = 0.0f;
    // rare: the pairs whose key is within lim (bit k = lexicographic
    // pair k, i <= j, the winner included) hold the reference's first
    // argmin (every other pair's objective exceeds the winner's): if
    // they all carry the winner's colour tuple, the first of them is
    // the pick; otherwise they are evaluated in double, in
    // lexicographic order (ascending bits).  The keys are recomputed
    // by the scan's instruction sequence, so they are the same values.
    unsigned long long close = 0;
#pragma unroll
    for (int j = 0; j < 9; ++j) {
        const float4 v = swin[(j / 3) * cw + j % 3];
        const float e0 = v.x - ip0, e1 = v.y - ip1, e2 = v.z - ip2;
        const float qj = __fmaf_rn(e2, e2, __fmaf_rn(e1, e1, __fmul_rn(e0, e0)));
        const float qm = __fmaf_rn(qj, kOneMinusE, -1e-36f);
#pragma unroll
        for (int i = 0; i <= j; ++i) {
            float key;
            if (i < j) {
                const float4 d = tab[i * 8 - i * (i - 1) / 2 + (j - i - 1)];
                const float dn = __fmaf_rn(e0, d.x, __fmaf_rn(e1, d.y, e2 * d.z));
                key = pack_key(__fmaf_rn(-dn, dn, qm), i, kmask);
            } else {
                key = pack_key(qm, j, kmask);
            }
            if (key <= lim) close |= 1ull << (i * 9 - i * (i - 1) / 2 + (j - i));
        }
    }
    bool mixed = false;
    int fi = -1, fj = -1;
    for (unsigned long long m = close; m; m &= m - 1) {
        int i, j;
        lex_pair(__ffsll(static_cast<long long>(m)) - 1, i, j);
        const float4 vi = swin[(i / 3) * cw + i % 3], vj = swin[(j / 3) * cw + j % 3];
        if (!(vi.x < kInf && vj.x < kInf)) ok = false;  // off-grid member (+inf sentinel)
        const bool same = same_rgb(vi, ci) && same_rgb(vj, cj);
        mixed |= !same;
        if (same && fi < 0) {
            fi = i;
            fj = j;
        }
    }
    if (ok && !mixed) {
        bi = fi;  // identical colours: identical objectives and weight
        bj = fj;
    } else if (ok && mixed) {
        const float ip[3] = {ip0, ip1, ip2};
        double best = 0, bw = 0;
        int ni = -1, nj = -1;
        for (unsigned long long m = close; m; m &= m - 1) {
            int i, j;
            lex_pair(__ffsll(static_cast<long long>(m)) - 1, i, j);
            const float4 vi = swin[(i / 3) * cw + i % 3];
            const float4 vj = swin[(j / 3) * cw + j % 3];
            const float a3[3] = {vi.x, vi.y, vi.z}, b3[3] = {vj.x, vj.y, vj.z};
            const double wv = weight_exact64(ip, a3, b3, eps);
            const double o = objective64(ip, a3, b3, wv, eps);
            if (ni < 0 || o < best) {
                best = o;
                bw = wv;
                ni = i;
                nj = j;
            }
        }
        bi = ni;
        bj = nj;
        wClose = float(bw);
        wSet = true;
        if (counters) atomicAdd(counters + 1, 1ull);
    }
    return ClosePick{bi, bj, wClose, ok, wSet};
}

// The reference's exact double-precision path for one pixel (NaN inputs,
// underflow-sized distances, off-grid close pairs, forced fallback): out of
// line like resolve_close.  Returns {a, b, bits(w)}.
__device__ __noinline__ uint3 solve_double(const float4* packed, int lw, int lh, double eps,
                                           unsigned long long* counters, int cx, int cy,
                                           float ip0, float ip1, float ip2) {
    const int pw = lw + 2;  // h = 1
    const int wx0 = max(0, cx - 1), wy0 = max(0, cy - 1);
    const int nwx = min(lw - 1, cx + 1) - wx0 + 1;
    const int nwy = min(lh - 1, cy + 1) - wy0 + 1;
    const float ip[3] = {ip0, ip1, ip2};
    PackedWindow pwin{packed + size_t(wy0 + 1) * pw + (wx0 + 1), pw, nwx};
    const Pick pk = pick_exact64(ip, pwin, nwx * nwy, eps);
    const int ar = pk.ai / nwx, br = pk.bi / nwx;
    if (counters) atomicAdd(counters, 1ull);
    return make_uint3(uint32_t(wy0 + ar) * uint32_t(lw) + uint32_t(wx0 + pk.ai - ar * nwx),
                      uint32_t(wy0 + br) * uint32_t(lw) + uint32_t(wx0 + pk.bi - br * nwx),
                      __float_as_uint(float(pk.w)));
}

// The tile's staged candidate cells and pair table (shared memory).
struct XTile {
    const float4* wcells;  // candidate cells of the tile's owner cells (+- 1), cw per row
    const float4* table;   // kCellStride float4 per owner cell: D' of its 36 pairs
    int cw, ncw, ocx0, ocy0;
#ifdef GLU_X_DEBUG
    int nrow, nwin, ntab;  // owner-cell rows, staged cells, table float4s (bounds checks)
#endif
};

// One HR pixel (x, y) with guide colour (ip0, ip1, ip2): the pair search,
// tie recovery, weight and the fused epilogues.
__device__ __forceinline__ void solve_pixel(const SolveArgs& a, const float4* packed, const XTile& t,
                                            int forceFallback, int x, int y, float ip0, float ip1,
                                            float ip2) {
    const int cw = t.cw;
    const size_t p = size_t(y) * a.W + x;
    const int cx = div_s(x, a), cy = div_s(y, a);
    // the window in shared memory: candidate j is swin[(j / 3) * cw + j % 3]
    const float4* swin = t.wcells + (cy - t.ocy0) * cw + (cx - t.ocx0);
    const float4* tab = t.table + ((cy - t.ocy0) * t.ncw + (cx - t.ocx0)) * kCellStride;
#ifdef GLU_X_DEBUG  // bounds of the staged window / table (debug builds)
    assert(cy >= t.ocy0 && cx >= t.ocx0 && cx - t.ocx0 < t.ncw && cy - t.ocy0 + 2 < t.nrow + 2);
    assert((cy - t.ocy0 + 2) * cw + (cx - t.ocx0) + 2 < t.nwin);
    assert(((cy - t.ocy0) * t.ncw + (cx - t.ocx0) + 1) * kCellStride <= t.ntab);
#endif

    // j-outer scan: pair (i, j) needs only e_j = I_j - I_p and q_j = |e_j|^2
    // (D'_ij = D_ij / sqrt(den) comes from the cell's table: obj = q_j -
    // (e_j . D')^2), so nothing per candidate stays live across the scan.
    //
    // Each pair is reduced to one key: t = q_j (1 - kE) - 1e-36 - (e_j . D')^2
    // (the fp32 objective lowered by its error bound) with the low 4 mantissa
    // bits replaced by i (the pair's row within column j).  |key - obj| is
    // within (kE +- 57u) q_j (objective 22u, t's roundings 3u, the packing
    // 15 ulp = 30u), so a key is a lower bound of its pair's objective and
    // key + kT q_j an upper bound.  The scan keeps the smallest key K1 (its
    // column bj, its row in the low bits) and the second smallest K2; if K2 >
    // K1 + kT q_bj the winner's objective is provably below every other pair's
    // and it is the reference's unique argmin.  Otherwise (close call, tie)
    // the close pairs are re-checked in the reference's lexicographic order
    // below.  Off-grid pairs give NaN keys (inf - inf, inf * 0), which the
    // NaN-ignoring min / max updates skip.
    constexpr float kE = kCE * kU;
    constexpr float kOneMinusE = 1.0f - kE;         // exact: 1 - 2^-18
    constexpr float kT = (2.0f * kCE + 8.0f) * kU;  // >= kE + 57u + the rounding of K1 + kT q
    // 0xfffffff0, opaque to the compiler (W > 0) so it stays in a register
    const unsigned kmask = 0xfffffff0u | (unsigned(a.W) >> 31);
    float qmin = kInf, K1 = kInf, K2 = kInf;
    int bj = 0;
#pragma unroll
    for (int j = 0; j < 9; ++j) {
        const float4 v = swin[(j / 3) * cw + j % 3];
        const float e0 = v.x - ip0, e1 = v.y - ip1, e2 = v.z - ip2;
        const float qj = __fmaf_rn(e2, e2, __fmaf_rn(e1, e1, __fmul_rn(e0, e0)));
        const float qm = __fmaf_rn(qj, kOneMinusE, -1e-36f);
        qmin = fminf(qmin, qj);
        const float k1in = K1;
        float pend = 0.0f;  // keys are tracked two at a time: (0, 1), (2, 3), ...
#pragma unroll
        for (int i = 0; i < j; ++i) {
            const float4 d = tab[i * 8 - i * (i - 1) / 2 + (j - i - 1)];
            const float dn = __fmaf_rn(e0, d.x, __fmaf_rn(e1, d.y, e2 * d.z));
            const float key = pack_key(__fmaf_rn(-dn, dn, qm), i, kmask);
            if (i & 1)
                track_key2(K1, K2, pend, key);
            else
                pend = key;
        }
        const float kd = pack_key(qm, j, kmask);  // (j, j): w = 0, obj = q_j
        if (j & 1)
            track_key2(K1, K2, pend, kd);
        else
            track_key(K1, K2, kd);
        bj = K1 != k1in ? j : bj;
    }
    int bi = int(__float_as_uint(K1) & 15u);
    bool ok = !forceFallback && K1 < kInf && ip0 == ip0 && ip1 == ip1 && ip2 == ip2 &&
              (qmin >= 1e-27f || qmin == 0.0f);
    // An exact colour match I_j0 == I_p: the pairs (i, j0) have objective 0
    // in double (w = 0, v = 0) and every other pair a positive one (a
    // non-matching colour has a nonzero double distance, even where its fp32
    // distance underflows), so the reference's pick is the lexicographically
    // first: (i0, j0), i0 the first in-grid candidate, j0 the first exact
    // match.  (Every LR sample pixel lands here.)  A zero fp32 distance
    // without an exact match (underflow) takes the double path.
    bool exactZero = false;
    if (ok && qmin == 0.0f) {
        int j0 = -1;
#pragma unroll
        for (int k = 8; k >= 0; --k) {
            const float4 v = swin[(k / 3) * cw + k % 3];
            j0 = (v.x == ip0 && v.y == ip1 && v.z == ip2) ? k : j0;
        }
        ok = j0 >= 0;
        exactZero = ok;
        bi = (cy == 0 ? 3 : 0) + (cx == 0 ? 1 : 0);
        bj = max(j0, 0);
    }
    bool wSet = false;  // w settled in double over the close set
    float wClose = 0.0f;
    if (ok && !exactZero) {
        // the winner's q (the scan's instruction sequence, so the same value)
        const float4 cj = swin[woff(bj, cw)];
        const float eb0 = cj.x - ip0, eb1 = cj.y - ip1, eb2 = cj.z - ip2;
        const float qb = __fmaf_rn(eb2, eb2, __fmaf_rn(eb1, eb1, __fmul_rn(eb0, eb0)));
        const float lim = K1 + __fmaf_rn(kT, qb, 2e-36f);
        if (K2 <= lim) {
#ifdef GLU_X_COUNT_RECHECK
            if (a.fallbacks) atomicAdd(a.fallbacks + 1, 1ull);
#endif
            const ClosePick c =
                resolve_close(swin, tab, cw, ip0, ip1, ip2, lim, kmask, bi, bj, a.eps, a.fallbacks);
            ok = c.ok;
            bi = c.bi;
            bj = c.bj;
            wSet = c.wSet;
            wClose = c.w;
        }
    }
    // (the pair's colours are re-read here rather than kept live across the
    // out-of-line call, which would spill them on every pixel)
    const float4 ci = swin[woff(bi, cw)], cj = swin[woff(bj, cw)];
    uint32_t ia, ib;
    float w;
    if (ok) {
        const int ri = (bi * 11) >> 5, rj = (bj * 11) >> 5;
        ia = uint32_t(cy - 1 + ri) * uint32_t(a.lw) + uint32_t(cx - 1 + bi - 3 * ri);
        ib = uint32_t(cy - 1 + rj) * uint32_t(a.lw) + uint32_t(cx - 1 + bj - 3 * rj);
        const float ip[3] = {ip0, ip1, ip2};
        const float a3[3] = {ci.x, ci.y, ci.z}, b3[3] = {cj.x, cj.y, cj.z};
        w = wSet ? wClose : weight_exact64_f(ip, a3, b3, a.eps);
    } else {
        const uint3 r = solve_double(packed, a.lw, a.lh, a.eps, a.fallbacks, cx, cy, ip0, ip1, ip2);
        ia = r.x;
        ib = r.y;
        w = __uint_as_float(r.z);
    }
    if (a.params) {
        unsigned* o = reinterpret_cast<unsigned*>(a.params + p);
        o[0] = ia + a.idxBase;
        o[1] = ib + a.idxBase;
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

__global__ void __launch_bounds__(kThreads, GLU_X_MIN_BLOCKS)
    k_solve32x(SolveArgs a, const float4* packed, int forceFallback, const unsigned* nanFlag,
               int maxCells, int maxWin, int rows) {
    extern __shared__ float4 smem[];
    float4* table = smem;                         // maxCells * kCellStride
    float4* wcells = smem + maxCells * kCellStride;  // the tile's candidate cells
    forceFallback |= int(__ldg(nanFlag));
    const int pw = a.lw + 2;  // h = 1
    const int tileH = kTY * rows;  // a CTA solves a kTX x tileH tile
    const int x0 = blockIdx.x * kTX, y0 = blockIdx.y * tileH;
    const int ocx0 = div_s(x0, a), ocy0 = div_s(y0, a);
    const int ncw = div_s(min(x0 + kTX - 1, a.W - 1), a) - ocx0 + 1;
    const int nch = div_s(min(y0 + tileH - 1, a.H - 1), a) - ocy0 + 1;
    const float eps = a.epsf;
    const int cw = ncw + 2;
    // the first pixel's guide colour is requested before the staging barriers
    const int x = x0 + (threadIdx.x % kTX), yb = y0 + (threadIdx.x / kTX);
    const bool xin = x < a.W;
    float g0 = 0.0f, g1 = 0.0f, g2 = 0.0f;
    if (xin && yb < a.H) {
        const float* g = a.high + 3 * (size_t(yb) * a.W + x);
        g0 = __ldg(g);
        g1 = __ldg(g + 1);
        g2 = __ldg(g + 2);
    }
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
    constexpr int kCellStep = kThreads / kPairs;  // cells per pass (the last threads idle)
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

#ifdef GLU_X_DEBUG
    assert(ncw * nch <= maxCells && cw * (nch + 2) <= maxWin);
    const XTile t{wcells, table, cw, ncw, ocx0, ocy0, nch, cw * (nch + 2), maxCells * kCellStride};
#else
    const XTile t{wcells, table, cw, ncw, ocx0, ocy0};
#endif
#pragma unroll 1
    for (int k = 0; k < rows; ++k) {
        const int y = yb + k * kTY;
        if (k > 0 && xin && y < a.H) {  // (prefetching one scan ahead measured slower)
            const float* g = a.high + 3 * (size_t(y) * a.W + x);
            g0 = __ldg(g);
            g1 = __ldg(g + 1);
            g2 = __ldg(g + 2);
        }
        const float ip0 = g0, ip1 = g1, ip2 = g2;
        if (xin && y < a.H) solve_pixel(a, packed, t, forceFallback, x, y, ip0, ip1, ip2);
    }
}

}  // namespace

bool solve32x_supported(int mode, int S, int s) {
    return mode == GLU_MODE_EXACT && S == 3 && s >= 3;
}

cudaError_t launch_solve32x(glu_ctx* ctx, const SolveArgs& a, const float4* packed,
                            int forceFallback, const unsigned* nanFlag) {
    // Rows per thread: more rows amortise a tile's staging (cells, pair
    // table, two barriers) over more pixels, fewer rows give more tiles and a
    // smaller partial last wave.  Pick the count minimising waves x (rows +
    // staging cost) among those whose tile fits kSmemCap.  Owner cells a tile
    // can touch: ncw <= (kTX - 1) / s + 2, nch <= (tileH - 1) / s + 2.
    int dev = 0;
    cudaGetDevice(&dev);
    const int mcw = (kTX - 1) / a.s + 2;
    const long tilesX = (a.W + kTX - 1) / kTX;
    thread_local int memo[5] = {-1, 0, 0, 0, 1};  // device, s, W, H -> rows
    if (memo[0] != dev || memo[1] != a.s || memo[2] != a.W || memo[3] != a.H) {
        int nsm = 148, rows = 1;
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        float best = -1.0f;
        for (int r = 1; r <= kMaxRows; ++r) {
            const int mch = (kTY * r - 1) / a.s + 2;
            const size_t sm =
                sizeof(float4) * (size_t(mcw * mch) * kCellStride + (mcw + 2) * (mch + 2));
            if (r > 1 && sm > kSmemCap) break;
            int per = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_solve32x, kThreads, sm);
            const long slots = long(max(per, 1)) * nsm;
            const long tiles = tilesX * ((a.H + kTY * r - 1) / (kTY * r));
            const float cost = float((tiles + slots - 1) / slots) * (float(r) + kStageCost);
            if (best < 0.0f || cost <= best) {
                best = cost;
                rows = r;
            }
        }
        memo[0] = dev;
        memo[1] = a.s;
        memo[2] = a.W;
        memo[3] = a.H;
        memo[4] = rows;
    }
    const int rows = memo[4];
    const int mch = (kTY * rows - 1) / a.s + 2;
    const int maxCells = mcw * mch;
    const size_t smem = sizeof(float4) * (size_t(maxCells) * kCellStride + (mcw + 2) * (mch + 2));
    if (smem > 48 * 1024)  // one row per thread at s = 3: 12 x 4 cells fit in 48 KB
        cudaFuncSetAttribute(k_solve32x, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    dim3 grid(unsigned(tilesX), (a.H + kTY * rows - 1) / (kTY * rows));
    k_solve32x<<<grid, kThreads, smem, ctx->stream>>>(a, packed, forceFallback, nanFlag, maxCells,
                                                        (mcw + 2) * (mch + 2), rows);
    ++ctx->launches;
    return cudaGetLastError();
}

}  // namespace glu_cu
