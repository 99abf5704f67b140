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
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cassert>
#include <cstdint>

#include "glu_internal.h"
#include "glu_math.cuh"

namespace glu_cu {

namespace {

#ifndef GLU_X_TY
#define GLU_X_TY 4  // warps per CTA (8: 0.7 % slower)
#endif
constexpr int kTX = 32, kTY = GLU_X_TY, kThreads = kTX * kTY;
constexpr int kPairs = 36;       // i < j over 9 candidates
#ifndef GLU_X_COMPACT
#define GLU_X_COMPACT 1  // the compact pair table (A/B knob; 0: 36 float4 slots per cell)
#endif
// float4 per owner cell, bank-spread (compact: 464 B; else 592 B)
constexpr int kCellStride = GLU_X_COMPACT ? 29 : 37;
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

// Packed fp32 pairs (sm_100 FMUL2 / FFMA2: two IEEE round-to-nearest
// operations per issued instruction, each lane bit-identical to the scalar
// mul / fma; glu_solve32f.cu).
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 pk2(float lo, float hi) {
    f32x2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void upk2(f32x2 v, float& lo, float& hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ f32x2 add2(f32x2 a, f32x2 b) {
    f32x2 r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f32x2 mul2(f32x2 a, f32x2 b) {
    f32x2 r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f32x2 fma2(f32x2 a, f32x2 b, f32x2 c) {
    f32x2 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

// The pair table of one owner cell: D'_ij (i < j) column by column, rows two
// at a time.  Compact layout (28 float4): the 16 two-row slots (column j's
// floor(j / 2) slots start at floor((j - 1)^2 / 4)) as float4 {x_i, x_i+1,
// y_i, y_i+1} at [0, 16) and float2 {z_i, z_i+1} at [16, 24) -- packed
// operands for one LDS.128 + one LDS.64 -- then the odd columns' last rows
// (j - 1, j) as plain {x, y, z, -} at 24 + (j - 1) / 2.  (The first version
// kept 36 float4 slots, column j at j (j - 1) / 2: 592 B per cell, 7 CTAs per
// SM at C3 instead of 8.)
__device__ __forceinline__ constexpr int col_base(int j) {
    return GLU_X_COMPACT ? (j - 1) * (j - 1) / 4 : j * (j - 1) / 2;
}
struct PairSlot {  // where the rows (i, i + 1), i even, of column j live
    const float4* xy;
    const float2* z;
};
__device__ __forceinline__ PairSlot pair_slot(const float4* tab, int i, int j) {
    if (GLU_X_COMPACT) {
        const int s = col_base(j) + i / 2;
        return PairSlot{tab + s, reinterpret_cast<const float2*>(tab + 16) + s};
    }
    return PairSlot{tab + col_base(j) + i, reinterpret_cast<const float2*>(tab + col_base(j) + i + 1)};
}
__device__ __forceinline__ const float4* single_slot(const float4* tab, int j) {  // (j - 1, j), j odd
    return GLU_X_COMPACT ? tab + 24 + (j - 1) / 2 : tab + col_base(j) + (j - 1);
}
__device__ __forceinline__ float3 tab_pair(const float4* tab, int i, int j) {
    if (!(i & 1) && i + 1 == j) {
        const float4 d = *single_slot(tab, j);
        return make_float3(d.x, d.y, d.z);
    }
    const PairSlot p = pair_slot(tab, i & ~1, j);
    const float* f = reinterpret_cast<const float*>(p.xy) + (i & 1);
    return make_float3(f[0], f[2], reinterpret_cast<const float*>(p.z)[i & 1]);
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
                const float3 d = tab_pair(tab, i, j);
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
    const float4* wcells;  // candidate cells of the tile's owner cells (+- 1), pitch cw;
                           // .w = the cell's LR index, or its 1-channel target value
    int cw;
};

enum Out { kOutParams = 0, kOutApply1 = 1, kOutGeneric = 2 };
#ifndef GLU_X_PCELLS
#define GLU_X_PCELLS 1  // e_j, q_j of candidates (3r, 3r + 1) in packed pairs (A/B knob)
#endif

// One HR pixel with guide colour (ip0, ip1, ip2): the pair search, tie
// recovery, weight and the fused epilogues.  `swin` = its owner cell's window
// (top-left candidate) in the staged cells, `tab` = the cell's pair table.
template <int OUT, int P>
__device__ __forceinline__ void solve_pixel(const SolveArgs& a, const float4* packed, const XTile& t,
                                            const float4* swin, const float4* tab,
                                            const float4* pwin, int forceFallback, size_t p, int cx,
                                            int cy, float ip0, float ip1, float ip2, size_t th) {
    // (pwin: the window in the pair cells -- position (r, c) holds the colours
    // of the staged cells (r, c) and (r, c + 1) as {x, x', y, y'}, {z, z'} --
    // so a window row's first two candidates are differenced and squared in
    // packed pairs, lane for lane the scalar sequence)
    // (p: the output index, th: the target offset -- both include this frame's
    // offset in a batched launch, which only the 1-ch video output uses)
    const int cw = P > 0 ? P : t.cw;

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
    f32x2 PE0 = 0, PE1 = 0, PE2 = 0, PQ = 0;  // candidates (3r, 3r + 1)
#pragma unroll
    for (int j = 0; j < 9; ++j) {
        float e0, e1, e2, qj;
        if (GLU_X_PCELLS && j % 3 != 2) {
            if (j % 3 == 0) {
                const float4* ps = pwin + 2 * ((j / 3) * cw);
                const ulonglong2 xy = *reinterpret_cast<const ulonglong2*>(ps);
                const f32x2 z = *reinterpret_cast<const f32x2*>(ps + 1);
                PE0 = add2(xy.x, pk2(-ip0, -ip0));
                PE1 = add2(xy.y, pk2(-ip1, -ip1));
                PE2 = add2(z, pk2(-ip2, -ip2));
                PQ = fma2(PE2, PE2, fma2(PE1, PE1, mul2(PE0, PE0)));
            }
            float o0, o1, o2, oq;  // the other lane
            if (j % 3 == 0) {
                upk2(PE0, e0, o0), upk2(PE1, e1, o1), upk2(PE2, e2, o2), upk2(PQ, qj, oq);
            } else {
                upk2(PE0, o0, e0), upk2(PE1, o1, e1), upk2(PE2, o2, e2), upk2(PQ, oq, qj);
            }
        } else {
            const float4 v = swin[(j / 3) * cw + j % 3];
            e0 = v.x - ip0, e1 = v.y - ip1, e2 = v.z - ip2;
            qj = __fmaf_rn(e2, e2, __fmaf_rn(e1, e1, __fmul_rn(e0, e0)));
        }
        const float qm = __fmaf_rn(qj, kOneMinusE, -1e-36f);
        qmin = fminf(qmin, qj);
        const float k1in = K1;
        float pend = 0.0f;  // keys are tracked two at a time: (0, 1), (2, 3), ...
        // rows (i, i + 1) of column j in packed pairs (e_j broadcast)
        const f32x2 E0 = pk2(e0, e0), E1 = pk2(e1, e1), E2 = pk2(e2, e2), Qm = pk2(qm, qm);
#pragma unroll
        for (int i = 0; i < j; i += 2) {
            if (i + 1 < j) {
                const PairSlot ps = pair_slot(tab, i, j);
                const ulonglong2 dxy = *reinterpret_cast<const ulonglong2*>(ps.xy);
                const f32x2 dz = *reinterpret_cast<const f32x2*>(ps.z);
                const f32x2 dn = fma2(E0, dxy.x, fma2(E1, dxy.y, mul2(E2, dz)));
                float n0, n1, t0, t1;
                upk2(dn, n0, n1);
                upk2(fma2(pk2(-n0, -n1), dn, Qm), t0, t1);
                track_key2(K1, K2, pack_key(t0, i, kmask), pack_key(t1, i + 1, kmask));
            } else {
                const float4 d = *single_slot(tab, j);
                const float dn = __fmaf_rn(e0, d.x, __fmaf_rn(e1, d.y, e2 * d.z));
                pend = pack_key(__fmaf_rn(-dn, dn, qm), i, kmask);
            }
        }
        const float kd = pack_key(qm, j, kmask);  // (j, j): w = 0, obj = q_j
        if (j & 1)
            track_key2(K1, K2, pend, kd);
        else
            track_key(K1, K2, kd);
        bj = K1 != k1in ? j : bj;
    }
    int bi = int(__float_as_uint(K1) & 15u);
    // (a NaN guide channel makes every key NaN: K1 stays +inf)
    bool ok = !forceFallback && K1 < kInf && (qmin >= 1e-27f || qmin == 0.0f);
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
    float w, wa = ci.w, wb = cj.w;
    if (ok) {
        const float ip[3] = {ip0, ip1, ip2};
        const float a3[3] = {ci.x, ci.y, ci.z}, b3[3] = {cj.x, cj.y, cj.z};
        w = wSet ? wClose : weight_exact64_f(ip, a3, b3, a.eps);
    } else {
        const uint3 r = solve_double(packed, a.lw, a.lh, a.eps, a.fallbacks, cx, cy, ip0, ip1, ip2);
        w = __uint_as_float(r.z);
        if (OUT == kOutApply1) {
            wa = __ldg(a.lowT + th + r.x);
            wb = __ldg(a.lowT + th + r.y);
        } else {
            wa = __uint_as_float(r.x);
            wb = __uint_as_float(r.y);
        }
    }
    if (OUT == kOutApply1) {  // the video path: 1-channel matte, no params
        a.out[p] = lerp_clamp(w, wa, wb, a.clamp != 0);
        return;
    }
    const uint32_t ia = __float_as_uint(wa), ib = __float_as_uint(wb);
    if (OUT == kOutParams || a.params) {
        unsigned* o = reinterpret_cast<unsigned*>(a.params + p);
        o[0] = ia + a.idxBase;
        o[1] = ib + a.idxBase;
        o[2] = __float_as_uint(w);
    }
    if (OUT == kOutGeneric) {
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
                r[k] = lerp_clamp(w, __ldg(a.low + 3 * size_t(ia) + k),
                                  __ldg(a.low + 3 * size_t(ib) + k), true);
            const float ipx[3] = {ip0, ip1, ip2};
            a.errOut[p] = pixel_error(ipx, r);
        }
    }
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

// A CTA solves a tile of kTX = 32 columns x tileH = kTY * rows rows; warp ty
// owns rows [ty * rows, (ty + 1) * rows).  Dynamic shared memory: [guide:
// tileH x 96 floats, one TMA (cp.async.bulk.tensor.2d) when useTma][pair
// table: maxCells x kCellStride][candidate cells: pitch x (mch + 2)].
template <int OUT, int P, bool BATCH>
__global__ void __launch_bounds__(kThreads, GLU_X_MIN_BLOCKS)
    k_solve32x(const __grid_constant__ CUtensorMap tmap, SolveArgs a, const float4* packed,
               int forceFallback, const unsigned* nanFlag, int maxCells, int rows, int useTma,
               FrameBatch fb) {
    // BATCH: frame blockIdx.z of a batch of video frames (glu_cu_upsample_frames;
    // k_solve32f's scheme); the single-frame instantiation compiles the offsets out
    const int fz = BATCH ? int(blockIdx.z) : 0;
    if (BATCH) {
        packed += size_t(fz) * fb.packed;
        nanFlag += fz;
    }
    const size_t fo = BATCH ? size_t(fz) * fb.px : 0, th = BATCH ? size_t(fz) * fb.lowT : 0,
                 hh = BATCH ? size_t(fz) * fb.high : 0;
    extern __shared__ __align__(1024) float xsm[];
    __shared__ __align__(8) unsigned long long bar;
    const int tileH = kTY * rows;
    float* gtile = xsm;
    float4* table = reinterpret_cast<float4*>(xsm + size_t(tileH) * 96);
    float4* wcells = table + maxCells * kCellStride;
    const int tx = threadIdx.x % kTX, ty = threadIdx.x / kTX;
    // (pair cells behind the cells: 2 float4 per position, the cells' pitch)
    float4* pcells = wcells + (P > 0 ? P : (kTX - 1) / a.s + 4) * ((tileH - 1) / a.s + 4);
    const int x0 = blockIdx.x * kTX, y0 = blockIdx.y * tileH;
    if (useTma && threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)),
                     "r"(unsigned(tileH * 96 * 4))
                     : "memory");
        if (BATCH)  // a 3-D map over the batch's frames
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(gtile)),
                "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(3 * x0), "r"(y0), "r"(fz),
                "r"(smem_u32(&bar))
                : "memory");
        else
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(gtile)),
                "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(3 * x0), "r"(y0), "r"(smem_u32(&bar))
                : "memory");
    }
    forceFallback |= int(__ldg(nanFlag));
    const int pw = a.lw + 2;  // h = 1
    const int ocx0 = div_s(x0, a), ocy0 = div_s(y0, a);
    const int ncw = div_s(min(x0 + kTX - 1, a.W - 1), a) - ocx0 + 1;
    const int nch = div_s(min(y0 + tileH - 1, a.H - 1), a) - ocy0 + 1;
    const float eps = a.epsf;
    const int cw = P > 0 ? P : ncw + 2;
    // packed cell (c - 1) of the LR grid is at padded index c; .w becomes what
    // the epilogue reads from a winning cell
    for (int k = threadIdx.x; k < cw * (nch + 2); k += kThreads) {
        const int r = k / cw, c = k - r * cw;
        if (c < ncw + 2) {
            float4 v = __ldg(packed + size_t(ocy0 + r) * pw + (ocx0 + c));
            const int lx = ocx0 + c - 1, ly = ocy0 + r - 1;
            const bool in = lx >= 0 && ly >= 0 && lx < a.lw && ly < a.lh;
            const unsigned li = in ? unsigned(ly) * unsigned(a.lw) + unsigned(lx) : 0u;
            v.w = OUT == kOutApply1 ? (in ? __ldg(a.lowT + th + li) : 0.0f) : __uint_as_float(li);
            wcells[k] = v;
            if (GLU_X_PCELLS && c < ncw + 1) {
                const float4 v1 = __ldg(packed + size_t(ocy0 + r) * pw + (ocx0 + c + 1));
                pcells[2 * k] = make_float4(v.x, v1.x, v.y, v1.y);
                pcells[2 * k + 1] = make_float4(v.z, v1.z, 0.0f, 0.0f);
            }
        }
    }
    if (!useTma) {  // the guide rows are not 16-byte aligned: staged by the threads
        for (int k = threadIdx.x; k < tileH * 96; k += kThreads) {
            const int r = k / 96, c = k - r * 96;
            const int y = y0 + r;
            gtile[k] = (y < a.H && x0 * 3 + c < a.W * 3)
                           ? __ldg(a.high + hh + 3 * (size_t(y) * a.W + x0) + c)
                           : 0.0f;
        }
    }
    __syncthreads();
    // thread t builds pair pr = t % 36 for cells t / 36, t / 36 + 7, ... (the
    // pair decode is paid once per thread)
    const int pr = int(threadIdx.x) % kPairs;
    const int ti = (pr >= 8) + (pr >= 15) + (pr >= 21) + (pr >= 26) + (pr >= 30) + (pr >= 33) +
                   (pr >= 35);
    const int tj = pr - (ti * 8 - ti * (ti - 1) / 2) + ti + 1;
    const int oi = (ti / 3) * cw + ti % 3, oj = (tj / 3) * cw + tj % 3;
    constexpr int kCellStep = kThreads / kPairs;  // cells per pass (the last threads idle)
    // (cell -> (ly, lx) advanced incrementally: kCellStep < ncw or one row step
    // at a time, no division per cell)
    int ly = 0, lx = int(threadIdx.x) / kPairs;
    while (lx >= ncw) {
        lx -= ncw;
        ++ly;
    }
    for (int cell = int(threadIdx.x) / kPairs; cell < ncw * nch && threadIdx.x < kCellStep * kPairs;
         cell += kCellStep) {
        const float4* w = wcells + ly * cw + lx;
        const float4 ci = w[oi], cj = w[oj];
        const float d0 = ci.x - cj.x, d1 = ci.y - cj.y, d2 = ci.z - cj.z;
        const float den = __fmaf_rn(d2, d2, __fmaf_rn(d1, d1, __fmaf_rn(d0, d0, eps)));
        // D' = D / sqrt(den): then obj_ij = q_j - (e_j . D')^2
        const float r = rsqrt_approx(den);
        float4* ctab = table + cell * kCellStride;
        if (!(ti & 1) && ti + 1 == tj) {
            *const_cast<float4*>(single_slot(ctab, tj)) = make_float4(d0 * r, d1 * r, d2 * r, 0.0f);
        } else {  // lane ti & 1 of the two-row slots
            const PairSlot ps = pair_slot(ctab, ti & ~1, tj);
            float* f = const_cast<float*>(reinterpret_cast<const float*>(ps.xy)) + (ti & 1);
            f[0] = d0 * r;
            f[2] = d1 * r;
            const_cast<float*>(reinterpret_cast<const float*>(ps.z))[ti & 1] = d2 * r;
        }
        lx += kCellStep;
        while (lx >= ncw) {
            lx -= ncw;
            ++ly;
        }
    }
    __syncthreads();
    if (useTma) {
        asm volatile(
            "{\n\t.reg .pred p;\n"
            "W:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t"
            "@!p bra W;\n}" ::"r"(smem_u32(&bar))
            : "memory");
    }
    const XTile t{wcells, cw};
    const int x = x0 + tx;
    if (x >= a.W) return;
    const int cx = div_s(x, a);
    const int yr = y0 + ty * rows;
    const int yEnd = min(yr + rows, a.H);
    const float* g = gtile + (ty * rows) * 96 + 3 * tx;
    size_t p = size_t(yr) * a.W + x + fo;
    // owner-cell row of the current row, advanced when y reaches yNext
    int cy = div_s(yr, a);
    int yNext = (cy + 1) * a.s;
    const float4* swin = wcells + (cy - ocy0) * cw + (cx - ocx0);
    const float4* tab = table + ((cy - ocy0) * ncw + (cx - ocx0)) * kCellStride;
    const float4* pwin = pcells + 2 * ((cy - ocy0) * cw + (cx - ocx0));
#pragma unroll 1
    for (int y = yr; y < yEnd; ++y, g += 96, p += a.W) {
        if (y == yNext) {
            ++cy;
            yNext += a.s;
            swin += cw;
            tab += ncw * kCellStride;
            pwin += 2 * cw;
        }
        solve_pixel<OUT, P>(a, packed, t, swin, tab, pwin, forceFallback, p, cx, cy, g[0], g[1], g[2],
                            th);
    }
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    }();
    return fn;
}

int max_pitch(int s) { return (kTX - 1) / s + 4; }

template <int OUT, int P>
cudaError_t launch_xp(glu_ctx* ctx, const SolveArgs& a, const float4* packed, int forceFallback,
                      const unsigned* nanFlag, const FrameBatch& fb) {
    // Rows per thread: more rows amortise a tile's staging (cells, pair
    // table, guide, two barriers) over more pixels, fewer rows give more
    // tiles and a smaller partial last wave.  Pick the count minimising waves
    // x (rows + staging cost) among those whose tile fits kSmemCap.  Owner
    // cells a tile can touch: ncw <= (kTX - 1) / s + 2, nch <= (tileH - 1) / s + 2.
    int dev = 0;
    cudaGetDevice(&dev);
    const int mcw = (kTX - 1) / a.s + 2;
    const int pitch = P > 0 ? P : max_pitch(a.s);
    const long tilesX = (a.W + kTX - 1) / kTX;
    auto smem_of = [&](int r) {
        const int mch = (kTY * r - 1) / a.s + 2;
        return sizeof(float) * size_t(kTY * r) * 96 +
               sizeof(float4) * (size_t(mcw * mch) * kCellStride +
                                 (GLU_X_PCELLS ? 3 : 1) * size_t(pitch) * (mch + 2));
    };
    thread_local int memo[6] = {-1, 0, 0, 0, -1, 1};  // device, s, W, H, key -> rows
    const int key = OUT * 64 + P;
    if (memo[0] != dev || memo[1] != a.s || memo[2] != a.W || memo[3] != a.H || memo[4] != key) {
        int nsm = 148, rows = 1;
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        float best = -1.0f;
        for (int r = 1; r <= kMaxRows; ++r) {
            const size_t sm = smem_of(r);
            if (r > 1 && sm > kSmemCap) break;
            cudaFuncSetAttribute(k_solve32x<OUT, P, false>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
            int per = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_solve32x<OUT, P, false>, kThreads,
                                                          sm);
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
        memo[4] = key;
        memo[5] = rows;
    }
#ifndef GLU_X_BATCH_ROWS
#define GLU_X_BATCH_ROWS 8  // rows per thread of a batched launch (no wave tail to fit; compact table: 6 / 7 / 8 = 0.1996 / 0.2007 / 0.1981 ms per 4K frame; 36-slot table: 5 / 6 / 7 / 8 = 0.2042 / 0.2000 / 0.2007 / 0.2029)
#endif
    // (as long as the taller tile respects kSmemCap: small scales keep the single-frame pick)
#ifndef GLU_X_ROWS
#define GLU_X_ROWS 0  // > 0: forces the single-frame rows per thread (A/B builds)
#endif
    if (GLU_X_ROWS > 0 && smem_of(GLU_X_ROWS) <= kSmemCap) memo[5] = GLU_X_ROWS;
    const int rows = GLU_X_BATCH_ROWS > 0 && fb.frames > 1 && GLU_X_BATCH_ROWS <= kMaxRows &&
                             smem_of(GLU_X_BATCH_ROWS) <= kSmemCap
                         ? GLU_X_BATCH_ROWS
                         : memo[5];
    const int tileH = kTY * rows;
    const int mch = (tileH - 1) / a.s + 2;
    const int maxCells = mcw * mch;
    CUtensorMap tmap{};
    int useTma = 0;
    if (a.W % 4 == 0 && (reinterpret_cast<uintptr_t>(a.high) & 15u) == 0) {
        if (auto enc = tensor_map_encoder()) {
            // (a batch: a third dimension over its frames, fb.high floats apart)
            const cuuint32_t rank = fb.frames > 1 ? 3u : 2u;
            const cuuint64_t dims[3] = {cuuint64_t(3) * a.W, cuuint64_t(a.H),
                                        cuuint64_t(fb.frames)};
            const cuuint64_t strides[2] = {cuuint64_t(12) * a.W, cuuint64_t(4) * fb.high};
            const cuuint32_t box[3] = {96u, cuuint32_t(tileH), 1u};
            const cuuint32_t estr[3] = {1u, 1u, 1u};
            useTma = (fb.frames == 1 || (fb.high * 4) % 16 == 0) &&
                     enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, const_cast<float*>(a.high),
                         dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
        }
    }
    const size_t smem = smem_of(rows);
    // (only the 1-ch video output is launched as a batch)
    constexpr bool kCanBatch = OUT == kOutApply1;
    const bool batch = kCanBatch && fb.frames > 1;
    if (fb.frames > 1 && !batch) return cudaErrorInvalidValue;
    auto kern = batch ? k_solve32x<OUT, P, kCanBatch> : k_solve32x<OUT, P, false>;
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    dim3 grid(unsigned(tilesX), (a.H + tileH - 1) / tileH, unsigned(fb.frames));
    kern<<<grid, kThreads, smem, ctx->stream>>>(tmap, a, packed, forceFallback, nanFlag, maxCells,
                                                rows, useTma, fb);
    ++ctx->launches;
    return cudaGetLastError();
}

template <int OUT>
cudaError_t launch_xo(glu_ctx* ctx, const SolveArgs& a, const float4* packed, int forceFallback,
                      const unsigned* nanFlag, const FrameBatch& fb) {
    switch (max_pitch(a.s)) {  // s = 8: 7; s = 16: 5; s >= 32: 4
        case 4: return launch_xp<OUT, 4>(ctx, a, packed, forceFallback, nanFlag, fb);
        case 5: return launch_xp<OUT, 5>(ctx, a, packed, forceFallback, nanFlag, fb);
        case 7: return launch_xp<OUT, 7>(ctx, a, packed, forceFallback, nanFlag, fb);
        default: return launch_xp<OUT, 0>(ctx, a, packed, forceFallback, nanFlag, fb);
    }
}

}  // namespace

bool solve32x_supported(int mode, int S, int s) {
    return mode == GLU_MODE_EXACT && S == 3 && s >= 3;
}

cudaError_t launch_solve32x(glu_ctx* ctx, const SolveArgs& a, const float4* packed,
                            int forceFallback, const unsigned* nanFlag, const FrameBatch& fb) {
    if (a.params && !a.lowT && !a.errOut)
        return launch_xo<kOutParams>(ctx, a, packed, forceFallback, nanFlag, fb);
    if (!a.params && a.lowT && a.channels == 1 && !a.errOut)
        return launch_xo<kOutApply1>(ctx, a, packed, forceFallback, nanFlag, fb);
    return launch_xo<kOutGeneric>(ctx, a, packed, forceFallback, nanFlag, fb);
}

}  // namespace glu_cu
