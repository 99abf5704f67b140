// glu_solve32f.cu -- Fast mode, S = 3: tile-staged candidates and a keyed
// closed-form stage B (fp32 filter + fp64 verify, bit-exact with the reference).
//
// The reference's pixelFast (upsample.cpp:49-71): a = first argmin of the
// distance |I_j - I_p|; then for every candidate j, w_j = d_j / (d_a + d_j +
// eps) and obj_j = |w_j I_a + (1 - w_j) I_j - I_p|^2 + eps w_j^2; b = first
// argmin of obj_j; all in double.
//
// Stage A is k_solve32's (glu_solve32.cu): fp32 squared distances, the first
// argmin, and a check that no candidate of a different colour lies within
// 32u q_min of it (else the pixel takes the double path).
//
// Stage B uses the closed form of the objective at w_j = d_j / s_j,
// s_j = d_a + eps + d_j (with q = d^2, c_j = e_a . e_j, e = I - I_p):
//     obj_j = (A q_j + B d_j c_j) / s_j^2,
//     A = q_a + (d_a + eps)^2 + eps,  B = 2 (d_a + eps),
// 12 instructions per candidate (k_solve32's form needs 22).  Each candidate
// becomes one key: the fp32 value lowered by G q_j / s_j^2, G = 96u (A + B
// d_a), with the candidate's index in the low 4 mantissa bits.  The fp32
// error of the closed form is below 49u T_j / s_j^2 (T_j = q_j (A + B d_a);
// the rounding of the key and the 15-ulp packing add 35u), and F = 2^-44 (M^2
// + eps) covers the reference's own double rounding (<= 2^-45.8 M^2 + 2^-51
// eps, M the largest |channel| of the pixel and its window), so a key is a
// lower bound of the reference's objective and key + 2 G q_j / s_j^2 + F an
// upper bound.  The smallest key K1 and the second
// smallest K2 decide b unless K2 is within the winner's upper bound; such
// close calls re-derive the keys and settle the close set in double in index
// order.  The stored weight is the reference's (float)(d_b / (d_a + d_b +
// eps)), verified in double (weight_fast_verified, glu_math.cuh).
//
// Layout: like k_solve32x, a CTA stages its tile's candidate cells (the
// packed LR image: float4 cells with a +inf border, .w = the cell's largest
// |channel|) in shared memory once and solves 1-8 rows of pixels per thread;
// the rare paths (close calls, the double path) are out of line with scalar
// arguments, so the scans stay in registers.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>

#include "glu_internal.h"
#include "glu_math.cuh"

namespace glu_cu {

namespace {

#ifndef GLU_F_TY
#define GLU_F_TY 4  // warps per CTA (rows of a tile per row step); 8 measured 1.3 % slower
#endif
constexpr int kTX = 32, kTY = GLU_F_TY, kThreads = kTX * kTY;
#ifndef GLU_F_MAX_ROWS
#define GLU_F_MAX_ROWS 8
#endif
constexpr int kMaxRows = GLU_F_MAX_ROWS;
constexpr float kStageCost = 0.3f;  // a tile's staging, in units of one row of pixels
constexpr float kU = 5.9604645e-08f;  // 2^-24
constexpr float kCA = 32.0f;          // stage A relative margin (in u)
constexpr float kG = 96.0f * kU;      // key offset, in u (A + B d_a)
constexpr float kF = 5.684342e-14f;   // 2^-44
constexpr float kInf = __builtin_huge_valf();
// Stage B's fp32 keys stay finite while every |channel| of the pixel and its
// tile is below 2^29 (A q_j and B d_j c_j <= 2 q_a q_j < 2^127); larger
// values take the double path.
constexpr float kMaxMag = 536870912.0f;

__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float fast_sqrt(float q) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(q));
    return r;
}
__device__ __forceinline__ float fmax_nan(float a, float b) {  // NaN if either is NaN
    float r;
    asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    return r;
}

// Packed fp32 pairs (sm_100 FADD2 / FMUL2 / FFMA2): two IEEE round-to-nearest
// operations per issued instruction, each lane bit-identical to the scalar
// add / mul / fma -- the kernel is bound by instruction issue, not by the FP32
// pipe.  A pair lives in an aligned 64-bit register pair (lo = first).
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
__device__ __forceinline__ float key_pack(float t, int j, unsigned mask) {  // (t & mask) | j
    unsigned r;
    asm("lop3.b32 %0, %1, %2, %3, 0xEC;" : "=r"(r) : "r"(__float_as_uint(t)), "r"(unsigned(j)),
        "r"(mask));
    return __uint_as_float(r);
}

// Pair table (compile-time pitches, s >= 8): per owner cell of the tile its 9
// window candidates as 5 slots of two candidates (2k, 2k + 1; slot 4 = {8, 8}):
// float4 {x0, x1, y0, y1} x 5, then float2 {z0, z1} x 5, so a pixel reads a
// slot with LDS.128 + LDS.64 straight into packed operands.  9 float4 per cell
// (144 B: the cells a warp reads at once fall in different banks), at a pitch
// of P - 2 owner cells per row.
constexpr int kCellF4 = 9;
// (GNU mode -- stage A only -- measured 2.5 % slower with the table: scalar)
template <int MODE, int P>
__host__ __device__ constexpr bool use_pairs() { return P > 0 && MODE == GLU_MODE_FAST; }
// GNU mode instead reads a pair-cell copy of the staged cells (position (r, c)
// = cells (r, c), (r, c + 1) interleaved: {x, x', y, y'}, {z, z'}): a window
// row's first two candidates in packed pairs, nothing to build per owner cell.
#ifndef GLU_F_GNU_PCELLS
#define GLU_F_GNU_PCELLS 1
#endif
template <int MODE, int P>
__host__ __device__ constexpr bool use_pcells() {
    return GLU_F_GNU_PCELLS && P > 0 && MODE == GLU_MODE_GNU;
}
#ifndef GLU_F_PK_A
#define GLU_F_PK_A 1  // stage A in packed pairs (A/B knob)
#endif
#ifndef GLU_F_PK_B
#define GLU_F_PK_B 1  // stage B in packed pairs (A/B knob)
#endif

__device__ __forceinline__ int div_s(int v, const SolveArgs& a) {
    return a.sdiv ? int(__umulhi(unsigned(v), a.sdiv)) : v / a.s;
}

__device__ __forceinline__ bool same_rgb(float4 a, float4 b) {
    return a.x == b.x && a.y == b.y && a.z == b.z;
}

// Offset of window candidate j (row j / 3, column j % 3) in a staged window of
// pitch cw; (j * 11) >> 5 == j / 3 for j < 9.
__device__ __forceinline__ int woff(int j, int cw) {
    const int r = (j * 11) >> 5;
    return r * cw + (j - 3 * r);
}

// Candidate j's key (see the header): the packed (B d_j c_j + (A - G) q_j) / s_j^2.  `mask` = 0xfffffff0 is held in a
// register so that (t & mask) | j is one LOP3.  Off-grid candidates (q = inf)
// give NaN keys.
// (b0, b1, b2) = B e_a, so the dot is B c_j directly.
__device__ __forceinline__ float fast_key(float e0, float e1, float e2, float qj, float b0,
                                          float b1, float b2, float at, float Ap, int j,
                                          unsigned mask) {
    const float bc = __fmaf_rn(e2, b2, __fmaf_rn(e1, b1, __fmul_rn(e0, b0)));
    const float dj = fast_sqrt(qj);
    const float nl = __fmaf_rn(dj, bc, __fmul_rn(Ap, qj));
    const float sj = __fadd_rn(at, dj);
    const float t = __fmul_rn(nl, rcp_approx(__fmul_rn(sj, sj)));
    return key_pack(t, j, mask);
}

// Smallest (K1) and second smallest (K2) key; NaN keys change neither.
__device__ __forceinline__ void track_key(float& K1, float& K2, float k) {
    K2 = fmaxf(fminf(K2, k), K1);
    K1 = fminf(K1, k);
}
// Two keys at once: second smallest of {K1 <= K2, a, b} = max(min(K2, a, b),
// min(K1, max(a, b))), with max propagating NaN (a NaN key drops out).
__device__ __forceinline__ void track_key2(float& K1, float& K2, float a, float b) {
    K2 = fmaxf(fminf(fminf(K2, a), b), fminf(K1, fmax_nan(a, b)));
    K1 = fminf(fminf(K1, a), b);
}

// The truncated window of the packed image as the reference's raster list.
struct PackedWindow {
    const float4* win;
    int pw, nwx;
    __device__ __forceinline__ const float* operator[](int i) const {
        const int r = i / nwx, q = i - r * nwx;
        return reinterpret_cast<const float*>(win + r * pw + q);
    }
};

// ---- rare paths, out of line (scalar arguments) ----------------------------

// The reference's double-precision pixelFast (upsample.cpp:49-71) for one
// pixel: NaN inputs, underflow-sized distances, uncertain stage-A picks,
// off-grid close members, forced fallback.  Returns {a, b, bits(w)}.
template <int MODE>
__device__ __noinline__ uint3 solve_double_fast(const float4* packed, int lw, int lh, double eps,
                                                unsigned long long* counters, int cx, int cy,
                                                float ip0, float ip1, float ip2) {
    const int pw = lw + 2;  // h = 1
    const int wx0 = max(0, cx - 1), wy0 = max(0, cy - 1);
    const int nwx = min(lw - 1, cx + 1) - wx0 + 1;
    const int nwy = min(lh - 1, cy + 1) - wy0 + 1;
    const float ip[3] = {ip0, ip1, ip2};
    PackedWindow pwin{packed + size_t(wy0 + 1) * pw + (wx0 + 1), pw, nwx};
    const Pick pk = MODE == GLU_MODE_GNU ? pick_gnu64(ip, pwin, nwx * nwy)
                                         : pick_fast64(ip, pwin, nwx * nwy, eps);
    const int ar = pk.ai / nwx, br = pk.bi / nwx;
    if (counters) atomicAdd(counters, 1ull);
    return make_uint3(uint32_t(wy0 + ar) * uint32_t(lw) + uint32_t(wx0 + pk.ai - ar * nwx),
                      uint32_t(wy0 + br) * uint32_t(lw) + uint32_t(wx0 + pk.bi - br * nwx),
                      __float_as_uint(float(pk.w)));
}

struct CloseFast {
    int jb;
    float w;
    bool ok, wExact;
};

// Stage-B close call: the candidates whose key is within lim hold the
// reference's first argmin (every other objective exceeds the winner's).  The
// keys are re-derived by the scan's instruction sequence (the same values).
// All of the winner's colour: the first of them; else the set is settled in
// double, in index order; an off-grid member sends the pixel to the double
// path.
__device__ __noinline__ CloseFast resolve_close_fast(const float4* swin, int cw, float ip0,
                                                     float ip1, float ip2, float at, float b0,
                                                     float b1, float b2, float Ap, float lim,
                                                     unsigned kmask, int ja, int jb, double eps,
                                                     unsigned long long* counters) {
    const float4 ca = swin[woff(ja, cw)], cb = swin[woff(jb, cw)];
    CloseFast r{jb, 0.0f, true, false};
    unsigned close = 0;
    bool mixed = false;
#pragma unroll
    for (int j = 0; j < 9; ++j) {
        const float4 v = swin[woff(j, cw)];
        const float d0 = v.x - ip0, d1 = v.y - ip1, d2 = v.z - ip2;
        const float qj = __fmaf_rn(d2, d2, __fmaf_rn(d1, d1, __fmul_rn(d0, d0)));
        const float key = fast_key(d0, d1, d2, qj, b0, b1, b2, at, Ap, j, kmask);
        if (key <= lim) {
            if (!(qj < kInf)) r.ok = false;
            close |= 1u << j;
            mixed |= !same_rgb(v, cb);
        }
    }
    if (!r.ok) return r;
    if (!mixed) {
        r.jb = __ffs(close) - 1;  // identical colours: identical objectives
        return r;
    }
    const float ip[3] = {ip0, ip1, ip2};
    const float a3[3] = {ca.x, ca.y, ca.z};
    const double dA = dist64(ip, a3);
    double best = 0, bw = 0;
    int bj = -1;
    for (unsigned m = close; m; m &= m - 1) {
        const int j = __ffs(m) - 1;
        const float4 v = swin[woff(j, cw)];
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
    r.jb = bj;
    r.w = float(bw);
    r.wExact = true;
    if (counters) atomicAdd(counters + 1, 1ull);
    return r;
}

// (float) of the reference's weight for (a, b) when the verified estimate is
// ambiguous (probability ~2^-24 per pixel): IEEE sqrt / division.
__device__ __noinline__ float weight_fast_ieee(float ip0, float ip1, float ip2, float4 ca,
                                               float4 cb, double eps) {
    const float ip[3] = {ip0, ip1, ip2};
    const float a3[3] = {ca.x, ca.y, ca.z}, b3[3] = {cb.x, cb.y, cb.z};
    const double dA = dist64(ip, a3), dB = dist64(ip, b3);
    return float(dB / (dA + dB + eps));
}

// ---- the kernel ---------------------------------------------------------------
//
// A CTA solves a tile of kTX = 32 columns x tileH = kTY * rows rows; warp ty
// owns the tile's rows [ty * rows, (ty + 1) * rows), one pixel per thread per
// row.  Before the rows are solved the CTA stages in shared memory:
//   * the tile's guide pixels (tileH x 96 floats), loaded by one TMA
//     (cp.async.bulk.tensor.2d, completion on an mbarrier) when the image rows
//     are 16-byte aligned, else by the threads;
//   * the candidate cells of the tile's owner cells +- 1 (the packed LR image)
//     at a pitch of P cells (a compile-time constant for the common scales, so
//     every candidate's offset is an immediate), with .w replaced by what the
//     epilogue needs from a winning cell: its LR index (params) or the
//     1-channel target value (the video path's fused apply);
//   * the tile's largest |channel| (k_pack_low's .w) for the rounding floor F.

// kOutParamsErr: the joint loop's initial solve (params + the self error map,
// jointopt.cpp:187-190) -- the reconstruction uses the winning cells' staged
// colours (the LR image itself) instead of gathering them again.
enum Out { kOutParams = 0, kOutApply1 = 1, kOutGeneric = 2, kOutParamsErr = 3 };

struct FTile {
    const float4* wcells;  // staged cells, pitch P (or cw when P = 0)
    int cw, ocx0, ocy0;
};

template <int P>
__device__ __forceinline__ int pitch_of(const FTile& t) { return P > 0 ? P : t.cw; }

// MODE: GLU_MODE_FAST, or GLU_MODE_GNU (stage A only: b = a, w = 1;
// upsample.cpp:93-104).  `swin` = the owner cell's window (top-left candidate),
// `wM` = the tile's largest |channel|.
template <int MODE, int OUT, int P>
__device__ __forceinline__ void solve_pixel(const SolveArgs& a, const float4* packed, const FTile& t,
                                            const float4* swin, const float4* ptab, float wM,
                                            int forceFallback, int x, int y, float ip0, float ip1,
                                            float ip2, size_t fo, size_t th) {
    // (fo / th: this frame's output / target offsets in a batched launch)
    const size_t p = size_t(y) * size_t(a.W) + size_t(x) + fo;
    const int cw = pitch_of<P>(t);

    // ---- stage A: a = first argmin |I_j - I_p| (compared as squares) -------
    // Each candidate's q_j as a key with its index in the low 4 mantissa bits
    // (<= 15 ulp = 30u): K1a (smallest) gives a = the first argmin of the fp32
    // distances up to keys within 30u of each other, and K2a (second
    // smallest) screens for the near ties that need the exact check below.
    const unsigned kmask = 0xfffffff0u | (unsigned(a.W) >> 31);  // opaque: a register
    float K1a = kInf, K2a = kInf, pa = 0.0f;
    // (P > 0) the candidates two at a time from the owner cell's pair table:
    // e = I_j - I_p and q_j for slot k's two candidates in packed registers,
    // lane for lane the scalar operations below
    f32x2 E0[5], E1[5], E2[5], Q[5];
    float keys[9];
    if (use_pairs<MODE, P>()) {
        const f32x2 n0 = pk2(-ip0, -ip0), n1 = pk2(-ip1, -ip1), n2 = pk2(-ip2, -ip2);
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            const ulonglong2 sxy = *reinterpret_cast<const ulonglong2*>(ptab + k);
            const f32x2 sz = reinterpret_cast<const f32x2*>(ptab + 5)[k];
            float q0, q1;
            if (GLU_F_PK_A) {
                E0[k] = add2(sxy.x, n0);
                E1[k] = add2(sxy.y, n1);
                E2[k] = add2(sz, n2);
                Q[k] = fma2(E2[k], E2[k], fma2(E1[k], E1[k], mul2(E0[k], E0[k])));
                upk2(Q[k], q0, q1);
            } else {
                float x0, x1, y0, y1, z0, z1;
                upk2(sxy.x, x0, x1);
                upk2(sxy.y, y0, y1);
                upk2(sz, z0, z1);
                x0 -= ip0, x1 -= ip0, y0 -= ip1, y1 -= ip1, z0 -= ip2, z1 -= ip2;
                q0 = __fmaf_rn(z0, z0, __fmaf_rn(y0, y0, __fmul_rn(x0, x0)));
                q1 = __fmaf_rn(z1, z1, __fmaf_rn(y1, y1, __fmul_rn(x1, x1)));
                E0[k] = pk2(x0, x1), E1[k] = pk2(y0, y1), E2[k] = pk2(z0, z1), Q[k] = pk2(q0, q1);
            }
            const float k0 = key_pack(q0, 2 * k, kmask);
            if (k < 4)
                track_key2(K1a, K2a, k0, key_pack(q1, 2 * k + 1, kmask));
            else
                track_key(K1a, K2a, k0);
        }
    } else if (use_pcells<MODE, P>()) {
        // (ptab = the window in the pair cells)
        const f32x2 n0 = pk2(-ip0, -ip0), n1 = pk2(-ip1, -ip1), n2 = pk2(-ip2, -ip2);
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            const float4* ps = ptab + 2 * (r * cw);
            const ulonglong2 sxy = *reinterpret_cast<const ulonglong2*>(ps);
            const f32x2 sz = *reinterpret_cast<const f32x2*>(ps + 1);
            const f32x2 e0 = add2(sxy.x, n0), e1 = add2(sxy.y, n1), e2 = add2(sz, n2);
            float q0, q1;
            upk2(fma2(e2, e2, fma2(e1, e1, mul2(e0, e0))), q0, q1);
            keys[3 * r] = key_pack(q0, 3 * r, kmask);
            keys[3 * r + 1] = key_pack(q1, 3 * r + 1, kmask);
            const float4 v = swin[r * cw + 2];
            const float d0 = v.x - ip0, d1 = v.y - ip1, d2 = v.z - ip2;
            keys[3 * r + 2] = key_pack(
                __fmaf_rn(d2, d2, __fmaf_rn(d1, d1, __fmul_rn(d0, d0))), 3 * r + 2, kmask);
        }
#pragma unroll
        for (int j = 0; j < 8; j += 2) track_key2(K1a, K2a, keys[j], keys[j + 1]);
        track_key(K1a, K2a, keys[8]);
    } else {
#pragma unroll
        for (int j = 0; j < 9; ++j) {
            const float4 v = swin[woff(j, cw)];
            const float d0 = v.x - ip0, d1 = v.y - ip1, d2 = v.z - ip2;
            const float qq = __fmaf_rn(d2, d2, __fmaf_rn(d1, d1, __fmul_rn(d0, d0)));
            const float key = key_pack(qq, j, kmask);
            if (j & 1)
                track_key2(K1a, K2a, pa, key);
            else if (j == 8)
                track_key(K1a, K2a, key);
            else
                pa = key;
        }
    }
    const int ja = int(__float_as_uint(K1a) & 15u);
    const float4 ca = swin[woff(ja, cw)];
    const float ea0 = ca.x - ip0, ea1 = ca.y - ip1, ea2 = ca.z - ip2;
    const float m1 = __fmaf_rn(ea2, ea2, __fmaf_rn(ea1, ea1, __fmul_rn(ea0, ea0)));  // q_a
    const bool exactA = ca.x == ip0 && ca.y == ip1 && ca.z == ip2;
    // NaN inputs and underflow-sized distances go to the exact path.
    // (a NaN guide channel makes every q_j and key NaN: K1a stays +inf)
    bool ok = !forceFallback && K1a < kInf && (m1 >= 1e-27f || exactA);
    // any other candidate within (1 + 32u) q_a has a key within K1a (1 + 128u)
    if (ok && K2a <= __fmaf_rn(K1a, 128.0f * kU, K1a) + 2e-36f) {
        const float lim = __fmaf_rn(m1, kCA * kU, m1) + 1e-36f;
#pragma unroll 1
        for (int j = 0; j < 9; ++j) {
            const float4 v = swin[woff(j, cw)];
            const float d0 = v.x - ip0, d1 = v.y - ip1, d2 = v.z - ip2;
            const float qq = __fmaf_rn(d2, d2, __fmaf_rn(d1, d1, __fmul_rn(d0, d0)));
            if (j != ja && !(qq > lim) && !same_rgb(v, ca)) ok = false;
        }
    }
    int jb = ja;
    float4 cb = ca;
    float w = 0.0f;
    bool wExact = false;  // w settled in double (close-set path)
    if (MODE == GLU_MODE_FAST && ok && !exactA) {
        // (exact match I_a == I_p: b = a, the first exact zero, and w = 0)
        // ---- stage B: b = first argmin of the objective at w_j ---------------
        const float eps = a.epsf;
        const float da = fast_sqrt(m1);
        const float at = da + eps;
        const float A = __fadd_rn(__fmaf_rn(at, at, m1), eps);
        const float B = at + at;
        const float G = kG * __fmaf_rn(B, da, A);
        const float Ap = A - G;
        const float b0 = B * ea0, b1 = B * ea1, b2 = B * ea2;
        float K1 = kInf, K2 = kInf, pend = 0.0f;
        if (use_pairs<MODE, P>()) {  // fast_key for two candidates per instruction
            const f32x2 B0 = pk2(b0, b0), B1 = pk2(b1, b1), B2 = pk2(b2, b2);
            const f32x2 at2 = pk2(at, at), Ap2 = pk2(Ap, Ap);
#pragma unroll
            for (int k = 0; k < 5; ++k) {
                float q0, q1;
                upk2(Q[k], q0, q1);
                float k0, k1 = 0.0f;
                if (GLU_F_PK_B) {
                    const f32x2 bc = fma2(E2[k], B2, fma2(E1[k], B1, mul2(E0[k], B0)));
                    const f32x2 dj = pk2(fast_sqrt(q0), k < 4 ? fast_sqrt(q1) : 0.0f);
                    const f32x2 nl = fma2(dj, bc, mul2(Ap2, Q[k]));
                    const f32x2 sj = add2(at2, dj);
                    float s0, s1;
                    upk2(mul2(sj, sj), s0, s1);
                    float t0, t1;
                    upk2(mul2(nl, pk2(rcp_approx(s0), k < 4 ? rcp_approx(s1) : 0.0f)), t0, t1);
                    k0 = key_pack(t0, 2 * k, kmask);
                    if (k < 4) k1 = key_pack(t1, 2 * k + 1, kmask);
                } else {
                    float x0, x1, y0, y1, z0, z1;
                    upk2(E0[k], x0, x1);
                    upk2(E1[k], y0, y1);
                    upk2(E2[k], z0, z1);
                    k0 = fast_key(x0, y0, z0, q0, b0, b1, b2, at, Ap, 2 * k, kmask);
                    if (k < 4) k1 = fast_key(x1, y1, z1, q1, b0, b1, b2, at, Ap, 2 * k + 1, kmask);
                }
                if (k < 4)
                    track_key2(K1, K2, k0, k1);
                else
                    track_key(K1, K2, k0);
            }
        } else {
#pragma unroll
            for (int j = 0; j < 9; ++j) {
                const float4 v = swin[woff(j, cw)];
                const float d0 = v.x - ip0, d1 = v.y - ip1, d2 = v.z - ip2;
                const float qj = __fmaf_rn(d2, d2, __fmaf_rn(d1, d1, __fmul_rn(d0, d0)));
                const float key = fast_key(d0, d1, d2, qj, b0, b1, b2, at, Ap, j, kmask);
                if (j & 1)
                    track_key2(K1, K2, pend, key);
                else if (j == 8)
                    track_key(K1, K2, key);
                else
                    pend = key;
            }
        }
        jb = int(__float_as_uint(K1) & 15u);
        // the winner's upper bound: K1 + 2 G q_b / s_b^2 + F
        cb = swin[woff(jb, cw)];
        const float qb = __fmaf_rn(cb.z - ip2, cb.z - ip2,
                                   __fmaf_rn(cb.y - ip1, cb.y - ip1, __fmul_rn(cb.x - ip0, cb.x - ip0)));
        const float sb = __fadd_rn(at, fast_sqrt(qb));
        const float m = fmaxf(wM, fmaxf(fabsf(ip0), fmaxf(fabsf(ip1), fabsf(ip2))));
        const float F = kF * __fmaf_rn(m, m, eps);
        const float lim = K1 + __fmaf_rn(2.0f * G * qb, rcp_approx(__fmul_rn(sb, sb)), F);
        if (!(K1 < kInf) || !(m < kMaxMag)) {
            ok = false;
        } else if (K2 <= lim) {
            const CloseFast c = resolve_close_fast(swin, cw, ip0, ip1, ip2, at, b0, b1, b2, Ap, lim,
                                                   kmask, ja, jb, a.eps, a.fallbacks);
            ok = c.ok;
            jb = c.jb;
            wExact = c.wExact;
            w = c.w;
            cb = swin[woff(jb, cw)];
        }
    }
    // the staged .w of the winning cells: LR indices, or the 1-channel target
    float wa = ca.w, wb = cb.w;
    float4 la = ca, lb = cb;  // the winning cells' LR colours (kOutParamsErr)
    if (ok) {
        if (MODE == GLU_MODE_GNU) {
            w = 1.0f;
        } else if (!wExact) {
            bool wok = false;
            w = weight_fast_lean(ip0, ip1, ip2, ca, cb, a.eps, &wok);
            if (!wok) w = weight_fast_ieee(ip0, ip1, ip2, ca, cb, a.eps);
        }
    } else {
        const uint3 r =
            solve_double_fast<MODE>(packed, a.lw, a.lh, a.eps, a.fallbacks, div_s(x, a), div_s(y, a),
                                    ip0, ip1, ip2);
        w = __uint_as_float(r.z);
        if (OUT == kOutApply1) {
            wa = __ldg(a.lowT + th + r.x);
            wb = __ldg(a.lowT + th + r.y);
        } else {
            wa = __uint_as_float(r.x);
            wb = __uint_as_float(r.y);
            if (OUT == kOutParamsErr) {
                const float* pa = a.low + 3 * size_t(r.x);
                const float* pb = a.low + 3 * size_t(r.y);
                la = make_float4(pa[0], pa[1], pa[2], 0.0f);
                lb = make_float4(pb[0], pb[1], pb[2], 0.0f);
            }
        }
    }
    if (OUT == kOutApply1) {  // the video path: 1-channel matte, no params
        a.out[p] = lerp_clamp(w, wa, wb, a.clamp != 0);
        return;
    }
    const uint32_t ia = __float_as_uint(wa), ib = __float_as_uint(wb);
    if (OUT == kOutParams || OUT == kOutParamsErr || a.params) {
        unsigned* o = reinterpret_cast<unsigned*>(a.params + p);
        o[0] = ia + a.idxBase;
        o[1] = ib + a.idxBase;
        o[2] = __float_as_uint(w);
    }
    if (OUT == kOutParamsErr) {  // pixel_error of the clamped self reconstruction
        const float r[3] = {lerp_clamp(w, la.x, lb.x, true), lerp_clamp(w, la.y, lb.y, true),
                            lerp_clamp(w, la.z, lb.z, true)};
        const float ipx[3] = {ip0, ip1, ip2};
        a.errOut[p] = pixel_error(ipx, r);
    }
    if (OUT == kOutGeneric) {
        if (a.lowT) {
            const bool clamp = a.clamp != 0;
            if (a.channels == 1) {
                a.out[p] = lerp_clamp(w, __ldg(a.lowT + th + ia), __ldg(a.lowT + th + ib), clamp);
            } else {
#pragma unroll
                for (int k = 0; k < 3; ++k)
                    a.out[3 * p + k] = lerp_clamp(w, __ldg(a.lowT + th + 3 * size_t(ia) + k),
                                                  __ldg(a.lowT + th + 3 * size_t(ib) + k), clamp);
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

#ifndef GLU_F_MIN_BLOCKS
#define GLU_F_MIN_BLOCKS 8  // 64 registers: 32 warps per SM (8 CTAs of 4 warps)
#endif

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

// Dynamic shared memory: [guide: tileH x 96 floats][cells: P x (mch + 2)]
// [Fast mode, P > 0: pair table, (P - 2) x mch owner cells x kCellF4 float4].
// `tmap` is a 2-D tensor map of the guide (3 W floats x H rows, box 96 x
// tileH) when useTma != 0.
template <int MODE, int OUT, int P, bool BATCH>
__global__ void __launch_bounds__(kThreads, GLU_F_MIN_BLOCKS)
    k_solve32f(const __grid_constant__ CUtensorMap tmap, SolveArgs a, const float4* packed,
               int forceFallback, const unsigned* nanFlag, int rows, int useTma, FrameBatch fb) {
    // BATCH: frame blockIdx.z of a batch of frames (glu_cu_upsample_frames);
    // the single-frame instantiation compiles the offsets out
    const int fz = BATCH ? int(blockIdx.z) : 0;
    if (BATCH) {
        packed += size_t(fz) * fb.packed;
        nanFlag += fz;
    }
    const size_t fo = BATCH ? size_t(fz) * fb.px : 0, th = BATCH ? size_t(fz) * fb.lowT : 0,
                 hh = BATCH ? size_t(fz) * fb.high : 0;
    extern __shared__ __align__(1024) float smem[];
    __shared__ __align__(8) unsigned long long bar;
    __shared__ float warpMax[kTY];
    const int tileH = kTY * rows;
    float* gtile = smem;                                                  // tileH x 96
    float4* wcells = reinterpret_cast<float4*>(smem + size_t(tileH) * 96);
    const int tx = threadIdx.x % kTX, ty = threadIdx.x / kTX;
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
    const int cw = P > 0 ? P : ncw + 2;
    GLU_DCHECK(ncw + 2 <= cw && nch <= (kTY * rows - 1) / a.s + 2);
    // packed cell (c - 1) of the LR grid is at padded index c
    float m = 0.0f;
    for (int k = threadIdx.x; k < cw * (nch + 2); k += kThreads) {
        const int r = k / cw, c = k - r * cw;
        if (c < ncw + 2) {
            float4 v = __ldg(packed + size_t(ocy0 + r) * pw + (ocx0 + c));
            m = fmaxf(m, v.w);
            const int lx = ocx0 + c - 1, ly = ocy0 + r - 1;
            const bool in = lx >= 0 && ly >= 0 && lx < a.lw && ly < a.lh;
            const unsigned li = in ? unsigned(ly) * unsigned(a.lw) + unsigned(lx) : 0u;
            v.w = OUT == kOutApply1 ? (in ? __ldg(a.lowT + th + li) : 0.0f) : __uint_as_float(li);
            wcells[k] = v;
            if (use_pcells<MODE, P>() && c < ncw + 1) {  // pair cells behind the cells
                const float4 v1 = __ldg(packed + size_t(ocy0 + r) * pw + (ocx0 + c + 1));
                float4* pc = wcells + P * ((tileH - 1) / a.s + 4) + 2 * k;
                pc[0] = make_float4(v.x, v1.x, v.y, v1.y);
                pc[1] = make_float4(v.z, v1.z, 0.0f, 0.0f);
            }
        }
    }
    float4* ptab = nullptr;
    if (use_pcells<MODE, P>()) ptab = wcells + P * ((tileH - 1) / a.s + 4);
    if (use_pairs<MODE, P>()) {
        // the pair table from the packed image (no barrier between the two
        // stagings): owner cell (r, c)'s slots at kCellF4 * (r * (P - 2) + c)
        const int mch = (tileH - 1) / a.s + 2;
        ptab = wcells + P * (mch + 2);
        for (int k = threadIdx.x; k < (P - 2) * nch * 5; k += kThreads) {
            const int cell = k / 5, sl = k - 5 * cell;
            const int r = cell / (P - 2), c = cell - r * (P - 2);
            if (c < ncw) {
                const int j0 = 2 * sl, j1 = sl < 4 ? j0 + 1 : j0;
                const int r0 = (j0 * 11) >> 5, r1 = (j1 * 11) >> 5;
                const float4 v0 = __ldg(packed + size_t(ocy0 + r + r0) * pw + (ocx0 + c + j0 - 3 * r0));
                const float4 v1 = __ldg(packed + size_t(ocy0 + r + r1) * pw + (ocx0 + c + j1 - 3 * r1));
                ptab[kCellF4 * cell + sl] = make_float4(v0.x, v1.x, v0.y, v1.y);
                reinterpret_cast<float2*>(ptab + kCellF4 * cell + 5)[sl] = make_float2(v0.z, v1.z);
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
    // the tile's largest |channel| (a NaN .w counts as +inf: every pixel then
    // settles its close calls in double)
    m = m == m ? m : kInf;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (tx == 0) warpMax[ty] = m;
    __syncthreads();
    float wM = warpMax[0];
#pragma unroll
    for (int k = 1; k < kTY; ++k) wM = fmaxf(wM, warpMax[k]);
    if (useTma) {
        asm volatile(
            "{\n\t.reg .pred p;\n"
            "W:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t"
            "@!p bra W;\n}" ::"r"(smem_u32(&bar))
            : "memory");
    }
    const FTile t{wcells, cw, ocx0, ocy0};
    const int x = x0 + tx;
    if (x >= a.W) return;
    const int yr = y0 + ty * rows;
    const int yEnd = min(yr + rows, a.H);
    const float* g = gtile + (ty * rows) * 96 + 3 * tx;
    // owner-cell row of the current row, advanced when y reaches yNext
    const int cy0 = div_s(yr, a);
    int yNext = (cy0 + 1) * a.s;
    // the owner cell's window in the staged cells (its top-left candidate)
    // and its slots in the pair table.  Fast carries the window as an offset
    // (0.1347 vs 0.1364 ms per fused 4K frame), GNU as a pointer (0.0626 vs
    // 0.0644 ms): one is dead code per instantiation.
    constexpr bool kCarryPtr = MODE == GLU_MODE_GNU;
    const int cxr = div_s(x, a) - ocx0;
    int co = (cy0 - ocy0) * cw + cxr;
    const float4* swinp = wcells + co;
    const float4* pt = use_pairs<MODE, P>()
                           ? ptab + kCellF4 * ((cy0 - ocy0) * (P - 2) + cxr)
                           : (use_pcells<MODE, P>() ? ptab + 2 * co : ptab);
#pragma unroll 1
    for (int y = yr; y < yEnd; ++y, g += 96) {
        if (y == yNext) {
            yNext += a.s;
            if (kCarryPtr)
                swinp += cw;
            else
                co += cw;
            if (use_pairs<MODE, P>()) pt += kCellF4 * (P - 2);
            if (use_pcells<MODE, P>()) pt += 2 * cw;
        }
        const float4* swin = kCarryPtr ? swinp : wcells + co;
        GLU_DCHECK(swin - wcells >= 0 && swin - wcells + 2 * cw + 2 < cw * (nch + 2));
        constexpr bool kPairs = use_pairs<MODE, P>();  // (no commas inside the macro)
        GLU_DCHECK(!kPairs || (pt - ptab >= 0 && pt - ptab < kCellF4 * (P - 2) * nch &&
                               (pt - ptab) / kCellF4 % (P - 2) < ncw));
        solve_pixel<MODE, OUT, P>(a, packed, t, swin, pt, wM, forceFallback, x, y, g[0], g[1], g[2],
                                  fo, th);
    }
}

}  // namespace

bool solve32f_supported(int mode, int S) {
    return (mode == GLU_MODE_FAST || mode == GLU_MODE_GNU) && S == 3;
}

namespace {

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

// Cells a tile touches: ncw <= (kTX - 1) / s + 2 (plus the +-1 border).
int max_pitch(int s) { return (kTX - 1) / s + 4; }

template <int MODE, int OUT, int P>
cudaError_t launch_fp(glu_ctx* ctx, const SolveArgs& a, const float4* packed, int forceFallback,
                      const unsigned* nanFlag, const FrameBatch& fb) {
    // Rows per thread: the count minimising waves x (rows + staging cost),
    // as k_solve32x.
    int dev = 0;
    cudaGetDevice(&dev);
    const int pitch = P > 0 ? P : max_pitch(a.s);
    const long tilesX = (a.W + kTX - 1) / kTX;
    auto smem_of = [&](int r) {
        const int mch = (kTY * r - 1) / a.s + 2;
        return sizeof(float) * size_t(kTY * r) * 96 + sizeof(float4) * size_t(pitch) * (mch + 2) +
               (use_pairs<MODE, P>() ? sizeof(float4) * size_t(kCellF4) * (P - 2) * mch : 0) +
               (use_pcells<MODE, P>() ? 2 * sizeof(float4) * size_t(pitch) * (mch + 2) : 0);
    };
    thread_local int memo[6] = {-1, 0, 0, 0, -1, 1};  // device, s, W, H, MODE/OUT/P -> rows
    const int key = (MODE * 4 + OUT) * 64 + P;
    if (memo[0] != dev || memo[1] != a.s || memo[2] != a.W || memo[3] != a.H || memo[4] != key) {
        int nsm = 148, rows = 1;
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        float best = -1.0f;
        for (int r = 1; r <= kMaxRows; ++r) {
            int per = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_solve32f<MODE, OUT, P, false>,
                                                          kThreads, smem_of(r));
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
#ifndef GLU_F_ROWS
#define GLU_F_ROWS 0  // 0: picked per launch (A/B builds force a count)
#endif
#ifndef GLU_F_BATCH_ROWS
#define GLU_F_BATCH_ROWS 10  // a batch has no wave tail to fit: taller tiles (8 / 10 / 12 / 14 / 16: 67.8 / 68.8 / 67.9 / 66.2 / 63.9 k HR Mpix/s)
#endif
    const int rows = GLU_F_ROWS > 0 ? GLU_F_ROWS
                                    : (OUT == kOutApply1 && fb.frames > 1
                                           ? (MODE == GLU_MODE_FAST ? GLU_F_BATCH_ROWS : 12)
                                           : memo[5]);
    const int tileH = kTY * rows;
    // TMA needs 16-byte aligned rows (3 W floats) and base; else the threads stage the guide.
    CUtensorMap tmap{};
    int useTma = 0;
#ifndef GLU_F_TMA
#define GLU_F_TMA 1
#endif
    if (GLU_F_TMA && a.W % 4 == 0 && (reinterpret_cast<uintptr_t>(a.high) & 15u) == 0) {
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
    auto kern = batch ? k_solve32f<MODE, OUT, P, kCanBatch> : k_solve32f<MODE, OUT, P, false>;
    if (fb.frames > 1 && !batch) return cudaErrorInvalidValue;
    if (smem > 48 * 1024) {
        const cudaError_t e =
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (e != cudaSuccess) return e;
    }
    dim3 grid(unsigned(tilesX), (a.H + tileH - 1) / tileH, unsigned(fb.frames));
    kern<<<grid, kThreads, smem, ctx->stream>>>(tmap, a, packed, forceFallback, nanFlag, rows,
                                                useTma, fb);
    ++ctx->launches;
    return cudaGetLastError();
}

template <int MODE, int OUT>
cudaError_t launch_fo(glu_ctx* ctx, const SolveArgs& a, const float4* packed, int forceFallback,
                      const unsigned* nanFlag, const FrameBatch& fb) {
    switch (max_pitch(a.s)) {  // s = 8 (C3, C2): 7; s = 16 (C4): 5; s >= 32: 4
        case 4: return launch_fp<MODE, OUT, 4>(ctx, a, packed, forceFallback, nanFlag, fb);
        case 5: return launch_fp<MODE, OUT, 5>(ctx, a, packed, forceFallback, nanFlag, fb);
        case 7: return launch_fp<MODE, OUT, 7>(ctx, a, packed, forceFallback, nanFlag, fb);
        default: return launch_fp<MODE, OUT, 0>(ctx, a, packed, forceFallback, nanFlag, fb);
    }
}

template <int MODE>
cudaError_t launch_f(glu_ctx* ctx, const SolveArgs& a, const float4* packed, int forceFallback,
                     const unsigned* nanFlag, const FrameBatch& fb) {
    if (a.params && !a.lowT && !a.errOut)
        return launch_fo<MODE, kOutParams>(ctx, a, packed, forceFallback, nanFlag, fb);
    if (a.params && !a.lowT && a.errOut)
        return launch_fo<MODE, kOutParamsErr>(ctx, a, packed, forceFallback, nanFlag, fb);
    if (!a.params && a.lowT && a.channels == 1 && !a.errOut)
        return launch_fo<MODE, kOutApply1>(ctx, a, packed, forceFallback, nanFlag, fb);
    return launch_fo<MODE, kOutGeneric>(ctx, a, packed, forceFallback, nanFlag, fb);
}

}  // namespace

cudaError_t launch_solve32f(glu_ctx* ctx, const SolveArgs& a, const float4* packed,
                            int forceFallback, const unsigned* nanFlag, const FrameBatch& fb) {
    return a.mode == GLU_MODE_GNU
               ? launch_f<GLU_MODE_GNU>(ctx, a, packed, forceFallback, nanFlag, fb)
               : launch_f<GLU_MODE_FAST>(ctx, a, packed, forceFallback, nanFlag, fb);
}

}  // namespace glu_cu
