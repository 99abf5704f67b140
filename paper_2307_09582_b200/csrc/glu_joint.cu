// glu_joint.cu -- joint downsampling optimisation on the device
// (jointopt.cpp:56-206): the replace / re-solve / accept-or-rollback trials and
// their schedules (find_large_error, jointopt.cpp:9-46, is glu_ccl.cu).
//
// Trials (jointopt.cpp:114-180, the loop 195-202) are strictly sequential in
// the reference.  A trial T_i writes the LR cells Q_i it replaces and the
// params / errors of the footprints of dilate(Q_i, h); it reads LR cells in
// dilate(Q_i, 2h) and errors in footprints of dilate(Q_i, h).  Two trials whose
// cell bounding boxes are more than 2h apart (Chebyshev) therefore touch
// disjoint state and commute.  k_trial_sched is a persistent, cooperatively
// launched dataflow scheduler over that conflict graph: each trial counts its
// earlier conflicting trials, CTAs pop trials whose count reached zero from a
// FIFO, run them with the whole CTA and release their successors.  Claiming
// in index order and blocking (round 1's first version) left every CTA parked
// on a dependency chain while independent trials queued behind them; the
// dataflow form runs at max(critical path, work / CTAs).  Conflicting trials
// still run in index order, so the final state is bit-identical to the
// sequential loop.  Trials too large for a CTA's private buffers get a
// whole-grid box (they conflict with everything, so they run alone) and use
// the global worst-case buffers.
//
// The accept test e1 <= e0 compares the reference's sequentially rounded
// double sums (150-165): the CTA forms parallel fp64 sums and decides when
// |e1 - e0| exceeds a rigorous bound on parallel-vs-sequential rounding;
// otherwise one thread redoes both sums in the exact reference order.
#include <cooperative_groups.h>
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "glu_internal.h"
#include "glu_filter32.cuh"
#include "glu_math.cuh"

namespace glu_cu {

namespace {

#ifndef GLU_SCHED_THREADS
#define GLU_SCHED_THREADS 512
#endif
#ifndef GLU_TRIAL_INCR
#define GLU_TRIAL_INCR 1  // trial re-solves keep provably unchanged pixels (Fast / GNU, S = 3)
#endif
constexpr int kSchedThreads = GLU_SCHED_THREADS;  // CTA size of the parallel trial scheduler
// A scheduled trial can run on a cluster of kCS CTAs (one per SM): each CTA
// stages the trial's window and offsets itself, the re-solve and the commit
// are split between them, partial sums meet in distributed shared memory.
// Measured (C2 / C4 joint): kCS = 1 2.43 / 3.65 ms, 2 2.64 / 3.56 ms, 4 3.56 /
// 4.49 ms -- a trial's latency is dominated by its staging, scans and
// barriers, not the re-solve, while clusters halve the trials in flight; so
// one CTA per trial is the default.
#ifndef GLU_TRIAL_CLUSTER
#define GLU_TRIAL_CLUSTER 1
#endif
constexpr int kCS = GLU_TRIAL_CLUSTER;
static_assert(kCS == 1 || kCS == 2 || kCS == 4, "trial cluster of 1, 2 or 4 CTAs");
constexpr int kSeqThreads = 1024;    // CTA size of the sequential (single-CTA) sweep
// Per-CTA private trial buffers (one 512-thread CTA per SM): a diagonal 200-pixel line
// at s = 8 has a 27 x 27-cell dilated box (46,656 pixels), so 64 Ki pixels
// keeps the serialising whole-grid fallback for genuinely huge components.
constexpr uint32_t kCtaPixels = 65536;  // per-CTA affected-pixel capacity
constexpr uint32_t kCtaCells = 8192;    // per-CTA replaced-cell capacity

// ---- trials -------------------------------------------------------------------

__device__ __forceinline__ unsigned cluster_rank() {
    return kCS > 1 ? cooperative_groups::this_cluster().block_rank() : 0u;
}
// Barrier over the trial's cluster (release / acquire at cluster scope: the
// CTAs' global and shared writes before it are visible to all after it).
__device__ __forceinline__ void cluster_barrier() {
    if (kCS > 1)
        cooperative_groups::this_cluster().sync();
    else
        __syncthreads();
}
// `v` into the same shared variable of every CTA of the cluster.
template <typename T>
__device__ __forceinline__ void cluster_bcast(T* var, T v) {
    if (kCS > 1) {
        auto cl = cooperative_groups::this_cluster();
        for (unsigned r = 0; r < unsigned(kCS); ++r) *cl.map_shared_rank(var, r) = v;
    } else {
        *var = v;
    }
}

#ifdef GLU_SCHED_TRACE
// Development builds only (-DGLU_SCHED_TRACE): per trial {claim, ready, end}
// %globaltimer stamps, dumped by run_sched to $GLU_SCHED_TRACE_FILE, and SM
// cycles per run_trial phase (thread 0, after the phase's barrier).
__device__ unsigned long long* g_trace;
__device__ unsigned long long g_phase[26];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
    return v;
}
#define GLU_PHASE(k)                                            \
    if (threadIdx.x == 0 && cluster_rank() == 0) {              \
        const long long c_ = clock64();                         \
        atomicAdd(&g_phase[k], (unsigned long long)(c_ - tph)); \
        tph = c_;                                               \
    }
#else
#define GLU_PHASE(k)
#endif


struct TrialState {
    const float* high;
    float* low;
    glu_pixel_params* field;
    float* errors;
    int W, H, s, lw, lh, S;
    double eps;
    int mode, literal;
    unsigned long long* cellKey;  // per LR cell, 0 between trials
    uint32_t* cellFlag;           // per LR cell, 0 between trials
    uint8_t* affMark;             // per LR cell, 0 between trials
    int* result;  // [0] accepted, [1] rejected, [2] sequential-sum fallbacks, [3] last verdict
    // Optional change log of accepted trials (distributed joint loop): cells
    // as {idx, r, g, b} words, pixels as {idx, a, b, w, e} words.
    uint32_t* dCount;  // [0] cells, [1] pixels, [2] overflow flag
    uint32_t* dCells;
    uint32_t* dPixels;
    uint32_t dCellCap, dPixelCap;
};

struct TrialBuffers {
    uint32_t* touched;  // replaced cells
    float* oldColor;    // 3 floats per replaced cell
    uint32_t* aff;      // affected pixels, reference order
    glu_pixel_params* bkParams;
    float* bkE;
};

struct GlobalLowWindow {
    const float* low;
    int lw, x0, y0, nwx;
    __device__ __forceinline__ const float* operator[](int i) const {
        const int r = i / nwx, q = i - r * nwx;
        return low + 3 * (size_t(y0 + r) * lw + x0 + q);
    }
};

template <int NT>
struct TrialSmem {
    using BlockScan = cub::BlockScan<uint32_t, NT>;
    using BlockReduce = cub::BlockReduce<double, NT>;
    union {
        typename BlockScan::TempStorage scan;
        typename BlockReduce::TempStorage reduce;
    } tmp;
    uint32_t touched, base;
    int box[4];
    double e0;
    int verdict;
    uint32_t logCells, logPixels;  // change-log bases of this trial
    uint32_t nFull;                // run_trial_smem: pixels listed for a full re-solve
    uint32_t parkWords;            // the speculative record's capacity (GLU_DCHECK)
};

// One trial (jointopt.cpp:114-180) executed by the whole CTA.  Returns the
// verdict (1 accepted) in every thread.
template <int NT>
__device__ int run_trial(const TrialState& t, const TrialBuffers& b, TrialSmem<NT>& sm,
                         const uint32_t* comp, uint32_t n) {
    using BlockScan = typename TrialSmem<NT>::BlockScan;
    using BlockReduce = typename TrialSmem<NT>::BlockReduce;
    const int tid = threadIdx.x;
    const int h = t.S / 2;
    const uint32_t W = uint32_t(t.W), s = uint32_t(t.s);
#ifdef GLU_SCHED_TRACE
    long long tph = clock64();
#endif
    if (tid == 0) {
        sm.touched = 0;
        sm.box[0] = t.lw;
        sm.box[1] = t.lh;
        sm.box[2] = -1;
        sm.box[3] = -1;
    }
    __syncthreads();
    // 1. groupByOwnerCell (jointopt.cpp:56-72) + worst pixel per cell: the
    //    first strict argmax over ascending pixels == max of (E, -pixel).
    for (uint32_t i = tid; i < n; i += NT) {
        const uint32_t p = comp[i];
        const uint32_t cx = (p % W) / s, cy = (p / W) / s;
        const uint32_t cell = cy * uint32_t(t.lw) + cx;
        const unsigned long long key =
            (static_cast<unsigned long long>(__float_as_uint(t.errors[p])) << 32) |
            (0xffffffffu - p);
        atomicMax(t.cellKey + cell, key);
        if (atomicExch(t.cellFlag + cell, 1u) == 0) {
            b.touched[atomicAdd(&sm.touched, 1u)] = cell;
            atomicMin(&sm.box[0], int(cx));
            atomicMin(&sm.box[1], int(cy));
            atomicMax(&sm.box[2], int(cx));
            atomicMax(&sm.box[3], int(cy));
        }
    }
    __syncthreads();
    GLU_PHASE(0)
    const uint32_t nt = sm.touched;
    // 2. replace each cell by its worst pixel (jointopt.cpp:130-142) and mark
    //    the cells whose windows reach it (affectedPixels, 76-110).
    for (uint32_t i = tid; i < nt; i += NT) {
        const uint32_t cell = b.touched[i];
        const uint32_t best = 0xffffffffu - uint32_t(t.cellKey[cell] & 0xffffffffu);
        float* lc = t.low + 3 * size_t(cell);
        const float* src = t.high + 3 * size_t(best);
        b.oldColor[3 * i] = lc[0];
        b.oldColor[3 * i + 1] = lc[1];
        b.oldColor[3 * i + 2] = lc[2];
        lc[0] = src[0];
        lc[1] = src[1];
        lc[2] = src[2];
        if (!t.literal) {
            const int cx = int(cell % uint32_t(t.lw)), cy = int(cell / uint32_t(t.lw));
            for (int y = max(0, cy - h); y <= min(t.lh - 1, cy + h); ++y)
                for (int x = max(0, cx - h); x <= min(t.lw - 1, cx + h); ++x)
                    t.affMark[size_t(y) * t.lw + x] = 1;
        }
    }
    __syncthreads();
    GLU_PHASE(1)
    // 3. affected pixels in the reference order: dilated bounding box in raster
    //    cell order, then each footprint in raster order.
    const uint32_t* aff = comp;
    uint32_t na = n;
    if (!t.literal) {
        const int bx0 = max(0, sm.box[0] - h), by0 = max(0, sm.box[1] - h);
        const int bx1 = min(t.lw - 1, sm.box[2] + h), by1 = min(t.lh - 1, sm.box[3] + h);
        const int bw = bx1 - bx0 + 1;
        const uint32_t nbox = uint32_t(bw) * uint32_t(by1 - by0 + 1);
        if (tid == 0) sm.base = 0;
        __syncthreads();
        for (uint32_t b0 = 0; b0 < nbox; b0 += NT) {
            const uint32_t k = b0 + tid;
            uint32_t fs = 0;
            int x = 0, y = 0;
            if (k < nbox) {
                x = bx0 + int(k % uint32_t(bw));
                y = by0 + int(k / uint32_t(bw));
                uint8_t* mk = t.affMark + size_t(y) * t.lw + x;
                if (*mk) {
                    *mk = 0;
                    fs = uint32_t(min(x * t.s + t.s, t.W) - x * t.s) *
                         uint32_t(min(y * t.s + t.s, t.H) - y * t.s);
                }
            }
            uint32_t pos, total;
            BlockScan(sm.tmp.scan).ExclusiveSum(fs, pos, total);
            if (fs) {
                uint32_t o = sm.base + pos;
                const int px0 = x * t.s, py0 = y * t.s;
                const int px1 = min(px0 + t.s, t.W), py1 = min(py0 + t.s, t.H);
                for (int py = py0; py < py1; ++py)
                    for (int pxx = px0; pxx < px1; ++pxx)
                        b.aff[o++] = uint32_t(py) * W + uint32_t(pxx);
            }
            __syncthreads();
            if (tid == 0) sm.base += total;
            __syncthreads();
        }
        aff = b.aff;
        na = sm.base;
    }
    GLU_PHASE(2)
    // 4. backup and e0 (jointopt.cpp:150-157).
    double part = 0;
    for (uint32_t i = tid; i < na; i += NT) {
        const uint32_t p = aff[i];
        b.bkParams[i] = t.field[p];
        b.bkE[i] = t.errors[p];
        part += double(b.bkE[i]);
    }
    const double e0 = BlockReduce(sm.tmp.reduce).Sum(part);
    if (tid == 0) sm.e0 = e0;
    __syncthreads();
    GLU_PHASE(3)
    // 5. re-solve (optimize_pixels, 159) and re-score (160-165).
    part = 0;
    bool changed = false;
    for (uint32_t i = tid; i < na; i += NT) {
        const uint32_t p = aff[i];
        const int x = int(p % W), y = int(p / W);
        const float* ip = t.high + 3 * size_t(p);
        const int cx = x / t.s, cy = y / t.s;
        const int x0 = max(0, cx - h), y0 = max(0, cy - h);
        const int nwx = min(t.lw - 1, cx + h) - x0 + 1, nwy = min(t.lh - 1, cy + h) - y0 + 1;
        glu_pixel_params np;
        bool done = false;
        if (t.S == 3) {
            // fp32 filter + fp64 verify (glu_filter32.cuh) on the live LR image
            float4 c[9];
#pragma unroll
            for (int k = 0; k < 9; ++k) {
                const int gx = cx - 1 + k % 3, gy = cy - 1 + k / 3;
                c[k] = make_float4(__int_as_float(0x7f800000), __int_as_float(0x7f800000),
                                   __int_as_float(0x7f800000), 0.0f);
                if (gx >= 0 && gy >= 0 && gx < t.lw && gy < t.lh) {
                    const float* s = t.low + 3 * (size_t(gy) * t.lw + gx);
                    c[k] = make_float4(s[0], s[1], s[2], max_abs3(s[0], s[1], s[2]));
                }
            }
            const Filter32Result fr =
                t.mode == GLU_MODE_EXACT
                    ? filter32x_pixel(c, ip, float(t.eps), t.eps)
                    : t.mode == GLU_MODE_GNU ? filter32_pixel(c, ip, float(t.eps), t.eps, true)
                                             : filter32k_pixel(c, ip, float(t.eps), t.eps);
            if (fr.ok) {
                np.a = uint32_t(cy - 1 + fr.ja / 3) * uint32_t(t.lw) + uint32_t(cx - 1 + fr.ja % 3);
                np.b = uint32_t(cy - 1 + fr.jb / 3) * uint32_t(t.lw) + uint32_t(cx - 1 + fr.jb % 3);
                np.w = fr.w;
                done = true;
            }
        }
#ifdef GLU_SCHED_TRACE
        atomicAdd(&g_phase[10], 1ull);
        if (!done) atomicAdd(&g_phase[9], 1ull);
#endif
        if (!done) {
            const Pick pk = pick64(t.mode, ip, GlobalLowWindow{t.low, t.lw, x0, y0, nwx},
                                   nwx * nwy, t.eps);
            const int ar = pk.ai / nwx, br = pk.bi / nwx;
            np.a = uint32_t(y0 + ar) * uint32_t(t.lw) + uint32_t(x0 + pk.ai - ar * nwx);
            np.b = uint32_t(y0 + br) * uint32_t(t.lw) + uint32_t(x0 + pk.bi - br * nwx);
            np.w = float(pk.w);
        }
        t.field[p] = np;
        float r[3];
        for (int k = 0; k < 3; ++k)
            r[k] = lerp_clamp(np.w, t.low[3 * size_t(np.a) + k], t.low[3 * size_t(np.b) + k],
                              true);
        const float e = pixel_error(ip, r);
        t.errors[p] = e;
        changed |= __float_as_uint(e) != __float_as_uint(b.bkE[i]);
        part += double(e);
    }
    GLU_PHASE(4)
    const double e1 = BlockReduce(sm.tmp.reduce).Sum(part);
    // Identical per-pixel errors give identical sequential sums: accept --
    // unless the sum is NaN (a NaN error in the set), where the reference's
    // `e1 <= e0` is false: the sequential re-check below then rejects.
    const bool anyChanged = __syncthreads_or(changed);
    if (tid == 0) {
        const double s0 = sm.e0;
        // |parallel - sequential| <= 2 * gamma_na * sum for non-negative terms.
        const double bound = 4.0 * (double(na) + 64.0) * 0x1.0p-53 * (s0 + e1);
        if ((!anyChanged && s0 == s0) || e1 + bound < s0)
            sm.verdict = 1;
        else if (e1 > s0 + bound)
            sm.verdict = 0;
        else
            sm.verdict = -1;  // too close: redo both sums in the reference order
    }
    __syncthreads();
    if (sm.verdict < 0) {
        // exact reference order (jointopt.cpp:150-165); the block stages each
        // chunk of old / new errors in shared memory for thread 0's chain
        double q0 = 0, q1 = 0;
        float* stage = reinterpret_cast<float*>(&sm.tmp);
        constexpr uint32_t kChunk = sizeof(sm.tmp) / (2 * sizeof(float));
        for (uint32_t c0 = 0; c0 < na; c0 += kChunk) {
            const uint32_t m = min(kChunk, na - c0);
            for (uint32_t k = tid; k < m; k += NT) {
                stage[2 * k] = b.bkE[c0 + k];
                stage[2 * k + 1] = t.errors[aff[c0 + k]];
            }
            __syncthreads();
            if (tid == 0)
                for (uint32_t k = 0; k < m; ++k) {
                    q0 += double(stage[2 * k]);
                    q1 += double(stage[2 * k + 1]);
                }
            __syncthreads();
        }
        if (tid == 0) {
            sm.verdict = q1 <= q0;
            atomicAdd(t.result + 2, 1);
        }
        __syncthreads();
    }
    GLU_PHASE(5)
    const int verdict = sm.verdict;
    // change log of an accepted trial (distributed joint loop)
    if (t.dCount && verdict) {
        if (tid == 0) {
            sm.logCells = atomicAdd(t.dCount, nt);
            sm.logPixels = atomicAdd(t.dCount + 1, na);
            if (sm.logCells + nt > t.dCellCap || sm.logPixels + na > t.dPixelCap) {
                atomicExch(t.dCount + 2, 1u);
                sm.logCells = sm.logPixels = 0xffffffffu;
            }
        }
        __syncthreads();
        if (sm.logCells != 0xffffffffu) {
            for (uint32_t i = tid; i < nt; i += NT) {
                const uint32_t cell = b.touched[i];
                uint32_t* o = t.dCells + 4 * size_t(sm.logCells + i);
                const float* lc = t.low + 3 * size_t(cell);
                o[0] = cell;
                o[1] = __float_as_uint(lc[0]);
                o[2] = __float_as_uint(lc[1]);
                o[3] = __float_as_uint(lc[2]);
            }
            for (uint32_t i = tid; i < na; i += NT) {
                const uint32_t p = aff[i];
                uint32_t* o = t.dPixels + 5 * size_t(sm.logPixels + i);
                const glu_pixel_params pp = t.field[p];
                o[0] = p;
                o[1] = pp.a;
                o[2] = pp.b;
                o[3] = __float_as_uint(pp.w);
                o[4] = __float_as_uint(t.errors[p]);
            }
        }
    }
    GLU_PHASE(6)
    // 6. rollback (jointopt.cpp:169-179) and reset per-cell state.
    if (!verdict) {
        for (uint32_t i = tid; i < na; i += NT) {
            const uint32_t p = aff[i];
            t.field[p] = b.bkParams[i];
            t.errors[p] = b.bkE[i];
        }
    }
    for (uint32_t i = tid; i < nt; i += NT) {
        const uint32_t cell = b.touched[i];
        if (!verdict) {
            float* lc = t.low + 3 * size_t(cell);
            lc[0] = b.oldColor[3 * i];
            lc[1] = b.oldColor[3 * i + 1];
            lc[2] = b.oldColor[3 * i + 2];
        }
        t.cellKey[cell] = 0;
        t.cellFlag[cell] = 0;
    }
    __syncthreads();
    GLU_PHASE(7)
    return verdict;
}

// ---- shared-memory trial path ---------------------------------------------------
//
// run_trial keeps its per-trial state in global memory (per-cell keys / marks
// and the affected-pixel list), so one trial is a dozen dependent L2 round
// trips.  A trial on the scheduler's critical path is pure latency, so the
// common case -- the component's cell box known up front (boxes[i]) and small
// -- keeps everything on chip instead: the LR colours of the box dilated by 2h
// (every candidate any re-solve reads), the worst-pixel key per box cell, the
// previous colours of the replaced cells and the affected-pixel offsets of
// the h-dilated box, from which thread-strided pixel indices are mapped in
// reference order by binary search.  Backup, re-solve and both error sums run
// in one pass (a pixel's re-solve writes only that pixel's params / error).
// Same results as run_trial, state for state.
constexpr int kSQ = 2048;  // cells of the component's box
constexpr int kSW = 4096;  // cells of the box dilated by 2h
constexpr int kSC = 2048;  // pixels of the component
constexpr int kSS = kSchedThreads > 512 ? kSchedThreads : 512;  // successors found by the early scan (>= the CTA size)
constexpr uint32_t kParkWords = 128u << 20;  // speculative-record arena (512 MB)
constexpr size_t kTrialSmemBytes = size_t(kSQ) * 8 + size_t(kSW) * 16 + size_t(kSC) * 16 +
                                   size_t(kSW + 1) * 4 + size_t(kSW) * 4 + size_t(kSQ) * 4 +
                                   size_t(kSQ) * 12 + size_t(kSW) * 2;

struct TrialShared {
    unsigned long long* key;  // [kSQ] worst-pixel key per box cell, 0: untouched
    float4* win;              // [kSW] LR colours of the 2h-dilated box
    float4* compC;            // [kSC] HR colours of the component's pixels
    uint32_t* pre;            // [kSW + 1] affected-pixel offsets over the h-dilated box
    uint32_t* cellOf;         // [kSW] affected cells in order, (y << 16) | x
    uint32_t* touched;        // [kSQ] replaced cells (box-local index, raster order)
    float* old;               // [3 kSQ] their previous colours
    uint16_t* rmask;          // [kSW] S = 3: replaced slots of each D cell's 3 x 3 window
    __device__ static TrialShared carve(char* base) {
        TrialShared s;
        s.key = reinterpret_cast<unsigned long long*>(base);
        s.win = reinterpret_cast<float4*>(base + size_t(kSQ) * 8);
        s.compC = s.win + kSW;
        s.pre = reinterpret_cast<uint32_t*>(s.compC + kSC);
        s.cellOf = s.pre + kSW + 1;
        s.touched = s.cellOf + kSW;
        s.old = reinterpret_cast<float*>(s.touched + kSQ);
        s.rmask = reinterpret_cast<uint16_t*>(s.old + 3 * kSQ);
        return s;
    }
};

// Box geometry of one trial (cells): Q = the component's cells, D = Q dilated
// by h (owner cells of the affected pixels), V = Q dilated by 2h (candidates).
struct TrialGeom {
    int qx0, qy0, qw, qh;
    int dx0, dy0, dw, dh;
    int vx0, vy0, vw, vh;
    bool full;  // every footprint in D is a full s x s block
    int sh;     // log2(s) when s is a power of two, else -1
    __device__ TrialGeom(int4 b, int h, int lw, int lh, int s, int W, int H) {
        qx0 = b.x;
        qy0 = b.y;
        qw = b.z - b.x + 1;
        qh = b.w - b.y + 1;
        dx0 = max(0, b.x - h);
        dy0 = max(0, b.y - h);
        dw = min(lw - 1, b.z + h) - dx0 + 1;
        dh = min(lh - 1, b.w + h) - dy0 + 1;
        // V is NOT clipped to the grid: cells outside it are staged as +inf
        // (like the packed LR image's border), so a pixel's 3 x 3 window is
        // always inside V and needs no bounds checks
        vx0 = b.x - 2 * h;
        vy0 = b.y - 2 * h;
        vw = b.z - b.x + 1 + 4 * h;
        vh = b.w - b.y + 1 + 4 * h;
        full = (dx0 + dw) * s <= W && (dy0 + dh) * s <= H && lw < 65536 && lh < 65536;
        sh = (s & (s - 1)) == 0 ? __ffs(s) - 1 : -1;
    }
    __device__ bool fits(uint32_t n) const {
        return qw * qh <= kSQ && vw * vh <= kSW && n <= uint32_t(kSC);
    }
};

struct SmemLowWindow {
    const float4* win;
    int vw, ox, oy, nwx;  // (ox, oy): window origin relative to V
    __device__ __forceinline__ const float* operator[](int i) const {
        const int r = i / nwx, q = i - r * nwx;
        return reinterpret_cast<const float*>(win + (oy + r) * vw + ox + q);
    }
};

__device__ __forceinline__ bool boxes_conflict(int4 a, int4 b, int reach) {
    const int dx = max(0, max(a.x - b.z, b.x - a.z));
    const int dy = max(0, max(a.y - b.w, b.y - a.w));
    return max(dx, dy) <= reach;
}

// Polling uses relaxed loads (served by L2, no L1 invalidation: an acquire load
// would flush the SM's L1 on every poll and starve the co-resident CTA doing
// real work); the waiting CTA issues one acquire fence after the flags are set.
__device__ __forceinline__ int ld_relaxed(const int* p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned long long ld_relaxed64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// The scheduler's view of one trial: its index and box, and where its
// conflicting successors found early (while pixel loads are in flight) go.
struct SuccScan {
    const int4* boxes;
    const int* sufTop;
    int ncomp, reach, self;
    int4 box;
    int* list;   // [kSS] shared
    int* count;  // shared; the caller zeroes it
    int* more;   // shared: successors may lie beyond the first kSS trials
    // speculation (nullptr: off): successors left waiting on this trial alone
    // are queued for an idle CTA to run speculatively (k_trial_sched)
    const unsigned long long* pred;
    int* specState;
    int* specQ;
    int* specTail;
};

// Affected pixel i (reference order) -> HR pixel index and its owner cell.
// When every affected footprint is a full s x s block (g.full), pixel i is
// pixel i % s^2 of the (i / s^2)-th affected cell; otherwise binary search.
__device__ __forceinline__ uint32_t affected_pixel(const TrialState& t, const TrialGeom& g,
                                                   const TrialShared& ss, uint32_t i, int& cx,
                                                   int& cy) {
    if (g.full) {
        uint32_t q, k, kx, ky;
        if (g.sh >= 0) {
            q = i >> (2 * g.sh);
            k = i & ((1u << (2 * g.sh)) - 1);
            ky = k >> g.sh;
            kx = k & ((1u << g.sh) - 1);
        } else {
            const uint32_t s = uint32_t(t.s);
            q = i / (s * s);
            k = i - q * s * s;
            ky = k / s;
            kx = k - ky * s;
        }
        const uint32_t cc = ss.cellOf[q];
        cx = int(cc & 0xffffu);
        cy = int(cc >> 16);
        return (uint32_t(cy * t.s) + ky) * uint32_t(t.W) + uint32_t(cx * t.s) + kx;
    }
    const uint32_t* pre = ss.pre;
    int lo = 0, hi = g.dw * g.dh;  // pre[lo] <= i < pre[hi]
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (pre[mid] <= i)
            lo = mid;
        else
            hi = mid;
    }
    cx = g.dx0 + lo % g.dw;
    cy = g.dy0 + lo / g.dw;
    const uint32_t k = i - pre[lo];
    const int fx0 = cx * t.s, fy0 = cy * t.s;
    const uint32_t fw = uint32_t(min(fx0 + t.s, t.W) - fx0);
    return uint32_t(fy0 + int(k / fw)) * uint32_t(t.W) + uint32_t(fx0) + k % fw;
}

struct PixIn {
    uint32_t p;
    int cx, cy;
    float oe, i0, i1, i2;
    glu_pixel_params old;  // the current params (S = 3, Fast / GNU)
};

template <int NT>
__device__ int run_trial_smem(const TrialState& t, const TrialBuffers& b, TrialSmem<NT>& sm,
                              const TrialShared& ss, const TrialGeom& g, const uint32_t* comp,
                              uint32_t n, const SuccScan& sc, uint32_t* park = nullptr) {
    using BlockScan = typename TrialSmem<NT>::BlockScan;
    __shared__ double red[2][NT / 32];
    __shared__ double xred[kCS][3];  // per-CTA partials {e0, e1, changed} of the cluster
    // park != nullptr (speculative run): the result goes to the trial's parked
    // record {verdict, nt, na, na x {p, a, b, w, e}, nt x {cell, r, g, b}}
    // instead of this CTA's buffers; see k_trial_sched.
    uint32_t* parkPix = park ? park + 3 : nullptr;
    const int tid = threadIdx.x;
    // Every CTA of the cluster stages the trial (phases A-C) in its own shared
    // memory; the affected pixels are split in blocks of NT (pixel i goes to
    // CTA (i / NT) % kCS) and the partial sums meet in distributed shared memory.
    const uint32_t rank = cluster_rank();
    const int h = t.S / 2;
    const uint32_t W = uint32_t(t.W), s = uint32_t(t.s);
#ifdef GLU_SCHED_TRACE
    long long tph = clock64();
#endif
    // A. stage the candidate colours and the component's colours; group its
    //    pixels by owner cell keeping the worst, i.e. the first strict argmax
    //    over ascending pixels = max of (E, -index) (jointopt.cpp:56-72,
    //    130-142).  Keys are zero on entry (the previous trial cleared them).
    const int nv = g.vw * g.vh, nq = g.qw * g.qh, nd = g.dw * g.dh;
    GLU_DCHECK(nv <= kSW && nq <= kSQ && nd <= kSW && n <= uint32_t(kSC));
    GLU_DCHECK(g.dx0 - g.vx0 >= h && g.dy0 - g.vy0 >= h &&
               g.dx0 + g.dw + h <= g.vx0 + g.vw && g.dy0 + g.dh + h <= g.vy0 + g.vh);
    for (int k = tid; k < nv; k += NT) {
        const int y = g.vy0 + k / g.vw, x = g.vx0 + k % g.vw;
        if (x >= 0 && y >= 0 && x < t.lw && y < t.lh) {
            const float* src = t.low + 3 * (size_t(y) * t.lw + x);
            ss.win[k] = make_float4(src[0], src[1], src[2], max_abs3(src[0], src[1], src[2]));
        } else {
            ss.win[k] = make_float4(__int_as_float(0x7f800000), __int_as_float(0x7f800000),
                                    __int_as_float(0x7f800000), 0.0f);
        }
    }
    for (uint32_t i = tid; i < n; i += NT) {
        const uint32_t p = comp[i];
        const float* src = t.high + 3 * size_t(p);
        const float e = t.errors[p];
        ss.compC[i] = make_float4(src[0], src[1], src[2], max_abs3(src[0], src[1], src[2]));
        const int cx = int((p % W) / s), cy = int((p / W) / s);
        const unsigned long long key =
            (static_cast<unsigned long long>(__float_as_uint(e)) << 32) | (0xffffffffu - i);
        atomicMax(ss.key + (cy - g.qy0) * g.qw + (cx - g.qx0), key);
    }
    if (sc.list && rank == 0) {
        // conflicting successors among the next NT trials (loads overlap the
        // staging above)
        const int j = sc.self + 1 + tid;
        if (j < sc.ncomp && boxes_conflict(sc.box, sc.boxes[j], sc.reach)) {
            const int at = atomicAdd(sc.count, 1);
            GLU_DCHECK(at < kSS);
            sc.list[at] = j;
            // a successor waiting on this trial alone: speculate it now (valid
            // iff this trial is rejected); the release pushes the others when
            // their last predecessor is left
            if (sc.specQ && uint32_t(ld_relaxed64(sc.pred + j)) == 1u &&
                atomicCAS(sc.specState + j, 0, 7) == 0) {
                const int at = atomicAdd(sc.specTail, 1);
                GLU_DCHECK(at < sc.ncomp);
                st_release(sc.specQ + at, j);
#ifdef GLU_SCHED_TRACE
                atomicAdd(&g_phase[19], 1ull);
#endif
            }
        }
        if (tid == 0)
            *sc.more = sc.self + 1 + NT < sc.ncomp && sc.sufTop[sc.self + 1 + NT] <= sc.box.w + sc.reach;
    }
    __syncthreads();
    GLU_PHASE(0)
    // C. replace the touched cells; affected-pixel offsets over D (76-110)
    // Fast / GNU at S = 3: a pixel whose a and b are not replaced keeps them
    // when no replaced candidate provably beats them (f32s_unchanged).  Worth
    // its extra pass from about three rounds of pixels per thread (C4: ~5;
    // C2: ~1.3, where it measured slower); decided from the box geometry so
    // the footprint scan below can record the replaced slots on the way.
    const bool incr = t.S == 3 && t.mode != GLU_MODE_EXACT && GLU_TRIAL_INCR && kCS == 1 &&
                      size_t(nd) * size_t(t.s) * size_t(t.s) > size_t(3 * NT);
    auto footprint = [&](int k) -> uint32_t {  // affected pixels of D cell k (0: not affected)
        const int x = g.dx0 + k % g.dw, y = g.dy0 + k / g.dw;
        if (incr) {
            // also which slots of the cell's 3 x 3 window hold a replaced cell
            uint32_t m = 0;
            for (int yy = max(y - 1, g.qy0); yy <= min(y + 1, g.qy0 + g.qh - 1); ++yy)
                for (int xx = max(x - 1, g.qx0); xx <= min(x + 1, g.qx0 + g.qw - 1); ++xx)
                    if (ss.key[(yy - g.qy0) * g.qw + (xx - g.qx0)])
                        m |= 1u << ((yy - y + 1) * 3 + (xx - x + 1));
            ss.rmask[k] = uint16_t(m);
            return m ? uint32_t(min(x * t.s + t.s, t.W) - x * t.s) *
                           uint32_t(min(y * t.s + t.s, t.H) - y * t.s)
                     : 0u;
        }
        for (int yy = max(y - h, g.qy0); yy <= min(y + h, g.qy0 + g.qh - 1); ++yy)
            for (int xx = max(x - h, g.qx0); xx <= min(x + h, g.qx0 + g.qw - 1); ++xx)
                if (ss.key[(yy - g.qy0) * g.qw + (xx - g.qx0)])
                    return uint32_t(min(x * t.s + t.s, t.W) - x * t.s) *
                           uint32_t(min(y * t.s + t.s, t.H) - y * t.s);
        return 0u;
    };
    auto replace = [&](int k, unsigned long long key, uint32_t slot) {
        const int qx = g.qx0 + k % g.qw, qy = g.qy0 + k / g.qw;
        const float4 bc = ss.compC[0xffffffffu - uint32_t(key & 0xffffffffu)];
        float4& wc = ss.win[(qy - g.vy0) * g.vw + (qx - g.vx0)];
        ss.touched[slot] = uint32_t(k);
        ss.old[3 * slot] = wc.x;
        ss.old[3 * slot + 1] = wc.y;
        ss.old[3 * slot + 2] = wc.z;
        wc = bc;  // global LR written at commit
    };
    auto place = [&](int k, uint32_t fs, uint32_t pos) {
        ss.pre[k] = pos;
        if (fs && g.full)
            ss.cellOf[pos / uint32_t(t.s * t.s)] =
                (uint32_t(g.dy0 + k / g.dw) << 16) | uint32_t(g.dx0 + k % g.dw);
    };
    uint32_t nt = 0, na = 0;
    if (nq <= NT && nd <= NT) {
        // the common case in one pass: both compactions by warp ballot /
        // shuffle scan, one barrier for the per-warp totals
        __shared__ uint32_t wtot[2][NT / 32];
        const int lane = tid & 31, wid = tid >> 5;
        const unsigned long long key = tid < nq ? ss.key[tid] : 0ull;
        const uint32_t fs = tid < nd ? footprint(tid) : 0u;
        const unsigned bal = __ballot_sync(0xffffffffu, key != 0);
        uint32_t incl = fs;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        if (lane == 31) {
            wtot[0][wid] = __popc(bal);
            wtot[1][wid] = incl;
        }
        __syncthreads();
        uint32_t baseT = 0, baseA = 0;
#pragma unroll
        for (int w = 0; w < NT / 32; ++w) {
            const uint32_t c0 = wtot[0][w], c1 = wtot[1][w];
            baseT += w < wid ? c0 : 0u;
            baseA += w < wid ? c1 : 0u;
            nt += c0;
            na += c1;
        }
        if (key) replace(tid, key, baseT + __popc(bal & ((1u << lane) - 1u)));
        if (tid < nd) place(tid, fs, baseA + incl - fs);
    } else {
        for (int b0 = 0; b0 < nq; b0 += NT) {
            const int k = b0 + tid;
            const unsigned long long key = k < nq ? ss.key[k] : 0ull;
            uint32_t pos, total;
            BlockScan(sm.tmp.scan).ExclusiveSum(key ? 1u : 0u, pos, total);
            if (key) replace(k, key, nt + pos);
            nt += total;
            __syncthreads();
        }
        for (int b0 = 0; b0 < nd; b0 += NT) {
            const int k = b0 + tid;
            const uint32_t fs = k < nd ? footprint(k) : 0u;
            uint32_t pos, total;
            BlockScan(sm.tmp.scan).ExclusiveSum(fs, pos, total);
            if (k < nd) place(k, fs, na + pos);
            na += total;
            __syncthreads();
        }
    }
    GLU_DCHECK(na <= kCtaPixels && nt <= uint32_t(kSQ));
    if (tid == 0) {
        ss.pre[nd] = na;
        sm.nFull = 0;
    }
    __syncthreads();
    GLU_PHASE(2)
    // D. backup + e0, re-solve + e1 (jointopt.cpp:150-165, optimize_pixels 159).
    //    Each thread's next pixel is loaded while the current one is solved.
    for (int k = tid; k < nq; k += NT) ss.key[k] = 0;
    auto load = [&](uint32_t i) {
        PixIn q;
        q.p = affected_pixel(t, g, ss, i, q.cx, q.cy);
        q.oe = t.errors[q.p];
        q.i0 = t.high[3 * size_t(q.p)];
        q.i1 = t.high[3 * size_t(q.p) + 1];
        q.i2 = t.high[3 * size_t(q.p) + 2];
        GLU_DCHECK(q.cx >= g.dx0 && q.cx < g.dx0 + g.dw && q.cy >= g.dy0 && q.cy < g.dy0 + g.dh &&
                   q.p < uint32_t(t.W) * uint32_t(t.H));
        if (incr) q.old = t.field[q.p];
        return q;
    };
    constexpr uint32_t kStride = uint32_t(kCS) * NT;
    double part0 = 0, part1 = 0;
    bool changed = false;
    // the full re-solve of pixel i (its e0 term already summed): the fp32
    // filter, else the exact double path; new params and error out, e1 term
    auto solve_full = [&](uint32_t i, const PixIn& q) {
        const uint32_t p = q.p;
        const int cx = q.cx, cy = q.cy;
        const float oe = q.oe;
        const float ip[3] = {q.i0, q.i1, q.i2};
        const int x0 = max(0, cx - h), y0 = max(0, cy - h);
        const int nwx = min(t.lw - 1, cx + h) - x0 + 1, nwy = min(t.lh - 1, cy + h) - y0 + 1;
        int ax, ay, bx, by;
        float w;
        bool done = false;
#ifdef GLU_SCHED_TRACE
        float4 c_dbg[9];
#endif
        if (t.S == 3) {
            // the window inside V (off-grid cells are the staged +inf cells)
            const float4* wv = ss.win + (cy - 1 - g.vy0) * g.vw + (cx - 1 - g.vx0);
            Filter32Result fr;
            if (t.mode == GLU_MODE_EXACT) {
                float4 c[9];
#pragma unroll
                for (int k = 0; k < 9; ++k) c[k] = wv[(k / 3) * g.vw + k % 3];
                fr = filter32x_pixel(c, ip, float(t.eps), t.eps);
            } else if (t.mode == GLU_MODE_GNU) {
                fr = filter32_smem<true>(wv, g.vw, ip, float(t.eps), t.eps);
            } else {
                fr = filter32_smem<false>(wv, g.vw, ip, float(t.eps), t.eps);
            }
#ifdef GLU_SCHED_TRACE
            for (int k = 0; k < 9; ++k) c_dbg[k] = wv[(k / 3) * g.vw + k % 3];
            if (fr.ok && fr.why == 6) atomicAdd(&g_phase[16], 1ull);
#endif
            if (fr.ok) {
                ax = cx - 1 + fr.ja % 3;
                ay = cy - 1 + fr.ja / 3;
                bx = cx - 1 + fr.jb % 3;
                by = cy - 1 + fr.jb / 3;
                w = fr.w;
                done = true;
            }
        }
#ifdef GLU_SCHED_TRACE
        atomicAdd(&g_phase[10], 1ull);
        if (!done) atomicAdd(&g_phase[9], 1ull);
        if (!done && t.S == 3 && t.mode != GLU_MODE_EXACT)
            atomicAdd(&g_phase[10 + filter32_pixel(c_dbg, ip, float(t.eps), t.eps,
                                                   t.mode == GLU_MODE_GNU).why], 1ull);
#endif
        if (!done) {
            const Pick pk = pick64(t.mode, ip,
                                   SmemLowWindow{ss.win, g.vw, x0 - g.vx0, y0 - g.vy0, nwx},
                                   nwx * nwy, t.eps);
            ay = y0 + pk.ai / nwx;
            ax = x0 + pk.ai % nwx;
            by = y0 + pk.bi / nwx;
            bx = x0 + pk.bi % nwx;
            w = float(pk.w);
        }
        glu_pixel_params np;
        np.a = uint32_t(ay) * uint32_t(t.lw) + uint32_t(ax);
        np.b = uint32_t(by) * uint32_t(t.lw) + uint32_t(bx);
        np.w = w;
        if (parkPix) {
            uint32_t* o = parkPix + 5 * size_t(i);
            o[0] = p;
            o[1] = np.a;
            o[2] = np.b;
            o[3] = __float_as_uint(np.w);
        } else {
            b.bkParams[i] = np;  // the trial's new state, written back at commit
        }
        const float4 la = ss.win[(ay - g.vy0) * g.vw + (ax - g.vx0)];
        const float4 lb = ss.win[(by - g.vy0) * g.vw + (bx - g.vx0)];
        const float r[3] = {lerp_clamp(w, la.x, lb.x, true), lerp_clamp(w, la.y, lb.y, true),
                            lerp_clamp(w, la.z, lb.z, true)};
        const float e = pixel_error(ip, r);
        if (parkPix)
            parkPix[5 * size_t(i) + 4] = __float_as_uint(e);
        else
            b.bkE[i] = e;
        changed |= __float_as_uint(e) != __float_as_uint(oe);
        part1 += double(e);
    };
    if (incr) {
        // Pass 1: every pixel's unchanged test (cheap); the pixels that fail
        // it are listed (this CTA's aff buffer) and re-solved in full in pass
        // 2, so full solves fill whole warps instead of diverging from the
        // ~90 % of pixels that keep their params (C4).
        PixIn cur{};
        if (tid < na) cur = load(tid);
        for (uint32_t i = tid; i < na; i += NT) {
            PixIn nxt{};
            if (i + NT < na) nxt = load(i + NT);
            const int cx = cur.cx, cy = cur.cy;
            const float oe = cur.oe;
            part0 += double(oe);
            const float ip[3] = {cur.i0, cur.i1, cur.i2};
            // slots of the current a and b in the window (both lie in it)
            const uint32_t o = uint32_t(cy - 1) * uint32_t(t.lw) + uint32_t(cx - 1);
            const uint32_t lw = uint32_t(t.lw);
            auto slot = [&](uint32_t idx) {
                const uint32_t d = idx - o;
                const uint32_t r = d >= 2 * lw ? 2u : (d >= lw ? 1u : 0u);
                return int(r * 3 + (d - r * lw));
            };
            const int sa = slot(cur.old.a), sb = slot(cur.old.b);
            GLU_DCHECK(sa >= 0 && sa < 9 && sb >= 0 && sb < 9);
            const uint32_t msk = ss.rmask[(cy - g.dy0) * g.dw + (cx - g.dx0)];
            const float4* wv = ss.win + (cy - 1 - g.vy0) * g.vw + (cx - 1 - g.vx0);
            if (!((msk >> sa) & 1u) && !((msk >> sb) & 1u) &&
                (t.mode == GLU_MODE_GNU
                     ? f32s_unchanged<true>(wv, g.vw, ip, sa, sb, msk, float(t.eps))
                     : f32s_unchanged<false>(wv, g.vw, ip, sa, sb, msk, float(t.eps)))) {
                // same a, b and w: the same params and, with a's and b's colours
                // unchanged, the same error
                if (parkPix) {
                    uint32_t* op = parkPix + 5 * size_t(i);
                    op[0] = cur.p;
                    op[1] = cur.old.a;
                    op[2] = cur.old.b;
                    op[3] = __float_as_uint(cur.old.w);
                    op[4] = __float_as_uint(oe);
                } else {
                    b.bkParams[i] = cur.old;
                    b.bkE[i] = oe;
                }
                part1 += double(oe);
#ifdef GLU_SCHED_TRACE
                atomicAdd(&g_phase[24], 1ull);
#endif
            } else {
                const uint32_t at = atomicAdd(&sm.nFull, 1u);
                GLU_DCHECK(at < na);
                b.aff[at] = i;
            }
            cur = nxt;
        }
        __syncthreads();
        const uint32_t nf = sm.nFull;
        // Pass 2: the listed pixels' full re-solves
        for (uint32_t k = tid; k < nf; k += NT) {
            const uint32_t i = b.aff[k];
            solve_full(i, load(i));
        }
    } else {
        PixIn cur{};
        if (rank * NT + tid < na) cur = load(rank * NT + tid);
        for (uint32_t i = rank * NT + tid; i < na; i += kStride) {
            PixIn nxt{};
            if (i + kStride < na) nxt = load(i + kStride);
            part0 += double(cur.oe);
            solve_full(i, cur);
            cur = nxt;
        }
    }
    GLU_PHASE(4)
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        part0 += __shfl_down_sync(0xffffffffu, part0, o);
        part1 += __shfl_down_sync(0xffffffffu, part1, o);
    }
    if ((tid & 31) == 0) {
        red[0][tid >> 5] = part0;
        red[1][tid >> 5] = part1;
    }
    const bool anyChangedCta = __syncthreads_or(changed);
    int verdict;
    if (kCS == 1) {
        // every thread forms the same sums in the same order: the same verdict
        double s0 = 0, e1 = 0;
#pragma unroll
        for (int k = 0; k < NT / 32; ++k) {
            s0 += red[0][k];
            e1 += red[1][k];
        }
        const double bound = 4.0 * (double(na) + 64.0) * 0x1.0p-53 * (s0 + e1);
        verdict = ((!anyChangedCta && s0 == s0) || e1 + bound < s0) ? 1 : (e1 > s0 + bound ? 0 : -1);
    } else {
        if (tid == 0) {
            double s0 = 0, e1 = 0;
            for (int k = 0; k < NT / 32; ++k) {
                s0 += red[0][k];
                e1 += red[1][k];
            }
            cluster_bcast(&xred[rank][0], s0);
            cluster_bcast(&xred[rank][1], e1);
            cluster_bcast(&xred[rank][2], anyChangedCta ? 1.0 : 0.0);
        }
        cluster_barrier();  // partials (and every CTA's new values in b / park) visible
        if (tid == 0) {
            // the same sums in the same order in every CTA: the same verdict
            double s0 = 0, e1 = 0;
            bool anyChanged = false;
            for (int r = 0; r < kCS; ++r) {
                s0 += xred[r][0];
                e1 += xred[r][1];
                anyChanged |= xred[r][2] != 0.0;
            }
            const double bound = 4.0 * (double(na) + 64.0) * 0x1.0p-53 * (s0 + e1);
            if ((!anyChanged && s0 == s0) || e1 + bound < s0)
                sm.verdict = 1;
            else if (e1 > s0 + bound)
                sm.verdict = 0;
            else
                sm.verdict = -1;
        }
        __syncthreads();
        verdict = sm.verdict;
    }
    if (verdict < 0) {
        // exact reference order, as in run_trial
        double q0 = 0, q1 = 0;
        float* stage = reinterpret_cast<float*>(&sm.tmp);
        constexpr uint32_t kChunk = sizeof(sm.tmp) / (2 * sizeof(float));
        for (uint32_t c0 = 0; c0 < na; c0 += kChunk) {
            const uint32_t m = min(kChunk, na - c0);
            for (uint32_t k = tid; k < m; k += NT) {
                int cx, cy;
                stage[2 * k] = t.errors[affected_pixel(t, g, ss, c0 + k, cx, cy)];
                stage[2 * k + 1] = parkPix ? __uint_as_float(parkPix[5 * size_t(c0 + k) + 4])
                                           : b.bkE[c0 + k];
            }
            __syncthreads();
            if (tid == 0)
                for (uint32_t k = 0; k < m; ++k) {
                    q0 += double(stage[2 * k]);
                    q1 += double(stage[2 * k + 1]);
                }
            __syncthreads();
        }
        if (tid == 0) {
            sm.verdict = q1 <= q0;
            if (rank == 0) atomicAdd(t.result + 2, 1);
        }
        __syncthreads();
        verdict = sm.verdict;
    }
    if (tid == 0) {
        sm.touched = nt;
        sm.base = na;
    }
    if (park && rank == 0) {
        GLU_DCHECK(3 + 5 * size_t(na) + 4 * size_t(nt) <= size_t(sm.parkWords));
        if (tid == 0) {
            park[0] = uint32_t(verdict);
            park[1] = nt;
            park[2] = na;
        }
        uint32_t* cells = parkPix + 5 * size_t(na);
        for (uint32_t i = tid; i < nt; i += NT) {
            const int k = int(ss.touched[i]);
            const int qx = g.qx0 + k % g.qw, qy = g.qy0 + k / g.qw;
            const float4 c = ss.win[(qy - g.vy0) * g.vw + (qx - g.vx0)];
            uint32_t* o = cells + 4 * size_t(i);
            o[0] = uint32_t(qy) * uint32_t(t.lw) + uint32_t(qx);
            o[1] = __float_as_uint(c.x);
            o[2] = __float_as_uint(c.y);
            o[3] = __float_as_uint(c.z);
        }
    }
    __syncthreads();
    GLU_PHASE(5)
    return verdict;
}

// Commit an accepted on-chip trial: the replaced LR cells, then the new params
// and errors of the affected pixels (a rejected trial wrote nothing: no
// rollback, jointopt.cpp:169-179 is implicit), plus the change log.
template <int NT>
__device__ void commit_trial_smem(const TrialState& t, const TrialBuffers& b, TrialSmem<NT>& sm,
                                  const TrialShared& ss, const TrialGeom& g) {
    const int tid = threadIdx.x;
    const uint32_t nt = sm.touched, na = sm.base, rank = cluster_rank();
#ifdef GLU_SCHED_TRACE
    long long tph = clock64();
#endif
    if (rank == 0)
        for (uint32_t i = tid; i < nt; i += NT) {
            const int k = int(ss.touched[i]);
            const int qx = g.qx0 + k % g.qw, qy = g.qy0 + k / g.qw;
            const float4 c = ss.win[(qy - g.vy0) * g.vw + (qx - g.vx0)];
            float* lc = t.low + 3 * (size_t(qy) * t.lw + qx);
            lc[0] = c.x;
            lc[1] = c.y;
            lc[2] = c.z;
        }
    // each CTA commits the pixels it solved
    for (uint32_t i = rank * NT + tid; i < na; i += uint32_t(kCS) * NT) {
        int cx, cy;
        const uint32_t p = affected_pixel(t, g, ss, i, cx, cy);
        t.field[p] = b.bkParams[i];
        t.errors[p] = b.bkE[i];
    }
    if (t.dCount && rank == 0) {
        if (tid == 0) {
            sm.logCells = atomicAdd(t.dCount, nt);
            sm.logPixels = atomicAdd(t.dCount + 1, na);
            if (sm.logCells + nt > t.dCellCap || sm.logPixels + na > t.dPixelCap) {
                atomicExch(t.dCount + 2, 1u);
                sm.logCells = sm.logPixels = 0xffffffffu;
            }
        }
        __syncthreads();
        if (sm.logCells != 0xffffffffu) {
            for (uint32_t i = tid; i < nt; i += NT) {
                const int k = int(ss.touched[i]);
                const int qx = g.qx0 + k % g.qw, qy = g.qy0 + k / g.qw;
                const float4 c = ss.win[(qy - g.vy0) * g.vw + (qx - g.vx0)];
                uint32_t* o = t.dCells + 4 * size_t(sm.logCells + i);
                o[0] = uint32_t(qy) * uint32_t(t.lw) + uint32_t(qx);
                o[1] = __float_as_uint(c.x);
                o[2] = __float_as_uint(c.y);
                o[3] = __float_as_uint(c.z);
            }
            for (uint32_t i = tid; i < na; i += NT) {
                int cx, cy;
                const uint32_t p = affected_pixel(t, g, ss, i, cx, cy);
                uint32_t* o = t.dPixels + 5 * size_t(sm.logPixels + i);
                const glu_pixel_params pp = b.bkParams[i];
                o[0] = p;
                o[1] = pp.a;
                o[2] = pp.b;
                o[3] = __float_as_uint(pp.w);
                o[4] = __float_as_uint(b.bkE[i]);
            }
        }
    }
    __syncthreads();
    GLU_PHASE(7)
}

// Commit a parked speculative record (see run_trial_smem); returns its verdict.
template <int NT>
__device__ int commit_parked(const TrialState& t, TrialSmem<NT>& sm, const uint32_t* park) {
    const int tid = threadIdx.x;
    const uint32_t rank = cluster_rank();
    const int verdict = int(park[0]);
    const uint32_t nt = park[1], na = park[2];
    const uint32_t* pix = park + 3;
    const uint32_t* cells = pix + 5 * size_t(na);
    if (verdict) {
        for (uint32_t i = rank * NT + tid; i < nt; i += uint32_t(kCS) * NT) {
            const uint32_t* c = cells + 4 * size_t(i);
            float* lc = t.low + 3 * size_t(c[0]);
            lc[0] = __uint_as_float(c[1]);
            lc[1] = __uint_as_float(c[2]);
            lc[2] = __uint_as_float(c[3]);
        }
        for (uint32_t i = rank * NT + tid; i < na; i += uint32_t(kCS) * NT) {
            const uint32_t* q = pix + 5 * size_t(i);
            glu_pixel_params pp;
            pp.a = q[1];
            pp.b = q[2];
            pp.w = __uint_as_float(q[3]);
            t.field[q[0]] = pp;
            t.errors[q[0]] = __uint_as_float(q[4]);
        }
        if (t.dCount && rank == 0) {
            if (tid == 0) {
                sm.logCells = atomicAdd(t.dCount, nt);
                sm.logPixels = atomicAdd(t.dCount + 1, na);
                if (sm.logCells + nt > t.dCellCap || sm.logPixels + na > t.dPixelCap) {
                    atomicExch(t.dCount + 2, 1u);
                    sm.logCells = sm.logPixels = 0xffffffffu;
                }
            }
            __syncthreads();
            if (sm.logCells != 0xffffffffu) {
                for (uint32_t i = tid; i < 4 * nt; i += NT)
                    t.dCells[4 * size_t(sm.logCells) + i] = cells[i];
                for (uint32_t i = tid; i < 5 * na; i += NT)
                    t.dPixels[5 * size_t(sm.logPixels) + i] = pix[i];
            }
        }
    }
    __syncthreads();
    return verdict;
}

// Parked-record size (32-bit words) of every trial that may run on chip.
__global__ void k_park_words(const int4* __restrict__ boxes, int n, int h, int s, int lw, int lh,
                             int W, int H, int literal, uint32_t* __restrict__ words) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i > n) return;
    if (i == n) {
        words[n] = 0;
        return;
    }
    const int4 b = boxes[i];
    uint32_t w = 0;
    if (b.x >= 0 && !literal) {
        const TrialGeom g(b, h, lw, lh, s, W, H);
        if (g.qw * g.qh <= kSQ && g.vw * g.vh <= kSW)
            w = 3 + 5 * uint32_t(g.dw * g.dh) * uint32_t(s * s) + 4 * uint32_t(g.qw * g.qh);
    }
    words[i] = w;
}

// Sequential sweep: one CTA runs the components in order (used for single
// trials and as the reference schedule in tests, GLU_OPT_TRIALS = 1).
__global__ void __launch_bounds__(kSeqThreads) k_trial_sweep(TrialState t, TrialBuffers b,
                                                             const uint32_t* off,
                                                             const uint32_t* px, int ncomp) {
    __shared__ TrialSmem<kSeqThreads> sm;
    for (int c = 0; c < ncomp; ++c) {
        const int v = run_trial<kSeqThreads>(t, b, sm, px + off[c], off[c + 1] - off[c]);
        if (threadIdx.x == 0) {
            t.result[v ? 0 : 1] += 1;
            t.result[3] = v;
        }
    }
}

// Cell bounding box of every component; components whose worst-case
// affected set exceeds a CTA's private buffers get the whole grid.
// With raw != 0 the plain cell box is written (for level scheduling); `ids`
// (optional) lists the components, box k belonging to component ids[k].
// The scheduler's per-trial state, initialised by the kernel that computes
// the trial's box (replaces five memsets per sweep): pred = 0 (with the 16
// counter words behind it), queue = specQ = -1, specState = 0, specSnap =
// 0x7f7f7f7f.  Null `pred`: boxes only.
struct SchedInit {
    unsigned long long* pred;
    int *queue, *specState, *specQ;
    uint32_t* specSnap;
};

__global__ void k_trial_boxes(const uint32_t* __restrict__ off, const uint32_t* __restrict__ px,
                              const uint32_t* __restrict__ ids, int ncomp, int W, int s, int lw,
                              int lh, int h, int literal, int raw, int4* __restrict__ boxes,
                              SchedInit si) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (si.pred && blockIdx.x == 0 && threadIdx.x < 8) si.pred[ncomp + threadIdx.x] = 0ull;
    if (warp >= ncomp) return;
    if (si.pred && lane == 0) {
        si.pred[warp] = 0ull;
        si.queue[warp] = -1;
        si.specState[warp] = 0;
        si.specSnap[warp] = 0x7f7f7f7fu;
        si.specQ[warp] = -1;
    }
    const uint32_t comp = ids ? ids[warp] : uint32_t(warp);
    const uint32_t b0 = off[comp], b1 = off[comp + 1];
    int x0 = lw, y0 = lh, x1 = -1, y1 = -1;
    for (uint32_t i = b0 + lane; i < b1; i += 32) {
        const uint32_t p = px[i];
        const int cx = int((p % uint32_t(W)) / uint32_t(s)), cy = int((p / uint32_t(W)) / uint32_t(s));
        x0 = min(x0, cx);
        y0 = min(y0, cy);
        x1 = max(x1, cx);
        y1 = max(y1, cy);
    }
    for (int o = 16; o; o >>= 1) {
        x0 = min(x0, __shfl_xor_sync(0xffffffffu, x0, o));
        y0 = min(y0, __shfl_xor_sync(0xffffffffu, y0, o));
        x1 = max(x1, __shfl_xor_sync(0xffffffffu, x1, o));
        y1 = max(y1, __shfl_xor_sync(0xffffffffu, y1, o));
    }
    if (lane == 0) {
        const uint64_t cells = uint64_t(x1 - x0 + 1) * uint64_t(y1 - y0 + 1);
        const uint64_t dil = uint64_t(min(lw - 1, x1 + h) - max(0, x0 - h) + 1) *
                             uint64_t(min(lh - 1, y1 + h) - max(0, y0 - h) + 1);
        const uint64_t affPx = literal ? uint64_t(b1 - b0) : dil * uint64_t(s) * uint64_t(s);
        const bool big = !raw && (cells > kCtaCells || affPx > kCtaPixels);
        boxes[warp] = big ? make_int4(-(1 << 28), -(1 << 28), 1 << 28, 1 << 28)
                          : make_int4(x0, y0, x1, y1);
    }
}



struct MinOp {
    __device__ __forceinline__ int operator()(int a, int b) const { return min(a, b); }
};

// sufTop[j] = smallest box top row over trials j..n-1 (a whole-grid box counts
// as -2^28).  No trial at or after j conflicts with a box whose bottom row +
// reach lies above sufTop[j], so successor scans stop there.  Components are
// in raster order of their first pixel, so box tops are non-decreasing and
// scans cover only the trials starting within the box's rows (+ reach).
__global__ void __launch_bounds__(1024) k_suffix_top(const int4* __restrict__ boxes, int n,
                                                     int* __restrict__ sufTop) {
    using Scan = cub::BlockScan<int, 1024>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ int carry;
    if (threadIdx.x == 0) carry = 0x7fffffff;
    __syncthreads();
    for (int end = n; end > 0; end -= 1024) {
        const int j = end - 1 - int(threadIdx.x);  // reversed: thread t holds end-1-t
        const int v = j >= 0 ? boxes[j].y : 0x7fffffff;
        int r;
        Scan(tmp).InclusiveScan(v, r, MinOp{});
        r = min(r, carry);
        if (j >= 0) sufTop[j] = r;
        __syncthreads();
        if (threadIdx.x == 1023) carry = r;
        __syncthreads();
    }
}

// pred[j] = number of earlier trials j conflicts with (one warp per trial i
// walks its successors j > i); first[i] = i's first conflicting successor (-1:
// none).
__global__ void k_trial_preds(const int4* __restrict__ boxes, const int* __restrict__ sufTop,
                              int n, int reach, unsigned long long* __restrict__ pred,
                              int* __restrict__ first) {
    const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (i >= n) return;
    const int4 bi = boxes[i];
    const int lim = bi.w + reach;
    int f = -1;
    for (int base = i + 1; base < n; base += 32) {
        if (sufTop[base] > lim) break;
        const int j = base + lane;
        const bool c = j < n && boxes_conflict(bi, boxes[j], reach);
        if (c) atomicAdd(pred + j, 1ull);
        const unsigned m = __ballot_sync(0xffffffffu, c);
        if (f < 0 && m) f = base + __ffs(m) - 1;
    }
    if (lane == 0) first[i] = f;
}

// Seeds ordered by priority (one CTA; n <= kPrioMax): trials with no earlier
// conflict, longest chain first.  A trial's chain length L(i) = 1 + L(first[i])
// -- the path through first successors, a lower bound of its height in the
// conflict DAG that tracks it closely (C4: correlation 0.999 over the seeds) --
// comes from pointer jumping in shared memory.  Index order (k_trial_seed)
// started the C4 critical chain ~300 us late: CTAs keep to their own chains,
// so a seed past the first grid-full waits for one to end.
constexpr int kPrioMax = 12288;
constexpr int kPrioPer = kPrioMax / 1024;
constexpr int kPrioBuckets = 1024;
__global__ void __launch_bounds__(1024) k_trial_seed_prio(const unsigned long long* __restrict__ pred,
                                                          const int* __restrict__ first, int n,
                                                          int* __restrict__ queue,
                                                          int* __restrict__ qTail) {
    extern __shared__ int dynp[];
    int* len = dynp;
    int* nxt = dynp + n;
    __shared__ int hist[kPrioBuckets];
    const int tid = threadIdx.x;
    for (int i = tid; i < n; i += 1024) {
        len[i] = 1;
        nxt[i] = first[i];
    }
    for (int b = tid; b < kPrioBuckets; b += 1024) hist[b] = 0;
    __syncthreads();
    for (;;) {
        int nl[kPrioPer], nn[kPrioPer];
        bool any = false;
#pragma unroll
        for (int k = 0; k < kPrioPer; ++k) {
            const int i = tid + 1024 * k;
            nl[k] = 0;
            nn[k] = -1;
            if (i < n && nxt[i] >= 0) {
                const int x = nxt[i];
                nl[k] = len[i] + len[x];
                nn[k] = nxt[x];
                any = true;
            }
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kPrioPer; ++k) {
            const int i = tid + 1024 * k;
            if (i < n && nxt[i] >= 0) {
                len[i] = nl[k];
                nxt[i] = nn[k];
            }
        }
        if (!__syncthreads_or(any)) break;
    }
    // counting sort of the seeds by descending L (clamped to the buckets)
    int key[kPrioPer];
#pragma unroll
    for (int k = 0; k < kPrioPer; ++k) {
        const int i = tid + 1024 * k;
        key[k] = -1;
        if (i < n && uint32_t(pred[i]) == 0u) {
            key[k] = kPrioBuckets - 1 - min(len[i], kPrioBuckets - 1);
            atomicAdd(hist + key[k], 1);
        }
    }
    __syncthreads();
    using Scan = cub::BlockScan<int, 1024>;
    __shared__ typename Scan::TempStorage tmp;
    int total = 0, pos = 0;
    Scan(tmp).ExclusiveSum(hist[tid], pos, total);
    __syncthreads();
    hist[tid] = pos;
    if (tid == 0) *qTail = total;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kPrioPer; ++k)
        if (key[k] >= 0) queue[atomicAdd(hist + key[k], 1)] = tid + 1024 * k;
}

// Trials with no earlier conflict start ready, in index order within a warp.
__global__ void k_trial_seed(const unsigned long long* __restrict__ pred, int n,
                             int* __restrict__ queue, int* __restrict__ qTail) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x, lane = threadIdx.x & 31;
    const bool ready = j < n && uint32_t(pred[j]) == 0;
    const unsigned m = __ballot_sync(0xffffffffu, ready);
    if (!m) return;
    int base = 0;
    if (lane == __ffs(m) - 1) base = atomicAdd(qTail, __popc(m));
    base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
    if (ready) queue[base + __popc(m & ((1u << lane) - 1))] = j;
}


// Persistent conflict-aware trial scheduler (see the file comment): a
// dependency-counting dataflow schedule with speculation.
//
// Dataflow: CTAs pop ready trials from a FIFO (slot k of `queue` is filled by
// the k-th trial to become ready); a finished trial decrements the counters of
// its conflicting successors and pushes the ones that reach zero, except one
// that runs next on the same CTA (a dependency chain stays put).
//
// Speculation (spec != 0): a trial left waiting on one running predecessor is
// queued for speculation; a CTA with no ready trial takes the newest queued
// one and runs it on chip against the current state, parking the result (its
// new LR cells, params and errors) instead of writing it.  Each trial's 64-bit
// counter holds {accepted predecessors (high), unfinished predecessors (low)};
// a finishing trial updates it with one atomic add.  The speculation snapshots
// the high word before reading any state; when the trial becomes ready its
// record is valid iff the high word is unchanged -- no conflicting predecessor
// was accepted (or wrote in place) meanwhile, and a rejected trial leaves the
// state bit for bit as it found it.  A valid record is committed (a copy
// instead of a re-solve); otherwise the trial runs normally.  Chains of mostly
// rejected trials thus overlap (C2: 57 % rejected, C4: 70 %).  Conflicting
// trials still take effect in index order: the state is bit-identical to the
// sequential loop.
__global__ void __launch_bounds__(kSchedThreads) k_trial_sched(
    TrialState t, TrialBuffers big, char* ctaBufs, const uint32_t* off, const uint32_t* px,
    const uint32_t* ids, int ncomp, const int4* boxes, const int* sufTop, unsigned long long* pred,
    int* queue, int* qHead, int* qTail, int* finished, int reach, int spec, int* specState,
    uint32_t* specSnap, int* specQ, int* specTail, const uint32_t* parkOff, uint32_t* parkBuf,
    uint32_t parkCap) {
    __shared__ TrialSmem<kSchedThreads> sm;
    __shared__ int sIdx, sMode, sUse;
    extern __shared__ __align__(16) char dyn[];
    const TrialShared ss = TrialShared::carve(dyn);
    // The cluster's private buffers (one set per cluster).  CTA rank 0 of the
    // cluster schedules; every CTA of the cluster runs the trial.
    const uint32_t rank = cluster_rank();
    const bool lead = rank == 0;
    char* mine = ctaBufs + size_t(blockIdx.x / kCS) *
                               (size_t(kCtaCells) * 16 + size_t(kCtaPixels) * 20);
    TrialBuffers local;
    local.touched = reinterpret_cast<uint32_t*>(mine);
    local.oldColor = reinterpret_cast<float*>(mine + size_t(kCtaCells) * 4);
    local.aff = reinterpret_cast<uint32_t*>(mine + size_t(kCtaCells) * 16);
    local.bkParams = reinterpret_cast<glu_pixel_params*>(mine + size_t(kCtaCells) * 16 +
                                                         size_t(kCtaPixels) * 4);
    local.bkE = reinterpret_cast<float*>(mine + size_t(kCtaCells) * 16 + size_t(kCtaPixels) * 16);
    static_assert(kSS >= kSchedThreads, "early successor scan covers one CTA width");
    __shared__ int sNext, sCount, sMore;
    __shared__ int sList[kSS];
    for (int k = threadIdx.x; k < kSQ; k += kSchedThreads) ss.key[k] = 0;
    if (threadIdx.x == 0) sNext = -1;
    enum { kExit = 0, kRun = 1, kSpec = 2 };
    for (;;) {
        if (lead && threadIdx.x == 0) {
            int i = sNext, mode = kRun;
#ifdef GLU_SCHED_TRACE
            const unsigned long long tc = gtimer();
#endif
            while (i < 0) {
                const int h = ld_relaxed(qHead);
                if (h < ld_relaxed(qTail)) {
                    // slot h is reserved by a pusher: it fills shortly
                    if (atomicCAS(qHead, h, h + 1) == h)
                        while ((i = ld_relaxed(queue + h)) < 0) __nanosleep(64);
                    continue;
                }
                if (ld_relaxed(finished) >= ncomp) {
                    mode = kExit;
                    break;
                }
                if (spec) {
                    // newest queued speculation first (older entries are mostly
                    // stale: their trials became ready meanwhile)
                    constexpr int kWin = 16;
                    const int tl = ld_relaxed(specTail);
                    int cand[kWin];
#pragma unroll
                    for (int k = 0; k < kWin; ++k)
                        cand[k] = tl - 1 - k >= 0 ? ld_relaxed(specQ + tl - 1 - k) : -1;
                    int got = -1;
#pragma unroll
                    for (int k = 0; k < kWin; ++k) {
                        const int j = cand[k];
                        if (got < 0 && j >= 0 && ld_relaxed(specState + j) == 7 &&
                            parkOff[j + 1] > parkOff[j] && parkOff[j + 1] <= parkCap &&
                            atomicCAS(specState + j, 7, 1) == 7)
                            got = j;
                    }
                    if (got >= 0) {
#ifdef GLU_SCHED_TRACE
                        atomicAdd(&g_phase[21], 1ull);
#endif
                        i = got;
                        mode = kSpec;
                        // accepted-predecessor count, before any of the trial's reads
                        specSnap[got] = uint32_t(ld_relaxed64(pred + got) >> 32);
                        continue;
                    }
                }
                __nanosleep(256);
            }
#ifdef GLU_SCHED_TRACE
            if (mode == kRun) {
                g_trace[3 * i] = tc;
                g_trace[3 * i + 1] = gtimer();
            }
#endif
            cluster_bcast(&sIdx, i);
            cluster_bcast(&sMode, mode);
            sNext = -1;
            sCount = 0;
            sMore = 1;
        }
        cluster_barrier();
        const int i = sIdx, mode = sMode;
        if (mode == kExit) break;
        GLU_DCHECK(i >= 0 && i < ncomp);
        __threadfence();  // acquire: the predecessors' committed writes are visible
        const int4 bi = boxes[i];
        const bool isBig = bi.x < 0;
        const uint32_t c = ids ? ids[i] : uint32_t(i);
        const uint32_t n = off[c + 1] - off[c];
        const TrialGeom geo(bi, t.S / 2, t.lw, t.lh, t.s, t.W, t.H);
        const bool onChip = !isBig && !t.literal && geo.fits(n);
        const SuccScan noScan{nullptr, nullptr, 0,       0,       0,      make_int4(0, 0, 0, 0),
                              nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
        if (mode == kSpec) {
#ifdef GLU_SCHED_TRACE
            if (threadIdx.x == 0) g_trace[3 * ncomp + 2 * i] = gtimer();
#endif
            if (onChip) {
                if (threadIdx.x == 0) sm.parkWords = parkOff[i + 1] - parkOff[i];
                run_trial_smem<kSchedThreads>(t, local, sm, ss, geo, px + off[c], n, noScan,
                                              parkBuf + parkOff[i]);
#ifdef GLU_SCHED_TRACE
                if (threadIdx.x == 0) atomicAdd(&g_phase[18], 1ull);
#endif
            }
            cluster_barrier();  // every CTA's share of the record is written
            if (lead && threadIdx.x == 0) {
#ifdef GLU_SCHED_TRACE
                g_trace[3 * ncomp + 2 * i + 1] = gtimer();
#endif
                __threadfence();
                atomicCAS(specState + i, 1, onChip ? 2 : 3);  // 2: record parked
            }
            cluster_barrier();
            continue;
        }
        // mode == kRun: all conflicting predecessors are final
        if (lead && threadIdx.x == 0) {
            int use = 0;
            if (spec) {
                int st = ld_relaxed(specState + i);
                // a speculation in flight that can still be valid is worth
                // waiting for (it started before this trial became ready)
#ifdef GLU_SCHED_TRACE
                if (st == 1) atomicAdd(&g_phase[22], 1ull);
                if (st == 7) atomicAdd(&g_phase[23], 1ull);
#endif
                const uint32_t acc = uint32_t(ld_relaxed64(pred + i) >> 32);  // final now
                while (st == 1 && acc == ld_relaxed(reinterpret_cast<int*>(specSnap) + i)) {
                    __nanosleep(64);
                    st = ld_relaxed(specState + i);
                }
                if (st == 2 && atomicCAS(specState + i, 2, 5) == 2) {
                    __threadfence();
                    use = acc == specSnap[i];
                }
            }
            cluster_bcast(&sUse, use);
        }
        cluster_barrier();
        int v = 0;
        bool dirty = false;
        if (sUse) {
            v = commit_parked<kSchedThreads>(t, sm, parkBuf + parkOff[i]);
#ifdef GLU_SCHED_TRACE
            if (threadIdx.x == 0) atomicAdd(&g_phase[17], 1ull);
#endif
        } else if (onChip) {
            const SuccScan sc{boxes,   sufTop, ncomp,     reach,     i,
                              bi,      sList,  &sCount,   &sMore,    pred,
                              spec ? specState : nullptr, spec ? specQ : nullptr, specTail};
            v = run_trial_smem<kSchedThreads>(t, local, sm, ss, geo, px + off[c], n, sc);
            if (v) commit_trial_smem<kSchedThreads>(t, local, sm, ss, geo);
        } else {
            if (lead) v = run_trial<kSchedThreads>(t, isBig ? big : local, sm, px + off[c], n);
            dirty = true;  // wrote in place (and rolled back if rejected)
        }
        cluster_barrier();  // the trial's writes, from every CTA, are complete
        if (!lead) continue;
        if (threadIdx.x == 0) {
            atomicAdd(t.result + (v ? 0 : 1), 1);
#ifdef GLU_SCHED_TRACE
            // bit 0: verdict, bit 1: a parked speculative record was committed
            g_trace[3 * i + 2] = (gtimer() & ~3ull) | unsigned(v != 0) | (sUse ? 2u : 0u);
#endif
        }
        __threadfence();  // release this trial's writes (after the trial's last barrier)
#ifdef GLU_SCHED_TRACE
        long long tph = clock64();
#endif
        // Release the conflicting successors (those found early, then the
        // rest).  One successor whose count reaches zero runs next on this CTA;
        // the others go to the FIFO.
        // one predecessor fewer; one more accepted (or in-place) predecessor
        const unsigned long long delta = spec && (v || dirty) ? 0xffffffffull : ~0ull;
        auto release = [&](int j) {
            const int left = int(uint32_t(atomicAdd(pred + j, delta)));
            if (left == 1 && atomicCAS(&sNext, -1, j) != -1) {
                __threadfence();
                const int at = atomicAdd(qTail, 1);
                GLU_DCHECK(at < ncomp);
                st_release(queue + at, j);
            } else if (left == 2 && spec && atomicCAS(specState + j, 0, 7) == 0) {
                const int at = atomicAdd(specTail, 1);  // one predecessor to go
                GLU_DCHECK(at < ncomp);
                st_release(specQ + at, j);
#ifdef GLU_SCHED_TRACE
                atomicAdd(&g_phase[20], 1ull);
#endif
            }
        };
        const int early = sUse ? 0 : sCount;
        if (threadIdx.x < early) release(sList[threadIdx.x]);
        if (sMore) {
            const int lim = bi.w + reach;
            for (int base = (onChip && !sUse) ? i + 1 + kSchedThreads : i + 1; base < ncomp;
                 base += kSchedThreads) {
                if (sufTop[base] > lim) break;
                const int j = base + int(threadIdx.x);
                if (j < ncomp && boxes_conflict(bi, boxes[j], reach)) release(j);
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) atomicAdd(finished, 1);  // after this trial's pushes
        GLU_PHASE(8)
    }
}

inline unsigned blocks_for(size_t n, int threads) {
    return unsigned((n + threads - 1) / threads);
}

struct JointScratch {
    unsigned long long* cellKey;
    uint32_t* cellFlag;
    uint8_t* affMark;
    TrialBuffers big;
    int* result;
};

// Per-context trial scratch: per-LR-cell state (kept zero between trials) and
// per-HR-pixel backup buffers sized for the worst case (every pixel affected).
int joint_scratch(glu_ctx* ctx, const glu_grid& g, JointScratch* js, bool reset) {
    const size_t lowN = size_t(g.lowW) * g.lowH, npx = size_t(g.highW) * g.highH;
    const size_t cellBytes = lowN * (8 + 4 + 1 + 4 + 12) + 64;
    char* cells = static_cast<char*>(scratch(ctx, S_TRIAL, cellBytes + 16 * sizeof(int)));
    char* pix = static_cast<char*>(scratch(ctx, S_TRIAL2, npx * (4 + 12 + 4)));
    if (!cells || !pix) return GLU_ENOMEM;
    js->cellKey = reinterpret_cast<unsigned long long*>(cells);
    js->cellFlag = reinterpret_cast<uint32_t*>(cells + lowN * 8);
    js->big.touched = reinterpret_cast<uint32_t*>(cells + lowN * 12);
    js->big.oldColor = reinterpret_cast<float*>(cells + lowN * 16);
    js->affMark = reinterpret_cast<uint8_t*>(cells + lowN * 28);
    js->result = reinterpret_cast<int*>(cells + ((cellBytes + 15) & ~size_t(15)));
    js->big.aff = reinterpret_cast<uint32_t*>(pix);
    js->big.bkParams = reinterpret_cast<glu_pixel_params*>(pix + npx * 4);
    js->big.bkE = reinterpret_cast<float*>(pix + npx * 16);
    if (reset) {
        cudaError_t e = cudaMemsetAsync(cells, 0, cellBytes + 16 * sizeof(int), ctx->stream);
        if (e != cudaSuccess) return fail_cuda(e, "joint scratch");
    }
    return GLU_OK;
}

TrialState trial_state(const float* high, float* low, glu_pixel_params* field, float* errors,
                       const glu_grid& g, const glu_config& cfg, int mode,
                       const JointScratch& js) {
    TrialState t;
    t.high = high;
    t.low = low;
    t.field = field;
    t.errors = errors;
    t.W = g.highW;
    t.H = g.highH;
    t.s = g.scale;
    t.lw = g.lowW;
    t.lh = g.lowH;
    t.S = cfg.windowSide;
    t.eps = double(cfg.epsilon);
    t.mode = mode;
    t.literal = cfg.literalComponentUpdate;
    t.cellKey = js.cellKey;
    t.cellFlag = js.cellFlag;
    t.affMark = js.affMark;
    t.result = js.result;
    t.dCount = nullptr;
    t.dCells = t.dPixels = nullptr;
    t.dCellCap = t.dPixelCap = 0;
    return t;
}

// Resident CTAs of the persistent scheduler: whole clusters of kCS CTAs.
template <typename K>
int sched_grid(glu_ctx* ctx, K kernel) {
    static thread_local int cached = -1, cachedDev = -1;
    if (cached > 0 && cachedDev == ctx->device) return cached;
    int sms = 0, per = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(kTrialSmemBytes));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, kSchedThreads, kTrialSmemBytes);
    cached = sms * std::max(1, std::min(per, 2));
    if (kCS > 1) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(unsigned(cached));
        cfg.blockDim = dim3(kSchedThreads);
        cfg.dynamicSmemBytes = kTrialSmemBytes;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = kCS;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int clusters = 0;
        if (cudaOccupancyMaxActiveClusters(&clusters, kernel, &cfg) == cudaSuccess && clusters > 0)
            cached = std::min(cached, clusters * kCS) / kCS * kCS;
        else
            cached = cached / kCS * kCS;
        cudaGetLastError();
    }
    cachedDev = ctx->device;
    return cached;
}

// Cooperative launch of the persistent scheduler in clusters of kCS CTAs.
cudaError_t launch_persistent(const void* kernel, int grid, void** args, cudaStream_t st) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(grid));
    cfg.blockDim = dim3(kSchedThreads);
    cfg.dynamicSmemBytes = kTrialSmemBytes;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    int na = 0;
    at[na].id = cudaLaunchAttributeCooperative;
    at[na++].val.cooperative = 1;
    if (kCS > 1) {
        at[na].id = cudaLaunchAttributeClusterDimension;
        at[na].val.clusterDim.x = kCS;
        at[na].val.clusterDim.y = 1;
        at[na++].val.clusterDim.z = 1;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    return cudaLaunchKernelExC(&cfg, kernel, args);
}

#ifdef GLU_SCHED_TRACE
unsigned long long* trace_begin(glu_ctx* ctx, size_t n) {
    unsigned long long* trace = nullptr;
    cudaMalloc(&trace, n * 40 + 8);
    cudaMemsetAsync(trace, 0, n * 40 + 8, ctx->stream);
    cudaMemcpyToSymbolAsync(g_trace, &trace, sizeof(trace), 0, cudaMemcpyHostToDevice,
                            ctx->stream);
    return trace;
}

void trace_end(glu_ctx* ctx, unsigned long long* trace, const int4* boxes, size_t n) {
    std::vector<unsigned long long> h(5 * n);
    std::vector<int4> hb(n);
    cudaMemcpyAsync(h.data(), trace, n * 40, cudaMemcpyDeviceToHost, ctx->stream);
    cudaMemcpyAsync(hb.data(), boxes, n * 16, cudaMemcpyDeviceToHost, ctx->stream);
    cudaStreamSynchronize(ctx->stream);
    cudaFree(trace);
    if (const char* f = getenv("GLU_SCHED_TRACE_FILE")) {
        if (FILE* fp = fopen(f, "ab")) {
            const unsigned long long hdr[2] = {0x5452414346ull, n};
            fwrite(hdr, 8, 2, fp);
            fwrite(h.data(), 8, 5 * n, fp);
            fwrite(hb.data(), 16, n, fp);
            fclose(fp);
        }
    }
    unsigned long long ph[26];
    cudaMemcpyFromSymbol(ph, g_phase, sizeof(ph));
    const unsigned long long z[26] = {};
    cudaMemcpyToSymbol(g_phase, z, sizeof(z));
    if (const char* f = getenv("GLU_SCHED_TRACE_FILE")) {
        if (FILE* fp = fopen((std::string(f) + ".phases").c_str(), "a")) {
            for (int k = 0; k < 26; ++k) fprintf(fp, "%llu ", ph[k]);
            fprintf(fp, "%zu\n", n);
            fclose(fp);
        }
    }
}
#endif

// Parallel conflict-aware schedule of the listed components (all when
// ids == NULL), k_trial_sched; `spec` enables speculation (one more host
// synchronisation: the parked-record sizes are summed to size their storage).
// Asynchronous on ctx->stream otherwise.
int run_sched(glu_ctx* ctx, const TrialState& t, const JointScratch& js, const glu_grid& g,
              const glu_config& cfg, const uint32_t* off, const uint32_t* px,
              const uint32_t* ids, size_t n, bool spec) {
    // No more CTAs than trials (each CTA owns 1.44 MB of private buffers; a
    // small problem needs neither the whole machine nor ~210 MB of them).
    const int grid = std::min(sched_grid(ctx, k_trial_sched),
                              int((std::max<size_t>(n, 1) + kCS - 1) / kCS) * kCS);
    const size_t per = size_t(kCtaCells) * 16 + size_t(kCtaPixels) * 20;
    char* ctaBufs = static_cast<char*>(scratch(ctx, S_SCHED, per * grid));
    // boxes (int4) | pred (u64: accepted << 32 | unfinished) | counters (16) | sufTop |
    // queue | specState | specSnap | specQ | parkOff (n + 1)
    char* meta = static_cast<char*>(scratch(ctx, S_SCHED_META, n * 52 + 128));
    if (!ctaBufs || !meta) return GLU_ENOMEM;
    int4* boxes = reinterpret_cast<int4*>(meta);
    unsigned long long* pred = reinterpret_cast<unsigned long long*>(meta + n * 16);
    int* ctr = reinterpret_cast<int*>(pred + n);
    int *qHead = ctr, *qTail = ctr + 1, *finished = ctr + 2, *specTail = ctr + 3;
    int* sufTop = ctr + 16;
    int* queue = sufTop + n;
    int* specState = queue + n;
    uint32_t* specSnap = reinterpret_cast<uint32_t*>(specState + n);
    int* specQ = reinterpret_cast<int*>(specSnap + n);
    uint32_t* parkOff = reinterpret_cast<uint32_t*>(specQ + n);
    cudaStream_t st = ctx->stream;
    cudaError_t e = cudaSuccess;
    const int reach = 2 * (cfg.windowSide / 2);
    // (the boxes kernel also initialises pred + the counters, the queues and
    // the speculation state: five memsets per sweep fewer, C2 2.26 -> 2.24 ms,
    // C4 2.82 -> 2.78 ms)
    k_trial_boxes<<<blocks_for(n * 32, 256), 256, 0, st>>>(
        off, px, ids, int(n), g.highW, g.scale, g.lowW, g.lowH, cfg.windowSide / 2,
        cfg.literalComponentUpdate, 0, boxes, SchedInit{pred, queue, specState, specQ, specSnap});
    k_suffix_top<<<1, 1024, 0, st>>>(boxes, int(n), sufTop);
    int* first = reinterpret_cast<int*>(parkOff + n + 1);
    k_trial_preds<<<blocks_for(n * 32, 256), 256, 0, st>>>(boxes, sufTop, int(n), reach, pred,
                                                           first);
#ifndef GLU_SEED_PRIO
#define GLU_SEED_PRIO 1
#endif
    // (with no more trials than CTAs every seed starts at once: no order needed)
    if (GLU_SEED_PRIO && n <= size_t(kPrioMax) && n > size_t(grid)) {
        const int smemP = int(n) * 8;
        // (static + dynamic shared memory above 48 KB needs the opt-in; a
        // function attribute is per device, so set on every call)
        const cudaError_t prioAttr = cudaFuncSetAttribute(
            k_trial_seed_prio, cudaFuncAttributeMaxDynamicSharedMemorySize, kPrioMax * 8);
        if (prioAttr != cudaSuccess) return fail_cuda(prioAttr, "trial schedule");
        k_trial_seed_prio<<<1, 1024, smemP, st>>>(pred, first, int(n), queue, qTail);
    } else {
        k_trial_seed<<<blocks_for(n, 256), 256, 0, st>>>(pred, int(n), queue, qTail);
    }
    ctx->launches += 4;
    uint32_t* parkBuf = nullptr;
    uint32_t parkCap = 0;
    if (spec) {
        size_t tb = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tb, parkOff, parkOff, int(n) + 1, st);
        // record sizes, then the scan's temporary storage, in one slot
        const size_t wBytes = ((n + 1) * 4 + 255) & ~size_t(255);
        char* temp = static_cast<char*>(scratch(ctx, S_PARK_TMP, wBytes + tb + 64));
        if (!temp) return GLU_ENOMEM;
        uint32_t* w = reinterpret_cast<uint32_t*>(temp);
        k_park_words<<<blocks_for(n + 1, 256), 256, 0, st>>>(
            boxes, int(n), cfg.windowSide / 2, g.scale, g.lowW, g.lowH, g.highW, g.highH,
            cfg.literalComponentUpdate, w);
        ++ctx->launches;
        e = cub::DeviceScan::ExclusiveSum(temp + wBytes, tb, w, parkOff, int(n) + 1, st);
        if (e != cudaSuccess) return fail_cuda(e, "trial schedule");
        ctx->launches += 2;
        // arena sized on the host without a round trip: n times the largest
        // record an on-chip trial can park (k_park_words: 3 + 5 words per
        // affected pixel of the h-dilated box, <= kSW cells and <= the image,
        // + 4 per replaced cell, <= kSQ), capped at kParkWords; records past
        // its end are simply not speculated (C4 needs ~280 MB, C2 ~60 MB)
        const size_t maxRec = 3 + 5 * std::min(size_t(kSW) * g.scale * g.scale,
                                               size_t(g.highW) * g.highH) + 4 * size_t(kSQ);
        parkCap = uint32_t(std::min(size_t(kParkWords), n * maxRec));
        parkBuf = static_cast<uint32_t*>(scratch(ctx, S_PARK, size_t(parkCap) * 4));
        if (!parkBuf) return GLU_ENOMEM;
    }
    TrialState ts = t;
    TrialBuffers big = js.big;
    int nc = int(n), rch = reach, sp = spec ? 1 : 0;
    void* args[] = {&ts,    &big,      &ctaBufs, &off,       &px,       &ids,
                    &nc,    &boxes,    &sufTop,  &pred,      &queue,    &qHead,
                    &qTail, &finished, &rch,     &sp,        &specState, &specSnap,
                    &specQ, &specTail, &parkOff, &parkBuf, &parkCap};
#ifdef GLU_SCHED_TRACE
    unsigned long long* trace = trace_begin(ctx, n);
#endif
    e = launch_persistent(reinterpret_cast<const void*>(k_trial_sched), grid, args, st);
    ++ctx->launches;
    if (e != cudaSuccess) return fail_cuda(e, "trial schedule");
#ifdef GLU_SCHED_TRACE
    trace_end(ctx, trace, boxes, n);
#endif
    return GLU_OK;
}

}  // namespace

int joint_sweep(glu_ctx* ctx, const float* high, float* low, glu_pixel_params* field,
                float* errors, const glu_grid& g, const glu_config& cfg, int mode,
                const uint32_t* off, const uint32_t* px, size_t ncomp, int* accepted,
                int* rejected) {
    JointScratch js;
    int rc = joint_scratch(ctx, g, &js, true);
    if (rc) return rc;
    const TrialState t = trial_state(high, low, field, errors, g, cfg, mode, js);
    cudaError_t e;
    if (ctx->trials == 1 || ncomp == 1) {
        k_trial_sweep<<<1, kSeqThreads, 0, ctx->stream>>>(t, js.big, off, px, int(ncomp));
        ++ctx->launches;
        e = cudaGetLastError();
    } else {
        rc = ctx->trials == 2 || cfg.literalComponentUpdate
                 ? run_sched(ctx, t, js, g, cfg, off, px, nullptr, ncomp, false)
                 : run_sched(ctx, t, js, g, cfg, off, px, nullptr, ncomp, true);
        if (rc) return rc;
        e = cudaSuccess;
    }
    int* res = reinterpret_cast<int*>(ctx->h_rb + 4);  // (pinned: glu_internal.h)
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(res, js.result, 4 * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) return fail_cuda(e, "trial sweep");
    *accepted = res[0];
    *rejected = res[1];
    return GLU_OK;
}

int trial_one(glu_ctx* ctx, const float* high, float* low, glu_pixel_params* field,
              float* errors, const glu_grid& g, const glu_config& cfg, int mode,
              const uint32_t* comp, size_t n, int* accepted) {
    uint32_t* off = static_cast<uint32_t*>(scratch(ctx, S_TRIAL3, 2 * sizeof(uint32_t)));
    if (!off) return GLU_ENOMEM;
    const uint32_t h[2] = {0, uint32_t(n)};
    cudaError_t e = cudaMemcpyAsync(off, h, sizeof(h), cudaMemcpyHostToDevice, ctx->stream);
    if (e != cudaSuccess) return fail_cuda(e, "trial");
    int acc = 0, rej = 0;
    const int rc = joint_sweep(ctx, high, low, field, errors, g, cfg, mode, off, comp, 1, &acc,
                               &rej);
    if (rc) return rc;
    *accepted = acc;
    return GLU_OK;
}

// ---- building blocks of the distributed joint loop --------------------------------
//
// Every rank holds the full (replicated) LR / params / errors state and finds the
// same components.  The components of a sweep are grouped into levels (level =
// 1 + the highest level of an earlier conflicting component); components of one
// level are mutually independent, so each rank runs its share of a level
// (run_trials with a change log), the ranks exchange the logs of accepted trials
// and apply each other's changes (apply_trial_log).  Any order of independent
// trials gives the sequential result, so every rank ends each level with the
// state the reference's sequential loop has after the same trials.

namespace {

__global__ void k_apply_log(float* __restrict__ low, glu_pixel_params* __restrict__ field,
                            float* __restrict__ errors, const uint32_t* __restrict__ cells,
                            size_t ncells, const uint32_t* __restrict__ pixels, size_t npixels) {
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < ncells; i += stride) {
        const uint32_t* c = cells + 4 * i;
        float* lc = low + 3 * size_t(c[0]);
        lc[0] = __uint_as_float(c[1]);
        lc[1] = __uint_as_float(c[2]);
        lc[2] = __uint_as_float(c[3]);
    }
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < npixels; i += stride) {
        const uint32_t* q = pixels + 5 * i;
        glu_pixel_params pp;
        pp.a = q[1];
        pp.b = q[2];
        pp.w = __uint_as_float(q[3]);
        field[q[0]] = pp;
        errors[q[0]] = __uint_as_float(q[4]);
    }
}

}  // namespace

int component_boxes(glu_ctx* ctx, const uint32_t* off, const uint32_t* px, size_t n,
                    const glu_grid& g, int32_t* boxes) {
    if (n == 0) return GLU_OK;
    k_trial_boxes<<<blocks_for(n * 32, 256), 256, 0, ctx->stream>>>(
        off, px, nullptr, int(n), g.highW, g.scale, g.lowW, g.lowH, 0, 0, 1,
        reinterpret_cast<int4*>(boxes), SchedInit{});
    ++ctx->launches;
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? GLU_OK : fail_cuda(e, "component boxes");
}

int run_trials(glu_ctx* ctx, const float* high, float* low, glu_pixel_params* field,
               float* errors, const glu_grid& g, const glu_config& cfg, int mode,
               const uint32_t* off, const uint32_t* px, const uint32_t* ids, size_t n,
               glu_trial_log* log, int* accepted, int* rejected) {
    JointScratch js;
    int rc = joint_scratch(ctx, g, &js, true);
    if (rc) return rc;
    TrialState t = trial_state(high, low, field, errors, g, cfg, mode, js);
    if (log) {
        t.dCount = log->counts;
        t.dCells = log->cells;
        t.dPixels = log->pixels;
        t.dCellCap = log->cellCapacity;
        t.dPixelCap = log->pixelCapacity;
        cudaError_t e = cudaMemsetAsync(log->counts, 0, 3 * sizeof(uint32_t), ctx->stream);
        if (e != cudaSuccess) return fail_cuda(e, "run_trials");
    }
    if (n) {
        rc = ctx->trials == 2 || cfg.literalComponentUpdate
                 ? run_sched(ctx, t, js, g, cfg, off, px, ids, n, false)
                 : run_sched(ctx, t, js, g, cfg, off, px, ids, n, true);
        if (rc) return rc;
    }
    int res[4];
    cudaError_t e =
        cudaMemcpyAsync(res, js.result, sizeof(res), cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) return fail_cuda(e, "run_trials");
    if (log) {
        uint32_t over = 0;
        e = cudaMemcpy(&over, log->counts + 2, sizeof(over), cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) return fail_cuda(e, "run_trials");
        if (over) {
            set_error("run_trials: change log capacity exceeded");
            return GLU_ENOMEM;
        }
    }
    *accepted = res[0];
    *rejected = res[1];
    return GLU_OK;
}

int apply_trial_log(glu_ctx* ctx, float* low, glu_pixel_params* field, float* errors,
                    const uint32_t* cells, size_t ncells, const uint32_t* pixels,
                    size_t npixels) {
    if (ncells == 0 && npixels == 0) return GLU_OK;
    const size_t work = ncells > npixels ? ncells : npixels;
    const unsigned blocks = unsigned(std::min<size_t>((work + 255) / 256, 148 * 16));
    k_apply_log<<<blocks, 256, 0, ctx->stream>>>(low, field, errors, cells, ncells, pixels,
                                                 npixels);
    ++ctx->launches;
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? GLU_OK : fail_cuda(e, "apply_trial_log");
}

}  // namespace glu_cu
