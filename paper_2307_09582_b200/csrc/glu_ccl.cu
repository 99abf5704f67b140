// glu_ccl.cu -- find_large_error (jointopt.cpp:9-46) on the device: the strict
// E > tau mask, 4-connected components, components in raster order of their
// first pixel, each component's pixel list ascending.
//
// A lock-free union-find whose roots are the smallest pixel index of each
// component, so the reference's component order is the order of the roots; a
// stable key sort of the raster-ordered mask pixels by component rank yields
// each component's ascending pixel list.  Two variants: dense (every pixel;
// used when the caller asks for the mask / label images) and sparse (inside
// the joint loop: one selection pass over the error map, then everything over
// the selected pixels' list indices).
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>

#include "glu_internal.h"

namespace glu_cu {

namespace {

constexpr uint32_t kNone = 0xffffffffu;

inline unsigned blocks_for(size_t n, int threads) {
    return unsigned((n + threads - 1) / threads);
}

// ---- connected components ---------------------------------------------------

__global__ void k_ccl_init(const float* __restrict__ e, size_t npx, float thr,
                           uint8_t* __restrict__ mask, uint32_t* __restrict__ parent) {
    const size_t p = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= npx) return;
    const bool m = e[p] > thr;  // strict, jointopt.cpp:17
    mask[p] = m;
    parent[p] = m ? uint32_t(p) : kNone;
}

__device__ __forceinline__ uint32_t find_root(const volatile uint32_t* parent, uint32_t x) {
    uint32_t p = parent[x];
    while (p != x) {
        x = p;
        p = parent[x];
    }
    return x;
}

// Link the larger root under the smaller one; parent[x] <= x always holds.
__device__ void unite(uint32_t* parent, uint32_t a, uint32_t b) {
    for (;;) {
        a = find_root(parent, a);
        b = find_root(parent, b);
        if (a == b) return;
        if (a < b) {
            const uint32_t t = a;
            a = b;
            b = t;
        }
        const uint32_t old = atomicMin(parent + a, b);
        if (old == a) return;
        a = old;  // a was re-linked meanwhile: keep its old parent connected too
    }
}

__global__ void k_ccl_union(const uint8_t* __restrict__ mask, uint32_t* parent, int W, int H) {
    const size_t p = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= size_t(W) * H || !mask[p]) return;
    const int x = int(p % W);
    if (x > 0 && mask[p - 1]) unite(parent, uint32_t(p), uint32_t(p - 1));
    if (p >= size_t(W) && mask[p - W]) unite(parent, uint32_t(p), uint32_t(p - W));
}

__global__ void k_ccl_flatten(uint32_t* parent, size_t npx, uint32_t* __restrict__ isRoot) {
    const size_t p = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= npx) return;
    const uint32_t q = parent[p];
    if (q == kNone) {
        isRoot[p] = 0;
        return;
    }
    const uint32_t r = find_root(parent, q);
    isRoot[p] = (r == p);
    parent[p] = r;
}

// Mask pixels in raster order with their component rank as the sort key.
__global__ void k_ccl_keys(const uint32_t* __restrict__ parent, const uint32_t* __restrict__ rank,
                           const uint32_t* __restrict__ slot, size_t npx,
                           uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
    const size_t p = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= npx) return;
    const uint32_t r = parent[p];
    if (r == kNone) return;
    const uint32_t i = slot[p];  // exclusive scan of mask flags
    keys[i] = rank[r];
    vals[i] = uint32_t(p);
}

__global__ void k_mask_flags(const uint32_t* __restrict__ parent, size_t npx,
                             uint32_t* __restrict__ flags) {
    const size_t p = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p < npx) flags[p] = parent[p] != kNone;
}

__global__ void k_ccl_offsets(const uint32_t* __restrict__ keys, size_t n, uint32_t ncomp,
                              uint32_t* __restrict__ off) {
    const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i == 0) off[ncomp] = uint32_t(n);
    if (i >= n) return;
    if (i == 0 || keys[i] != keys[i - 1]) off[keys[i]] = uint32_t(i);
}

// Sparse variant (the joint loop: no dense mask / label output).  Large-error
// pixels are a small fraction of the image, so after one selection pass over
// the error map (raster-ordered list mp) everything runs over list indices;
// idx[p] maps a mask pixel back to its list index (written for mask pixels
// only -- a neighbour is looked up only after the error map says it is one).
// List order is raster order, so min-index roots are again the components'
// first pixels.
struct AboveThreshold {
    const float* e;
    float thr;
    __device__ __forceinline__ bool operator()(const uint32_t& p) const { return e[p] > thr; }
};

// The selection of the mask pixels in raster order, in two passes over
// chunks of kSelChunk pixels: k_sel_mask reads the error map once (float4
// loads) and writes the chunk's mask as bits and its count; after an
// exclusive scan of the counts, k_sel_write expands each chunk's bits into
// pixel indices at the chunk's offset.  (CUB's DeviceSelect over a counting
// iterator read the map with scalar loads: ~2.5x slower.)
constexpr int kSelChunk = 4096, kSelThreads = 256;  // 16 pixels per thread
constexpr int kSelWords = kSelChunk / 32;

__global__ void __launch_bounds__(kSelThreads) k_sel_mask(const float* __restrict__ e, size_t npx,
                                                          float thr, uint32_t* __restrict__ bits,
                                                          uint32_t* __restrict__ counts) {
    const size_t c0 = size_t(blockIdx.x) * kSelChunk;
    const int lane = threadIdx.x & 31;
    uint32_t cnt = 0;
    const bool vec = (reinterpret_cast<uintptr_t>(e) & 15u) == 0;
#pragma unroll
    for (int k = 0; k < kSelChunk / (4 * kSelThreads); ++k) {
        const int q = k * kSelThreads + threadIdx.x;  // quad of the chunk
        const size_t p = c0 + 4 * size_t(q);
        float v[4];
        if (vec && p + 4 <= npx) {
            const float4 f = __ldcs(reinterpret_cast<const float4*>(e + p));
            v[0] = f.x, v[1] = f.y, v[2] = f.z, v[3] = f.w;
        } else {
#pragma unroll
            for (int c = 0; c < 4; ++c) v[c] = p + c < npx ? e[p + c] : thr;
        }
        uint32_t nib = 0;
#pragma unroll
        for (int c = 0; c < 4; ++c) nib |= uint32_t(v[c] > thr) << c;  // strict, NaN: no
        cnt += __popc(nib);
        // the word of quads 8j .. 8j + 7 (32 pixels): 8 lanes' nibbles
        uint32_t w = nib << (4 * (lane & 7));
        w |= __shfl_xor_sync(0xffffffffu, w, 1);
        w |= __shfl_xor_sync(0xffffffffu, w, 2);
        w |= __shfl_xor_sync(0xffffffffu, w, 4);
        if ((lane & 7) == 0) bits[size_t(blockIdx.x) * kSelWords + q / 8] = w;
    }
    using BR = cub::BlockReduce<uint32_t, kSelThreads>;
    __shared__ typename BR::TempStorage tmp;
    const uint32_t total = BR(tmp).Sum(cnt);
    if (threadIdx.x == 0) counts[blockIdx.x] = total;
}

__global__ void __launch_bounds__(kSelWords) k_sel_write(const uint32_t* __restrict__ bits,
                                                         const uint32_t* __restrict__ off,
                                                         uint32_t* __restrict__ mp) {
    using BS = cub::BlockScan<uint32_t, kSelWords>;
    __shared__ typename BS::TempStorage tmp;
    uint32_t w = bits[size_t(blockIdx.x) * kSelWords + threadIdx.x];
    uint32_t pre;
    BS(tmp).ExclusiveSum(uint32_t(__popc(w)), pre);
    uint32_t* o = mp + off[blockIdx.x] + pre;
    const uint32_t base = blockIdx.x * uint32_t(kSelChunk) + 32u * threadIdx.x;
    for (; w; w &= w - 1) *o++ = base + uint32_t(__ffs(w) - 1);
}

__global__ void k_sparse_init(const uint32_t* __restrict__ mp, uint32_t m,
                              uint32_t* __restrict__ idx, uint32_t* __restrict__ parent) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= m) return;
    idx[mp[k]] = k;
    parent[k] = k;
}

__global__ void k_sparse_union(const uint32_t* __restrict__ mp, uint32_t m,
                               const float* __restrict__ e, float thr,
                               const uint32_t* __restrict__ idx, uint32_t* parent, int W) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= m) return;
    const uint32_t p = mp[k];
    if (p % uint32_t(W) > 0 && e[p - 1] > thr) unite(parent, k, idx[p - 1]);
    if (p >= uint32_t(W) && e[p - W] > thr) unite(parent, k, idx[p - W]);
}

__global__ void k_sparse_flatten(uint32_t* parent, uint32_t m, uint32_t* __restrict__ isRoot) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= m) return;
    const uint32_t r = find_root(parent, parent[k]);
    isRoot[k] = r == k;
    parent[k] = r;
}

__global__ void k_sparse_keys(const uint32_t* __restrict__ parent, const uint32_t* __restrict__ rank,
                              uint32_t m, uint32_t* __restrict__ keys) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < m) keys[k] = rank[parent[k]];
}

}  // namespace

namespace {

int ccl_sparse(glu_ctx* ctx, const float* errors, int W, int H, float thr, size_t* count,
               const uint32_t** offOut, const uint32_t** pxOut) {
    const size_t npx = size_t(W) * H;
    cudaStream_t st = ctx->stream;
    uint32_t* mp = static_cast<uint32_t*>(scratch(ctx, S_CCL_LIST, npx * 4 + 64));
    uint32_t* idx = static_cast<uint32_t*>(scratch(ctx, S_CCL_LABEL, npx * 4));
    if (!mp || !idx) return GLU_ENOMEM;
    // selection: chunk masks + counts, scan, expansion (k_sel_mask / k_sel_write)
    const size_t nch = (npx + kSelChunk - 1) / kSelChunk;
    size_t tbSel = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tbSel, static_cast<uint32_t*>(nullptr),
                                  static_cast<uint32_t*>(nullptr), int(nch) + 1, st);
    // bits (nch * kSelWords) | counts (nch + 1) | offsets (nch + 1) | scan temp
    const size_t selWords = nch * kSelWords + 2 * (nch + 1);
    char* sel = static_cast<char*>(scratch(ctx, S_CCL_OFF, selWords * 4 + 256 + tbSel));
    if (!sel) return GLU_ENOMEM;
    uint32_t* selBits = reinterpret_cast<uint32_t*>(sel);
    uint32_t* cnts = selBits + nch * kSelWords;
    uint32_t* coff = cnts + nch + 1;
    void* tsel = sel + ((selWords * 4 + 255) & ~size_t(255));
    cudaError_t e = cudaMemsetAsync(cnts + nch, 0, 4, st);
    if (e == cudaSuccess) {
        k_sel_mask<<<unsigned(nch), kSelThreads, 0, st>>>(errors, npx, thr, selBits, cnts);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess)
        e = cub::DeviceScan::ExclusiveSum(tsel, tbSel, cnts, coff, int(nch) + 1, st);
    if (e == cudaSuccess) {
        k_sel_write<<<unsigned(nch), kSelWords, 0, st>>>(selBits, coff, mp);
        e = cudaGetLastError();
    }
    // (read-backs through the context's pinned words)
    if (e == cudaSuccess) e = cudaMemcpyAsync(ctx->h_rb, coff + nch, 4, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return fail_cuda(e, "ccl select");
    const uint32_t m = ctx->h_rb[0];
    ctx->launches += 4;
    // parent | isRoot | rank | keys | keys2 | vals2 (m words each)
    uint32_t* w = static_cast<uint32_t*>(scratch(ctx, S_CCL_MISC, size_t(m) * 24 + 64));
    if (!w) return GLU_ENOMEM;
    uint32_t* parent = w;
    uint32_t* isRoot = w + m;
    uint32_t* rank = w + 2 * size_t(m);
    uint32_t* keys = w + 3 * size_t(m);
    uint32_t* keys2 = w + 4 * size_t(m);
    uint32_t* vals2 = w + 5 * size_t(m);
    *count = 0;
    *pxOut = vals2;
    if (m == 0) {
        *offOut = vals2;
        return GLU_OK;
    }
    k_sparse_init<<<blocks_for(m, 256), 256, 0, st>>>(mp, m, idx, parent);
    k_sparse_union<<<blocks_for(m, 256), 256, 0, st>>>(mp, m, errors, thr, idx, parent, W);
    k_sparse_flatten<<<blocks_for(m, 256), 256, 0, st>>>(parent, m, isRoot);
    ctx->launches += 3;
    size_t tbScan = 0, tbSort = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tbScan, isRoot, rank, int(m), st);
    cub::DeviceRadixSort::SortPairs(nullptr, tbSort, keys, keys2, mp, vals2, int(m), 0, 32, st);
    const size_t tb = std::max(tbScan, tbSort);
    void* temp = scratch(ctx, S_CCL_OFF, ((tb + 255) & ~size_t(255)) + size_t(m) * 4 + 64);
    if (!temp) return GLU_ENOMEM;
    uint32_t* off = reinterpret_cast<uint32_t*>(static_cast<char*>(temp) + ((tb + 255) & ~size_t(255)));
    e = cub::DeviceScan::ExclusiveSum(temp, tbScan, isRoot, rank, int(m), st);
    uint32_t* tail = ctx->h_rb + 2;
    if (e == cudaSuccess) e = cudaMemcpyAsync(tail, rank + m - 1, 4, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(tail + 1, isRoot + m - 1, 4, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return fail_cuda(e, "ccl rank");
    const uint32_t ncomp = tail[0] + tail[1];
    k_sparse_keys<<<blocks_for(m, 256), 256, 0, st>>>(parent, rank, m, keys);
    ++ctx->launches;
    int bits = 1;
    while (bits < 32 && (uint64_t(1) << bits) <= ncomp) ++bits;
    // stable: each component's pixels stay in raster order
    e = cub::DeviceRadixSort::SortPairs(temp, tbSort, keys, keys2, mp, vals2, int(m), 0, bits, st);
    if (e != cudaSuccess) return fail_cuda(e, "ccl sort");
    k_ccl_offsets<<<blocks_for(m, 256), 256, 0, st>>>(keys2, m, ncomp, off);
    ++ctx->launches;
    e = cudaGetLastError();
    if (e != cudaSuccess) return fail_cuda(e, "ccl");
    *count = ncomp;
    *offOut = off;
    return GLU_OK;
}

}  // namespace

int ccl_find_large_error(glu_ctx* ctx, const float* errors, int W, int H, float thr,
                         uint8_t* mask, uint32_t* label, size_t* count, const uint32_t** offOut,
                         const uint32_t** pxOut) {
    const size_t npx = size_t(W) * H;
    if (!mask && !label && offOut && pxOut && npx < (size_t(1) << 31))
        return ccl_sparse(ctx, errors, W, H, thr, count, offOut, pxOut);
    cudaStream_t st = ctx->stream;
    uint8_t* dmask = mask ? mask : static_cast<uint8_t*>(scratch(ctx, S_CCL_MISC, npx));
    uint32_t* parent = label ? label : static_cast<uint32_t*>(scratch(ctx, S_CCL_LABEL, npx * 4));
    // flags/rank/slot + keys/vals (+ sorted copies)
    uint32_t* work = static_cast<uint32_t*>(scratch(ctx, S_CCL_LIST, npx * 4 * 6 + 64));
    if (!dmask || !parent || !work) return GLU_ENOMEM;
    uint32_t* flags = work;
    uint32_t* rank = work + npx;
    uint32_t* keys = work + 2 * npx;
    uint32_t* vals = work + 3 * npx;
    uint32_t* keys2 = work + 4 * npx;
    uint32_t* vals2 = work + 5 * npx;
    cudaError_t e;
    k_ccl_init<<<blocks_for(npx, 256), 256, 0, st>>>(errors, npx, thr, dmask, parent);
    k_ccl_union<<<blocks_for(npx, 256), 256, 0, st>>>(dmask, parent, W, H);
    k_ccl_flatten<<<blocks_for(npx, 256), 256, 0, st>>>(parent, npx, flags);
    ctx->launches += 3;
    // rank of each root = component id (raster order of the smallest pixel).
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, flags, rank, int(npx), st);
    size_t tbSort = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tbSort, keys, keys2, vals, vals2, int(npx), 0, 32,
                                    st);
    void* temp = scratch(ctx, S_CCL_OFF, std::max(tb, tbSort) + npx * 4 + 64);
    if (!temp) return GLU_ENOMEM;
    uint32_t* off = reinterpret_cast<uint32_t*>(static_cast<char*>(temp) +
                                                ((std::max(tb, tbSort) + 255) & ~size_t(255)));
    e = cub::DeviceScan::ExclusiveSum(temp, tb, flags, rank, int(npx), st);
    if (e != cudaSuccess) return fail_cuda(e, "ccl scan");
    // totals: ncomp = rank[last] + flags[last]
    uint32_t ncomp = 0, nmask = 0;
    {
        uint32_t lastRank, lastFlag;
        e = cudaMemcpyAsync(&lastRank, rank + npx - 1, 4, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(&lastFlag, flags + npx - 1, 4, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) return fail_cuda(e, "ccl count");
        ncomp = lastRank + lastFlag;
    }
    // mask slots
    k_mask_flags<<<blocks_for(npx, 256), 256, 0, st>>>(parent, npx, flags);
    ++ctx->launches;
    e = cub::DeviceScan::ExclusiveSum(temp, tb, flags, keys2, int(npx), st);  // keys2 = slots
    if (e != cudaSuccess) return fail_cuda(e, "ccl slots");
    {
        uint32_t lastSlot, lastFlag;
        e = cudaMemcpyAsync(&lastSlot, keys2 + npx - 1, 4, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(&lastFlag, flags + npx - 1, 4, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) return fail_cuda(e, "ccl count");
        nmask = lastSlot + lastFlag;
    }
    *count = ncomp;
    if (ncomp == 0) {
        if (offOut) *offOut = off;
        if (pxOut) *pxOut = vals2;
        return GLU_OK;
    }
    k_ccl_keys<<<blocks_for(npx, 256), 256, 0, st>>>(parent, rank, keys2, npx, keys, vals);
    ++ctx->launches;
    int bits = 1;
    while (bits < 32 && (uint64_t(1) << bits) <= ncomp) ++bits;
    e = cub::DeviceRadixSort::SortPairs(temp, tbSort, keys, keys2, vals, vals2, int(nmask), 0,
                                        bits, st);
    if (e != cudaSuccess) return fail_cuda(e, "ccl sort");
    k_ccl_offsets<<<blocks_for(nmask, 256), 256, 0, st>>>(keys2, nmask, ncomp, off);
    ++ctx->launches;
    e = cudaGetLastError();
    if (e != cudaSuccess) return fail_cuda(e, "ccl");
    if (offOut) *offOut = off;
    if (pxOut) *pxOut = vals2;
    return GLU_OK;
}

}  // namespace glu_cu
