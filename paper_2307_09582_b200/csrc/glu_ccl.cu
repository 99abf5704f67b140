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
    uint32_t* nsel = mp + npx;  // device counters
    size_t tbSel = 0;
    const AboveThreshold pred{errors, thr};
    thrust::counting_iterator<uint32_t> pix(0);
    cub::DeviceSelect::If(nullptr, tbSel, pix, mp, nsel, int(npx), pred, st);
    void* tsel = scratch(ctx, S_CCL_OFF, tbSel + 64);
    if (!tsel) return GLU_ENOMEM;
    cudaError_t e = cub::DeviceSelect::If(tsel, tbSel, pix, mp, nsel, int(npx), pred, st);
    uint32_t m = 0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&m, nsel, 4, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return fail_cuda(e, "ccl select");
    ctx->launches += 2;
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
    uint32_t tail[2] = {0, 0};
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
