// glu_glup.cu -- GLUP parameter files on device buffers (
// reference: proj/src/io_glup.cpp:48-139, format in proj/README.md:97-117).
//
// Layout (little endian): 32-byte header {"GLUP", u32 version = 1, u32 highW,
// highH, scale, lowW, lowH, u8 mode, u8 optimized, u8 0, u8 0}, then the LR
// image as lowW*lowH*3 f32, then one {u32 a, u32 b, f32 w} record per HR
// pixel.  The device buffers already hold exactly these bytes, so encoding is
// a header plus two straight copies (device -> pinned host) and decoding is
// the reverse plus one validation kernel that finds the first offending LR
// sample / pixel record in the reference's check order (io_glup.cpp:121-137).
#include <cuda_runtime.h>

#include <cstring>
#include <string>

#include "glu_internal.h"

namespace glu_cu {

namespace {

constexpr unsigned long long kNoViolation = ~0ull;

// key = 2 * position + kind; the smallest key is the reference's first error.
__global__ void k_glup_validate(const float* __restrict__ low, size_t lowFloats,
                                const glu_pixel_params* __restrict__ field, size_t npx,
                                unsigned lowCount, unsigned long long* firstBad) {
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < lowFloats; i += stride) {
        const float v = low[i];
        if (!(isfinite(v) && v >= 0.0f && v <= 1.0f)) atomicMin(firstBad, 2ull * i);
    }
    const unsigned long long base = 2ull * lowFloats;
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < npx; i += stride) {
        const glu_pixel_params pp = field[i];
        if (pp.a >= lowCount || pp.b >= lowCount)
            atomicMin(firstBad, base + 2ull * i);
        else if (!isfinite(pp.w))
            atomicMin(firstBad, base + 2ull * i + 1);
    }
}

void put32(uint8_t* p, uint32_t v) {
    p[0] = uint8_t(v);
    p[1] = uint8_t(v >> 8);
    p[2] = uint8_t(v >> 16);
    p[3] = uint8_t(v >> 24);
}

uint32_t get32(const uint8_t* p) {
    return uint32_t(p[0]) | uint32_t(p[1]) << 8 | uint32_t(p[2]) << 16 | uint32_t(p[3]) << 24;
}

thread_local std::string g_field;

int format_error(const char* field, const std::string& msg) {
    g_field = field;
    set_error(msg);
    return GLU_EFORMAT;
}

}  // namespace

}  // namespace glu_cu

using namespace glu_cu;

extern "C" {

const char* glu_last_error_field(void) { return g_field.c_str(); }

size_t glu_glup_size(const glu_grid* g) {
    if (!g) return 0;
    return 32 + 12 * size_t(g->lowW) * g->lowH + 12 * size_t(g->highW) * g->highH;
}

int glu_cu_glup_encode(glu_ctx* ctx, const glu_pixel_params* field, const float* low,
                       const glu_grid* g, int mode, int optimized, uint8_t* out, size_t cap) {
    if (!ctx) {
        set_error("ctx must not be null");
        return GLU_EINVAL;
    }
    if (!g || g->highW <= 0 || g->highH <= 0 || g->scale < 2) {
        set_error("encode_glup: field has no grid");
        return GLU_EINVAL;
    }
    if (g->lowW != (g->highW + g->scale - 1) / g->scale ||
        g->lowH != (g->highH + g->scale - 1) / g->scale) {
        set_error("encode_glup: low-res image does not match grid");
        return GLU_EINVAL;
    }
    if (mode < 0 || mode > 2) {
        set_error("encode_glup: unknown mode");
        return GLU_EINVAL;
    }
    const size_t lowBytes = 12 * size_t(g->lowW) * g->lowH;
    const size_t parBytes = 12 * size_t(g->highW) * g->highH;
    if (!out || cap < 32 + lowBytes + parBytes) {
        set_error("encode_glup: output buffer too small");
        return GLU_EINVAL;
    }
    uint8_t h[32];
    std::memcpy(h, "GLUP", 4);
    put32(h + 4, 1);
    put32(h + 8, uint32_t(g->highW));
    put32(h + 12, uint32_t(g->highH));
    put32(h + 16, uint32_t(g->scale));
    put32(h + 20, uint32_t(g->lowW));
    put32(h + 24, uint32_t(g->lowH));
    h[28] = uint8_t(mode);
    h[29] = optimized ? 1 : 0;
    h[30] = h[31] = 0;
    cudaPointerAttributes attr{};
    const bool hostOut = cudaPointerGetAttributes(&attr, out) != cudaSuccess ||
                         attr.type != cudaMemoryTypeDevice;
    cudaGetLastError();
    const cudaMemcpyKind kind = hostOut ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
    cudaError_t e = cudaMemcpyAsync(out, h, 32, hostOut ? cudaMemcpyHostToHost
                                                        : cudaMemcpyHostToDevice, ctx->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(out + 32, low, lowBytes, kind, ctx->stream);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(out + 32 + lowBytes, field, parBytes, kind, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) return fail_cuda(e, "encode_glup");
    return GLU_OK;
}

int glu_cu_glup_decode(glu_ctx* ctx, const uint8_t* bytes, size_t n, glu_grid* gOut,
                       int* modeOut, int* optimizedOut, float* low, glu_pixel_params* field) {
    if (!ctx) {
        set_error("ctx must not be null");
        return GLU_EINVAL;
    }
    g_field.clear();
    if (n < 32 || !bytes)
        return format_error("length", "parameter file shorter than its 32-byte header");
    uint8_t h[32];
    cudaPointerAttributes attr{};
    const bool hostIn = cudaPointerGetAttributes(&attr, bytes) != cudaSuccess ||
                        attr.type != cudaMemoryTypeDevice;
    cudaGetLastError();
    if (hostIn)
        std::memcpy(h, bytes, 32);
    else if (cudaMemcpy(h, bytes, 32, cudaMemcpyDeviceToHost) != cudaSuccess)
        return fail_cuda(cudaGetLastError(), "decode_glup");
    if (std::memcmp(h, "GLUP", 4) != 0) return format_error("magic", "not a GLUP parameter file");
    const uint32_t version = get32(h + 4);
    if (version != 1)
        return format_error("version",
                            "unsupported parameter file version " + std::to_string(version));
    const uint32_t W = get32(h + 8), H = get32(h + 12), s = get32(h + 16);
    const uint32_t lw = get32(h + 20), lh = get32(h + 24);
    const uint8_t mode = h[28], flag = h[29];
    if (W == 0 || H == 0 || s < 2 || lw == 0 || lh == 0)
        return format_error("dims", "parameter file has degenerate dimensions");
    if (s >= (W < H ? W : H)) return format_error("dims", "scale is not smaller than the image");
    if (lw != (size_t(W) + s - 1) / s || lh != (size_t(H) + s - 1) / s)
        return format_error("dims", "low-res dimensions do not match size and scale");
    if (mode > 2) return format_error("mode", "unknown mode byte " + std::to_string(mode));
    if (flag > 1) return format_error("flag", "optimized flag must be 0 or 1");
    if (h[30] != 0 || h[31] != 0)
        return format_error("reserved", "reserved header bytes must be zero");
    const size_t lowCount = size_t(lw) * lh, npx = size_t(W) * H;
    const size_t expect = 32 + 12 * lowCount + 12 * npx;
    if (n != expect)
        return format_error("length", "parameter file is " + std::to_string(n) +
                                          " bytes, expected " + std::to_string(expect));
    if (W > 0x7fffffffu || H > 0x7fffffffu || npx > 0xffffffffull) {
        set_error("decode_glup: image exceeds 2^32 pixels");
        return GLU_EINVAL;
    }
    if (gOut) {
        gOut->scale = int(s);
        gOut->highW = int(W);
        gOut->highH = int(H);
        gOut->lowW = int(lw);
        gOut->lowH = int(lh);
        gOut->sampleOffset = int(s / 2);
    }
    if (modeOut) *modeOut = mode;
    if (optimizedOut) *optimizedOut = flag;
    if (!low || !field) return GLU_OK;  // header-only ("peek") call
    const cudaMemcpyKind kind = hostIn ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
    cudaError_t e = cudaMemcpyAsync(low, bytes + 32, 12 * lowCount, kind, ctx->stream);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(field, bytes + 32 + 12 * lowCount, 12 * npx, kind, ctx->stream);
    unsigned long long* bad = ctx->d_counters + 2;
    const unsigned long long none = kNoViolation;
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(bad, &none, sizeof(none), cudaMemcpyHostToDevice, ctx->stream);
    if (e == cudaSuccess) {
        k_glup_validate<<<148 * 8, 256, 0, ctx->stream>>>(low, 3 * lowCount, field, npx,
                                                          unsigned(lowCount), bad);
        ++ctx->launches;
        e = cudaGetLastError();
    }
    unsigned long long first = none;
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(&first, bad, sizeof(first), cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) return fail_cuda(e, "decode_glup");
    if (first != none) {
        if (first < 2ull * 3 * lowCount)
            return format_error("lowres", "low-res sample outside [0, 1]");
        if ((first & 1ull) == 0)
            return format_error("index", "pixel record references a cell outside the grid");
        return format_error("weight", "pixel record has a non-finite weight");
    }
    return GLU_OK;
}

}  // extern "C"
