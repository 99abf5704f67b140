// glu_capi.cu -- the C-ABI (include/glu_cuda.h): contexts, validation with
// the reference's error texts, device-pointer and host-pointer entry points.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "glu_internal.h"

namespace glu_cu {

namespace {
thread_local std::string g_last_error;
}

void set_error(const std::string& msg) { g_last_error = msg; }

int fail_cuda(cudaError_t e, const char* where) {
    set_error(std::string(where) + ": " + cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? GLU_ENOMEM : GLU_ECUDA;
}

void* scratch(glu_ctx* ctx, int slot, size_t bytes) {
    if (bytes == 0) bytes = 1;
    if (ctx->cap[slot] >= bytes) return ctx->buf[slot];
    if (ctx->buf[slot]) {
        cudaStreamSynchronize(ctx->stream);
        cudaFree(ctx->buf[slot]);
        ctx->buf[slot] = nullptr;
        ctx->cap[slot] = 0;
    }
    const size_t want = bytes + bytes / 8;
    if (cudaMalloc(&ctx->buf[slot], want) != cudaSuccess) {
        cudaGetLastError();
        set_error("out of device memory");
        return nullptr;
    }
    ctx->cap[slot] = want;
    return ctx->buf[slot];
}

}  // namespace glu_cu

using namespace glu_cu;

namespace {

int einval(const char* msg) {
    set_error(msg);
    return GLU_EINVAL;
}

int check_grid(const glu_grid* g) {
    if (!g) return einval("grid must not be null");
    if (g->highW <= 0 || g->highH <= 0) return einval("GridSpec: dimensions must be positive");
    if (g->scale < 2) return einval("GridSpec: scale must be >= 2");
    if (g->scale >= (g->highW < g->highH ? g->highW : g->highH))
        return einval("GridSpec: scale must be < min(width, height)");
    if (g->lowW != (g->highW + g->scale - 1) / g->scale ||
        g->lowH != (g->highH + g->scale - 1) / g->scale)
        return einval("GridSpec: low-res dimensions inconsistent with scale");
    if (size_t(g->highW) * size_t(g->highH) > 0xffffffffull)
        return einval("GridSpec: image exceeds 2^32 pixels");
    return GLU_OK;
}

size_t npx_of(const glu_grid* g) { return size_t(g->highW) * g->highH; }
size_t lown_of(const glu_grid* g) { return size_t(g->lowW) * g->lowH; }

// Records and floats are read / written as 4-byte words (the vector apply
// peels any head that is not 16-byte aligned, launch_apply).
int check_apply_alignment(const void* field, const void* target, const void* out) {
    if ((reinterpret_cast<uintptr_t>(field) | reinterpret_cast<uintptr_t>(target) |
         reinterpret_cast<uintptr_t>(out)) % 4 != 0)
        return einval("apply_field: buffers must be 4-byte aligned");
    return GLU_OK;
}

int check_mode(int mode) {
    if (mode < 0 || mode > 2) return einval("unknown mode (expected fast|exact|gnu)");
    return GLU_OK;
}

#define GLU_TRY(expr)              \
    do {                           \
        const int rc_ = (expr);    \
        if (rc_ != GLU_OK) return rc_; \
    } while (0)

#define GLU_CUDA(expr, where)                              \
    do {                                                   \
        const cudaError_t e_ = (expr);                     \
        if (e_ != cudaSuccess) return fail_cuda(e_, where); \
    } while (0)

SolveArgs solve_args(const float* high, const float* low, const glu_grid* g,
                     const glu_config* cfg, int mode) {
    SolveArgs a{};
    a.high = high;
    a.low = low;
    a.W = g->highW;
    a.H = g->highH;
    a.s = g->scale;
    a.lw = g->lowW;
    a.lh = g->lowH;
    a.S = cfg->windowSide;
    a.eps = double(cfg->epsilon);  // GluConfig::epsilon is a float (upsample.cpp:201)
    a.mode = mode;
    return a;
}

template <typename T>
T* dev(glu_ctx* ctx, int slot, size_t count) {
    return static_cast<T*>(scratch(ctx, slot, count * sizeof(T)));
}

int h2d(glu_ctx* ctx, void* d, const void* h, size_t bytes) {
    GLU_CUDA(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, ctx->stream), "copy to device");
    return GLU_OK;
}

int d2h_sync(glu_ctx* ctx, void* h, const void* d, size_t bytes) {
    if (bytes) GLU_CUDA(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, ctx->stream),
                        "copy to host");
    GLU_CUDA(cudaStreamSynchronize(ctx->stream), "synchronize");
    return GLU_OK;
}

}  // namespace

extern "C" {

int glu_abi_version(void) { return GLU_CUDA_ABI_VERSION; }

const char* glu_last_error(void) { return g_last_error.c_str(); }

const char* glu_build_info(void) {
    return "glu_cuda sm_100a; fp32 filter + fp64 verify selection (bit-exact); -fmad=false; "
           "built " __DATE__ " " __TIME__;
}

int glu_grid_create(int highW, int highH, int scale, glu_grid* out) {
    if (!out) return einval("grid must not be null");
    if (highW <= 0 || highH <= 0) return einval("GridSpec: dimensions must be positive");
    if (scale < 2) return einval("GridSpec: scale must be >= 2");
    if (scale >= (highW < highH ? highW : highH))
        return einval("GridSpec: scale must be < min(width, height)");
    out->scale = scale;
    out->highW = highW;
    out->highH = highH;
    out->lowW = (highW + scale - 1) / scale;
    out->lowH = (highH + scale - 1) / scale;
    out->sampleOffset = scale / 2;
    return GLU_OK;
}

int glu_config_validate(const glu_config* c) {
    if (!c) return einval("config must not be null");
    if (c->windowSide < 3 || c->windowSide % 2 == 0)
        return einval("GluConfig: windowSide must be odd and >= 3");
    if (!(c->errorThreshold >= 0)) return einval("GluConfig: errorThreshold must be >= 0");
    if (c->maxIterations < 0) return einval("GluConfig: maxIterations must be >= 0");
    if (!(c->epsilon > 0)) return einval("GluConfig: epsilon must be > 0");
    return GLU_OK;
}

glu_config glu_config_default(void) {
    glu_config c;
    c.windowSide = 3;
    c.errorThreshold = 30.0f / 255.0f;
    c.maxIterations = 3;
    c.epsilon = 1e-3f;
    c.literalComponentUpdate = 0;
    return c;
}

int glu_current_device(int* device) {
    if (!device) return einval("device must not be null");
    GLU_CUDA(cudaGetDevice(device), "cudaGetDevice");
    return GLU_OK;
}

int glu_ctx_create(int device, glu_ctx** out) {
    if (!out) return einval("ctx must not be null");
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
        cudaGetLastError();
        set_error("no CUDA device available");
        return GLU_ECUDA;
    }
    if (device < 0 || device >= n) return einval("device index out of range");
    GLU_CUDA(cudaSetDevice(device), "cudaSetDevice");
    glu_ctx* c = new glu_ctx();
    c->device = device;
    e = cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        delete c;
        return fail_cuda(e, "stream");
    }
    c->stream = c->own;
    e = cudaEventCreateWithFlags(&c->switchEv, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaMalloc(&c->d_counters, 8 * sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMemset(c->d_counters, 0, 8 * sizeof(unsigned long long));
    if (e == cudaSuccess)
        e = cudaHostAlloc(reinterpret_cast<void**>(&c->h_rb), 16 * sizeof(uint32_t),
                          cudaHostAllocDefault);
    if (e != cudaSuccess) {
        cudaStreamDestroy(c->own);
        delete c;
        return fail_cuda(e, "counters");
    }
    *out = c;
    return GLU_OK;
}

int glu_ctx_destroy(glu_ctx* ctx) {
    if (!ctx) return GLU_OK;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    for (int i = 0; i < glu_ctx::kSlots; ++i)
        if (ctx->buf[i]) cudaFree(ctx->buf[i]);
    for (void* h : ctx->hbuf)
        if (h) cudaFreeHost(h);
    cudaFree(ctx->d_counters);
    if (ctx->h_rb) cudaFreeHost(ctx->h_rb);
    for (cudaEvent_t ev : ctx->ev)
        if (ev) cudaEventDestroy(ev);
    if (ctx->switchEv) cudaEventDestroy(ctx->switchEv);
    for (cudaEvent_t ev : ctx->pev)
        if (ev) cudaEventDestroy(ev);
    if (ctx->side) cudaStreamDestroy(ctx->side);
    if (ctx->h2d) cudaStreamDestroy(ctx->h2d);
    if (ctx->d2h) cudaStreamDestroy(ctx->d2h);
    cudaStreamDestroy(ctx->own);
    delete ctx;
    return GLU_OK;
}

int glu_ctx_set_stream(glu_ctx* ctx, void* s) {
    if (!ctx) return einval("ctx must not be null");
    cudaStream_t next = s ? static_cast<cudaStream_t>(s) : ctx->own;
    if (next != ctx->stream) {
        // The scratch slots and counters are shared by every stream this
        // context is bound to: order the new stream after everything already
        // issued on the old one.
        GLU_CUDA(cudaEventRecord(ctx->switchEv, ctx->stream), "stream switch");
        GLU_CUDA(cudaStreamWaitEvent(next, ctx->switchEv, 0), "stream switch");
        ctx->stream = next;
    }
    return GLU_OK;
}

void* glu_ctx_stream(glu_ctx* ctx) { return ctx ? ctx->stream : nullptr; }

int glu_ctx_set_option(glu_ctx* ctx, int option, int value) {
    if (!ctx) return einval("ctx must not be null");
    if (option == GLU_OPT_SOLVER) {
        if (value < 0 || value > 2) return einval("GLU_OPT_SOLVER: value must be 0, 1 or 2");
        ctx->solver = value;
        return GLU_OK;
    }
    if (option == GLU_OPT_TRIALS) {
        if (value < 0 || value > 2) return einval("GLU_OPT_TRIALS: value must be 0, 1 or 2");
        ctx->trials = value;
        return GLU_OK;
    }
    return einval("unknown option");
}

int glu_ctx_synchronize(glu_ctx* ctx) {
    if (!ctx) return einval("ctx must not be null");
    GLU_CUDA(cudaStreamSynchronize(ctx->stream), "synchronize");
    return GLU_OK;
}

unsigned long long glu_ctx_launch_count(glu_ctx* ctx) { return ctx ? ctx->launches : 0; }

unsigned long long glu_ctx_fallback_count(glu_ctx* ctx) {
    if (!ctx) return 0;
    unsigned long long v = 0;
    cudaMemcpy(&v, ctx->d_counters, sizeof(v), cudaMemcpyDeviceToHost);
    return v;
}

unsigned long long glu_ctx_close_set_count(glu_ctx* ctx) {
    if (!ctx) return 0;
    unsigned long long v = 0;
    cudaMemcpy(&v, ctx->d_counters + 1, sizeof(v), cudaMemcpyDeviceToHost);
    return v;
}

// ---- device entry points ------------------------------------------------------

int glu_cu_copy(glu_ctx* ctx, void* dst, const void* src, size_t bytes) {
    if (!ctx) return einval("ctx must not be null");
    if (bytes == 0) return GLU_OK;
    GLU_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, ctx->stream), "copy");
    return GLU_OK;
}

int glu_cu_alloc(glu_ctx* ctx, void** ptr, size_t bytes) {
    if (!ctx || !ptr) return einval("ctx and ptr must not be null");
    GLU_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
    GLU_CUDA(cudaMalloc(ptr, bytes ? bytes : 1), "cudaMalloc");
    return GLU_OK;
}

int glu_cu_free(glu_ctx* ctx, void* ptr) {
    if (!ctx) return einval("ctx must not be null");
    GLU_CUDA(cudaStreamSynchronize(ctx->stream), "synchronize");
    GLU_CUDA(cudaFree(ptr), "cudaFree");
    return GLU_OK;
}

int glu_cu_upload(glu_ctx* ctx, void* dst, const void* src, size_t bytes) {
    if (!ctx) return einval("ctx must not be null");
    if (bytes == 0) return GLU_OK;
    GLU_TRY(h2d(ctx, dst, src, bytes));
    GLU_CUDA(cudaStreamSynchronize(ctx->stream), "synchronize");
    return GLU_OK;
}

int glu_cu_download(glu_ctx* ctx, void* dst, const void* src, size_t bytes) {
    if (!ctx) return einval("ctx must not be null");
    return d2h_sync(ctx, dst, src, bytes);
}

int glu_cu_grid_downsample(glu_ctx* ctx, const float* high, const glu_grid* g, float* low) {
    if (!ctx) return einval("ctx must not be null");
    GLU_TRY(check_grid(g));
    GLU_CUDA(launch_grid_downsample(ctx, high, g->highW, g->highH, g->scale, g->lowW, g->lowH,
                                    low),
             "grid_downsample");
    return GLU_OK;
}

int glu_cu_optimize_field(glu_ctx* ctx, const float* high, const float* low, const glu_grid* g,
                          const glu_config* cfg, int mode, glu_pixel_params* out) {
    if (!ctx) return einval("ctx must not be null");
    GLU_TRY(glu_config_validate(cfg));
    GLU_TRY(check_grid(g));
    GLU_TRY(check_mode(mode));
    SolveArgs a = solve_args(high, low, g, cfg, mode);
    a.params = out;
    a.fallbacks = ctx->d_counters;
    GLU_CUDA(launch_solve(ctx, a), "optimize_field");
    return GLU_OK;
}

int glu_cu_optimize_pixels(glu_ctx* ctx, const float* high, const float* low, const glu_grid* g,
                           const glu_config* cfg, int mode, const uint32_t* pixels, size_t count,
                           glu_pixel_params* field) {
    if (!ctx) return einval("ctx must not be null");
    GLU_TRY(glu_config_validate(cfg));
    GLU_TRY(check_grid(g));
    GLU_TRY(check_mode(mode));
    SolveArgs a = solve_args(high, low, g, cfg, mode);
    a.params = field;
    GLU_CUDA(launch_solve_list(ctx, a, pixels, count), "optimize_pixels");
    return GLU_OK;
}

int glu_cu_apply_field(glu_ctx* ctx, const glu_pixel_params* field, const glu_grid* g,
                       const float* lowTarget, int channels, int clampOutput, float* out) {
    if (!ctx) return einval("ctx must not be null");
    GLU_TRY(check_grid(g));
    if (channels != 1 && channels != 3) return einval("apply_field: channels must be 1 or 3");
    GLU_TRY(check_apply_alignment(field, lowTarget, out));
    GLU_CUDA(launch_apply(ctx, field, npx_of(g), lowTarget, lown_of(g), channels, clampOutput, out),
             "apply_field");
    return GLU_OK;
}

int glu_cu_apply_field_band(glu_ctx* ctx, const glu_pixel_params* bandField, size_t bandPixels,
                            const glu_grid* g, const float* lowTarget, int channels,
                            int clampOutput, float* out) {
    if (!ctx) return einval("ctx must not be null");
    GLU_TRY(check_grid(g));
    if (channels != 1 && channels != 3) return einval("apply_field: channels must be 1 or 3");
    if (bandPixels > npx_of(g)) return einval("apply_field: band exceeds the grid");
    if (bandPixels == 0) return GLU_OK;
    GLU_TRY(check_apply_alignment(bandField, lowTarget, out));
    GLU_CUDA(launch_apply(ctx, bandField, bandPixels, lowTarget, lown_of(g), channels,
                          clampOutput, out),
             "apply_field");
    return GLU_OK;
}

int glu_cu_error_map(glu_ctx* ctx, const float* high, const float* recon, size_t n,
                     float* errors) {
    if (!ctx) return einval("ctx must not be null");
    if (n == 0) return GLU_OK;
    GLU_CUDA(launch_error_map(ctx, high, recon, n, errors), "error_map");
    return GLU_OK;
}

int glu_cu_self_error_map(glu_ctx* ctx, const float* high, const glu_pixel_params* field,
                          const glu_grid* g, const float* low, float* errors) {
    if (!ctx) return einval("ctx must not be null");
    GLU_TRY(check_grid(g));
    GLU_CUDA(launch_self_error(ctx, high, field, npx_of(g), low, errors), "self_error_map");
    return GLU_OK;
}

int glu_cu_solve_apply(glu_ctx* ctx, const float* high, const float* low, const glu_grid* g,
                       const glu_config* cfg, int mode, const float* lowTarget, int channels,
                       int clampOutput, float* out, glu_pixel_params* paramsOut) {
    if (!ctx) return einval("ctx must not be null");
    GLU_TRY(glu_config_validate(cfg));
    GLU_TRY(check_grid(g));
    GLU_TRY(check_mode(mode));
    if (channels != 1 && channels != 3) return einval("apply_field: channels must be 1 or 3");
    if (!lowTarget || !out) return einval("solve_apply: target and output required");
    SolveArgs a = solve_args(high, low, g, cfg, mode);
    a.params = paramsOut;
    a.lowT = lowTarget;
    a.channels = channels;
    a.clamp = clampOutput;
    a.out = out;
    a.fallbacks = ctx->d_counters;
    GLU_CUDA(launch_solve(ctx, a), "solve_apply");
    return GLU_OK;
}

int glu_cu_find_large_error(glu_ctx* ctx, const float* errors, int width, int height,
                            float threshold, uint8_t* mask, uint32_t* label, size_t* count,
                            const uint32_t** compOffsets, const uint32_t** compPixels) {
    if (!ctx) return einval("ctx must not be null");
    if (width <= 0 || height <= 0) return einval("find_large_error: empty error map");
    size_t n = 0;
    GLU_TRY(ccl_find_large_error(ctx, errors, width, height, threshold, mask, label, &n,
                                 compOffsets, compPixels));
    if (count) *count = n;
    return GLU_OK;
}

int glu_cu_trial_update_component(glu_ctx* ctx, const float* high, float* low,
                                  glu_pixel_params* field, float* errors, const glu_grid* g,
                                  const glu_config* cfg, int mode, const uint32_t* component,
                                  size_t count, int* accepted) {
    if (!ctx) return einval("ctx must not be null");
    GLU_TRY(glu_config_validate(cfg));
    if (count == 0) return einval("trial_update_component: empty component");
    GLU_TRY(check_grid(g));
    GLU_TRY(check_mode(mode));
    int acc = 0;
    GLU_TRY(trial_one(ctx, high, low, field, errors, *g, *cfg, mode, component, count, &acc));
    if (accepted) *accepted = acc;
    return GLU_OK;
}

int glu_cu_joint_optimize(glu_ctx* ctx, const float* high, const glu_grid* g,
                          const glu_config* cfg, int mode, float* low, glu_pixel_params* field,
                          float* errors, glu_joint_stats* stats) {
    if (!ctx) return einval("ctx must not be null");
    GLU_TRY(glu_config_validate(cfg));
    GLU_TRY(check_grid(g));
    GLU_TRY(check_mode(mode));
    // jointopt.cpp:182-206: downsample, solve, self error map, then sweeps.
    GLU_CUDA(launch_grid_downsample(ctx, high, g->highW, g->highH, g->scale, g->lowW, g->lowH,
                                    low),
             "joint_optimize");
    SolveArgs a = solve_args(high, low, g, cfg, mode);
    a.params = field;
    a.errOut = errors;  // self error map fused into the solve
    a.fallbacks = ctx->d_counters;
    GLU_CUDA(launch_solve(ctx, a), "joint_optimize");
    glu_joint_stats st{0, 0, 0, 0};
    for (int it = 0; it < cfg->maxIterations; ++it) {
        size_t ncomp = 0;
        const uint32_t* off = nullptr;
        const uint32_t* px = nullptr;
        GLU_TRY(ccl_find_large_error(ctx, errors, g->highW, g->highH, cfg->errorThreshold,
                                     nullptr, nullptr, &ncomp, &off, &px));
        if (ncomp == 0) break;
        ++st.iterations;
        st.components += int(ncomp);
        int acc = 0, rej = 0;
        GLU_TRY(joint_sweep(ctx, high, low, field, errors, *g, *cfg, mode, off, px, ncomp, &acc,
                            &rej));
        st.trialsAccepted += acc;
        st.trialsRejected += rej;
        if (acc == 0) break;
    }
    if (stats) *stats = st;
    return GLU_OK;
}

}  // extern "C"

namespace {

// One frame of the pipeline on ctx->stream: downsample -> target op -> fused solve+apply.
int frame_kernels(glu_ctx* ctx, const float* frame, const glu_grid* g, const glu_config* cfg,
                  int mode, int targetOp, float* low, float* target, float* out,
                  glu_pixel_params* params) {
    if (ctx->solver != 1 && solve32_supported(mode, cfg->windowSide, g->scale)) {
        // downsample + matte + LR packing fused into one launch before the solve
        const bool matte = targetOp == GLU_TARGET_MATTE;
        SolveArgs a = solve_args(frame, low, g, cfg, mode);
        a.params = params;
        a.lowT = matte ? target : low;
        a.channels = matte ? 1 : 3;
        a.clamp = 1;
        a.out = out;
        a.fallbacks = ctx->d_counters;
        GLU_CUDA(launch_frame_solve32(ctx, a, low, matte ? target : nullptr, ctx->solver == 2),
                 "upsample_frames");
        return GLU_OK;
    }
    GLU_CUDA(launch_grid_downsample(ctx, frame, g->highW, g->highH, g->scale, g->lowW, g->lowH,
                                    low),
             "upsample_frames");
    const float* t = low;
    int ch = 3;
    if (targetOp == GLU_TARGET_MATTE) {
        GLU_CUDA(launch_op_matte(ctx, low, lown_of(g), target), "upsample_frames");
        t = target;
        ch = 1;
    }
    SolveArgs a = solve_args(frame, low, g, cfg, mode);
    a.params = params;
    a.lowT = t;
    a.channels = ch;
    a.clamp = 1;
    a.out = out;
    a.fallbacks = ctx->d_counters;
    GLU_CUDA(launch_solve(ctx, a), "upsample_frames");
    return GLU_OK;
}

// Device frames (all resident at the call): frame k's k_frame_prep runs on a
// side stream into buffer set k % 2 while frame k - 1 is solved on the
// context stream (the prep is a small grid: it fills the solve's last wave).
// Prep k waits for solve k - 2 (its buffers); solve k waits for prep k.
#ifndef GLU_FRAME_BATCH_EXACT
#define GLU_FRAME_BATCH_EXACT 1  // Exact mode (k_solve32x) also in one launch per batch
#endif
#ifndef GLU_FRAME_BATCH
#define GLU_FRAME_BATCH 1
#endif

int frames_pipelined(glu_ctx* ctx, const float* frames, int count, const glu_grid* g,
                     const glu_config* cfg, int mode, int targetOp, float* out,
                     glu_pixel_params* paramsOut) {
    const size_t n = npx_of(g), ln = lown_of(g);
    const bool matte = targetOp == GLU_TARGET_MATTE;
    const int ch = matte ? 1 : 3;
    const int h = cfg->windowSide / 2;
    const size_t cells = size_t(g->lowW + 2 * h) * (g->lowH + 2 * h);
    // per buffer set: low (3 ln floats) | matte (ln) | packed (cells float4) | nanFlag
    const size_t setBytes = ((ln * 16 + 255) & ~size_t(255)) + cells * 16 + 256;
    char* base = static_cast<char*>(scratch(ctx, S_SPARE2, 2 * setBytes));
    if (!base) return GLU_ENOMEM;
    if (!ctx->side) {
        GLU_CUDA(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking), "stream");
        for (cudaEvent_t& ev : ctx->pev)
            GLU_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event");
    }
    cudaEvent_t* prepped = ctx->pev;     // [2]
    cudaEvent_t* solved = ctx->pev + 2;  // [2]
    cudaEvent_t entry = ctx->pev[4];
    // the side stream starts after everything already issued on the context stream
    GLU_CUDA(cudaEventRecord(entry, ctx->stream), "pipeline");
    GLU_CUDA(cudaStreamWaitEvent(ctx->side, entry, 0), "pipeline");
    for (int k = 0; k < count; ++k) {
        const int b = k & 1;
        char* set = base + b * setBytes;
        float* low = reinterpret_cast<float*>(set);
        float* tgt = low + 3 * ln;
        float4* packed = reinterpret_cast<float4*>(set + ((ln * 16 + 255) & ~size_t(255)));
        unsigned* nanFlag = reinterpret_cast<unsigned*>(packed + cells);
        SolveArgs a = solve_args(frames + size_t(k) * n * 3, low, g, cfg, mode);
        a.params = paramsOut ? paramsOut + size_t(k) * n : nullptr;
        a.lowT = matte ? tgt : low;
        a.channels = ch;
        a.clamp = 1;
        a.out = out + size_t(k) * n * ch;
        a.fallbacks = ctx->d_counters;
        if (k >= 2) GLU_CUDA(cudaStreamWaitEvent(ctx->side, solved[b], 0), "pipeline");
        GLU_CUDA(launch_frame_prep(ctx, ctx->side, a, low, matte ? tgt : nullptr, packed, nanFlag),
                 "upsample_frames");
        GLU_CUDA(cudaEventRecord(prepped[b], ctx->side), "pipeline");
        GLU_CUDA(cudaStreamWaitEvent(ctx->stream, prepped[b], 0), "pipeline");
        GLU_CUDA(launch_prepped_solve32(ctx, a, packed, ctx->solver == 2, nanFlag),
                 "upsample_frames");
        GLU_CUDA(cudaEventRecord(solved[b], ctx->stream), "pipeline");
    }
    return GLU_OK;
}

// Fast / GNU / Exact, S = 3, matte target, no params: the frames go through
// k_solve32f (Exact: k_solve32x) in batches of up to kFrameBatch per launch
// (grid z = frame), so
// the SMs never drain between frames; one batched prep launch per batch, the
// next batch's on the side stream while this one solves.
#ifndef GLU_FRAME_BATCH_MAX
#define GLU_FRAME_BATCH_MAX 16
#endif
constexpr int kFrameBatch = GLU_FRAME_BATCH_MAX;

int frames_batched(glu_ctx* ctx, const float* frames, int count, const glu_grid* g,
                   const glu_config* cfg, int mode, float* out) {
    const size_t n = npx_of(g), ln = lown_of(g);
    const int h = cfg->windowSide / 2;
    const size_t cells = size_t(g->lowW + 2 * h) * (g->lowH + 2 * h);
    // per frame: low (3 ln floats) | matte (ln floats) | packed (cells float4)
    const size_t offMatte = (ln * 12 + 255) & ~size_t(255);
    const size_t offPacked = offMatte + ((ln * 4 + 255) & ~size_t(255));
    const size_t set = (offPacked + cells * 16 + 255) & ~size_t(255);
    const int B = std::min(count, kFrameBatch);
    char* base = static_cast<char*>(scratch(ctx, S_SPARE2, 2 * size_t(B) * set + 2 * B * 4 + 64));
    if (!base) return GLU_ENOMEM;
    unsigned* flagBase = reinterpret_cast<unsigned*>(base + 2 * size_t(B) * set);
    if (!ctx->side) {
        GLU_CUDA(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking), "stream");
        for (cudaEvent_t& ev : ctx->pev)
            GLU_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event");
    }
    cudaEvent_t* prepped = ctx->pev;     // [2] per batch buffer group
    cudaEvent_t* solved = ctx->pev + 2;  // [2]
    GLU_CUDA(cudaEventRecord(ctx->pev[4], ctx->stream), "pipeline");
    GLU_CUDA(cudaStreamWaitEvent(ctx->side, ctx->pev[4], 0), "pipeline");
    for (int k0 = 0, bi = 0; k0 < count; k0 += B, ++bi) {
        const int nb = std::min(B, count - k0), grp = bi & 1;
        char* gb = base + size_t(grp) * B * set;
        unsigned* flags = flagBase + grp * B;
        SolveArgs a = solve_args(frames + size_t(k0) * n * 3, reinterpret_cast<float*>(gb), g,
                                 cfg, mode);
        a.params = nullptr;
        a.lowT = reinterpret_cast<float*>(gb + offMatte);
        a.channels = 1;
        a.clamp = 1;
        a.out = out + size_t(k0) * n;
        a.fallbacks = ctx->d_counters;
        FrameBatch fb;
        fb.frames = nb;
        fb.high = n * 3;
        fb.px = n;
        fb.lowT = set / 4;
        fb.packed = set / 16;
        if (bi >= 2) GLU_CUDA(cudaStreamWaitEvent(ctx->side, solved[grp], 0), "pipeline");
        GLU_CUDA(launch_frame_prep_batch(ctx, ctx->side, a, fb, gb, set, offMatte, offPacked, flags),
                 "upsample_frames");
        GLU_CUDA(cudaEventRecord(prepped[grp], ctx->side), "pipeline");
        GLU_CUDA(cudaStreamWaitEvent(ctx->stream, prepped[grp], 0), "pipeline");
        GLU_CUDA(launch_prepped_solve32f_batch(ctx, a, reinterpret_cast<float4*>(gb + offPacked),
                                               ctx->solver == 2, flags, fb),
                 "upsample_frames");
        GLU_CUDA(cudaEventRecord(solved[grp], ctx->stream), "pipeline");
    }
    return GLU_OK;
}

int check_frames(glu_ctx* ctx, int count, const glu_grid* g, const glu_config* cfg, int mode,
                 int targetOp) {
    if (!ctx) return einval("ctx must not be null");
    GLU_TRY(glu_config_validate(cfg));
    GLU_TRY(check_grid(g));
    GLU_TRY(check_mode(mode));
    if (count < 0) return einval("upsample_frames: count must be >= 0");
    if (targetOp != GLU_TARGET_IDENTITY && targetOp != GLU_TARGET_MATTE)
        return einval("upsample_frames: unknown target operator");
    return GLU_OK;
}

}  // namespace

extern "C" {

int glu_cu_upsample_frames(glu_ctx* ctx, const float* frames, int count, const glu_grid* g,
                           const glu_config* cfg, int mode, int targetOp, float* out,
                           glu_pixel_params* paramsOut) {
    GLU_TRY(check_frames(ctx, count, g, cfg, mode, targetOp));
    const size_t n = npx_of(g), ln = lown_of(g);
    const int ch = targetOp == GLU_TARGET_MATTE ? 1 : 3;
    if (count > 1 && ctx->solver != 1 && !paramsOut && targetOp == GLU_TARGET_MATTE &&
        (solve32f_supported(mode, cfg->windowSide) ||
         (GLU_FRAME_BATCH_EXACT && solve32x_supported(mode, cfg->windowSide, g->scale))) &&
        GLU_FRAME_BATCH)
        return frames_batched(ctx, frames, count, g, cfg, mode, out);
    if (count > 1 && ctx->solver != 1 && solve32_supported(mode, cfg->windowSide, g->scale))
        return frames_pipelined(ctx, frames, count, g, cfg, mode, targetOp, out, paramsOut);
    float* low = dev<float>(ctx, S_LOW, ln * 3);
    float* tgt = dev<float>(ctx, S_AUX, ln);
    if (!low || !tgt) return GLU_ENOMEM;
    for (int k = 0; k < count; ++k)
        GLU_TRY(frame_kernels(ctx, frames + size_t(k) * n * 3, g, cfg, mode, targetOp, low, tgt,
                              out + size_t(k) * n * ch, paramsOut ? paramsOut + size_t(k) * n
                                                                  : nullptr));
    return GLU_OK;
}

int glu_h_upsample_frames(glu_ctx* ctx, const float* frames, int count, const glu_grid* g,
                          const glu_config* cfg, int mode, int targetOp, float* out,
                          glu_pixel_params* paramsOut) {
    GLU_TRY(check_frames(ctx, count, g, cfg, mode, targetOp));
    if (count == 0) return GLU_OK;
    const size_t n = npx_of(g), ln = lown_of(g);
    const int ch = targetOp == GLU_TARGET_MATTE ? 1 : 3;
    if (!ctx->h2d) {
        GLU_CUDA(cudaStreamCreateWithFlags(&ctx->h2d, cudaStreamNonBlocking), "stream");
        GLU_CUDA(cudaStreamCreateWithFlags(&ctx->d2h, cudaStreamNonBlocking), "stream");
        for (cudaEvent_t& ev : ctx->ev)
            GLU_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event");
    }
    // Two device slots per buffer: frame k uses slot k % 2.
    float* dframe = dev<float>(ctx, S_HIGH, 2 * n * 3);
    float* dout = dev<float>(ctx, S_OUT, 2 * n * ch);
    glu_pixel_params* dpar = paramsOut ? dev<glu_pixel_params>(ctx, S_PARAMS, 2 * n) : nullptr;
    float* low = dev<float>(ctx, S_LOW, ln * 3);
    float* tgt = dev<float>(ctx, S_AUX, ln);
    if (!dframe || !dout || !low || !tgt || (paramsOut && !dpar)) return GLU_ENOMEM;
    cudaEvent_t* inReady = ctx->ev;      // [2] frame slot filled
    cudaEvent_t* computed = ctx->ev + 2;  // [2] frame slot consumed, output slot written
    cudaEvent_t* drained = ctx->ev + 4;   // [2] output slot copied out
    for (int k = 0; k < count; ++k) {
        const int sl = k & 1;
        float* f = dframe + size_t(sl) * n * 3;
        float* o = dout + size_t(sl) * n * ch;
        glu_pixel_params* pp = dpar ? dpar + size_t(sl) * n : nullptr;
        if (k >= 2) GLU_CUDA(cudaStreamWaitEvent(ctx->h2d, computed[sl], 0), "pipeline");
        GLU_CUDA(cudaMemcpyAsync(f, frames + size_t(k) * n * 3, n * 12, cudaMemcpyHostToDevice,
                                 ctx->h2d),
                 "copy to device");
        GLU_CUDA(cudaEventRecord(inReady[sl], ctx->h2d), "pipeline");
        GLU_CUDA(cudaStreamWaitEvent(ctx->stream, inReady[sl], 0), "pipeline");
        if (k >= 2) GLU_CUDA(cudaStreamWaitEvent(ctx->stream, drained[sl], 0), "pipeline");
        GLU_TRY(frame_kernels(ctx, f, g, cfg, mode, targetOp, low, tgt, o, pp));
        GLU_CUDA(cudaEventRecord(computed[sl], ctx->stream), "pipeline");
        GLU_CUDA(cudaStreamWaitEvent(ctx->d2h, computed[sl], 0), "pipeline");
        GLU_CUDA(cudaMemcpyAsync(out + size_t(k) * n * ch, o, n * ch * 4, cudaMemcpyDeviceToHost,
                                 ctx->d2h),
                 "copy to host");
        if (pp)
            GLU_CUDA(cudaMemcpyAsync(paramsOut + size_t(k) * n, pp, n * 12,
                                     cudaMemcpyDeviceToHost, ctx->d2h),
                     "copy to host");
        GLU_CUDA(cudaEventRecord(drained[sl], ctx->d2h), "pipeline");
    }
    GLU_CUDA(cudaStreamSynchronize(ctx->d2h), "synchronize");
    GLU_CUDA(cudaStreamSynchronize(ctx->stream), "synchronize");
    return GLU_OK;
}

int glu_cu_fp32_peak(glu_ctx* ctx, double* tflops, double* sm_mhz) {
    if (!ctx) return einval("ctx must not be null");
    int sms = 0, clk = 0;
    GLU_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device), "attr");
    float* sink = dev<float>(ctx, S_SPARE2, 1024);
    if (!sink) return GLU_ENOMEM;
    cudaEvent_t e0, e1;
    GLU_CUDA(cudaEventCreate(&e0), "event");
    GLU_CUDA(cudaEventCreate(&e1), "event");
    const int threads = 256, blocks = sms * 8, iters = 1 << 14;
    GLU_CUDA(launch_ffma_probe(ctx, sink, iters / 16, blocks, threads), "ffma");  // warm-up
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0, ctx->stream);
        GLU_CUDA(launch_ffma_probe(ctx, sink, iters, blocks, threads), "ffma");
        cudaEventRecord(e1, ctx->stream);
        GLU_CUDA(cudaEventSynchronize(e1), "ffma");
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    const double flops = 2.0 * 8.0 * double(iters) * double(blocks) * threads;
    if (tflops) *tflops = flops / (best * 1e-3) / 1e12;
    // 128 FP32 lanes per SM: clock = FFMA rate / (128 * SMs)
    if (sm_mhz) *sm_mhz = flops / 2.0 / (best * 1e-3) / (128.0 * sms) / 1e6;
    (void)clk;
    return GLU_OK;
}

int glu_cu_component_boxes(glu_ctx* ctx, const uint32_t* off, const uint32_t* px, size_t n,
                           const glu_grid* g, int32_t* boxes) {
    if (!ctx) return einval("ctx must not be null");
    GLU_TRY(check_grid(g));
    return component_boxes(ctx, off, px, n, *g, boxes);
}

int glu_trial_levels(const int32_t* boxes, size_t n, int reach, int32_t* levels) {
    if ((n && (!boxes || !levels)) || reach < 0) return einval("glu_trial_levels: bad arguments");
    // Spatial bins of kBin x kBin cells; a component only has to be checked
    // against earlier components registered in the bins its dilated box covers.
    constexpr int kBin = 16;
    int maxX = 0, maxY = 0;
    for (size_t i = 0; i < n; ++i) {
        maxX = std::max(maxX, boxes[4 * i + 2]);
        maxY = std::max(maxY, boxes[4 * i + 3]);
    }
    const int bw = maxX / kBin + 1, bh = maxY / kBin + 1;
    std::vector<std::vector<uint32_t>> bins(size_t(bw) * bh);
    for (size_t i = 0; i < n; ++i) {
        const int32_t* b = boxes + 4 * i;
        const int x0 = std::max(0, b[0] - reach), y0 = std::max(0, b[1] - reach);
        const int x1 = b[2] + reach, y1 = b[3] + reach;
        int lvl = 1;
        for (int by = y0 / kBin; by <= std::min(bh - 1, y1 / kBin); ++by)
            for (int bx = x0 / kBin; bx <= std::min(bw - 1, x1 / kBin); ++bx)
                for (uint32_t j : bins[size_t(by) * bw + bx]) {
                    const int32_t* c = boxes + 4 * size_t(j);
                    const int dx = std::max(0, std::max(c[0] - b[2], b[0] - c[2]));
                    const int dy = std::max(0, std::max(c[1] - b[3], b[1] - c[3]));
                    if (std::max(dx, dy) <= reach) lvl = std::max(lvl, levels[j] + 1);
                }
        levels[i] = lvl;
        for (int by = b[1] / kBin; by <= b[3] / kBin; ++by)
            for (int bx = b[0] / kBin; bx <= b[2] / kBin; ++bx)
                bins[size_t(by) * bw + bx].push_back(uint32_t(i));
    }
    return GLU_OK;
}

int glu_trial_rounds(const int32_t* boxes, size_t n, int reach, const int32_t* owners,
                     int32_t* rounds) {
    if ((n && (!boxes || !owners || !rounds)) || reach < 0)
        return einval("glu_trial_rounds: bad arguments");
    // the bins of glu_trial_levels
    constexpr int kBin = 16;
    int maxX = 0, maxY = 0;
    for (size_t i = 0; i < n; ++i) {
        maxX = std::max(maxX, boxes[4 * i + 2]);
        maxY = std::max(maxY, boxes[4 * i + 3]);
    }
    const int bw = maxX / kBin + 1, bh = maxY / kBin + 1;
    std::vector<std::vector<uint32_t>> bins(size_t(bw) * bh);
    for (size_t i = 0; i < n; ++i) {
        const int32_t* b = boxes + 4 * i;
        const int x0 = std::max(0, b[0] - reach), y0 = std::max(0, b[1] - reach);
        const int x1 = b[2] + reach, y1 = b[3] + reach;
        int r = 0;
        for (int by = y0 / kBin; by <= std::min(bh - 1, y1 / kBin); ++by)
            for (int bx = x0 / kBin; bx <= std::min(bw - 1, x1 / kBin); ++bx)
                for (uint32_t j : bins[size_t(by) * bw + bx]) {
                    const int32_t* c = boxes + 4 * size_t(j);
                    const int dx = std::max(0, std::max(c[0] - b[2], b[0] - c[2]));
                    const int dy = std::max(0, std::max(c[1] - b[3], b[1] - c[3]));
                    if (std::max(dx, dy) <= reach)
                        r = std::max(r, rounds[j] + (owners[j] != owners[i] ? 1 : 0));
                }
        rounds[i] = r;
        for (int by = b[1] / kBin; by <= b[3] / kBin; ++by)
            for (int bx = b[0] / kBin; bx <= b[2] / kBin; ++bx)
                bins[size_t(by) * bw + bx].push_back(uint32_t(i));
    }
    return GLU_OK;
}

int glu_cu_downsample_band(glu_ctx* ctx, const float* high, const glu_grid* g, int r0, int r1,
                           float* low) {
    if (!ctx) return einval("ctx must not be null");
    GLU_TRY(check_grid(g));
    if (r0 < 0 || r1 > g->lowH || r0 > r1) return einval("band: LR rows out of range");
    if (r0 == r1) return GLU_OK;
    // the band's sample pixels min(cy s + s/2, H - 1) lie in its HR rows
    const int y0 = r0 * g->scale, y1 = std::min(r1 * g->scale, g->highH);
    GLU_CUDA(launch_grid_downsample(ctx, high + size_t(y0) * g->highW * 3, g->highW, y1 - y0,
                                    g->scale, g->lowW, r1 - r0, low + size_t(r0) * g->lowW * 3),
             "downsample_band");
    return GLU_OK;
}

int glu_cu_solve_band(glu_ctx* ctx, const float* high, const float* low, const glu_grid* g,
                      const glu_config* cfg, int mode, int r0, int r1, glu_pixel_params* field,
                      float* errors) {
    if (!ctx) return einval("ctx must not be null");
    GLU_TRY(glu_config_validate(cfg));
    GLU_TRY(check_grid(g));
    GLU_TRY(check_mode(mode));
    if (r0 < 0 || r1 > g->lowH || r0 > r1) return einval("band: LR rows out of range");
    if (r0 == r1) return GLU_OK;
    // The band plus its h-row LR halo as a sub-image: its owned rows see the
    // same (unclipped) windows as in the full grid; stored indices are
    // rebased to the full grid (idxBase); the halo rows' outputs are scratch.
    const int h = cfg->windowSide / 2;
    const int ls = std::max(0, r0 - h), le = std::min(g->lowH, r1 + h);
    const int y0 = ls * g->scale, y1 = std::min(le * g->scale, g->highH);
    glu_grid sub = *g;
    sub.highH = y1 - y0;
    sub.lowH = le - ls;
    const size_t off = size_t(y0) * g->highW;
    SolveArgs a = solve_args(high + 3 * off, low + size_t(ls) * g->lowW * 3, &sub, cfg, mode);
    a.params = field + off;
    a.errOut = errors + off;
    a.idxBase = unsigned(ls) * unsigned(g->lowW);
    a.fallbacks = ctx->d_counters;
    GLU_CUDA(launch_solve(ctx, a), "solve_band");
    return GLU_OK;
}

int glu_cu_run_trials(glu_ctx* ctx, const float* high, float* low, glu_pixel_params* field,
                      float* errors, const glu_grid* g, const glu_config* cfg, int mode,
                      const uint32_t* off, const uint32_t* px, const uint32_t* ids, size_t n,
                      glu_trial_log* log, int* accepted, int* rejected) {
    if (!ctx) return einval("ctx must not be null");
    GLU_TRY(glu_config_validate(cfg));
    GLU_TRY(check_grid(g));
    GLU_TRY(check_mode(mode));
    int acc = 0, rej = 0;
    GLU_TRY(run_trials(ctx, high, low, field, errors, *g, *cfg, mode, off, px, ids, n, log, &acc,
                       &rej));
    if (accepted) *accepted = acc;
    if (rejected) *rejected = rej;
    return GLU_OK;
}

int glu_cu_apply_trial_log(glu_ctx* ctx, float* low, glu_pixel_params* field, float* errors,
                           const uint32_t* cells, size_t ncells, const uint32_t* pixels,
                           size_t npixels) {
    if (!ctx) return einval("ctx must not be null");
    return apply_trial_log(ctx, low, field, errors, cells, ncells, pixels, npixels);
}

int glu_cu_op_color(glu_ctx* ctx, const float* in, size_t n, const double* M,
                    const double* bias, double gammaExp, float* out) {
    if (!ctx) return einval("ctx must not be null");
    if (n == 0) return GLU_OK;
    GLU_CUDA(launch_op_color(ctx, in, n, M, bias, gammaExp, out), "op_color");
    return GLU_OK;
}

namespace {
// The reference's constructors' checks (simop.cpp:44-87).
int check_sim_operator(const glu_sim_operator* op) {
    if (!op) return einval("operator must not be null");
    if (op->kind < GLU_OP_IDENTITY || op->kind > GLU_OP_INVERT) return einval("unknown operator");
    if (op->kind == GLU_OP_GAIN && !(op->gain >= 0))
        return einval("scalar_gain_op: gain must be >= 0");
    if (op->kind == GLU_OP_GAMMA && !(op->gamma > 0))
        return einval("gamma_op: gamma must be > 0");
    return GLU_OK;
}
}  // namespace

int glu_cu_apply_operator(glu_ctx* ctx, const glu_sim_operator* op, const float* in, size_t n,
                          float* out) {
    if (!ctx) return einval("ctx must not be null");
    GLU_TRY(check_sim_operator(op));
    if (n == 0) return GLU_OK;
    GLU_CUDA(launch_apply_operator(ctx, *op, in, n, out), "apply_operator");
    return GLU_OK;
}

int glu_cu_apply_operator_field(glu_ctx* ctx, const glu_pixel_params* field, const glu_grid* g,
                                const glu_sim_operator* op, const float* lowIn, int clampOutput,
                                float* out) {
    if (!ctx) return einval("ctx must not be null");
    GLU_TRY(check_grid(g));
    GLU_TRY(check_sim_operator(op));
    if ((reinterpret_cast<uintptr_t>(field) | reinterpret_cast<uintptr_t>(out)) % 16 != 0)
        return einval("apply_operator_field: field and out must be 16-byte aligned");
    GLU_CUDA(launch_apply_operator_field(ctx, field, npx_of(g), *op, lowIn, lown_of(g),
                                         clampOutput, out),
             "apply_operator_field");
    return GLU_OK;
}

int glu_cu_apply_operator_field_band(glu_ctx* ctx, const glu_pixel_params* bandField,
                                     size_t bandPixels, const glu_grid* g,
                                     const glu_sim_operator* op, const float* lowIn,
                                     int clampOutput, float* out) {
    if (!ctx) return einval("ctx must not be null");
    GLU_TRY(check_grid(g));
    GLU_TRY(check_sim_operator(op));
    if (bandPixels > npx_of(g)) return einval("apply_field: band exceeds the grid");
    if ((reinterpret_cast<uintptr_t>(bandField) | reinterpret_cast<uintptr_t>(out)) % 16 != 0)
        return einval("apply_operator_field: field and out must be 16-byte aligned");
    if (bandPixels == 0) return GLU_OK;
    GLU_CUDA(launch_apply_operator_field(ctx, bandField, bandPixels, *op, lowIn, lown_of(g),
                                         clampOutput, out),
             "apply_operator_field");
    return GLU_OK;
}

int glu_cu_op_matte(glu_ctx* ctx, const float* in, size_t n, float* out) {
    if (!ctx) return einval("ctx must not be null");
    if (n == 0) return GLU_OK;
    GLU_CUDA(launch_op_matte(ctx, in, n, out), "op_matte");
    return GLU_OK;
}

int glu_cu_optimize_pixel_batch(glu_ctx* ctx, const float* ip, const uint32_t* offsets,
                                const uint32_t* candIdx, const float* candRgb, size_t count,
                                double eps, int mode, glu_pixel_params* out) {
    if (!ctx) return einval("ctx must not be null");
    GLU_TRY(check_mode(mode));
    GLU_CUDA(launch_pixel_batch(ctx, ip, offsets, candIdx, candRgb, count, eps, mode, out),
             "optimize_pixel");
    return GLU_OK;
}

int glu_cu_pair_eval(glu_ctx* ctx, const float* ip, const float* ia, const float* ib,
                     const double* w, size_t count, double eps, double* we, double* wf,
                     double* obj) {
    if (!ctx) return einval("ctx must not be null");
    GLU_CUDA(launch_pair_eval(ctx, ip, ia, ib, w, count, eps, we, wf, obj), "pair_eval");
    return GLU_OK;
}

// ---- host entry points ----------------------------------------------------------

int glu_h_grid_downsample(glu_ctx* ctx, const float* high, const glu_grid* g, float* low) {
    if (!ctx) return einval("ctx must not be null");
    GLU_TRY(check_grid(g));
    float* dh = dev<float>(ctx, S_HIGH, npx_of(g) * 3);
    float* dl = dev<float>(ctx, S_LOW, lown_of(g) * 3);
    if (!dh || !dl) return GLU_ENOMEM;
    GLU_TRY(h2d(ctx, dh, high, npx_of(g) * 12));
    GLU_TRY(glu_cu_grid_downsample(ctx, dh, g, dl));
    return d2h_sync(ctx, low, dl, lown_of(g) * 12);
}

int glu_h_optimize_field(glu_ctx* ctx, const float* high, const float* low, const glu_grid* g,
                         const glu_config* cfg, int mode, glu_pixel_params* out) {
    if (!ctx) return einval("ctx must not be null");
    GLU_TRY(glu_config_validate(cfg));
    GLU_TRY(check_grid(g));
    float* dh = dev<float>(ctx, S_HIGH, npx_of(g) * 3);
    float* dl = dev<float>(ctx, S_LOW, lown_of(g) * 3);
    glu_pixel_params* dp = dev<glu_pixel_params>(ctx, S_PARAMS, npx_of(g));
    if (!dh || !dl || !dp) return GLU_ENOMEM;
    GLU_TRY(h2d(ctx, dh, high, npx_of(g) * 12));
    GLU_TRY(h2d(ctx, dl, low, lown_of(g) * 12));
    GLU_TRY(glu_cu_optimize_field(ctx, dh, dl, g, cfg, mode, dp));
    return d2h_sync(ctx, out, dp, npx_of(g) * sizeof(glu_pixel_params));
}

int glu_h_optimize_pixels(glu_ctx* ctx, const float* high, const float* low, const glu_grid* g,
                          const glu_config* cfg, int mode, const uint32_t* pixels, size_t count,
                          glu_pixel_params* field) {
    if (!ctx) return einval("ctx must not be null");
    GLU_TRY(glu_config_validate(cfg));
    GLU_TRY(check_grid(g));
    for (size_t i = 0; i < count; ++i)
        if (pixels[i] >= npx_of(g)) return einval("optimize_pixels: pixel index out of range");
    if (count == 0) return GLU_OK;
    float* dh = dev<float>(ctx, S_HIGH, npx_of(g) * 3);
    float* dl = dev<float>(ctx, S_LOW, lown_of(g) * 3);
    glu_pixel_params* dp = dev<glu_pixel_params>(ctx, S_PARAMS, npx_of(g));
    uint32_t* dx = dev<uint32_t>(ctx, S_PIX, count);
    if (!dh || !dl || !dp || !dx) return GLU_ENOMEM;
    GLU_TRY(h2d(ctx, dh, high, npx_of(g) * 12));
    GLU_TRY(h2d(ctx, dl, low, lown_of(g) * 12));
    GLU_TRY(h2d(ctx, dp, field, npx_of(g) * sizeof(glu_pixel_params)));
    GLU_TRY(h2d(ctx, dx, pixels, count * 4));
    GLU_TRY(glu_cu_optimize_pixels(ctx, dh, dl, g, cfg, mode, dx, count, dp));
    return d2h_sync(ctx, field, dp, npx_of(g) * sizeof(glu_pixel_params));
}

int glu_h_apply_field(glu_ctx* ctx, const glu_pixel_params* field, const glu_grid* g,
                      const float* lowTarget, int channels, int clampOutput, float* out) {
    if (!ctx) return einval("ctx must not be null");
    GLU_TRY(check_grid(g));
    if (channels != 1 && channels != 3) return einval("apply_field: channels must be 1 or 3");
    glu_pixel_params* dp = dev<glu_pixel_params>(ctx, S_PARAMS, npx_of(g));
    float* dl = dev<float>(ctx, S_LOW, lown_of(g) * channels);
    float* dout = dev<float>(ctx, S_OUT, npx_of(g) * channels);
    if (!dp || !dl || !dout) return GLU_ENOMEM;
    GLU_TRY(h2d(ctx, dp, field, npx_of(g) * sizeof(glu_pixel_params)));
    GLU_TRY(h2d(ctx, dl, lowTarget, lown_of(g) * channels * 4));
    GLU_TRY(glu_cu_apply_field(ctx, dp, g, dl, channels, clampOutput, dout));
    return d2h_sync(ctx, out, dout, npx_of(g) * channels * 4);
}

int glu_h_error_map(glu_ctx* ctx, const float* high, const float* recon, size_t n,
                    float* errors) {
    if (!ctx) return einval("ctx must not be null");
    if (n == 0) return GLU_OK;
    float* dh = dev<float>(ctx, S_HIGH, n * 3);
    float* dr = dev<float>(ctx, S_OUT, n * 3);
    float* de = dev<float>(ctx, S_ERR, n);
    if (!dh || !dr || !de) return GLU_ENOMEM;
    GLU_TRY(h2d(ctx, dh, high, n * 12));
    GLU_TRY(h2d(ctx, dr, recon, n * 12));
    GLU_TRY(glu_cu_error_map(ctx, dh, dr, n, de));
    return d2h_sync(ctx, errors, de, n * 4);
}

int glu_h_solve_apply(glu_ctx* ctx, const float* high, const float* low, const glu_grid* g,
                      const glu_config* cfg, int mode, const float* lowTarget, int channels,
                      int clampOutput, float* out, glu_pixel_params* paramsOut) {
    if (!ctx) return einval("ctx must not be null");
    GLU_TRY(glu_config_validate(cfg));
    GLU_TRY(check_grid(g));
    if (channels != 1 && channels != 3) return einval("apply_field: channels must be 1 or 3");
    float* dh = dev<float>(ctx, S_HIGH, npx_of(g) * 3);
    float* dl = dev<float>(ctx, S_LOW, lown_of(g) * 3);
    float* dt = dev<float>(ctx, S_AUX, lown_of(g) * channels);
    float* dout = dev<float>(ctx, S_OUT, npx_of(g) * channels);
    glu_pixel_params* dp =
        paramsOut ? dev<glu_pixel_params>(ctx, S_PARAMS, npx_of(g)) : nullptr;
    if (!dh || !dl || !dt || !dout || (paramsOut && !dp)) return GLU_ENOMEM;
    GLU_TRY(h2d(ctx, dh, high, npx_of(g) * 12));
    GLU_TRY(h2d(ctx, dl, low, lown_of(g) * 12));
    GLU_TRY(h2d(ctx, dt, lowTarget, lown_of(g) * channels * 4));
    GLU_TRY(glu_cu_solve_apply(ctx, dh, dl, g, cfg, mode, dt, channels, clampOutput, dout, dp));
    if (paramsOut)
        GLU_CUDA(cudaMemcpyAsync(paramsOut, dp, npx_of(g) * sizeof(glu_pixel_params),
                                 cudaMemcpyDeviceToHost, ctx->stream),
                 "copy to host");
    return d2h_sync(ctx, out, dout, npx_of(g) * channels * 4);
}

int glu_h_find_large_error(glu_ctx* ctx, const float* errors, int width, int height,
                           float threshold, uint8_t* mask, uint32_t* compOffsets,
                           uint32_t* compPixels, size_t* count) {
    if (!ctx) return einval("ctx must not be null");
    if (width <= 0 || height <= 0) return einval("find_large_error: empty error map");
    const size_t n = size_t(width) * height;
    float* de = dev<float>(ctx, S_ERR, n);
    uint8_t* dm = dev<uint8_t>(ctx, S_AUX, n);
    if (!de || !dm) return GLU_ENOMEM;
    GLU_TRY(h2d(ctx, de, errors, n * 4));
    size_t nc = 0;
    const uint32_t* off = nullptr;
    const uint32_t* px = nullptr;
    GLU_TRY(ccl_find_large_error(ctx, de, width, height, threshold, dm, nullptr, &nc, &off, &px));
    if (mask) GLU_CUDA(cudaMemcpyAsync(mask, dm, n, cudaMemcpyDeviceToHost, ctx->stream), "copy");
    GLU_CUDA(cudaMemcpyAsync(compOffsets, off, (nc + 1) * 4, cudaMemcpyDeviceToHost, ctx->stream),
             "copy");
    GLU_CUDA(cudaStreamSynchronize(ctx->stream), "synchronize");
    if (nc == 0) compOffsets[0] = 0;
    const size_t total = compOffsets[nc];
    if (total) GLU_TRY(d2h_sync(ctx, compPixels, px, total * 4));
    if (count) *count = nc;
    return GLU_OK;
}

int glu_h_trial_update_component(glu_ctx* ctx, const float* high, float* low,
                                 glu_pixel_params* field, float* errors, const glu_grid* g,
                                 const glu_config* cfg, int mode, const uint32_t* component,
                                 size_t count, int* accepted) {
    if (!ctx) return einval("ctx must not be null");
    GLU_TRY(glu_config_validate(cfg));
    if (count == 0) return einval("trial_update_component: empty component");
    GLU_TRY(check_grid(g));
    for (size_t i = 0; i < count; ++i)
        if (component[i] >= npx_of(g))
            return einval("trial_update_component: pixel index out of range");
    const size_t n = npx_of(g);
    float* dh = dev<float>(ctx, S_HIGH, n * 3);
    float* dl = dev<float>(ctx, S_LOW, lown_of(g) * 3);
    glu_pixel_params* dp = dev<glu_pixel_params>(ctx, S_PARAMS, n);
    float* de = dev<float>(ctx, S_ERR, n);
    uint32_t* dc = dev<uint32_t>(ctx, S_PIX, count);
    if (!dh || !dl || !dp || !de || !dc) return GLU_ENOMEM;
    GLU_TRY(h2d(ctx, dh, high, n * 12));
    GLU_TRY(h2d(ctx, dl, low, lown_of(g) * 12));
    GLU_TRY(h2d(ctx, dp, field, n * sizeof(glu_pixel_params)));
    GLU_TRY(h2d(ctx, de, errors, n * 4));
    GLU_TRY(h2d(ctx, dc, component, count * 4));
    GLU_TRY(glu_cu_trial_update_component(ctx, dh, dl, dp, de, g, cfg, mode, dc, count,
                                          accepted));
    GLU_CUDA(cudaMemcpyAsync(low, dl, lown_of(g) * 12, cudaMemcpyDeviceToHost, ctx->stream),
             "copy");
    GLU_CUDA(cudaMemcpyAsync(field, dp, n * sizeof(glu_pixel_params), cudaMemcpyDeviceToHost,
                             ctx->stream),
             "copy");
    return d2h_sync(ctx, errors, de, n * 4);
}

int glu_h_joint_optimize(glu_ctx* ctx, const float* high, const glu_grid* g,
                         const glu_config* cfg, int mode, float* low, glu_pixel_params* field,
                         float* errors, glu_joint_stats* stats) {
    if (!ctx) return einval("ctx must not be null");
    GLU_TRY(glu_config_validate(cfg));
    GLU_TRY(check_grid(g));
    const size_t n = npx_of(g);
    float* dh = dev<float>(ctx, S_HIGH, n * 3);
    float* dl = dev<float>(ctx, S_LOW, lown_of(g) * 3);
    glu_pixel_params* dp = dev<glu_pixel_params>(ctx, S_PARAMS, n);
    float* de = dev<float>(ctx, S_ERR, n);
    if (!dh || !dl || !dp || !de) return GLU_ENOMEM;
    GLU_TRY(h2d(ctx, dh, high, n * 12));
    GLU_TRY(glu_cu_joint_optimize(ctx, dh, g, cfg, mode, dl, dp, de, stats));
    GLU_CUDA(cudaMemcpyAsync(low, dl, lown_of(g) * 12, cudaMemcpyDeviceToHost, ctx->stream),
             "copy");
    GLU_CUDA(cudaMemcpyAsync(field, dp, n * sizeof(glu_pixel_params), cudaMemcpyDeviceToHost,
                             ctx->stream),
             "copy");
    return d2h_sync(ctx, errors, de, n * 4);
}

int glu_h_optimize_pixel_batch(glu_ctx* ctx, const float* ip, const uint32_t* offsets,
                               const uint32_t* candIdx, const float* candRgb, size_t count,
                               double eps, int mode, glu_pixel_params* out) {
    if (!ctx) return einval("ctx must not be null");
    GLU_TRY(check_mode(mode));
    for (size_t k = 0; k < count; ++k)
        if (offsets[k + 1] <= offsets[k]) return einval("candidate list must not be empty");
    if (count == 0) return GLU_OK;
    const size_t nc = offsets[count];
    // one slot, carved: ip | offsets | idx | rgb | out
    const size_t bytes = count * 12 + (count + 1) * 4 + nc * 4 + nc * 12 + count * 12 + 64;
    char* base = static_cast<char*>(scratch(ctx, S_SPARE1, bytes));
    if (!base) return GLU_ENOMEM;
    float* dip = reinterpret_cast<float*>(base);
    uint32_t* doff = reinterpret_cast<uint32_t*>(base + count * 12);
    uint32_t* didx = doff + count + 1;
    float* drgb = reinterpret_cast<float*>(didx + nc);
    glu_pixel_params* dout = reinterpret_cast<glu_pixel_params*>(drgb + nc * 3);
    GLU_TRY(h2d(ctx, dip, ip, count * 12));
    GLU_TRY(h2d(ctx, doff, offsets, (count + 1) * 4));
    GLU_TRY(h2d(ctx, didx, candIdx, nc * 4));
    GLU_TRY(h2d(ctx, drgb, candRgb, nc * 12));
    GLU_TRY(glu_cu_optimize_pixel_batch(ctx, dip, doff, didx, drgb, count, eps, mode, dout));
    return d2h_sync(ctx, out, dout, count * sizeof(glu_pixel_params));
}

int glu_h_pair_eval(glu_ctx* ctx, const float* ip, const float* ia, const float* ib,
                    const double* w, size_t count, double eps, double* we, double* wf,
                    double* obj) {
    if (!ctx) return einval("ctx must not be null");
    if (count == 0) return GLU_OK;
    const size_t bytes = count * (12 * 3 + 8 * 4) + 64;
    char* base = static_cast<char*>(scratch(ctx, S_SPARE2, bytes));
    if (!base) return GLU_ENOMEM;
    float* dp = reinterpret_cast<float*>(base);
    float* da = dp + 3 * count;
    float* db = da + 3 * count;
    double* dw = reinterpret_cast<double*>(base + count * 36 + 8 - (count * 36) % 8);
    double* dwe = dw + count;
    double* dwf = dwe + count;
    double* dob = dwf + count;
    GLU_TRY(h2d(ctx, dp, ip, count * 12));
    GLU_TRY(h2d(ctx, da, ia, count * 12));
    GLU_TRY(h2d(ctx, db, ib, count * 12));
    if (w) GLU_TRY(h2d(ctx, dw, w, count * 8));
    GLU_TRY(glu_cu_pair_eval(ctx, dp, da, db, w ? dw : nullptr, count, eps, dwe, dwf, dob));
    if (we) GLU_CUDA(cudaMemcpyAsync(we, dwe, count * 8, cudaMemcpyDeviceToHost, ctx->stream),
                     "copy");
    if (wf) GLU_CUDA(cudaMemcpyAsync(wf, dwf, count * 8, cudaMemcpyDeviceToHost, ctx->stream),
                     "copy");
    return d2h_sync(ctx, obj, dob, obj ? count * 8 : 0);
}

}  // extern "C"
