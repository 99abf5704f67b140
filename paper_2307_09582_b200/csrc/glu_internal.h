// glu_internal.h -- shared declarations of the CUDA implementation.
#pragma once

#include <cuda_runtime.h>

#include <string>

#include "glu_cuda.h"

// Bounds / invariant checks of the device code, compiled in with
// -DGLU_DEBUG_CHECKS (tools/debug_checks.sh): a failed check prints where and
// traps, so the test that ran it fails loudly.  (compute-sanitizer is not
// available on the GPU pool; this build stands in for its memcheck.)
#ifdef GLU_DEBUG_CHECKS
#include <cstdio>
#define GLU_DCHECK(cond)                                                                     \
    do {                                                                                     \
        if (!(cond)) {                                                                       \
            printf("GLU_DCHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__,    \
                   __LINE__, int(blockIdx.x), int(threadIdx.x));                             \
            __trap();                                                                        \
        }                                                                                    \
    } while (0)
#else
#define GLU_DCHECK(cond) \
    do {                 \
    } while (0)
#endif

struct glu_ctx {
    int device = 0;
    cudaStream_t own = nullptr;
    cudaStream_t stream = nullptr;
    unsigned long long launches = 0;
    unsigned long long* d_counters = nullptr;  // [0] = fp64 fallback pixels
    // Pinned host words for the joint loop's small read-backs (component
    // counts, sweep verdicts): a device-to-host copy into pageable memory is
    // staged by the driver and costs several microseconds more per sync.
    uint32_t* h_rb = nullptr;  // 16 words
    // Grow-only scratch slots (device memory).
    static constexpr int kSlots = 24;
    void* buf[kSlots] = {};
    size_t cap[kSlots] = {};
    // Grow-only pinned host slots.
    void* hbuf[4] = {};
    size_t hcap[4] = {};
    // GLU_OPT_SOLVER: 0 auto, 1 fp64 reference-order kernel only, 2 fp32
    // filter with every pixel forced through the fp64 verify path (testing).
    int solver = 0;
    // GLU_OPT_TRIALS: 0 speculative parallel schedule, 1 one CTA in order,
    // 2 dependency-counting dataflow schedule (literal scope always uses 2).
    int trials = 0;
    // Copy streams + events of the host frame pipeline (created lazily).
    cudaStream_t h2d = nullptr, d2h = nullptr;
    cudaEvent_t ev[8] = {};
    // Side stream + events of the device frame pipeline (created lazily):
    // frame k + 1's preparation overlaps frame k's solve.
    cudaStream_t side = nullptr;
    cudaEvent_t pev[5] = {};
    // Recorded on the previous stream when glu_ctx_set_stream switches
    // streams: the new stream waits on it, so work issued on different
    // streams never overlaps on the shared scratch slots / counters.
    cudaEvent_t switchEv = nullptr;
};

namespace glu_cu {

// Scratch slot ids.
enum Slot {
    S_HIGH = 0, S_LOW, S_PARAMS, S_OUT, S_ERR, S_AUX, S_PIX,
    S_CCL_LABEL, S_CCL_LIST, S_CCL_OFF, S_CCL_MISC, S_TRIAL, S_TRIAL2, S_TRIAL3,
    S_SPARE1, S_SPARE2, S_PACKED, S_SCHED, S_SCHED_META, S_PARK, S_PARK_TMP, S_TARGET4
};

void set_error(const std::string& msg);
int fail_cuda(cudaError_t e, const char* where);
void* scratch(glu_ctx* ctx, int slot, size_t bytes);  // nullptr on OOM (error set)

struct SolveArgs {
    const float* high;
    const float* low;
    int W, H, s, lw, lh, S;
    double eps;
    int mode;
    glu_pixel_params* params;  // may be null when fused with apply
    const float* lowT;         // apply target (null: no apply)
    int channels;
    int clamp;
    float* out;
    unsigned long long* fallbacks;
    unsigned sdiv;  // ceil(2^32 / s) when W, H < 2^16 (x / s = umulhi(x, sdiv)), else 0
    float epsf;     // (float)eps for the fp32 filter
    float* errOut;  // optional: self reconstruction error per pixel (k_self_error fused)
    // Added to the stored LR indices: a row band solved as a sub-image whose
    // LR rows start at global row r (idxBase = r * lowW of the full grid).
    unsigned idxBase;
};

// Launchers (return cudaError_t of the launch).
cudaError_t launch_grid_downsample(glu_ctx* ctx, const float* high, int W, int H, int s,
                                   int lw, int lh, float* low);
cudaError_t launch_solve(glu_ctx* ctx, const SolveArgs& a);
// glu_solve32.cu: fp32 filter + fp64 verify (Fast / GNU, S in {3, 5}; Exact
// S = 3, s >= 3 via glu_solve32x.cu).
bool solve32_supported(int mode, int S, int s);
cudaError_t launch_solve32(glu_ctx* ctx, const SolveArgs& a, int forceFallback);
// One frame of the video path: grid_downsample of a.high into `low`, optional
// 1-ch matte of it into `matte`, and the LR packing in one kernel, then the
// solve (a.lowT must already point at `low` or `matte`).
cudaError_t launch_frame_solve32(glu_ctx* ctx, const SolveArgs& a, float* low, float* matte,
                                 int forceFallback);
// The same split in two, for the multi-frame pipeline: k_frame_prep into the
// given buffers on stream `st`, then the solve on ctx->stream.
cudaError_t launch_frame_prep(glu_ctx* ctx, cudaStream_t st, const SolveArgs& a, float* low,
                              float* matte, float4* packed, unsigned* nanFlag);
cudaError_t launch_prepped_solve32(glu_ctx* ctx, const SolveArgs& a, const float4* packed,
                                   int forceFallback, const unsigned* nanFlag);
// A batch of video frames in ONE solve launch (glu_cu_upsample_frames, 1-ch
// matte target): frame f = blockIdx.z reads the guide at high + f * high,
// its packed LR at packed + f * packed, its NaN flag at nanFlag[f] and its
// target at lowT + f * lowT, and writes out + f * px.  frames = 1: one frame.
struct FrameBatch {
    int frames = 1;
    size_t high = 0, px = 0, lowT = 0, packed = 0;
};
// glu_solve32f.cu: Fast, S = 3 (tile-staged, keyed closed-form stage B).
bool solve32f_supported(int mode, int S);
cudaError_t launch_solve32f(glu_ctx* ctx, const SolveArgs& a, const float4* packed,
                            int forceFallback, const unsigned* nanFlag,
                            const FrameBatch& fb = FrameBatch{});
// k_frame_prep for fb.frames frames in one launch (frame f: the guide at
// a.high + f * fb.high; low / matte / packed / flag at their bases + f * the
// set stride `set` bytes), on stream st.
cudaError_t launch_frame_prep_batch(glu_ctx* ctx, cudaStream_t st, const SolveArgs& a,
                                    const FrameBatch& fb, char* base, size_t set,
                                    size_t offMatte, size_t offPacked, unsigned* flags);
// The batch's solve (k_solve32f over fb.frames frames; a = frame 0's args).
// (Fast / GNU: k_solve32f; Exact: k_solve32x)
cudaError_t launch_prepped_solve32f_batch(glu_ctx* ctx, const SolveArgs& a, const float4* packed,
                                          int forceFallback, const unsigned* flags,
                                          const FrameBatch& fb);
bool solve32x_supported(int mode, int S, int s);
cudaError_t launch_solve32x(glu_ctx* ctx, const SolveArgs& a, const float4* packed,
                            int forceFallback, const unsigned* nanFlag,
                            const FrameBatch& fb = FrameBatch{});
cudaError_t launch_solve_list(glu_ctx* ctx, const SolveArgs& a, const uint32_t* pixels,
                              size_t count);
cudaError_t launch_apply(glu_ctx* ctx, const glu_pixel_params* field, size_t npx,
                         const float* lowT, size_t lowN, int channels, int clamp, float* out);
cudaError_t launch_error_map(glu_ctx* ctx, const float* high, const float* recon, size_t npx,
                             float* e);
cudaError_t launch_self_error(glu_ctx* ctx, const float* high, const glu_pixel_params* field,
                              size_t npx, const float* low, float* e);
cudaError_t launch_op_color(glu_ctx* ctx, const float* in, size_t n, const double* M,
                            const double* bias, double gammaExp, float* out);
cudaError_t launch_op_matte(glu_ctx* ctx, const float* in, size_t n, float* out);
cudaError_t launch_apply_operator(glu_ctx* ctx, const glu_sim_operator& op, const float* in,
                                  size_t n, float* out);
// k_op_pack_target4 + k_apply3v (field and out 16-byte aligned).
cudaError_t launch_apply_operator_field(glu_ctx* ctx, const glu_pixel_params* field, size_t npx,
                                        const glu_sim_operator& op, const float* lowIn,
                                        size_t lowN, int clamp, float* out);
cudaError_t launch_ffma_probe(glu_ctx* ctx, float* sink, int iters, int blocks, int threads);
cudaError_t launch_pixel_batch(glu_ctx* ctx, const float* ip, const uint32_t* offsets,
                               const uint32_t* candIdx, const float* candRgb, size_t count,
                               double eps, int mode, glu_pixel_params* out);
cudaError_t launch_pair_eval(glu_ctx* ctx, const float* ip, const float* ia, const float* ib,
                             const double* w, size_t count, double eps, double* we,
                             double* wf, double* obj);

// Joint optimisation (glu_joint.cu).
int ccl_find_large_error(glu_ctx* ctx, const float* errors, int W, int H, float thr,
                         uint8_t* mask, uint32_t* label, size_t* count,
                         const uint32_t** off, const uint32_t** px);
int trial_one(glu_ctx* ctx, const float* high, float* low, glu_pixel_params* field,
              float* errors, const glu_grid& g, const glu_config& cfg, int mode,
              const uint32_t* comp, size_t n, int* accepted);
int component_boxes(glu_ctx* ctx, const uint32_t* off, const uint32_t* px, size_t n,
                    const glu_grid& g, int32_t* boxes);
int run_trials(glu_ctx* ctx, const float* high, float* low, glu_pixel_params* field,
               float* errors, const glu_grid& g, const glu_config& cfg, int mode,
               const uint32_t* off, const uint32_t* px, const uint32_t* ids, size_t n,
               glu_trial_log* log, int* accepted, int* rejected);
int apply_trial_log(glu_ctx* ctx, float* low, glu_pixel_params* field, float* errors,
                    const uint32_t* cells, size_t ncells, const uint32_t* pixels,
                    size_t npixels);
int joint_sweep(glu_ctx* ctx, const float* high, float* low, glu_pixel_params* field,
                float* errors, const glu_grid& g, const glu_config& cfg, int mode,
                const uint32_t* off, const uint32_t* px, size_t ncomp, int* accepted,
                int* rejected);

}  // namespace glu_cu
