/*
 * glu_cuda.h -- C-ABI of the B200 (sm_100a) Guided Linear Upsampling hot path.
 *
 * The reference exposes this path only as the C++ API in
 * /root/reference/proj/include/glu/{grid,params,upsample,jointopt}.hpp (there
 * is no plugin registry or FFI).  This header is the thin, torch-free C
 * boundary underneath the drop-in C++ API (include/glu/ headers, implemented in
 * paper_2307_09582_b200/csrc/glu_api.cpp): plain pointers and sizes, status
 * codes, a per-device context.  Each entry point names the reference function
 * it replaces.
 *
 * Buffer layouts are byte-identical to the reference containers:
 *   image   : row-major, interleaved RGB float32, 12 B/pixel (image.hpp:13-23)
 *   params  : row-major glu_pixel_params {u32 a, u32 b, f32 w}, 12 B (params.hpp:42-46)
 *   errors  : row-major float32 (params.hpp:57-69)
 * A single-channel target/output (1 float per pixel) is an extension
 * (channels = 1) that the C++ API does not expose.
 *
 * Two families of entry points:
 *   glu_cu_*  device pointers, asynchronous on the context's stream;
 *   glu_h_*   host pointers (what the C++ API calls): copies in, runs, copies
 *             out and synchronises.
 *
 * Status codes: GLU_OK, GLU_EINVAL (message = the reference's
 * std::invalid_argument text), GLU_ECUDA, GLU_ENOMEM; glu_last_error() returns
 * the thread's last message.  Every call is reentrant per context; contexts
 * are not shared between host threads without external locking.
 */
#ifndef GLU_CUDA_H
#define GLU_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GLU_CUDA_ABI_VERSION 1

enum glu_status { GLU_OK = 0, GLU_EINVAL = 1, GLU_ECUDA = 2, GLU_ENOMEM = 3, GLU_EFORMAT = 4 };
/* glu::Mode (params.hpp:11-15) */
enum glu_mode { GLU_MODE_FAST = 0, GLU_MODE_EXACT = 1, GLU_MODE_GNU = 2 };

/* glu::PixelParams (params.hpp:42-46) */
typedef struct glu_pixel_params {
    uint32_t a;
    uint32_t b;
    float w;
} glu_pixel_params;

/* glu::GridSpec (grid.hpp:19-39) */
typedef struct glu_grid {
    int scale;
    int highW, highH;
    int lowW, lowH;
    int sampleOffset;
} glu_grid;

/* glu::GluConfig (params.hpp:20-39) */
typedef struct glu_config {
    int windowSide;
    float errorThreshold;
    int maxIterations;
    float epsilon;
    int literalComponentUpdate;
} glu_config;

/* Per-trial-phase statistics of glu_*_joint_optimize (glu::JointResult counters). */
typedef struct glu_joint_stats {
    int iterations;
    int trialsAccepted;
    int trialsRejected;
    int components; /* total components visited over all sweeps */
} glu_joint_stats;

typedef struct glu_ctx glu_ctx;

int glu_abi_version(void);
const char* glu_last_error(void);
const char* glu_build_info(void);

/* GridSpec::create (grid.cpp:8-23); validation messages as the reference. */
int glu_grid_create(int highW, int highH, int scale, glu_grid* out);
/* GluConfig::validate (params.hpp:30-38). */
int glu_config_validate(const glu_config* cfg);
/* GluConfig{} defaults: S=3, tau=30/255, N=3, eps=1e-3, literal=false. */
glu_config glu_config_default(void);

/* The calling thread's current CUDA device (cudaGetDevice). */
int glu_current_device(int* device);

/* Context: owns a CUDA stream on `device` and grow-only scratch buffers. */
int glu_ctx_create(int device, glu_ctx** out);
int glu_ctx_destroy(glu_ctx* ctx);
/* Use an external cudaStream_t (NULL = the context's own stream). */
int glu_ctx_set_stream(glu_ctx* ctx, void* cuda_stream);
void* glu_ctx_stream(glu_ctx* ctx);
int glu_ctx_synchronize(glu_ctx* ctx);
/* Context options.  GLU_OPT_SOLVER selects the solve kernel:
 *   0 (default) fp32 filter + fp64 verify where supported (Fast/GNU, S 3 or 5),
 *     the fp64 reference-order kernel otherwise;
 *   1 the fp64 reference-order kernel everywhere;
 *   2 fp32 filter with every pixel forced through the fp64 verify (testing).
 * GLU_OPT_TRIALS selects the joint-loop trial schedule:
 *   0 (default) speculative parallel schedule over all SMs (trials start at
 *     once, commit in conflict order, re-run if an overlapping earlier trial
 *     was accepted meanwhile);
 *   1 one CTA runs the trials in sweep order;
 *   2 dependency-counting dataflow schedule over all SMs.
 * All settings produce bit-identical results. */
enum glu_option { GLU_OPT_SOLVER = 1, GLU_OPT_TRIALS = 2 };
int glu_ctx_set_option(glu_ctx* ctx, int option, int value);
/* Number of kernels this context has launched (bench.py's gpu_launches). */
unsigned long long glu_ctx_launch_count(glu_ctx* ctx);
/* Pixels this context's solves re-evaluated on the exact fp64 path
 * (cumulative). */
unsigned long long glu_ctx_fallback_count(glu_ctx* ctx);
/* Pixels whose fp32 near-tie was settled in double over the close set only
 * (cumulative; diagnostics for the fp32 filter). */
unsigned long long glu_ctx_close_set_count(glu_ctx* ctx);

/* ---- device-pointer entry points (async on the context stream) ---------- */

/* Device-to-device copy on the context stream (e.g. out of the context-owned
 * component buffers of glu_cu_find_large_error). */
int glu_cu_copy(glu_ctx* ctx, void* dst, const void* src, size_t bytes);
/* Device memory for C/C++ callers without their own allocator; upload /
 * download are synchronous host <-> device copies on the context stream. */
int glu_cu_alloc(glu_ctx* ctx, void** ptr, size_t bytes);
int glu_cu_free(glu_ctx* ctx, void* ptr);
int glu_cu_upload(glu_ctx* ctx, void* dst, const void* hostSrc, size_t bytes);
int glu_cu_download(glu_ctx* ctx, void* hostDst, const void* src, size_t bytes);

/* grid_downsample (grid.cpp:41-52). low: lowW*lowH*3 floats. */
int glu_cu_grid_downsample(glu_ctx* ctx, const float* high, const glu_grid* grid, float* low);

/* optimize_field (upsample.cpp:194-216). */
int glu_cu_optimize_field(glu_ctx* ctx, const float* high, const float* low,
                          const glu_grid* grid, const glu_config* cfg, int mode,
                          glu_pixel_params* out);

/* optimize_pixels (upsample.cpp:218-233): listed linear indices, in place.
 * Duplicate indices resolve to the same value, so list order is immaterial. */
int glu_cu_optimize_pixels(glu_ctx* ctx, const float* high, const float* low,
                           const glu_grid* grid, const glu_config* cfg, int mode,
                           const uint32_t* pixels, size_t count, glu_pixel_params* field);

/* apply_field + reconstruct_pixel (upsample.cpp:235-252, upsample.hpp:54-65).
 * lowTarget/out have `channels` (1 or 3) floats per pixel. */
int glu_cu_apply_field(glu_ctx* ctx, const glu_pixel_params* field, const glu_grid* grid,
                       const float* lowTarget, int channels, int clampOutput, float* out);

/* apply_field over a contiguous range of HR pixels (a row band of the field;
 * multi-GPU C5): `bandField` / `out` hold `bandPixels`
 * consecutive raster pixels whose params index the whole grid's LR target. */
int glu_cu_apply_field_band(glu_ctx* ctx, const glu_pixel_params* bandField, size_t bandPixels,
                            const glu_grid* grid, const float* lowTarget, int channels,
                            int clampOutput, float* out);

/* error_map + pixel_error (upsample.cpp:254-267, upsample.hpp:67-74). */
int glu_cu_error_map(glu_ctx* ctx, const float* high, const float* recon, size_t pixelCount,
                     float* errors);

/* error_map(high, apply_field(field, low)) fused, without the HR image. */
int glu_cu_self_error_map(glu_ctx* ctx, const float* high, const glu_pixel_params* field,
                          const glu_grid* grid, const float* low, float* errors);

/* optimize_field then apply_field on lowTarget, fused in one kernel (no
 * parameter round trip through HBM).  paramsOut may be NULL. */
int glu_cu_solve_apply(glu_ctx* ctx, const float* high, const float* low,
                       const glu_grid* grid, const glu_config* cfg, int mode,
                       const float* lowTarget, int channels, int clampOutput, float* out,
                       glu_pixel_params* paramsOut);

/* find_large_error (jointopt.cpp:9-46).  mask: W*H bytes; label: W*H u32 =
 * the component's smallest pixel index, 0xffffffff outside the mask.
 * Components are returned in CSR form in device memory owned by the context
 * (valid until the next call): *compOffsets[0..*count], *compPixels.  Pass
 * NULL for outputs that are not needed.  *count is written on the host. */
int glu_cu_find_large_error(glu_ctx* ctx, const float* errors, int width, int height,
                            float threshold, uint8_t* mask, uint32_t* label, size_t* count,
                            const uint32_t** compOffsets, const uint32_t** compPixels);

/* trial_update_component (jointopt.cpp:114-180) for one component (device
 * pixel list, sorted ascending).  *accepted written on the host. */
int glu_cu_trial_update_component(glu_ctx* ctx, const float* high, float* low,
                                  glu_pixel_params* field, float* errors,
                                  const glu_grid* grid, const glu_config* cfg, int mode,
                                  const uint32_t* component, size_t count, int* accepted);

/* joint_optimize (jointopt.cpp:182-206).  low/field/errors are outputs. */
int glu_cu_joint_optimize(glu_ctx* ctx, const float* high, const glu_grid* grid,
                          const glu_config* cfg, int mode, float* low, glu_pixel_params* field,
                          float* errors, glu_joint_stats* stats);

/* LR target operators the frame pipeline can apply between downsample and
 * upsample (stand-ins for the black-box operator). */
enum glu_target_op { GLU_TARGET_IDENTITY = 0, GLU_TARGET_MATTE = 1 };

/* Frame pipeline (BASELINE.json configs[2]): for each of `count` HR frames
 * (count*W*H*3 floats): grid_downsample -> target = op(LR) -> fused
 * optimize_field + apply_field.  out: count*W*H*channels floats (channels = 1
 * for GLU_TARGET_MATTE, else 3); paramsOut (count*W*H records) may be NULL. */
int glu_cu_upsample_frames(glu_ctx* ctx, const float* frames, int count, const glu_grid* grid,
                           const glu_config* cfg, int mode, int targetOp, float* out,
                           glu_pixel_params* paramsOut);

/* FP32 roofline denominator: FFMA throughput of this device, measured with
 * CUDA events over a dependent-chain-free FFMA kernel (TFLOP/s, FFMA = 2). */
int glu_cu_fp32_peak(glu_ctx* ctx, double* tflops, double* sm_mhz_estimate);

/* Black-box operator stand-ins on LR images (harness
 * operators of BASELINE.json).  n = LR pixel count. */
/* out = clamp01(M * in + bias) per pixel, fp64 row-major M, bias may be NULL;
 * gammaExp > 0 applies clamp01(pow(in, gammaExp)) first (simop.cpp:33-36). */
int glu_cu_op_color(glu_ctx* ctx, const float* in, size_t n, const double* M3x3,
                    const double* bias3, double gammaExp, float* out);
/* 1-channel matte: out = 1 / (1 + exp(-10 (Y - 0.5))), Y = BT.601 luma. */
int glu_cu_op_matte(glu_ctx* ctx, const float* in, size_t n, float* out);

/* The reference's black-box operator stand-ins (glu::SimOperator,
 * simop.hpp:11-26): kind, gain (ScalarGain), gamma (Gamma), row-major 3x3
 * mix (ChannelMix).  Every output channel is clamp01 of the reference's
 * double expression (simop.cpp:16-41). */
enum glu_sim_kind { GLU_OP_IDENTITY = 0, GLU_OP_GAIN = 1, GLU_OP_MIX = 2, GLU_OP_GRAY = 3,
                    GLU_OP_GAMMA = 4, GLU_OP_INVERT = 5 };
typedef struct glu_sim_operator {
    int kind;
    double gain;
    double gamma;
    double mix[9];
} glu_sim_operator;
/* apply_operator (simop.cpp:120-132) on n RGB pixels (LR targets). */
int glu_cu_apply_operator(glu_ctx* ctx, const glu_sim_operator* op, const float* in, size_t n,
                          float* out);
/* The edit loop's "edit T-down, then upsample" in one pass over the HR field:
 * apply_field(field, apply_operator(op, lowIn), clampOutput) -- the operator
 * runs once per LR cell inside the target packing, the HR pass is the RGB
 * apply (out: W*H*3 floats). */
int glu_cu_apply_operator_field(glu_ctx* ctx, const glu_pixel_params* field, const glu_grid* grid,
                                const glu_sim_operator* op, const float* lowIn, int clampOutput,
                                float* out);
/* The same over a row band of the field (multi-GPU C5, as glu_cu_apply_field_band). */
int glu_cu_apply_operator_field_band(glu_ctx* ctx, const glu_pixel_params* bandField,
                                     size_t bandPixels, const glu_grid* grid,
                                     const glu_sim_operator* op, const float* lowIn,
                                     int clampOutput, float* out);

/* Batched per-pixel selection (optimize_pixel_{fast,exact,gnu},
 * upsample.cpp:178-192): instance k has pixel colour ip[3k..], counts[k]
 * candidates starting at offsets[k] in candIdx/candRgb. */
int glu_cu_optimize_pixel_batch(glu_ctx* ctx, const float* ip, const uint32_t* offsets,
                                const uint32_t* candIdx, const float* candRgb, size_t count,
                                double eps, int mode, glu_pixel_params* out);
/* Batched scalar helpers (weight_exact, weight_fast, pair_objective;
 * upsample.cpp:158-176).  Any output may be NULL. */
int glu_cu_pair_eval(glu_ctx* ctx, const float* ip, const float* ia, const float* ib,
                     const double* w, size_t count, double eps, double* weightExact,
                     double* weightFast, double* objective);

/* ---- distributed joint loop building blocks ---------- *
 * Every rank keeps the full LR / params / errors state (replicas) and finds
 * the same components (glu_cu_find_large_error).  glu_trial_levels groups
 * the components of a sweep into levels of mutually independent trials
 * (Chebyshev box distance > 2h to every earlier member of other levels it
 * depends on); each rank runs its share of a level with a change log, the
 * logs are exchanged (NCCL / gloo all-gather), and every rank applies the
 * others' logs.  The result is bit-identical to the sequential loop. */
typedef struct glu_trial_log {
    uint32_t* counts; /* device: [0] cells, [1] pixels, [2] overflow flag */
    uint32_t* cells;  /* device: 4 words per replaced cell {idx, r, g, b} (accepted trials) */
    uint32_t* pixels; /* device: 5 words per affected pixel {idx, a, b, w, e} */
    uint32_t cellCapacity, pixelCapacity;
} glu_trial_log;

/* ---- banded joint loop (SURVEY §8(e), C4 over HR row bands) -------------- *
 * A rank owns the LR rows [r0, r1) of the grid and the HR rows of their
 * footprints; paper_2307_09582_b200/bands.py runs the loop of
 * jointopt.cpp:182-206 over bands (downsample + solve per band, band CCL with a
 * seam merge, trials owned by the band of their first pixel in rounds, change
 * logs exchanged between rounds).  Buffers are full-size (global indices);
 * only the band (and its halo rows) is ever written or read. */
/* grid_downsample (grid.cpp:41-52) of the LR rows [r0, r1) into `low` (the full
 * LR buffer); reads only the HR rows of the band. */
int glu_cu_downsample_band(glu_ctx* ctx, const float* high, const glu_grid* grid, int r0, int r1,
                           float* low);
/* joint_optimize's initial optimize_field + self error map (jointopt.cpp:187-190)
 * for the LR rows [r0, r1): `low` must hold LR rows [r0 - h, r1 + h) (h = S / 2,
 * the solve's halo).  Writes field / errors for the band's HR rows; the rows of
 * the h LR rows around the band are used as scratch (refreshed by the caller's
 * halo exchange). */
int glu_cu_solve_band(glu_ctx* ctx, const float* high, const float* low, const glu_grid* grid,
                      const glu_config* cfg, int mode, int r0, int r1, glu_pixel_params* field,
                      float* errors);
/* Host: the round of each component of a sweep for a banded schedule: owners[i]
 * = the rank running trial i; round(i) = max over earlier components j within
 * Chebyshev `reach` of i of round(j) (same owner) or round(j) + 1 (other owner). */
int glu_trial_rounds(const int32_t* boxes, size_t count, int reach, const int32_t* owners,
                     int32_t* rounds);

/* Cell bounding boxes {x0, y0, x1, y1} of components (device, 4 int32 each). */
int glu_cu_component_boxes(glu_ctx* ctx, const uint32_t* compOffsets,
                           const uint32_t* compPixels, size_t count, const glu_grid* grid,
                           int32_t* boxes);
/* Host: level of each component (1-based) for Chebyshev reach `reach` (= 2h). */
int glu_trial_levels(const int32_t* boxes, size_t count, int reach, int32_t* levels);
/* Run the listed components (device ids, mutually independent or ordered by
 * index) as trials; accepted trials are appended to `log` (may be NULL). */
int glu_cu_run_trials(glu_ctx* ctx, const float* high, float* low, glu_pixel_params* field,
                      float* errors, const glu_grid* grid, const glu_config* cfg, int mode,
                      const uint32_t* compOffsets, const uint32_t* compPixels,
                      const uint32_t* ids, size_t count, glu_trial_log* log, int* accepted,
                      int* rejected);
/* Apply another rank's change log. */
int glu_cu_apply_trial_log(glu_ctx* ctx, float* low, glu_pixel_params* field, float* errors,
                           const uint32_t* cells, size_t cellCount, const uint32_t* pixels,
                           size_t pixelCount);

/* ---- GLUP parameter files (io_glup.cpp:48-139; proj/README.md:97-117) --- */

/* Bytes of the GLUP encoding of a field on `grid`. */
size_t glu_glup_size(const glu_grid* grid);
/* encode_glup: header + the LR image + the records, streamed from device
 * buffers straight into `out` (pinned host memory or device memory). */
int glu_cu_glup_encode(glu_ctx* ctx, const glu_pixel_params* field, const float* low,
                       const glu_grid* grid, int mode, int optimized, uint8_t* out,
                       size_t capacity);
/* decode_glup: validates the header (host), copies the payload into device
 * buffers and validates it on the device.  With low or field NULL only the
 * header is checked and the grid / mode / flag are returned ("peek").
 * Format violations return GLU_EFORMAT; glu_last_error() holds the
 * reference's message and glu_last_error_field() its field name (length,
 * magic, version, dims, mode, flag, reserved, lowres, index, weight). */
int glu_cu_glup_decode(glu_ctx* ctx, const uint8_t* bytes, size_t size, glu_grid* grid,
                       int* mode, int* optimized, float* low, glu_pixel_params* field);
const char* glu_last_error_field(void);

/* ---- quality metrics (metrics.cpp:62-107) -------------------------------- */

/* mse: mean of squared differences over `count` floats (device pointers). */
int glu_cu_mse(glu_ctx* ctx, const float* a, const float* b, size_t count, double* out);
/* ssim: luma SSIM, 11x11 Gaussian sigma 1.5, valid windows, RGB images. */
int glu_cu_ssim(glu_ctx* ctx, const float* a, const float* b, int width, int height,
                double* out);

/* ---- comparison upsamplers (baseline.cpp:30-129) ------------------------- */

int glu_cu_nearest_upsample(glu_ctx* ctx, const float* lowTarget, const glu_grid* grid,
                            float* out);
int glu_cu_bilinear_upsample(glu_ctx* ctx, const float* lowTarget, const glu_grid* grid,
                             float* out);
/* JbuParams {window (odd >= 1), sigmaD, sigmaR} (baseline.hpp:8-14). */
int glu_cu_jbu_upsample(glu_ctx* ctx, const float* guideHigh, const float* guideLow,
                        const float* targetLow, const glu_grid* grid, int window,
                        double sigmaD, double sigmaR, float* out);

/* ---- host-pointer entry points (the C++ API's calls) ------------------- */

int glu_h_grid_downsample(glu_ctx* ctx, const float* high, const glu_grid* grid, float* low);
int glu_h_optimize_field(glu_ctx* ctx, const float* high, const float* low,
                         const glu_grid* grid, const glu_config* cfg, int mode,
                         glu_pixel_params* out);
int glu_h_optimize_pixels(glu_ctx* ctx, const float* high, const float* low,
                          const glu_grid* grid, const glu_config* cfg, int mode,
                          const uint32_t* pixels, size_t count, glu_pixel_params* field);
int glu_h_apply_field(glu_ctx* ctx, const glu_pixel_params* field, const glu_grid* grid,
                      const float* lowTarget, int channels, int clampOutput, float* out);
int glu_h_error_map(glu_ctx* ctx, const float* high, const float* recon, size_t pixelCount,
                    float* errors);
int glu_h_solve_apply(glu_ctx* ctx, const float* high, const float* low, const glu_grid* grid,
                      const glu_config* cfg, int mode, const float* lowTarget, int channels,
                      int clampOutput, float* out, glu_pixel_params* paramsOut);
/* find_large_error with host outputs: mask (W*H), compOffsets (cap W*H+1),
 * compPixels (cap W*H); *count = number of components. */
int glu_h_find_large_error(glu_ctx* ctx, const float* errors, int width, int height,
                           float threshold, uint8_t* mask, uint32_t* compOffsets,
                           uint32_t* compPixels, size_t* count);
int glu_h_trial_update_component(glu_ctx* ctx, const float* high, float* low,
                                 glu_pixel_params* field, float* errors, const glu_grid* grid,
                                 const glu_config* cfg, int mode, const uint32_t* component,
                                 size_t count, int* accepted);
int glu_h_joint_optimize(glu_ctx* ctx, const float* high, const glu_grid* grid,
                         const glu_config* cfg, int mode, float* low, glu_pixel_params* field,
                         float* errors, glu_joint_stats* stats);
/* glu_cu_upsample_frames from host memory: frame k+1's host-to-device copy
 * and frame k-1's device-to-host copy overlap frame k's kernels (two copy
 * streams, double-buffered device slots).  Pass pinned memory for full PCIe
 * bandwidth. */
int glu_h_upsample_frames(glu_ctx* ctx, const float* frames, int count, const glu_grid* grid,
                          const glu_config* cfg, int mode, int targetOp, float* out,
                          glu_pixel_params* paramsOut);
int glu_h_optimize_pixel_batch(glu_ctx* ctx, const float* ip, const uint32_t* offsets,
                               const uint32_t* candIdx, const float* candRgb, size_t count,
                               double eps, int mode, glu_pixel_params* out);
int glu_h_pair_eval(glu_ctx* ctx, const float* ip, const float* ia, const float* ib,
                    const double* w, size_t count, double eps, double* weightExact,
                    double* weightFast, double* objective);

#ifdef __cplusplus
}
#endif

#endif /* GLU_CUDA_H */
