// glu_b200.hpp -- drop-in C++ API of the B200 GLU hot path.
//
// Declares, in namespace glu, the types and functions of the reference's
// public headers proj/include/glu/{image,grid,params,upsample,jointopt,
// parallel}.hpp with identical signatures and semantics, so code written
// against the reference recompiles and relinks against lib/libglu.so
// unchanged.  The per-header files in this directory (image.hpp, grid.hpp,
// ...) only include this one.  The bulk entry points run on the GPU through
// the C-ABI of include/glu_cuda.h; value semantics (host std::vectors in,
// host std::vectors out) are kept, so each call copies in and out.
#pragma once

#include <array>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <functional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

namespace glu {

// ---- image.hpp -----------------------------------------------------------------

using Rgb = std::array<float, 3>;

/// Interleaved RGB float image, row-major, 3 floats per pixel.
struct ImageF32 {
    int width = 0;
    int height = 0;
    std::vector<float> data;

    ImageF32() = default;
    ImageF32(int w, int h) : width(w), height(h) {
        if (w <= 0 || h <= 0) throw std::invalid_argument("ImageF32: dimensions must be positive");
        data.assign(size_t(w) * size_t(h) * 3, 0.0f);
    }
    ImageF32(int w, int h, Rgb fill) : ImageF32(w, h) {
        for (size_t k = 0; k + 2 < data.size(); k += 3) {
            data[k] = fill[0];
            data[k + 1] = fill[1];
            data[k + 2] = fill[2];
        }
    }

    size_t pixelCount() const { return size_t(width) * size_t(height); }
    float* px(int x, int y) { return data.data() + 3 * (size_t(y) * width + x); }
    const float* px(int x, int y) const { return data.data() + 3 * (size_t(y) * width + x); }
    float* px(uint32_t i) { return data.data() + 3 * size_t(i); }
    const float* px(uint32_t i) const { return data.data() + 3 * size_t(i); }
    float& at(int x, int y, int c) { return px(x, y)[c]; }
    float at(int x, int y, int c) const { return px(x, y)[c]; }
    Rgb rgb(int x, int y) const {
        const float* p = px(x, y);
        return {p[0], p[1], p[2]};
    }
    Rgb rgb(uint32_t i) const {
        const float* p = px(i);
        return {p[0], p[1], p[2]};
    }
    void setRgb(int x, int y, Rgb v) {
        float* p = px(x, y);
        p[0] = v[0];
        p[1] = v[1];
        p[2] = v[2];
    }
    bool sameShape(const ImageF32& o) const { return width == o.width && height == o.height; }
};

inline void requireSameShape(const ImageF32& a, const ImageF32& b, const char* what) {
    if (!a.sameShape(b)) throw std::invalid_argument(std::string(what) + ": image dimensions differ");
}

// ---- grid.hpp ------------------------------------------------------------------

struct Coord {
    int x = 0;
    int y = 0;
    bool operator==(const Coord&) const = default;
};

/// LR cell (cx, cy) samples HR pixel min(c*s + s/2, dim-1) and owns the s x s
/// block starting at (cx*s, cy*s), clipped to the image.
struct GridSpec {
    int scale = 0;
    int highW = 0, highH = 0;
    int lowW = 0, lowH = 0;
    int sampleOffset = 0;

    static GridSpec create(int highW, int highH, int scale);
    uint32_t lowIndex(int cx, int cy) const { return uint32_t(cy) * uint32_t(lowW) + uint32_t(cx); }
    size_t lowCount() const { return size_t(lowW) * size_t(lowH); }
    Coord mapDown(Coord p) const { return {p.x / scale, p.y / scale}; }
    Coord sampleCoord(Coord cell) const;
    void windowBounds(Coord cell, int windowSide, int& x0, int& y0, int& x1, int& y1) const;
};

ImageF32 grid_downsample(const ImageF32& high, int scale, GridSpec* outGrid = nullptr);
std::vector<uint32_t> neighborhood(Coord p, const GridSpec& grid, int windowSide);
std::vector<Coord> footprint(Coord cell, const GridSpec& grid);

// ---- params.hpp ----------------------------------------------------------------

enum class Mode : uint8_t { Fast = 0, Exact = 1, Gnu = 2 };

const char* mode_name(Mode m);
Mode mode_from_name(const std::string& name);

struct GluConfig {
    int windowSide = 3;
    float errorThreshold = 30.0f / 255.0f;
    int maxIterations = 3;
    float epsilon = 1e-3f;
    bool literalComponentUpdate = false;

    void validate() const {
        if (windowSide < 3 || windowSide % 2 == 0)
            throw std::invalid_argument("GluConfig: windowSide must be odd and >= 3");
        if (!(errorThreshold >= 0))
            throw std::invalid_argument("GluConfig: errorThreshold must be >= 0");
        if (maxIterations < 0) throw std::invalid_argument("GluConfig: maxIterations must be >= 0");
        if (!(epsilon > 0)) throw std::invalid_argument("GluConfig: epsilon must be > 0");
    }
};

/// out = w * low[a] + (1 - w) * low[b]; 12 bytes, same layout as glu_pixel_params.
struct PixelParams {
    uint32_t a = 0;
    uint32_t b = 0;
    float w = 0.0f;
};

struct ParamField {
    GridSpec grid;
    Mode mode = Mode::Fast;
    std::vector<PixelParams> params;
    size_t size() const { return params.size(); }
};

struct ErrorMap {
    int width = 0;
    int height = 0;
    std::vector<float> e;
    float& at(int x, int y) { return e[size_t(y) * width + x]; }
    float at(int x, int y) const { return e[size_t(y) * width + x]; }
    double total() const {
        double sum = 0;
        for (float v : e) sum += v;
        return sum;
    }
};

// ---- upsample.hpp --------------------------------------------------------------

struct Candidate {
    uint32_t index = 0;
    Rgb color{};
};

double weight_exact(Rgb ip, Rgb ia, Rgb ib, double eps);
double weight_fast(Rgb ip, Rgb ia, Rgb ib, double eps);
double pair_objective(Rgb ip, Rgb ia, Rgb ib, double w, double eps);

PixelParams optimize_pixel_fast(Rgb ip, std::span<const Candidate> cands, double eps);
PixelParams optimize_pixel_exact(Rgb ip, std::span<const Candidate> cands, double eps);
PixelParams optimize_pixel_gnu(Rgb ip, std::span<const Candidate> cands);

ParamField optimize_field(const ImageF32& high, const ImageF32& low, const GridSpec& grid,
                          const GluConfig& cfg, Mode mode);
void optimize_pixels(const ImageF32& high, const ImageF32& low, const GridSpec& grid,
                     const GluConfig& cfg, Mode mode, std::span<const uint32_t> pixels,
                     ParamField& field);
ImageF32 apply_field(const ParamField& field, const ImageF32& lowTarget, bool clampOutput = true);
ErrorMap error_map(const ImageF32& high, const ImageF32& reconstructed);

/// Single-pixel apply_field; bitwise equal to the bulk kernel (float maths,
/// no contraction).
inline Rgb reconstruct_pixel(const PixelParams& pp, const ImageF32& lowTarget,
                             bool clampOutput = true) {
    const float* ta = lowTarget.px(pp.a);
    const float* tb = lowTarget.px(pp.b);
    Rgb r;
    for (int c = 0; c < 3; ++c) {
        const float wa = pp.w * ta[c];
        const float wb = (1.0f - pp.w) * tb[c];
        float v = wa + wb;
        if (clampOutput) v = v < 0.0f ? 0.0f : (v > 1.0f ? 1.0f : v);
        r[c] = v;
    }
    return r;
}

/// Single-pixel error_map: Euclidean RGB distance in double, rounded to float.
inline float pixel_error(Rgb truth, Rgb recon) {
    double acc = 0;
    for (int c = 0; c < 3; ++c) {
        const double d = double(truth[c]) - double(recon[c]);
        acc += d * d;
    }
    return float(std::sqrt(acc));
}

// ---- jointopt.hpp --------------------------------------------------------------

struct LargeErrorSet {
    int width = 0;
    int height = 0;
    std::vector<uint8_t> mask;
    std::vector<std::vector<uint32_t>> components;
};

LargeErrorSet find_large_error(const ErrorMap& errors, float threshold);

bool trial_update_component(const ImageF32& high, ImageF32& low, ParamField& field,
                            ErrorMap& errors, std::span<const uint32_t> component,
                            const GluConfig& cfg, Mode mode);

struct JointResult {
    ImageF32 low;
    ParamField field;
    ErrorMap errors;
    int iterations = 0;
    int trialsAccepted = 0;
    int trialsRejected = 0;
};

JointResult joint_optimize(const ImageF32& high, int scale, const GluConfig& cfg, Mode mode);

// ---- baseline.hpp: comparison upsamplers -----------------------------------------

struct JbuParams {
    int window = 5;
    double sigmaD = 0.5;
    double sigmaR = 0.1;

    void validate() const {
        if (window < 1 || window % 2 == 0)
            throw std::invalid_argument("JbuParams: window must be odd and >= 1");
        if (!(sigmaD > 0) || !(sigmaR > 0))
            throw std::invalid_argument("JbuParams: sigmas must be > 0");
    }
};

ImageF32 jbu_upsample(const ImageF32& guideHigh, const ImageF32& guideLow,
                      const ImageF32& targetLow, const GridSpec& grid, const JbuParams& params);
ImageF32 nearest_upsample(const ImageF32& targetLow, const GridSpec& grid);
ImageF32 bilinear_upsample(const ImageF32& targetLow, const GridSpec& grid);

// ---- metrics.hpp -----------------------------------------------------------------

struct QualityReport {
    double mse = 0;
    double psnrDb = 0;
    double ssim = 0;
};

double mse(const ImageF32& a, const ImageF32& b);
double psnr(const ImageF32& a, const ImageF32& b);
double ssim(const ImageF32& a, const ImageF32& b);
QualityReport quality_report(const ImageF32& reference, const ImageF32& test);

// ---- io.hpp: GLUP parameter files (PNG/PPM image I/O is out of scope) --------

struct IoError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct FormatError : std::runtime_error {
    std::string field;
    FormatError(std::string fieldName, const std::string& msg)
        : std::runtime_error(msg), field(std::move(fieldName)) {}
};

struct GlupFile {
    ParamField field;
    ImageF32 low;
    bool optimized = false;
};

void write_glup(const std::string& path, const GlupFile& f);
GlupFile read_glup(const std::string& path);
std::vector<uint8_t> encode_glup(const GlupFile& f);
GlupFile decode_glup(const std::vector<uint8_t>& bytes);

// ---- parallel.hpp (host utility kept for drop-in; the GPU path ignores it) ----

void set_num_threads(int n);
int num_threads();
void parallel_for(int count, const std::function<void(int, int)>& fn, int minGrain = 1024);

}  // namespace glu
