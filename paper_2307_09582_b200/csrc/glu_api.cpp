// glu_api.cpp -- the drop-in C++ API (include/glu/glu_b200.hpp) over the
// C-ABI (include/glu_cuda.h).  Host code only: validation with the
// reference's messages, value-semantics marshalling, and exceptions.  Every
// bulk computation is a glu_h_* call into the sm_100a kernels; there is no
// CPU implementation of the hot path here.
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <thread>

#include "glu/glu_b200.hpp"
#include "glu_cuda.h"

namespace glu {

namespace {

// One C-ABI context per host thread and device.
struct CtxHolder {
    glu_ctx* ctx = nullptr;
    int device = -1;
    ~CtxHolder() {
        if (ctx) glu_ctx_destroy(ctx);
    }
};

glu_ctx* ctx() {
    thread_local CtxHolder h;
    int dev = 0;
    if (glu_current_device(&dev) != GLU_OK) dev = 0;
    if (!h.ctx || h.device != dev) {
        if (h.ctx) glu_ctx_destroy(h.ctx);
        h.ctx = nullptr;
        if (glu_ctx_create(dev, &h.ctx) != GLU_OK)
            throw std::runtime_error(std::string("glu: ") + glu_last_error());
        h.device = dev;
    }
    return h.ctx;
}

void check(int rc) {
    if (rc == GLU_OK) return;
    if (rc == GLU_EINVAL) throw std::invalid_argument(glu_last_error());
    if (rc == GLU_ENOMEM) throw std::bad_alloc();
    throw std::runtime_error(std::string("glu: ") + glu_last_error());
}

glu_grid cgrid(const GridSpec& g) {
    return {g.scale, g.highW, g.highH, g.lowW, g.lowH, g.sampleOffset};
}

glu_config ccfg(const GluConfig& c) {
    return {c.windowSide, c.errorThreshold, c.maxIterations, c.epsilon,
            c.literalComponentUpdate ? 1 : 0};
}

glu_pixel_params* cparams(PixelParams* p) { return reinterpret_cast<glu_pixel_params*>(p); }
const glu_pixel_params* cparams(const PixelParams* p) {
    return reinterpret_cast<const glu_pixel_params*>(p);
}

static_assert(sizeof(PixelParams) == sizeof(glu_pixel_params), "PixelParams layout");
static_assert(sizeof(Rgb) == 12, "Rgb layout");

// checkFieldInputs (upsample.cpp:147-154)
void checkFieldInputs(const ImageF32& high, const ImageF32& low, const GridSpec& grid,
                      const GluConfig& cfg) {
    cfg.validate();
    if (high.width != grid.highW || high.height != grid.highH)
        throw std::invalid_argument("optimize: guide image does not match grid");
    if (low.width != grid.lowW || low.height != grid.lowH)
        throw std::invalid_argument("optimize: low-res image does not match grid");
}

PixelParams selectOne(Rgb ip, std::span<const Candidate> cands, double eps, Mode mode) {
    if (cands.empty()) throw std::invalid_argument("candidate list must not be empty");
    std::vector<uint32_t> idx(cands.size());
    std::vector<float> rgb(cands.size() * 3);
    for (size_t i = 0; i < cands.size(); ++i) {
        idx[i] = cands[i].index;
        for (int c = 0; c < 3; ++c) rgb[3 * i + c] = cands[i].color[c];
    }
    const uint32_t off[2] = {0, uint32_t(cands.size())};
    PixelParams out;
    check(glu_h_optimize_pixel_batch(ctx(), ip.data(), off, idx.data(), rgb.data(), 1, eps,
                                     int(mode), cparams(&out)));
    return out;
}

std::atomic<int> g_threads{0};

}  // namespace

// ---- grid ---------------------------------------------------------------------

GridSpec GridSpec::create(int highW, int highH, int scale) {
    glu_grid g;
    check(glu_grid_create(highW, highH, scale, &g));
    GridSpec r;
    r.scale = g.scale;
    r.highW = g.highW;
    r.highH = g.highH;
    r.lowW = g.lowW;
    r.lowH = g.lowH;
    r.sampleOffset = g.sampleOffset;
    return r;
}

Coord GridSpec::sampleCoord(Coord cell) const {
    return {std::min(cell.x * scale + sampleOffset, highW - 1),
            std::min(cell.y * scale + sampleOffset, highH - 1)};
}

void GridSpec::windowBounds(Coord cell, int windowSide, int& x0, int& y0, int& x1,
                            int& y1) const {
    if (windowSide < 3 || windowSide % 2 == 0)
        throw std::invalid_argument("windowSide must be odd and >= 3");
    const int h = windowSide / 2;
    x0 = std::max(0, cell.x - h);
    y0 = std::max(0, cell.y - h);
    x1 = std::min(lowW - 1, cell.x + h);
    y1 = std::min(lowH - 1, cell.y + h);
}

ImageF32 grid_downsample(const ImageF32& high, int scale, GridSpec* outGrid) {
    const GridSpec g = GridSpec::create(high.width, high.height, scale);
    ImageF32 low(g.lowW, g.lowH);
    const glu_grid cg = cgrid(g);
    check(glu_h_grid_downsample(ctx(), high.data.data(), &cg, low.data.data()));
    if (outGrid) *outGrid = g;
    return low;
}

std::vector<uint32_t> neighborhood(Coord p, const GridSpec& grid, int windowSide) {
    if (p.x < 0 || p.y < 0 || p.x >= grid.highW || p.y >= grid.highH)
        throw std::invalid_argument("neighborhood: pixel outside image");
    int x0, y0, x1, y1;
    grid.windowBounds(grid.mapDown(p), windowSide, x0, y0, x1, y1);
    std::vector<uint32_t> out;
    for (int cy = y0; cy <= y1; ++cy)
        for (int cx = x0; cx <= x1; ++cx) out.push_back(grid.lowIndex(cx, cy));
    return out;
}

std::vector<Coord> footprint(Coord cell, const GridSpec& grid) {
    if (cell.x < 0 || cell.y < 0 || cell.x >= grid.lowW || cell.y >= grid.lowH)
        throw std::invalid_argument("footprint: cell outside grid");
    std::vector<Coord> out;
    for (int y = cell.y * grid.scale; y < std::min((cell.y + 1) * grid.scale, grid.highH); ++y)
        for (int x = cell.x * grid.scale; x < std::min((cell.x + 1) * grid.scale, grid.highW); ++x)
            out.push_back({x, y});
    return out;
}

// ---- params -------------------------------------------------------------------

const char* mode_name(Mode m) {
    switch (m) {
        case Mode::Exact: return "exact";
        case Mode::Gnu: return "gnu";
        default: return "fast";
    }
}

Mode mode_from_name(const std::string& name) {
    if (name == "fast") return Mode::Fast;
    if (name == "exact") return Mode::Exact;
    if (name == "gnu") return Mode::Gnu;
    throw std::invalid_argument("unknown mode: " + name + " (expected fast|exact|gnu)");
}

// ---- upsample -----------------------------------------------------------------

double weight_exact(Rgb ip, Rgb ia, Rgb ib, double eps) {
    double r = 0;
    check(glu_h_pair_eval(ctx(), ip.data(), ia.data(), ib.data(), nullptr, 1, eps, &r, nullptr,
                          nullptr));
    return r;
}

double weight_fast(Rgb ip, Rgb ia, Rgb ib, double eps) {
    double r = 0;
    check(glu_h_pair_eval(ctx(), ip.data(), ia.data(), ib.data(), nullptr, 1, eps, nullptr, &r,
                          nullptr));
    return r;
}

double pair_objective(Rgb ip, Rgb ia, Rgb ib, double w, double eps) {
    double r = 0;
    check(glu_h_pair_eval(ctx(), ip.data(), ia.data(), ib.data(), &w, 1, eps, nullptr, nullptr,
                          &r));
    return r;
}

PixelParams optimize_pixel_fast(Rgb ip, std::span<const Candidate> c, double eps) {
    return selectOne(ip, c, eps, Mode::Fast);
}

PixelParams optimize_pixel_exact(Rgb ip, std::span<const Candidate> c, double eps) {
    return selectOne(ip, c, eps, Mode::Exact);
}

PixelParams optimize_pixel_gnu(Rgb ip, std::span<const Candidate> c) {
    return selectOne(ip, c, 1e-3, Mode::Gnu);
}

ParamField optimize_field(const ImageF32& high, const ImageF32& low, const GridSpec& grid,
                          const GluConfig& cfg, Mode mode) {
    checkFieldInputs(high, low, grid, cfg);
    ParamField f;
    f.grid = grid;
    f.mode = mode;
    f.params.resize(high.pixelCount());
    const glu_grid cg = cgrid(grid);
    const glu_config cc = ccfg(cfg);
    check(glu_h_optimize_field(ctx(), high.data.data(), low.data.data(), &cg, &cc, int(mode),
                               cparams(f.params.data())));
    return f;
}

void optimize_pixels(const ImageF32& high, const ImageF32& low, const GridSpec& grid,
                     const GluConfig& cfg, Mode mode, std::span<const uint32_t> pixels,
                     ParamField& field) {
    checkFieldInputs(high, low, grid, cfg);
    if (field.params.size() != high.pixelCount())
        throw std::invalid_argument("optimize_pixels: field does not match image");
    if (pixels.empty()) return;
    const glu_grid cg = cgrid(grid);
    const glu_config cc = ccfg(cfg);
    check(glu_h_optimize_pixels(ctx(), high.data.data(), low.data.data(), &cg, &cc, int(mode),
                                pixels.data(), pixels.size(), cparams(field.params.data())));
}

ImageF32 apply_field(const ParamField& field, const ImageF32& lowTarget, bool clampOutput) {
    if (lowTarget.width != field.grid.lowW || lowTarget.height != field.grid.lowH)
        throw std::invalid_argument("apply_field: low-res image does not match grid");
    if (field.params.size() != size_t(field.grid.highW) * field.grid.highH)
        throw std::invalid_argument("apply_field: field size does not match grid");
    ImageF32 out(field.grid.highW, field.grid.highH);
    const glu_grid cg = cgrid(field.grid);
    check(glu_h_apply_field(ctx(), cparams(field.params.data()), &cg, lowTarget.data.data(), 3,
                            clampOutput ? 1 : 0, out.data.data()));
    return out;
}

ErrorMap error_map(const ImageF32& high, const ImageF32& reconstructed) {
    requireSameShape(high, reconstructed, "error_map");
    ErrorMap em;
    em.width = high.width;
    em.height = high.height;
    em.e.resize(high.pixelCount());
    check(glu_h_error_map(ctx(), high.data.data(), reconstructed.data.data(), high.pixelCount(),
                          em.e.data()));
    return em;
}

// ---- jointopt -----------------------------------------------------------------

LargeErrorSet find_large_error(const ErrorMap& errors, float threshold) {
    if (errors.width <= 0 || errors.height <= 0)
        throw std::invalid_argument("find_large_error: empty error map");
    const size_t n = size_t(errors.width) * errors.height;
    LargeErrorSet out;
    out.width = errors.width;
    out.height = errors.height;
    out.mask.resize(n);
    std::vector<uint32_t> off(n + 1), px(n);
    size_t count = 0;
    check(glu_h_find_large_error(ctx(), errors.e.data(), errors.width, errors.height, threshold,
                                 out.mask.data(), off.data(), px.data(), &count));
    out.components.resize(count);
    for (size_t c = 0; c < count; ++c)
        out.components[c].assign(px.begin() + off[c], px.begin() + off[c + 1]);
    return out;
}

bool trial_update_component(const ImageF32& high, ImageF32& low, ParamField& field,
                            ErrorMap& errors, std::span<const uint32_t> component,
                            const GluConfig& cfg, Mode mode) {
    cfg.validate();
    if (component.empty()) throw std::invalid_argument("trial_update_component: empty component");
    const GridSpec& g = field.grid;
    if (high.width != g.highW || high.height != g.highH || low.width != g.lowW ||
        low.height != g.lowH || errors.width != g.highW || errors.height != g.highH)
        throw std::invalid_argument("trial_update_component: shape mismatch");
    // The reference reaches optimize_pixels (upsample.cpp:222-223) with a
    // field of the wrong size and throws there; the host buffers below are
    // copied by size, so check every container before any device work.
    if (field.params.size() != high.pixelCount())
        throw std::invalid_argument("optimize_pixels: field does not match image");
    if (high.data.size() != 3 * high.pixelCount() || low.data.size() != 3 * low.pixelCount() ||
        errors.e.size() != high.pixelCount())
        throw std::invalid_argument("trial_update_component: shape mismatch");
    const glu_grid cg = cgrid(g);
    const glu_config cc = ccfg(cfg);
    int accepted = 0;
    check(glu_h_trial_update_component(ctx(), high.data.data(), low.data.data(),
                                       cparams(field.params.data()), errors.e.data(), &cg, &cc,
                                       int(mode), component.data(), component.size(), &accepted));
    return accepted != 0;
}

JointResult joint_optimize(const ImageF32& high, int scale, const GluConfig& cfg, Mode mode) {
    cfg.validate();
    const GridSpec g = GridSpec::create(high.width, high.height, scale);
    JointResult r;
    r.low = ImageF32(g.lowW, g.lowH);
    r.field.grid = g;
    r.field.mode = mode;
    r.field.params.resize(high.pixelCount());
    r.errors.width = high.width;
    r.errors.height = high.height;
    r.errors.e.resize(high.pixelCount());
    const glu_grid cg = cgrid(g);
    const glu_config cc = ccfg(cfg);
    glu_joint_stats st{};
    check(glu_h_joint_optimize(ctx(), high.data.data(), &cg, &cc, int(mode), r.low.data.data(),
                               cparams(r.field.params.data()), r.errors.e.data(), &st));
    r.iterations = st.iterations;
    r.trialsAccepted = st.trialsAccepted;
    r.trialsRejected = st.trialsRejected;
    return r;
}

// ---- GLUP files (io_glup.cpp:48-159) -------------------------------------------

namespace {

// Device staging for the codec: field + LR image + raw bytes.
struct DevBuf {
    void* p = nullptr;
    explicit DevBuf(size_t n) {
        if (n && glu_cu_alloc(ctx(), &p, n) != GLU_OK) throw std::bad_alloc();
    }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p) { o.p = nullptr; }
    ~DevBuf() {
        if (p) glu_cu_free(ctx(), p);
    }
};

}  // namespace

std::vector<uint8_t> encode_glup(const GlupFile& f) {
    const GridSpec& g = f.field.grid;
    if (g.highW <= 0 || g.highH <= 0 || g.scale < 2)
        throw std::invalid_argument("encode_glup: field has no grid");
    if (f.field.params.size() != size_t(g.highW) * g.highH)
        throw std::invalid_argument("encode_glup: param count does not match grid");
    if (f.low.width != g.lowW || f.low.height != g.lowH)
        throw std::invalid_argument("encode_glup: low-res image does not match grid");
    const glu_grid cg = cgrid(g);
    std::vector<uint8_t> out(glu_glup_size(&cg));
    DevBuf dp(f.field.params.size() * sizeof(PixelParams)), dl(f.low.data.size() * 4);
    check(glu_cu_upload(ctx(), dp.p, f.field.params.data(), f.field.params.size() * 12));
    check(glu_cu_upload(ctx(), dl.p, f.low.data.data(), f.low.data.size() * 4));
    check(glu_cu_glup_encode(ctx(), static_cast<const glu_pixel_params*>(dp.p),
                             static_cast<const float*>(dl.p), &cg, int(f.field.mode),
                             f.optimized ? 1 : 0, out.data(), out.size()));
    return out;
}

GlupFile decode_glup(const std::vector<uint8_t>& bytes) {
    glu_grid g{};
    int mode = 0, opt = 0;
    auto rethrow = [](int rc) {
        if (rc == GLU_EFORMAT) throw FormatError(glu_last_error_field(), glu_last_error());
        check(rc);
    };
    rethrow(glu_cu_glup_decode(ctx(), bytes.data(), bytes.size(), &g, &mode, &opt, nullptr,
                               nullptr));
    GlupFile f;
    f.field.grid = GridSpec::create(g.highW, g.highH, g.scale);
    f.field.mode = static_cast<Mode>(mode);
    f.optimized = opt == 1;
    f.low = ImageF32(g.lowW, g.lowH);
    f.field.params.resize(size_t(g.highW) * g.highH);
    DevBuf dp(f.field.params.size() * 12), dl(f.low.data.size() * 4);
    rethrow(glu_cu_glup_decode(ctx(), bytes.data(), bytes.size(), &g, &mode, &opt,
                               static_cast<float*>(dl.p), static_cast<glu_pixel_params*>(dp.p)));
    check(glu_cu_download(ctx(), f.field.params.data(), dp.p, f.field.params.size() * 12));
    check(glu_cu_download(ctx(), f.low.data.data(), dl.p, f.low.data.size() * 4));
    return f;
}

void write_glup(const std::string& path, const GlupFile& f) {
    const std::vector<uint8_t> bytes = encode_glup(f);
    std::FILE* fp = std::fopen(path.c_str(), "wb");
    if (!fp) throw IoError("cannot open for writing: " + path);
    const size_t n = std::fwrite(bytes.data(), 1, bytes.size(), fp);
    const bool bad = n != bytes.size() || std::fclose(fp) != 0;
    if (bad) throw IoError("write failed: " + path);
}

GlupFile read_glup(const std::string& path) {
    std::FILE* fp = std::fopen(path.c_str(), "rb");
    if (!fp) throw IoError("cannot open: " + path);
    std::vector<uint8_t> bytes;
    uint8_t buf[1 << 16];
    size_t n;
    while ((n = std::fread(buf, 1, sizeof(buf), fp)) > 0) bytes.insert(bytes.end(), buf, buf + n);
    const bool bad = std::ferror(fp) != 0;
    std::fclose(fp);
    if (bad) throw IoError("read failed: " + path);
    return decode_glup(bytes);
}

// ---- metrics (metrics.cpp:62-115) ------------------------------------------------

namespace {

struct DevPair {
    DevBuf a, b;
    DevPair(const ImageF32& x, const ImageF32& y)
        : a(x.data.size() * sizeof(float)), b(y.data.size() * sizeof(float)) {
        check(glu_cu_upload(ctx(), a.p, x.data.data(), x.data.size() * sizeof(float)));
        check(glu_cu_upload(ctx(), b.p, y.data.data(), y.data.size() * sizeof(float)));
    }
    const float* fa() const { return static_cast<const float*>(a.p); }
    const float* fb() const { return static_cast<const float*>(b.p); }
};

}  // namespace

double mse(const ImageF32& a, const ImageF32& b) {
    requireSameShape(a, b, "mse");
    DevPair d(a, b);
    double m = 0;
    check(glu_cu_mse(ctx(), d.fa(), d.fb(), a.data.size(), &m));
    return m;
}

double psnr(const ImageF32& a, const ImageF32& b) {
    const double m = mse(a, b);
    if (m == 0) return 99.0;
    return 10.0 * std::log10(1.0 / m);
}

double ssim(const ImageF32& a, const ImageF32& b) {
    requireSameShape(a, b, "ssim");
    if (a.width < 11 || a.height < 11)
        throw std::invalid_argument("ssim: images smaller than the 11x11 window");
    DevPair d(a, b);
    double s = 0;
    check(glu_cu_ssim(ctx(), d.fa(), d.fb(), a.width, a.height, &s));
    return s;
}

QualityReport quality_report(const ImageF32& reference, const ImageF32& test) {
    QualityReport q;
    q.mse = mse(reference, test);
    q.psnrDb = q.mse == 0 ? 99.0 : 10.0 * std::log10(1.0 / q.mse);
    q.ssim = ssim(reference, test);
    return q;
}

// ---- comparison upsamplers (baseline.cpp:30-129) -----------------------------------

namespace {

void checkLowGrid(const ImageF32& low, const GridSpec& grid, const char* what) {
    if (low.width != grid.lowW || low.height != grid.lowH)
        throw std::invalid_argument(std::string(what) + ": low-res image does not match grid");
}

ImageF32 downloadImage(const DevBuf& d, int w, int h) {
    ImageF32 out(w, h);
    check(glu_cu_download(ctx(), out.data.data(), d.p, out.data.size() * sizeof(float)));
    return out;
}

DevBuf uploadImage(const ImageF32& img) {
    DevBuf d(img.data.size() * sizeof(float));
    check(glu_cu_upload(ctx(), d.p, img.data.data(), img.data.size() * sizeof(float)));
    return d;
}

}  // namespace

ImageF32 jbu_upsample(const ImageF32& guideHigh, const ImageF32& guideLow,
                      const ImageF32& targetLow, const GridSpec& grid, const JbuParams& params) {
    params.validate();
    if (guideHigh.width != grid.highW || guideHigh.height != grid.highH)
        throw std::invalid_argument("jbu_upsample: guide image does not match grid");
    checkLowGrid(guideLow, grid, "jbu_upsample");
    checkLowGrid(targetLow, grid, "jbu_upsample");
    const DevBuf gh = uploadImage(guideHigh), gl = uploadImage(guideLow),
                 tl = uploadImage(targetLow);
    DevBuf out(size_t(grid.highW) * grid.highH * 3 * sizeof(float));
    const glu_grid cg = cgrid(grid);
    check(glu_cu_jbu_upsample(ctx(), static_cast<const float*>(gh.p),
                              static_cast<const float*>(gl.p), static_cast<const float*>(tl.p),
                              &cg, params.window, params.sigmaD, params.sigmaR,
                              static_cast<float*>(out.p)));
    return downloadImage(out, grid.highW, grid.highH);
}

ImageF32 nearest_upsample(const ImageF32& targetLow, const GridSpec& grid) {
    checkLowGrid(targetLow, grid, "nearest_upsample");
    const DevBuf tl = uploadImage(targetLow);
    DevBuf out(size_t(grid.highW) * grid.highH * 3 * sizeof(float));
    const glu_grid cg = cgrid(grid);
    check(glu_cu_nearest_upsample(ctx(), static_cast<const float*>(tl.p), &cg,
                                  static_cast<float*>(out.p)));
    return downloadImage(out, grid.highW, grid.highH);
}

ImageF32 bilinear_upsample(const ImageF32& targetLow, const GridSpec& grid) {
    checkLowGrid(targetLow, grid, "bilinear_upsample");
    const DevBuf tl = uploadImage(targetLow);
    DevBuf out(size_t(grid.highW) * grid.highH * 3 * sizeof(float));
    const glu_grid cg = cgrid(grid);
    check(glu_cu_bilinear_upsample(ctx(), static_cast<const float*>(tl.p), &cg,
                                   static_cast<float*>(out.p)));
    return downloadImage(out, grid.highW, grid.highH);
}

// ---- parallel (host utility) --------------------------------------------------

void set_num_threads(int n) {
    if (n < 0) throw std::invalid_argument("set_num_threads: n must be >= 0");
    g_threads.store(n);
}

int num_threads() {
    const int n = g_threads.load();
    if (n > 0) return n;
    const unsigned hw = std::thread::hardware_concurrency();
    return hw ? int(hw) : 1;
}

void parallel_for(int count, const std::function<void(int, int)>& fn, int minGrain) {
    if (count <= 0) return;
    const int workers = std::min(num_threads(), (count + minGrain - 1) / minGrain);
    if (workers <= 1) {
        fn(0, count);
        return;
    }
    const int chunk = (count + workers - 1) / workers;
    std::vector<std::thread> pool;
    for (int t = 1; t < workers && t * chunk < count; ++t)
        pool.emplace_back(fn, t * chunk, std::min(count, (t + 1) * chunk));
    fn(0, std::min(count, chunk));
    for (auto& th : pool) th.join();
}

}  // namespace glu
