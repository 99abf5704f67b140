// ref_shim.cpp -- C-ABI shim over the UNMODIFIED reference library.
//
// TEST / BASELINE INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file
// together with the reference's own sources (read in place under
// /root/reference/proj/src, never copied) into oracle/_ref/libglu_ref.so.
// It is used (1) to generate the golden vectors in tests/golden/ that pin
// oracle/glu_oracle.c, and (2) as the CPU baseline ("kind": "reference") timed
// by bench.py.  Nothing in the product links it.
#include <array>
#include <cstdio>
#include <cstring>
#include <span>
#include <thread>
#include <vector>

#include "glu/baseline.hpp"
#include "glu/grid.hpp"
#include "glu/io.hpp"
#include "glu/jointopt.hpp"
#include "glu/metrics.hpp"
#include "glu/parallel.hpp"
#include "glu/simop.hpp"
#include "glu/synth.hpp"
#include "glu/upsample.hpp"

using namespace glu;

namespace {

ImageF32 wrap(const float* d, int w, int h) {
    ImageF32 img(w, h);
    std::memcpy(img.data.data(), d, img.data.size() * sizeof(float));
    return img;
}

GluConfig config(int S, double eps, float thr, int maxIter, int literal) {
    GluConfig c;
    c.windowSide = S;
    c.epsilon = static_cast<float>(eps);
    c.errorThreshold = thr;
    c.maxIterations = maxIter;
    c.literalComponentUpdate = literal != 0;
    return c;
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

}  // namespace

extern "C" {

void glu_r_set_num_threads(int n) { set_num_threads(n); }

// apply_operator (simop.cpp:120-132) with an operator built by the
// reference's own constructors: kind 0 identity, 1 gain, 2 mix, 3 gray,
// 4 gamma, 5 invert.
int glu_r_apply_operator(int kind, double gain, double gamma, const double* mix, const float* in,
                         int w, int h, float* out) {
    return guarded([&] {
        SimOperator op;
        switch (kind) {
            case 0: op = identity_op(); break;
            case 1: op = scalar_gain_op(gain); break;
            case 2: {
                std::array<double, 9> m{};
                for (int i = 0; i < 9; ++i) m[i] = mix[i];
                op = channel_mix_op(m);
                break;
            }
            case 3: op = grayscale_op(); break;
            case 4: op = gamma_op(gamma); break;
            case 5: op = invert_op(); break;
            default: throw std::invalid_argument("kind");
        }
        const ImageF32 r = apply_operator(op, wrap(in, w, h));
        std::memcpy(out, r.data.data(), r.data.size() * sizeof(float));
    });
}
int glu_r_num_threads() { return num_threads(); }

// Synthetic generators of the reference (synth.cpp), used to build the same
// images the reference unit tests use.
int glu_r_synth(const char* kind, int w, int h, unsigned long long seed, float* out) {
    return guarded([&] {
        ImageF32 img;
        if (!std::strcmp(kind, "mixture"))
            img = synth_mixture(w, h, seed);
        else if (!std::strcmp(kind, "photo"))
            img = synth_photo(w, h, seed);
        else
            throw std::invalid_argument("kind");
        std::memcpy(out, img.data.data(), img.data.size() * sizeof(float));
    });
}

// optimize_pixel_{fast,exact,gnu} (upsample.cpp:178-192) on one candidate list.
int glu_r_optimize_pixel(const float* ip, const uint32_t* idx, const float* rgb, size_t n,
                         double eps, int mode, PixelParams* out) {
    return guarded([&] {
        std::vector<Candidate> c(n);
        for (size_t i = 0; i < n; ++i) c[i] = {idx[i], {rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2]}};
        const Rgb p{ip[0], ip[1], ip[2]};
        if (mode == 1)
            *out = optimize_pixel_exact(p, c, eps);
        else if (mode == 2)
            *out = optimize_pixel_gnu(p, c);
        else
            *out = optimize_pixel_fast(p, c, eps);
    });
}

int glu_r_grid_downsample(const float* high, int W, int H, int s, float* low) {
    return guarded([&] {
        const ImageF32 l = grid_downsample(wrap(high, W, H), s);
        std::memcpy(low, l.data.data(), l.data.size() * sizeof(float));
    });
}

// optimize_field with eps passed as the float GluConfig::epsilon holds.
int glu_r_optimize_field(const float* high, int W, int H, const float* low, int s, int S,
                         double eps, int mode, PixelParams* out) {
    return guarded([&] {
        const GridSpec g = GridSpec::create(W, H, s);
        const ParamField f = optimize_field(wrap(high, W, H), wrap(low, g.lowW, g.lowH), g,
                                            config(S, eps, 30.0f / 255.0f, 3, 0),
                                            static_cast<Mode>(mode));
        std::memcpy(out, f.params.data(), f.params.size() * sizeof(PixelParams));
    });
}

// "Reference API on all cores": optimize_pixels on disjoint
// contiguous row bands of one field from `threads` std::threads.  Bitwise equal
// to optimize_field (upsample_test.cpp:226-237).
int glu_r_optimize_field_allcores(const float* high, int W, int H, const float* low, int s,
                                  int S, double eps, int mode, int threads, PixelParams* out) {
    return guarded([&] {
        const GridSpec g = GridSpec::create(W, H, s);
        const ImageF32 hi = wrap(high, W, H), lo = wrap(low, g.lowW, g.lowH);
        const GluConfig cfg = config(S, eps, 30.0f / 255.0f, 3, 0);
        ParamField f;
        f.grid = g;
        f.mode = static_cast<Mode>(mode);
        f.params.resize(static_cast<size_t>(W) * H);
        if (threads <= 0) threads = static_cast<int>(std::thread::hardware_concurrency());
        if (threads <= 0) threads = 1;
        const int rows = (H + threads - 1) / threads;
        std::vector<std::thread> pool;
        for (int t = 0; t < threads; ++t) {
            const int y0 = t * rows, y1 = std::min(H, y0 + rows);
            if (y0 >= y1) break;
            pool.emplace_back([&, y0, y1] {
                std::vector<uint32_t> px(static_cast<size_t>(y1 - y0) * W);
                for (size_t i = 0; i < px.size(); ++i)
                    px[i] = static_cast<uint32_t>(static_cast<size_t>(y0) * W + i);
                optimize_pixels(hi, lo, g, cfg, f.mode, px, f);
            });
        }
        for (auto& th : pool) th.join();
        std::memcpy(out, f.params.data(), f.params.size() * sizeof(PixelParams));
    });
}

int glu_r_apply_field(const PixelParams* params, int W, int H, int s, const float* lowT,
                      int clampOutput, float* out) {
    return guarded([&] {
        ParamField f;
        f.grid = GridSpec::create(W, H, s);
        f.params.assign(params, params + static_cast<size_t>(W) * H);
        const ImageF32 o = apply_field(f, wrap(lowT, f.grid.lowW, f.grid.lowH), clampOutput != 0);
        std::memcpy(out, o.data.data(), o.data.size() * sizeof(float));
    });
}

int glu_r_error_map(const float* high, const float* recon, int W, int H, float* e) {
    return guarded([&] {
        const ErrorMap em = error_map(wrap(high, W, H), wrap(recon, W, H));
        std::memcpy(e, em.e.data(), em.e.size() * sizeof(float));
    });
}

long glu_r_find_large_error(const float* e, int W, int H, float thr, uint8_t* mask,
                            uint32_t* off, uint32_t* px) {
    long n = -1;
    guarded([&] {
        ErrorMap em;
        em.width = W;
        em.height = H;
        em.e.assign(e, e + static_cast<size_t>(W) * H);
        const LargeErrorSet les = find_large_error(em, thr);
        std::memcpy(mask, les.mask.data(), les.mask.size());
        off[0] = 0;
        uint32_t used = 0;
        for (size_t c = 0; c < les.components.size(); ++c) {
            for (uint32_t p : les.components[c]) px[used++] = p;
            off[c + 1] = used;
        }
        n = static_cast<long>(les.components.size());
    });
    return n;
}

int glu_r_trial_update_component(const float* high, int W, int H, float* low, int s, int S,
                                 double eps, int mode, int literal, PixelParams* field,
                                 float* errors, const uint32_t* comp, size_t n) {
    int accepted = -1;
    guarded([&] {
        const GridSpec g = GridSpec::create(W, H, s);
        ImageF32 lo = wrap(low, g.lowW, g.lowH);
        ParamField f;
        f.grid = g;
        f.mode = static_cast<Mode>(mode);
        f.params.assign(field, field + static_cast<size_t>(W) * H);
        ErrorMap em;
        em.width = W;
        em.height = H;
        em.e.assign(errors, errors + static_cast<size_t>(W) * H);
        accepted = trial_update_component(wrap(high, W, H), lo, f, em,
                                          std::span<const uint32_t>(comp, n),
                                          config(S, eps, 30.0f / 255.0f, 3, literal),
                                          static_cast<Mode>(mode))
                       ? 1
                       : 0;
        std::memcpy(low, lo.data.data(), lo.data.size() * sizeof(float));
        std::memcpy(field, f.params.data(), f.params.size() * sizeof(PixelParams));
        std::memcpy(errors, em.e.data(), em.e.size() * sizeof(float));
    });
    return accepted;
}

int glu_r_joint_optimize(const float* high, int W, int H, int s, int S, float thr, int maxIter,
                         double eps, int mode, int literal, float* low, PixelParams* field,
                         float* errors, int* counters) {
    return guarded([&] {
        const JointResult r = joint_optimize(wrap(high, W, H), s,
                                             config(S, eps, thr, maxIter, literal),
                                             static_cast<Mode>(mode));
        std::memcpy(low, r.low.data.data(), r.low.data.size() * sizeof(float));
        std::memcpy(field, r.field.params.data(), r.field.params.size() * sizeof(PixelParams));
        std::memcpy(errors, r.errors.e.data(), r.errors.e.size() * sizeof(float));
        counters[0] = r.iterations;
        counters[1] = r.trialsAccepted;
        counters[2] = r.trialsRejected;
    });
}

// jbu / nearest / bilinear (baseline.cpp:30-129); kind 0 nearest, 1 bilinear, 2 jbu.
int glu_r_baseline(int kind, const float* guideHigh, const float* guideLow, const float* target,
                   int W, int H, int s, int window, double sigmaD, double sigmaR, float* out) {
    return guarded([&] {
        const GridSpec g = GridSpec::create(W, H, s);
        const ImageF32 t = wrap(target, g.lowW, g.lowH);
        ImageF32 o;
        if (kind == 0)
            o = nearest_upsample(t, g);
        else if (kind == 1)
            o = bilinear_upsample(t, g);
        else {
            JbuParams p;
            p.window = window;
            p.sigmaD = sigmaD;
            p.sigmaR = sigmaR;
            o = jbu_upsample(wrap(guideHigh, W, H), wrap(guideLow, g.lowW, g.lowH), t, g, p);
        }
        std::memcpy(out, o.data.data(), o.data.size() * sizeof(float));
    });
}

// mse / psnr / ssim (metrics.cpp:62-107); out = {mse, psnr, ssim}.
int glu_r_quality(const float* a, const float* b, int W, int H, double* out) {
    return guarded([&] {
        const QualityReport q = quality_report(wrap(a, W, H), wrap(b, W, H));
        out[0] = q.mse;
        out[1] = q.psnrDb;
        out[2] = q.ssim;
    });
}

// encode_glup (io_glup.cpp:48-77): writes up to cap bytes, returns the size.
long glu_r_encode_glup(const PixelParams* params, const float* low, int W, int H, int s,
                       int mode, int optimized, uint8_t* out, size_t cap) {
    long n = -1;
    guarded([&] {
        GlupFile f;
        f.field.grid = GridSpec::create(W, H, s);
        f.field.mode = static_cast<Mode>(mode);
        f.field.params.assign(params, params + static_cast<size_t>(W) * H);
        f.low = wrap(low, f.field.grid.lowW, f.field.grid.lowH);
        f.optimized = optimized != 0;
        const std::vector<uint8_t> b = encode_glup(f);
        if (b.size() <= cap) std::memcpy(out, b.data(), b.size());
        n = static_cast<long>(b.size());
    });
    return n;
}

// decode_glup (io_glup.cpp:79-139): 0 ok, 1 FormatError (field copied into
// `field`), 2 other exception.  Outputs are written only on success.
int glu_r_decode_glup(const uint8_t* bytes, size_t n, int* dims, float* low, PixelParams* params,
                      char* field, size_t fieldCap) {
    try {
        const GlupFile f = decode_glup(std::vector<uint8_t>(bytes, bytes + n));
        const GridSpec& g = f.field.grid;
        dims[0] = g.highW;
        dims[1] = g.highH;
        dims[2] = g.scale;
        dims[3] = static_cast<int>(f.field.mode);
        dims[4] = f.optimized ? 1 : 0;
        if (low) std::memcpy(low, f.low.data.data(), f.low.data.size() * sizeof(float));
        if (params)
            std::memcpy(params, f.field.params.data(), f.field.params.size() * sizeof(PixelParams));
        return 0;
    } catch (const FormatError& e) {
        std::snprintf(field, fieldCap, "%s", e.field.c_str());
        return 1;
    } catch (const std::exception&) {
        return 2;
    }
}

}  // extern "C"
