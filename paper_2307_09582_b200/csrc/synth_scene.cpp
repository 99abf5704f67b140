// synth_scene.cpp -- seeded synthetic workloads for BASELINE.json's configs.
//
// Host-side harness code (not on the hot path): builds the guide images that
// the tests and bench.py feed to both the CUDA path and the CPU checkers, so
// generator parity across devices is never needed.  All randomness is the
// reference's SplitMix64 (proj/include/glu/synth.hpp:12-34), restated here.
//
// Scene (BASELINE.json configs[0]): 64 Voronoi regions, seeds uniform over the
// image; region colour = base U[0,1]^3 + per-channel slope U[-0.5,0.5] * (x -
// seed_x) / W; 200 one-pixel lines (start uniform, angle U[0,2pi), length
// U[10,200], colour U[0,1]^3, DDA raster); Gaussian noise sigma 0.01; clamp.
// Video (configs[2]): per frame, every Voronoi seed drifts 2 px along its own
// random direction and every line translates rigidly 2 px along its own
// direction; noise is fresh per frame.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <thread>
#include <vector>

namespace {

struct SplitMix64 {
    uint64_t state;
    explicit SplitMix64(uint64_t s) : state(s) {}
    uint64_t next() {
        state += 0x9e3779b97f4a7c15ull;
        uint64_t z = state;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        return z ^ (z >> 31);
    }
    double uniform() { return double(next() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
};

constexpr double kTwoPi = 6.283185307179586;

struct Region {
    double x, y, dx, dy;
    float base[3], slope[3];
};

struct Line {
    double x0, y0, ang, len, dx, dy;
    float color[3];
};

template <typename F>
void parallel_rows(int H, int threads, F&& fn) {
    if (threads <= 0) threads = static_cast<int>(std::thread::hardware_concurrency());
    threads = std::max(1, std::min(threads, H));
    const int chunk = (H + threads - 1) / threads;
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) {
        const int y0 = t * chunk, y1 = std::min(H, y0 + chunk);
        if (y0 < y1) pool.emplace_back([&fn, y0, y1] { fn(y0, y1); });
    }
    for (auto& th : pool) th.join();
}

}  // namespace

extern "C" {

// Writes W*H*3 floats (interleaved RGB, [0,1]) for frame `frame` of scene `seed`.
int glu_synth_scene(int W, int H, unsigned long long seed, int frame, int threads, float* out) {
    if (W <= 0 || H <= 0 || !out) return 1;
    SplitMix64 rng(seed);
    std::vector<Region> regions(64);
    for (Region& r : regions) {
        r.x = rng.uniform(0, W);
        r.y = rng.uniform(0, H);
        const double a = rng.uniform(0, kTwoPi);
        r.dx = 2.0 * std::cos(a);
        r.dy = 2.0 * std::sin(a);
        for (int c = 0; c < 3; ++c) r.base[c] = static_cast<float>(rng.uniform());
        for (int c = 0; c < 3; ++c) r.slope[c] = static_cast<float>(rng.uniform(-0.5, 0.5));
        r.x += frame * r.dx;
        r.y += frame * r.dy;
    }
    std::vector<Line> lines(200);
    for (Line& l : lines) {
        l.x0 = rng.uniform(0, W);
        l.y0 = rng.uniform(0, H);
        l.ang = rng.uniform(0, kTwoPi);
        l.len = rng.uniform(10, 200);
        for (int c = 0; c < 3; ++c) l.color[c] = static_cast<float>(rng.uniform());
        const double a = rng.uniform(0, kTwoPi);
        l.dx = 2.0 * std::cos(a);
        l.dy = 2.0 * std::sin(a);
        l.x0 += frame * l.dx;
        l.y0 += frame * l.dy;
    }
    const uint64_t noiseSeed = seed * 0x100000001b3ull + static_cast<uint64_t>(frame) + 1;

    // Voronoi + gradient, nearest seed by squared distance, ties -> lower index.
    // Per 32x32 tile only seeds that can be nearest somewhere in the tile are
    // scanned (min distance to the tile <= smallest max distance over seeds),
    // in index order, so the result equals the brute-force scan.
    constexpr int kT = 32;
    parallel_rows((H + kT - 1) / kT, threads, [&](int t0, int t1) {
        int cand[64];
        for (int ty = t0; ty < t1; ++ty) {
            for (int tx = 0; tx < (W + kT - 1) / kT; ++tx) {
                const double x0 = tx * kT, y0 = ty * kT;
                const double x1 = std::min(W, (tx + 1) * kT) - 1.0;
                const double y1 = std::min(H, (ty + 1) * kT) - 1.0;
                double m = 1e300;
                double dmin[64];
                for (int k = 0; k < 64; ++k) {
                    const Region& r = regions[k];
                    const double nx = std::clamp(r.x, x0, x1), ny = std::clamp(r.y, y0, y1);
                    dmin[k] = (nx - r.x) * (nx - r.x) + (ny - r.y) * (ny - r.y);
                    const double fx = std::max(std::fabs(r.x - x0), std::fabs(r.x - x1));
                    const double fy = std::max(std::fabs(r.y - y0), std::fabs(r.y - y1));
                    m = std::min(m, fx * fx + fy * fy);
                }
                int nc = 0;
                for (int k = 0; k < 64; ++k)
                    if (dmin[k] <= m * (1 + 1e-12) + 1e-9) cand[nc++] = k;
                for (int y = int(y0); y <= int(y1); ++y) {
                    for (int x = int(x0); x <= int(x1); ++x) {
                        int best = cand[0];
                        double bd = 1e300;
                        for (int i = 0; i < nc; ++i) {
                            const int k = cand[i];
                            const double dx = x - regions[k].x, dy = y - regions[k].y;
                            const double d = dx * dx + dy * dy;
                            if (d < bd) {
                                bd = d;
                                best = k;
                            }
                        }
                        const Region& r = regions[best];
                        float* o = out + 3 * (static_cast<size_t>(y) * W + x);
                        const double t = (x - r.x) / W;
                        for (int c = 0; c < 3; ++c)
                            o[c] = static_cast<float>(r.base[c] + r.slope[c] * t);
                    }
                }
            }
        }
    });
    // One-pixel lines, DDA with max(|dx|,|dy|) steps, clipped.
    for (const Line& l : lines) {
        const double ex = l.x0 + l.len * std::cos(l.ang), ey = l.y0 + l.len * std::sin(l.ang);
        const int steps = static_cast<int>(std::ceil(std::max(std::fabs(ex - l.x0),
                                                              std::fabs(ey - l.y0))));
        for (int i = 0; i <= steps; ++i) {
            const double t = steps ? double(i) / steps : 0.0;
            const int x = static_cast<int>(std::lround(l.x0 + t * (ex - l.x0)));
            const int y = static_cast<int>(std::lround(l.y0 + t * (ey - l.y0)));
            if (x < 0 || y < 0 || x >= W || y >= H) continue;
            float* o = out + 3 * (static_cast<size_t>(y) * W + x);
            for (int c = 0; c < 3; ++c) o[c] = l.color[c];
        }
    }
    // Gaussian noise (Box-Muller over a per-row SplitMix64 stream), clamp.
    parallel_rows(H, threads, [&](int y0, int y1) {
        for (int y = y0; y < y1; ++y) {
            SplitMix64 nr(noiseSeed ^ (static_cast<uint64_t>(y) * 0xd1b54a32d192ed03ull));
            float* row = out + 3 * static_cast<size_t>(y) * W;
            for (int i = 0; i < 3 * W; i += 2) {
                const double u1 = 1.0 - nr.uniform(), u2 = nr.uniform();
                const double rad = std::sqrt(-2.0 * std::log(u1));
                const double n0 = 0.01 * rad * std::cos(kTwoPi * u2);
                const double n1 = 0.01 * rad * std::sin(kTwoPi * u2);
                row[i] = static_cast<float>(std::clamp(row[i] + n0, 0.0, 1.0));
                if (i + 1 < 3 * W)
                    row[i + 1] = static_cast<float>(std::clamp(row[i + 1] + n1, 0.0, 1.0));
            }
        }
    });
    return 0;
}

}  // extern "C"
