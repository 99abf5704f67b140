// Drop-in C++ API under concurrent host callers (SURVEY 8(b) "Threading"):
// every thread gets its own context and stream (thread_local in glu_api.cpp),
// so optimize_field / apply_field / joint_optimize from several std::threads
// at once give exactly the single-threaded results.
#include <cstdio>
#include <thread>
#include <vector>

#include "glu/grid.hpp"
#include "glu/jointopt.hpp"
#include "glu/upsample.hpp"

using namespace glu;

static ImageF32 scene(int w, int h, unsigned seed) {
    ImageF32 img(w, h);
    unsigned long long x = seed * 0x9E3779B97F4A7C15ull + 1;
    for (size_t i = 0; i < img.data.size(); ++i) {
        x ^= x << 13;
        x ^= x >> 7;
        x ^= x << 17;
        // blocky colour plus a little noise: real components and ties
        const size_t px = i / 3, c = i % 3;
        const int bx = int(px % size_t(w)) / 11, by = int(px / size_t(w)) / 7;
        img.data[i] = float(((bx * 31 + by * 17 + int(c) * 7 + int(seed)) % 23) / 22.0 +
                            double(x % 1000) * 1e-5);
    }
    return img;
}

struct Result {
    std::vector<PixelParams> params;
    std::vector<float> out, low, errors;
    int accepted = 0, rejected = 0;
};

static Result run(unsigned seed) {
    Result r;
    const ImageF32 img = scene(160 + 8 * int(seed % 3), 120, seed);
    GridSpec grid;
    const ImageF32 low = grid_downsample(img, 4, &grid);
    const ParamField f = optimize_field(img, low, grid, GluConfig{}, Mode::Fast);
    r.params = f.params;
    r.out = apply_field(f, low).data;
    const JointResult j = joint_optimize(img, 4, GluConfig{}, Mode::Fast);
    r.low = j.low.data;
    r.errors = j.errors.e;
    r.accepted = j.trialsAccepted;
    r.rejected = j.trialsRejected;
    return r;
}

static bool same(const Result& a, const Result& b) {
    if (a.params.size() != b.params.size()) return false;
    for (size_t i = 0; i < a.params.size(); ++i)
        if (a.params[i].a != b.params[i].a || a.params[i].b != b.params[i].b ||
            a.params[i].w != b.params[i].w)
            return false;
    return a.out == b.out && a.low == b.low && a.errors == b.errors &&
           a.accepted == b.accepted && a.rejected == b.rejected;
}

int main() {
    constexpr int kThreads = 4, kRounds = 3;
    std::vector<Result> want;
    for (int t = 0; t < kThreads; ++t) want.push_back(run(unsigned(t)));
    int fails = 0, trials = 0;
    for (const Result& r : want) trials += r.accepted + r.rejected;
    if (trials == 0) {
        std::fprintf(stderr, "the scenes produced no joint trials\n");
        ++fails;
    }
    for (int round = 0; round < kRounds; ++round) {
        std::vector<Result> got(kThreads);
        std::vector<std::thread> th;
        for (int t = 0; t < kThreads; ++t)
            th.emplace_back([&got, t] { got[t] = run(unsigned(t)); });
        for (auto& x : th) x.join();
        for (int t = 0; t < kThreads; ++t)
            if (!same(got[t], want[t])) {
                std::fprintf(stderr, "round %d thread %d differs\n", round, t);
                ++fails;
            }
    }
    std::printf("%s (%d trials per round)\n", fails ? "FAIL" : "OK", trials);
    return fails ? 1 : 0;
}
