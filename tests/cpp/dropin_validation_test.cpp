// Host-side validation of the drop-in C++ API, runnable without a GPU: every
// check below throws std::invalid_argument with the reference's message
// before any device work (no context is created).
//   trial_update_component with a field of the wrong size: the reference
//   throws "optimize_pixels: field does not match image" (upsample.cpp:222-223)
//   once its re-solve is reached; the drop-in copies the field by size, so it
//   must refuse up front instead of overflowing the host vector.
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "glu/grid.hpp"
#include "glu/jointopt.hpp"
#include "glu/upsample.hpp"

using namespace glu;

static int failures = 0;

template <typename F>
static void expect_invalid(const char* what, const char* msg, F&& f) {
    try {
        f();
        std::printf("FAIL %s: no exception\n", what);
        ++failures;
    } catch (const std::invalid_argument& e) {
        if (std::strstr(e.what(), msg) == nullptr) {
            std::printf("FAIL %s: message '%s'\n", what, e.what());
            ++failures;
        }
    }
}

int main() {
    ImageF32 high(32, 24, {0.5f, 0.25f, 0.75f});
    GridSpec grid;
    ImageF32 low(8, 6, {0.5f, 0.25f, 0.75f});
    grid = GridSpec::create(32, 24, 4);
    ParamField field;
    field.grid = grid;
    field.params.resize(10);  // wrong size
    ErrorMap errors;
    errors.width = 32;
    errors.height = 24;
    errors.e.assign(32 * 24, 1.0f);
    const std::vector<uint32_t> comp = {0, 1, 2};
    expect_invalid("field size", "optimize_pixels: field does not match image", [&] {
        trial_update_component(high, low, field, errors, comp, GluConfig{}, Mode::Fast);
    });
    field.params.resize(32 * 24);
    expect_invalid("empty component", "trial_update_component: empty component", [&] {
        trial_update_component(high, low, field, errors, {}, GluConfig{}, Mode::Fast);
    });
    errors.e.resize(7);
    expect_invalid("error vector size", "trial_update_component: shape mismatch", [&] {
        trial_update_component(high, low, field, errors, comp, GluConfig{}, Mode::Fast);
    });
    errors.e.resize(32 * 24);
    ImageF32 wrongLow(7, 6);
    expect_invalid("low dims", "trial_update_component: shape mismatch", [&] {
        trial_update_component(high, wrongLow, field, errors, comp, GluConfig{}, Mode::Fast);
    });
    GluConfig bad;
    bad.windowSide = 4;
    expect_invalid("config", "windowSide must be odd", [&] {
        trial_update_component(high, low, field, errors, comp, bad, Mode::Fast);
    });
    if (failures == 0) std::printf("OK\n");
    return failures;
}
