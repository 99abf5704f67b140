// Drop-in C++ API smoke for the GLUP codec (include/glu/io.hpp): round trip
// through encode/decode and disk, and FormatError field names on corruption
// (the cases of proj/tests/unit/io_test.cpp:166-269, restated).
#include <cstdio>
#include <cstring>

#include "glu/grid.hpp"
#include "glu/io.hpp"
#include "glu/upsample.hpp"

using namespace glu;

static int fails = 0;
#define EXPECT(c)                                                  \
    do {                                                           \
        if (!(c)) {                                                \
            std::fprintf(stderr, "%s:%d: %s\n", __FILE__, __LINE__, #c); \
            ++fails;                                               \
        }                                                          \
    } while (0)

static void put32(std::vector<uint8_t>& b, size_t off, uint32_t v) {
    for (int k = 0; k < 4; ++k) b[off + k] = uint8_t(v >> (8 * k));
}

static std::string fieldOf(const std::vector<uint8_t>& b) {
    try {
        decode_glup(b);
    } catch (const FormatError& e) {
        return e.field;
    }
    return "";
}

int main(int argc, char** argv) {
    ImageF32 img(20, 16);
    for (size_t i = 0; i < img.data.size(); ++i) img.data[i] = float((i * 37) % 101) / 100.0f;
    GridSpec grid;
    const ImageF32 low = grid_downsample(img, 4, &grid);
    GlupFile f;
    f.field = optimize_field(img, low, grid, GluConfig{}, Mode::Fast);
    f.low = low;
    f.optimized = true;
    const std::vector<uint8_t> bytes = encode_glup(f);
    EXPECT(bytes.size() == 32 + 12 * 20 + 12 * 320);
    const GlupFile g = decode_glup(bytes);
    EXPECT(g.field.grid.highW == 20 && g.field.grid.highH == 16 && g.field.grid.scale == 4);
    EXPECT(g.optimized && g.field.mode == Mode::Fast);
    EXPECT(std::memcmp(g.field.params.data(), f.field.params.data(), 320 * 12) == 0);
    EXPECT(std::memcmp(g.low.data.data(), f.low.data.data(), 60 * 4) == 0);
    const std::string path = argc > 1 ? argv[1] : "/tmp/glu_dropin.glup";
    write_glup(path, f);
    const GlupFile h = read_glup(path);
    EXPECT(std::memcmp(h.field.params.data(), f.field.params.data(), 320 * 12) == 0);
    std::remove(path.c_str());
    bool threw = false;
    try {
        read_glup(path);
    } catch (const IoError&) {
        threw = true;
    }
    EXPECT(threw);
    std::vector<uint8_t> b = bytes;
    b[0] = 'X';
    EXPECT(fieldOf(b) == "magic");
    b = bytes;
    b.pop_back();
    EXPECT(fieldOf(b) == "length");
    b = bytes;
    put32(b, 16, 16);
    EXPECT(fieldOf(b) == "dims");
    b = bytes;
    put32(b, 32, 0x3fc00000u);
    EXPECT(fieldOf(b) == "lowres");
    b = bytes;
    put32(b, 272, 20);
    EXPECT(fieldOf(b) == "index");
    b = bytes;
    put32(b, 280, 0x7fc00000u);
    EXPECT(fieldOf(b) == "weight");
    EXPECT(fieldOf({}) == "length");
    threw = false;
    try {
        GlupFile bad = f;
        bad.field.params.pop_back();
        encode_glup(bad);
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    EXPECT(threw);
    std::printf("dropin_io_test: %s\n", fails ? "FAILED" : "ok");
    return fails ? 1 : 0;
}
