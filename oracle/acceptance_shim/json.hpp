// Minimal stand-in for nlohmann/json.hpp (TEST INFRASTRUCTURE).
//
// The reference's acceptance gate (proj/tests/acceptance/acceptance_main.cpp)
// includes "json.hpp" from its un-vendored proj/vendor/ directory, only for
// criterion 10 (comparing two CLI JSON reports).  The CLI is out of scope
// here, so criterion 10 cannot run; this header lets the file compile
// UNCHANGED, and any attempt to use it throws (reported by the gate as a
// FAIL with the message below, never as a pass).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <vector>

namespace nlohmann {

struct json {
    static json parse(const std::vector<uint8_t>&) {
        throw std::runtime_error("json.hpp stand-in: JSON parsing is not available");
    }
    size_t erase(const char*) { return 0; }
    bool operator==(const json&) const { return false; }
};

}  // namespace nlohmann
