"""The drop-in boundary, checked without a GPU: the C-ABI library loads and
exports every symbol include/glu_cuda.h declares; host-only validation returns
the reference's std::invalid_argument texts; contexts fail cleanly (no CPU
fallback) when no device is visible."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "glu_cuda.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(glu_\w+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    from paper_2307_09582_b200 import _native, build
    if not os.path.exists(_native.LIB_PATH):
        build.build()
    return _native.lib()


def test_every_declared_symbol_is_exported(lib):
    from paper_2307_09582_b200 import _native
    syms = header_symbols()
    assert len(syms) >= 40
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_native.SIGNATURES), set(syms) ^ set(_native.SIGNATURES)


def test_cpp_api_library_exports_reference_signatures():
    from paper_2307_09582_b200 import build
    if not os.path.exists(build.CPP_SO):
        build.build()
    out = os.popen(f"nm -DC --defined-only {build.CPP_SO}").read()
    for sig in [
        "glu::optimize_field(glu::ImageF32 const&, glu::ImageF32 const&, glu::GridSpec const&, "
        "glu::GluConfig const&, glu::Mode)",
        "glu::optimize_pixels(glu::ImageF32 const&, glu::ImageF32 const&, glu::GridSpec const&, "
        "glu::GluConfig const&, glu::Mode, std::span<unsigned int const, 18446744073709551615ul>, "
        "glu::ParamField&)",
        "glu::apply_field(glu::ParamField const&, glu::ImageF32 const&, bool)",
        "glu::error_map(glu::ImageF32 const&, glu::ImageF32 const&)",
        "glu::grid_downsample(glu::ImageF32 const&, int, glu::GridSpec*)",
        "glu::find_large_error(glu::ErrorMap const&, float)",
        "glu::joint_optimize(glu::ImageF32 const&, int, glu::GluConfig const&, glu::Mode)",
        "glu::weight_exact(std::array<float, 3ul>, std::array<float, 3ul>, "
        "std::array<float, 3ul>, double)",
    ]:
        assert sig in out, sig


def test_abi_version_and_build_info(lib):
    assert lib.glu_abi_version() == 1
    assert b"sm_100a" in lib.glu_build_info()


def test_grid_create_matches_reference(lib):
    from paper_2307_09582_b200 import _native
    g = _native.GluGrid()
    assert lib.glu_grid_create(17, 17, 8, C.byref(g)) == 0
    assert (g.lowW, g.lowH, g.sampleOffset) == (3, 3, 4)  # grid_test.cpp:24-34
    assert lib.glu_grid_create(17, 16, 15, C.byref(g)) == 0 and g.lowW == 2
    for args, msg in [((16, 16, 1), b"scale must be >= 2"),
                      ((16, 16, 16), b"scale must be < min(width, height)"),
                      ((16, 32, 16), b"scale must be < min(width, height)"),
                      ((0, 16, 2), b"dimensions must be positive")]:
        assert lib.glu_grid_create(*args, C.byref(g)) == 1
        assert msg in lib.glu_last_error()


def test_config_validate_messages(lib):
    from paper_2307_09582_b200 import _native
    c = lib.glu_config_default()
    assert (c.windowSide, c.maxIterations) == (3, 3)
    assert abs(c.errorThreshold - 30 / 255) < 1e-7 and abs(c.epsilon - 1e-3) < 1e-10
    assert lib.glu_config_validate(C.byref(c)) == 0
    for field, val, msg in [("windowSide", 4, b"windowSide must be odd and >= 3"),
                            ("windowSide", 1, b"windowSide must be odd and >= 3"),
                            ("errorThreshold", -1.0, b"errorThreshold must be >= 0"),
                            ("maxIterations", -1, b"maxIterations must be >= 0"),
                            ("epsilon", 0.0, b"epsilon must be > 0")]:
        bad = _native.GluConfigC(c.windowSide, c.errorThreshold, c.maxIterations, c.epsilon, 0)
        setattr(bad, field, val)
        assert lib.glu_config_validate(C.byref(bad)) == 1
        assert msg in lib.glu_last_error()


def test_python_mirror_validation():
    import paper_2307_09582_b200 as glu
    assert glu.GridSpec.create(17, 17, 8).sampleCoord(2, 0) == (16, 4)
    with pytest.raises(ValueError, match="unknown mode"):
        glu.mode_from_name("bogus")
    assert glu.neighborhood(9, 5, glu.GridSpec.create(10, 10, 2), 5) == [
        cy * 5 + cx for cy in range(0, 5) for cx in range(2, 5)]  # grid_test.cpp:88-97
    with pytest.raises(ValueError):
        glu.neighborhood(0, 0, glu.GridSpec.create(20, 20, 2), 4)


def test_no_cpu_fallback_without_gpu(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    h = C.c_void_p()
    assert lib.glu_ctx_create(0, C.byref(h)) == 2
    assert b"no CUDA device" in lib.glu_last_error()
    import paper_2307_09582_b200 as glu
    with pytest.raises(Exception):
        glu.glu.context()


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2307_09582_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "glu_oracle" not in txt and "libglu_ref" not in txt, f


def test_cpp_dropin_validation_without_gpu(tmp_path):
    """Host-side validation of the drop-in C++ API (tests/cpp/
    dropin_validation_test.cpp): the reference's std::invalid_argument texts,
    thrown before any device work -- including a field of the wrong size in
    trial_update_component, which must not reach the size-based host copy."""
    import subprocess
    from paper_2307_09582_b200 import build
    if not os.path.exists(build.CPP_SO):
        build.build()
    lib = os.path.dirname(build.CPP_SO)
    exe = tmp_path / "dropin_validation_test"
    subprocess.run(["g++", "-std=c++20", "-O1", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "dropin_validation_test.cpp"),
                    "-L" + lib, "-lglu", "-lglu_cuda", "-Wl,-rpath," + lib, "-o", str(exe)],
                   check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout + r.stderr
