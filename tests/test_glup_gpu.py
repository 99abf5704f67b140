"""GLUP parameter files on device buffers against the
reference codec (proj/src/io_glup.cpp, built in oracle/_ref); corruption cases
follow proj/tests/unit/io_test.cpp:196-259."""
import struct

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _sample(glu):
    # io_test.cpp sampleGlup(): a 20x16 field at scale 4 (20 LR cells)
    from paper_2307_09582_b200 import workloads
    img = torch.from_numpy(workloads.scene(20, 16, 77)).cuda()
    low, grid = glu.grid_downsample(img, 4)
    field = glu.optimize_field(img, low, grid, None, glu.Mode.Exact)
    return field, low


def test_encode_matches_reference_bytes(glu, reference):
    field, low = _sample(glu)
    ours = bytes(glu.glu.encode_glup(field, low, optimized=True).numpy())
    ref = reference.encode_glup(field.numpy(), low.cpu().numpy(), 4, mode=1, optimized=True)
    assert len(ours) == 32 + 12 * 20 + 12 * 320 == len(ref)
    assert ours == ref


def test_round_trip_bitwise(glu):
    field, low = _sample(glu)
    data = glu.glu.encode_glup(field, low)
    f2, low2, opt = glu.glu.decode_glup(data)
    assert f2.grid == field.grid and f2.mode == field.mode and not opt
    assert torch.equal(f2.params, field.params) and torch.equal(low2, low)
    # device-resident bytes decode the same way
    f3, low3, _ = glu.glu.decode_glup(data.cuda())
    assert torch.equal(f3.params, field.params) and torch.equal(low3, low)


def _put(b, off, v):
    b[off:off + 4] = struct.pack("<I", v)


def test_corruption_names_the_field_like_the_reference(glu, reference):
    field, low = _sample(glu)
    good = bytearray(bytes(glu.glu.encode_glup(field, low).numpy()))
    params = 32 + 12 * 20
    cases = []
    b = bytearray(good); b[0] = ord("X"); cases.append((b, "magic"))
    b = bytearray(good); b[4] = 2; cases.append((b, "version"))
    cases.append((good[:31], "length"))
    cases.append((good[:-1], "length"))
    cases.append((good + b"\0", "length"))
    b = bytearray(good); _put(b, 8, 0); cases.append((b, "dims"))
    b = bytearray(good); _put(b, 16, 16); cases.append((b, "dims"))
    b = bytearray(good); _put(b, 20, 6); cases.append((b, "dims"))
    b = bytearray(good); b[28] = 3; cases.append((b, "mode"))
    b = bytearray(good); b[29] = 2; cases.append((b, "flag"))
    b = bytearray(good); b[30] = 1; cases.append((b, "reserved"))
    b = bytearray(good); _put(b, 32, 0x7FC00000); cases.append((b, "lowres"))
    b = bytearray(good); _put(b, 32, 0x3FC00000); cases.append((b, "lowres"))
    b = bytearray(good); _put(b, params, 20); cases.append((b, "index"))
    b = bytearray(good); _put(b, params + 8, 0x7FC00000); cases.append((b, "weight"))
    # first violation in the reference's order wins: a bad weight before a bad index
    b = bytearray(good); _put(b, params + 8, 0x7FC00000); _put(b, params + 24, 99)
    cases.append((b, "weight"))
    cases.append((bytearray(), "length"))
    for data, want in cases:
        ok, fld, _ = reference.decode_glup(bytes(data))
        assert not ok and fld == want
        with pytest.raises(glu.glu.FormatError) as ei:
            glu.glu.decode_glup(bytes(data))
        assert ei.value.field == want, (want, ei.value.field, str(ei.value))


def test_encode_validates_input(glu):
    field, low = _sample(glu)
    with pytest.raises(ValueError):
        glu.glu.encode_glup(field, torch.zeros((3, 3, 3), device="cuda"))


def test_cpp_dropin_io_api(glu, tmp_path):
    """include/glu/io.hpp through lib/libglu.so from a C++ program."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    lib = os.path.join(root, "paper_2307_09582_b200", "lib")
    exe = tmp_path / "dropin_io_test"
    subprocess.run(["g++", "-std=c++20", "-O1", "-I" + os.path.join(root, "include"),
                    os.path.join(root, "tests", "cpp", "dropin_io_test.cpp"), "-L" + lib,
                    "-lglu", "-lglu_cuda", "-Wl,-rpath," + lib, "-o", str(exe)], check=True)
    r = subprocess.run([str(exe), str(tmp_path / "x.glup")], capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr


def test_dropin_api_concurrent_host_threads(tmp_path):
    """The drop-in C++ API from four std::threads at once (thread-local contexts
    and streams) gives the single-threaded results bit for bit: optimize_field,
    apply_field and joint_optimize (SURVEY 8(b) threading contract)."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    lib = os.path.join(root, "paper_2307_09582_b200", "lib")
    exe = tmp_path / "dropin_threads_test"
    subprocess.run(["g++", "-std=c++20", "-O1", "-I" + os.path.join(root, "include"),
                    os.path.join(root, "tests", "cpp", "dropin_threads_test.cpp"), "-L" + lib,
                    "-lglu", "-lglu_cuda", "-Wl,-rpath," + lib, "-pthread", "-o", str(exe)],
                   check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout + r.stderr
