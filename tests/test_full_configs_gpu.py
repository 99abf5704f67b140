"""Bitwise parity at the BASELINE.json sizes, against the reference itself.

Every test here compares the CUDA path with ``oracle/_ref`` (the UNMODIFIED
reference sources compiled by oracle/Makefile; the built .so travels to the GPU
box) on the config's own seeded synthetic input:

* C2  joint_optimize 2048x2048, s = 8              (jointopt.cpp:182-206)
* C4  joint_optimize 7680x4320, s = 16             (jointopt.cpp:182-206)
* C5  apply_field of 4 of the 64 colour-mix targets on the C4 JOINT field
      (upsample.cpp:235-252; configs[4])
* C3  one 3840x2160 frame, s = 8, through the frame pipeline in Exact and GNU
      mode (Fast is checked by bench.py's cpu_baseline on every frame and by
      test_parity_gpu.py::test_full_size_properties)

Tolerance: none -- LR images, params, error maps, counts and HR outputs must be
byte-identical.
"""
import numpy as np
import pytest
import torch

from oracle import PARAMS_DTYPE

pytestmark = pytest.mark.gpu


def _host_params(t):
    return t.cpu().numpy().view(PARAMS_DTYPE)[..., 0]


def _same(a, b):
    a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
    return a.nbytes == b.nbytes and a.tobytes() == b.tobytes()


def _first_diff(a, b):
    a = np.ascontiguousarray(a).view(np.uint8).reshape(-1)
    b = np.ascontiguousarray(b).view(np.uint8).reshape(-1)
    d = np.nonzero(a != b)[0]
    return int(d[0]) if d.size else None


@pytest.fixture(scope="module")
def c4(glu, reference):
    """C4 joint solve on both sides (shared by the C4 and C5 tests)."""
    from paper_2307_09582_b200 import workloads
    cfg = workloads.CONFIGS[4]
    img = workloads.scene(cfg["W"], cfg["H"], 4, 0)
    reference.set_num_threads(0)
    want = reference.joint_optimize(img, cfg["scale"])
    got = glu.joint_optimize(torch.from_numpy(img).cuda(), cfg["scale"])
    torch.cuda.synchronize()
    return img, want, got


def _check_joint(want, got):
    assert [got.iterations, got.trialsAccepted, got.trialsRejected] == \
        [want["iterations"], want["accepted"], want["rejected"]]
    assert _same(got.low.cpu().numpy(), want["low"])
    gp = _host_params(got.field.params)
    assert _same(gp, want["field"]), _first_diff(gp, want["field"])
    ge = got.errors.cpu().numpy()
    assert _same(ge, want["errors"]), _first_diff(ge, want["errors"])


def test_c2_joint_matches_reference(glu, reference):
    from paper_2307_09582_b200 import workloads
    cfg = workloads.CONFIGS[2]
    img = workloads.scene(cfg["W"], cfg["H"], 2, 0)
    reference.set_num_threads(0)
    want = reference.joint_optimize(img, cfg["scale"])
    got = glu.joint_optimize(torch.from_numpy(img).cuda(), cfg["scale"])
    assert want["accepted"] + want["rejected"] > 1000  # the trial loop is exercised
    _check_joint(want, got)


def test_c4_joint_matches_reference(c4):
    _, want, got = c4
    assert want["accepted"] + want["rejected"] > 1000
    _check_joint(want, got)


def test_c5_apply_on_c4_joint_field_matches_reference(glu, reference, c4):
    """configs[4]: params = C4's joint PixelParams, targets = seeded channel-mix
    edits of C4's optimised LR image (seeds 1000 + 5 + k); 4 of the 64."""
    from paper_2307_09582_b200 import workloads
    _, want, got = c4
    s = workloads.CONFIGS[4]["scale"]
    for k in (0, 21, 42, 63):
        tgt = glu.op_color(got.low, workloads.mix_op(1005 + k).M)
        t_np = tgt.cpu().numpy()
        out = glu.apply_field(got.field, tgt).cpu().numpy()
        ref = reference.apply_field(want["field"], s, t_np)
        assert _same(out, ref), (k, _first_diff(out, ref))
        # the banded (multi-GPU) apply of the same target tiles the same bytes
        H = got.field.params.shape[0]
        y = (H // 3) // s * s
        band = glu.glu.apply_field_band(got.field.params[y:], got.field.grid, tgt)
        assert _same(band.cpu().numpy(), ref[y:]), k


@pytest.mark.parametrize("mode", ["exact", "gnu"])
def test_c3_frame_matches_reference(glu, reference, mode):
    """One C3 frame (3840x2160, s = 8) through glu_cu_upsample_frames
    (k_frame_prep + the fused solve / 1-channel apply) against the reference's
    grid_downsample -> matte -> optimize_field -> apply_field (matte replicated
    to RGB; channel 0 compared), plus the params through optimize_field."""
    from paper_2307_09582_b200 import workloads
    W, H, s = 3840, 2160, 8
    frame = workloads.scene(W, H, 3, 5)
    md = glu.mode_from_name(mode)
    dev = torch.from_numpy(frame).cuda()
    got = glu.glu.upsample_frames(dev[None], s, "matte", mode=md)[0].cpu().numpy()
    reference.set_num_threads(0)
    low = reference.grid_downsample(frame, s)
    field = reference.optimize_field_allcores(frame, low, s, 3, mode=mode)
    matte = workloads.matte_numpy(low)
    ref = reference.apply_field(field, s, np.repeat(matte[..., None], 3, axis=2))
    want = np.ascontiguousarray(ref[..., 0])
    assert _same(got, want), _first_diff(got, want)
    lo, grid = glu.grid_downsample(dev, s)
    f = glu.optimize_field(dev, lo, grid, None, md)
    gp = _host_params(f.params)
    assert _same(gp, field), _first_diff(gp, field)


def test_beyond_4gib_image_sampled_rows(glu, oracle):
    """A 20480 x 20480 guide (4.7 GiB of RGB fp32, 419 M pixels): byte offsets
    pass 2^31 and 2^32, so every 32-bit index product in the solve, the apply
    and the frame path would show.  grid_downsample is compared whole; the
    solve (Fast), the RGB apply and the video path's fused solve + matte apply
    on LR cell rows around both thresholds and at the edges, each against the
    oracle on a crop of the cell row with its LR neighbours (a pixel's window
    only reaches one LR row either side, so the crop solve is the full solve)."""
    from oracle import low_dims
    from paper_2307_09582_b200 import workloads
    W = H = 20480
    s = 16
    img = workloads.scene(W, H, 41)
    dev = torch.from_numpy(img).cuda()
    low, grid = glu.grid_downsample(dev, s)
    lo = low.cpu().numpy()
    assert _same(lo, oracle.grid_downsample(img, s))
    lw, lh = low_dims(W, H, s)
    field = glu.optimize_field(dev, low, grid)
    rec = glu.apply_field(field, low)
    matte = glu.op_matte(low)
    video = glu.glu.upsample_frames(dev[None], s, "matte")[0]
    # two frames through the batched launch (3-D tensor map; frame 1's guide
    # starts 4.7 GiB in): frame 1 (a mirrored copy) must match its own solve
    mirrored = torch.flip(dev, dims=[1]).contiguous()
    pair = torch.stack([dev, mirrored])
    video2 = glu.glu.upsample_frames(pair, s, "matte")
    del pair
    assert torch.equal(video2[0], video)
    lowm, gridm = glu.grid_downsample(mirrored, s)
    fieldm = glu.optimize_field(mirrored, lowm, gridm)
    assert torch.equal(video2[1], glu.apply_field(fieldm, glu.op_matte(lowm)))
    del video2, fieldm, mirrored
    mat = matte.cpu().numpy()
    # cell rows holding HR rows whose byte offsets cross 2^31 and 2^32
    rows = sorted({0, (2**31 // 12) // W // s, (2**32 // 12) // W // s, lh // 2, lh - 1})
    for cy in rows:
        r0, r1 = max(0, cy - 1), min(lh, cy + 2)  # LR rows of the crop
        y0, y1 = r0 * s, min(H, r1 * s)             # its HR rows
        want = oracle.optimize_field(img[y0:y1], lo[r0:r1], s)
        hy0, hy1 = cy * s - y0, min(H, cy * s + s) - y0  # the cell row inside the crop
        want = want[hy0:hy1]
        got = _host_params(field.params[cy * s:cy * s + (hy1 - hy0)])
        shifted = want.copy()
        shifted["a"] += np.uint32(r0 * lw)
        shifted["b"] += np.uint32(r0 * lw)
        assert _same(got, shifted), (cy, _first_diff(got, shifted))
        ref_rgb = oracle.apply_field(want, lo[r0:r1])
        assert _same(rec[cy * s:cy * s + (hy1 - hy0)].cpu().numpy(), ref_rgb), cy
        ref_m = oracle.apply_field(want, np.repeat(mat[r0:r1, :, None], 3, axis=2))
        assert _same(video[cy * s:cy * s + (hy1 - hy0)].cpu().numpy(),
                     np.ascontiguousarray(ref_m[..., 0])), cy


@pytest.mark.parametrize("mode", ["exact", "gnu"])
def test_beyond_4gib_image_other_modes(glu, oracle, mode):
    """The same 20480 x 20480 guide through optimize_field in Exact and GNU
    mode (k_solve32x, k_solve32f<GNU>), checked on the LR cell row whose HR
    byte offsets cross 2^32 and on the last one."""
    from oracle import low_dims
    from paper_2307_09582_b200 import workloads
    W = H = 20480
    s = 16
    img = workloads.scene(W, H, 43)
    dev = torch.from_numpy(img).cuda()
    low, grid = glu.grid_downsample(dev, s)
    lo = low.cpu().numpy()
    lw, lh = low_dims(W, H, s)
    field = glu.optimize_field(dev, low, grid, None, glu.mode_from_name(mode))
    for cy in ((2**32 // 12) // W // s, lh - 1):
        r0, r1 = max(0, cy - 1), min(lh, cy + 2)
        y0, y1 = r0 * s, min(H, r1 * s)
        want = oracle.optimize_field(img[y0:y1], lo[r0:r1], s, mode=mode)
        hy0, hy1 = cy * s - y0, min(H, cy * s + s) - y0
        want = want[hy0:hy1].copy()
        want["a"] += np.uint32(r0 * lw)
        want["b"] += np.uint32(r0 * lw)
        got = _host_params(field.params[cy * s:cy * s + (hy1 - hy0)])
        assert _same(got, want), (mode, cy, _first_diff(got, want))
