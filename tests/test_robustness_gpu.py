"""Robustness of the CUDA path beyond the reference's own test inputs:
misaligned row-band slices of a field, NaN guide pixels inside joint trials,
and one context shared by several torch streams.  Bit-exact against the
oracle / the single-stream results."""
import numpy as np
import pytest
import torch

from oracle import PARAMS_DTYPE

pytestmark = pytest.mark.gpu


def _host_params(t):
    return t.cpu().numpy().view(PARAMS_DTYPE)[..., 0]


@pytest.mark.parametrize("channels", [1, 3])
@pytest.mark.parametrize("W,s", [(101, 3), (67, 5), (640, 16)])
def test_band_apply_any_row_offset(glu, channels, W, s):
    """glu_cu_apply_field_band on slices starting at every row offset: odd W
    puts the slice's first record mid-quad (not 16-byte aligned); the launcher
    peels the head per pixel (launch_apply) and the bytes equal the full apply."""
    from paper_2307_09582_b200 import workloads
    H = 9 * s + 2
    high = torch.from_numpy(workloads.scene(W, H, 77)).cuda()
    low, grid = glu.grid_downsample(high, s)
    field = glu.optimize_field(high, low, grid)
    tgt = glu.op_matte(low) if channels == 1 else low
    full = glu.apply_field(field, tgt)
    for y0 in range(0, 8):
        for y1 in (y0 + 1, H):
            band = glu.glu.apply_field_band(field.params[y0:y1], grid, tgt)
            assert torch.equal(band, full[y0:y1]), (y0, y1)
    # an output buffer that is 4- but not 16-byte aligned
    buf = torch.empty(full.numel() + 1, device="cuda")
    out = buf[1:].view(full.shape)
    glu.glu.apply_field_band(field.params, grid, tgt, out=out)
    assert torch.equal(out, full)


@pytest.mark.parametrize("mode", ["fast", "exact", "gnu"])
def test_joint_with_nan_guide_pixels_matches_oracle(glu, oracle, mode):
    """NaN guide pixels inside trial footprints: their error is NaN, so the
    reference's `e1 <= e0` (jointopt.cpp:167) is false and the trial is
    rejected even when every error is unchanged (no identical-errors accept
    shortcut on a NaN sum).  Every trial schedule against the oracle."""
    from test_oracle import nan_joint_scene
    img = nan_joint_scene()
    o = oracle.joint_optimize(img, 8, mode=mode)
    ctx = glu.glu.context()
    try:
        for trials in (1, 0, 2):
            ctx.set_trials(trials)
            r = glu.joint_optimize(torch.from_numpy(img).cuda(), 8, None,
                                   glu.mode_from_name(mode))
            assert [r.iterations, r.trialsAccepted, r.trialsRejected] == \
                [o["iterations"], o["accepted"], o["rejected"]], trials
            assert r.low.cpu().numpy().tobytes() == o["low"].tobytes(), trials
            assert _host_params(r.field.params).tobytes() == o["field"].tobytes(), trials
            assert r.errors.cpu().numpy().tobytes() == o["errors"].tobytes(), trials
    finally:
        ctx.set_trials(0)
    assert o["rejected"] > 0


@pytest.mark.parametrize("mode", ["fast", "gnu", "exact"])
def test_joint_with_huge_values_matches_oracle(glu, oracle, mode):
    """Channels near 1e12: the fp32 closed-form objective of the Fast filters
    (k_solve32f's stage B, the trials' filter32k_pixel) would overflow, so
    those pixels must take the double path instead of losing candidates.
    Every trial schedule against the oracle."""
    from paper_2307_09582_b200 import workloads
    rng = np.random.default_rng(11)
    img = workloads.scene(160, 112, 23)
    img[rng.random((112, 160)) < 0.03] *= 1e12
    img = np.ascontiguousarray(img.astype(np.float32))
    o = oracle.joint_optimize(img, 8, mode=mode)
    ctx = glu.glu.context()
    try:
        for trials in (1, 0, 2):
            ctx.set_trials(trials)
            r = glu.joint_optimize(torch.from_numpy(img).cuda(), 8, None,
                                   glu.mode_from_name(mode))
            assert [r.iterations, r.trialsAccepted, r.trialsRejected] == \
                [o["iterations"], o["accepted"], o["rejected"]], trials
            assert r.low.cpu().numpy().tobytes() == o["low"].tobytes(), trials
            assert _host_params(r.field.params).tobytes() == o["field"].tobytes(), trials
            assert r.errors.cpu().numpy().tobytes() == o["errors"].tobytes(), trials
    finally:
        ctx.set_trials(0)
    assert o["accepted"] + o["rejected"] > 0


def test_one_context_many_streams(glu):
    """The per-device context's scratch (packed LR image, NaN flag, trial
    buffers) is shared by every stream it is bound to; binding a new stream
    orders it after the old one (glu_ctx_set_stream), so solves and joint runs
    issued back to back on different torch streams give the one-stream results."""
    from paper_2307_09582_b200 import workloads
    imgs = [torch.from_numpy(workloads.scene(640, 384, 50 + k)).cuda() for k in range(4)]
    want = []
    for im in imgs:
        low, grid = glu.grid_downsample(im, 8)
        want.append((glu.optimize_field(im, low, grid).params.clone(),
                     glu.joint_optimize(im, 8).errors.clone()))
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in range(4)]
    got = []
    for _ in range(3):
        for im, st in zip(imgs, streams):
            with torch.cuda.stream(st):
                low, grid = glu.grid_downsample(im, 8)
                got.append((glu.optimize_field(im, low, grid).params,
                            glu.joint_optimize(im, 8).errors))
    torch.cuda.synchronize()
    for k, (p, e) in enumerate(got):
        assert torch.equal(p, want[k % 4][0]) and torch.equal(e, want[k % 4][1]), k


@pytest.mark.parametrize("clamp", [True, False])
def test_nonfinite_apply_and_error_map_bits_match_reference(glu, reference, clamp):
    """NaN / inf guide pixels reach the LR image, the reconstruction and the
    error map: NaN results must carry the reference host's bits (first NaN
    operand quieted, or the x86 default NaN), not the GPU's canonical NaN."""
    from test_oracle import nonfinite_scene
    img = nonfinite_scene()
    for s in (4, 8):
        high = torch.from_numpy(img).cuda()
        low, grid = glu.grid_downsample(high, s)
        field = glu.optimize_field(high, low, grid)
        P = _host_params(field.params)
        want = reference.apply_field(P, s, low.cpu().numpy(), clamp)
        got = glu.apply_field(field, low, clampOutput=clamp)
        assert got.cpu().numpy().tobytes() == want.tobytes(), (s, clamp)
        e_want = reference.error_map(img, want)
        assert glu.error_map(high, got).cpu().numpy().tobytes() == e_want.tobytes(), s
        if clamp:
            se = glu.self_error_map(high, field, low).cpu().numpy()
            assert se.tobytes() == e_want.tobytes(), s
