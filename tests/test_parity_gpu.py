"""Parity of the CUDA path (through the C-ABI) with the reference.

Bit-exact against the reference's golden vectors and against the pinned oracle
on fresh seeded inputs; size-independent properties at BASELINE sizes.
Tolerance: none -- indices, weights, images and error maps must match
bit for bit (stronger than north_star's 1e-5 / 1e-4 bars).
"""
import numpy as np
import pytest
import torch

from oracle import EPS_DEFAULT, PARAMS_DTYPE, TAU_DEFAULT

pytestmark = pytest.mark.gpu

SOLVES = ["mix67x45_s4", "mix41x33_s4", "photo40x28_s4", "mix37x29_s4_S5", "mix50x38_s3_S7",
          "mix45x45_s5_S9", "mix33x21_s2", "scene96x64_s8", "scene100x70_s16"]
JOINTS = ["joint_missed_line", "joint_missed_line_literal", "joint_mix72x60_s6",
          "joint_mix64x56_s8", "joint_mix48_s6_tau05", "joint_mix128_s8", "joint_mix60x52_s4_S5",
          "joint_scene160x96_s8", "joint_harmful"]


def dev(a):
    a = np.ascontiguousarray(a)
    if a.dtype == PARAMS_DTYPE:
        a = a.view(np.int32).reshape(a.shape + (3,))
    elif a.dtype == np.uint32:
        a = a.view(np.int32)
    return torch.from_numpy(a.copy()).cuda()


def host_params(t):
    return t.cpu().numpy().view(PARAMS_DTYPE)[..., 0]


def same(a, b):
    a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
    return a.nbytes == b.nbytes and a.tobytes() == b.tobytes()


def mode_of(glu, m):
    return glu.mode_from_name(m)


@pytest.mark.parametrize("name", SOLVES)
def test_solve_apply_error_golden(glu, golden, name):
    img, (s, S) = golden[f"{name}/high"], golden[f"{name}/meta"]
    high = dev(img)
    low, grid = glu.grid_downsample(high, int(s))
    assert same(low.cpu().numpy(), golden[f"{name}/low"])
    cfg = glu.GluConfig(windowSide=int(S))
    for m in ("fast", "exact", "gnu"):
        field = glu.optimize_field(high, low, grid, cfg, mode_of(glu, m))
        want = golden[f"{name}/params_{m}"]
        got = host_params(field.params)
        assert same(got, want), (m, int((got != want.view(PARAMS_DTYPE).reshape(
            got.shape)).sum()))
        rec = glu.apply_field(field, low)
        assert same(rec.cpu().numpy(), golden[f"{name}/apply_{m}"]), m
        assert same(glu.error_map(high, rec).cpu().numpy(), golden[f"{name}/errors_{m}"]), m
        assert same(glu.self_error_map(high, field, low).cpu().numpy(),
                    golden[f"{name}/errors_{m}"]), m
        out, pf = glu.solve_apply(high, low, grid, low, cfg, mode_of(glu, m), keep_params=True)
        assert same(out.cpu().numpy(), golden[f"{name}/apply_{m}"]), m
        assert same(host_params(pf.params), want), m
    field = glu.optimize_field(high, low, grid, cfg, glu.Mode.Fast)
    half = glu.apply_field(field, low * 0.5, clampOutput=False)
    assert same(half.cpu().numpy(), golden[f"{name}/apply_fast_noclamp_half"])


@pytest.mark.parametrize("name", JOINTS)
def test_joint_golden(glu, golden, name):
    img, (s, S, lit) = golden[f"{name}/high"], golden[f"{name}/meta"]
    tau = float(golden[f"{name}/tau"][0])
    cfg = glu.GluConfig(windowSide=int(S), errorThreshold=tau, literalComponentUpdate=bool(lit))
    modes = ("fast", "exact", "gnu") if name == "joint_mix72x60_s6" else ("fast",)
    for m in modes:
        r = glu.joint_optimize(dev(img), int(s), cfg, mode_of(glu, m))
        key = f"{name}/{m}"
        assert [r.iterations, r.trialsAccepted, r.trialsRejected] == \
            golden[f"{key}/counts"].tolist(), m
        assert same(r.low.cpu().numpy(), golden[f"{key}/low"]), m
        assert same(host_params(r.field.params), golden[f"{key}/params"]), m
        assert same(r.errors.cpu().numpy(), golden[f"{key}/errors"]), m


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_trial_sequence_golden(glu, golden, seed):
    """Per-trial verdicts, bitwise rollback (jointopt_test.cpp:76-109)."""
    img = golden[f"trials_mix48_{seed}/high"]
    s = 6
    cfg = glu.GluConfig(errorThreshold=0.05)
    high = dev(img)
    low, grid = glu.grid_downsample(high, s)
    field = glu.optimize_field(high, low, grid, cfg)
    errors = glu.error_map(high, glu.apply_field(field, low))
    les = glu.find_large_error(errors, 0.05)
    verdicts = []
    for comp in les.components:
        before = (low.clone(), field.params.clone(), errors.clone())
        ok = glu.trial_update_component(high, low, field, errors, comp, cfg)
        verdicts.append(ok)
        if not ok:
            assert torch.equal(low, before[0]) and torch.equal(field.params, before[1])
            assert torch.equal(errors, before[2])
    assert verdicts == golden[f"trials_mix48_{seed}/verdicts"].astype(bool).tolist()
    assert same(low.cpu().numpy(), golden[f"trials_mix48_{seed}/low"])
    assert same(host_params(field.params), golden[f"trials_mix48_{seed}/params"])
    assert same(errors.cpu().numpy(), golden[f"trials_mix48_{seed}/errors"])


@pytest.mark.parametrize("name", ["ccl_pin", "ccl_scene"])
def test_find_large_error_golden(glu, golden, name):
    les = glu.find_large_error(dev(golden[f"{name}/errors"]), float(golden[f"{name}/tau"][0]))
    assert same(les.mask.cpu().numpy(), golden[f"{name}/mask"])
    assert same(les.offsets.cpu().numpy().astype(np.uint32), golden[f"{name}/offsets"])
    assert same(les.pixels.cpu().numpy().view(np.uint32), golden[f"{name}/pixels"])


@pytest.mark.parametrize("mode", ["fast", "exact", "gnu"])
def test_pixel_batch_golden(glu, golden, mode):
    ip, rgb, idx, off = (golden[f"pixels/{k}"] for k in ("ip", "rgb", "idx", "off"))
    cands = [(idx[off[k]:off[k + 1]], rgb[off[k]:off[k + 1]]) for k in range(len(ip))]
    got = glu.optimize_pixel_batch(ip, cands, 1e-3, mode_of(glu, mode))
    assert same(got.view(np.uint32).reshape(-1, 3), golden[f"pixels/{mode}"])


def test_scalar_pins(glu):
    # upsample_test.cpp:39-63, 134-159, 178-189
    assert glu.weight_exact([0.25, 0, 0], [1, 0, 0], [0, 0, 0], 1e-3) == pytest.approx(
        0.25 / 1.001, rel=1e-9)
    assert glu.weight_fast([0.5] * 3, [1] * 3, [0] * 3, 1e-3) == pytest.approx(0.4997, rel=1e-4)
    rng = np.random.default_rng(424242)
    w = glu.weight_fast(rng.random((5000, 3)), rng.random((5000, 3)), rng.random((5000, 3)), 1e-3)
    assert (w >= 0).all() and (w < 1).all()
    p = glu.optimize_pixel_exact([0.9, 0.1, 0.5], (np.arange(6) + 40,
                                                   np.tile([0.3, 0.7, 0.2], (6, 1))), 1e-3)
    assert (int(p["a"]), int(p["b"]), float(p["w"])) == (40, 40, 0.0)
    p = glu.optimize_pixel_exact([1.0] * 3, ([0, 1], [[0.8] * 3, [0.4] * 3]), 1e-3)
    assert float(p["w"]) > 1.0
    with pytest.raises(ValueError):
        glu.optimize_pixel_gnu([0, 0, 0], ([], np.zeros((0, 3))))


CASES = [  # (W, H, s, S, seed): ragged sizes, every supported window class
    (131, 77, 4, 3, 11), (200, 120, 8, 3, 12), (97, 203, 3, 5, 13), (160, 90, 5, 7, 14),
    (64, 64, 2, 9, 15), (257, 129, 16, 3, 16), (33, 300, 6, 11, 17),
    # degenerate geometries: 2 x N / N x 2 LR grids, one-cell-wide LR, scale 32,
    # tiles narrower than a warp, windows wider than the LR grid
    (33, 5, 4, 3, 18), (7, 300, 3, 5, 19), (1000, 9, 8, 3, 20), (257, 129, 32, 5, 21),
    (5, 5, 2, 3, 22), (17, 200, 16, 7, 23), (96, 64, 2, 3, 24),
    # the exact kernel's tile shapes: s = 3 (one row per thread, 12 x 4 owner
    # cells per tile) and a larger s = 5 / s = 7 frame (several rows per thread)
    (301, 211, 3, 3, 25), (1203, 1001, 5, 3, 26), (1500, 700, 7, 3, 27),
    # k_solve32f's tile shapes at the extremes: s = 32 (5 x 3 LR grid), a 40 x 3
    # image at s = 2 (one tile row, 2-row LR grid)
    (129, 77, 32, 3, 28), (40, 3, 2, 3, 29),
    # the pair-table path (packed fp32 pairs) at every compile-time pitch and
    # its edges: s = 8 / 9 / 10 (pitch 7), 11 / 15 (generic), 16 / 17 / 31
    # (pitch 5), 33 / 40 (pitch 4); widths off the 32-pixel tile, heights off
    # the tile rows, LR grids narrower than the pitch
    (333, 219, 9, 3, 30), (650, 411, 10, 3, 31), (407, 230, 11, 3, 32), (500, 300, 15, 3, 33),
    (523, 389, 17, 3, 34), (700, 500, 31, 3, 35), (431, 303, 33, 3, 36), (90, 650, 40, 3, 37),
    (27, 500, 8, 3, 38), (1040, 17, 8, 3, 39), (47, 49, 16, 3, 40),
]


@pytest.mark.parametrize("W,H,s,S,seed", CASES)
def test_solve_vs_oracle_seeded(glu, oracle, W, H, s, S, seed):
    from paper_2307_09582_b200 import workloads
    img = workloads.scene(W, H, seed)
    high = dev(img)
    low, grid = glu.grid_downsample(high, s)
    lo = oracle.grid_downsample(img, s)
    assert same(low.cpu().numpy(), lo)
    for m in ("fast", "exact", "gnu"):
        f = glu.optimize_field(high, low, grid, glu.GluConfig(windowSide=S), mode_of(glu, m))
        want = oracle.optimize_field(img, lo, s, S, EPS_DEFAULT, m)
        assert same(host_params(f.params), want), m


def test_optimize_pixels_matches_field(glu):
    # upsample_test.cpp:226-237: sparse re-solve of every pixel == optimize_field
    from paper_2307_09582_b200 import workloads
    img = dev(workloads.scene(123, 77, 5))
    low, grid = glu.grid_downsample(img, 4)
    full = glu.optimize_field(img, low, grid)
    sparse = full.clone()
    sparse.params.fill_(-1)
    order = torch.randperm(123 * 77, device="cuda").to(torch.int32)
    glu.optimize_pixels(img, low, grid, None, glu.Mode.Fast, order, sparse)
    assert torch.equal(full.params, sparse.params)


def test_single_channel_apply_matches_rgb(glu, oracle):
    from paper_2307_09582_b200 import workloads
    img = workloads.scene(240, 136, 6)
    high = dev(img)
    low, grid = glu.grid_downsample(high, 8)
    matte = glu.op_matte(low)
    field = glu.optimize_field(high, low, grid)
    one = glu.apply_field(field, matte).cpu().numpy()
    rgb = oracle.apply_field(host_params(field.params),
                             np.repeat(matte.cpu().numpy()[..., None], 3, axis=2))
    assert same(one, np.ascontiguousarray(rgb[..., 0]))
    fused, _ = glu.solve_apply(high, low, grid, matte)
    assert same(fused.cpu().numpy(), one)


@pytest.mark.parametrize("mode", ["fast", "gnu", "exact"])
def test_joint_vs_oracle_seeded(glu, oracle, mode):
    from paper_2307_09582_b200 import workloads
    # regular, ragged, tall-thin, scale-2 and scale-32 grids
    for (W, H, s, seed) in ((256, 192, 8, 21), (300, 170, 6, 22), (40, 260, 4, 23),
                            (130, 90, 2, 24), (400, 200, 32, 25)):
        img = workloads.scene(W, H, seed)
        r = glu.joint_optimize(dev(img), s, None, mode_of(glu, mode))
        o = oracle.joint_optimize(img, s, mode=mode)
        assert [r.iterations, r.trialsAccepted, r.trialsRejected] == \
            [o["iterations"], o["accepted"], o["rejected"]]
        assert same(r.low.cpu().numpy(), o["low"])
        assert same(host_params(r.field.params), o["field"])
        assert same(r.errors.cpu().numpy(), o["errors"])


@pytest.mark.parametrize("mode", ["fast", "gnu", "exact"])
def test_joint_vs_oracle_tie_heavy(glu, oracle, mode):
    """Joint loop on quantised (duplicate-colour, tie-heavy) and noise images:
    the trial filters' exact-zero, close-call and close-set paths against the
    oracle."""
    from paper_2307_09582_b200 import workloads
    rng = np.random.default_rng(5)
    base = workloads.scene(200, 144, 31)
    for img in ((np.round(base * 3) / 3).astype(np.float32),
                rng.random((120, 160, 3), dtype=np.float32)):
        r = glu.joint_optimize(dev(img), 4, None, mode_of(glu, mode))
        o = oracle.joint_optimize(img, 4, mode=mode)
        assert [r.iterations, r.trialsAccepted, r.trialsRejected] == \
            [o["iterations"], o["accepted"], o["rejected"]]
        assert same(r.low.cpu().numpy(), o["low"])
        assert same(host_params(r.field.params), o["field"])
        assert same(r.errors.cpu().numpy(), o["errors"])


def test_full_size_properties(glu, oracle):
    """C3 size (3840x2160, s=8): determinism, oracle rows, gain linearity."""
    from paper_2307_09582_b200 import workloads
    img = workloads.scene(3840, 2160, 3, 0)
    high = dev(img)
    low, grid = glu.grid_downsample(high, 8)
    f1 = glu.optimize_field(high, low, grid)
    f2 = glu.optimize_field(high, low, grid)
    assert torch.equal(f1.params, f2.params)
    # every pixel against the oracle (fast mode, the reference default)
    want = oracle.optimize_field(img, low.cpu().numpy(), 8)
    assert same(host_params(f1.params), want)
    out = glu.apply_field(f1, low, clampOutput=False)
    half = glu.apply_field(f1, low * 0.5, clampOutput=False)
    assert torch.equal(half, out * 0.5)


def test_validation_messages(glu):
    img = torch.zeros((16, 16, 3), device="cuda")
    low, grid = glu.grid_downsample(img, 4)
    with pytest.raises(ValueError, match="windowSide must be odd"):
        glu.optimize_field(img, low, grid, glu.GluConfig(windowSide=4))
    with pytest.raises(ValueError, match="epsilon must be > 0"):
        glu.optimize_field(img, low, grid, glu.GluConfig(epsilon=0.0))
    with pytest.raises(ValueError, match="low-res image does not match grid"):
        glu.optimize_field(img, torch.zeros((4, 3, 3), device="cuda"), grid)
    with pytest.raises(ValueError, match="image dimensions differ"):
        glu.error_map(img, torch.zeros((4, 4, 3), device="cuda"))
    with pytest.raises(ValueError, match="empty component"):
        f = glu.optimize_field(img, low, grid)
        glu.trial_update_component(img, low, f, torch.zeros((16, 16), device="cuda"), [])


def _stress_images():
    """Inputs built to provoke near-ties in the fp32 filter: quantised colours
    (exact duplicate candidates), smooth colinear ramps, pure noise, tiny values."""
    from paper_2307_09582_b200 import workloads
    rng = np.random.default_rng(7)
    base = workloads.scene(320, 200, 31)
    yield "scene", base
    yield "quantised", (np.round(base * 4) / 4).astype(np.float32)
    yy, xx = np.mgrid[0:200, 0:320].astype(np.float32)
    ramp = np.stack([xx / 320, yy / 200, (xx + yy) / 520], axis=2).astype(np.float32)
    yield "ramp", ramp
    yield "noise", rng.random((200, 320, 3), dtype=np.float32)
    yield "tiny", (rng.random((200, 320, 3)) * 1e-6).astype(np.float32)
    yield "two_level", (rng.random((200, 320, 1)) < 0.5).repeat(3, 2).astype(np.float32)
    # magnitudes where the fp32 closed-form objective would overflow (products
    # of two squared distances): the solve must fall back, not drop candidates
    yield "huge", (base * 3e11).astype(np.float32)
    spiky = base.copy()
    spiky[rng.random((200, 320)) < 0.05] *= 1e15
    yield "huge_spikes", spiky.astype(np.float32)


@pytest.mark.parametrize("mode", ["fast", "gnu", "exact"])
@pytest.mark.parametrize("S", [3, 5])
def test_fp32_filter_matches_oracle_on_stress_images(glu, oracle, mode, S):
    ctx = glu.glu.context()
    close0 = ctx.close_sets
    for name, img in _stress_images():
        for s in (4, 8):
            high = dev(img)
            low, grid = glu.grid_downsample(high, s)
            want = oracle.optimize_field(img, low.cpu().numpy(), s, S, EPS_DEFAULT, mode)
            for solver in (0, 1, 2):
                ctx.set_solver(solver)
                f = glu.optimize_field(high, low, grid, glu.GluConfig(windowSide=S),
                                       mode_of(glu, mode))
                got = host_params(f.params)
                ctx.set_solver(0)
                assert same(got, want), (name, s, solver, int((got != want).sum()))
    if mode in ("fast", "exact") and S == 3:
        # the near-tie close-set path (settled in double) ran and stayed exact
        assert ctx.close_sets > close0


def test_reference_unit_tests_pass_against_dropin_api(glu):
    """The reference's own unit tests (proj/tests/unit/{grid,upsample,jointopt,
    parallel}_test.cpp, 47 cases) compiled UNCHANGED against include/glu and
    linked with lib/libglu.so (oracle/Makefile `reftests`, built where
    /root/reference exists; the binary travels with the tree)."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = os.path.join(root, "oracle", "_ref", "ref_unit_tests_b200")
    if not os.path.exists(exe):
        if not os.path.isdir("/root/reference/proj/tests/unit"):
            pytest.skip("ref_unit_tests_b200 not built and /root/reference absent")
        subprocess.run(["make", "-s", "-C", os.path.join(root, "oracle"), "reftests"], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    import re
    m = re.search(r"test cases: (\d+) \| (\d+) passed \| 0 failed", r.stdout)
    assert m and int(m.group(1)) >= 55 and m.group(1) == m.group(2), r.stdout


@pytest.mark.parametrize("W,H,s,S,literal,mode", [
    (512, 384, 8, 3, False, "fast"), (640, 360, 4, 3, False, "fast"),
    (480, 320, 6, 5, False, "fast"), (400, 300, 8, 3, True, "fast"),
    (480, 360, 6, 3, False, "fast"), (512, 384, 8, 3, False, "gnu"),
    (384, 256, 8, 3, False, "exact"), (250, 190, 5, 5, False, "exact")])
def test_parallel_trial_schedule_matches_sequential(glu, W, H, s, S, literal, mode):
    """The parallel trial schedules -- speculative (default) and dataflow -- on
    the on-chip trial path (full and clipped footprints, power-of-two and other
    scales) are bit-identical to the reference's sequential component loop
    (jointopt.cpp:195-202)."""
    from paper_2307_09582_b200 import workloads
    high = dev(workloads.scene(W, H, 40 + s))
    cfg = glu.GluConfig(windowSide=S, literalComponentUpdate=literal)
    md = {"fast": glu.Mode.Fast, "gnu": glu.Mode.Gnu, "exact": glu.Mode.Exact}[mode]
    ctx = glu.glu.context()
    out = []
    for trials in (1, 0, 2):
        ctx.set_trials(trials)
        out.append(glu.joint_optimize(high, s, cfg, md))
    ctx.set_trials(0)
    a = out[0]
    assert a.trialsAccepted + a.trialsRejected > 10
    for b in out[1:]:  # speculative and dataflow schedules
        assert (a.iterations, a.trialsAccepted, a.trialsRejected) == \
            (b.iterations, b.trialsAccepted, b.trialsRejected)
        assert torch.equal(a.low, b.low) and torch.equal(a.field.params, b.field.params)
        assert torch.equal(a.errors, b.errors)


@pytest.mark.parametrize("mode", ["fast", "gnu", "exact"])
@pytest.mark.parametrize("target", ["matte", "identity"])
@pytest.mark.parametrize("solver", [0, 1, 2])
def test_frame_pipeline_matches_composed_reference_path(glu, oracle, mode, target, solver):
    """glu_cu_upsample_frames / glu_h_upsample_frames (fused k_frame_prep +
    solve + apply) equal the composition of the reference calls: grid_downsample
    (grid.cpp:41-52), the matte operator, optimize_field (upsample.cpp:194-216)
    and apply_field (235-252) -- checked against the oracle, bit for bit."""
    from paper_2307_09582_b200 import workloads
    W, H, s = 328, 200, 8
    frames = np.stack([workloads.scene(W, H, 30 + k, k) for k in range(3)])
    ctx = glu.glu.context()
    ctx.set_solver(solver)
    try:
        got = glu.glu.upsample_frames(dev(frames), s, target, mode=mode_of(glu, mode)).cpu()
        pin_in = torch.from_numpy(frames).pin_memory()
        host = torch.empty(tuple(got.shape), dtype=torch.float32).pin_memory()
        glu.glu.upsample_frames_host(pin_in, s, host, target, mode=mode_of(glu, mode))
    finally:
        ctx.set_solver(0)
    assert torch.equal(got, host)
    for k in range(3):
        low = oracle.grid_downsample(frames[k], s)
        tgt = glu.op_matte(dev(low)).cpu().numpy() if target == "matte" else low
        P = oracle.optimize_field(frames[k], low, s, 3, EPS_DEFAULT, mode)
        want = oracle.apply_field(P, tgt)
        assert got[k].numpy().tobytes() == want.tobytes(), (k, mode, target)


@pytest.mark.parametrize("kind", ["noise", "blocks"])
def test_parallel_schedule_with_off_chip_and_whole_grid_trials(glu, kind):
    """Components too large for the on-chip trial (box > 2048 cells, > 2048
    pixels) take the global-memory path inside the speculative and dataflow
    schedules -- in place, never speculated, invalidating speculating
    successors -- and whole-grid trials run alone; all bit-identical to the
    sequential loop."""
    rng = np.random.default_rng(11)
    if kind == "noise":
        img = rng.random((192, 256, 3), dtype=np.float32)  # one huge component
    else:
        img = np.zeros((200, 240, 3), np.float32)
        img[:, :, :] = rng.random((1, 1, 3))
        for k in range(12):  # large noisy blocks = big components, plus small ones
            y, x = rng.integers(0, 150), rng.integers(0, 190)
            hh, ww = rng.integers(8, 60), rng.integers(8, 60)
            img[y:y + hh, x:x + ww] = rng.random((hh, ww, 3))
    high = dev(img)
    r0 = glu.joint_optimize(high, 4, glu.GluConfig(maxIterations=0))
    sizes = [len(c) for c in glu.find_large_error(r0.errors, glu.GluConfig().errorThreshold)
             .components]
    assert max(sizes) > 2048 and min(sizes) < 2048  # off-chip and on-chip trials
    ctx = glu.glu.context()
    out = []
    for trials in (1, 0, 2):
        ctx.set_trials(trials)
        out.append(glu.joint_optimize(high, 4))
    ctx.set_trials(0)
    a = out[0]
    assert a.trialsAccepted + a.trialsRejected > 0
    for b in out[1:]:
        assert (a.iterations, a.trialsAccepted, a.trialsRejected) == \
            (b.iterations, b.trialsAccepted, b.trialsRejected)
        assert torch.equal(a.low, b.low) and torch.equal(a.field.params, b.field.params)
        assert torch.equal(a.errors, b.errors)


@pytest.mark.parametrize("S", [3, 5])
def test_nonfinite_inputs_match_oracle(glu, oracle, S):
    # NaN / +inf / -inf channels in the guide (and, through grid_downsample, in
    # the LR image): every solver setting must follow the reference's IEEE
    # comparisons bit for bit (the fp32 filters route such pixels / solves to
    # the double path)
    from test_oracle import nonfinite_scene
    img = nonfinite_scene()
    ctx = glu.glu.context()
    for s in (4, 8):
        high = dev(img)
        low, grid = glu.grid_downsample(high, s)
        lo = oracle.grid_downsample(img, s)
        assert same(low.cpu().numpy(), lo)
        for m in ("fast", "exact", "gnu"):
            want = oracle.optimize_field(img, lo, s, S, EPS_DEFAULT, m)
            for solver in (0, 1, 2):
                ctx.set_solver(solver)
                f = glu.optimize_field(high, low, grid, glu.GluConfig(windowSide=S), mode_of(glu, m))
                ctx.set_solver(0)
                got = host_params(f.params)
                assert same(got, want), (s, m, solver, int((got != want).sum()))


@pytest.mark.parametrize("mode", ["fast", "gnu"])
@pytest.mark.parametrize("image", ["scene", "quantised", "noise"])
@pytest.mark.parametrize("s", [16, 12])
def test_joint_unchanged_pixel_pass_matches_oracle(glu, oracle, mode, image, s):
    """Scales where a trial's box spans about three rounds of pixels per CTA
    thread, so the on-chip trials screen their affected pixels with the
    unchanged-pixel certificate (f32s_unchanged) and re-solve the rest in a
    compacted pass: every schedule against the oracle (itself pinned to the
    reference) -- including quantised colours, whose exact distance ties must
    fail the certificate and go to the full solve."""
    from paper_2307_09582_b200 import workloads
    W, H = 640, 480
    img = workloads.scene(W, H, 57)
    if image == "quantised":
        img = (np.round(img * 4) / 4).astype(np.float32)
    elif image == "noise":
        img = np.random.default_rng(5).random((H, W, 3), dtype=np.float32)
    img = np.ascontiguousarray(img)
    o = oracle.joint_optimize(img, s, mode=mode)
    ctx = glu.glu.context()
    try:
        for trials in (0, 2, 1):
            ctx.set_trials(trials)
            r = glu.joint_optimize(dev(img), s, None, mode_of(glu, mode))
            assert [r.iterations, r.trialsAccepted, r.trialsRejected] == \
                [o["iterations"], o["accepted"], o["rejected"]], trials
            assert r.low.cpu().numpy().tobytes() == o["low"].tobytes(), trials
            assert host_params(r.field.params).tobytes() == o["field"].tobytes(), trials
            assert r.errors.cpu().numpy().tobytes() == o["errors"].tobytes(), trials
    finally:
        ctx.set_trials(0)
    assert o["accepted"] + o["rejected"] > 0


@pytest.mark.parametrize("W,H,s,mode", [(200, 136, 8, "fast"), (198, 131, 6, "fast"),
                                        (256, 96, 4, "gnu"), (200, 136, 8, "exact"),
                                        (198, 131, 5, "exact"), (320, 200, 16, "exact")])
def test_frame_batches_match_single_frames(glu, W, H, s, mode):
    """glu_cu_upsample_frames with a 1-channel matte launches k_solve32f (Exact
    mode: k_solve32x) over
    batches of up to 16 frames (grid z = frame; a 3-D tensor map when the rows
    are 16-byte aligned, else the threads stage each frame's guide); 35 frames
    = batches of 16, 16 and 3 on two buffer groups.  Every frame equals its
    own single-frame solve + apply, bit for bit."""
    from paper_2307_09582_b200 import workloads
    frames = np.stack([workloads.scene(W, H, 70 + k, k) for k in range(35)])
    md = mode_of(glu, mode)
    got = glu.glu.upsample_frames(dev(frames), s, "matte", mode=md)
    for k in range(frames.shape[0]):
        f = dev(frames[k])
        low, grid = glu.grid_downsample(f, s)
        want, _ = glu.solve_apply(f, low, grid, glu.op_matte(low), None, md)
        assert torch.equal(got[k], want), k
