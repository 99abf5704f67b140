"""Pin the CPU oracle (oracle/glu_oracle.c) before trusting it.

1. Bit-exact against the golden vectors the UNMODIFIED reference produced
   (tests/golden/make_golden.py).
2. The known-answer values of the reference's own unit tests
   (proj/tests/unit/{upsample,jointopt,grid}_test.cpp), restated.
3. When oracle/_ref is built: bit-exact against the reference on fresh seeds.
"""
import math

import numpy as np
import pytest

from oracle import EPS_DEFAULT, PARAMS_DTYPE, TAU_DEFAULT

SOLVES = ["mix67x45_s4", "mix41x33_s4", "photo40x28_s4", "mix37x29_s4_S5", "mix50x38_s3_S7",
          "mix45x45_s5_S9", "mix33x21_s2", "scene96x64_s8", "scene100x70_s16"]
JOINTS = ["joint_missed_line", "joint_missed_line_literal", "joint_mix72x60_s6",
          "joint_mix64x56_s8", "joint_mix48_s6_tau05", "joint_mix128_s8", "joint_mix60x52_s4_S5",
          "joint_scene160x96_s8", "joint_harmful"]


def same(a, b):
    return a.shape == b.shape and a.tobytes() == b.tobytes()


@pytest.mark.parametrize("name", SOLVES)
def test_field_solves_match_golden(oracle, golden, name):
    img, (s, S) = golden[f"{name}/high"], golden[f"{name}/meta"]
    low = oracle.grid_downsample(img, int(s))
    assert same(low, golden[f"{name}/low"])
    for m in ("fast", "exact", "gnu"):
        f = oracle.optimize_field(img, low, int(s), int(S), EPS_DEFAULT, m)
        assert same(f, golden[f"{name}/params_{m}"].view(PARAMS_DTYPE).reshape(f.shape)), m
        rec = oracle.apply_field(f, low)
        assert same(rec, golden[f"{name}/apply_{m}"]), m
        assert same(oracle.error_map(img, rec), golden[f"{name}/errors_{m}"]), m
    half = oracle.apply_field(golden[f"{name}/params_fast"].view(PARAMS_DTYPE).reshape(
        img.shape[:2]), low * np.float32(0.5), clamp=False)
    assert same(half, golden[f"{name}/apply_fast_noclamp_half"])


@pytest.mark.parametrize("name", JOINTS)
def test_joint_matches_golden(oracle, golden, name):
    img, (s, S, lit) = golden[f"{name}/high"], golden[f"{name}/meta"]
    tau = float(golden[f"{name}/tau"][0])
    modes = ("fast", "exact", "gnu") if name == "joint_mix72x60_s6" else ("fast",)
    for m in modes:
        r = oracle.joint_optimize(img, int(s), int(S), tau, 3, EPS_DEFAULT, m, bool(lit))
        key = f"{name}/{m}"
        assert same(r["low"], golden[f"{key}/low"])
        assert same(r["field"], golden[f"{key}/params"].view(PARAMS_DTYPE).reshape(
            r["field"].shape))
        assert same(r["errors"], golden[f"{key}/errors"])
        assert [r["iterations"], r["accepted"], r["rejected"]] == golden[f"{key}/counts"].tolist()


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_trial_sequence_matches_golden(oracle, golden, seed):
    img = golden[f"trials_mix48_{seed}/high"]
    s, tau = 6, 0.05
    low = oracle.grid_downsample(img, s)
    field = oracle.optimize_field(img, low, s)
    errors = oracle.error_map(img, oracle.apply_field(field, low))
    _, comps = oracle.find_large_error(errors, tau)
    verdicts = [oracle.trial_update_component(img, low, field, errors, c, s) for c in comps]
    assert verdicts == golden[f"trials_mix48_{seed}/verdicts"].astype(bool).tolist()
    assert same(low, golden[f"trials_mix48_{seed}/low"])
    assert same(errors, golden[f"trials_mix48_{seed}/errors"])


@pytest.mark.parametrize("name", ["ccl_pin", "ccl_scene"])
def test_find_large_error_matches_golden(oracle, golden, name):
    mask, comps = oracle.find_large_error(golden[f"{name}/errors"],
                                          float(golden[f"{name}/tau"][0]))
    assert same(mask, golden[f"{name}/mask"])
    off, px = golden[f"{name}/offsets"], golden[f"{name}/pixels"]
    assert len(comps) == len(off) - 1
    for c, comp in enumerate(comps):
        assert comp.tolist() == px[off[c]:off[c + 1]].tolist()


@pytest.mark.parametrize("mode", ["fast", "exact", "gnu"])
def test_pixel_selection_matches_golden(oracle, golden, mode):
    ip, rgb, idx, off = (golden[f"pixels/{k}"] for k in ("ip", "rgb", "idx", "off"))
    want = golden[f"pixels/{mode}"]
    for k in range(len(ip)):
        a, b, w = oracle.optimize_pixel(ip[k], idx[off[k]:off[k + 1]], rgb[off[k]:off[k + 1]],
                                        1e-3, mode)
        assert (a, b, np.float32(w).view(np.uint32)) == tuple(want[k].tolist()), k


# ---- known answers of the reference unit tests ------------------------------------

def test_weight_pins(oracle):
    # upsample_test.cpp:39-54
    assert oracle.weight_exact([0.25, 0, 0], [1, 0, 0], [0, 0, 0], 1e-3) == pytest.approx(
        0.25 / 1.001, rel=1e-9)
    assert oracle.weight_exact([0.5, 0.5, 0], [1, 0, 0], [0, 0, 0], 1e-3) == pytest.approx(
        0.5 / 1.001, rel=1e-9)
    assert oracle.weight_fast([0.5] * 3, [1] * 3, [0] * 3, 1e-3) == pytest.approx(0.4997, rel=1e-4)
    assert oracle.weight_fast([0.25, 0, 0], [1, 0, 0], [0, 0, 0], 1e-3) == pytest.approx(
        0.25 / 1.001, rel=1e-6)


def test_pixel_pins(oracle):
    # upsample_test.cpp:123-159
    levels = np.array([[v] * 3 for v in (0.0, 0.25, 0.5, 0.75, 1.0)], np.float32)
    a, b, w = oracle.optimize_pixel([0.3] * 3, np.arange(5), levels, 1e-3, "fast")
    assert (a, b) == (1, 2) and w == pytest.approx(0.798, rel=2e-3)
    same6 = np.tile(np.array([0.3, 0.7, 0.2], np.float32), (6, 1))
    assert oracle.optimize_pixel([0.9, 0.1, 0.5], np.arange(6) + 40, same6, 1e-3,
                                 "exact") == (40, 40, 0.0)
    a, b, w = oracle.optimize_pixel([1.0] * 3, [0, 1], np.array([[0.8] * 3, [0.4] * 3]), 1e-3,
                                    "exact")
    assert (a, b) == (0, 1) and w > 1.0
    with pytest.raises(ValueError):
        oracle.optimize_pixel([0, 0, 0], [], np.zeros((0, 3)), 1e-3, "gnu")


def test_dominance_chain(oracle):
    # upsample_test.cpp:161-176 / acceptance crit5: exact <= fast <= gnu
    from paper_2307_09582_b200.workloads import SplitMix64
    rng = SplitMix64(20230801)
    for _ in range(300):
        ip = np.array(rng.color(), np.float32)
        c = np.array([rng.color() for _ in range(9)], np.float32)
        r = {}
        for m in ("exact", "fast", "gnu"):
            a, b, w = oracle.optimize_pixel(ip, np.arange(9), c, 1e-3, m)
            r[m] = oracle.pair_objective(ip, c[a], c[b], w, 1e-3)
        assert r["exact"] <= r["fast"] + 1e-12
        assert r["fast"] <= r["gnu"] + 1e-12


def test_grid_pins(oracle):
    # grid_test.cpp:46-55: 4x4 ramp k/16, s = 2
    img = np.repeat((np.arange(16, dtype=np.float32) / 16).reshape(4, 4, 1), 3, axis=2)
    low = oracle.grid_downsample(img, 2)
    assert low[..., 0].tolist() == [[5 / 16, 7 / 16], [13 / 16, 15 / 16]]
    with pytest.raises(ValueError):
        oracle.grid_downsample(np.zeros((16, 16, 3), np.float32), 16)


def test_ccl_pin(oracle):
    # jointopt_test.cpp:32-51
    em = np.zeros((4, 6), np.float32)
    em[0, 0], em[0, 5], em[1, 1], em[1, 2], em[2, 3], em[3, 4] = 0.1, 0.15, 0.2, 0.3, 0.2, 0.2
    mask, comps = oracle.find_large_error(em, 0.1)
    assert mask[0, 0] == 0
    assert [c.tolist() for c in comps] == [[5], [7, 8], [15], [22]]


def test_missed_line_recovered(oracle):
    # jointopt_test.cpp:53-74, 111-119
    img = np.full((16, 16, 3), 0.1, np.float32)
    img[0, :] = (0.9, 0.2, 0.3)
    r = oracle.joint_optimize(img, 4)
    assert r["iterations"] >= 1 and r["accepted"] >= 1
    assert float(r["errors"].astype(np.float64).sum()) == 0.0
    fresh = oracle.error_map(img, oracle.apply_field(r["field"], r["low"]))
    assert same(fresh, r["errors"])


def test_error_map_pins(oracle):
    # upsample_test.cpp:285-302
    a = np.tile(np.array([0.4, 0.5, 0.6], np.float32), (8, 8, 1))
    b = a.copy()
    b[..., 0] += np.float32(0.1)
    assert np.allclose(oracle.error_map(a, b), 0.1, rtol=1e-6)
    c = a + np.float32(0.1)
    assert np.allclose(oracle.error_map(a, c), 0.1 * math.sqrt(3), rtol=1e-6)


def test_oracle_vs_reference_fresh_seeds(oracle, reference):
    for seed in (501, 502, 503):
        img = reference.synth("mixture", 57 + seed % 5, 43, seed)
        for s, S in ((4, 3), (5, 5)):
            low = reference.grid_downsample(img, s)
            for m in ("fast", "exact", "gnu"):
                assert same(oracle.optimize_field(img, low, s, S, EPS_DEFAULT, m),
                            reference.optimize_field(img, low, s, S, EPS_DEFAULT, m))
        a = oracle.joint_optimize(img, 4, 3, TAU_DEFAULT)
        b = reference.joint_optimize(img, 4, 3, TAU_DEFAULT)
        assert same(a["low"], b["low"]) and same(a["errors"], b["errors"])
        assert (a["accepted"], a["rejected"]) == (b["accepted"], b["rejected"])


def nonfinite_scene(W=96, H=72, seed=41):
    """A seeded scene with NaN / +inf / -inf channels sprinkled over it (some on
    LR sample pixels, so the LR image holds them too)."""
    from paper_2307_09582_b200 import workloads
    img = workloads.scene(W, H, seed).copy()
    rng = np.random.default_rng(seed)
    for val in (np.nan, np.inf, -np.inf):
        ys, xs, cs = rng.integers(0, H, 12), rng.integers(0, W, 12), rng.integers(0, 3, 12)
        img[ys, xs, cs] = val
    img[2, 2, :] = np.inf          # an LR sample pixel at s = 4 (centre offset 2)
    img[6, 10, 1] = np.nan
    return img


@pytest.mark.parametrize("S", [3, 5])
def test_oracle_vs_reference_nonfinite(oracle, reference, S):
    # IEEE comparisons with NaN / inf in the reference's scans (upsample.cpp:49-104):
    # the restatement must follow them operation for operation
    img = nonfinite_scene()
    for s in (4, 8):
        low = reference.grid_downsample(img, s)
        assert same(oracle.grid_downsample(img, s), low)
        for m in ("fast", "exact", "gnu"):
            want = reference.optimize_field(img, low, s, S, EPS_DEFAULT, m)
            got = oracle.optimize_field(img, low, s, S, EPS_DEFAULT, m)
            assert same(got, want), (s, m)


def nan_joint_scene():
    """tests/test_robustness_gpu.py's joint input: NaN channels on 40 guide
    pixels, so many trials see a NaN error in their affected set."""
    from paper_2307_09582_b200 import workloads
    img = workloads.scene(256, 192, 91)
    rng = np.random.default_rng(3)
    ys, xs = rng.integers(0, 192, 40), rng.integers(0, 256, 40)
    img[ys, xs, rng.integers(0, 3, 40)] = np.nan
    return img


@pytest.mark.parametrize("mode", ["fast", "exact", "gnu"])
def test_oracle_vs_reference_joint_nan_guide(oracle, reference, mode):
    # NaN <= NaN is false in jointopt.cpp:167: such trials are rejected
    img = nan_joint_scene()
    a = oracle.joint_optimize(img, 8, mode=mode)
    b = reference.joint_optimize(img, 8, mode=mode)
    assert (a["iterations"], a["accepted"], a["rejected"]) == \
        (b["iterations"], b["accepted"], b["rejected"])
    for k in ("low", "field", "errors"):
        assert same(a[k], b[k]), k
