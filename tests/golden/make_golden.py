"""Generate tests/golden/glu_golden.npz from the UNMODIFIED reference library.

Runs only in the build container (it needs oracle/_ref/libglu_ref.so, built by
oracle/Makefile from /root/reference/proj/src).  Every output array below is
produced by the reference's own functions through oracle/ref_shim.cpp; the
inputs are the reference's own synthetic images (synth_mixture / synth_photo,
proj/src/synth.cpp) with the shapes and seeds its unit tests use, plus a few
cases from this repo's BASELINE-config generator.  The committed .npz pins both
oracle/glu_oracle.c (tests/test_oracle.py) and the CUDA path
(tests/test_parity_gpu.py).

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import EPS_DEFAULT, TAU_DEFAULT, Reference  # noqa: E402
from paper_2307_09582_b200 import workloads  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "glu_golden.npz")
MODES = ("fast", "exact", "gnu")


def missed_line_image() -> np.ndarray:
    """jointopt_test.cpp:19-23: 16x16 background, one-pixel line on y = 0."""
    img = np.full((16, 16, 3), 0.1, np.float32)
    img[0, :] = (0.9, 0.2, 0.3)
    return img


def harmful_image() -> np.ndarray:
    """jointopt_test.cpp:162-171."""
    img = np.zeros((8, 8, 3), np.float32)
    img[2, 2] = (0, 1, 0)
    img[0, 0] = (0.13, 0, 0)
    img[0, 1] = (0.09, 1.0, 0.09)
    return img


def main() -> None:
    ref = Reference()
    ref.set_num_threads(1)
    g: dict[str, np.ndarray] = {}

    # --- field solves: (name, image, s, S) --------------------------------------
    solves = [
        ("mix67x45_s4", ref.synth("mixture", 67, 45, 3), 4, 3),      # upsample_test.cpp:212-224
        ("mix41x33_s4", ref.synth("mixture", 41, 33, 5), 4, 3),      # upsample_test.cpp:226-237
        ("photo40x28_s4", ref.synth("photo", 40, 28, 17), 4, 3),     # upsample_test.cpp:239-251
        ("mix37x29_s4_S5", ref.synth("mixture", 37, 29, 99), 4, 5),  # grid_test.cpp:69-78
        ("mix50x38_s3_S7", ref.synth("mixture", 50, 38, 21), 3, 7),
        ("mix45x45_s5_S9", ref.synth("mixture", 45, 45, 22), 5, 9),
        ("mix33x21_s2", ref.synth("mixture", 33, 21, 23), 2, 3),     # ragged, smallest s
        ("scene96x64_s8", workloads.scene(96, 64, 3, 0), 8, 3),       # configs[2] generator
        ("scene100x70_s16", workloads.scene(100, 70, 4, 0), 16, 3),   # ragged, s = 16
    ]
    for name, img, s, S in solves:
        low = ref.grid_downsample(img, s)
        g[f"{name}/high"] = img
        g[f"{name}/meta"] = np.array([s, S], np.int32)
        g[f"{name}/low"] = low
        for m in MODES:
            f = ref.optimize_field(img, low, s, S, EPS_DEFAULT, m)
            g[f"{name}/params_{m}"] = f
            rec = ref.apply_field(f, s, low, True)
            g[f"{name}/apply_{m}"] = rec
            g[f"{name}/errors_{m}"] = ref.error_map(img, rec)
        g[f"{name}/apply_fast_noclamp_half"] = ref.apply_field(
            g[f"{name}/params_fast"], s, (low * np.float32(0.5)).astype(np.float32), False)

    # --- joint optimisation: (name, image, s, S, tau, literal) ----------------------
    joints = [
        ("joint_missed_line", missed_line_image(), 4, 3, TAU_DEFAULT, 0),
        ("joint_missed_line_literal", missed_line_image(), 4, 3, TAU_DEFAULT, 1),
        ("joint_mix72x60_s6", ref.synth("mixture", 72, 60, 12), 6, 3, TAU_DEFAULT, 0),
        ("joint_mix64x56_s8", ref.synth("mixture", 64, 56, 101), 8, 3, TAU_DEFAULT, 0),
        ("joint_mix48_s6_tau05", ref.synth("mixture", 48, 48, 2), 6, 3, 0.05, 0),
        ("joint_mix128_s8", ref.synth("mixture", 128, 128, 1000), 8, 3, TAU_DEFAULT, 0),
        ("joint_mix60x52_s4_S5", ref.synth("mixture", 60, 52, 31), 4, 5, 0.05, 0),
        ("joint_scene160x96_s8", workloads.scene(160, 96, 2, 0), 8, 3, TAU_DEFAULT, 0),
        ("joint_harmful", harmful_image(), 4, 3, TAU_DEFAULT, 0),
    ]
    for name, img, s, S, tau, lit in joints:
        for m in (("fast", "exact", "gnu") if name == "joint_mix72x60_s6" else ("fast",)):
            r = ref.joint_optimize(img, s, S, tau, 3, EPS_DEFAULT, m, bool(lit))
            key = f"{name}/{m}"
            g[f"{name}/high"] = img
            g[f"{name}/meta"] = np.array([s, S, lit], np.int32)
            g[f"{name}/tau"] = np.array([tau], np.float32)
            g[f"{key}/low"] = r["low"]
            g[f"{key}/params"] = r["field"]
            g[f"{key}/errors"] = r["errors"]
            g[f"{key}/counts"] = np.array([r["iterations"], r["accepted"], r["rejected"]],
                                          np.int32)

    # --- per-trial states on the rollback sweep (jointopt_test.cpp:76-109) ---------
    for seed in (1, 2, 3):
        img = ref.synth("mixture", 48, 48, seed)
        s, tau = 6, 0.05
        low = ref.grid_downsample(img, s)
        field = ref.optimize_field(img, low, s, 3)
        errors = ref.error_map(img, ref.apply_field(field, s, low))
        _, comps = ref.find_large_error(errors, tau)
        verdicts = []
        for comp in comps:
            verdicts.append(ref.trial_update_component(img, low, field, errors, comp, s))
        g[f"trials_mix48_{seed}/high"] = img
        g[f"trials_mix48_{seed}/verdicts"] = np.array(verdicts, np.uint8)
        g[f"trials_mix48_{seed}/low"] = low
        g[f"trials_mix48_{seed}/params"] = field
        g[f"trials_mix48_{seed}/errors"] = errors

    # --- find_large_error (jointopt_test.cpp:32-51 pin + a real error map) ---------
    em = np.zeros((4, 6), np.float32)
    em[0, 0], em[0, 5], em[1, 1], em[1, 2], em[2, 3], em[3, 4] = 0.1, 0.15, 0.2, 0.3, 0.2, 0.2
    for name, e, tau in (("ccl_pin", em, 0.1),
                         ("ccl_scene", g["scene96x64_s8/errors_fast"], 0.05)):
        mask, comps = ref.find_large_error(e, tau)
        g[f"{name}/errors"] = e
        g[f"{name}/tau"] = np.array([tau], np.float32)
        g[f"{name}/mask"] = mask
        g[f"{name}/offsets"] = np.cumsum([0] + [len(c) for c in comps]).astype(np.uint32)
        g[f"{name}/pixels"] = (np.concatenate(comps).astype(np.uint32) if comps
                               else np.zeros(0, np.uint32))

    # --- per-pixel selection on random candidate lists (acceptance crit5 style) ----
    rng = workloads.SplitMix64(42)
    K = 400
    ip = np.array([rng.color() for _ in range(K)], np.float32)
    counts = np.array([9 if k % 4 else 1 + (k // 4) % 9 for k in range(K)], np.int64)
    rgb = np.array([rng.color() for _ in range(int(counts.sum()))], np.float32)
    idx = np.arange(int(counts.sum()), dtype=np.uint32) * 7 + 3
    off = np.concatenate([[0], np.cumsum(counts)]).astype(np.uint32)
    g["pixels/ip"], g["pixels/rgb"], g["pixels/idx"], g["pixels/off"] = ip, rgb, idx, off
    for m in MODES:
        out = np.zeros((K, 3), np.uint32)
        for k in range(K):
            a, b, w = ref.optimize_pixel(ip[k], idx[off[k]:off[k + 1]], rgb[off[k]:off[k + 1]],
                                         1e-3, m)
            out[k] = (a, b, np.array([w], np.float32).view(np.uint32)[0])
        g[f"pixels/{m}"] = out

    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT}: {len(g)} arrays, {os.path.getsize(OUT) / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
