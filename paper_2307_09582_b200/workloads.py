"""Seeded synthetic stand-ins for BASELINE.json's five configs.

No public dataset is used: the guide images come from the seeded generator in
csrc/synth_scene.cpp (Voronoi regions + gradients + 200 one-pixel lines +
Gaussian noise, BASELINE.json configs[0]); the LR operators below are the
harness-side "black box" operators the configs name.  All randomness is the
reference's SplitMix64 (proj/include/glu/synth.hpp:12-34).  Seeds: image seed =
config number, operator seed = 1000 + config number.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _native as N

MASK64 = (1 << 64) - 1


class SplitMix64:
    """glu::Rng (synth.hpp:12-34)."""

    def __init__(self, seed: int):
        self.state = seed & MASK64

    def next(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & MASK64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        return z ^ (z >> 31)

    def uniform(self, lo: float = 0.0, hi: float = 1.0) -> float:
        return lo + (hi - lo) * ((self.next() >> 11) * 2.0 ** -53)

    def normal(self, sigma: float = 1.0) -> float:
        u1 = 1.0 - self.uniform()
        u2 = self.uniform()
        return sigma * math.sqrt(-2.0 * math.log(u1)) * math.cos(2.0 * math.pi * u2)

    def color(self) -> list[float]:
        return [float(np.float32(self.uniform())) for _ in range(3)]


def scene(W: int, H: int, seed: int, frame: int = 0, threads: int = 0) -> np.ndarray:
    """Guide image (H, W, 3) float32 in [0, 1] (csrc/synth_scene.cpp)."""
    out = np.empty((H, W, 3), np.float32)
    rc = N.synth_lib().glu_synth_scene(int(W), int(H), int(seed), int(frame), int(threads),
                                       C.c_void_p(out.ctypes.data))
    if rc:
        raise ValueError("scene: invalid dimensions")
    return out


def box_downsample(img: np.ndarray, s: int) -> np.ndarray:
    """s x s box mean (configs[0]); dimensions must divide evenly."""
    H, W, _ = img.shape
    if H % s or W % s:
        raise ValueError("box_downsample: dimensions must be multiples of s")
    return img.reshape(H // s, s, W // s, s, 3).mean(axis=(1, 3), dtype=np.float64).astype(
        np.float32)


@dataclass
class ColorOp:
    """clamp01(M @ g(x) + b), g = optional gamma (simop.cpp:22-36)."""
    M: np.ndarray
    bias: np.ndarray
    gamma: float = 0.0

    def apply_numpy(self, low: np.ndarray) -> np.ndarray:
        x = low.astype(np.float64)
        if self.gamma > 0:
            x = np.clip(np.power(x, self.gamma), 0, 1).astype(np.float32).astype(np.float64)
        y = x @ self.M.T + self.bias
        return np.clip(y, 0, 1).astype(np.float32)


def affine_op(seed: int) -> ColorOp:
    """configs[0]: M = I + N(0, 0.2) entries, b ~ U[-0.1, 0.1]^3."""
    r = SplitMix64(seed)
    M = np.eye(3) + np.array([r.normal(0.2) for _ in range(9)]).reshape(3, 3)
    b = np.array([r.uniform(-0.1, 0.1) for _ in range(3)])
    return ColorOp(M, b, 0.0)


def gamma_mix_op(seed: int) -> ColorOp:
    """configs[1]/[3]: gamma 1/2.2 followed by the seeded 3x3 colour matrix."""
    r = SplitMix64(seed)
    M = np.eye(3) + np.array([r.normal(0.2) for _ in range(9)]).reshape(3, 3)
    return ColorOp(M, np.zeros(3), 1.0 / 2.2)


def mix_op(seed: int) -> ColorOp:
    """configs[4]: a seeded colour-matrix edit (no gamma, no bias)."""
    r = SplitMix64(seed)
    M = np.eye(3) + np.array([r.normal(0.2) for _ in range(9)]).reshape(3, 3)
    return ColorOp(M, np.zeros(3), 0.0)


def matte_numpy(low: np.ndarray) -> np.ndarray:
    """configs[2]: 1-channel matte sigmoid(10 (luma - 0.5)) of the LR image."""
    x = low.astype(np.float64)
    Y = 0.299 * x[..., 0] + 0.587 * x[..., 1] + 0.114 * x[..., 2]
    return (1.0 / (1.0 + np.exp(-10.0 * (Y - 0.5)))).astype(np.float32)


# The five configs (BASELINE.json).  W, H, scale, joint?, frames/targets.
CONFIGS = {
    1: dict(W=512, H=512, scale=4, joint=False, name="C1 512x512 s4 box-LR GLU-"),
    2: dict(W=2048, H=2048, scale=8, joint=True, name="C2 2048x2048 s8 joint"),
    3: dict(W=3840, H=2160, scale=8, joint=False, frames=16,
            name="C3 3840x2160 s8 video x16, 1-ch matte"),
    4: dict(W=7680, H=4320, scale=16, joint=True, name="C4 7680x4320 s16 joint"),
    5: dict(W=7680, H=4320, scale=16, joint=False, targets=64,
            name="C5 7680x4320 upsample-only x64 targets"),
}
