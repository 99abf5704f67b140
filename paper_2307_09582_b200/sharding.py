"""Host-side work decomposition for 1/2/4/8 GPUs of one node.

* C3 video: frames are independent -> every rank solves its own frames, no
  data-path collective (weak scaling).
* C4 / C5 bands: HR row bands aligned to multiples of s, so every LR cell's
  footprint lies in one band; a band owning LR rows [r0, r1) reads LR rows
  [r0 - h, r1 + h) for the solve (h = S // 2) and [r0 - 2h, r1 + 2h) for the
  joint trials (SURVEY §8(a) conflict rule).
"""
from __future__ import annotations

from dataclasses import dataclass


def frame_seeds(rank: int, world: int, nframes: int, base_seed: int) -> list[tuple[int, int]]:
    """(scene seed, frame index) pairs of one rank: each rank owns a full clip."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    return [(base_seed + 1000 * rank, f) for f in range(nframes)]


@dataclass(frozen=True)
class Band:
    rank: int
    lr_rows: tuple[int, int]       # owned LR rows [r0, r1)
    hr_rows: tuple[int, int]       # owned HR rows [r0*s, min(r1*s, H))
    solve_halo: tuple[int, int]    # LR rows read by the solve
    trial_halo: tuple[int, int]    # LR rows read by joint trials

    @property
    def halo_rows(self) -> int:
        return (self.lr_rows[0] - self.solve_halo[0]) + (self.solve_halo[1] - self.lr_rows[1])


def row_bands(H: int, s: int, S: int, world: int) -> list[Band]:
    """Balanced LR-row bands (270 rows over 8 ranks -> 34 x 6 + 33 x 2)."""
    lh = (H + s - 1) // s
    if world < 1 or world > lh:
        raise ValueError("world size must be in [1, lowH]")
    h = S // 2
    base, extra = divmod(lh, world)
    bands, r0 = [], 0
    for r in range(world):
        r1 = r0 + base + (1 if r < extra else 0)
        bands.append(Band(r, (r0, r1), (r0 * s, min(r1 * s, H)),
                          (max(0, r0 - h), min(lh, r1 + h)),
                          (max(0, r0 - 2 * h), min(lh, r1 + 2 * h))))
        r0 = r1
    return bands


def halo_bytes(band: Band, lw: int, channels: int = 3) -> int:
    """Bytes of LR halo a band receives per exchange (f32)."""
    return band.halo_rows * lw * channels * 4
