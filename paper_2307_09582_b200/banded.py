"""Multi-GPU upsample-only editing: C5 over HR row bands.

The interactive-editing path applies a resident parameter field to a stream
of LR targets (apply_field, upsample.cpp:235-252).  Split over GPUs, each rank
keeps only its HR row band of the field (sharding.row_bands: bands aligned to
multiples of s); the params hold *global* LR indices, so a band's apply needs
the whole LR target (1.56 MB at 8K / s16) but no halo.  A target arrives at
one rank (`src`) and is broadcast (NCCL over NVLink; gloo for CPU tests),
double-buffered: target k+1 is in flight while target k is applied.  Total
work is fixed as ranks are added (strong scaling); the band outputs tile the
full frame and are bit-identical to a single-GPU apply (tests/test_multiproc.py,
tests/test_distributed_gpu.py).
"""
from __future__ import annotations

from typing import Callable, Sequence

import torch
import torch.distributed as dist

from . import sharding
from .glu import GridSpec, apply_field_band


def band_rows(grid: GridSpec, windowSide: int, world: int, rank: int) -> tuple[int, int]:
    """HR rows [y0, y1) owned by `rank`."""
    return sharding.row_bands(grid.highH, grid.scale, windowSide, world)[rank].hr_rows


def run_banded_apply(bandParams: torch.Tensor, grid: GridSpec,
                     targets: Sequence[torch.Tensor] | None, ntargets: int, channels: int = 3,
                     src: int = 0, clampOutput: bool = True,
                     apply: Callable | None = None,
                     sink: Callable[[int, torch.Tensor], None] | None = None) -> None:
    """Apply `ntargets` LR targets (given on rank `src`) to this rank's band.

    `apply(bandParams, grid, target, clampOutput)` defaults to the device
    kernel (glu_cu_apply_field_band); `sink(k, out)` receives each band output.
    """
    rank = dist.get_rank()
    if rank == src and (targets is None or len(targets) < ntargets):
        raise ValueError("banded apply: the source rank must hold every target")
    apply = apply or (lambda p, g, t, c: apply_field_band(p, g, t, c))
    shape = (grid.lowH, grid.lowW, 3) if channels == 3 else (grid.lowH, grid.lowW)
    bufs = [torch.empty(shape, dtype=torch.float32, device=bandParams.device) for _ in range(2)]

    def post(k: int):
        buf = bufs[k % 2]
        if rank == src:
            buf.copy_(targets[k])
        # the collective is ordered after every op already queued on the
        # current stream (the apply of target k - 1 that read this buffer)
        return dist.broadcast(buf, src, async_op=True)

    if ntargets <= 0:
        return
    work = post(0)
    for k in range(ntargets):
        work.wait()
        nxt = post(k + 1) if k + 1 < ntargets else None
        out = apply(bandParams, grid, bufs[k % 2], clampOutput)
        if sink is not None:
            sink(k, out)
        work = nxt
