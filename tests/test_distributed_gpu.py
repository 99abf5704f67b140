"""The level-synchronous multi-rank joint loop (paper_2307_09582_b200/distributed.py)
is bit-identical to the single-GPU joint_optimize (itself bit-identical to the
reference).  One GPU is available, so W ranks are emulated in one process:
each keeps its own replica, runs only its share of every level, and applies the
other ranks' change logs."""
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("W,H,s,S", [(512, 384, 8, 3), (480, 320, 6, 5)])
def test_local_ranks_match_single_gpu(glu, world, W, H, s, S):
    from paper_2307_09582_b200 import distributed, workloads
    high = torch.from_numpy(workloads.scene(W, H, 60 + s)).cuda()
    cfg = glu.GluConfig(windowSide=S)
    ref = glu.joint_optimize(high, s, cfg)
    results, stats = distributed.joint_optimize_local(high, s, world, cfg)
    assert stats["iterations"] == ref.iterations
    assert (stats["accepted"], stats["rejected"]) == (ref.trialsAccepted, ref.trialsRejected)
    assert ref.trialsAccepted > 0
    for r in results:
        assert torch.equal(r.low, ref.low)
        assert torch.equal(r.field.params, ref.field.params)
        assert torch.equal(r.errors, ref.errors)


def test_levels_are_independent_sets(glu):
    """Within a level no two component boxes are within 2h (the conflict rule)."""
    import numpy as np
    from paper_2307_09582_b200 import distributed, workloads
    high = torch.from_numpy(workloads.scene(640, 480, 9)).cuda()
    r = glu.joint_optimize(high, 8, glu.GluConfig(maxIterations=0))
    les = glu.find_large_error(r.errors, glu.GluConfig().errorThreshold)
    lv = distributed.trial_levels(les, r.field.grid, 3, high.device)
    comps = les.components
    W, s = 640, 8
    bx = np.array([[((c % W) // s).min(), ((c // W) // s).min(), ((c % W) // s).max(),
                    ((c // W) // s).max()] for c in comps], dtype=np.int64)
    for L in range(1, lv.max() + 1):
        ids = np.nonzero(lv == L)[0]
        b = bx[ids]
        dx = np.maximum(0, np.maximum(b[:, None, 0] - b[None, :, 2], b[None, :, 0] - b[:, None, 2]))
        dy = np.maximum(0, np.maximum(b[:, None, 1] - b[None, :, 3], b[None, :, 1] - b[:, None, 3]))
        cheb = np.maximum(dx, dy)
        np.fill_diagonal(cheb, 99)
        assert (cheb > 2).all()
    # and each component's level exceeds that of every earlier conflicting one
    for i in range(len(comps)):
        for j in range(i):
            d = max(0, bx[j, 0] - bx[i, 2], bx[i, 0] - bx[j, 2], bx[j, 1] - bx[i, 3],
                    bx[i, 1] - bx[j, 3])
            if d <= 2:
                assert lv[i] > lv[j]


@pytest.mark.parametrize("world,channels", [(2, 3), (8, 3), (3, 1)])
def test_banded_apply_tiles_full_apply(glu, world, channels):
    """C5 row bands: per-band applies of a field through
    glu_cu_apply_field_band concatenate to the single-GPU apply, bit for bit."""
    from paper_2307_09582_b200 import banded, workloads
    W, H, s = 640, 480, 16
    high = torch.from_numpy(workloads.scene(W, H, 5)).cuda()
    low, grid = glu.grid_downsample(high, s)
    field = glu.optimize_field(high, low, grid)
    target = glu.op_color(low, workloads.mix_op(1005).M)
    if channels == 1:
        target = glu.op_matte(target)
    full = glu.apply_field(field, target)
    parts = []
    for r in range(world):
        y0, y1 = banded.band_rows(grid, 3, world, r)
        parts.append(glu.glu.apply_field_band(field.params[y0:y1], grid, target))
    assert torch.equal(torch.cat(parts), full)
