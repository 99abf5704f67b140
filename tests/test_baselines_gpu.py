"""Comparison upsamplers on device buffers against the
reference (proj/src/baseline.cpp, built in oracle/_ref).  nearest / bilinear:
bit-exact.  JBU: CUDA's double exp is within 1 ulp of glibc's, so outputs are
compared within 1e-6 absolute (one float rounding step at values <= 1)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("W,H,s", [(66, 50, 3), (640, 360, 8), (257, 129, 16)])
def test_baselines_match_reference(glu, reference, W, H, s):
    from paper_2307_09582_b200 import workloads
    img = workloads.scene(W, H, W + s)
    high = torch.from_numpy(img).cuda()
    low, grid = glu.grid_downsample(high, s)
    target = glu.op_color(low, workloads.mix_op(7).M)
    lo, t = low.cpu().numpy(), target.cpu().numpy()
    nn = glu.glu.nearest_upsample(target, grid).cpu().numpy()
    assert nn.tobytes() == reference.baseline("nearest", t, s, img, lo).tobytes()
    bl = glu.glu.bilinear_upsample(target, grid).cpu().numpy()
    assert bl.tobytes() == reference.baseline("bilinear", t, s, img, lo).tobytes()
    for p in (glu.glu.JbuParams(), glu.glu.JbuParams(window=3, sigmaD=1.0, sigmaR=0.05)):
        jb = glu.glu.jbu_upsample(high, low, target, grid, p).cpu().numpy()
        ref = reference.baseline("jbu", t, s, img, lo, p.window, p.sigmaD, p.sigmaR)
        assert np.abs(jb - ref).max() <= 1e-6
        assert (jb == ref).mean() > 0.99


def test_jbu_validation(glu):
    img = torch.zeros((16, 16, 3), device="cuda")
    low, grid = glu.grid_downsample(img, 4)
    with pytest.raises(ValueError, match="window must be odd"):
        glu.glu.jbu_upsample(img, low, low, grid, glu.glu.JbuParams(window=4))
    with pytest.raises(ValueError, match="sigmas must be > 0"):
        glu.glu.jbu_upsample(img, low, low, grid, glu.glu.JbuParams(sigmaR=0.0))
