"""Quality metrics on device buffers against the reference
(proj/src/metrics.cpp, built in oracle/_ref).  Per-window SSIM statistics are
bit-identical; the final means are fixed-order parallel sums, so the tolerance
is the n * 2^-53 bound of a sequential sum (the reference sums sequentially)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("W,H,seed", [(11, 11, 1), (64, 48, 2), (513, 257, 3), (2048, 2048, 4)])
def test_metrics_match_reference(glu, reference, W, H, seed):
    from paper_2307_09582_b200 import workloads
    a = workloads.scene(W, H, seed)
    rng = np.random.default_rng(seed)
    b = np.clip(a + rng.normal(0, 0.02, a.shape), 0, 1).astype(np.float32)
    ref = reference.quality(a, b)
    A, B = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    got = glu.glu.quality_report(A, B)
    # the reference's sequential double sum over n terms is only good to
    # n * 2^-53 relative; ours is a fixed-order tree sum
    tol = max(1e-12, 2 * a.size * 2.0 ** -53)
    assert got["mse"] == pytest.approx(ref[0], rel=tol)
    assert got["psnrDb"] == pytest.approx(ref[1], rel=tol)
    assert got["ssim"] == pytest.approx(ref[2], rel=tol)


def test_metric_pins(glu):
    a = torch.full((16, 16, 3), 0.5, device="cuda")
    assert glu.glu.psnr(a, a) == 99.0          # metrics.cpp:74 sentinel
    assert glu.glu.ssim(a, a) == pytest.approx(1.0, abs=1e-12)
    b = a + 0.1
    assert glu.glu.mse(a, b) == pytest.approx(0.01, rel=1e-6)
    with pytest.raises(ValueError, match="smaller than the 11x11 window"):
        glu.glu.ssim(torch.zeros((10, 10, 3), device="cuda"), torch.zeros((10, 10, 3),
                                                                           device="cuda"))
