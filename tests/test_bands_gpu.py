"""The banded multi-GPU joint loop (paper_2307_09582_b200/bands.py: init per
HR row band with an LR halo, band CCL + seam merge, trials owned by bands in
rounds with change logs) is bit-identical to the single-GPU joint_optimize
(itself bit-identical to the reference, tests/test_full_configs_gpu.py).

One GPU is available: W ranks are emulated in one process (separate state per
rank, collectives as list operations), and the real torch.distributed path runs
as 2 processes on the same GPU over gloo (host-staged collectives: no kernel of
one process waits on the other's)."""
import os
import socket

import pytest
import torch

pytestmark = pytest.mark.gpu


def _same(a, b):
    return (a.iterations, a.trialsAccepted, a.trialsRejected) == \
        (b.iterations, b.trialsAccepted, b.trialsRejected) and torch.equal(a.low, b.low) and \
        torch.equal(a.field.params, b.field.params) and torch.equal(a.errors, b.errors)


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("W,H,s,S,mode", [(1024, 1024, 8, 3, "fast"), (960, 720, 6, 5, "fast"),
                                          (800, 640, 8, 3, "exact"), (800, 600, 4, 3, "gnu")])
def test_banded_emulated_matches_single_gpu(glu, world, W, H, s, S, mode):
    from paper_2307_09582_b200 import bands, workloads
    high = torch.from_numpy(workloads.scene(W, H, 70 + s)).cuda()
    cfg = glu.GluConfig(windowSide=S)
    md = glu.mode_from_name(mode)
    ref = glu.joint_optimize(high, s, cfg, md)
    res, states, stats = bands.joint_optimize_banded_local(high, s, world, cfg, md)
    assert ref.trialsAccepted > 10
    assert _same(res, ref), (stats, ref.iterations, ref.trialsAccepted, ref.trialsRejected)
    if world > 1:  # (a component taller than the halo makes its sweep replicated)
        assert stats["replicated_sweeps"] < stats["iterations"] or stats["iterations"] == 0


def test_banded_c4_eight_ranks(glu):
    """BASELINE configs[3] (7680x4320, s = 16) over 8 emulated bands (34 x 6 + 33 x 2
    LR rows): the same LR image, params, errors and counts as one GPU."""
    from paper_2307_09582_b200 import bands, workloads
    high = torch.from_numpy(workloads.scene(7680, 4320, 4, 0)).cuda()
    ref = glu.joint_optimize(high, 16)
    for world in (2, 8):
        res, _, stats = bands.joint_optimize_banded_local(high, 16, world)
        assert _same(res, ref), (world, stats)
        assert stats["replicated_sweeps"] == 0


def test_banded_seam_components_and_replicated_sweep(glu):
    """Components crossing seams (merged by the seam union-find) and a noise
    image whose single huge component exceeds every band's halo (that sweep runs
    replicated); literal scope."""
    import numpy as np
    from paper_2307_09582_b200 import bands, workloads
    rng = np.random.default_rng(3)
    img = workloads.scene(640, 512, 12).copy()
    for x in range(0, 640, 37):  # vertical lines cross every seam
        img[:, x, :] = rng.random(3)
    high = torch.from_numpy(img).cuda()
    for lit in (False, True):
        cfg = glu.GluConfig(literalComponentUpdate=lit)
        ref = glu.joint_optimize(high, 4, cfg)
        for world in (2, 5):
            res, _, stats = bands.joint_optimize_banded_local(high, 4, world, cfg)
            assert _same(res, ref), (lit, world, stats)
    noise = torch.from_numpy(rng.random((256, 320, 3), dtype=np.float32)).cuda()
    ref = glu.joint_optimize(noise, 4)
    res, _, stats = bands.joint_optimize_banded_local(noise, 4, 4)
    assert stats["replicated_sweeps"] >= 1
    assert _same(res, ref)


def _free_port():
    with socket.socket() as sck:
        sck.bind(("127.0.0.1", 0))
        return sck.getsockname()[1]


def _dist_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2307_09582_b200 as glu
        from paper_2307_09582_b200 import bands, workloads
        torch.cuda.set_device(0)
        high = torch.from_numpy(workloads.scene(768, 640, 81)).cuda()
        st, g, stats = bands.joint_optimize_banded(high, 8)
        ref = glu.joint_optimize(high, 8)
        y0, y1 = st.band.hr_rows
        ok = torch.equal(st.params[y0:y1], ref.field.params[y0:y1]) and \
            torch.equal(st.errors[y0:y1], ref.errors[y0:y1]) and torch.equal(st.low, ref.low) and \
            (stats["iterations"], stats["accepted"], stats["rejected"]) == \
            (ref.iterations, ref.trialsAccepted, ref.trialsRejected)
        q.put((rank, bool(ok), stats["rounds"]))
    finally:
        dist.destroy_process_group()


def test_banded_two_processes_torch_distributed(glu):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dist_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    res = [q.get(timeout=10) for _ in range(2)]
    assert all(ok for _, ok, _ in res), res
