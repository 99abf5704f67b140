"""World-size-2 CPU (gloo) tests of the multi-GPU host logic: frame sharding,
row bands with LR halos, and the max-over-ranks timing reduction bench.py uses."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2307_09582_b200 import sharding


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # frame sharding: disjoint clips, nothing exchanged on the data path
        mine = sharding.frame_seeds(rank, world, 16, 3)
        got = [None] * world
        dist.all_gather_object(got, mine)
        flat = [x for r in got for x in r]
        assert len(set(flat)) == 16 * world
        # bands: every rank derives the same partition; owned rows tile the grid
        bands = sharding.row_bands(4320, 16, 3, world)
        allb = [None] * world
        dist.all_gather_object(allb, bands[rank])
        assert [b.lr_rows for b in allb] == [b.lr_rows for b in bands]
        # halo exchange of LR rows: each rank sends its edge rows to neighbours
        lw = 480
        me = bands[rank]
        block = torch.full(((me.lr_rows[1] - me.lr_rows[0]), lw), float(rank))
        halo = {}
        reqs = []
        for nb in (rank - 1, rank + 1):
            if 0 <= nb < world:
                edge = block[:1] if nb < rank else block[-1:]
                reqs.append(dist.isend(edge.contiguous(), nb))
                buf = torch.empty((1, lw))
                reqs.append(dist.irecv(buf, nb))
                halo[nb] = buf
        for r in reqs:
            r.wait()
        for nb, buf in halo.items():
            assert torch.all(buf == float(nb))
        # max-over-ranks timing (bench.py)
        t = torch.tensor([10.0 + rank])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        q.put((rank, float(t.item())))
    finally:
        dist.destroy_process_group()


def test_two_rank_sharding_and_halo_exchange():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(2))
    assert res == [(0, 11.0), (1, 11.0)]


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_row_bands_partition_c4(world):
    bands = sharding.row_bands(4320, 16, 3, world)
    rows = [r for b in bands for r in range(*b.lr_rows)]
    assert rows == list(range(270))
    assert all(b.hr_rows[0] % 16 == 0 for b in bands)
    sizes = [b.lr_rows[1] - b.lr_rows[0] for b in bands]
    assert max(sizes) - min(sizes) <= 1
    if world == 8:
        assert sizes == [34] * 6 + [33] * 2
        assert sharding.halo_bytes(bands[3], 480) == 2 * 480 * 12  # 5,760 B per side


def _log_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2307_09582_b200.distributed import TorchComm
        comm = TorchComm()
        cells = torch.arange(4 * (rank + 1), dtype=torch.int32).reshape(-1, 4) + 100 * rank
        pixels = torch.arange(5 * (2 - rank), dtype=torch.int32).reshape(-1, 5) + 1000 * rank
        logs = comm.all_gather_logs(cells, pixels)
        sums = comm.all_reduce_sum([rank + 1, 10 * rank])
        q.put((rank, [(c.tolist(), p.tolist()) for c, p in logs], sums))
    finally:
        dist.destroy_process_group()


def test_two_rank_change_log_exchange():
    """The distributed joint loop's all-gather of variable-size change logs."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_log_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = dict((r, (logs, sums)) for r, logs, sums in (q.get(timeout=10) for _ in range(2)))
    want = [([[0, 1, 2, 3]], [[0, 1, 2, 3, 4], [5, 6, 7, 8, 9]]),
            ([[100, 101, 102, 103], [104, 105, 106, 107]], [[1000, 1001, 1002, 1003, 1004]])]
    for r in (0, 1):
        assert res[r][0] == want
        assert res[r][1] == [3, 10]


def _banded_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import numpy as np

        import oracle
        from paper_2307_09582_b200 import banded
        from paper_2307_09582_b200.glu import GridSpec
        g = GridSpec.create(40, 48, 8)
        rng = np.random.default_rng(7)
        lown = g.lowW * g.lowH
        full = np.zeros((g.highH, g.highW, 3), np.int32)
        full[..., 0] = rng.integers(0, lown, (g.highH, g.highW))
        full[..., 1] = rng.integers(0, lown, (g.highH, g.highW))
        full[..., 2] = rng.uniform(-0.2, 1.2, (g.highH, g.highW)).astype(np.float32).view(np.int32)
        targets = [torch.from_numpy(rng.uniform(-0.1, 1.1, (g.lowH, g.lowW, 3)).astype(np.float32))
                   for _ in range(3)]
        y0, y1 = banded.band_rows(g, 3, world, rank)
        ora = oracle.Oracle()

        def ora_apply(p, grid, t, clamp):
            P = np.ascontiguousarray(p.numpy()).view(oracle.PARAMS_DTYPE).reshape(p.shape[0], -1)
            return torch.from_numpy(ora.apply_field(P, t.numpy().copy(), clamp))

        outs = {}
        banded.run_banded_apply(torch.from_numpy(full[y0:y1].copy()), g,
                                targets if rank == 0 else None, 3, apply=ora_apply,
                                sink=lambda k, o: outs.__setitem__(k, o.clone()))
        got = [None] * world
        dist.all_gather_object(got, (y0, y1, [outs[k].numpy() for k in range(3)]))
        ok = True
        if rank == 0:
            P = full.view(oracle.PARAMS_DTYPE).reshape(g.highH, g.highW)
            for k in range(3):
                want = ora.apply_field(P, targets[k].numpy())
                cat = np.concatenate([o[2][k] for o in sorted(got, key=lambda o: o[0])])
                ok &= cat.tobytes() == want.tobytes()
            ok &= [o[0] for o in sorted(got)] == [0] + [o[1] for o in sorted(got)][:-1]
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


def test_two_rank_banded_apply_matches_full_apply():
    """C5 over row bands: broadcast targets, per-band apply, outputs tile the frame."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_banded_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = dict(q.get(timeout=10) for _ in range(2))
    assert res == {0: True, 1: True}


def _bands_comm_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2307_09582_b200 import bands
        comm = bands.DistBandComm()
        # variable-length all-gather (change logs, CSR lists, LR rows)
        mine = torch.arange(3 * (rank + 2), dtype=torch.int32).reshape(-1, 3) + 100 * rank
        got = comm.all_gather([mine])[0]
        shapes = [tuple(t.shape) for t in got]
        firsts = [int(t[0, 0]) for t in got]
        sums = comm.all_reduce_sum([[rank + 1, 5]])
        # halo rows of params / errors between neighbouring bands (send / recv)
        H, W = 32, 8
        st = bands.BandState(rank, sharding.row_bands(H, 4, 3, world)[rank],
                             torch.zeros(1), torch.full((H, W, 3), rank, dtype=torch.int32),
                             torch.full((H, W), float(rank)))
        comm.exchange_rows([st], [(0, 1, 12, 16), (1, 0, 16, 20)])
        ok = (bool(torch.all(st.params[12:16] == 0)) and bool(torch.all(st.params[16:20] == 1))
              and bool(torch.all(st.errors[12:20] == torch.tensor([0.0] * 4 + [1.0] * 4)[:, None])))
        q.put((rank, shapes, firsts, sums, ok))
    finally:
        dist.destroy_process_group()


def test_two_rank_band_comm():
    """bands.DistBandComm over gloo: variable-size all-gather, sum all-reduce and
    the neighbour halo exchange of params / errors rows."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bands_comm_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    for _ in range(2):
        rank, shapes, firsts, sums, ok = q.get(timeout=10)
        assert shapes == [(2, 3), (3, 3)] and firsts == [0, 100] and sums == [3, 10] and ok


@pytest.mark.parametrize("world", [2, 3, 5])
def test_seam_merge_matches_full_find_large_error(world):
    """bands._merge (the seam union-find and the global component list) on band
    CCL results equals find_large_error on the whole map (jointopt.cpp:9-46):
    the band CCL is the oracle's here (test stand-in for the kernel); the merge
    is the product code."""
    import numpy as np

    import oracle
    from paper_2307_09582_b200 import bands
    from paper_2307_09582_b200.glu import GridSpec
    ora = oracle.Oracle()
    rng = np.random.default_rng(world)
    H, W, s = 96, 70, 4
    e = (rng.random((H, W)) < 0.45).astype(np.float32)   # percolating blobs cross seams
    e[:, 33] = 1.0                                         # a column through every seam
    g = GridSpec.create(W, H, s)
    bl = sharding.row_bands(H, s, 3, world)
    parts, states = [], []
    for b in bl:
        y0, y1 = b.hr_rows
        mask, comps = ora.find_large_error(e[y0:y1], 0.5)
        lab = np.full((y1 - y0, W), -1, np.int64)
        for c in comps:
            lab.reshape(-1)[c.astype(np.int64)] = int(c[0]) + y0 * W
        off = np.zeros(len(comps) + 1, np.int64)
        off[1:] = np.cumsum([len(c) for c in comps])
        px = (np.concatenate(comps).astype(np.int64) if comps else np.zeros(0, np.int64)) + y0 * W
        parts.append((torch.from_numpy(np.stack([lab[0], lab[-1]])), torch.from_numpy(off),
                      torch.from_numpy(px)))
        states.append(bands.BandState(b.rank, b, torch.zeros(1), torch.zeros(1, dtype=torch.int32),
                                      torch.zeros(1)))
    comm = bands.LocalBandComm(world)
    off, px = bands._merge(states, g, comm, parts)[0]
    _, want = ora.find_large_error(e, 0.5)
    got = [px[off[k]:off[k + 1]].numpy().astype(np.uint32) for k in range(off.numel() - 1)]
    assert len(got) == len(want)
    assert all(a.tobytes() == b.tobytes() for a, b in zip(got, want))
