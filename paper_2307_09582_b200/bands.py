"""joint_optimize over HR row bands, one band per rank.

The reference loop (jointopt.cpp:182-206) -- downsample, solve, self error map,
then up to N sweeps of find_large_error + trial_update_component -- split into
HR row bands aligned to LR rows (sharding.row_bands: 270 LR rows over 8 ranks
= 34 x 6 + 33 x 2).  Rank b owns the LR rows [L0, L1) and their HR rows and
keeps full-size buffers of which only its band and an R-row halo are valid:

1. **init** -- the band's LR rows are downsampled from its HR rows
   (glu_cu_downsample_band), the LR rows are all-gathered (1.56 MB at 8K; the
   solve needs h rows of halo, the trials read LR anywhere), and the band is
   solved with the self error map fused (glu_cu_solve_band: the band + h LR
   rows as a sub-image, indices rebased).  Then R LR rows (R * s HR rows) of
   params / errors are exchanged with each neighbour (NCCL send/recv).
2. **components** -- find_large_error on the band's error rows
   (glu_cu_find_large_error: union-find with min-index roots), labels made
   global; the seam rows of the labels are all-gathered and a union-find over
   the vertical pairs across seams merges the components that cross a seam
   (root = smallest pixel index, the reference's raster order of first
   pixels).  The band CSR lists are all-gathered, so every rank holds the same
   global component list (a merged component's pixel list is re-sorted).
3. **trials** -- trial i is owned by the band of its first pixel.  Trials i <
   j conflict when their LR cell boxes are within Chebyshev 2h (SURVEY §8(a)
   conflict rule: T_i writes Q_i and params / errors of fp(dilate(Q_i, h)),
   reads LR in dilate(Q_i, 2h)).  round(j) = max over conflicting earlier i of
   round(i) (same owner) or round(i) + 1 (other owner) (glu_trial_rounds).
   Each round, every rank runs its trials of the round with the conflict-aware
   dataflow scheduler (glu_cu_run_trials: conflicting trials in index order),
   logging accepted trials' LR cells and (params, error) pixels; the logs are
   all-gathered and applied.  Every conflicting pair therefore takes effect in
   index order and every trial reads exactly the state the sequential loop
   gives it: the result is bit-identical to the single-GPU loop.  A trial is
   *local* when its affected rows [q0 - h, q1 + h] lie in its owner's band +
   halo; a sweep with a non-local trial (a component taller than the halo)
   all-gathers the bands and runs replicated on every rank instead.
4. **counts** -- accepted / rejected counts are all-reduced per sweep; the loop
   stops exactly where the reference stops.

Measured on the C4 scene (tools/exp_band_rounds.py): 2 rounds per sweep at 4
and 8 ranks (C2: 2), 419..1155 trials per band at 8 ranks, no non-local trial
with R = 4.  `joint_optimize_banded_local` emulates W ranks in one process on
one device (the tests; one GPU is available); `joint_optimize_banded` runs over
torch.distributed (NCCL on GPUs; gloo stages through the host).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from . import sharding
from .glu import (GluConfig, GridSpec, JointResult, Mode, ParamField, _ptr, context,
                  find_large_error)

HALO = 4  # LR rows of params / errors halo around a band (>= 2h + 2 for S = 3)


@dataclass
class BandState:
    rank: int
    band: sharding.Band
    low: torch.Tensor      # (lh, lw, 3): full LR replica
    params: torch.Tensor   # (H, W, 3) int32: band + halo valid
    errors: torch.Tensor   # (H, W): band + halo valid
    log: object = None


class _Log:
    """Device change log of glu_cu_run_trials (accepted trials only), grown to
    the bound of a round's trials: <= qw qh replaced cells and (qw + 2h)(qh + 2h)
    s^2 affected pixels per trial (q = the component's cell box)."""

    def __init__(self, device):
        self.device = device
        self.counts = torch.zeros(3, dtype=torch.int32, device=device)
        self.cells = self.pixels = None
        self.c = None

    def reserve(self, ncells: int, npixels: int):
        if self.c is not None and self.c.cellCapacity >= ncells and \
                self.c.pixelCapacity >= npixels:
            return
        ncells, npixels = max(ncells, 1024), max(npixels, 1 << 16)
        self.cells = torch.empty((ncells, 4), dtype=torch.int32, device=self.device)
        self.pixels = torch.empty((npixels, 5), dtype=torch.int32, device=self.device)
        self.c = N.GluTrialLog(self.counts.data_ptr(), self.cells.data_ptr(),
                               self.pixels.data_ptr(), ncells, npixels)

    def used(self):
        """The logged (cells, pixels), one entry per index: trials of a round
        that conflict commit in index order and log at commit time, so the
        last entry of an index is its final value (the apply kernel writes
        the entries in parallel, in no order)."""
        n = self.counts[:2].cpu().tolist()
        return _last_per_index(self.cells[:n[0]]), _last_per_index(self.pixels[:n[1]])

    def used_raw(self):
        n = self.counts[:2].cpu().tolist()
        return self.cells[:n[0]], self.pixels[:n[1]]


def _last_per_index(entries: torch.Tensor) -> torch.Tensor:
    """Rows of an (n, k) int32 log whose column 0 (the index) is not repeated
    later in the log."""
    n = entries.shape[0]
    if n == 0:
        return entries
    idx = entries[:, 0].to(torch.int64) & 0xFFFFFFFF
    uniq, inv = torch.unique(idx, return_inverse=True)
    pos = torch.arange(n, device=entries.device)
    last = torch.full((uniq.numel(),), -1, dtype=torch.int64, device=entries.device)
    last = last.scatter_reduce(0, inv, pos, reduce="amax")
    return entries[last]


# ---- communication: real ranks (torch.distributed) or emulated ranks --------------

class LocalBandComm:
    """Every rank of the job lives in this process (emulation on one device):
    collectives are list operations, the halo exchange device copies."""

    def __init__(self, world: int):
        self.world = world
        self.ranks = list(range(world))

    def all_gather(self, mine: list[torch.Tensor]) -> list[list[torch.Tensor]]:
        return [mine for _ in mine]

    def all_reduce_sum(self, vals: list[list[int]]) -> list[int]:
        return [int(sum(v[k] for v in vals)) for k in range(len(vals[0]))]

    def exchange_rows(self, states: list[BandState], rows: list[tuple[int, int, int, int]]):
        """rows[k] = (src rank, dst rank, y0, y1): copy HR rows [y0, y1) of
        params and errors from src's buffers into dst's."""
        for src, dst, y0, y1 in rows:
            states[dst].params[y0:y1] = states[src].params[y0:y1]
            states[dst].errors[y0:y1] = states[src].errors[y0:y1]


class DistBandComm:
    """One rank per process over torch.distributed (NCCL for CUDA tensors; a
    gloo group stages through the host)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.ranks = [self.rank]
        self.cpu = dist.get_backend(group) == "gloo"

    def _stage(self, t):
        return t.cpu() if self.cpu else t

    def all_gather(self, mine: list[torch.Tensor]) -> list[list[torch.Tensor]]:
        """Variable-length first dimension, same trailing shape and dtype."""
        (t,) = mine
        dev = t.device
        n = self._stage(torch.tensor([t.shape[0]], dtype=torch.int64, device=dev))
        ns = [torch.empty_like(n) for _ in range(self.world)]
        self.dist.all_gather(ns, n, group=self.group)
        m = max(int(x.item()) for x in ns)
        pad = torch.zeros((max(m, 1),) + tuple(t.shape[1:]), dtype=t.dtype, device=dev)
        pad[:t.shape[0]] = t
        pad = self._stage(pad)
        outs = [torch.empty_like(pad) for _ in range(self.world)]
        self.dist.all_gather(outs, pad, group=self.group)
        return [[o[:int(k.item())].to(dev) for o, k in zip(outs, ns)]]

    def all_reduce_sum(self, vals: list[list[int]]) -> list[int]:
        t = torch.tensor(vals[0], dtype=torch.int64)
        if not self.cpu:
            t = t.cuda()
        self.dist.all_reduce(t, group=self.group)
        return [int(v) for v in t.cpu().tolist()]

    def exchange_rows(self, states: list[BandState], rows: list[tuple[int, int, int, int]]):
        (st,) = states
        ops, recvs = [], []
        for src, dst, y0, y1 in rows:
            for buf in (st.params, st.errors):
                if src == self.rank:
                    ops.append(self.dist.P2POp(self.dist.isend, self._stage(buf[y0:y1].contiguous()),
                                               dst, self.group))
                elif dst == self.rank:
                    tmp = self._stage(torch.empty_like(buf[y0:y1]))
                    recvs.append((buf, y0, y1, tmp))
                    ops.append(self.dist.P2POp(self.dist.irecv, tmp, src, self.group))
        if ops:
            for w in self.dist.batch_isend_irecv(ops):
                w.wait()
        for buf, y0, y1, tmp in recvs:
            buf[y0:y1] = tmp.to(buf.device)


# ---- the loop ------------------------------------------------------------------------

def _ctx(t: torch.Tensor):
    return context(t.device.index)


def _band_components(st: BandState, grid: GridSpec, tau: float):
    """Band-local find_large_error (glu_cu_find_large_error, the sparse
    variant the joint loop uses) made global: the labels (first pixel, -1
    outside the mask) of the band's first and last HR rows, the band CSR
    offsets and the pixels as global indices."""
    y0, y1 = st.band.hr_rows
    W, hb = grid.highW, y1 - y0
    dev = st.errors.device
    n = C.c_size_t()
    off, px = C.c_void_p(), C.c_void_p()
    ctx = _ctx(st.errors)
    N.check(N.lib().glu_cu_find_large_error(ctx.handle, _ptr(st.errors[y0:y1]), W, hb,
                                            float(tau), C.c_void_p(0), C.c_void_p(0), C.byref(n),
                                            C.byref(off), C.byref(px)))
    offsets = torch.zeros(n.value + 1, dtype=torch.int32, device=dev)
    pixels = torch.empty(0, dtype=torch.int32, device=dev)
    m = 0
    if n.value:
        N.check(N.lib().glu_cu_copy(ctx.handle, _ptr(offsets), off, (n.value + 1) * 4))
        m = int(offsets[-1].item())
        pixels = torch.empty(m, dtype=torch.int32, device=dev)
        N.check(N.lib().glu_cu_copy(ctx.handle, _ptr(pixels), px, m * 4))
    base = y0 * W
    offsets, pixels = offsets.to(torch.int64), pixels.to(torch.int64)
    edge = torch.full((2, W), -1, dtype=torch.int64, device=dev)
    if m:
        # each pixel's label (its component's first pixel), scattered into
        # the band's first and last rows
        comp = torch.repeat_interleave(torch.arange(n.value, device=dev), torch.diff(offsets),
                                       output_size=m)
        lab = pixels[offsets[:-1]][comp] + base
        top = pixels < W
        edge[0, pixels[top]] = lab[top]
        bot = pixels >= (hb - 1) * W
        edge[1, pixels[bot] - (hb - 1) * W] = lab[bot]
    return edge, offsets, pixels + base


def _merge(states, grid: GridSpec, comm, parts):
    """The global component CSR (identical on every rank) from the band parts:
    components touching across a seam are merged (union-find over the labels
    of the vertical pixel pairs across each seam; root = smallest label, i.e.
    the component's first pixel)."""
    dev = states[0].params.device
    edges = comm.all_gather([p[0] for p in parts])
    offs = comm.all_gather([p[1] for p in parts])
    pixs = comm.all_gather([p[2] for p in parts])
    out = []
    for k in range(len(states)):
        rows = [e.cpu().numpy() for e in edges[k]]          # per band: (2, W) labels
        parent: dict[int, int] = {}

        def find(x):
            root = x
            while parent.get(root, root) != root:
                root = parent[root]
            while parent.get(x, x) != root:
                parent[x], x = root, parent[x]
            return root

        for b in range(len(rows) - 1):
            lo, up = rows[b][1], rows[b + 1][0]
            both = (lo >= 0) & (up >= 0)
            for u, v in set(zip(lo[both].tolist(), up[both].tolist())):
                ru, rv = find(u), find(v)
                if ru != rv:
                    parent[max(ru, rv)] = min(ru, rv)
        bpix = list(pixs[k])
        boff = list(offs[k])
        # every band component in band order: global first pixel, start, size
        # (the band lists concatenated are the global list in first-pixel
        # order when nothing merges)
        shift, starts, sizes_l = 0, [], []
        for o in boff:
            starts.append(o[:-1] + shift)
            sizes_l.append(torch.diff(o))
            shift += int(o[-1]) if o.numel() else 0
        allpix = torch.cat(bpix) if bpix else torch.zeros(0, dtype=torch.int64)
        start = torch.cat(starts) if starts else torch.zeros(0, dtype=torch.int64)
        sizes = torch.cat(sizes_l) if sizes_l else torch.zeros(0, dtype=torch.int64)
        pixels = allpix
        if parent:
            member = {}
            for x in list(parent):
                r = find(x)
                member[x] = r
                member[r] = r  # (a root is never a key of `parent`)
            # the few components that merge: the root keeps its place with the
            # group's pixels re-sorted, the other members are dropped; the
            # lists between them are copied as whole slices
            firsts = allpix[start.to(allpix.device)].cpu().numpy() if start.numel() else []
            special = [c for c, f in enumerate(firsts.tolist()) if f in member]
            start_h, size_h = start.tolist(), sizes.tolist()
            groups: dict[int, list] = {}
            for c in special:
                groups.setdefault(member[int(firsts[c])], []).append(c)
            chunks, new_sizes, prev = [], [], 0
            for c in special:
                chunks.append(allpix[start_h[prev] if prev < len(start_h) else 0:start_h[c]]
                              if c > prev else allpix[0:0])
                new_sizes.append(sizes[prev:c])
                root = member[int(firsts[c])]
                if int(firsts[c]) == root:
                    merged = torch.sort(torch.cat([allpix[start_h[m]:start_h[m] + size_h[m]]
                                                   for m in groups[root]])).values
                    chunks.append(merged)
                    new_sizes.append(torch.tensor([merged.numel()], dtype=torch.int64,
                                                  device=sizes.device))
                prev = c + 1
            if prev < len(start_h):
                chunks.append(allpix[start_h[prev]:])
                new_sizes.append(sizes[prev:])
            pixels = torch.cat(chunks)
            sizes = torch.cat(new_sizes)
        off = torch.zeros(sizes.numel() + 1, dtype=torch.int32, device=dev)
        if sizes.numel():
            off[1:] = torch.cumsum(sizes.to(dev), 0).to(torch.int32)
        out.append((off, pixels.to(torch.int32).to(dev)))
    return out


def _boxes(off, pixels, grid: GridSpec, device) -> np.ndarray:
    n = off.numel() - 1
    boxes = torch.empty((max(n, 1), 4), dtype=torch.int32, device=device)
    if n:
        N.check(N.lib().glu_cu_component_boxes(context(device.index).handle, _ptr(off),
                                               _ptr(pixels), n, C.byref(grid.c()), _ptr(boxes)))
    return np.ascontiguousarray(boxes[:n].cpu().numpy())


def _rounds(boxes: np.ndarray, owners: np.ndarray, reach: int) -> np.ndarray:
    n = boxes.shape[0]
    rounds = np.zeros(n, np.int32)
    ow = np.ascontiguousarray(owners, np.int32)
    N.check(N.lib().glu_trial_rounds(C.c_void_p(boxes.ctypes.data), n, reach,
                                     C.c_void_p(ow.ctypes.data), C.c_void_p(rounds.ctypes.data)))
    return rounds


def _run(st: BandState, high, grid, cfg, mode, off, pixels, ids: np.ndarray, log):
    acc, rej = C.c_int(), C.c_int()
    dids = torch.as_tensor(ids.astype(np.int32), device=high.device)
    N.check(N.lib().glu_cu_run_trials(
        _ctx(high).handle, _ptr(high), _ptr(st.low), _ptr(st.params), _ptr(st.errors),
        C.byref(grid.c()), C.byref(cfg.c()), int(mode), _ptr(off), _ptr(pixels),
        _ptr(dids) if ids.size else C.c_void_p(0), int(ids.size),
        C.byref(log.c) if log is not None else None, C.byref(acc), C.byref(rej)))
    return acc.value, rej.value


def _apply_log(st: BandState, high, cells, pixels):
    if cells.shape[0] == 0 and pixels.shape[0] == 0:
        return
    cells, pixels = cells.contiguous(), pixels.contiguous()
    N.check(N.lib().glu_cu_apply_trial_log(
        _ctx(high).handle, _ptr(st.low), _ptr(st.params), _ptr(st.errors),
        _ptr(cells) if cells.numel() else C.c_void_p(0), cells.shape[0],
        _ptr(pixels) if pixels.numel() else C.c_void_p(0), pixels.shape[0]))


def _banded_loop(high: torch.Tensor, scale: int, cfg: GluConfig, mode, comm, stats: dict):
    cfg.validate()
    H, W = high.shape[:2]
    g = GridSpec.create(W, H, scale)
    h = cfg.windowSide // 2
    R = max(HALO, 2 * h + 2)
    bands = sharding.row_bands(H, scale, cfg.windowSide, comm.world)
    if min(b.lr_rows[1] - b.lr_rows[0] for b in bands) < R and comm.world > 1:
        raise ValueError(f"banded joint_optimize: every band needs >= {R} LR rows")
    dev = high.device
    states = []
    for r in comm.ranks:
        states.append(BandState(
            r, bands[r],
            torch.empty((g.lowH, g.lowW, 3), dtype=torch.float32, device=dev),
            torch.empty((H, W, 3), dtype=torch.int32, device=dev),
            torch.empty((H, W), dtype=torch.float32, device=dev)))
    ctx = _ctx(high)
    # 1. init: band downsample, LR all-gather, band solve + self error, halo exchange
    for st in states:
        r0, r1 = st.band.lr_rows
        N.check(N.lib().glu_cu_downsample_band(ctx.handle, _ptr(high), C.byref(g.c()), r0, r1,
                                               _ptr(st.low)))
    rows = comm.all_gather([st.low[st.band.lr_rows[0]:st.band.lr_rows[1]] for st in states])
    for k, st in enumerate(states):
        st.low.copy_(torch.cat(rows[k]))
    for st in states:
        r0, r1 = st.band.lr_rows
        N.check(N.lib().glu_cu_solve_band(ctx.handle, _ptr(high), _ptr(st.low), C.byref(g.c()),
                                          C.byref(cfg.c()), int(mode), r0, r1, _ptr(st.params),
                                          _ptr(st.errors)))
    halo = []
    for b in range(comm.world - 1):
        ya = max(0, bands[b].lr_rows[1] - R) * scale       # band b's bottom R rows -> b + 1
        yb = bands[b].hr_rows[1]
        yc = bands[b + 1].hr_rows[0]                       # band b+1's top R rows -> b
        yd = min(H, (bands[b + 1].lr_rows[0] + R) * scale)
        halo += [(b, b + 1, ya, yb), (b + 1, b, yc, yd)]
    comm.exchange_rows(states, halo)
    for st in states:
        st.log = _Log(dev)
    # 2-4. sweeps
    reach = 2 * h
    starts = np.array([b.lr_rows[0] for b in bands])
    for _ in range(cfg.maxIterations):
        parts = [_band_components(st, g, cfg.errorThreshold) for st in states]
        comps = _merge(states, g, comm, parts)
        n = comps[0][0].numel() - 1
        if n == 0:
            break
        stats["iterations"] += 1
        stats["components"] += n
        boxes = _boxes(comps[0][0], comps[0][1], g, dev)
        owners = np.searchsorted(starts, boxes[:, 1], side="right") - 1
        lo = starts[owners] - R
        hi = np.array([bands[o].lr_rows[1] for o in owners]) + R
        local = ((boxes[:, 1] - h >= lo) & (boxes[:, 3] + h < hi)) | (comm.world == 1)
        acc = rej = 0
        if local.all():
            rounds = _rounds(boxes, owners, reach)
            stats["rounds"].append(int(rounds.max()) + 1)
            for rd in range(int(rounds.max()) + 1):
                logs = []
                for k, st in enumerate(states):
                    ids = np.nonzero((rounds == rd) & (owners == st.rank))[0]
                    log = None
                    if comm.world > 1:
                        qw = (boxes[ids, 2] - boxes[ids, 0] + 1).astype(np.int64)
                        qh = (boxes[ids, 3] - boxes[ids, 1] + 1).astype(np.int64)
                        st.log.reserve(int((qw * qh).sum()),
                                       int(((qw + 2 * h) * (qh + 2 * h)).sum()) * scale * scale)
                        log = st.log
                    a, b = _run(st, high, g, cfg, mode, comps[k][0], comps[k][1], ids, log)
                    acc += a
                    rej += b
                    if log is not None:
                        logs.append(log.used())
                if comm.world > 1:
                    cells = comm.all_gather([c for c, _ in logs])
                    pixels = comm.all_gather([p for _, p in logs])
                    for k, st in enumerate(states):
                        for src in range(comm.world):
                            if src != st.rank:
                                _apply_log(st, high, cells[k][src], pixels[k][src])
        else:
            # a trial reaches beyond its owner's halo: gather every band and
            # run the sweep replicated (identical on every rank)
            stats["replicated_sweeps"] += 1
            for name in ("params", "errors"):
                got = comm.all_gather([getattr(st, name)[st.band.hr_rows[0]:st.band.hr_rows[1]]
                                       for st in states])
                for k, st in enumerate(states):
                    getattr(st, name).copy_(torch.cat(got[k]))
            for k, st in enumerate(states):
                a, b = _run(st, high, g, cfg, mode, comps[k][0], comps[k][1],
                            np.arange(n, dtype=np.int32), None)
                if st.rank == 0:  # every rank ran every trial: count them once
                    acc, rej = a, b
        tot = comm.all_reduce_sum([[acc, rej]])
        stats["accepted"] += tot[0]
        stats["rejected"] += tot[1]
        if tot[0] == 0:
            break
    return g, states


def _new_stats():
    return {"iterations": 0, "accepted": 0, "rejected": 0, "components": 0, "rounds": [],
            "replicated_sweeps": 0}


def joint_optimize_banded(high: torch.Tensor, scale: int, cfg: GluConfig | None = None,
                          mode: Mode = Mode.Fast, group=None):
    """joint_optimize over the ranks of a torch.distributed group, one HR row
    band per rank.  Returns (this rank's BandState, grid, stats); the band's
    HR rows of params / errors and the full LR image are the reference's."""
    comm = DistBandComm(group)
    stats = _new_stats()
    g, states = _banded_loop(high, scale, cfg or GluConfig(), mode, comm, stats)
    return states[0], g, stats


def joint_optimize_banded_local(high: torch.Tensor, scale: int, world: int,
                                cfg: GluConfig | None = None, mode: Mode = Mode.Fast):
    """Emulate a `world`-rank banded job in this process; returns the
    assembled JointResult (each band's rows from its rank, LR from rank 0),
    the per-rank states and stats."""
    comm = LocalBandComm(world)
    stats = _new_stats()
    g, states = _banded_loop(high, scale, cfg or GluConfig(), mode, comm, stats)
    params = torch.empty_like(states[0].params)
    errors = torch.empty_like(states[0].errors)
    for st in states:
        y0, y1 = st.band.hr_rows
        params[y0:y1] = st.params[y0:y1]
        errors[y0:y1] = st.errors[y0:y1]
    res = JointResult(states[0].low, ParamField(g, Mode(mode), params), errors,
                      stats["iterations"], stats["accepted"], stats["rejected"],
                      stats["components"])
    return res, states, stats
