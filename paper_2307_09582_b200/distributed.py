"""Multi-GPU joint optimisation (BASELINE.json configs[3] / SURVEY §8(e)).

Level-synchronous, replicated-state decomposition of joint_optimize
(jointopt.cpp:182-206):

* every rank holds the full LR image, parameter field and error map and runs
  the (cheap, deterministic) init and find_large_error itself, so all ranks see
  the same components in the same order;
* the components of a sweep are grouped into levels (glu_trial_levels): a
  component's level is one more than the highest level of any earlier component
  whose cell box is within 2h (Chebyshev).  Trials of one level touch disjoint
  state, so any order -- and any split across ranks -- gives the reference's
  sequential result;
* per level each rank runs its round-robin share of the trials with a change
  log of the accepted ones (glu_cu_run_trials), the logs are all-gathered and
  every rank applies the others' changes (glu_cu_apply_trial_log);
* the sweep's accept / reject counts are summed across ranks; the loop stops
  exactly where the reference stops.

The first sweep of the C4 scene has 122 levels (C2: 159: chains of nearby
components), so a sweep costs a few hundred small all-gathers; on one GPU the
dataflow scheduler (glu_joint.cu k_trial_sched) is faster than any level
schedule, and this module is the multi-rank decomposition.  `joint_optimize_local` runs W ranks inside one process on one
device (what the tests use: one GPU is available); `joint_optimize_distributed`
uses torch.distributed (NCCL for CUDA tensors, gloo via host staging).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .glu import (GluConfig, GridSpec, JointResult, Mode, ParamField, _ptr, context,
                  find_large_error, joint_optimize)


@dataclass
class RankState:
    low: torch.Tensor
    params: torch.Tensor
    errors: torch.Tensor


class TorchComm:
    """All-gather of per-rank change logs over torch.distributed."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.cpu = dist.get_backend(group) == "gloo"

    def all_gather_logs(self, cells: torch.Tensor, pixels: torch.Tensor):
        """cells (n, 4) and pixels (m, 5) int32 of this rank -> [(cells, pixels)] per rank."""
        dev = cells.device
        stage = (lambda t: t.cpu()) if self.cpu else (lambda t: t)
        sizes = stage(torch.tensor([cells.shape[0], pixels.shape[0]], dtype=torch.int64,
                                   device=dev))
        all_sizes = [torch.empty_like(sizes) for _ in range(self.world)]
        self.dist.all_gather(all_sizes, sizes, group=self.group)
        mc = max(int(s[0]) for s in all_sizes)
        mp = max(int(s[1]) for s in all_sizes)
        pc = torch.zeros((max(mc, 1), 4), dtype=torch.int32, device=dev)
        pp = torch.zeros((max(mp, 1), 5), dtype=torch.int32, device=dev)
        pc[:cells.shape[0]] = cells
        pp[:pixels.shape[0]] = pixels
        pc, pp = stage(pc), stage(pp)
        gc = [torch.empty_like(pc) for _ in range(self.world)]
        gp = [torch.empty_like(pp) for _ in range(self.world)]
        self.dist.all_gather(gc, pc, group=self.group)
        self.dist.all_gather(gp, pp, group=self.group)
        return [(gc[r][:int(all_sizes[r][0])].to(dev), gp[r][:int(all_sizes[r][1])].to(dev))
                for r in range(self.world)]

    def all_reduce_sum(self, values: list[int]) -> list[int]:
        t = torch.tensor(values, dtype=torch.int64)
        if not self.cpu:
            t = t.cuda()
        self.dist.all_reduce(t, group=self.group)
        return [int(v) for v in t.cpu().tolist()]


class _Log:
    def __init__(self, npx: int, lowN: int, device):
        self.counts = torch.zeros(3, dtype=torch.int32, device=device)
        self.cells = torch.empty((lowN, 4), dtype=torch.int32, device=device)
        self.pixels = torch.empty((npx, 5), dtype=torch.int32, device=device)
        self.c = N.GluTrialLog(self.counts.data_ptr(), self.cells.data_ptr(),
                               self.pixels.data_ptr(), lowN, npx)

    def used(self):
        n = self.counts[:2].cpu().tolist()
        return self.cells[:n[0]].clone(), self.pixels[:n[1]].clone()


def _run_level(st: RankState, high, g, cfg: GluConfig, mode, les, ids: np.ndarray, log: _Log):
    ctx = context(high.device.index)
    dids = torch.as_tensor(ids.astype(np.int32), device=high.device)
    acc, rej = C.c_int(), C.c_int()
    N.check(N.lib().glu_cu_run_trials(ctx.handle, _ptr(high), _ptr(st.low), _ptr(st.params),
                                      _ptr(st.errors), C.byref(g.c()), C.byref(cfg.c()),
                                      int(mode), _ptr(les.offsets), _ptr(les.pixels),
                                      _ptr(dids) if ids.size else C.c_void_p(0), int(ids.size),
                                      C.byref(log.c), C.byref(acc), C.byref(rej)))
    return acc.value, rej.value


def _apply(st: RankState, high, cells: torch.Tensor, pixels: torch.Tensor):
    if cells.shape[0] == 0 and pixels.shape[0] == 0:
        return
    ctx = context(high.device.index)
    cells, pixels = cells.contiguous(), pixels.contiguous()
    N.check(N.lib().glu_cu_apply_trial_log(ctx.handle, _ptr(st.low), _ptr(st.params),
                                           _ptr(st.errors),
                                           _ptr(cells) if cells.numel() else C.c_void_p(0),
                                           cells.shape[0],
                                           _ptr(pixels) if pixels.numel() else C.c_void_p(0),
                                           pixels.shape[0]))


def trial_levels(les, grid: GridSpec, windowSide: int, device) -> np.ndarray:
    """Level (1-based) of every component of `les` (glu_trial_levels)."""
    n = len(les)
    boxes = torch.empty((n, 4), dtype=torch.int32, device=device)
    ctx = context(device.index)
    N.check(N.lib().glu_cu_component_boxes(ctx.handle, _ptr(les.offsets), _ptr(les.pixels), n,
                                           C.byref(grid.c()), _ptr(boxes)))
    hb = np.ascontiguousarray(boxes.cpu().numpy())
    levels = np.zeros(n, np.int32)
    N.check(N.lib().glu_trial_levels(C.c_void_p(hb.ctypes.data), n, 2 * (windowSide // 2),
                                     C.c_void_p(levels.ctypes.data)))
    return levels


def _joint_ranks(high, scale, cfg: GluConfig, mode, ranks: list[int], world: int, exchange,
                 reduce):
    """The loop for the ranks `ranks` (of a `world`-rank job) living in this
    process.  exchange(list of this process's logs) -> every rank's log;
    reduce([accepted, rejected]) -> job-wide sums."""
    init_cfg = GluConfig(cfg.windowSide, cfg.errorThreshold, 0, cfg.epsilon,
                         cfg.literalComponentUpdate)
    r0 = joint_optimize(high, scale, init_cfg, mode)  # downsample + solve + error map
    g = r0.field.grid
    states = [RankState(r0.low.clone(), r0.field.params.clone(), r0.errors.clone())
              for _ in ranks]
    logs = [_Log(g.highW * g.highH, g.lowW * g.lowH, high.device) for _ in ranks]
    stats = {"iterations": 0, "accepted": 0, "rejected": 0, "levels": []}
    for _ in range(cfg.maxIterations):
        les = find_large_error(states[0].errors, cfg.errorThreshold)
        n = len(les)
        if n == 0:
            break
        stats["iterations"] += 1
        levels = trial_levels(les, g, cfg.windowSide, high.device)
        stats["levels"].append(int(levels.max()))
        owner = np.arange(n) % world
        acc = rej = 0
        for L in range(1, int(levels.max()) + 1):
            mine = []
            for k, (rk, st) in enumerate(zip(ranks, states)):
                ids = np.nonzero((levels == L) & (owner == rk))[0]
                a, b = _run_level(st, high, g, cfg, mode, les, ids, logs[k])
                acc += a
                rej += b
                mine.append(logs[k].used())
            everyone = exchange(mine)
            for k, (rk, st) in enumerate(zip(ranks, states)):
                for src, (cells, pixels) in enumerate(everyone):
                    if src != rk:
                        _apply(st, high, cells, pixels)
        acc, rej = reduce([acc, rej])
        stats["accepted"] += acc
        stats["rejected"] += rej
        if acc == 0:
            break
    return g, states, stats


def joint_optimize_distributed(high: torch.Tensor, scale: int, cfg: GluConfig | None = None,
                               mode: Mode = Mode.Fast, group=None) -> JointResult:
    """joint_optimize across the ranks of a torch.distributed group (one rank per
    GPU); returns this rank's replica of the (identical) result."""
    comm = TorchComm(group)
    g, states, st = _joint_ranks(high, scale, cfg or GluConfig(), mode, [comm.rank], comm.world,
                                 lambda mine: comm.all_gather_logs(*mine[0]),
                                 comm.all_reduce_sum)
    s = states[0]
    return JointResult(s.low, ParamField(g, Mode(mode), s.params), s.errors, st["iterations"],
                       st["accepted"], st["rejected"])


def joint_optimize_local(high: torch.Tensor, scale: int, world: int,
                         cfg: GluConfig | None = None, mode: Mode = Mode.Fast):
    """Emulate a `world`-rank job inside this process (all replicas on one
    device); returns (one JointResult per rank, stats)."""
    g, states, st = _joint_ranks(high, scale, cfg or GluConfig(), mode, list(range(world)),
                                 world, lambda mine: mine, lambda v: v)
    return [JointResult(s.low, ParamField(g, Mode(mode), s.params), s.errors, st["iterations"],
                        st["accepted"], st["rejected"]) for s in states], st
