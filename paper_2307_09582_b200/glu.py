"""Host-side mirror of the reference's hot-path interface over device tensors.

Same names, argument meaning and error behaviour as
/root/reference/proj/include/glu/{grid,params,upsample,jointopt}.hpp; every
call goes through the C-ABI (include/glu_cuda.h) into the sm_100a kernels.

Data lives in torch CUDA tensors (torch is only the allocator / stream owner):
  image  : float32 (H, W, 3) contiguous, interleaved RGB (image.hpp:13-23)
  params : int32 (H, W, 3) contiguous = the 12-byte {u32 a, u32 b, f32 w}
           records of params.hpp:42-46 (use ParamField.numpy() to view them)
  errors : float32 (H, W)
Validation failures raise ValueError carrying the reference's
std::invalid_argument text.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field as dc_field

import numpy as np
import torch

from . import _native as N

PARAMS_DTYPE = np.dtype([("a", "<u4"), ("b", "<u4"), ("w", "<f4")])


class Mode(enum.IntEnum):
    """glu::Mode (params.hpp:11-15)."""
    Fast = 0
    Exact = 1
    Gnu = 2


def mode_from_name(name: str) -> Mode:
    """mode_from_name (upsample.cpp:19-24)."""
    table = {"fast": Mode.Fast, "exact": Mode.Exact, "gnu": Mode.Gnu}
    if name not in table:
        raise ValueError(f"unknown mode: {name} (expected fast|exact|gnu)")
    return table[name]


def mode_name(m: Mode) -> str:
    return {Mode.Fast: "fast", Mode.Exact: "exact", Mode.Gnu: "gnu"}[Mode(m)]


@dataclass(frozen=True)
class GridSpec:
    """glu::GridSpec (grid.hpp:19-39; create: grid.cpp:8-23)."""
    scale: int
    highW: int
    highH: int
    lowW: int
    lowH: int
    sampleOffset: int

    @staticmethod
    def create(highW: int, highH: int, scale: int) -> "GridSpec":
        g = N.GluGrid()
        N.check(N.lib().glu_grid_create(int(highW), int(highH), int(scale), C.byref(g)))
        return GridSpec(g.scale, g.highW, g.highH, g.lowW, g.lowH, g.sampleOffset)

    def c(self) -> N.GluGrid:
        return N.GluGrid(self.scale, self.highW, self.highH, self.lowW, self.lowH,
                         self.sampleOffset)

    def lowIndex(self, cx: int, cy: int) -> int:
        return cy * self.lowW + cx

    def lowCount(self) -> int:
        return self.lowW * self.lowH

    def mapDown(self, x: int, y: int) -> tuple[int, int]:
        return x // self.scale, y // self.scale

    def sampleCoord(self, cx: int, cy: int) -> tuple[int, int]:
        return (min(cx * self.scale + self.sampleOffset, self.highW - 1),
                min(cy * self.scale + self.sampleOffset, self.highH - 1))


@dataclass
class GluConfig:
    """glu::GluConfig (params.hpp:20-39)."""
    windowSide: int = 3
    errorThreshold: float = float(np.float32(30.0 / 255.0))
    maxIterations: int = 3
    epsilon: float = float(np.float32(1e-3))
    literalComponentUpdate: bool = False

    def c(self) -> N.GluConfigC:
        return N.GluConfigC(int(self.windowSide), float(self.errorThreshold),
                            int(self.maxIterations), float(self.epsilon),
                            int(bool(self.literalComponentUpdate)))

    def validate(self) -> None:
        N.check(N.lib().glu_config_validate(C.byref(self.c())))


@dataclass
class ParamField:
    """glu::ParamField (params.hpp:48-54); params is int32 (H, W, 3) on the device."""
    grid: GridSpec
    mode: Mode
    params: torch.Tensor

    def size(self) -> int:
        return self.grid.highW * self.grid.highH

    def numpy(self) -> np.ndarray:
        return self.params.cpu().numpy().view(PARAMS_DTYPE).reshape(self.grid.highH,
                                                                   self.grid.highW)

    def clone(self) -> "ParamField":
        return ParamField(self.grid, self.mode, self.params.clone())


@dataclass
class LargeErrorSet:
    """glu::LargeErrorSet (jointopt.hpp:12-17); components stay on the device."""
    width: int
    height: int
    mask: torch.Tensor            # uint8 (H, W)
    offsets: torch.Tensor         # int32 (ncomp + 1,)
    pixels: torch.Tensor          # int32 (sum of sizes,), each component ascending

    @property
    def components(self) -> list[np.ndarray]:
        off = self.offsets.cpu().numpy().astype(np.int64)
        px = self.pixels.cpu().numpy().view(np.uint32)
        return [px[off[c]:off[c + 1]].copy() for c in range(len(off) - 1)]

    def __len__(self) -> int:
        return int(self.offsets.numel()) - 1


@dataclass
class JointResult:
    """glu::JointResult (jointopt.hpp:30-37)."""
    low: torch.Tensor
    field: ParamField
    errors: torch.Tensor
    iterations: int = 0
    trialsAccepted: int = 0
    trialsRejected: int = 0
    components: int = 0


class Context:
    """A C-ABI context (stream + scratch) bound to one CUDA device.

    The context follows torch's current stream at each call so device work is
    ordered with the caller's torch work."""

    def __init__(self, device: int | None = None):
        if not torch.cuda.is_available():
            raise N.GluError("no CUDA device: the GLU hot path has no CPU fallback")
        self.device = torch.cuda.current_device() if device is None else int(device)
        h = C.c_void_p()
        N.check(N.lib().glu_ctx_create(self.device, C.byref(h)))
        self.handle = h

    def bind_stream(self) -> None:
        s = torch.cuda.current_stream(self.device).cuda_stream
        # torch's default stream is the legacy NULL stream; the C-ABI reads NULL
        # as "the context's own stream", so name the legacy stream explicitly
        # (cudaStreamLegacy == 0x1) to stay ordered with torch work and events.
        N.check(N.lib().glu_ctx_set_stream(self.handle, C.c_void_p(s if s else 1)))

    def set_solver(self, value: int) -> None:
        """GLU_OPT_SOLVER: 0 auto (fp32 filter + fp64 verify), 1 fp64 kernel only,
        2 fp32 filter with every pixel forced through the fp64 verify."""
        N.check(N.lib().glu_ctx_set_option(self.handle, 1, int(value)))

    def set_trials(self, value: int) -> None:
        """GLU_OPT_TRIALS: 0 speculative parallel schedule, 1 one CTA in order,
        2 dependency-counting dataflow schedule."""
        N.check(N.lib().glu_ctx_set_option(self.handle, 2, int(value)))

    @property
    def launches(self) -> int:
        return int(N.lib().glu_ctx_launch_count(self.handle))

    @property
    def fallbacks(self) -> int:
        return int(N.lib().glu_ctx_fallback_count(self.handle))

    @property
    def close_sets(self) -> int:
        """Pixels whose near-tie was settled in double over the close set."""
        return int(N.lib().glu_ctx_close_set_count(self.handle))

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                N.lib().glu_ctx_destroy(self.handle)
        except Exception:
            pass


_ctx: dict[int, Context] = {}


def context(device: int | None = None) -> Context:
    d = torch.cuda.current_device() if device is None else int(device)
    if d not in _ctx:
        _ctx[d] = Context(d)
    c = _ctx[d]
    c.bind_stream()
    return c


def _ptr(t: torch.Tensor | None) -> C.c_void_p:
    if t is None:
        return C.c_void_p(0)
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    return C.c_void_p(t.data_ptr())


def _image(t: torch.Tensor, what: str) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or t.dtype != torch.float32 or t.dim() != 3 \
            or t.shape[2] != 3:
        raise ValueError(f"{what}: expected a float32 (H, W, 3) tensor")
    return t.contiguous()


# ---- grid.hpp ------------------------------------------------------------------

def grid_downsample(high: torch.Tensor, scale: int) -> tuple[torch.Tensor, GridSpec]:
    """grid_downsample (grid.cpp:41-52); returns (low, grid)."""
    high = _image(high, "grid_downsample")
    g = GridSpec.create(high.shape[1], high.shape[0], scale)
    low = torch.empty((g.lowH, g.lowW, 3), dtype=torch.float32, device=high.device)
    ctx = context(high.device.index)
    N.check(N.lib().glu_cu_grid_downsample(ctx.handle, _ptr(high), C.byref(g.c()), _ptr(low)))
    return low, g


def neighborhood(x: int, y: int, grid: GridSpec, windowSide: int) -> list[int]:
    """neighborhood (grid.cpp:54-65): candidate cell indices, raster order."""
    if x < 0 or y < 0 or x >= grid.highW or y >= grid.highH:
        raise ValueError("neighborhood: pixel outside image")
    if windowSide < 3 or windowSide % 2 == 0:
        raise ValueError("windowSide must be odd and >= 3")
    cx, cy = grid.mapDown(x, y)
    h = windowSide // 2
    return [yy * grid.lowW + xx
            for yy in range(max(0, cy - h), min(grid.lowH - 1, cy + h) + 1)
            for xx in range(max(0, cx - h), min(grid.lowW - 1, cx + h) + 1)]


# ---- upsample.hpp --------------------------------------------------------------

def _check_field_inputs(high, low, grid: GridSpec, cfg: GluConfig) -> None:
    cfg.validate()
    if high.shape[1] != grid.highW or high.shape[0] != grid.highH:
        raise ValueError("optimize: guide image does not match grid")
    if low.shape[1] != grid.lowW or low.shape[0] != grid.lowH:
        raise ValueError("optimize: low-res image does not match grid")


def optimize_field(high: torch.Tensor, low: torch.Tensor, grid: GridSpec,
                   cfg: GluConfig | None = None, mode: Mode = Mode.Fast) -> ParamField:
    """optimize_field (upsample.cpp:194-216)."""
    cfg = cfg or GluConfig()
    high, low = _image(high, "optimize_field"), _image(low, "optimize_field")
    _check_field_inputs(high, low, grid, cfg)
    out = torch.empty((grid.highH, grid.highW, 3), dtype=torch.int32, device=high.device)
    ctx = context(high.device.index)
    N.check(N.lib().glu_cu_optimize_field(ctx.handle, _ptr(high), _ptr(low), C.byref(grid.c()),
                                          C.byref(cfg.c()), int(mode), _ptr(out)))
    return ParamField(grid, Mode(mode), out)


def optimize_pixels(high: torch.Tensor, low: torch.Tensor, grid: GridSpec, cfg: GluConfig | None,
                    mode: Mode, pixels: torch.Tensor, field: ParamField) -> None:
    """optimize_pixels (upsample.cpp:218-233): in place on field."""
    cfg = cfg or GluConfig()
    high, low = _image(high, "optimize_pixels"), _image(low, "optimize_pixels")
    _check_field_inputs(high, low, grid, cfg)
    if field.params.numel() != 3 * high.shape[0] * high.shape[1]:
        raise ValueError("optimize_pixels: field does not match image")
    pixels = pixels.to(device=high.device, dtype=torch.int32).contiguous()
    ctx = context(high.device.index)
    N.check(N.lib().glu_cu_optimize_pixels(ctx.handle, _ptr(high), _ptr(low), C.byref(grid.c()),
                                           C.byref(cfg.c()), int(mode), _ptr(pixels),
                                           pixels.numel(), _ptr(field.params)))


def apply_field(field: ParamField, lowTarget: torch.Tensor, clampOutput: bool = True
                ) -> torch.Tensor:
    """apply_field (upsample.cpp:235-252).  A (lowH, lowW) target is the
    single-channel extension and yields an (H, W) output."""
    g = field.grid
    ch = 1 if lowTarget.dim() == 2 else lowTarget.shape[2]
    if lowTarget.shape[1] != g.lowW or lowTarget.shape[0] != g.lowH or ch not in (1, 3):
        raise ValueError("apply_field: low-res image does not match grid")
    if field.params.numel() != 3 * g.highW * g.highH:
        raise ValueError("apply_field: field size does not match grid")
    lowTarget = lowTarget.contiguous()
    shape = (g.highH, g.highW, 3) if ch == 3 else (g.highH, g.highW)
    out = torch.empty(shape, dtype=torch.float32, device=lowTarget.device)
    ctx = context(lowTarget.device.index)
    N.check(N.lib().glu_cu_apply_field(ctx.handle, _ptr(field.params), C.byref(g.c()),
                                       _ptr(lowTarget), ch, int(bool(clampOutput)), _ptr(out)))
    return out


def apply_field_band(bandParams: torch.Tensor, grid: GridSpec, lowTarget: torch.Tensor,
                     clampOutput: bool = True, out: torch.Tensor | None = None) -> torch.Tensor:
    """apply_field over a row band (multi-GPU C5): `bandParams` is a
    (rows, W, 3) int32 slice of a field of `grid`, indexing the whole LR
    target; returns (rows, W[, 3])."""
    ch = 1 if lowTarget.dim() == 2 else lowTarget.shape[2]
    if lowTarget.shape[1] != grid.lowW or lowTarget.shape[0] != grid.lowH or ch not in (1, 3):
        raise ValueError("apply_field: low-res image does not match grid")
    if bandParams.dim() != 3 or bandParams.shape[1] != grid.highW or bandParams.shape[2] != 3:
        raise ValueError("apply_field: band does not match grid")
    bandParams, lowTarget = bandParams.contiguous(), lowTarget.contiguous()
    rows = bandParams.shape[0]
    shape = (rows, grid.highW, 3) if ch == 3 else (rows, grid.highW)
    if out is None:
        out = torch.empty(shape, dtype=torch.float32, device=lowTarget.device)
    ctx = context(lowTarget.device.index)
    N.check(N.lib().glu_cu_apply_field_band(ctx.handle, _ptr(bandParams), rows * grid.highW,
                                            C.byref(grid.c()), _ptr(lowTarget), ch,
                                            int(bool(clampOutput)), _ptr(out)))
    return out


def error_map(high: torch.Tensor, reconstructed: torch.Tensor) -> torch.Tensor:
    """error_map (upsample.cpp:254-267)."""
    if high.shape != reconstructed.shape:
        raise ValueError("error_map: image dimensions differ")
    high, rec = _image(high, "error_map"), _image(reconstructed, "error_map")
    e = torch.empty(high.shape[:2], dtype=torch.float32, device=high.device)
    ctx = context(high.device.index)
    N.check(N.lib().glu_cu_error_map(ctx.handle, _ptr(high), _ptr(rec),
                                     high.shape[0] * high.shape[1], _ptr(e)))
    return e


def self_error_map(high: torch.Tensor, field: ParamField, low: torch.Tensor) -> torch.Tensor:
    """error_map(high, apply_field(field, low)) in one pass (jointopt.cpp:188)."""
    high = _image(high, "self_error_map")
    e = torch.empty(high.shape[:2], dtype=torch.float32, device=high.device)
    ctx = context(high.device.index)
    N.check(N.lib().glu_cu_self_error_map(ctx.handle, _ptr(high), _ptr(field.params),
                                          C.byref(field.grid.c()), _ptr(low.contiguous()),
                                          _ptr(e)))
    return e


def solve_apply(high: torch.Tensor, low: torch.Tensor, grid: GridSpec, lowTarget: torch.Tensor,
                cfg: GluConfig | None = None, mode: Mode = Mode.Fast, clampOutput: bool = True,
                keep_params: bool = False):
    """Fused optimize_field + apply_field; returns (out, ParamField | None)."""
    cfg = cfg or GluConfig()
    high, low = _image(high, "solve_apply"), _image(low, "solve_apply")
    _check_field_inputs(high, low, grid, cfg)
    ch = 1 if lowTarget.dim() == 2 else lowTarget.shape[2]
    if lowTarget.shape[1] != grid.lowW or lowTarget.shape[0] != grid.lowH or ch not in (1, 3):
        raise ValueError("apply_field: low-res image does not match grid")
    shape = (grid.highH, grid.highW, 3) if ch == 3 else (grid.highH, grid.highW)
    out = torch.empty(shape, dtype=torch.float32, device=high.device)
    params = (torch.empty((grid.highH, grid.highW, 3), dtype=torch.int32, device=high.device)
              if keep_params else None)
    ctx = context(high.device.index)
    N.check(N.lib().glu_cu_solve_apply(ctx.handle, _ptr(high), _ptr(low), C.byref(grid.c()),
                                       C.byref(cfg.c()), int(mode), _ptr(lowTarget.contiguous()),
                                       ch, int(bool(clampOutput)), _ptr(out), _ptr(params)))
    return out, (ParamField(grid, Mode(mode), params) if keep_params else None)


# Scalar helpers (upsample.hpp:17-31), evaluated by the device batch kernels.

def _pair_eval(ip, ia, ib, w, eps):
    dev = torch.device("cuda", torch.cuda.current_device())
    t = lambda v: torch.as_tensor(np.asarray(v, np.float32).reshape(-1, 3), device=dev)
    P, A, B = t(ip), t(ia), t(ib)
    n = P.shape[0]
    W = torch.as_tensor(np.asarray(w if w is not None else np.zeros(n), np.float64).reshape(-1),
                        device=dev)
    we, wf, ob = (torch.empty(n, dtype=torch.float64, device=dev) for _ in range(3))
    ctx = context()
    N.check(N.lib().glu_cu_pair_eval(ctx.handle, _ptr(P), _ptr(A), _ptr(B), _ptr(W), n,
                                     float(eps), _ptr(we), _ptr(wf), _ptr(ob)))
    return we.cpu().numpy(), wf.cpu().numpy(), ob.cpu().numpy()


def weight_exact(ip, ia, ib, eps: float):
    """weight_exact (upsample.cpp:158-167); batched over leading dims."""
    r = _pair_eval(ip, ia, ib, None, eps)[0]
    return float(r[0]) if r.size == 1 else r


def weight_fast(ip, ia, ib, eps: float):
    """weight_fast (upsample.cpp:169-172)."""
    r = _pair_eval(ip, ia, ib, None, eps)[1]
    return float(r[0]) if r.size == 1 else r


def pair_objective(ip, ia, ib, w, eps: float):
    """pair_objective (upsample.cpp:174-176)."""
    r = _pair_eval(ip, ia, ib, w, eps)[2]
    return float(r[0]) if r.size == 1 else r


def optimize_pixel_batch(ips, cand_lists, eps: float, mode: Mode) -> np.ndarray:
    """optimize_pixel_{fast,exact,gnu} (upsample.cpp:178-192) over many
    instances; cand_lists[k] = (indices, colours (n, 3))."""
    counts = [len(c[0]) for c in cand_lists]
    if any(n == 0 for n in counts):
        raise ValueError("candidate list must not be empty")
    dev = torch.device("cuda", torch.cuda.current_device())
    off = np.zeros(len(counts) + 1, np.uint32)
    off[1:] = np.cumsum(counts)
    idx = np.concatenate([np.asarray(c[0], np.uint32) for c in cand_lists])
    rgb = np.concatenate([np.asarray(c[1], np.float32).reshape(-1, 3) for c in cand_lists])
    T = lambda a: torch.as_tensor(np.ascontiguousarray(a).view(np.int32)
                                  if a.dtype == np.uint32 else np.ascontiguousarray(a),
                                  device=dev)
    # keep every device buffer referenced until the (asynchronous) kernel has run
    ip, doff, didx, drgb = (T(np.asarray(ips, np.float32).reshape(-1, 3)), T(off), T(idx),
                            T(rgb))
    out = torch.empty((len(counts), 3), dtype=torch.int32, device=dev)
    ctx = context()
    N.check(N.lib().glu_cu_optimize_pixel_batch(ctx.handle, _ptr(ip), _ptr(doff), _ptr(didx),
                                                _ptr(drgb), len(counts), float(eps), int(mode),
                                                _ptr(out)))
    return out.cpu().numpy().view(PARAMS_DTYPE).reshape(-1)


def optimize_pixel_fast(ip, cands, eps: float):
    return optimize_pixel_batch([ip], [cands], eps, Mode.Fast)[0]


def optimize_pixel_exact(ip, cands, eps: float):
    return optimize_pixel_batch([ip], [cands], eps, Mode.Exact)[0]


def optimize_pixel_gnu(ip, cands):
    return optimize_pixel_batch([ip], [cands], 1e-3, Mode.Gnu)[0]


# ---- jointopt.hpp --------------------------------------------------------------

def find_large_error(errors: torch.Tensor, threshold: float) -> LargeErrorSet:
    """find_large_error (jointopt.cpp:9-46)."""
    if errors.dim() != 2 or errors.numel() == 0:
        raise ValueError("find_large_error: empty error map")
    errors = errors.contiguous()
    H, W = errors.shape
    mask = torch.empty((H, W), dtype=torch.uint8, device=errors.device)
    n = C.c_size_t()
    off, px = C.c_void_p(), C.c_void_p()
    ctx = context(errors.device.index)
    N.check(N.lib().glu_cu_find_large_error(ctx.handle, _ptr(errors), W, H, float(threshold),
                                            _ptr(mask), C.c_void_p(0), C.byref(n), C.byref(off),
                                            C.byref(px)))
    ncomp = n.value
    offsets = torch.zeros(ncomp + 1, dtype=torch.int32, device=errors.device)
    pixels = torch.empty(0, dtype=torch.int32, device=errors.device)
    if ncomp:
        # copy out of the context-owned buffers (valid until the next call)
        N.check(N.lib().glu_cu_copy(ctx.handle, _ptr(offsets), off, (ncomp + 1) * 4))
        total = int(offsets[-1].item())
        pixels = torch.empty(total, dtype=torch.int32, device=errors.device)
        N.check(N.lib().glu_cu_copy(ctx.handle, _ptr(pixels), px, total * 4))
    return LargeErrorSet(W, H, mask, offsets, pixels)


def trial_update_component(high: torch.Tensor, low: torch.Tensor, field: ParamField,
                           errors: torch.Tensor, component, cfg: GluConfig | None = None,
                           mode: Mode = Mode.Fast) -> bool:
    """trial_update_component (jointopt.cpp:114-180): in place on low, field, errors."""
    cfg = cfg or GluConfig()
    cfg.validate()
    comp = torch.as_tensor(np.asarray(component, np.uint32).view(np.int32)
                           if not isinstance(component, torch.Tensor) else component,
                           device=high.device).to(torch.int32).contiguous()
    if comp.numel() == 0:
        raise ValueError("trial_update_component: empty component")
    g = field.grid
    if (high.shape[1] != g.highW or high.shape[0] != g.highH or low.shape[1] != g.lowW
            or low.shape[0] != g.lowH or errors.shape[1] != g.highW or errors.shape[0] != g.highH):
        raise ValueError("trial_update_component: shape mismatch")
    acc = C.c_int()
    ctx = context(high.device.index)
    N.check(N.lib().glu_cu_trial_update_component(ctx.handle, _ptr(high), _ptr(low),
                                                  _ptr(field.params), _ptr(errors),
                                                  C.byref(g.c()), C.byref(cfg.c()), int(mode),
                                                  _ptr(comp), comp.numel(), C.byref(acc)))
    return bool(acc.value)


def joint_optimize(high: torch.Tensor, scale: int, cfg: GluConfig | None = None,
                   mode: Mode = Mode.Fast) -> JointResult:
    """joint_optimize (jointopt.cpp:182-206)."""
    cfg = cfg or GluConfig()
    cfg.validate()
    high = _image(high, "joint_optimize")
    g = GridSpec.create(high.shape[1], high.shape[0], scale)
    low = torch.empty((g.lowH, g.lowW, 3), dtype=torch.float32, device=high.device)
    params = torch.empty((g.highH, g.highW, 3), dtype=torch.int32, device=high.device)
    errors = torch.empty((g.highH, g.highW), dtype=torch.float32, device=high.device)
    st = N.GluJointStats()
    ctx = context(high.device.index)
    N.check(N.lib().glu_cu_joint_optimize(ctx.handle, _ptr(high), C.byref(g.c()),
                                          C.byref(cfg.c()), int(mode), _ptr(low), _ptr(params),
                                          _ptr(errors), C.byref(st)))
    return JointResult(low, ParamField(g, Mode(mode), params), errors, st.iterations,
                       st.trialsAccepted, st.trialsRejected, st.components)


# ---- LR operator stand-ins ---------------------------------

def op_color(low: torch.Tensor, M=None, bias=None, gamma: float = 0.0) -> torch.Tensor:
    """clamp01(M @ (gamma ? clamp01(x**gamma) : x) + bias) per LR pixel."""
    low = _image(low, "op_color")
    out = torch.empty_like(low)
    Mh = (C.c_double * 9)(*np.asarray(M, np.float64).reshape(9)) if M is not None else None
    Bh = (C.c_double * 3)(*np.asarray(bias, np.float64).reshape(3)) if bias is not None else None
    ctx = context(low.device.index)
    N.check(N.lib().glu_cu_op_color(ctx.handle, _ptr(low), low.shape[0] * low.shape[1],
                                    C.cast(Mh, C.c_void_p) if Mh else None,
                                    C.cast(Bh, C.c_void_p) if Bh else None, float(gamma),
                                    _ptr(out)))
    return out


def op_matte(low: torch.Tensor) -> torch.Tensor:
    """1-channel matte 1 / (1 + exp(-10 (luma - 0.5))) (BASELINE.json configs[2])."""
    low = _image(low, "op_matte")
    out = torch.empty(low.shape[:2], dtype=torch.float32, device=low.device)
    ctx = context(low.device.index)
    N.check(N.lib().glu_cu_op_matte(ctx.handle, _ptr(low), low.shape[0] * low.shape[1],
                                    _ptr(out)))
    return out


# ---- SimOperator (simop.hpp:11-37): the reference's black-box operator stand-ins ----

class SimOperator:
    """glu::SimOperator (simop.hpp:11-26): a pointwise colour operator, applied
    on the device (glu_cu_apply_operator) with the reference's double
    expressions and clamp01 (simop.cpp:16-41)."""

    class Kind(enum.IntEnum):
        Identity = 0
        ScalarGain = 1
        ChannelMix = 2
        Grayscale = 3
        Gamma = 4
        Invert = 5

    def __init__(self, kind: "SimOperator.Kind" = Kind.Identity, gain: float = 1.0,
                 gamma: float = 1.0, mix=(1, 0, 0, 0, 1, 0, 0, 0, 1), name: str = "identity"):
        self.kind, self.gain, self.gamma = SimOperator.Kind(kind), float(gain), float(gamma)
        self.mix = tuple(float(v) for v in np.asarray(mix, np.float64).reshape(9))
        self.name = name

    def linear(self) -> bool:
        K = SimOperator.Kind
        return self.kind in (K.Identity, K.ScalarGain, K.ChannelMix, K.Grayscale)

    def c(self) -> N.GluSimOperator:
        return N.GluSimOperator(int(self.kind), self.gain, self.gamma, (C.c_double * 9)(*self.mix))


def identity_op() -> SimOperator:
    return SimOperator()


def scalar_gain_op(gain: float) -> SimOperator:
    if not gain >= 0:
        raise ValueError("scalar_gain_op: gain must be >= 0")
    return SimOperator(SimOperator.Kind.ScalarGain, gain=gain, name=f"gain({gain:g})")


def channel_mix_op(m) -> SimOperator:
    return SimOperator(SimOperator.Kind.ChannelMix, mix=m, name="mix")


def grayscale_op() -> SimOperator:
    return SimOperator(SimOperator.Kind.Grayscale, name="gray")


def gamma_op(gamma: float) -> SimOperator:
    if not gamma > 0:
        raise ValueError("gamma_op: gamma must be > 0")
    return SimOperator(SimOperator.Kind.Gamma, gamma=gamma, name=f"gamma({gamma:g})")


def invert_op() -> SimOperator:
    return SimOperator(SimOperator.Kind.Invert, name="invert")


def parse_operator(text: str) -> SimOperator:
    """identity | gain:<c> | gamma:<g> | gray | invert | mix:m00,...,m22 (simop.cpp:89-118)."""
    if text == "identity":
        return identity_op()
    if text == "gray":
        return grayscale_op()
    if text == "invert":
        return invert_op()
    head, sep, rest = text.partition(":")
    if sep:
        if head == "gain":
            return scalar_gain_op(float(rest))
        if head == "gamma":
            return gamma_op(float(rest))
        if head == "mix":
            vals = rest.split(",")
            if len(vals) < 9:
                raise ValueError("mix needs 9 comma-separated values")
            if len(vals) > 9:
                raise ValueError("mix needs exactly 9 values")
            return channel_mix_op([float(v) for v in vals])
    raise ValueError("unknown operator: " + text)


def apply_operator(op: SimOperator, img: torch.Tensor) -> torch.Tensor:
    """apply_operator (simop.cpp:120-132) on a device RGB image."""
    img = _image(img, "apply_operator")
    out = torch.empty_like(img)
    ctx = context(img.device.index)
    N.check(N.lib().glu_cu_apply_operator(ctx.handle, C.byref(op.c()), _ptr(img),
                                          img.shape[0] * img.shape[1], _ptr(out)))
    return out


def apply_operator_field(field: ParamField, op: SimOperator, lowIn: torch.Tensor,
                         clampOutput: bool = True, out: torch.Tensor | None = None
                         ) -> torch.Tensor:
    """apply_field(field, apply_operator(op, lowIn)) in one pass over the HR
    field: the edit loop's "operator on T-down, then upsample"
    (glu_cu_apply_operator_field)."""
    g = field.grid
    lowIn = _image(lowIn, "apply_operator_field")
    if lowIn.shape[1] != g.lowW or lowIn.shape[0] != g.lowH:
        raise ValueError("apply_field: low-res image does not match grid")
    if out is None:
        out = torch.empty((g.highH, g.highW, 3), dtype=torch.float32, device=lowIn.device)
    ctx = context(lowIn.device.index)
    N.check(N.lib().glu_cu_apply_operator_field(ctx.handle, _ptr(field.params), C.byref(g.c()),
                                                C.byref(op.c()), _ptr(lowIn),
                                                int(bool(clampOutput)), _ptr(out)))
    return out


def apply_operator_field_band(bandParams: torch.Tensor, grid: GridSpec, op: SimOperator,
                              lowIn: torch.Tensor, clampOutput: bool = True,
                              out: torch.Tensor | None = None) -> torch.Tensor:
    """apply_operator_field over a (rows, W, 3) int32 row band of a field of
    `grid` (multi-GPU C5); returns (rows, W, 3)."""
    lowIn = _image(lowIn, "apply_operator_field")
    if lowIn.shape[1] != grid.lowW or lowIn.shape[0] != grid.lowH:
        raise ValueError("apply_field: low-res image does not match grid")
    if bandParams.dim() != 3 or bandParams.shape[1] != grid.highW or bandParams.shape[2] != 3:
        raise ValueError("apply_field: band does not match grid")
    bandParams = bandParams.contiguous()
    rows = bandParams.shape[0]
    if out is None:
        out = torch.empty((rows, grid.highW, 3), dtype=torch.float32, device=lowIn.device)
    ctx = context(lowIn.device.index)
    N.check(N.lib().glu_cu_apply_operator_field_band(
        ctx.handle, _ptr(bandParams), rows * grid.highW, C.byref(grid.c()), C.byref(op.c()),
        _ptr(lowIn), int(bool(clampOutput)), _ptr(out)))
    return out


# ---- frame pipeline (BASELINE.json configs[2]) -----------------------------------

TARGET_OPS = {"identity": 0, "matte": 1}


def upsample_frames(frames: torch.Tensor, scale: int, target: str = "matte",
                    cfg: GluConfig | None = None, mode: Mode = Mode.Fast,
                    out: torch.Tensor | None = None) -> torch.Tensor:
    """Per frame: grid_downsample -> target op -> fused solve + apply (device-resident)."""
    cfg = cfg or GluConfig()
    if frames.dim() != 4 or frames.shape[3] != 3 or frames.dtype != torch.float32:
        raise ValueError("upsample_frames: expected float32 (F, H, W, 3)")
    F_, H, W, _ = frames.shape
    g = GridSpec.create(W, H, scale)
    ch = 1 if target == "matte" else 3
    shape = (F_, H, W) if ch == 1 else (F_, H, W, 3)
    if out is None:
        out = torch.empty(shape, dtype=torch.float32, device=frames.device)
    ctx = context(frames.device.index)
    N.check(N.lib().glu_cu_upsample_frames(ctx.handle, _ptr(frames), F_, C.byref(g.c()),
                                           C.byref(cfg.c()), int(mode), TARGET_OPS[target],
                                           _ptr(out), C.c_void_p(0)))
    return out


def upsample_frames_host(frames: torch.Tensor, scale: int, out: torch.Tensor,
                         target: str = "matte", cfg: GluConfig | None = None,
                         mode: Mode = Mode.Fast, device: int | None = None) -> None:
    """Same, from host (ideally pinned) memory through glu_h_upsample_frames:
    copies in and out overlap the kernels; returns after the last copy-out."""
    cfg = cfg or GluConfig()
    if frames.is_cuda or out.is_cuda:
        raise ValueError("upsample_frames_host: expected host tensors")
    F_, H, W, _ = frames.shape
    g = GridSpec.create(W, H, scale)
    ctx = context(device)
    N.check(N.lib().glu_h_upsample_frames(ctx.handle, C.c_void_p(frames.data_ptr()), F_,
                                          C.byref(g.c()), C.byref(cfg.c()), int(mode),
                                          TARGET_OPS[target], C.c_void_p(out.data_ptr()),
                                          C.c_void_p(0)))


def fp32_peak(device: int | None = None) -> tuple[float, float]:
    """(TFLOP/s, implied SM MHz) of an FFMA probe on this device."""
    ctx = context(device)
    t, m = C.c_double(), C.c_double()
    N.check(N.lib().glu_cu_fp32_peak(ctx.handle, C.byref(t), C.byref(m)))
    return t.value, m.value


# ---- GLUP parameter files (io_glup.cpp:48-139) ----------------------------------

FormatError = N.FormatError


def encode_glup(field: ParamField, low: torch.Tensor, optimized: bool = False,
                out: torch.Tensor | None = None) -> torch.Tensor:
    """encode_glup: device field + LR image -> GLUP bytes (uint8 tensor, pinned
    host memory by default, or a device tensor passed as `out`)."""
    g = field.grid
    if low.shape[1] != g.lowW or low.shape[0] != g.lowH:
        raise ValueError("encode_glup: low-res image does not match grid")
    if field.params.numel() != 3 * g.highW * g.highH:
        raise ValueError("encode_glup: param count does not match grid")
    n = int(N.lib().glu_glup_size(C.byref(g.c())))
    if out is None:
        out = torch.empty(n, dtype=torch.uint8).pin_memory()
    ctx = context(field.params.device.index)
    N.check(N.lib().glu_cu_glup_encode(ctx.handle, _ptr(field.params), _ptr(low.contiguous()),
                                       C.byref(g.c()), int(field.mode), int(bool(optimized)),
                                       C.c_void_p(out.data_ptr()), out.numel()))
    return out


def decode_glup(data, device: int | None = None):
    """decode_glup: GLUP bytes (bytes / numpy / uint8 tensor, host or device) ->
    (ParamField, low, optimized) on the device; raises FormatError(field, msg)."""
    if isinstance(data, (bytes, bytearray)):
        data = torch.frombuffer(bytearray(data), dtype=torch.uint8) if len(data) else \
            torch.empty(0, dtype=torch.uint8)
    elif isinstance(data, np.ndarray):
        data = torch.from_numpy(np.ascontiguousarray(data, np.uint8))
    data = data.contiguous()
    ctx = context(device)
    g, mode, opt = N.GluGrid(), C.c_int(), C.c_int()
    ptr = C.c_void_p(data.data_ptr() if data.numel() else 0)
    N.check(N.lib().glu_cu_glup_decode(ctx.handle, ptr, data.numel(), C.byref(g), C.byref(mode),
                                       C.byref(opt), None, None))
    dev = torch.device("cuda", ctx.device)
    low = torch.empty((g.lowH, g.lowW, 3), dtype=torch.float32, device=dev)
    params = torch.empty((g.highH, g.highW, 3), dtype=torch.int32, device=dev)
    N.check(N.lib().glu_cu_glup_decode(ctx.handle, ptr, data.numel(), C.byref(g), C.byref(mode),
                                       C.byref(opt), _ptr(low), _ptr(params)))
    grid = GridSpec(g.scale, g.highW, g.highH, g.lowW, g.lowH, g.sampleOffset)
    return ParamField(grid, Mode(mode.value), params), low, bool(opt.value)


# ---- quality metrics (metrics.cpp:62-117) ----------------------------------------

def mse(a: torch.Tensor, b: torch.Tensor) -> float:
    """mse (metrics.cpp:62-70)."""
    if a.shape != b.shape:
        raise ValueError("mse: image dimensions differ")
    a, b = a.contiguous(), b.contiguous()
    out = C.c_double()
    ctx = context(a.device.index)
    N.check(N.lib().glu_cu_mse(ctx.handle, _ptr(a), _ptr(b), a.numel(), C.byref(out)))
    return out.value


def psnr(a: torch.Tensor, b: torch.Tensor) -> float:
    """psnr (metrics.cpp:72-76): 99 dB for identical images."""
    import math
    m = mse(a, b)
    return 99.0 if m == 0 else 10.0 * math.log10(1.0 / m)


def ssim(a: torch.Tensor, b: torch.Tensor) -> float:
    """ssim (metrics.cpp:78-107) on the BT.601 luma channel."""
    if a.shape != b.shape:
        raise ValueError("ssim: image dimensions differ")
    a, b = _image(a, "ssim"), _image(b, "ssim")
    out = C.c_double()
    ctx = context(a.device.index)
    N.check(N.lib().glu_cu_ssim(ctx.handle, _ptr(a), _ptr(b), a.shape[1], a.shape[0],
                                C.byref(out)))
    return out.value


@dataclass
class JbuParams:
    """glu::JbuParams (baseline.hpp:8-14)."""
    window: int = 5
    sigmaD: float = 0.5
    sigmaR: float = 0.1


def _baseline_out(g: GridSpec, ref: torch.Tensor) -> torch.Tensor:
    return torch.empty((g.highH, g.highW, 3), dtype=torch.float32, device=ref.device)


def nearest_upsample(targetLow: torch.Tensor, grid: GridSpec) -> torch.Tensor:
    """nearest_upsample (baseline.cpp:87-98)."""
    if targetLow.shape[1] != grid.lowW or targetLow.shape[0] != grid.lowH:
        raise ValueError("nearest_upsample: low-res image does not match grid")
    t = _image(targetLow, "nearest_upsample")
    out = _baseline_out(grid, t)
    ctx = context(t.device.index)
    N.check(N.lib().glu_cu_nearest_upsample(ctx.handle, _ptr(t), C.byref(grid.c()), _ptr(out)))
    return out


def bilinear_upsample(targetLow: torch.Tensor, grid: GridSpec) -> torch.Tensor:
    """bilinear_upsample (baseline.cpp:100-129)."""
    if targetLow.shape[1] != grid.lowW or targetLow.shape[0] != grid.lowH:
        raise ValueError("bilinear_upsample: low-res image does not match grid")
    t = _image(targetLow, "bilinear_upsample")
    out = _baseline_out(grid, t)
    ctx = context(t.device.index)
    N.check(N.lib().glu_cu_bilinear_upsample(ctx.handle, _ptr(t), C.byref(grid.c()), _ptr(out)))
    return out


def jbu_upsample(guideHigh: torch.Tensor, guideLow: torch.Tensor, targetLow: torch.Tensor,
                 grid: GridSpec, params: JbuParams | None = None) -> torch.Tensor:
    """jbu_upsample (baseline.cpp:30-85)."""
    p = params or JbuParams()
    gh, gl, t = (_image(x, "jbu_upsample") for x in (guideHigh, guideLow, targetLow))
    if gh.shape[1] != grid.highW or gh.shape[0] != grid.highH:
        raise ValueError("jbu_upsample: guide image does not match grid")
    for x in (gl, t):
        if x.shape[1] != grid.lowW or x.shape[0] != grid.lowH:
            raise ValueError("jbu_upsample: low-res image does not match grid")
    out = _baseline_out(grid, t)
    ctx = context(t.device.index)
    N.check(N.lib().glu_cu_jbu_upsample(ctx.handle, _ptr(gh), _ptr(gl), _ptr(t),
                                        C.byref(grid.c()), int(p.window), float(p.sigmaD),
                                        float(p.sigmaR), _ptr(out)))
    return out


def quality_report(reference: torch.Tensor, test: torch.Tensor) -> dict:
    """quality_report (metrics.cpp:109-115)."""
    m = mse(reference, test)
    import math
    return {"mse": m, "psnrDb": 99.0 if m == 0 else 10.0 * math.log10(1.0 / m),
            "ssim": ssim(reference, test)}
