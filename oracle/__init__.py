"""CPU ORACLE bindings -- TEST INFRASTRUCTURE ONLY.

Two checkers, both reached through ctypes over numpy buffers:

* ``Oracle``  -- oracle/_build/libglu_oracle.so, the plain-C restatement of the
  reference hot path (glu_oracle.c; every function cites the reference
  file:line it follows).
* ``Reference`` -- oracle/_ref/libglu_ref.so, the UNMODIFIED reference library
  compiled from /root/reference/proj/src by oracle/Makefile plus ref_shim.cpp.
  It exists wherever it was built in this container (the built .so travels to
  the GPU box); it is used to pin the restatement and as bench.py's
  ``cpu_baseline`` (``"kind": "reference"``).

Only tests/, __graft_entry__.smoke() and bench.py's cpu-baseline / reference
arm may import this package.  The product (paper_2307_09582_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libglu_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libglu_ref.so")

PARAMS_DTYPE = np.dtype([("a", "<u4"), ("b", "<u4"), ("w", "<f4")])
MODES = {"fast": 0, "exact": 1, "gnu": 2}
EPS_DEFAULT = float(np.float32(1e-3))  # GluConfig::epsilon is a float (params.hpp:24)
TAU_DEFAULT = float(np.float32(30.0 / 255.0))

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_parp = np.ctypeslib.ndpointer(PARAMS_DTYPE, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")


def build(force: bool = False) -> None:
    """Compile the checkers with oracle/Makefile (gcc/g++ only)."""
    if force or not os.path.exists(ORACLE_SO) or os.path.isdir("/root/reference/proj/src"):
        # incremental; the reference-derived targets exist only where the
        # reference sources do (oracle/Makefile)
        subprocess.run(["make", "-s", "-C", HERE], check=True)


def _mode(m) -> int:
    return MODES[m] if isinstance(m, str) else int(m)


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def low_dims(W: int, H: int, s: int) -> tuple[int, int]:
    return (W + s - 1) // s, (H + s - 1) // s


class _Common:
    """Bindings shared by the restatement (prefix glu_o_) and the reference shim (glu_r_)."""

    prefix = ""

    def __init__(self, path: str):
        if not os.path.exists(path):
            build()
        self.lib = C.CDLL(path)
        p = self.prefix
        L = self.lib
        self._ds = getattr(L, p + "grid_downsample")
        self._ds.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, _f32p]
        self._of = getattr(L, p + "optimize_field")
        self._of.argtypes = [_f32p, C.c_int, C.c_int, _f32p, C.c_int, C.c_int, C.c_double,
                             C.c_int, _parp]
        self._fle = getattr(L, p + "find_large_error")
        self._fle.restype = C.c_long
        self._fle.argtypes = [_f32p, C.c_int, C.c_int, C.c_float, _u8p, _u32p, _u32p]
        self._trial = getattr(L, p + "trial_update_component")
        self._trial.argtypes = [_f32p, C.c_int, C.c_int, _f32p, C.c_int, C.c_int, C.c_double,
                                C.c_int, C.c_int, _parp, _f32p, _u32p, C.c_size_t]
        self._joint = getattr(L, p + "joint_optimize")
        self._joint.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_float, C.c_int,
                                C.c_double, C.c_int, C.c_int, _f32p, _parp, _f32p, _i32p]

    def grid_downsample(self, high: np.ndarray, s: int) -> np.ndarray:
        high = _f32(high)
        H, W = high.shape[:2]
        lw, lh = low_dims(W, H, s)
        low = np.zeros((lh, lw, 3), np.float32)
        if self._ds(high, W, H, s, low):
            raise ValueError("grid_downsample: invalid arguments")
        return low

    def optimize_field(self, high, low, s, S=3, eps=EPS_DEFAULT, mode="fast") -> np.ndarray:
        high, low = _f32(high), _f32(low)
        H, W = high.shape[:2]
        out = np.zeros((H, W), PARAMS_DTYPE)
        if self._of(high, W, H, low, s, S, eps, _mode(mode), out):
            raise ValueError("optimize_field: invalid arguments")
        return out

    def find_large_error(self, e, threshold=TAU_DEFAULT):
        e = _f32(e)
        H, W = e.shape
        mask = np.zeros((H, W), np.uint8)
        off = np.zeros(W * H + 1, np.uint32)
        px = np.zeros(W * H, np.uint32)
        n = self._fle(e, W, H, threshold, mask, off, px)
        if n < 0:
            raise ValueError("find_large_error: empty error map")
        return mask, [px[off[c]:off[c + 1]].copy() for c in range(n)]

    def trial_update_component(self, high, low, field, errors, comp, s, S=3, eps=EPS_DEFAULT,
                               mode="fast", literal=False) -> bool:
        """In place on low/field/errors (numpy arrays, C-contiguous)."""
        high = _f32(high)
        H, W = high.shape[:2]
        comp = np.ascontiguousarray(comp, np.uint32)
        r = self._trial(high, W, H, low, s, S, eps, _mode(mode), int(literal), field, errors,
                        comp, comp.size)
        if r < 0:
            raise ValueError("trial_update_component: invalid arguments")
        return bool(r)

    def joint_optimize(self, high, s, S=3, threshold=TAU_DEFAULT, max_iterations=3,
                       eps=EPS_DEFAULT, mode="fast", literal=False):
        high = _f32(high)
        H, W = high.shape[:2]
        lw, lh = low_dims(W, H, s)
        low = np.zeros((lh, lw, 3), np.float32)
        field = np.zeros((H, W), PARAMS_DTYPE)
        errors = np.zeros((H, W), np.float32)
        cnt = np.zeros(3, np.int32)
        if self._joint(high, W, H, s, S, threshold, max_iterations, eps, _mode(mode),
                       int(literal), low, field, errors, cnt):
            raise ValueError("joint_optimize: invalid arguments")
        return dict(low=low, field=field, errors=errors, iterations=int(cnt[0]),
                    accepted=int(cnt[1]), rejected=int(cnt[2]))


class Oracle(_Common):
    prefix = "glu_o_"

    def __init__(self):
        super().__init__(ORACLE_SO)
        L = self.lib
        for name in ("weight_exact", "weight_fast"):
            fn = getattr(L, "glu_o_" + name)
            fn.restype = C.c_double
            fn.argtypes = [_f32p, _f32p, _f32p, C.c_double]
        L.glu_o_pair_objective.restype = C.c_double
        L.glu_o_pair_objective.argtypes = [_f32p, _f32p, _f32p, C.c_double, C.c_double]
        L.glu_o_optimize_pixel.argtypes = [_f32p, _u32p, _f32p, C.c_size_t, C.c_double, C.c_int,
                                           C.POINTER(C.c_uint32 * 3)]
        L.glu_o_optimize_pixels.argtypes = [_f32p, C.c_int, C.c_int, _f32p, C.c_int, C.c_int,
                                            C.c_double, C.c_int, _u32p, C.c_size_t, _parp]
        L.glu_o_apply_field.argtypes = [_parp, C.c_int, C.c_int, _f32p, C.c_int, C.c_int, C.c_int,
                                        C.c_int, _f32p]
        L.glu_o_error_map.argtypes = [_f32p, _f32p, C.c_size_t, _f32p]

    def weight_exact(self, ip, ia, ib, eps=1e-3) -> float:
        return self.lib.glu_o_weight_exact(_f32(ip), _f32(ia), _f32(ib), eps)

    def weight_fast(self, ip, ia, ib, eps=1e-3) -> float:
        return self.lib.glu_o_weight_fast(_f32(ip), _f32(ia), _f32(ib), eps)

    def pair_objective(self, ip, ia, ib, w, eps=1e-3) -> float:
        return self.lib.glu_o_pair_objective(_f32(ip), _f32(ia), _f32(ib), w, eps)

    def optimize_pixel(self, ip, idx, rgb, eps=1e-3, mode="fast"):
        idx = np.ascontiguousarray(idx, np.uint32)
        rgb = _f32(rgb).reshape(-1)
        out = (C.c_uint32 * 3)()
        if self.lib.glu_o_optimize_pixel(_f32(ip), idx, rgb, idx.size, eps, _mode(mode),
                                         C.byref(out)):
            raise ValueError("candidate list must not be empty")
        w = np.array([out[2]], np.uint32).view(np.float32)[0]
        return int(out[0]), int(out[1]), float(w)

    def optimize_pixels(self, high, low, s, pixels, field, S=3, eps=EPS_DEFAULT, mode="fast"):
        high, low = _f32(high), _f32(low)
        H, W = high.shape[:2]
        pixels = np.ascontiguousarray(pixels, np.uint32)
        if self.lib.glu_o_optimize_pixels(high, W, H, low, s, S, eps, _mode(mode), pixels,
                                          pixels.size, field):
            raise ValueError("optimize_pixels: invalid arguments")

    def apply_field(self, field, low_target, clamp=True) -> np.ndarray:
        field = np.ascontiguousarray(field)
        H, W = field.shape
        lt = _f32(low_target)
        ch = 1 if lt.ndim == 2 else lt.shape[2]
        out = np.zeros((H, W, ch) if ch == 3 else (H, W), np.float32)
        if self.lib.glu_o_apply_field(field, W, H, lt, lt.shape[1], lt.shape[0], ch, int(clamp),
                                      out):
            raise ValueError("apply_field: invalid arguments")
        return out

    def error_map(self, high, recon) -> np.ndarray:
        high, recon = _f32(high), _f32(recon)
        if high.shape != recon.shape:
            raise ValueError("error_map: image dimensions differ")
        e = np.zeros(high.shape[:2], np.float32)
        self.lib.glu_o_error_map(high, recon, e.size, e)
        return e


class Reference(_Common):
    prefix = "glu_r_"

    def __init__(self):
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(f"{REF_SO} not built (needs /root/reference at build time)")
        super().__init__(REF_SO)
        L = self.lib
        L.glu_r_synth.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_ulonglong, _f32p]
        L.glu_r_set_num_threads.argtypes = [C.c_int]
        L.glu_r_optimize_field_allcores.argtypes = [_f32p, C.c_int, C.c_int, _f32p, C.c_int,
                                                    C.c_int, C.c_double, C.c_int, C.c_int, _parp]
        L.glu_r_apply_field.argtypes = [_parp, C.c_int, C.c_int, C.c_int, _f32p, C.c_int, _f32p]
        L.glu_r_error_map.argtypes = [_f32p, _f32p, C.c_int, C.c_int, _f32p]
        L.glu_r_optimize_pixel.argtypes = [_f32p, _u32p, _f32p, C.c_size_t, C.c_double, C.c_int,
                                           C.POINTER(C.c_uint32 * 3)]

    def optimize_pixel(self, ip, idx, rgb, eps=1e-3, mode="fast"):
        idx = np.ascontiguousarray(idx, np.uint32)
        out = (C.c_uint32 * 3)()
        if self.lib.glu_r_optimize_pixel(_f32(ip), idx, _f32(rgb).reshape(-1), idx.size, eps,
                                         _mode(mode), C.byref(out)):
            raise ValueError("candidate list must not be empty")
        w = np.array([out[2]], np.uint32).view(np.float32)[0]
        return int(out[0]), int(out[1]), float(w)

    def apply_operator(self, kind: int, img, gain=1.0, gamma=1.0, mix=None) -> np.ndarray:
        """apply_operator (simop.cpp:120-132) with the reference's operator
        constructors (kind: 0 identity, 1 gain, 2 mix, 3 gray, 4 gamma, 5 invert)."""
        L = self.lib
        f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
        L.glu_r_apply_operator.argtypes = [C.c_int, C.c_double, C.c_double, f64p, _f32p, C.c_int,
                                           C.c_int, _f32p]
        img = _f32(img)
        m = np.ascontiguousarray(np.eye(3) if mix is None else mix, np.float64).reshape(9)
        out = np.zeros_like(img)
        if L.glu_r_apply_operator(int(kind), float(gain), float(gamma), m, img, img.shape[1],
                                  img.shape[0], out):
            raise ValueError("apply_operator: invalid operator")
        return out

    def set_num_threads(self, n: int) -> None:
        self.lib.glu_r_set_num_threads(n)

    def baseline(self, kind: str, target, s, guide_high=None, guide_low=None, window=5,
                 sigma_d=0.5, sigma_r=0.1):
        """nearest / bilinear / jbu upsampling of the reference (baseline.cpp:30-129)."""
        L = self.lib
        L.glu_r_baseline.argtypes = [C.c_int, C.c_void_p, C.c_void_p, _f32p, C.c_int, C.c_int,
                                     C.c_int, C.c_int, C.c_double, C.c_double, _f32p]
        t = _f32(target)
        lh, lw = t.shape[:2]
        if guide_high is not None:
            gh = _f32(guide_high)
            H, W = gh.shape[:2]
        else:
            H, W = lh * s, lw * s
            gh = None
        out = np.zeros((H, W, 3), np.float32)
        k = {"nearest": 0, "bilinear": 1, "jbu": 2}[kind]
        gl = _f32(guide_low) if guide_low is not None else None
        if L.glu_r_baseline(k, gh.ctypes.data if gh is not None else None,
                            gl.ctypes.data if gl is not None else None, t, W, H, s, window,
                            sigma_d, sigma_r, out):
            raise ValueError(kind + ": invalid arguments")
        return out

    def quality(self, a, b):
        """(mse, psnr, ssim) of the reference (metrics.cpp:62-115)."""
        L = self.lib
        L.glu_r_quality.argtypes = [_f32p, _f32p, C.c_int, C.c_int,
                                    np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")]
        a = _f32(a)
        out = np.zeros(3, np.float64)
        if L.glu_r_quality(a, _f32(b), a.shape[1], a.shape[0], out):
            raise ValueError("quality: invalid images")
        return tuple(out.tolist())

    def encode_glup(self, field, low, s, mode=0, optimized=False) -> bytes:
        """encode_glup (io_glup.cpp:48-77) of the reference."""
        L = self.lib
        L.glu_r_encode_glup.restype = C.c_long
        L.glu_r_encode_glup.argtypes = [_parp, _f32p, C.c_int, C.c_int, C.c_int, C.c_int,
                                        C.c_int, C.c_void_p, C.c_size_t]
        field = np.ascontiguousarray(field)
        H, W = field.shape
        n = L.glu_r_encode_glup(field, _f32(low), W, H, s, int(mode), int(optimized), None, 0)
        if n < 0:
            raise ValueError("encode_glup: invalid input")
        out = (C.c_uint8 * n)()
        L.glu_r_encode_glup(field, _f32(low), W, H, s, int(mode), int(optimized), out, n)
        return bytes(out)

    def decode_glup(self, data: bytes):
        """decode_glup (io_glup.cpp:79-139): (ok, field-or-error-field, dims)."""
        L = self.lib
        L.glu_r_decode_glup.restype = C.c_int
        L.glu_r_decode_glup.argtypes = [C.c_void_p, C.c_size_t, _i32p, C.c_void_p, C.c_void_p,
                                        C.c_char_p, C.c_size_t]
        dims = np.zeros(5, np.int32)
        buf = (C.c_uint8 * max(1, len(data))).from_buffer_copy(data or b"\0")
        fld = C.create_string_buffer(32)
        rc = L.glu_r_decode_glup(buf, len(data), dims, None, None, fld, 32)
        if rc == 1:
            return False, fld.value.decode(), None
        if rc != 0:
            raise RuntimeError("decode_glup failed")
        return True, None, dims.tolist()

    def synth(self, kind: str, w: int, h: int, seed: int) -> np.ndarray:
        out = np.zeros((h, w, 3), np.float32)
        if self.lib.glu_r_synth(kind.encode(), w, h, seed, out):
            raise ValueError(kind)
        return out

    def optimize_field_allcores(self, high, low, s, S=3, eps=EPS_DEFAULT, mode="fast",
                                threads=0) -> np.ndarray:
        high, low = _f32(high), _f32(low)
        H, W = high.shape[:2]
        out = np.zeros((H, W), PARAMS_DTYPE)
        if self.lib.glu_r_optimize_field_allcores(high, W, H, low, s, S, eps, _mode(mode),
                                                  threads, out):
            raise ValueError("optimize_field: invalid arguments")
        return out

    def apply_field(self, field, s, low_target, clamp=True) -> np.ndarray:
        field = np.ascontiguousarray(field)
        H, W = field.shape
        out = np.zeros((H, W, 3), np.float32)
        if self.lib.glu_r_apply_field(field, W, H, s, _f32(low_target), int(clamp), out):
            raise ValueError("apply_field: invalid arguments")
        return out

    def error_map(self, high, recon) -> np.ndarray:
        high = _f32(high)
        H, W = high.shape[:2]
        e = np.zeros((H, W), np.float32)
        if self.lib.glu_r_error_map(high, _f32(recon), W, H, e):
            raise ValueError("error_map: image dimensions differ")
        return e
