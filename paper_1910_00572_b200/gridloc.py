"""Python mirror of the reference ``gridloc`` hot-path API over the C-ABI.

Same names, argument meaning and error behaviour as
/root/reference/proj/include/gridloc/{belief_tensor,observation,localizer,
occupancy_map}.hpp, with the belief tensor resident on the GPU. The
reference's ``ThreadPool&`` / ``StepScratch&`` parameters become an optional
:class:`Context` (one CUDA device + stream).
"""
from __future__ import annotations

import ctypes as C
import os
import math
from dataclasses import dataclass, field as dc_field

import numpy as np

from . import _lib
from ._lib import (BeliefExtinguishedError, CudaError, GridlocError, KernelInfo, LikelihoodC, MapParseError,
                   PoseEstimateC, check)

__all__ = [
    "Context", "OccupancyMap", "DistanceField", "KernelSet", "Activation", "BeliefTensor", "MotionNoise",
    "OdometryDelta", "Pose2", "PoseEstimate", "SampleSet", "LidarScan", "LikelihoodParams", "StepScratch",
    "load_map", "init_uniform", "motion_vector", "build_kernels", "make_activation", "step", "step_async",
    "apply_motion", "belief_map", "argmax_state", "dither_samples", "scan_likelihood", "observation_update",
    "distance_field", "wrap_angle", "compose_delta", "Localizer", "LocalizerConfig",
    "write_belief_snapshot", "read_belief_snapshot", "DifficultyConfig", "map_difficulty",
    "BeliefExtinguishedError", "MapParseError", "CudaError", "GridlocError", "Engine",
    "raycast", "simulate_scans", "simulate_scan", "sequential_sum",
]


def _d(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _i(a):
    return a.ctypes.data_as(C.POINTER(C.c_int))


def _u8(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint8))


# ----------------------------------------------------------------- geometry
@dataclass
class Pose2:
    x: float = 0.0
    y: float = 0.0
    theta: float = 0.0


@dataclass
class OdometryDelta:
    """Body-frame motion: forward u, left v, heading change w (geometry.hpp:27-31)."""
    u: float = 0.0
    v: float = 0.0
    w: float = 0.0


@dataclass
class MotionNoise:
    """belief_tensor.hpp:16-20."""
    sigma_x: float = 0.03
    sigma_y: float = 0.03
    sigma_theta: float = 0.012


@dataclass
class LikelihoodParams:
    """observation.hpp:21-25."""
    sigma_hit: float = 0.2
    weight_floor: float = 0.05
    beam_stride: int = 4


@dataclass
class LidarScan:
    angles: np.ndarray
    ranges: np.ndarray
    max_range: float = 0.0


@dataclass
class SampleSet:
    cells: np.ndarray  # (n, 2) int32 (i, j) in emission order
    source_mass: float = 0.0


@dataclass
class PoseEstimate:
    pose: Pose2
    confidence: float
    i: int
    j: int
    k: int


@dataclass
class StepScratch:
    """belief_tensor.hpp:121-128; the fused kernel has no phase boundaries,
    so the whole step's device time lands in t_motion."""
    t_motion: float = 0.0
    t_diffusion: float = 0.0
    t_masking: float = 0.0


def wrap_angle(a: float) -> float:
    """geometry.hpp:8-13."""
    a = math.fmod(a, 2.0 * math.pi)
    if a < -math.pi:
        a += 2.0 * math.pi
    if a >= math.pi:
        a -= 2.0 * math.pi
    return a


def compose_delta(a: OdometryDelta, b: OdometryDelta) -> OdometryDelta:
    """geometry.hpp:56-60."""
    c, s = math.cos(a.w), math.sin(a.w)
    return OdometryDelta(a.u + c * b.u - s * b.v, a.v + s * b.u + c * b.v, a.w + b.w)


def compose(a: Pose2, d: OdometryDelta) -> Pose2:
    """geometry.hpp:36-45."""
    c, s = math.cos(a.theta), math.sin(a.theta)
    return Pose2(a.x + c * d.u - s * d.v, a.y + s * d.u + c * d.v, wrap_angle(a.theta + d.w))


# ------------------------------------------------------------------ context
class Context:
    """One CUDA device + stream; replaces ThreadPool& and StepScratch&."""

    _default: dict = {}

    def __init__(self, device: int = 0):
        self.lib = _lib.load()
        h = C.c_void_p()
        check(self.lib.gl_context_create(device, C.byref(h)))
        self.h = h
        self.device = device

    @classmethod
    def default(cls, device: int = 0) -> "Context":
        if device not in cls._default:
            cls._default[device] = Context(device)
        return cls._default[device]

    def set_path(self, path: int):
        check(self.lib.gl_context_set_path(self.h, path))

    def set_fast(self, enable: bool):
        """FAST fused variant on clean tensors (bitwise-identical results)."""
        check(self.lib.gl_context_set_fast(self.h, int(enable)))

    def set_himax(self, mode: int):
        """0 auto, 1 always, 2 never: the fused step's high-word max."""
        check(self.lib.gl_context_set_himax(self.h, int(mode)))

    def set_channel_chunks(self, n: int):
        """Fused-step channel chunks: 0 auto, n >= 1 fixed (1 for batches of
        small tensors on concurrent streams). Bit-identical either way."""
        check(self.lib.gl_context_set_channel_chunks(self.h, int(n)))

    def set_wave_tail(self, ctas: int, chunks: int = 3):
        """Fused-step wave-tail split: the grid's last `ctas` CTAs run their
        channels in `chunks` chunks (-1 auto: last ~1/5 of the partial wave,
        3 chunks; 0 off). Bit-identical."""
        check(self.lib.gl_context_set_wave_tail(self.h, int(ctas), int(chunks)))

    def set_host_exp(self, enable: bool):
        """scan_likelihood's final exp: host glibc (default, bit-exact) or
        CUDA's exp on the device (<= 1 ulp)."""
        check(self.lib.gl_context_set_host_exp(self.h, int(enable)))

    def set_wall_mask(self, enable: bool):
        """The wall-crossing mask extension (off by default; not in the
        reference): step() drops taps whose motion segment crosses a wall."""
        check(self.lib.gl_context_set_wall_mask(self.h, int(enable)))

    def set_tile_order(self, strip_tiles: int, stack: int = 0):
        """Fused-step tile order: strip_tiles -1 auto, 0 row-major, n =
        vertical strips of n tiles; stack n >= 2: a CTA's warps take n
        vertically adjacent tiles (L2 reuse of the vertical halo rows).
        Bit-identical for every setting."""
        check(self.lib.gl_context_set_tile_order(self.h, int(strip_tiles), int(stack)))

    def synchronize(self):
        check(self.lib.gl_context_synchronize(self.h))

    def set_step_timing(self, enable: bool):
        """CUDA events around every step for last_step_ms() (off by default:
        ~5 us of host time per step)."""
        check(self.lib.gl_context_set_step_timing(self.h, int(enable)))

    def last_step_ms(self) -> float:
        ms = C.c_double()
        check(self.lib.gl_context_last_step_ms(self.h, C.byref(ms)))
        return ms.value

    def launch_count(self) -> int:
        n = C.c_uint64()
        check(self.lib.gl_context_launch_count(self.h, C.byref(n)))
        return n.value

    def stream(self) -> int:
        s = C.c_void_p()
        check(self.lib.gl_context_stream(self.h, C.byref(s)))
        return s.value or 0

    def mark(self, i: int):
        """Record CUDA-event marker i on the context stream."""
        check(self.lib.gl_context_mark(self.h, i))

    def marks_ms(self, i: int, j: int) -> float:
        ms = C.c_double()
        check(self.lib.gl_context_marks_ms(self.h, i, j, C.byref(ms)))
        return ms.value

    def time_steps(self, enable, stride: int = 1):
        """Bracket every `stride`-th step kernel with CUDA events on the
        context stream (enable False: off)."""
        check(self.lib.gl_context_time_steps(self.h, max(1, int(stride)) if enable else 0))

    def step_times(self):
        """(total ms, count) of the timed step kernels since the last call."""
        tot = C.c_double()
        n = C.c_int()
        check(self.lib.gl_context_step_times(self.h, C.byref(tot), C.byref(n)))
        return tot.value, n.value

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.lib.gl_context_destroy(self.h)
                self.h = None
        except Exception:
            pass


def _ctx(ctx):
    return ctx if ctx is not None else Context.default()


# --------------------------------------------------------------------- maps
class OccupancyMap:
    """occupancy_map.hpp:35-81 (boundary ring forced occupied)."""

    def __init__(self, width, height, resolution, occupied, origin_x=0.0, origin_y=0.0, ctx=None):
        self.ctx = _ctx(ctx)
        occ = np.ascontiguousarray(np.asarray(occupied, dtype=np.uint8).reshape(height, width))
        h = C.c_void_p()
        check(self.ctx.lib.gl_map_create(self.ctx.h, width, height, resolution, origin_x, origin_y, _u8(occ),
                                         C.byref(h)))
        self.h = h
        w_, h_, fc = C.c_int(), C.c_int(), C.c_int()
        res, ox, oy = C.c_double(), C.c_double(), C.c_double()
        check(self.ctx.lib.gl_map_info(h, C.byref(w_), C.byref(h_), C.byref(res), C.byref(ox), C.byref(oy),
                                       C.byref(fc)))
        self._w, self._h, self._fc = w_.value, h_.value, fc.value
        self._res, self._ox, self._oy = res.value, ox.value, oy.value

    def width(self):
        return self._w

    def height(self):
        return self._h

    def resolution(self):
        return self._res

    def origin_x(self):
        return self._ox

    def origin_y(self):
        return self._oy

    def free_count(self):
        return self._fc

    def cells(self) -> np.ndarray:
        out = np.empty((self._h, self._w), np.uint8)
        check(self.ctx.lib.gl_map_cells(self.h, _u8(out)))
        return out

    def occupied(self, i, j):
        return bool(self.cells()[j, i])

    def free(self, i, j):
        return not self.occupied(i, j)

    def center_x(self, i):
        return self._ox + (i + 0.5) * self._res

    def center_y(self, j):
        return self._oy + (j + 0.5) * self._res

    def __del__(self):
        try:
            self.ctx.lib.gl_map_destroy(self.h)
        except Exception:
            pass


def load_map(data: bytes, threshold: int, resolution: float, origin_x=0.0, origin_y=0.0, ctx=None) -> OccupancyMap:
    """occupancy_map.hpp:106-108 (PGM P2/P5)."""
    lib = _lib.load()
    buf = np.frombuffer(bytes(data), dtype=np.uint8).copy()
    w, h = C.c_int(), C.c_int()
    check(lib.gl_load_map(_u8(buf), len(buf), threshold, C.byref(w), C.byref(h), None))
    occ = np.empty((h.value, w.value), np.uint8)
    check(lib.gl_load_map(_u8(buf), len(buf), threshold, C.byref(w), C.byref(h), _u8(occ)))
    return OccupancyMap(w.value, h.value, resolution, occ, origin_x, origin_y, ctx)


class DistanceField:
    """occupancy_map.hpp:85-101."""

    def __init__(self, m: OccupancyMap, ctx=None):
        self.ctx = _ctx(ctx)
        self.map = m
        h = C.c_void_p()
        check(self.ctx.lib.gl_field_create(self.ctx.h, m.h, C.byref(h)))
        self.h = h

    def values(self) -> np.ndarray:
        out = np.empty((self.map.height(), self.map.width()))
        check(self.ctx.lib.gl_field_values(self.h, _d(out)))
        return out

    def at(self, i, j):
        return float(self.values()[j, i])

    def __del__(self):
        try:
            self.ctx.lib.gl_field_destroy(self.h)
        except Exception:
            pass


def distance_field(m: OccupancyMap, ctx=None) -> DistanceField:
    return DistanceField(m, ctx)


# ------------------------------------------------------------------ kernels
class KernelSet:
    """belief_tensor.hpp:79-89 (host taps + device copy)."""

    def __init__(self, handle, lib):
        self.h = handle
        self.lib = lib
        info = KernelInfo()
        check(lib.gl_kernels_info(handle, C.byref(info)))
        self.info = info
        self.radius = info.radius
        self.separable = bool(info.separable)
        self.degenerate_spatial = bool(info.degenerate_spatial)
        self.degenerate_angular = bool(info.degenerate_angular)
        kw = 2 * info.radius + 1
        sep = np.zeros(kw if info.separable else 1)
        spatial = np.zeros(info.channels * kw * kw)
        off = np.zeros(info.n_angular, np.int32)
        w = np.zeros(info.n_angular)
        check(lib.gl_kernels_get(handle, _d(sep), _d(spatial), _i(off), _d(w)))
        self.sep = sep[: kw if info.separable else 0]
        self.spatial = spatial.reshape(info.channels, kw * kw)
        self.angular = [(int(o), float(x)) for o, x in zip(off, w)]

    @classmethod
    def from_arrays(cls, radius, separable, sep, spatial, angular, channels, degenerate_spatial=False,
                    degenerate_angular=False, ctx=None):
        """Wrap an explicit KernelSet (e.g. the reference's own)."""
        ctx = _ctx(ctx)
        info = KernelInfo(channels, radius, int(separable), int(degenerate_spatial), int(degenerate_angular),
                          len(angular))
        sep = np.ascontiguousarray(sep if sep is not None else np.zeros(1), dtype=np.float64)
        sp = None if spatial is None else np.ascontiguousarray(spatial, dtype=np.float64)
        off = np.array([a[0] for a in angular], np.int32)
        w = np.array([a[1] for a in angular], np.float64)
        h = C.c_void_p()
        check(ctx.lib.gl_kernels_create(ctx.h, C.byref(info), _d(sep), None if sp is None else _d(sp), _i(off),
                                        _d(w), C.byref(h)))
        return cls(h, ctx.lib)

    def __del__(self):
        try:
            self.lib.gl_kernels_destroy(self.h)
        except Exception:
            pass


def build_kernels(noise: MotionNoise, channels: int, cell_size: float, delta_theta: float) -> KernelSet:
    """belief_tensor.cpp:243-338 (host libm, like the reference)."""
    lib = _lib.load()
    h = C.c_void_p()
    check(lib.gl_build_kernels(noise.sigma_x, noise.sigma_y, noise.sigma_theta, channels, cell_size, delta_theta,
                               C.byref(h)))
    return KernelSet(h, lib)


class Activation:
    """belief_tensor.hpp:93-96, device-resident."""

    def __init__(self, handle, ctx, channels, w, h):
        self.h, self.ctx, self.channels, self._w, self._h = handle, ctx, channels, w, h

    def _get(self, which):
        out = np.empty((self.channels, self._h, self._w))
        args = [None, None]
        args[which] = _d(out)
        check(self.ctx.lib.gl_activation_get(self.ctx.h, self.h, *args))
        return out

    @property
    def values(self):
        return self._get(0)

    @property
    def inverse(self):
        return self._get(1)

    def __del__(self):
        try:
            self.ctx.lib.gl_activation_destroy(self.h)
        except Exception:
            pass


def make_activation(m: OccupancyMap, kernels: KernelSet, channels: int, ctx=None) -> Activation:
    """belief_tensor.cpp:354-394, computed on the device."""
    ctx = _ctx(ctx)
    h = C.c_void_p()
    check(ctx.lib.gl_make_activation(ctx.h, m.h, kernels.h, channels, C.byref(h)))
    return Activation(h, ctx, channels, m.width(), m.height())


# ------------------------------------------------------------------- tensor
class BeliefTensor:
    """belief_tensor.hpp:30-75 with the values resident in HBM."""

    def __init__(self, width=None, height=None, channels=None, cell_size=0.1, origin_x=0.0, origin_y=0.0,
                 ctx=None, _handle=None):
        self.ctx = _ctx(ctx)
        if _handle is None:
            h = C.c_void_p()
            check(self.ctx.lib.gl_tensor_create(self.ctx.h, width, height, channels, cell_size, origin_x, origin_y,
                                                C.byref(h)))
            _handle = h
        self.h = _handle
        w, hh, c = C.c_int(), C.c_int(), C.c_int()
        cs, ox, oy = C.c_double(), C.c_double(), C.c_double()
        check(self.ctx.lib.gl_tensor_info(self.h, C.byref(w), C.byref(hh), C.byref(c), C.byref(cs), C.byref(ox),
                                          C.byref(oy)))
        self._w, self._h, self._c = w.value, hh.value, c.value
        self._cell, self._ox, self._oy = cs.value, ox.value, oy.value

    def width(self):
        return self._w

    def height(self):
        return self._h

    def channels(self):
        return self._c

    def cell_size(self):
        return self._cell

    def origin_x(self):
        return self._ox

    def origin_y(self):
        return self._oy

    def delta_theta(self):
        return 2.0 * math.pi / self._c

    def theta_t(self) -> float:
        t = C.c_double()
        check(self.ctx.lib.gl_tensor_theta(self.h, C.byref(t)))
        return t.value

    def set_theta_t(self, t: float):
        check(self.ctx.lib.gl_tensor_set_theta(self.h, t))

    def channel_angle(self, k):
        return k * self.delta_theta() + self.theta_t()

    def plane_size(self):
        return self._w * self._h

    def size(self):
        return self._w * self._h * self._c

    def values(self) -> np.ndarray:
        """Download: (C, H, W) float64, layout [k][j][i]."""
        out = np.empty((self._c, self._h, self._w))
        check(self.ctx.lib.gl_tensor_download(self.ctx.h, self.h, _d(out)))
        return out

    def at(self, i: int, j: int, k: int) -> float:
        """One element (belief_tensor.hpp:55-60), read from the device."""
        x = C.c_double()
        off = (k * self._h + j) * self._w + i
        check(self.ctx.lib.gl_tensor_read(self.ctx.h, self.h, off, 1, C.byref(x)))
        return x.value

    def set_values(self, vals):
        v = np.ascontiguousarray(vals, dtype=np.float64).reshape(self._c, self._h, self._w)
        check(self.ctx.lib.gl_tensor_upload(self.ctx.h, self.h, _d(v)))

    def hash(self) -> int:
        hv = C.c_uint64()
        check(self.ctx.lib.gl_tensor_hash(self.ctx.h, self.h, C.byref(hv)))
        return hv.value

    def device_ptr(self) -> int:
        p = C.POINTER(C.c_double)()
        check(self.ctx.lib.gl_tensor_device_ptr(self.ctx.h, self.h, C.byref(p)))
        return C.cast(p, C.c_void_p).value

    def __del__(self):
        try:
            self.ctx.lib.gl_tensor_destroy(self.h)
        except Exception:
            pass


def tensor_hash_host(vals: np.ndarray) -> int:
    """Host restatement of gl_tensor_hash (order-independent splitmix sum)."""
    bits = np.ascontiguousarray(vals, dtype=np.float64).view(np.uint64).reshape(-1)
    idx = np.arange(bits.size, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = bits + idx * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
        return int(np.sum(z, dtype=np.uint64))


def init_uniform(m: OccupancyMap, channels: int, ctx=None) -> BeliefTensor:
    """belief_tensor.cpp:35-53."""
    ctx = _ctx(ctx) if ctx is not None else m.ctx
    h = C.c_void_p()
    check(ctx.lib.gl_init_uniform(ctx.h, m.h, channels, C.byref(h)))
    return BeliefTensor(ctx=ctx, _handle=h)


def motion_vector(u: OdometryDelta, k: int, theta_t: float, delta_theta: float, cell_size: float):
    """belief_tensor.cpp:55-62 (host libm; the library uses the same formula)."""
    angle = k * delta_theta + theta_t
    c, s = math.cos(angle), math.sin(angle)
    return (c * u.u - s * u.v) / cell_size, (s * u.u + c * u.v) / cell_size


def step(tensor: BeliefTensor, u: OdometryDelta, m: OccupancyMap, kernels: KernelSet, act: Activation, ctx=None,
         scratch: StepScratch | None = None):
    """belief_tensor.cpp:396-498. Raises BeliefExtinguishedError like the reference."""
    ctx = _ctx(ctx) if ctx is not None else tensor.ctx
    rc = ctx.lib.gl_step(ctx.h, tensor.h, u.u, u.v, u.w, m.h, kernels.h, act.h)
    if scratch is not None:
        scratch.t_motion = ctx.last_step_ms() * 1e-3
        scratch.t_diffusion = scratch.t_masking = 0.0
    check(rc)


def step_async(tensor: BeliefTensor, u: OdometryDelta, m: OccupancyMap, kernels: KernelSet, act: Activation,
               ctx=None):
    """Enqueue a step without reading back the status (see gl_step_async)."""
    ctx = _ctx(ctx) if ctx is not None else tensor.ctx
    check(ctx.lib.gl_step_async(ctx.h, tensor.h, u.u, u.v, u.w, m.h, kernels.h, act.h))


def tensor_status(tensor: BeliefTensor):
    check(tensor.ctx.lib.gl_tensor_status(tensor.ctx.h, tensor.h))


def tensors_status(tensors, ctx=None):
    """The latest step status of tensors stepped on one context, read in one
    round trip (gl_tensors_status); raises BeliefExtinguishedError if any is
    extinguished."""
    tensors = list(tensors)
    if not tensors:
        return
    ctx = _ctx(ctx) if ctx is not None else tensors[0].ctx
    arr = (C.c_void_p * len(tensors))(*[t.h for t in tensors])
    out = (C.c_int * len(tensors))()
    check(ctx.lib.gl_tensors_status(ctx.h, C.cast(arr, C.POINTER(C.c_void_p)), len(tensors), out))


def apply_motion(tensor: BeliefTensor, u: OdometryDelta):
    """belief_tensor.cpp:340-352."""
    check(tensor.ctx.lib.gl_apply_motion(tensor.ctx.h, tensor.h, u.u, u.v, u.w))


def belief_map(tensor: BeliefTensor) -> np.ndarray:
    """belief_tensor.cpp:500-510: (H, W) per-cell max over channels."""
    out = np.empty((tensor.height(), tensor.width()))
    check(tensor.ctx.lib.gl_belief_map(tensor.ctx.h, tensor.h, _d(out)))
    return out


@dataclass
class DifficultyConfig:
    """evaluation.hpp:21-29."""
    error_threshold: float = 1.0
    beam_count: int = 8
    fov: float = 2.0 * math.pi
    max_range: float = 8.0
    stride: int = 1
    theta_bins: int = 8
    likelihood: LikelihoodParams = dc_field(default_factory=lambda: LikelihoodParams(0.2, 0.05, 1))


def map_difficulty(m: OccupancyMap, f: DistanceField, cfg: DifficultyConfig = None, ctx=None) -> float:
    """evaluation.cpp:25-72 on the device (bit-exact)."""
    from ._lib import DifficultyC
    cfg = cfg or DifficultyConfig()
    ctx = _ctx(ctx)
    lk = cfg.likelihood
    c = DifficultyC(cfg.error_threshold, cfg.beam_count, cfg.fov, cfg.max_range, cfg.stride, cfg.theta_bins,
                    LikelihoodC(lk.sigma_hit, lk.weight_floor, lk.beam_stride))
    out = C.c_double()
    check(ctx.lib.gl_map_difficulty(ctx.h, m.h, f.h, C.byref(c), C.byref(out)))
    return out.value


def write_belief_snapshot(tensor: BeliefTensor, path: str):
    """belief_tensor.cpp:543-563: BLF1, float32 payload (lossy)."""
    check(tensor.ctx.lib.gl_write_belief_snapshot(tensor.ctx.h, tensor.h, os.fsencode(path)))


def read_belief_snapshot(path: str, cell_size: float, origin_x: float, origin_y: float, ctx=None) -> BeliefTensor:
    """belief_tensor.cpp:565-587."""
    ctx = _ctx(ctx)
    h = C.c_void_p()
    check(ctx.lib.gl_read_belief_snapshot(ctx.h, os.fsencode(path), cell_size, origin_x, origin_y, C.byref(h)))
    return BeliefTensor(ctx=ctx, _handle=h)


def argmax_state(tensor: BeliefTensor) -> PoseEstimate:
    """belief_tensor.cpp:512-541."""
    e = PoseEstimateC()
    check(tensor.ctx.lib.gl_argmax(tensor.ctx.h, tensor.h, C.byref(e)))
    return PoseEstimate(Pose2(e.x, e.y, e.theta), e.confidence, e.i, e.j, e.k)


def dither_samples(bm, budget: int, ctx=None) -> SampleSet:
    """observation.cpp:11-71. ``bm`` is a host (H, W) belief map or a
    BeliefTensor (then belief_map is taken on the device)."""
    n = C.c_int()
    mass = C.c_double()
    if isinstance(bm, BeliefTensor):
        ctx = bm.ctx
        cap = max(1, min(bm.plane_size(), 4 * max(budget, 1) + 64))
        cells = np.zeros(2 * cap, np.int32)
        check(ctx.lib.gl_dither_tensor(ctx.h, bm.h, budget, _i(cells), cap, C.byref(n), C.byref(mass)))
    else:
        ctx = _ctx(ctx)
        g = np.ascontiguousarray(bm, dtype=np.float64)
        h, w = g.shape
        cap = max(1, min(h * w, 4 * max(budget, 1) + 64))
        cells = np.zeros(2 * cap, np.int32)
        check(ctx.lib.gl_dither(ctx.h, _d(g), w, h, budget, _i(cells), cap, C.byref(n), C.byref(mass)))
    if n.value > cap:
        raise GridlocError("sample capacity exceeded")
    return SampleSet(cells[: 2 * n.value].reshape(-1, 2).copy(), mass.value)


def _lp(p: LikelihoodParams):
    return LikelihoodC(p.sigma_hit, p.weight_floor, p.beam_stride)


def scan_likelihood(m: OccupancyMap, f: DistanceField, pose: Pose2, scan: LidarScan,
                    params: LikelihoodParams = LikelihoodParams(), ctx=None) -> float:
    """observation.cpp:73-111 (one pose, evaluated by the device kernel)."""
    ctx = _ctx(ctx) if ctx is not None else m.ctx
    a = np.ascontiguousarray(scan.angles, dtype=np.float64)
    r = np.ascontiguousarray(scan.ranges, dtype=np.float64)
    if a.size == 0 or a.size != r.size:
        raise ValueError("scan must have matching, nonempty beams")
    out = C.c_double()
    check(ctx.lib.gl_scan_likelihood(ctx.h, m.h, f.h, pose.x, pose.y, pose.theta, _d(a), _d(r), a.size,
                                     scan.max_range, _lp(params), C.byref(out)))
    return out.value


def observation_update(tensor: BeliefTensor, samples: SampleSet, scan: LidarScan, m: OccupancyMap,
                       f: DistanceField, params: LikelihoodParams = LikelihoodParams(), ctx=None):
    """observation.cpp:113-170."""
    ctx = _ctx(ctx) if ctx is not None else tensor.ctx
    cells = np.ascontiguousarray(samples.cells, dtype=np.int32).reshape(-1)
    a = np.ascontiguousarray(scan.angles, dtype=np.float64)
    r = np.ascontiguousarray(scan.ranges, dtype=np.float64)
    if cells.size and (a.size == 0 or a.size != r.size):
        raise ValueError("scan must have matching, nonempty beams")
    check(ctx.lib.gl_observation_update(ctx.h, tensor.h, _i(cells), cells.size // 2, _d(a), _d(r), a.size,
                                        scan.max_range, m.h, f.h, _lp(params)))


# ---------------------------------------------------------------- localizer
@dataclass
class LocalizerConfig:
    """localizer.hpp:17-26."""
    channels: int = 128
    motion_noise: MotionNoise = dc_field(default_factory=MotionNoise)
    likelihood: LikelihoodParams = dc_field(default_factory=LikelihoodParams)
    sample_budget: int = 512
    use_samples: bool = True
    trigger_cells: float = 1.0


class Localizer:
    """Drop-in for gridloc::Localizer (localizer.hpp:28-71, localizer.cpp:7-66)
    with the tensor, kernels and activations resident on the device."""

    def __init__(self, m: OccupancyMap, field: DistanceField, config: LocalizerConfig = LocalizerConfig(),
                 ctx=None):
        self.ctx = _ctx(ctx) if ctx is not None else m.ctx
        self.map, self.field, self.config = m, field, config
        C_ = config.channels
        dth = 2.0 * math.pi / C_
        self.kernels = build_kernels(config.motion_noise, C_, m.resolution(), dth)
        self.activation = make_activation(m, self.kernels, C_, self.ctx)
        self.rot_kernels = build_kernels(MotionNoise(1e-4, 1e-4, config.motion_noise.sigma_theta), C_,
                                         m.resolution(), dth)
        self.rot_activation = make_activation(m, self.rot_kernels, C_, self.ctx)
        self.tensor = init_uniform(m, C_, self.ctx)
        self.pending = OdometryDelta()
        self.trigger_trans_m = config.trigger_cells * m.resolution()
        self.trigger_rot = math.pi / C_
        self._steps = 0

    def integrate_odometry(self, delta: OdometryDelta) -> bool:
        self.pending = compose_delta(self.pending, delta)
        if (math.hypot(self.pending.u, self.pending.v) >= self.trigger_trans_m
                or abs(self.pending.w) >= self.trigger_rot):
            self.flush()
            return True
        return False

    def flush(self):
        translated = math.hypot(self.pending.u, self.pending.v) >= 0.5 * self.trigger_trans_m
        if translated:
            step(self.tensor, self.pending, self.map, self.kernels, self.activation, self.ctx)
        else:
            step(self.tensor, self.pending, self.map, self.rot_kernels, self.rot_activation, self.ctx)
        self.pending = OdometryDelta()
        self._steps += 1

    def observe(self, scan: LidarScan):
        if not self.config.use_samples:
            return
        eps = 1e-12
        if abs(self.pending.u) > eps or abs(self.pending.v) > eps or abs(self.pending.w) > eps:
            self.flush()
        samples = dither_samples(self.tensor, self.config.sample_budget)
        observation_update(self.tensor, samples, scan, self.map, self.field, self.config.likelihood, self.ctx)

    def estimate(self) -> PoseEstimate:
        est = argmax_state(self.tensor)
        est.pose = compose(est.pose, self.pending)
        est.pose.theta = wrap_angle(est.pose.theta)
        return est

    def belief(self) -> BeliefTensor:
        return self.tensor

    def steps_run(self) -> int:
        return self._steps


def sequential_sum(values, ctx=None) -> float:
    """dither_samples' total (observation.cpp:16-17): the reference's
    sequential FP64 sum in order, bit-exact, computed on the device by a
    parallel binade scan. Values must be finite and >= 0."""
    ctx = _ctx(ctx)
    v = np.ascontiguousarray(values, dtype=np.float64).reshape(-1)
    out = C.c_double()
    check(ctx.lib.gl_sequential_sum(ctx.h, _d(v), v.size, C.byref(out)))
    return out.value


# ------------------------------------------------------ raycast / scans
def raycast(m: OccupancyMap, rays, max_range: float, ctx=None) -> np.ndarray:
    """occupancy_map.cpp:273-332 for a batch of rays: rays (n, 3) = (x, y,
    angle); returns (n,) ranges in meters, bit-exact, on the device."""
    ctx = _ctx(ctx) if ctx is not None else m.ctx
    r = np.ascontiguousarray(np.asarray(rays, dtype=np.float64).reshape(-1, 3))
    out = np.empty(len(r))
    check(ctx.lib.gl_raycast(ctx.h, m.h, _d(r), len(r), max_range, _d(out)))
    return out


def simulate_scans(m: OccupancyMap, poses, beam_count: int, fov: float, max_range: float,
                   range_noise_sigma: float = 0.0, rng=None, ctx=None):
    """simulator.cpp:63-94 for a batch of poses (n, 3) = (x, y, theta):
    returns (angles (beams,), ranges (n, beams)). With range noise, `rng`
    (the reference's xoshiro256++ generator, floorplan.Rng) draws one normal
    per beam in pose-major order, exactly as n successive simulate_scan
    calls on the reference's Rng would."""
    ctx = _ctx(ctx) if ctx is not None else m.ctx
    p = np.ascontiguousarray(np.asarray(poses, dtype=np.float64).reshape(-1, 3))
    n = len(p)
    noise = None
    if range_noise_sigma > 0.0:
        if rng is None:
            raise ValueError("range noise needs an rng (reference draw order)")
        noise = np.array([rng.normal() for _ in range(n * beam_count)], dtype=np.float64)
    angles = np.empty(max(beam_count, 0))
    ranges = np.empty((n, max(beam_count, 0)))
    check(ctx.lib.gl_simulate_scans(ctx.h, m.h, _d(p), n, beam_count, fov, max_range, range_noise_sigma,
                                    None if noise is None else _d(noise), _d(angles), _d(ranges)))
    return angles, ranges


def simulate_scan(m: OccupancyMap, pose: Pose2, beam_count: int, fov: float, max_range: float,
                  range_noise_sigma: float = 0.0, rng=None, ctx=None) -> LidarScan:
    """simulator.cpp:63-94 (one pose)."""
    a, r = simulate_scans(m, [(pose.x, pose.y, pose.theta)], beam_count, fov, max_range, range_noise_sigma, rng,
                          ctx)
    return LidarScan(a, r[0], max_range)


# ------------------------------------------------------------------ engine
class Engine:
    """gl_engine: ONE process driving a theta-slab sharded belief over a
    device list; the Python face of the C++ callers'
    multi-GPU path. Shard s owns channels [s*C/n, (s+1)*C/n) on devices[s];
    halo planes are read over peer memory inside the step kernel, the 8-byte
    step max is all-reduced by NCCL (distinct devices) or a peer-memory
    gather (P2P). Bitwise the unsharded tensor. Slot 0 = main kernels,
    slot 1 = rotation-only (Localizer)."""

    def __init__(self, devices, m: "OccupancyMap", channels: int, mode: int = 0):
        self.lib = _lib.load()
        devs = (C.c_int * len(devices))(*devices)
        occ = np.ascontiguousarray(m.cells(), dtype=np.uint8)
        h = C.c_void_p()
        check(self.lib.gl_engine_create(devs, len(devices), m.width(), m.height(), m.resolution(), m.origin_x(),
                                        m.origin_y(), _u8(occ), channels, mode, C.byref(h)))
        self.h = h
        self.W, self.H, self.C = m.width(), m.height(), channels
        self.cell, self.ox, self.oy = m.resolution(), m.origin_x(), m.origin_y()

    def info(self):
        n, mode, halo = C.c_int(), C.c_int(), C.c_int()
        check(self.lib.gl_engine_info(self.h, C.byref(n), C.byref(mode), C.byref(halo)))
        return {"shards": n.value, "mode": {1: "nccl", 2: "p2p"}.get(mode.value, mode.value), "halo": halo.value}

    def set_kernels(self, slot: int, kernels: "KernelSet"):
        check(self.lib.gl_engine_set_kernels(self.h, slot, kernels.h))

    def init_uniform(self):
        check(self.lib.gl_engine_init_uniform(self.h))

    def step(self, u: "OdometryDelta", slot: int = 0):
        check(self.lib.gl_engine_step(self.h, u.u, u.v, u.w, slot))

    def step_async(self, u: "OdometryDelta", slot: int = 0):
        check(self.lib.gl_engine_step_async(self.h, u.u, u.v, u.w, slot))

    def status(self):
        check(self.lib.gl_engine_status(self.h))

    def argmax(self) -> PoseEstimate:
        e = PoseEstimateC()
        check(self.lib.gl_engine_argmax(self.h, C.byref(e)))
        return PoseEstimate(Pose2(e.x, e.y, e.theta), e.confidence, e.i, e.j, e.k)

    def belief_map(self) -> np.ndarray:
        out = np.empty((self.H, self.W))
        check(self.lib.gl_engine_belief_map(self.h, _d(out)))
        return out

    def observe(self, scan: "LidarScan", params: "LikelihoodParams" = None, budget: int = 512) -> SampleSet:
        params = params or LikelihoodParams()
        a = np.ascontiguousarray(scan.angles, dtype=np.float64)
        r = np.ascontiguousarray(scan.ranges, dtype=np.float64)
        cap = max(1, min(self.W * self.H, 4 * max(budget, 1) + 64))
        cells = np.zeros(2 * cap, np.int32)
        n, mass = C.c_int(), C.c_double()
        check(self.lib.gl_engine_observe(self.h, budget, _d(a), _d(r), a.size, scan.max_range, _lp(params),
                                         _i(cells), cap, C.byref(n), C.byref(mass)))
        return SampleSet(cells[: 2 * min(n.value, cap)].reshape(-1, 2).copy(), mass.value)

    def values(self):
        out = np.empty((self.C, self.H, self.W))
        th = C.c_double()
        check(self.lib.gl_engine_download(self.h, _d(out), C.byref(th)))
        return out, th.value

    def set_values(self, vals, theta_t: float = 0.0):
        v = np.ascontiguousarray(vals, dtype=np.float64)
        check(self.lib.gl_engine_upload(self.h, _d(v), theta_t))

    def hash(self) -> int:
        hv = C.c_uint64()
        check(self.lib.gl_engine_hash(self.h, C.byref(hv)))
        return hv.value

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.gl_engine_destroy(self.h)
            self.h = None
