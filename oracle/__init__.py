"""TEST INFRASTRUCTURE ONLY — Python bindings for the two CPU checkers.

* ``port``: our plain-C restatement ``oracle/liboracle.so`` (gl_oracle.c).
* ``ref``:  the UNMODIFIED reference compiled from /root/reference into
  ``oracle/_ref/libgridloc_ref.so`` by ``oracle/Makefile`` (extern "C" shim in
  ``oracle/ref/ref_shim.cpp``). Present here and, as a prebuilt file, on the
  GPU box.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU legs may import
this package, and only as the checker / CPU baseline. The product
(``paper_1910_00572_b200``) never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libgridloc_ref.so")

OK, EXTINGUISHED, INVALID, MAP_PARSE, RUNTIME = 0, 1, 2, 3, 4

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_u8p = C.POINTER(C.c_uint8)
_vp = C.c_void_p


def build() -> None:
    """Compile the checkers (make -C oracle)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _d(a):
    return a.ctypes.data_as(_dp)


def _i(a):
    return a.ctypes.data_as(_ip)


def _u8(a):
    return a.ctypes.data_as(_u8p)


class OracleError(RuntimeError):
    def __init__(self, code, msg=""):
        super().__init__(f"oracle status {code}: {msg}")
        self.code = code


# --------------------------------------------------------------------- port
class _Kernels(C.Structure):
    _fields_ = [
        ("channels", C.c_int),
        ("radius", C.c_int),
        ("separable", C.c_int),
        ("degenerate_spatial", C.c_int),
        ("degenerate_angular", C.c_int),
        ("sep", C.c_double * 64),
        ("spatial", _dp),
        ("n_ang", C.c_int),
        ("ang_off", C.c_int * 4096),
        ("ang_w", C.c_double * 4096),
    ]


class Kernels:
    """KernelSet (belief_tensor.hpp:79-89) as numpy arrays."""

    def __init__(self, radius, separable, sep, spatial, ang_off, ang_w,
                 degenerate_spatial=False, degenerate_angular=False):
        self.radius = int(radius)
        self.separable = bool(separable)
        self.sep = np.ascontiguousarray(sep, dtype=np.float64)
        self.spatial = np.ascontiguousarray(spatial, dtype=np.float64)
        self.ang_off = np.ascontiguousarray(ang_off, dtype=np.int32)
        self.ang_w = np.ascontiguousarray(ang_w, dtype=np.float64)
        self.degenerate_spatial = bool(degenerate_spatial)
        self.degenerate_angular = bool(degenerate_angular)

    def __repr__(self):
        return (f"Kernels(r={self.radius}, sep={self.separable}, "
                f"n_ang={len(self.ang_w)})")


class Port:
    """ctypes wrapper of liboracle.so (the C restatement)."""

    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            build()
        L = self.lib = C.CDLL(path)
        L.glo_build_kernels.argtypes = [C.c_double] * 3 + [C.c_int, C.c_double, C.c_double, C.POINTER(_Kernels)]
        L.glo_kernels_free.argtypes = [C.POINTER(_Kernels)]
        L.glo_motion_vector.argtypes = [C.c_double, C.c_double, C.c_int, C.c_double, C.c_double, C.c_double, _dp, _dp]
        L.glo_make_activation.argtypes = [_u8p, C.c_int, C.c_int, C.POINTER(_Kernels), _dp, _dp]
        L.glo_init_uniform.argtypes = [_u8p, C.c_int, C.c_int, C.c_int, _dp]
        L.glo_step.argtypes = [_dp, C.c_int, C.c_int, C.c_int, C.c_double, _dp, C.c_double, C.c_double, C.c_double,
                               _u8p, C.POINTER(_Kernels), _dp]
        L.glo_step_wall.argtypes = [_dp, C.c_int, C.c_int, C.c_int, C.c_double, _dp, C.c_double, C.c_double,
                                    C.c_double, _u8p, C.POINTER(_Kernels), _dp, C.c_int]
        L.glo_seg_cells.argtypes = [C.c_int, C.c_int, _ip, _ip, C.c_int]
        L.glo_apply_motion.argtypes = [_dp, C.c_int, C.c_int, C.c_int, C.c_double, _dp, C.c_double, C.c_double, C.c_double]
        L.glo_belief_map.argtypes = [_dp, C.c_int, C.c_int, C.c_int, _dp]
        L.glo_argmax.argtypes = [_dp, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, C.c_double,
                                 _ip, _dp, _dp]
        L.glo_dither.argtypes = [_dp, C.c_int, C.c_int, C.c_int, _ip, C.c_int, _ip, _dp]
        L.glo_distance_field.argtypes = [_u8p, C.c_int, C.c_int, C.c_double, _dp]
        L.glo_scan_likelihood.argtypes = [_u8p, _dp, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                          C.c_double, C.c_double, C.c_double, _dp, _dp, C.c_int, C.c_double,
                                          C.c_double, C.c_double, C.c_int, _dp]
        L.glo_observation_update.argtypes = [_dp, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                             C.c_double, _ip, C.c_int, _dp, _dp, C.c_int, C.c_double, _u8p, _dp,
                                             C.c_double, C.c_double, C.c_int]
        L.glo_load_map.argtypes = [_u8p, C.c_size_t, C.c_int, _ip, _ip, _u8p]

    # kernels ------------------------------------------------------------
    def _ks(self, ks: Kernels, channels: int) -> _Kernels:
        s = _Kernels()
        s.channels = channels
        s.radius = ks.radius
        s.separable = int(ks.separable)
        for t, v in enumerate(ks.sep):
            s.sep[t] = v
        s.spatial = _d(ks.spatial)
        s.n_ang = len(ks.ang_w)
        for t in range(len(ks.ang_w)):
            s.ang_off[t] = int(ks.ang_off[t])
            s.ang_w[t] = float(ks.ang_w[t])
        s._keep = ks  # keep spatial alive
        return s

    def build_kernels(self, sx, sy, st, channels, cell, dtheta=None) -> Kernels:
        if dtheta is None:
            dtheta = 2.0 * np.pi / channels
        s = _Kernels()
        rc = self.lib.glo_build_kernels(sx, sy, st, channels, cell, dtheta, C.byref(s))
        if rc:
            raise OracleError(rc, "build_kernels")
        kw = 2 * s.radius + 1
        spatial = np.ctypeslib.as_array(s.spatial, shape=(channels * kw * kw,)).copy()
        ks = Kernels(s.radius, s.separable, np.array(s.sep[: kw if s.separable else 0]), spatial,
                     np.array(s.ang_off[: s.n_ang]), np.array(s.ang_w[: s.n_ang]),
                     s.degenerate_spatial, s.degenerate_angular)
        self.lib.glo_kernels_free(C.byref(s))
        return ks

    def motion_vector(self, u, v, k, theta_t, dtheta, cell):
        dx, dy = C.c_double(), C.c_double()
        self.lib.glo_motion_vector(u, v, k, theta_t, dtheta, cell, C.byref(dx), C.byref(dy))
        return dx.value, dy.value

    def make_activation(self, occ, ks: Kernels, channels):
        h, w = occ.shape
        occ = np.ascontiguousarray(occ, dtype=np.uint8)
        vals = np.empty((channels, h, w))
        inv = np.empty((channels, h, w))
        self.lib.glo_make_activation(_u8(occ), w, h, C.byref(self._ks(ks, channels)), _d(vals), _d(inv))
        return vals, inv

    def init_uniform(self, occ, channels):
        h, w = occ.shape
        occ = np.ascontiguousarray(occ, dtype=np.uint8)
        out = np.empty((channels, h, w))
        rc = self.lib.glo_init_uniform(_u8(occ), w, h, channels, _d(out))
        if rc:
            raise OracleError(rc, "init_uniform")
        return out

    def step(self, B, theta_t, u, v, dw, occ, cell, ks: Kernels, inv, wall: bool = False):
        """In-place step on B (C,H,W) float64; returns (status, theta_t).
        wall: the wall-crossing mask extension (glo_step_wall)."""
        Cn, h, w = B.shape
        th = C.c_double(theta_t)
        occ = np.ascontiguousarray(occ, dtype=np.uint8)
        if wall:
            rc = self.lib.glo_step_wall(_d(B), w, h, Cn, cell, C.byref(th), u, v, dw, _u8(occ),
                                        C.byref(self._ks(ks, Cn)), _d(inv), 1)
        else:
            rc = self.lib.glo_step(_d(B), w, h, Cn, cell, C.byref(th), u, v, dw, _u8(occ),
                                   C.byref(self._ks(ks, Cn)), _d(inv))
        return rc, th.value

    def seg_cells(self, ox, oy, cap=64):
        """Cells the tap offset (ox, oy) crosses, relative to the destination."""
        qx = np.zeros(cap, np.int32)
        qy = np.zeros(cap, np.int32)
        n = self.lib.glo_seg_cells(ox, oy, _i(qx), _i(qy), cap)
        return list(zip(qx[:min(n, cap)].tolist(), qy[:min(n, cap)].tolist())), n

    def apply_motion(self, B, theta_t, u, v, dw, cell):
        Cn, h, w = B.shape
        th = C.c_double(theta_t)
        self.lib.glo_apply_motion(_d(B), w, h, Cn, cell, C.byref(th), u, v, dw)
        return th.value

    def belief_map(self, B):
        Cn, h, w = B.shape
        out = np.empty((h, w))
        self.lib.glo_belief_map(_d(np.ascontiguousarray(B)), w, h, Cn, _d(out))
        return out

    def argmax(self, B, cell, ox, oy, theta_t):
        Cn, h, w = B.shape
        ijk = np.zeros(3, np.int32)
        pose = np.zeros(3)
        conf = C.c_double()
        rc = self.lib.glo_argmax(_d(np.ascontiguousarray(B)), w, h, Cn, cell, ox, oy, theta_t, _i(ijk), _d(pose),
                                 C.byref(conf))
        if rc:
            raise OracleError(rc, "argmax")
        return tuple(int(x) for x in ijk), tuple(float(x) for x in pose), conf.value

    def dither(self, bm, budget):
        h, w = bm.shape
        bm = np.ascontiguousarray(bm, dtype=np.float64)
        cap = max(1, min(h * w, 4 * budget + 16))
        cells = np.zeros(2 * cap, np.int32)
        n = C.c_int()
        mass = C.c_double()
        rc = self.lib.glo_dither(_d(bm), w, h, budget, _i(cells), cap, C.byref(n), C.byref(mass))
        if rc:
            raise OracleError(rc, "dither")
        assert n.value <= cap
        return cells[: 2 * n.value].reshape(-1, 2).copy(), mass.value

    def distance_field(self, occ, res):
        h, w = occ.shape
        out = np.empty((h, w))
        self.lib.glo_distance_field(_u8(np.ascontiguousarray(occ, dtype=np.uint8)), w, h, res, _d(out))
        return out

    def scan_likelihood(self, occ, field, res, ox, oy, pose, angles, ranges, max_range, sigma_hit=0.2,
                        weight_floor=0.05, beam_stride=4):
        h, w = occ.shape
        out = C.c_double()
        a = np.ascontiguousarray(angles, dtype=np.float64)
        r = np.ascontiguousarray(ranges, dtype=np.float64)
        rc = self.lib.glo_scan_likelihood(_u8(np.ascontiguousarray(occ, dtype=np.uint8)), _d(field), w, h, res, ox,
                                          oy, pose[0], pose[1], pose[2], _d(a), _d(r), len(a), max_range, sigma_hit,
                                          weight_floor, beam_stride, C.byref(out))
        if rc:
            raise OracleError(rc, "scan_likelihood")
        return out.value

    def observation_update(self, B, cell, ox, oy, theta_t, cells, angles, ranges, max_range, occ, field,
                           sigma_hit=0.2, weight_floor=0.05, beam_stride=4):
        Cn, h, w = B.shape
        cells = np.ascontiguousarray(cells, dtype=np.int32).reshape(-1)
        a = np.ascontiguousarray(angles, dtype=np.float64)
        r = np.ascontiguousarray(ranges, dtype=np.float64)
        return self.lib.glo_observation_update(_d(B), w, h, Cn, cell, ox, oy, theta_t, _i(cells), len(cells) // 2,
                                               _d(a), _d(r), len(a), max_range,
                                               _u8(np.ascontiguousarray(occ, dtype=np.uint8)),
                                               _d(np.ascontiguousarray(field)), sigma_hit, weight_floor, beam_stride)

    def load_map(self, data: bytes, threshold=250):
        buf = np.frombuffer(data, dtype=np.uint8).copy()
        w, h = C.c_int(), C.c_int()
        rc = self.lib.glo_load_map(_u8(buf), len(buf), threshold, C.byref(w), C.byref(h), None)
        if rc:
            raise OracleError(rc, "load_map")
        occ = np.empty((h.value, w.value), np.uint8)
        rc = self.lib.glo_load_map(_u8(buf), len(buf), threshold, C.byref(w), C.byref(h), _u8(occ))
        if rc:
            raise OracleError(rc, "load_map")
        return occ


# ---------------------------------------------------------------------- ref
def ref_available() -> bool:
    return os.path.exists(REF_SO)


class Ref:
    """ctypes wrapper of the reference library (oracle/_ref)."""

    def __init__(self, path: str = REF_SO):
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_pool_new.restype = _vp
        L.ref_pool_new.argtypes = [C.c_int]
        L.ref_pool_free.argtypes = [_vp]
        L.ref_pool_threads.argtypes = [_vp]
        L.ref_map_new.argtypes = [C.c_int, C.c_int, C.c_double, _u8p, C.c_double, C.c_double, C.POINTER(_vp)]
        L.ref_map_load.argtypes = [_u8p, C.c_size_t, C.c_int, C.c_double, C.c_double, C.c_double, C.POINTER(_vp)]
        L.ref_map_free.argtypes = [_vp]
        L.ref_map_dims.argtypes = [_vp, _ip, _ip, _ip]
        L.ref_map_cells.argtypes = [_vp, _u8p]
        L.ref_write_pgm.argtypes = [_vp, _u8p, C.c_size_t, C.POINTER(C.c_size_t)]
        L.ref_field_new.restype = _vp
        L.ref_field_new.argtypes = [_vp]
        L.ref_field_free.argtypes = [_vp]
        L.ref_field_values.argtypes = [_vp, _dp]
        L.ref_kernels_new.argtypes = [C.c_double] * 3 + [C.c_int, C.c_double, C.c_double, C.POINTER(_vp)]
        L.ref_kernels_free.argtypes = [_vp]
        L.ref_kernels_info.argtypes = [_vp] + [_ip] * 6
        L.ref_kernels_get.argtypes = [_vp, _dp, _dp, _ip, _dp]
        L.ref_activation_new.restype = _vp
        L.ref_activation_new.argtypes = [_vp, _vp, C.c_int, _vp]
        L.ref_activation_free.argtypes = [_vp]
        L.ref_activation_get.argtypes = [_vp, _dp, _dp]
        L.ref_tensor_new.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, C.POINTER(_vp)]
        L.ref_tensor_init_uniform.argtypes = [_vp, C.c_int, C.POINTER(_vp)]
        L.ref_tensor_free.argtypes = [_vp]
        L.ref_tensor_set.argtypes = [_vp, _dp, C.c_double]
        L.ref_tensor_get.argtypes = [_vp, _dp, _dp]
        L.ref_write_snapshot.argtypes = [_vp, C.c_char_p]
        L.ref_read_snapshot.argtypes = [C.c_char_p, C.c_double, C.c_double, C.c_double, C.POINTER(_vp)]
        L.ref_tensor_dims.argtypes = [_vp, _ip, _ip, _ip]
        L.ref_map_difficulty.argtypes = [_vp, _vp, C.c_double, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int,
                                         C.c_double, C.c_double, C.c_int, _vp, _dp]
        L.ref_world.argtypes = [C.c_int, C.POINTER(_vp)]
        L.ref_scratch_new.restype = _vp
        L.ref_scratch_free.argtypes = [_vp]
        L.ref_scratch_times.argtypes = [_vp, _dp]
        L.ref_step.argtypes = [_vp, C.c_double, C.c_double, C.c_double, _vp, _vp, _vp, _vp, _vp]
        L.ref_apply_motion.argtypes = [_vp, C.c_double, C.c_double, C.c_double]
        L.ref_motion_vector.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int, C.c_double, C.c_double,
                                        C.c_double, _dp, _dp]
        L.ref_belief_map.argtypes = [_vp, _dp]
        L.ref_argmax.argtypes = [_vp, _ip, _dp, _dp]
        L.ref_dither.argtypes = [_dp, C.c_int, C.c_int, C.c_int, _ip, C.c_int, _ip, _dp]
        L.ref_scan_likelihood.argtypes = [_vp, _vp, C.c_double, C.c_double, C.c_double, _dp, _dp, C.c_int,
                                          C.c_double, C.c_double, C.c_double, C.c_int, _dp]
        L.ref_observation_update.argtypes = [_vp, _ip, C.c_int, _dp, _dp, C.c_int, C.c_double, _vp, _vp,
                                             C.c_double, C.c_double, C.c_int, _vp]
        L.ref_simulate_scan.argtypes = [_vp, C.c_double, C.c_double, C.c_double, C.c_int, C.c_double, C.c_double,
                                        C.c_double, C.c_uint64, _dp, _dp]
        L.ref_gen_trace.argtypes = [_vp, C.c_int, C.c_double, C.c_double, C.c_double, C.c_uint64, C.c_int,
                                    C.c_double, C.c_double, C.c_int, C.c_double, C.c_double, _dp, C.c_int, _ip,
                                    _dp, C.c_int, _ip]

    def err(self):
        return self.lib.ref_last_error().decode()

    def check(self, rc, what):
        if rc:
            raise OracleError(rc, f"{what}: {self.err()}")


class RefMap:
    def __init__(self, ref: Ref, occ=None, res=0.1, ox=0.0, oy=0.0, pgm: bytes | None = None, threshold=250):
        self.ref = ref
        h = _vp()
        if pgm is not None:
            buf = np.frombuffer(pgm, dtype=np.uint8).copy()
            ref.check(ref.lib.ref_map_load(_u8(buf), len(buf), threshold, res, ox, oy, C.byref(h)), "load_map")
        else:
            o = np.ascontiguousarray(occ, dtype=np.uint8)
            ref.check(ref.lib.ref_map_new(o.shape[1], o.shape[0], res, _u8(o), ox, oy, C.byref(h)), "map")
        self.h = h
        self.res, self.ox, self.oy = res, ox, oy
        w, hh, fc = C.c_int(), C.c_int(), C.c_int()
        ref.lib.ref_map_dims(h, C.byref(w), C.byref(hh), C.byref(fc))
        self.w, self.height, self.free_count = w.value, hh.value, fc.value
        self._field = None

    @property
    def cells(self):
        out = np.empty((self.height, self.w), np.uint8)
        self.ref.lib.ref_map_cells(self.h, _u8(out))
        return out

    def pgm(self) -> bytes:
        cap = self.w * self.height + 64
        buf = np.empty(cap, np.uint8)
        n = C.c_size_t()
        self.ref.check(self.ref.lib.ref_write_pgm(self.h, _u8(buf), cap, C.byref(n)), "write_pgm")
        return buf[: n.value].tobytes()

    @property
    def field(self):
        if self._field is None:
            self._field = self.ref.lib.ref_field_new(self.h)
        return self._field

    def field_values(self):
        out = np.empty((self.height, self.w))
        self.ref.lib.ref_field_values(self.field, _d(out))
        return out

    def __del__(self):
        try:
            if self._field:
                self.ref.lib.ref_field_free(self._field)
            self.ref.lib.ref_map_free(self.h)
        except Exception:
            pass


class RefEngine:
    """Reference tensor + kernels + activation + pool, like the Localizer's
    members (localizer.cpp:7-23): slot 0 main kernels, slot 1 rotation-only."""

    def __init__(self, ref: Ref, rmap: RefMap, channels: int, noise=(0.03, 0.03, 0.012), threads: int = 0,
                 rot_slot: bool = True, tensor: np.ndarray | None = None):
        self.ref, self.map, self.C = ref, rmap, channels
        L = ref.lib
        self.pool = L.ref_pool_new(threads)
        self.threads = L.ref_pool_threads(self.pool)
        dth = 2.0 * np.pi / channels
        self.kern, self.act = [], []
        noises = [noise] + ([(1e-4, 1e-4, noise[2])] if rot_slot else [])
        for n in noises:
            kh = _vp()
            ref.check(L.ref_kernels_new(n[0], n[1], n[2], channels, rmap.res, dth, C.byref(kh)), "build_kernels")
            self.kern.append(kh)
            self.act.append(L.ref_activation_new(rmap.h, kh, channels, self.pool))
        th = _vp()
        if tensor is None:
            ref.check(L.ref_tensor_init_uniform(rmap.h, channels, C.byref(th)), "init_uniform")
        else:
            ref.check(L.ref_tensor_new(rmap.w, rmap.height, channels, rmap.res, rmap.ox, rmap.oy, C.byref(th)),
                      "tensor")
        self.t = th
        if tensor is not None:
            self.set(tensor, 0.0)
        self.scratch = L.ref_scratch_new()

    def kernels(self, slot=0) -> Kernels:
        L = self.ref.lib
        kh = self.kern[slot]
        v = [C.c_int() for _ in range(6)]
        L.ref_kernels_info(kh, *[C.byref(x) for x in v])
        r, sep, na, ds, da, ns = (x.value for x in v)
        kw = 2 * r + 1
        sepv = np.zeros(kw if sep else 1)
        spatial = np.zeros(ns * kw * kw)
        off = np.zeros(na, np.int32)
        wt = np.zeros(na)
        L.ref_kernels_get(kh, _d(sepv), _d(spatial), _i(off), _d(wt))
        return Kernels(r, sep, sepv[: kw if sep else 0], spatial, off, wt, ds, da)

    def activation(self, slot=0):
        n = self.C * self.map.w * self.map.height
        vals = np.empty(n)
        inv = np.empty(n)
        self.ref.lib.ref_activation_get(self.act[slot], _d(vals), _d(inv))
        shp = (self.C, self.map.height, self.map.w)
        return vals.reshape(shp), inv.reshape(shp)

    def set(self, B, theta_t):
        B = np.ascontiguousarray(B, dtype=np.float64)
        self.ref.lib.ref_tensor_set(self.t, _d(B), theta_t)

    def get(self):
        out = np.empty((self.C, self.map.height, self.map.w))
        th = C.c_double()
        self.ref.lib.ref_tensor_get(self.t, _d(out), C.byref(th))
        return out, th.value

    def step(self, u, v, w, slot=0):
        return self.ref.lib.ref_step(self.t, u, v, w, self.map.h, self.kern[slot], self.act[slot], self.pool,
                                     self.scratch)

    def apply_motion(self, u, v, w):
        self.ref.lib.ref_apply_motion(self.t, u, v, w)

    def belief_map(self):
        out = np.empty((self.map.height, self.map.w))
        self.ref.lib.ref_belief_map(self.t, _d(out))
        return out

    def argmax(self):
        ijk = np.zeros(3, np.int32)
        pose = np.zeros(3)
        conf = C.c_double()
        self.ref.check(self.ref.lib.ref_argmax(self.t, _i(ijk), _d(pose), C.byref(conf)), "argmax")
        return tuple(int(x) for x in ijk), tuple(float(x) for x in pose), conf.value

    def observation_update(self, cells, angles, ranges, max_range, sigma_hit=0.2, weight_floor=0.05, beam_stride=4):
        cells = np.ascontiguousarray(cells, dtype=np.int32).reshape(-1)
        a = np.ascontiguousarray(angles, dtype=np.float64)
        r = np.ascontiguousarray(ranges, dtype=np.float64)
        return self.ref.lib.ref_observation_update(self.t, _i(cells), len(cells) // 2, _d(a), _d(r), len(a),
                                                   max_range, self.map.h, self.map.field, sigma_hit, weight_floor,
                                                   beam_stride, self.pool)

    def __del__(self):
        try:
            L = self.ref.lib
            L.ref_scratch_free(self.scratch)
            L.ref_tensor_free(self.t)
            for a in self.act:
                L.ref_activation_free(a)
            for k in self.kern:
                L.ref_kernels_free(k)
            L.ref_pool_free(self.pool)
        except Exception:
            pass


def ref_map_difficulty(ref: Ref, rmap: "RefMap", cfg: dict, threads: int = 0) -> float:
    """The reference's map_difficulty (evaluation.cpp:25-72) on its own pool."""
    pool = ref.lib.ref_pool_new(threads)
    try:
        out = C.c_double()
        sh, fl, bs = cfg["lik"]
        rc = ref.lib.ref_map_difficulty(rmap.h, rmap.field, cfg["thr"], cfg["beams"], cfg["fov"], cfg["max_range"],
                                        cfg["stride"], cfg["bins"], sh, fl, bs, pool, C.byref(out))
        if rc != 0:
            raise RuntimeError(ref.lib.ref_last_error().decode())
        return out.value
    finally:
        ref.lib.ref_pool_free(pool)


def ref_world_cells(ref: Ref, which: int):
    """Occupancy of one of the reference's fixed worlds (worlds.cpp)."""
    h = _vp()
    if ref.lib.ref_world(which, C.byref(h)) != 0:
        raise RuntimeError(ref.lib.ref_last_error().decode())
    try:
        w, hh, fc = C.c_int(), C.c_int(), C.c_int()
        ref.lib.ref_map_dims(h, C.byref(w), C.byref(hh), C.byref(fc))
        out = np.empty((hh.value, w.value), np.uint8)
        ref.lib.ref_map_cells(h, _u8(out))
        return out
    finally:
        ref.lib.ref_map_free(h)


def ref_write_snapshot(ref: Ref, values, theta_t: float, path: str, cell=0.1):
    """The reference's write_belief_snapshot of a (C, H, W) FP64 array."""
    c, h, w = values.shape
    t = _vp()
    assert ref.lib.ref_tensor_new(w, h, c, cell, 0.0, 0.0, C.byref(t)) == 0
    try:
        v = np.ascontiguousarray(values, dtype=np.float64)
        ref.lib.ref_tensor_set(t, v.ctypes.data_as(_dp), theta_t)
        if ref.lib.ref_write_snapshot(t, os.fsencode(path)) != 0:
            raise RuntimeError(ref.lib.ref_last_error().decode())
    finally:
        ref.lib.ref_tensor_free(t)


def ref_read_snapshot(ref: Ref, path: str, cell=0.1):
    """The reference's read_belief_snapshot -> ((C, H, W) FP64 values, theta_t)."""
    t = _vp()
    if ref.lib.ref_read_snapshot(os.fsencode(path), cell, 0.0, 0.0, C.byref(t)) != 0:
        raise RuntimeError(ref.lib.ref_last_error().decode())
    try:
        w, h, c = C.c_int(), C.c_int(), C.c_int()
        ref.lib.ref_tensor_dims(t, C.byref(w), C.byref(h), C.byref(c))
        out = np.empty((c.value, h.value, w.value))
        th = C.c_double()
        ref.lib.ref_tensor_get(t, out.ctypes.data_as(_dp), C.byref(th))
        return out, th.value
    finally:
        ref.lib.ref_tensor_free(t)


def ref_dither(ref: Ref, bm, budget):
    h, w = bm.shape
    bm = np.ascontiguousarray(bm, dtype=np.float64)
    cap = max(1, min(h * w, 4 * budget + 16))
    cells = np.zeros(2 * cap, np.int32)
    n = C.c_int()
    mass = C.c_double()
    ref.check(ref.lib.ref_dither(_d(bm), w, h, budget, _i(cells), cap, C.byref(n), C.byref(mass)), "dither")
    return cells[: 2 * n.value].reshape(-1, 2).copy(), mass.value


def ref_gen_trace(ref: Ref, rmap: RefMap, channels: int, start, seed: int, max_steps: int, dt=0.05,
                  scan_period=0.0, beams=24, fov=2 * np.pi, max_range=8.0):
    """Record the step()/observe() calls a reference Localizer would issue
    along a simulated random walk (see ref_shim.cpp:ref_gen_trace)."""
    max_events = 4 * max_steps + 64
    max_scans = max_events if scan_period > 0 else 1
    ev = np.zeros(6 * max_events)
    sc = np.zeros(2 * beams * max_scans)
    ne, ns = C.c_int(), C.c_int()
    ref.check(ref.lib.ref_gen_trace(rmap.h, channels, start[0], start[1], start[2], seed, max_steps, dt, scan_period,
                                    beams, fov, max_range, _d(ev), max_events, C.byref(ne), _d(sc), max_scans,
                                    C.byref(ns)), "gen_trace")
    return ev[: 6 * ne.value].reshape(-1, 6).copy(), sc[: 2 * beams * ns.value].reshape(-1, 2, beams).copy()
