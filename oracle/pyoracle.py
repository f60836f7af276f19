"""TEST INFRASTRUCTURE ONLY — Python handles on the two CPU checkers:

* ``Port``: oracle/_build/liboracle.so, our plain-C restatement (pathrec_oracle.c),
  built on demand with gcc (present on every box).
* ``Reference``: oracle/_ref/libpathrec_ref.so, the unmodified reference compiled in
  place from /root/reference (only buildable where the reference tree exists; the .so
  travels to the GPU box with the snapshot).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this module.  The product never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional

import numpy as np

from paper_2110_00085_b200 import abi
from paper_2110_00085_b200.scene import ParamsHolder, ParamSet, Scene

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libpathrec_ref.so")

_u32p = C.POINTER(C.c_uint32)
_u64p = C.POINTER(C.c_uint64)
_i32p = C.POINTER(C.c_int32)
_dp = abi.c_double_p


def _ptr(a: Optional[np.ndarray], t):
    return None if a is None else a.ctypes.data_as(t)


def build_port() -> str:
    src = os.path.join(HERE, "pathrec_oracle.c")
    if not os.path.exists(PORT_SO) or os.path.getmtime(PORT_SO) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", HERE, "port"])
    return PORT_SO


def build_ref() -> Optional[str]:
    if os.path.isdir("/root/reference/proj/src"):
        subprocess.check_call(["make", "-s", "-C", HERE, "ref"])
    return REF_SO if os.path.exists(REF_SO) else None


class _Store:
    """Handle on an oracle path store (AoS records as in the reference)."""

    def __init__(self, lib, ptr):
        self.lib, self.ptr = lib, ptr

    def __del__(self):
        if getattr(self, "ptr", None):
            self.lib.orc_store_free(self.ptr)
            self.ptr = None

    def __len__(self):
        return int(self.lib.orc_store_count(self.ptr))

    def streams(self) -> np.ndarray:
        out = np.zeros(len(self), np.uint64)
        self.lib.orc_store_streams(self.ptr, _ptr(out, _u64p))
        return out

    def sizes(self) -> np.ndarray:
        out = np.zeros(len(self), np.uint32)
        self.lib.orc_store_sizes(self.ptr, _ptr(out, _u32p))
        return out

    def stats(self) -> dict:
        o = np.zeros(7)
        self.lib.orc_store_stats(self.ptr, _ptr(o, _dp))
        keys = ["segments", "vertices", "events", "le_spans", "live_path_spans", "path_spans",
                "truncated"]
        return dict(zip(keys, o.tolist()))

    def slice(self, lo: int, hi: int) -> "_Store":
        return _Store(self.lib, self.lib.orc_store_slice(self.ptr, lo, hi))

    def sort_by_size(self):
        if self.lib.orc_sort_by_size(self.ptr):
            raise ValueError(self.lib.orc_last_error().decode())

    def save(self, path: str):
        if self.lib.orc_save_pstr(self.ptr, path.encode()):
            raise IOError(self.lib.orc_last_error().decode())


class Port:
    """The plain-C restatement oracle."""

    def __init__(self, path: Optional[str] = None):
        self.lib = C.CDLL(path or build_port())
        L = self.lib
        L.orc_last_error.restype = C.c_char_p
        L.orc_store_count.restype = C.c_uint64
        L.orc_store_count.argtypes = [C.c_void_p]
        L.orc_store_free.argtypes = [C.c_void_p]
        L.orc_store_streams.argtypes = [C.c_void_p, _u64p]
        L.orc_store_sizes.argtypes = [C.c_void_p, _u32p]
        L.orc_store_stats.argtypes = [C.c_void_p, _dp]
        L.orc_sort_by_size.argtypes = [C.c_void_p]
        L.orc_save_pstr.argtypes = [C.c_void_p, C.c_char_p]
        L.orc_load_pstr.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
        L.orc_render.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64, C.c_int, C.c_int,
                                 C.c_int, _dp, _u64p, C.POINTER(C.c_void_p)]
        L.orc_evaluate.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, _dp, _dp, _dp, _dp,
                                   _dp, _u64p, _dp]
        L.orc_philox.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, _u32p]
        L.orc_store_slice.restype = C.c_void_p
        L.orc_store_slice.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64]
        L.orc_walk.argtypes = [C.c_void_p, C.c_uint64, _dp, _u32p, _u32p, _dp, C.c_uint64]
        L.orc_pixel_of.argtypes = [C.c_void_p, C.c_int, C.c_uint64, _dp, _i32p]

    def _err(self):
        return self.lib.orc_last_error().decode()

    def philox(self, seed: int, stream: int, n: int) -> np.ndarray:
        out = np.zeros(n, np.uint32)
        self.lib.orc_philox(seed, stream, n, _ptr(out, _u32p))
        return out

    def walk(self, scene: Scene, rays: np.ndarray):
        rays = np.ascontiguousarray(rays, dtype=np.float64).reshape(-1, 7)
        n = rays.shape[0]
        h = scene.desc()
        counts = np.zeros(n, np.uint32)
        self.lib.orc_walk(h.ptr, n, _ptr(rays, _dp), _ptr(counts, _u32p), None, None, 0)
        tot = int(counts.sum())
        vox = np.zeros(max(tot, 1), np.uint32)
        ln = np.zeros(max(tot, 1))
        self.lib.orc_walk(h.ptr, n, _ptr(rays, _dp), _ptr(counts, _u32p), _ptr(vox, _u32p),
                          _ptr(ln, _dp), tot)
        return counts, vox[:tot], ln[:tot]

    def pixel_of(self, scene: Scene, det: int, pts: np.ndarray) -> np.ndarray:
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
        out = np.zeros(pts.shape[0], np.int32)
        h = scene.desc()
        if self.lib.orc_pixel_of(h.ptr, det, pts.shape[0], _ptr(pts, _dp), _ptr(out, _i32p)):
            raise ValueError(self._err())
        return out

    def render(self, scene: Scene, n: int, seed: int, params: Optional[ParamSet] = None,
               max_bounces: int = 500, max_events: int = -1, keep: bool = True):
        h = scene.desc()
        ph = ParamsHolder(params)
        img = np.zeros(scene.pixel_count)
        tr = C.c_uint64(0)
        st = C.c_void_p()
        if self.lib.orc_render(h.ptr, ph.ptr, n, seed, max_bounces, max_events, 1 if keep else 0,
                               _ptr(img, _dp), C.byref(tr), C.byref(st)):
            raise ValueError(self._err())
        return img, int(tr.value), (_Store(self.lib, st.value) if keep else None)

    def load(self, path: str) -> _Store:
        st = C.c_void_p()
        if self.lib.orc_load_pstr(path.encode(), C.byref(st)):
            raise IOError(self._err())
        return _Store(self.lib, st.value)

    def evaluate(self, scene: Scene, store: _Store, params: Optional[ParamSet] = None,
                 flags: int = abi.PRC_EVAL_NORMALIZE, weights: Optional[np.ndarray] = None):
        h = scene.desc()
        ph = ParamsHolder(params)
        img = np.zeros(scene.pixel_count)
        grad = np.zeros(max(scene.voxel_count, 1))
        gk, gg, mc = C.c_double(), C.c_double(), C.c_double()
        cl = C.c_uint64()
        w = None if weights is None else np.ascontiguousarray(weights, dtype=np.float64)
        if self.lib.orc_evaluate(h.ptr, store.ptr, ph.ptr, flags, _ptr(w, _dp), _ptr(img, _dp),
                                 _ptr(grad, _dp), C.byref(gk), C.byref(gg), C.byref(cl),
                                 C.byref(mc)):
            raise ValueError(self._err())
        return dict(images=img, grad=grad[:scene.voxel_count], grad_kappa=gk.value,
                    grad_gamma=gg.value, clamp_events=int(cl.value), mean_correction=mc.value)


class Reference:
    """The unmodified reference library compiled in place (oracle/_ref)."""

    def __init__(self, path: Optional[str] = None):
        path = path or (REF_SO if os.path.exists(REF_SO) else build_ref())
        if not path or not os.path.exists(path):
            raise FileNotFoundError("oracle/_ref/libpathrec_ref.so not built")
        self.lib = C.CDLL(path)
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        L.ref_philox.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, _u32p]
        L.ref_walk.argtypes = [C.c_void_p, C.c_uint64, _dp, _u32p, _u32p, _dp, C.c_uint64]
        L.ref_pixel_of.argtypes = [C.c_void_p, C.c_int, C.c_uint64, _dp, _i32p]
        L.ref_render.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64, C.c_int, C.c_int,
                                 C.c_int, C.c_int, C.c_char_p, _dp, _u64p]
        L.ref_sort_pstr.argtypes = [C.c_char_p, C.c_char_p, _u64p]
        L.ref_evaluate.argtypes = [C.c_void_p, C.c_char_p, C.c_void_p, C.c_int, _dp, C.c_int, _dp,
                                   _dp, _dp, _dp, _u64p, _dp]
        L.ref_time_iteration.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64,
                                         C.c_uint64, C.c_int, C.c_int, C.c_int, _dp]
        L.ref_reconstruct.argtypes = [C.c_void_p, C.c_void_p, _dp, C.c_double, _dp, C.c_int,
                                      C.c_uint64, C.c_uint64, C.c_int, C.c_int, C.c_int, _dp, _dp,
                                      _dp, _dp, _u64p]
        L.ref_space_carve.argtypes = [C.c_void_p, _dp, C.c_double, C.c_double, C.POINTER(C.c_uint8), _dp]
        L.ref_downsample.argtypes = [C.c_int, _i32p, _i32p, _dp, C.c_int, C.c_int, _dp]
        L.ref_metrics.argtypes = [_dp, _dp, C.c_uint64, _dp, _dp]
        L.ref_save_grid.argtypes = [C.c_char_p, _i32p, _dp, _dp, C.c_int, _dp]
        L.ref_save_csv.argtypes = [C.c_char_p, C.c_int, _i32p, _dp, _dp, _dp, _dp, _i32p]
        L.ref_render_json.argtypes = [C.c_char_p, C.c_uint64, C.c_uint64, _dp, C.c_uint64]
        L.ref_save_pfm.argtypes = [C.c_char_p, C.c_int, C.c_int, _dp]
        L.ref_load_pfm.argtypes = [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int), _dp, C.c_uint64]
        L.ref_adam.argtypes = [C.c_uint64, _dp, _dp, C.c_int, C.c_double, C.c_double, C.c_double,
                               C.c_double, C.c_int, _dp, C.c_int, C.c_int, _dp]
        L.ref_loss.argtypes = [C.c_void_p, _dp, _dp, _dp]
        L.ref_reconstruct_schedule.argtypes = [C.c_void_p, C.c_void_p, _dp, C.c_double, C.c_uint64, C.c_int,
                                               _i32p, _u64p, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int,
                                               _dp, _i32p, _u64p, _u64p]
        L.ref_segment_lengths.argtypes = [C.c_void_p, C.c_char_p, _u64p, _u32p, _u32p, _dp]

    def _err(self):
        return self.lib.ref_last_error().decode()

    def philox(self, seed, stream, n):
        out = np.zeros(n, np.uint32)
        self.lib.ref_philox(seed, stream, n, _ptr(out, _u32p))
        return out

    def walk(self, scene: Scene, rays: np.ndarray):
        rays = np.ascontiguousarray(rays, dtype=np.float64).reshape(-1, 7)
        n = rays.shape[0]
        h = scene.desc()
        counts = np.zeros(n, np.uint32)
        self.lib.ref_walk(h.ptr, n, _ptr(rays, _dp), _ptr(counts, _u32p), None, None, 0)
        tot = int(counts.sum())
        vox = np.zeros(max(tot, 1), np.uint32)
        ln = np.zeros(max(tot, 1))
        self.lib.ref_walk(h.ptr, n, _ptr(rays, _dp), _ptr(counts, _u32p), _ptr(vox, _u32p),
                          _ptr(ln, _dp), tot)
        return counts, vox[:tot], ln[:tot]

    def pixel_of(self, scene: Scene, det: int, pts: np.ndarray) -> np.ndarray:
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
        out = np.zeros(pts.shape[0], np.int32)
        h = scene.desc()
        if self.lib.ref_pixel_of(h.ptr, det, pts.shape[0], _ptr(pts, _dp), _ptr(out, _i32p)):
            raise ValueError(self._err())
        return out

    def render(self, scene: Scene, n: int, seed: int, params: Optional[ParamSet] = None,
               max_bounces: int = 500, max_events: int = -1, workers: int = 1,
               pstr_out: Optional[str] = None, sort: bool = False):
        h = scene.desc()
        ph = ParamsHolder(params)
        img = np.zeros(scene.pixel_count)
        tr = C.c_uint64(0)
        if self.lib.ref_render(h.ptr, ph.ptr, n, seed, max_bounces, max_events, workers,
                               1 if sort else 0, pstr_out.encode() if pstr_out else None,
                               _ptr(img, _dp), C.byref(tr)):
            raise ValueError(self._err())
        return img, int(tr.value)

    def sort_pstr(self, path_in: str, n: int, path_out: Optional[str] = None) -> np.ndarray:
        out = np.zeros(n, np.uint64)
        if self.lib.ref_sort_pstr(path_in.encode(), path_out.encode() if path_out else None,
                                  _ptr(out, _u64p)):
            raise ValueError(self._err())
        return out

    def evaluate(self, scene: Scene, pstr: str, params: Optional[ParamSet] = None,
                 flags: int = abi.PRC_EVAL_NORMALIZE, weights: Optional[np.ndarray] = None,
                 workers: int = 1):
        h = scene.desc()
        ph = ParamsHolder(params)
        img = np.zeros(scene.pixel_count)
        grad = np.zeros(max(scene.voxel_count, 1))
        gk, gg, mc = C.c_double(), C.c_double(), C.c_double()
        cl = C.c_uint64()
        w = None if weights is None else np.ascontiguousarray(weights, dtype=np.float64)
        if self.lib.ref_evaluate(h.ptr, pstr.encode(), ph.ptr, flags, _ptr(w, _dp), workers,
                                 _ptr(img, _dp), _ptr(grad, _dp), C.byref(gk), C.byref(gg),
                                 C.byref(cl), C.byref(mc)):
            raise ValueError(self._err())
        return dict(images=img, grad=grad[:scene.voxel_count], grad_kappa=gk.value,
                    grad_gamma=gg.value, clamp_events=int(cl.value), mean_correction=mc.value)

    def adam(self, x0, grads, alpha, eta1=0.9, eta2=0.999, eps=1e-8, nonneg=True, step_scale=None,
             phong=False):
        """adam_step (inverse.cpp:41-67) over the rows of grads; the unknowns after each step."""
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
        grads = np.ascontiguousarray(grads, dtype=np.float64).reshape(-1, x0.size)
        ss = None if step_scale is None else np.ascontiguousarray(step_scale, dtype=np.float64)
        out = np.zeros_like(grads)
        if self.lib.ref_adam(x0.size, _ptr(x0, _dp), _ptr(grads, _dp), grads.shape[0], alpha, eta1, eta2, eps,
                             1 if nonneg else 0, _ptr(ss, _dp), 0 if ss is None else ss.size, 1 if phong else 0,
                             _ptr(out, _dp)):
            raise ValueError(self._err())
        return out

    def loss(self, scene: Scene, F, gt) -> float:
        h = scene.desc()
        F = np.ascontiguousarray(F, dtype=np.float64)
        gt = np.ascontiguousarray(gt, dtype=np.float64)
        out = C.c_double()
        if self.lib.ref_loss(h.ptr, _ptr(F, _dp), _ptr(gt, _dp), C.byref(out)):
            raise ValueError(self._err())
        return out.value

    def reconstruct_schedule(self, scene: Scene, initial: ParamSet, gt, alpha: float, seed: int, stages,
                             recycle_period: int, max_iterations: int, window: int, rel: float,
                             workers: int = 1) -> dict:
        h = scene.desc()
        ph = ParamsHolder(initial)
        gt = np.ascontiguousarray(gt, dtype=np.float64)
        rc = np.array([[r, c] for r, c, _ in stages], np.int32).reshape(-1)
        ns = np.array([n for _, _, n in stages], np.uint64)
        loss = np.zeros(max_iterations)
        stage = np.zeros(max_iterations, np.int32)
        phases, trunc = C.c_uint64(), C.c_uint64()
        if self.lib.ref_reconstruct_schedule(h.ptr, ph.ptr, _ptr(gt, _dp), alpha, seed, len(stages),
                                             _ptr(rc, _i32p), _ptr(ns, _u64p), recycle_period, max_iterations,
                                             window, rel, workers, _ptr(loss, _dp), _ptr(stage, _i32p),
                                             C.byref(phases), C.byref(trunc)):
            raise ValueError(self._err())
        return dict(loss=loss, stage=stage, sampling_phases=int(phases.value), truncated_paths=int(trunc.value))

    def segment_lengths(self, scene: Scene, pstr: str):
        """segment_lengths (pathstore.cpp:296-313) of every record: (counts per segment, voxels,
        lengths), records in file order, segments b = 1..B."""
        h = scene.desc()
        sz = np.zeros(2, np.uint64)
        if self.lib.ref_segment_lengths(h.ptr, pstr.encode(), _ptr(sz, _u64p), None, None, None):
            raise ValueError(self._err())
        counts = np.zeros(max(int(sz[0]), 1), np.uint32)
        vox = np.zeros(max(int(sz[1]), 1), np.uint32)
        ln = np.zeros(max(int(sz[1]), 1))
        if self.lib.ref_segment_lengths(h.ptr, pstr.encode(), _ptr(sz, _u64p), _ptr(counts, _u32p),
                                        _ptr(vox, _u32p), _ptr(ln, _dp)):
            raise ValueError(self._err())
        return counts[:int(sz[0])], vox[:int(sz[1])], ln[:int(sz[1])]

    def time_iteration(self, scene: Scene, ref: Optional[ParamSet], t: ParamSet, n: int, seed: int,
                       workers: int, reps: int = 1, warmup: int = 0) -> dict:
        h = scene.desc()
        pr, pt = ParamsHolder(ref), ParamsHolder(t)
        st = np.zeros(9)
        if self.lib.ref_time_iteration(h.ptr, pr.ptr, pt.ptr, n, seed, workers, warmup, reps,
                                       _ptr(st, _dp)):
            raise ValueError(self._err())
        keys = ["segments", "trace_s", "sort_s", "forward_s", "grad_s", "events", "le_spans",
                "live_path_spans", "vertices"]
        return dict(zip(keys, st.tolist()))

    def reconstruct(self, scene: Scene, initial: ParamSet, gt: np.ndarray, alpha: float,
                    seed: int, n_paths: int, recycle_period: int, max_iterations: int,
                    step_scale=None, workers: int = 1):
        h = scene.desc()
        ph = ParamsHolder(initial)
        gt = np.ascontiguousarray(gt, dtype=np.float64)
        ss = None if step_scale is None else np.ascontiguousarray(step_scale, dtype=np.float64)
        loss = np.zeros(max_iterations)
        beta = np.zeros(max(scene.voxel_count, 1))
        k, g = C.c_double(), C.c_double()
        ph_ = C.c_uint64()
        if self.lib.ref_reconstruct(h.ptr, ph.ptr, _ptr(gt, _dp), alpha, _ptr(ss, _dp),
                                    0 if ss is None else ss.size, seed, n_paths, recycle_period,
                                    max_iterations, workers, _ptr(loss, _dp), _ptr(beta, _dp),
                                    C.byref(k), C.byref(g), C.byref(ph_)):
            raise ValueError(self._err())
        return dict(loss=loss, beta=beta[:scene.voxel_count], kappa_s=k.value, gamma=g.value,
                    sampling_phases=int(ph_.value))

    # -------------------------------------------------- the driver around the loop (§8(f) 1)
    def space_carve(self, scene: Scene, gt: np.ndarray, thr: float, fill: float):
        h = scene.desc()
        gt = np.ascontiguousarray(gt, dtype=np.float64)
        V = scene.voxel_count
        mask = np.zeros(max(V, 1), np.uint8)
        beta = np.zeros(max(V, 1))
        if self.lib.ref_space_carve(h.ptr, _ptr(gt, _dp), thr, fill, mask.ctypes.data_as(C.POINTER(C.c_uint8)),
                                    _ptr(beta, _dp)):
            raise ValueError(self._err())
        return mask[:V], beta[:V]

    def downsample(self, images, ro: int, co: int):
        rows = np.array([im.shape[0] for im in images], np.int32)
        cols = np.array([im.shape[1] for im in images], np.int32)
        flat = np.ascontiguousarray(np.concatenate([np.asarray(im, np.float64).reshape(-1) for im in images]))
        out = np.zeros(len(images) * ro * co)
        if self.lib.ref_downsample(len(images), _ptr(rows, _i32p), _ptr(cols, _i32p), _ptr(flat, _dp), ro, co,
                                   _ptr(out, _dp)):
            raise ValueError(self._err())
        return [out[k * ro * co:(k + 1) * ro * co].reshape(ro, co) for k in range(len(images))]

    def metrics(self, e, t):
        e = np.ascontiguousarray(e, dtype=np.float64)
        t = np.ascontiguousarray(t, dtype=np.float64)
        a, b = C.c_double(), C.c_double()
        if self.lib.ref_metrics(_ptr(e, _dp), _ptr(t, _dp), t.size, C.byref(a), C.byref(b)):
            raise ValueError(self._err())
        return a.value, b.value

    def save_grid(self, path: str, dims, origin, vs, values, unit: int = 0):
        d = np.array(dims, np.int32)
        o = np.array(origin, np.float64)
        v = np.array(vs, np.float64)
        x = np.ascontiguousarray(values, dtype=np.float64)
        if self.lib.ref_save_grid(path.encode(), _ptr(d, _i32p), _ptr(o, _dp), _ptr(v, _dp), unit, _ptr(x, _dp)):
            raise ValueError(self._err())

    def save_csv(self, path: str, history):
        n = len(history)
        it = np.ascontiguousarray(history["iter"], np.int32)
        st = np.ascontiguousarray(history["stage"], np.int32)
        cols = [np.ascontiguousarray(history[k], np.float64) for k in ("time_s", "loss", "eps", "delta")]
        if self.lib.ref_save_csv(path.encode(), n, _ptr(it, _i32p), *[_ptr(c, _dp) for c in cols], _ptr(st, _i32p)):
            raise ValueError(self._err())

    def render_json(self, path: str, n: int, seed: int, n_pix: int) -> np.ndarray:
        out = np.zeros(n_pix)
        if self.lib.ref_render_json(path.encode(), n, seed, _ptr(out, _dp), n_pix):
            raise ValueError(self._err())
        return out

    def save_pfm(self, path: str, image: np.ndarray):
        im = np.ascontiguousarray(image, dtype=np.float64)
        if self.lib.ref_save_pfm(path.encode(), im.shape[0], im.shape[1], _ptr(im, _dp)):
            raise ValueError(self._err())

    def load_pfm(self, path: str) -> np.ndarray:
        r, c = C.c_int(), C.c_int()
        if self.lib.ref_load_pfm(path.encode(), C.byref(r), C.byref(c), None, 0):
            raise ValueError(self._err())
        out = np.zeros(r.value * c.value)
        if self.lib.ref_load_pfm(path.encode(), C.byref(r), C.byref(c), _ptr(out, _dp), out.size):
            raise ValueError(self._err())
        return out.reshape(r.value, c.value)
