"""Python mirror of the reference hot-path API over the C ABI (include/pathrec_gpu.h).

Names and argument meanings follow the reference C++ API so parity tests read like the
reference's own tests:

    render(scene, RenderOptions)            -> transport.hpp:174   (prc_gpu_render)
    sort_by_size(store)                     -> pathstore.hpp:28    (prc_gpu_sort_by_size)
    evaluate_store(scene, store, t, opt)    -> pathstore.hpp:64    (prc_gpu_evaluate)
    recycled_render(scene, store, t)        -> pathstore.hpp:68
    grad_forward(scene, store, t, opt)      -> gradient.hpp:40
    reconstruct(scene, gt, initial, opt)    -> inverse.hpp:294     (prc_gpu_reconstruct)

Errors map to exceptions with the reference's classes: PRC_ERR_CONFIG -> ValueError
(std::invalid_argument / logic_error), PRC_ERR_IO -> IOError, PRC_ERR_NUMERIC ->
FloatingPointError, PRC_ERR_INVALID -> ValueError, PRC_ERR_CUDA -> RuntimeError.
There is no CPU fallback: without the CUDA library or a B200 every call raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import abi
from .scene import ParamSet, ParamsHolder, Scene

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libpathrec_gpu.so")

_lib = None
_u32p = C.POINTER(C.c_uint32)
_u64p = C.POINTER(C.c_uint64)
_i32p = C.POINTER(C.c_int32)
_dp = abi.c_double_p


class PrcError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class PrcConfigError(PrcError, ValueError):
    pass


class PrcIOError(PrcError, IOError):
    pass


class PrcNumericError(PrcError, FloatingPointError):
    pass


class PrcInvalidError(PrcError, ValueError):
    pass


_ERR = {abi.PRC_ERR_CONFIG: PrcConfigError, abi.PRC_ERR_IO: PrcIOError,
        abi.PRC_ERR_NUMERIC: PrcNumericError, abi.PRC_ERR_INVALID: PrcInvalidError}


def load_library(path: Optional[str] = None):
    """Loads libpathrec_gpu.so (building it with nvcc if it is missing or stale)."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("PRC_LIB") or LIB_PATH  # PRC_LIB: A/B experiment builds
    if path == LIB_PATH:
        from .build import build  # in-tree build; the .so normally ships prebuilt
        try:
            build()
        except Exception:
            if not os.path.exists(LIB_PATH):
                raise
    lib = C.CDLL(path)
    lib.prc_gpu_version.restype = C.c_char_p
    lib.prc_gpu_last_error.restype = C.c_char_p
    vp = C.c_void_p
    sig = {
        "prc_gpu_ctx_create": [C.c_int, C.POINTER(vp)],
        "prc_gpu_nccl_unique_id": [vp],
        "prc_gpu_ctx_create_rank": [C.c_int, C.c_int, C.c_int, vp, C.POINTER(vp)],
        "prc_gpu_shard_range": [C.c_uint64, C.c_int, C.c_int, _u64p, _u64p],
        "prc_gpu_ctx_destroy": [vp],
        "prc_gpu_ctx_rank": [vp, C.POINTER(C.c_int), C.POINTER(C.c_int)],
        "prc_gpu_release_cached_memory": [],
        "prc_gpu_ctx_set_option": [vp, C.c_char_p, C.c_int64],
        "prc_gpu_scene_upload": [vp, vp],
        "prc_gpu_scene_voxel_count": [vp, _u64p],
        "prc_gpu_scene_pixel_count": [vp, _u64p],
        "prc_gpu_render": [vp, vp, vp, _dp, _u64p, C.POINTER(vp)],
        "prc_gpu_sort_by_size": [vp, vp],
        "prc_gpu_store_info_get": [vp, C.POINTER(abi.StoreInfo)],
        "prc_gpu_store_streams": [vp, _u64p],
        "prc_gpu_correction_factors": [vp, vp, vp, _dp],
        "prc_gpu_store_sizes": [vp, _u32p],
        "prc_gpu_store_export_pstr": [vp, vp, C.c_char_p],
        "prc_gpu_store_import_pstr": [vp, C.c_char_p, C.POINTER(vp)],
        "prc_gpu_store_import_pstr_ex": [vp, C.c_char_p, C.c_int, C.POINTER(vp)],
        "prc_gpu_store_set_generation": [vp, C.c_uint64],
        "prc_gpu_store_free": [vp],
        "prc_gpu_evaluate": [vp, vp, vp, C.POINTER(abi.EvalOpts), C.POINTER(abi.EvalResult)],
        "prc_gpu_opt_init": [vp, vp, _dp, C.POINTER(abi.AdamConfig)],
        "prc_gpu_opt_step": [vp, vp, _dp],
        "prc_gpu_opt_params": [vp, _dp, _dp, _dp],
        "prc_gpu_opt_adam_step": [vp, _dp, C.c_uint64],
        "prc_gpu_opt_images": [vp, _dp],
        "prc_gpu_reconstruct": [vp, vp, _dp, C.POINTER(abi.AdamConfig),
                                C.POINTER(abi.ReconstructOpts), _dp, _u64p],
        "prc_gpu_reconstruct_schedule": [vp, vp, _dp, C.POINTER(abi.AdamConfig), C.POINTER(abi.Schedule),
                                         C.POINTER(abi.IterationLog), _u64p, _u64p],
        "prc_gpu_space_carve": [vp, _dp, C.c_double, C.c_double, C.POINTER(C.c_uint8), _dp],
        "prc_gpu_metrics": [_dp, _dp, C.c_uint64, _dp, _dp],
        "prc_gpu_downsample_images": [C.c_int, _i32p, _i32p, _dp, C.c_int, C.c_int, _dp],
        "prc_gpu_save_grid": [C.c_char_p, _i32p, C.POINTER(abi.Vec3), C.POINTER(abi.Vec3), C.c_int, _dp],
        "prc_gpu_load_grid": [C.c_char_p, _i32p, C.POINTER(abi.Vec3), C.POINTER(abi.Vec3),
                              C.POINTER(C.c_int), _dp, C.c_uint64],
        "prc_gpu_last_timings": [vp, _dp],
        "prc_gpu_kernel_launches": [vp, _u64p],
        "prc_gpu_debug_checks": [vp, _u32p, C.POINTER(C.c_int)],
        "prc_gpu_timer_start": [vp],
        "prc_gpu_timer_stop": [vp, _dp],
        "prc_gpu_store_stats": [vp, vp, _u64p],
        "prc_gpu_debug_philox": [vp, C.c_uint64, C.c_uint64, C.c_uint64, _u32p],
        "prc_gpu_debug_walk": [vp, C.c_uint64, _dp, _u32p, _u32p, _dp, C.c_uint64],
        "prc_gpu_debug_walk_padded": [vp, C.c_uint64, _dp, _u32p, _u32p, _dp, C.c_uint64],
        "prc_gpu_debug_pixel_of": [vp, C.c_int, C.c_uint64, _dp, _i32p],
    }
    for name, args in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = None if name in ("prc_gpu_ctx_destroy", "prc_gpu_store_free") else C.c_int
    _lib = lib
    return lib


def _check(rc: int):
    if rc != abi.PRC_OK:
        msg = _lib.prc_gpu_last_error().decode()
        raise _ERR.get(rc, PrcError)(rc, msg)


def _ptr(a, t):
    return None if a is None else a.ctypes.data_as(t)


@dataclass
class RenderOptions:
    """transport.hpp:154-161 (workers is meaningless on the GPU and ignored)."""
    n_paths: int = 1
    seed: int = 0
    workers: int = 1
    max_bounces: int = 500
    max_scatter_events: int = -1
    keep_paths: bool = False
    images: bool = True  # False: trace only, no fresh evaluation (images None)


@dataclass
class EvalOptions:
    """pathstore.hpp:41-50 (+ per_species: per-type gradients, config (c))."""
    workers: int = 1
    normalize: bool = True
    want_grad: bool = False
    legacy_score: bool = False
    self_normalize: bool = False
    pixel_weights: Optional[np.ndarray] = None
    per_species: bool = False
    deterministic: bool = False  # bit-reproducible images (PRC_EVAL_DETERMINISTIC)

    def flags(self) -> int:
        f = 0
        if self.normalize:
            f |= abi.PRC_EVAL_NORMALIZE
        if self.want_grad:
            f |= abi.PRC_EVAL_WANT_GRAD
        if self.legacy_score:
            f |= abi.PRC_EVAL_LEGACY_SCORE
        if self.self_normalize:
            f |= abi.PRC_EVAL_SELF_NORMALIZE
        if self.per_species:
            f |= abi.PRC_EVAL_PER_SPECIES
        if self.deterministic:
            f |= abi.PRC_EVAL_DETERMINISTIC
        return f


@dataclass
class EvalResult:
    images: np.ndarray
    grad_beta: Optional[np.ndarray]
    grad_kappa: float
    grad_gamma: float
    clamp_events: int
    mean_correction: float


@dataclass
class RenderResult:
    images: np.ndarray
    truncated_paths: int
    store: Optional["PathStore"]


class PathStore:
    """Handle on a device-resident path store (one shard per rank)."""

    def __init__(self, ctx: "Context", ptr: int):
        self.ctx, self.ptr = ctx, ptr

    def free(self):
        if getattr(self, "ptr", None):
            _lib.prc_gpu_store_free(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    def info(self) -> dict:
        i = abi.StoreInfo()
        _check(_lib.prc_gpu_store_info_get(self.ptr, C.byref(i)))
        return {k: getattr(i, k) for k, _ in abi.StoreInfo._fields_}

    def __len__(self):
        return int(self.info()["n_paths"])

    def streams(self) -> np.ndarray:
        out = np.zeros(len(self), np.uint64)
        _check(_lib.prc_gpu_store_streams(self.ptr, _ptr(out, _u64p)))
        return out

    def sizes(self) -> np.ndarray:
        out = np.zeros(len(self), np.uint32)
        _check(_lib.prc_gpu_store_sizes(self.ptr, _ptr(out, _u32p)))
        return out

    @property
    def sorted_flag(self) -> bool:
        return bool(self.info()["sorted"])

    def save(self, path: str):
        _check(_lib.prc_gpu_store_export_pstr(self.ctx.ptr, self.ptr, path.encode()))

    def set_generation(self, g: int):
        _check(_lib.prc_gpu_store_set_generation(self.ptr, g))


class Context:
    """One process's view of the engine: a CUDA device, a scene and (world > 1) an NCCL
    communicator.  Paths are sharded over ranks by contiguous stream ranges."""

    def __init__(self, device: int = 0, rank: int = 0, world: int = 1,
                 nccl_id: Optional[bytes] = None):
        load_library()
        p = C.c_void_p()
        if world == 1 and nccl_id is None:
            _check(_lib.prc_gpu_ctx_create(device, C.byref(p)))
        else:  # nccl_id None with world > 1: a detached shard (partial sums, no communicator)
            buf = None if nccl_id is None else C.create_string_buffer(bytes(nccl_id), 128)
            _check(_lib.prc_gpu_ctx_create_rank(device, rank, world, buf, C.byref(p)))
        self.ptr = p.value
        self.scene: Optional[Scene] = None
        self.rank, self.world = rank, world

    @staticmethod
    def shard_range(n: int, rank: int, world: int):
        """[lo, hi) of the global stream ids rank `rank` owns (host-only)."""
        load_library()
        lo, hi = C.c_uint64(), C.c_uint64()
        _check(_lib.prc_gpu_shard_range(n, rank, world, C.byref(lo), C.byref(hi)))
        return int(lo.value), int(hi.value)

    @staticmethod
    def nccl_unique_id() -> bytes:
        load_library()
        buf = C.create_string_buffer(128)
        _check(_lib.prc_gpu_nccl_unique_id(buf))
        return buf.raw

    def close(self):
        if getattr(self, "ptr", None):
            _lib.prc_gpu_ctx_destroy(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_option(self, key: str, value: int):
        """'mode': 0 event-major wavefront (default) / 1 fused thread-per-path;
        'packet': LE rays per thread in the gradient kernel (1..4, default 3); 'spread';
        'events': compact event list for scenes without a medium (default 1); see
        include/pathrec_gpu.h for the rest."""
        _check(_lib.prc_gpu_ctx_set_option(self.ptr, key.encode(), int(value)))

    # ------------------------------------------------------------------ scene
    def upload(self, scene: Scene):
        h = scene.desc()
        _check(_lib.prc_gpu_scene_upload(self.ptr, h.ptr))
        self.scene = scene

    def _use(self, scene: Optional[Scene]):
        if scene is not None and scene is not self.scene:
            self.upload(scene)
        if self.scene is None:
            raise PrcInvalidError(abi.PRC_ERR_INVALID, "no scene uploaded")
        return self.scene

    # ------------------------------------------------------------------ K1
    def render(self, scene: Optional[Scene], opt: RenderOptions,
               params: Optional[ParamSet] = None) -> RenderResult:
        s = self._use(scene)
        o = abi.RenderOpts(opt.n_paths, opt.seed, opt.max_bounces, opt.max_scatter_events)
        ph = ParamsHolder(params)
        img = np.zeros(s.pixel_count) if opt.images else None
        tr = C.c_uint64()
        st = C.c_void_p()
        _check(_lib.prc_gpu_render(self.ptr, C.byref(o), ph.ptr, _ptr(img, _dp), C.byref(tr),
                                   C.byref(st) if opt.keep_paths else None))
        return RenderResult(img, int(tr.value), PathStore(self, st.value) if opt.keep_paths else None)

    # ------------------------------------------------------------------ K2
    def sort_by_size(self, store: PathStore):
        _check(_lib.prc_gpu_sort_by_size(self.ptr, store.ptr))

    def load_store(self, path: str, materialized: bool = False) -> PathStore:
        """load_store (pathstore.cpp:455-516).  materialized=True evaluates the file's own
        stored spans (PRC_IMPORT_MATERIALIZE); otherwise spans are recomputed on the device."""
        st = C.c_void_p()
        if materialized:
            _check(_lib.prc_gpu_store_import_pstr_ex(self.ptr, path.encode(), abi.PRC_IMPORT_MATERIALIZE,
                                                     C.byref(st)))
        else:
            _check(_lib.prc_gpu_store_import_pstr(self.ptr, path.encode(), C.byref(st)))
        return PathStore(self, st.value)

    # ------------------------------------------------------------------ K3-K5
    def evaluate_store(self, scene: Optional[Scene], store: PathStore,
                       params: Optional[ParamSet] = None,
                       opt: Optional[EvalOptions] = None) -> EvalResult:
        s = self._use(scene)
        opt = opt or EvalOptions()
        ph = ParamsHolder(params)
        w = None
        if opt.pixel_weights is not None:
            w = np.ascontiguousarray(opt.pixel_weights, dtype=np.float64).reshape(-1)
            if w.size != s.pixel_count:
                raise PrcConfigError(abi.PRC_ERR_CONFIG, "pixel_weights size != pixel count")
        eo = abi.EvalOpts(opt.flags(), _ptr(w, _dp))
        img = np.zeros(s.pixel_count)
        n_out = len(s.species) if opt.per_species else 1
        grad = np.zeros(max(1, n_out * s.voxel_count)) if opt.want_grad else None
        r = abi.EvalResult()
        r.images = _ptr(img, _dp)
        r.grad_beta = _ptr(grad, _dp)
        _check(_lib.prc_gpu_evaluate(self.ptr, store.ptr, ph.ptr, C.byref(eo), C.byref(r)))
        g = None
        if opt.want_grad and s.voxel_count and (s.unknown_species() >= 0 or opt.per_species):
            g = grad[:n_out * s.voxel_count]
            if opt.per_species:
                g = g.reshape(n_out, s.voxel_count)
        return EvalResult(img, g, r.grad_kappa, r.grad_gamma, int(r.clamp_events), r.mean_correction)

    def correction_factors(self, scene: Optional[Scene], store: PathStore,
                           params: Optional[ParamSet] = None) -> np.ndarray:
        """correction_factor (pathstore.cpp:269-294) of every path of the store, in storage
        order (store.streams() gives the stream ids)."""
        self._use(scene)
        ph = ParamsHolder(params)
        out = np.zeros(max(1, len(store)))
        _check(_lib.prc_gpu_correction_factors(self.ptr, store.ptr, ph.ptr, _ptr(out, _dp)))
        return out[:len(store)]

    def recycled_render(self, scene: Optional[Scene], store: PathStore,
                        params: Optional[ParamSet] = None) -> np.ndarray:
        return self.evaluate_store(scene, store, params, EvalOptions()).images

    def grad_forward(self, scene: Optional[Scene], store: PathStore,
                     params: Optional[ParamSet] = None, opt: Optional[EvalOptions] = None) -> dict:
        """gradient.cpp:111-128: {'kind': 'tomography', 'grad': V} or {'kind': 'phong', ...}."""
        opt = EvalOptions(**{**(opt.__dict__ if opt else {}), "want_grad": True})
        r = self.evaluate_store(scene, store, params, opt)
        s = self.scene
        if s.unknown_species() >= 0 or opt.per_species:
            return {"kind": "tomography", "grad": r.grad_beta}
        return {"kind": "phong", "grad": np.array([r.grad_kappa, r.grad_gamma])}

    # ------------------------------------------------------------------ Algorithm 2
    def opt_init(self, initial: Optional[ParamSet], gt: np.ndarray, alpha: float = 1e7,
                 eta1: float = 0.9, eta2: float = 0.999, eps_guard: float = 1e-8,
                 project_nonneg: bool = True, step_scale=None):
        self._adam = _adam(alpha, eta1, eta2, eps_guard, project_nonneg, step_scale)
        self._gt = np.ascontiguousarray(gt, dtype=np.float64).reshape(-1)
        ph = ParamsHolder(initial)
        _check(_lib.prc_gpu_opt_init(self.ptr, ph.ptr, _ptr(self._gt, _dp), C.byref(self._adam[0])))

    def opt_step(self, store: PathStore) -> float:
        loss = C.c_double()
        _check(_lib.prc_gpu_opt_step(self.ptr, store.ptr, C.byref(loss)))
        return loss.value

    def opt_params(self) -> ParamSet:
        s = self.scene
        beta = np.zeros(max(1, s.voxel_count))
        k, g = C.c_double(), C.c_double()
        _check(_lib.prc_gpu_opt_params(self.ptr, _ptr(beta, _dp), C.byref(k), C.byref(g)))
        return ParamSet(beta[:s.voxel_count] if s.unknown_species() >= 0 else None, k.value, g.value)

    def opt_adam_step(self, grad: np.ndarray):
        """adam_step (inverse.cpp:41-67) with a given gradient over the flattened unknowns."""
        g = np.ascontiguousarray(grad, dtype=np.float64).reshape(-1)
        _check(_lib.prc_gpu_opt_adam_step(self.ptr, _ptr(g, _dp), g.size))

    def opt_images(self) -> np.ndarray:
        out = np.zeros(self.scene.pixel_count)
        _check(_lib.prc_gpu_opt_images(self.ptr, _ptr(out, _dp)))
        return out

    def reconstruct(self, scene: Optional[Scene], gt: np.ndarray, initial: Optional[ParamSet],
                    n_paths: int, seed: int = 0, recycle_period: int = 30,
                    max_iterations: int = 100, max_bounces: int = 500, alpha: float = 1e7,
                    step_scale=None) -> dict:
        self._use(scene)
        adam = _adam(alpha, 0.9, 0.999, 1e-8, True, step_scale)
        gt = np.ascontiguousarray(gt, dtype=np.float64).reshape(-1)
        ph = ParamsHolder(initial)
        ro = abi.ReconstructOpts(seed, n_paths, max_bounces, recycle_period, max_iterations)
        loss = np.zeros(max_iterations)
        phases = C.c_uint64()
        _check(_lib.prc_gpu_reconstruct(self.ptr, ph.ptr, _ptr(gt, _dp), C.byref(adam[0]),
                                        C.byref(ro), _ptr(loss, _dp), C.byref(phases)))
        return {"loss": loss, "params": self.opt_params(), "sampling_phases": int(phases.value)}

    def reconstruct_schedule(self, scene: Optional[Scene], gt: np.ndarray, initial: Optional[ParamSet],
                             stages, seed: int = 0, recycle_period: int = 30, max_iterations: int = 100,
                             max_bounces: int = 500, alpha: float = 1e7, step_scale=None,
                             saturation_window: int = 20, saturation_rel_improvement: float = 0.01,
                             checkpoint_every: int = 0, checkpoint_dir: Optional[str] = None,
                             length_unit: int = 0, truth: Optional[ParamSet] = None) -> dict:
        """reconstruct() with a stage schedule (inverse.cpp:154-263).  stages: sequence of
        (rows, cols, n_paths).  Returns the per-iteration history (iter, time_s, loss, eps,
        delta, stage), the final unknowns and the sampling-phase / truncation counters."""
        self._use(scene)
        adam = _adam(alpha, 0.9, 0.999, 1e-8, True, step_scale)
        gt = np.ascontiguousarray(gt, dtype=np.float64).reshape(-1)
        ph = ParamsHolder(initial)
        th = ParamsHolder(truth)
        st = (abi.Stage * len(stages))(*[abi.Stage(int(r), int(c), int(n)) for r, c, n in stages])
        sch = abi.Schedule(seed, max_bounces, recycle_period, max_iterations, st, len(stages),
                           saturation_window, saturation_rel_improvement, checkpoint_every,
                           checkpoint_dir.encode() if checkpoint_dir else None, length_unit,
                           C.pointer(th.p) if truth is not None else None)
        hist = (abi.IterationLog * max(1, max_iterations))()
        phases, trunc = C.c_uint64(), C.c_uint64()
        _check(_lib.prc_gpu_reconstruct_schedule(self.ptr, ph.ptr, _ptr(gt, _dp), C.byref(adam[0]), C.byref(sch),
                                                 hist, C.byref(phases), C.byref(trunc)))
        rows = [(h.iter, h.time_s, h.loss, h.eps, h.delta, h.stage) for h in hist[:max_iterations]]
        return {"history": np.array(rows, dtype=[("iter", "i4"), ("time_s", "f8"), ("loss", "f8"), ("eps", "f8"),
                                                 ("delta", "f8"), ("stage", "i4")]),
                "params": self.opt_params(), "sampling_phases": int(phases.value),
                "truncated_paths": int(trunc.value)}

    def space_carve(self, scene: Optional[Scene], gt: np.ndarray, threshold_fraction: float,
                    fill_extinction: float):
        """space_carve (inverse.cpp:69-101) on the device: (mask, initial beta)."""
        self._use(scene)
        gt = np.ascontiguousarray(gt, dtype=np.float64).reshape(-1)
        V = self.scene.voxel_count
        mask = np.zeros(max(V, 1), np.uint8)
        beta = np.zeros(max(V, 1))
        _check(_lib.prc_gpu_space_carve(self.ptr, _ptr(gt, _dp), threshold_fraction, fill_extinction,
                                        mask.ctypes.data_as(C.POINTER(C.c_uint8)), _ptr(beta, _dp)))
        return mask[:V], beta[:V]

    # ------------------------------------------------------------------ diagnostics
    def last_timings(self) -> dict:
        ms = np.zeros(8)
        _check(_lib.prc_gpu_last_timings(self.ptr, _ptr(ms, _dp)))
        return dict(zip(["prep", "forward", "image_allreduce", "gradient", "grad_allreduce_adam",
                         "total", "forward_per_path", "gradient_per_path"], ms.tolist()))

    def timer_start(self):
        _check(_lib.prc_gpu_timer_start(self.ptr))

    def timer_stop(self) -> float:
        ms = C.c_double()
        _check(_lib.prc_gpu_timer_stop(self.ptr, C.byref(ms)))
        return ms.value

    def store_stats(self, store: "PathStore") -> dict:
        out = np.zeros(4, np.uint64)
        _check(_lib.prc_gpu_store_stats(self.ptr, store.ptr, _ptr(out, _u64p)))
        return dict(zip(["events", "live_path_spans", "le_spans", "path_spans"], out.tolist()))

    def debug_checks(self):
        """(flags, checked_build): the checked build's range-violation word (read and cleared)."""
        f, cb = C.c_uint32(), C.c_int()
        _check(_lib.prc_gpu_debug_checks(self.ptr, C.byref(f), C.byref(cb)))
        return int(f.value), bool(cb.value)

    def kernel_launches(self) -> int:
        n = C.c_uint64()
        _check(_lib.prc_gpu_kernel_launches(self.ptr, C.byref(n)))
        return int(n.value)

    def debug_philox(self, seed: int, stream: int, n: int) -> np.ndarray:
        out = np.zeros(n, np.uint32)
        _check(_lib.prc_gpu_debug_philox(self.ptr, seed, stream, n, _ptr(out, _u32p)))
        return out

    def debug_walk(self, rays: np.ndarray, padded: bool = False):
        """Device DDA spans of n rays (n x 7); padded=True: the guard-free walk over the
        padded layout (voxel ids are padded indices)."""
        fn = _lib.prc_gpu_debug_walk_padded if padded else _lib.prc_gpu_debug_walk
        rays = np.ascontiguousarray(rays, dtype=np.float64).reshape(-1, 7)
        n = rays.shape[0]
        counts = np.zeros(n, np.uint32)
        _check(fn(self.ptr, n, _ptr(rays, _dp), _ptr(counts, _u32p), None, None, 0))
        tot = int(counts.sum())
        vox = np.zeros(max(tot, 1), np.uint32)
        ln = np.zeros(max(tot, 1))
        _check(fn(self.ptr, n, _ptr(rays, _dp), _ptr(counts, _u32p), _ptr(vox, _u32p), _ptr(ln, _dp), tot))
        return counts, vox[:tot], ln[:tot]

    def debug_pixel_of(self, det: int, pts: np.ndarray) -> np.ndarray:
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
        out = np.zeros(pts.shape[0], np.int32)
        _check(_lib.prc_gpu_debug_pixel_of(self.ptr, det, pts.shape[0], _ptr(pts, _dp),
                                           _ptr(out, _i32p)))
        return out


def release_cached_memory():
    """Returns the engine's cached device blocks (freed stores' arrays) to the driver."""
    _check(load_library().prc_gpu_release_cached_memory())


def metrics(estimate: np.ndarray, truth: np.ndarray):
    """metrics (inverse.cpp:103-114): (eps, delta)."""
    load_library()
    e = np.ascontiguousarray(estimate, dtype=np.float64)
    t = np.ascontiguousarray(truth, dtype=np.float64)
    if e.size != t.size:
        raise PrcConfigError(abi.PRC_ERR_CONFIG, "metrics: dimension mismatch")
    eps, delta = C.c_double(), C.c_double()
    _check(_lib.prc_gpu_metrics(_ptr(e, _dp), _ptr(t, _dp), t.size, C.byref(eps), C.byref(delta)))
    return eps.value, delta.value


def downsample_images(images, rows_out: int, cols_out: int):
    """downsample_images (inverse.cpp:116-133): list of 2-D arrays -> list of block sums."""
    load_library()
    rows = np.array([im.shape[0] for im in images], np.int32)
    cols = np.array([im.shape[1] for im in images], np.int32)
    flat = np.ascontiguousarray(np.concatenate([np.asarray(im, np.float64).reshape(-1) for im in images]))
    out = np.zeros(len(images) * rows_out * cols_out)
    _check(_lib.prc_gpu_downsample_images(len(images), _ptr(rows, _i32p), _ptr(cols, _i32p), _ptr(flat, _dp),
                                          rows_out, cols_out, _ptr(out, _dp)))
    return [out[k * rows_out * cols_out:(k + 1) * rows_out * cols_out].reshape(rows_out, cols_out)
            for k in range(len(images))]


def save_grid(path: str, dims, origin, voxel_size, values, length_unit: int = 0):
    """VGRD v1 writer (io.cpp:59-76)."""
    load_library()
    d = np.array(dims, np.int32)
    v = np.ascontiguousarray(values, dtype=np.float64)
    _check(_lib.prc_gpu_save_grid(path.encode(), _ptr(d, _i32p), C.byref(abi.Vec3(*origin)),
                                  C.byref(abi.Vec3(*voxel_size)), length_unit, _ptr(v, _dp)))


def load_grid(path: str) -> dict:
    """VGRD v1 reader (io.cpp:32-57)."""
    load_library()
    d = np.zeros(3, np.int32)
    o, vs, unit = abi.Vec3(), abi.Vec3(), C.c_int()
    _check(_lib.prc_gpu_load_grid(path.encode(), _ptr(d, _i32p), C.byref(o), C.byref(vs), C.byref(unit), None, 0))
    vals = np.zeros(int(np.prod(d)))
    _check(_lib.prc_gpu_load_grid(path.encode(), _ptr(d, _i32p), C.byref(o), C.byref(vs), C.byref(unit),
                                  _ptr(vals, _dp), vals.size))
    return {"dims": tuple(int(x) for x in d), "origin": (o.x, o.y, o.z), "voxel_size": (vs.x, vs.y, vs.z),
            "unit": unit.value, "values": vals}


def _adam(alpha, eta1, eta2, eps, nonneg, step_scale):
    ss = None if step_scale is None else np.ascontiguousarray(step_scale, dtype=np.float64)
    a = abi.AdamConfig(alpha, eta1, eta2, eps, 1 if nonneg else 0, _ptr(ss, _dp),
                       0 if ss is None else ss.size)
    return a, ss


# ---------------------------------------------------------------- reference-style free functions
_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(int(os.environ.get("LOCAL_RANK", "0")))
    return _default_ctx


def render(scene: Scene, opt: RenderOptions, params: Optional[ParamSet] = None) -> RenderResult:
    return default_context().render(scene, opt, params)


def sort_by_size(store: PathStore):
    store.ctx.sort_by_size(store)


def evaluate_store(scene: Scene, store: PathStore, params: Optional[ParamSet] = None,
                   opt: Optional[EvalOptions] = None) -> EvalResult:
    return store.ctx.evaluate_store(scene, store, params, opt)


def recycled_render(scene: Scene, store: PathStore, params: Optional[ParamSet] = None):
    return store.ctx.recycled_render(scene, store, params)


def grad_forward(scene: Scene, store: PathStore, params: Optional[ParamSet] = None,
                 opt: Optional[EvalOptions] = None) -> dict:
    return store.ctx.grad_forward(scene, store, params, opt)
