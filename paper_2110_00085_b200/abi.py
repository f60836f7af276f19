"""ctypes mirror of include/pathrec_gpu.h (the C-ABI boundary).

Struct layouts here must match the header field for field; tests/test_abi.py checks the
sizes against a C compile of the header.
"""
import ctypes as C

PRC_OK, PRC_ERR_CONFIG, PRC_ERR_IO, PRC_ERR_NUMERIC, PRC_ERR_INVALID, PRC_ERR_CUDA = range(6)
PRC_PHASE_HG, PRC_PHASE_RAYLEIGH = 0, 1
PRC_SURF_SPHERE, PRC_SURF_FACE = 0, 1
PRC_BRDF_DIFFUSE, PRC_BRDF_PHONG = 0, 1
PRC_LIGHT_SUN, PRC_LIGHT_POINT = 0, 1
PRC_EVAL_NORMALIZE = 1
PRC_EVAL_WANT_GRAD = 2
PRC_EVAL_LEGACY_SCORE = 4
PRC_EVAL_SELF_NORMALIZE = 8
PRC_EVAL_PER_SPECIES = 16
PRC_EVAL_DETERMINISTIC = 32
PRC_IMPORT_MATERIALIZE = 1

c_double_p = C.POINTER(C.c_double)


class Vec3(C.Structure):
    _fields_ = [("x", C.c_double), ("y", C.c_double), ("z", C.c_double)]


class SpeciesDesc(C.Structure):
    _fields_ = [("extinction", c_double_p), ("albedo", C.c_double), ("phase_kind", C.c_int),
                ("g", C.c_double), ("unknown", C.c_int)]


class SurfaceDesc(C.Structure):
    _fields_ = [("kind", C.c_int), ("center", Vec3), ("radius", C.c_double), ("axis", C.c_int),
                ("coord", C.c_double), ("lo", C.c_double * 2), ("hi", C.c_double * 2),
                ("normal_sign", C.c_double), ("brdf_kind", C.c_int), ("albedo", C.c_double),
                ("kappa_s", C.c_double), ("gamma", C.c_double), ("target", C.c_int)]


class LightDesc(C.Structure):
    _fields_ = [("kind", C.c_int), ("position", Vec3), ("direction", Vec3),
                ("radiance", C.c_double)]


class DetectorDesc(C.Structure):
    _fields_ = [("position", Vec3), ("direction", Vec3), ("up", Vec3), ("rows", C.c_int),
                ("cols", C.c_int), ("fov", C.c_double)]


class SceneDesc(C.Structure):
    _fields_ = [("bounds_min", Vec3), ("bounds_max", Vec3), ("dims", C.c_int * 3),
                ("grid_origin", Vec3), ("voxel_size", Vec3), ("n_species", C.c_int),
                ("species", C.POINTER(SpeciesDesc)), ("n_surfaces", C.c_int),
                ("surfaces", C.POINTER(SurfaceDesc)), ("light", LightDesc),
                ("n_detectors", C.c_int), ("detectors", C.POINTER(DetectorDesc)), ("finalized", C.c_int)]


class Params(C.Structure):
    _fields_ = [("beta", c_double_p), ("n_beta", C.c_uint64), ("kappa_s", C.c_double),
                ("gamma", C.c_double), ("species_beta", C.POINTER(c_double_p))]


class RenderOpts(C.Structure):
    _fields_ = [("n_paths", C.c_uint64), ("seed", C.c_uint64), ("max_bounces", C.c_int),
                ("max_scatter_events", C.c_int)]


class StoreInfo(C.Structure):
    _fields_ = [("n_paths", C.c_uint64), ("n_paths_global", C.c_uint64),
                ("stream_base", C.c_uint64), ("segments", C.c_uint64), ("vertices", C.c_uint64),
                ("interaction_vertices", C.c_uint64), ("truncated", C.c_uint64),
                ("seed", C.c_uint64), ("generation", C.c_uint64), ("sorted", C.c_int),
                ("max_size", C.c_int), ("device_bytes", C.c_uint64), ("materialized", C.c_int)]


class EvalOpts(C.Structure):
    _fields_ = [("flags", C.c_int), ("pixel_weights", c_double_p)]


class EvalResult(C.Structure):
    _fields_ = [("images", c_double_p), ("grad_beta", c_double_p), ("grad_kappa", C.c_double),
                ("grad_gamma", C.c_double), ("clamp_events", C.c_uint64),
                ("mean_correction", C.c_double)]


class AdamConfig(C.Structure):
    _fields_ = [("alpha", C.c_double), ("eta1", C.c_double), ("eta2", C.c_double),
                ("eps_guard", C.c_double), ("project_nonneg", C.c_int),
                ("step_scale", c_double_p), ("n_step_scale", C.c_int)]


class ReconstructOpts(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("n_paths", C.c_uint64), ("max_bounces", C.c_int),
                ("recycle_period", C.c_int), ("max_iterations", C.c_int)]


class Stage(C.Structure):  # prc_gpu_stage (Stage, inverse.hpp:23-26)
    _fields_ = [("rows", C.c_int), ("cols", C.c_int), ("n_paths", C.c_uint64)]


class Schedule(C.Structure):  # prc_gpu_schedule (Schedule + ReconstructOptions, inverse.hpp:28-76)
    _fields_ = [("seed", C.c_uint64), ("max_bounces", C.c_int), ("recycle_period", C.c_int),
                ("max_iterations", C.c_int), ("stages", C.POINTER(Stage)), ("n_stages", C.c_int),
                ("saturation_window", C.c_int), ("saturation_rel_improvement", C.c_double),
                ("checkpoint_every", C.c_int), ("checkpoint_dir", C.c_char_p), ("length_unit", C.c_int),
                ("truth", C.POINTER(Params)), ("on_iteration", C.c_void_p), ("user", C.c_void_p)]


class IterationLog(C.Structure):  # prc_gpu_iteration_log (IterationLog, inverse.hpp:46-53)
    _fields_ = [("iter", C.c_int), ("time_s", C.c_double), ("loss", C.c_double), ("eps", C.c_double),
                ("delta", C.c_double), ("stage", C.c_int)]
