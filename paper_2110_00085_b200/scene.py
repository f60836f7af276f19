"""Scene / ParamSet value types — Python mirror of pathrec::Scene (scene.hpp:26-107) and
pathrec::ParamSet (transport.hpp:63-67), convertible to the C-ABI prc_scene_desc.

Also holds the scene builders used by tests and bench: the reference's own test
fixtures (tests/helpers.hpp:9-118) and the synthetic workloads of SURVEY.md §8(d)
(the cloud of acceptance.cpp:402-426 at 32^3 / 128^3, two species, reflectometry).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import abi


def _v(t) -> abi.Vec3:
    return abi.Vec3(float(t[0]), float(t[1]), float(t[2]))


@dataclass
class Grid:
    dims: tuple = (1, 1, 1)
    origin: tuple = (0.0, 0.0, 0.0)
    voxel_size: tuple = (1.0, 1.0, 1.0)

    @property
    def voxel_count(self) -> int:
        return int(self.dims[0]) * int(self.dims[1]) * int(self.dims[2])

    def voxel_centers(self) -> np.ndarray:
        """Voxel centres in flat (x-fastest) order (grid.hpp:57-63)."""
        nx, ny, nz = self.dims
        iz, iy, ix = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
        c = np.stack([self.origin[0] + (ix + 0.5) * self.voxel_size[0],
                      self.origin[1] + (iy + 0.5) * self.voxel_size[1],
                      self.origin[2] + (iz + 0.5) * self.voxel_size[2]], axis=-1)
        return c.reshape(-1, 3)


@dataclass
class Species:
    extinction: np.ndarray
    albedo: float = 1.0
    phase: str = "rayleigh"  # "hg" | "rayleigh"
    g: float = 0.0
    unknown: bool = False


@dataclass
class Surface:
    kind: str = "sphere"  # "sphere" | "face"
    center: tuple = (0.0, 0.0, 0.0)
    radius: float = 1.0
    axis: int = 2
    coord: float = 0.0
    lo: tuple = (0.0, 0.0)
    hi: tuple = (1.0, 1.0)
    normal_sign: float = 1.0
    brdf: str = "diffuse"  # "diffuse" | "phong"
    albedo: float = 1.0
    kappa_s: float = 0.0
    gamma: float = 0.0
    target: bool = False


@dataclass
class Light:
    kind: str = "point"  # "sun" | "point"
    position: tuple = (0.0, 0.0, 0.0)
    direction: tuple = (0.0, 0.0, -1.0)
    radiance: float = 1.0


@dataclass
class Detector:
    position: tuple
    direction: tuple
    up: tuple = (0.0, 0.0, 1.0)
    rows: int = 1
    cols: int = 1
    fov: float = 1.0


@dataclass
class Scene:
    bounds_min: tuple = (0.0, 0.0, 0.0)
    bounds_max: tuple = (1.0, 1.0, 1.0)
    grid: Grid = field(default_factory=Grid)
    species: List[Species] = field(default_factory=list)
    surfaces: List[Surface] = field(default_factory=list)
    light: Light = field(default_factory=Light)
    detectors: List[Detector] = field(default_factory=list)
    unit: int = 0  # LengthUnit tag (0 m, 1 km): informational, carried into VGRD checkpoints

    @property
    def voxel_count(self) -> int:
        return self.grid.voxel_count if self.species else 0

    @property
    def pixel_count(self) -> int:
        return sum(d.rows * d.cols for d in self.detectors)

    def image_offsets(self) -> List[int]:
        off = [0]
        for d in self.detectors:
            off.append(off[-1] + d.rows * d.cols)
        return off

    def split_images(self, flat: np.ndarray) -> List[np.ndarray]:
        off = self.image_offsets()
        return [flat[off[k]:off[k + 1]].reshape(d.rows, d.cols) for k, d in enumerate(self.detectors)]

    def unknown_species(self) -> int:
        for j, s in enumerate(self.species):
            if s.unknown:
                return j
        return -1

    def target_surface(self) -> int:
        for k, s in enumerate(self.surfaces):
            if s.target:
                return k
        return -1

    def desc(self) -> "SceneDescHolder":
        return SceneDescHolder(self)


class SceneDescHolder:
    """Owns the ctypes arrays backing one prc_scene_desc."""

    def __init__(self, s: Scene):
        self.keep = []
        d = abi.SceneDesc()
        d.bounds_min = _v(s.bounds_min)
        d.bounds_max = _v(s.bounds_max)
        for a in range(3):
            d.dims[a] = int(s.grid.dims[a])
        d.grid_origin = _v(s.grid.origin)
        d.voxel_size = _v(s.grid.voxel_size)
        d.n_species = len(s.species)
        if s.species:
            arr = (abi.SpeciesDesc * len(s.species))()
            for j, sp in enumerate(s.species):
                ext = np.ascontiguousarray(sp.extinction, dtype=np.float64)
                assert ext.size == s.grid.voxel_count, "species extinction size != voxel count"
                self.keep.append(ext)
                arr[j].extinction = ext.ctypes.data_as(abi.c_double_p)
                arr[j].albedo = sp.albedo
                arr[j].phase_kind = abi.PRC_PHASE_RAYLEIGH if sp.phase == "rayleigh" else abi.PRC_PHASE_HG
                arr[j].g = sp.g
                arr[j].unknown = 1 if sp.unknown else 0
            self.keep.append(arr)
            d.species = arr
        d.n_surfaces = len(s.surfaces)
        if s.surfaces:
            arr = (abi.SurfaceDesc * len(s.surfaces))()
            for k, sf in enumerate(s.surfaces):
                a = arr[k]
                a.kind = abi.PRC_SURF_FACE if sf.kind == "face" else abi.PRC_SURF_SPHERE
                a.center = _v(sf.center)
                a.radius = sf.radius
                a.axis = sf.axis
                a.coord = sf.coord
                a.lo[0], a.lo[1] = sf.lo
                a.hi[0], a.hi[1] = sf.hi
                a.normal_sign = sf.normal_sign
                a.brdf_kind = abi.PRC_BRDF_PHONG if sf.brdf == "phong" else abi.PRC_BRDF_DIFFUSE
                a.albedo = sf.albedo
                a.kappa_s = sf.kappa_s
                a.gamma = sf.gamma
                a.target = 1 if sf.target else 0
            self.keep.append(arr)
            d.surfaces = arr
        d.light.kind = abi.PRC_LIGHT_SUN if s.light.kind == "sun" else abi.PRC_LIGHT_POINT
        d.light.position = _v(s.light.position)
        d.light.direction = _v(s.light.direction)
        d.light.radiance = s.light.radiance
        d.n_detectors = len(s.detectors)
        arr = (abi.DetectorDesc * max(1, len(s.detectors)))()
        for k, dt in enumerate(s.detectors):
            arr[k].position = _v(dt.position)
            arr[k].direction = _v(dt.direction)
            arr[k].up = _v(dt.up)
            arr[k].rows = dt.rows
            arr[k].cols = dt.cols
            arr[k].fov = dt.fov
        self.keep.append(arr)
        d.detectors = arr
        self.desc = d

    @property
    def ptr(self):
        return C.byref(self.desc)


@dataclass
class ParamSet:
    """pathrec::ParamSet (transport.hpp:63-67) + optional per-species overrides."""
    beta: Optional[np.ndarray] = None
    kappa_s: float = 0.0
    gamma: float = 0.0
    species_beta: Optional[List[Optional[np.ndarray]]] = None

    def holder(self) -> "ParamsHolder":
        return ParamsHolder(self)


class ParamsHolder:
    def __init__(self, p: Optional[ParamSet]):
        self.keep = []
        self.p = None
        if p is None:
            return
        c = abi.Params()
        if p.beta is not None:
            b = np.ascontiguousarray(p.beta, dtype=np.float64)
            self.keep.append(b)
            c.beta = b.ctypes.data_as(abi.c_double_p)
            c.n_beta = b.size
        c.kappa_s = p.kappa_s
        c.gamma = p.gamma
        if p.species_beta is not None:
            arr = (abi.c_double_p * len(p.species_beta))()
            for j, sb in enumerate(p.species_beta):
                if sb is not None:
                    a = np.ascontiguousarray(sb, dtype=np.float64)
                    self.keep.append(a)
                    arr[j] = a.ctypes.data_as(abi.c_double_p)
            self.keep.append(arr)
            c.species_beta = arr
        self.p = c

    @property
    def ptr(self):
        return C.byref(self.p) if self.p is not None else None


def params_from_scene(s: Scene) -> ParamSet:
    """params_from_scene (transport.cpp:119-128)."""
    p = ParamSet()
    u = s.unknown_species()
    if u >= 0:
        p.beta = np.array(s.species[u].extinction, dtype=np.float64)
    t = s.target_surface()
    if t >= 0 and s.surfaces[t].brdf == "phong":
        p.kappa_s = s.surfaces[t].kappa_s
        p.gamma = s.surfaces[t].gamma
    return p


# ----------------------------------------------------------------------------------
# Fixtures of the reference test-suite (tests/helpers.hpp:9-118)
# ----------------------------------------------------------------------------------

def cube_grid(n: int, side: float = 1.0) -> Grid:
    vs = side / n
    return Grid((n, n, n), (0.0, 0.0, 0.0), (vs, vs, vs))


def top_detector(rows: int, cols: int, fov: float = 0.6) -> Detector:
    return Detector((0.5, 0.5, 3.0), (0.0, 0.0, -1.0), (0.0, 1.0, 0.0), rows, cols, fov)


def homogeneous_cube(beta: float, albedo: float, phase: str = "rayleigh", g: float = 0.0,
                     grid_n: int = 4, rows: int = 8, cols: int = 8) -> Scene:
    g_ = cube_grid(grid_n)
    return Scene(grid=g_, species=[Species(np.full(g_.voxel_count, beta), albedo, phase, g)],
                 light=Light("point", (0.5, 0.5, 0.5), (0, 0, -1), 1.0),
                 detectors=[top_detector(rows, cols)])


def two_species_cube(cloud_beta: np.ndarray, grid_n: int, air_beta: float = 0.04,
                     rows: int = 8, cols: int = 8) -> Scene:
    g_ = cube_grid(grid_n)
    return Scene(grid=g_,
                 species=[Species(np.asarray(cloud_beta, dtype=np.float64), 0.99, "hg", 0.5, True),
                          Species(np.full(g_.voxel_count, air_beta), 0.912, "rayleigh", 0.0, False)],
                 light=Light("point", (0.5, 0.5, 0.5), (0, 0, -1), 1.0),
                 detectors=[top_detector(rows, cols)])


def phong_box(kappa_s: float, gamma: float, rows: int = 16, cols: int = 16,
              wall_albedo: float = 0.8) -> Scene:
    def wall(axis, coord, sign):
        return Surface("face", axis=axis, coord=coord, lo=(0.0, 0.0), hi=(1.0, 1.0),
                       normal_sign=sign, brdf="diffuse", albedo=wall_albedo)
    floor = wall(2, 0.0, 1.0)
    floor.brdf = "phong"
    floor.kappa_s = kappa_s
    floor.gamma = gamma
    floor.target = True
    d = np.array([-0.2, 0.0, -1.0])
    d = d / math.sqrt(float(d @ d))
    return Scene(surfaces=[floor, wall(0, 0.0, 1.0), wall(0, 1.0, -1.0), wall(1, 0.0, 1.0),
                           wall(1, 1.0, -1.0)],
                 light=Light("point", (0.35, 0.5, 0.75), (0, 0, -1), 1.0),
                 detectors=[Detector((0.65, 0.5, 0.9), tuple(d), (0.0, 1.0, 0.0), rows, cols, 1.1)])


# ----------------------------------------------------------------------------------
# Synthetic workloads of SURVEY.md §8(d)
# ----------------------------------------------------------------------------------

def cloud_field(n: int, peak: float = 20.0, sigma: float = 0.22,
                centre=(0.5, 0.5, 0.5)) -> np.ndarray:
    """beta(v) = peak * exp(-|c_v - centre|^2 / (2 sigma^2)) (shape of acceptance.cpp:402-406)."""
    c = cube_grid(n).voxel_centers() - np.asarray(centre)
    return peak * np.exp(-(c * c).sum(axis=1) / (2.0 * sigma * sigma))


def ring_cameras(rows: int, cols: int, fov: float = 0.9, n_ring: int = 8) -> List[Detector]:
    """Zenith camera plus a ring of radius 1.4 at z = 1.6, looking at the centre
    (acceptance.cpp:411-426)."""
    def cam(pos):
        d = np.array([0.5, 0.5, 0.5]) - np.asarray(pos)
        d = d / math.sqrt(float(d @ d))
        up = (0.0, 0.0, 1.0)
        if abs(d[2]) > 0.99:
            up = (0.0, 1.0, 0.0)
        return Detector(tuple(pos), tuple(d), up, rows, cols, fov)
    dets = [cam((0.5, 0.5, 2.6))]
    for k in range(n_ring):
        a = 2.0 * math.pi * k / n_ring
        dets.append(cam((0.5 + 1.4 * math.cos(a), 0.5 + 1.4 * math.sin(a), 1.6)))
    return dets


def cloud_scene(n: int = 32, rows: int = 64, cols: int = 64, two_species: bool = False,
                n_ring: int = 8, fov: float = 0.9) -> Scene:
    """Config (a)/(b)/(c): unit cube, Gaussian cloud (peak 20, sigma 0.22), albedo 0.99,
    HG g = 0.85, sun at zenith, 9 cameras.  (c) adds a Rayleigh species 2."""
    g_ = cube_grid(n)
    sp = [Species(cloud_field(n), 0.99, "hg", 0.85, True)]
    if two_species:
        c = g_.voxel_centers() - np.array([0.35, 0.6, 0.45])
        b2 = 0.04 + 4.0 * np.exp(-(c * c).sum(axis=1) / (2.0 * 0.15 * 0.15))
        sp.append(Species(b2, 0.912, "rayleigh", 0.0, False))
    return Scene(grid=g_, species=sp, light=Light("sun", (0, 0, 0), (0.0, 0.0, -1.0), 1.0),
                 detectors=ring_cameras(rows, cols, fov, n_ring))


def recycle_point(beta_ref: np.ndarray) -> np.ndarray:
    """beta_t = beta_ref * (1 + 0.01 * (v mod 5))."""
    v = np.arange(beta_ref.size)
    return beta_ref * (1.0 + 0.01 * (v % 5))


def reflectometry_scene(rows: int = 256, cols: int = 256, n_cams: int = 16) -> Scene:
    """Config (d): phong_box geometry (walls albedo 0.3) + a central Phong sphere
    (kappa_s 0.7, gamma 50; the target) + 14 small diffuse spheres, 16 inward cameras."""
    s = phong_box(0.7, 50.0, rows, cols, 0.3)
    # The box floor stays Phong but is no longer the unknown; the central sphere is.
    s.surfaces[0].target = False
    s.surfaces.insert(0, Surface("sphere", center=(0.5, 0.5, 0.25), radius=0.18, brdf="phong",
                                 kappa_s=0.7, gamma=50.0, target=True))
    rng = np.random.default_rng(2110)
    for k in range(14):
        c = (0.12 + 0.76 * rng.random(), 0.12 + 0.76 * rng.random(), 0.05 + 0.3 * rng.random())
        s.surfaces.append(Surface("sphere", center=c, radius=0.04, brdf="diffuse", albedo=0.6))
    s.light = Light("point", (0.5, 0.5, 0.8), (0, 0, -1), 1.0)
    dets = []
    for k in range(n_cams):
        a = 2.0 * math.pi * k / n_cams
        pos = np.array([0.5 + 0.3 * math.cos(a), 0.5 + 0.3 * math.sin(a), 0.92])
        d = np.array([0.5, 0.5, 0.2]) - pos
        d = d / math.sqrt(float(d @ d))
        dets.append(Detector(tuple(pos), tuple(d), (0.0, 0.0, 1.0), rows, cols, 1.0))
    s.detectors = dets
    return s
