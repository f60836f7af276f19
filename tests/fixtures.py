"""Fixture scenes shared by the golden generator and the tests.

They restate the reference test fixtures (tests/helpers.hpp:9-118) and miniature
versions of the SURVEY.md §8(d) workloads, small enough for the CPU oracles.
"""
import numpy as np

from paper_2110_00085_b200 import scene as S
from paper_2110_00085_b200.scene import ParamSet, params_from_scene


def _tomo2():
    n = 6
    c = S.cube_grid(n).voxel_centers() - 0.5
    cloud = 1.0 + 5.0 * np.exp(-(c * c).sum(1) / (2 * 0.25 ** 2))
    return S.two_species_cube(cloud, n, 0.04, 6, 6)


def _tomo2_flip():
    s = _tomo2()
    s.species[0].unknown = False
    s.species[1].unknown = True
    return s


def _cloud():
    return S.cloud_scene(12, 10, 10)


def _mixed():
    """Medium + surfaces: a homogeneous HG cube with a diffuse floor strip and a
    blocking sphere (visibility tests inside the DDA path)."""
    s = S.homogeneous_cube(2.5, 0.9, "hg", 0.5, grid_n=5, rows=7, cols=7)
    s.species[0].unknown = True
    s.surfaces = [S.Surface("face", axis=2, coord=0.05, lo=(0.1, 0.1), hi=(0.9, 0.9), normal_sign=1.0,
                            brdf="diffuse", albedo=0.7),
                  S.Surface("sphere", center=(0.3, 0.6, 0.7), radius=0.12, brdf="diffuse", albedo=0.5)]
    return s


def _phong():
    return S.phong_box(0.7, 50.0, 8, 8)


FIXTURES = {
    "tomo2": {"scene": _tomo2, "n": 700, "flip_unknown": _tomo2_flip},
    "cloud": {"scene": _cloud, "n": 250},
    "mixed": {"scene": _mixed, "n": 500},
    "phong": {"scene": _phong, "n": 1500, "max_bounces": 40},
}


def perturbed(scene) -> ParamSet:
    p = params_from_scene(scene)
    if p.beta is not None:
        v = np.arange(p.beta.size)
        p.beta = p.beta * (1.0 + 0.02 * (v % 7)) + 0.01 * (v % 3 == 0)
    else:
        p.kappa_s, p.gamma = 0.55, 38.0
    return p


def weight_patterns(scene):
    k = np.arange(scene.pixel_count)
    return {"none": None, "w": 1.0 + (k % 5).astype(np.float64),
            "res": np.sin(0.37 * k + 0.1)}


def walk_rays(scene, n, seed=0):
    """Random rays with origins inside/outside the grid, axis-aligned and diagonal
    directions, exact voxel-boundary origins (the nudge branch of traverse.hpp:83)."""
    rng = np.random.default_rng(seed)
    g = scene.grid
    lo = np.asarray(g.origin)
    hi = lo + np.asarray(g.dims) * np.asarray(g.voxel_size)
    o = rng.uniform(lo - 0.3, hi + 0.3, size=(n, 3))
    d = rng.normal(size=(n, 3))
    q = n // 8
    d[:q] = np.eye(3)[rng.integers(0, 3, q)] * rng.choice([-1.0, 1.0], size=(q, 1))
    d[q:2 * q, rng.integers(0, 3)] = 0.0
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    # origins exactly on voxel faces
    vs = np.asarray(g.voxel_size)
    m = slice(2 * q, 3 * q)
    o[m] = lo + np.floor(rng.uniform(0, 1, size=(q, 3)) * np.asarray(g.dims)) * vs
    maxd = rng.uniform(0.0, 2.0, size=n)
    maxd[:q // 2] = 10.0
    return np.concatenate([o, d, maxd[:, None]], axis=1)


def golden(name):
    import os
    return dict(np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", name + ".npz")))
