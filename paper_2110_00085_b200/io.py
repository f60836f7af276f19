"""Host formats around the loop: the reference's JSON scene
(io.cpp:190-278), VGRD grids (io.cpp:32-76, through the C ABI) and PFM images
(io.cpp:94-129).  These are file I/O for end-to-end runs from reference inputs; none of
it is on the device path."""
from __future__ import annotations

import json
import math
import os
import struct
from typing import List

import numpy as np

from . import gpu
from .scene import Detector, Grid, Light, Scene, Species, Surface


def _vec3(j) -> tuple:  # vec3_of, io.cpp:159-162
    if not isinstance(j, list) or len(j) != 3:
        raise ValueError("scene: expected a 3-vector")
    return (float(j[0]), float(j[1]), float(j[2]))


def _normalized(v) -> tuple:  # Vec3::normalized, vec3.hpp:24-25 (same operation order)
    n = math.sqrt((v[0] * v[0] + v[1] * v[1]) + v[2] * v[2])
    return (v[0] / n, v[1] / n, v[2] / n)


def _geom(j) -> Grid:  # geom_of, io.cpp:178-185
    d = j["dims"]
    return Grid((int(d[0]), int(d[1]), int(d[2])), _vec3(j["origin"]), _vec3(j["voxel_size"]))


def load_scene(path: str) -> Scene:
    """load_scene (io.cpp:190-278): the reference's JSON scene, with species extinction
    from VGRD files (relative to the scene file) or constants.  Every species must share
    one grid geometry (the engine keeps one voxel lattice)."""
    try:
        with open(path) as f:
            j = json.load(f)
    except OSError as e:
        raise IOError(f"load_scene: cannot open {path}") from e
    except json.JSONDecodeError as e:
        raise ValueError(f"load_scene: parse error in {path}: {e}") from e
    base = os.path.dirname(path)
    unit = j.get("unit", "m")
    if unit not in ("m", "km"):
        raise ValueError("load_scene: unit must be 'm' or 'km'")
    s = Scene(bounds_min=_vec3(j["bounds"]["min"]), bounds_max=_vec3(j["bounds"]["max"]),
              unit=0 if unit == "m" else 1)
    jl = j["light"]
    lt = jl["type"]
    if lt == "point":
        s.light = Light("point", position=_vec3(jl["position"]), radiance=float(jl.get("radiance", 1.0)))
    elif lt == "sun":
        s.light = Light("sun", direction=_normalized(_vec3(jl["direction"])), radiance=float(jl.get("radiance", 1.0)))
    else:
        raise ValueError(f"load_scene: unknown light type '{lt}'")
    grid = None
    for js in j.get("species", []):
        ph = js["phase"]
        if ph["type"] not in ("hg", "rayleigh"):
            raise ValueError(f"scene: unknown phase type '{ph['type']}'")
        je = js["extinction"]
        if "grid" in je:
            g = gpu.load_grid(os.path.join(base, je["grid"]))
            geom = Grid(g["dims"], g["origin"], g["voxel_size"])
            ext = g["values"]
        else:
            geom = _geom(je)
            ext = np.full(geom.voxel_count, float(je["constant"]))
        if grid is not None and (geom.dims, geom.origin, geom.voxel_size) != (grid.dims, grid.origin, grid.voxel_size):
            raise ValueError("load_scene: species grids differ (one voxel lattice per scene)")
        grid = geom
        s.species.append(Species(ext, albedo=float(js["albedo"]), phase=ph["type"], g=float(ph.get("g", 0.0)),
                                 unknown=bool(js.get("unknown", False))))
    if grid is not None:
        s.grid = grid
    for js in j.get("surfaces", []):
        br = js["brdf"]
        if br["type"] not in ("diffuse", "phong"):
            raise ValueError(f"scene: unknown brdf type '{br['type']}'")
        kw = dict(brdf=br["type"], albedo=float(br.get("albedo", 1.0)), kappa_s=float(br.get("kappa_s", 0.0)),
                  gamma=float(br.get("gamma", 0.0)), target=bool(js.get("target", False)))
        t = js["type"]
        if t == "sphere":
            s.surfaces.append(Surface("sphere", center=_vec3(js["center"]), radius=float(js["radius"]), **kw))
        elif t == "face":
            s.surfaces.append(Surface("face", axis=int(js["axis"]), coord=float(js["coord"]),
                                      lo=(float(js["lo"][0]), float(js["lo"][1])),
                                      hi=(float(js["hi"][0]), float(js["hi"][1])),
                                      normal_sign=float(js.get("normal", 1.0)), **kw))
        else:
            raise ValueError(f"load_scene: unknown surface type '{t}'")
    for jd in j["detectors"]:
        s.detectors.append(Detector(_vec3(jd["position"]), _vec3(jd["direction"]),
                                    _vec3(jd["up"]) if "up" in jd else (0.0, 0.0, 1.0),
                                    int(jd["rows"]), int(jd["cols"]), float(jd["fov"])))
    return s


def save_pfm(image: np.ndarray, path: str):
    """save_pfm (io.cpp:94-108): grayscale PFM, little-endian f32, rows bottom-to-top."""
    im = np.asarray(image, dtype=np.float64)
    bad = ~np.isfinite(im.reshape(-1))
    if bad.any():
        raise ValueError(f"save_pfm: {int(bad.sum())} non-finite pixel(s), first at index {int(np.argmax(bad))}")
    rows, cols = im.shape
    with open(path, "wb") as f:
        f.write(f"Pf\n{cols} {rows}\n-1.0\n".encode())
        f.write(im[::-1].astype("<f4").tobytes())


def load_pfm(path: str) -> np.ndarray:
    """load_pfm (io.cpp:110-129)."""
    with open(path, "rb") as f:
        data = f.read()
    toks: List[bytes] = []
    pos = 0
    while len(toks) < 4:  # "Pf", cols, rows, scale, separated by whitespace
        while pos < len(data) and data[pos:pos + 1].isspace():
            pos += 1
        start = pos
        while pos < len(data) and not data[pos:pos + 1].isspace():
            pos += 1
        if start == pos:
            raise ValueError(f"load_pfm: unsupported header in {path}")
        toks.append(data[start:pos])
    if toks[0] != b"Pf":
        raise ValueError(f"load_pfm: not a grayscale PFM: {path}")
    cols, rows, scale = int(toks[1]), int(toks[2]), float(toks[3])
    if cols <= 0 or rows <= 0 or scale >= 0.0:
        raise ValueError(f"load_pfm: unsupported header in {path}")
    pos += 1  # single whitespace before the payload
    n = rows * cols * 4
    if len(data) - pos < n:
        raise ValueError(f"load_pfm: truncated payload in {path}")
    return np.frombuffer(data[pos:pos + n], dtype="<f4").astype(np.float64).reshape(rows, cols)[::-1].copy()
