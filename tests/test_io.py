"""Host formats around the loop: the reference's JSON scene loader
(io.cpp:190-278) and PFM images (io.cpp:94-129), pinned against the reference library.
A scene loaded by paper_2110_00085_b200.io.load_scene renders, through the reference's
own render(), to the same bits as the reference's load_scene of the same file."""
import json
import os

import numpy as np
import pytest

from paper_2110_00085_b200 import gpu
from paper_2110_00085_b200 import io as pio
from tests.fixtures import FIXTURES


def write_scene_json(scene, d, name="scene.json", sun_raw=None):
    """Test helper: a Scene as the reference's JSON schema, species grids as VGRD files."""
    j = {"unit": "km" if scene.unit == 1 else "m",
         "bounds": {"min": list(scene.bounds_min), "max": list(scene.bounds_max)}}
    L = scene.light
    if L.kind == "point":
        j["light"] = {"type": "point", "position": list(L.position), "radiance": L.radiance}
    else:
        j["light"] = {"type": "sun", "direction": list(sun_raw or L.direction), "radiance": L.radiance}
    sp = []
    for k, s in enumerate(scene.species):
        f = f"species{k}.vgrd"
        gpu.save_grid(os.path.join(d, f), scene.grid.dims, scene.grid.origin, scene.grid.voxel_size, s.extinction)
        ph = {"type": s.phase} if s.phase == "rayleigh" else {"type": "hg", "g": s.g}
        sp.append({"name": f"s{k}", "albedo": s.albedo, "phase": ph, "unknown": s.unknown,
                   "extinction": {"grid": f}})
    if sp:
        j["species"] = sp
    sf = []
    for s in scene.surfaces:
        br = {"type": "diffuse", "albedo": s.albedo} if s.brdf == "diffuse" else \
            {"type": "phong", "kappa_s": s.kappa_s, "gamma": s.gamma}
        if s.kind == "sphere":
            sf.append({"type": "sphere", "center": list(s.center), "radius": s.radius, "brdf": br, "target": s.target})
        else:
            sf.append({"type": "face", "axis": s.axis, "coord": s.coord, "lo": list(s.lo), "hi": list(s.hi),
                       "normal": s.normal_sign, "brdf": br, "target": s.target})
    if sf:
        j["surfaces"] = sf
    j["detectors"] = [{"position": list(x.position), "direction": list(x.direction), "up": list(x.up),
                       "rows": x.rows, "cols": x.cols, "fov": x.fov} for x in scene.detectors]
    p = os.path.join(d, name)
    with open(p, "w") as f:
        json.dump(j, f)
    return p


@pytest.mark.parametrize("name", list(FIXTURES))
def test_json_scene_renders_like_reference_loader(ref, tmp_path, name):
    scene = FIXTURES[name]["scene"]()
    path = write_scene_json(scene, str(tmp_path), sun_raw=(0.3, -0.2, -2.0) if scene.light.kind == "sun" else None)
    ours = pio.load_scene(path)
    assert ours.pixel_count == scene.pixel_count and ours.voxel_count == scene.voxel_count
    a = ref.render(ours, 400, 17)[0]
    b = ref.render_json(path, 400, 17, ours.pixel_count)
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


def test_json_scene_constant_extinction_and_defaults(ref, tmp_path):
    j = {"bounds": {"min": [0, 0, 0], "max": [1, 1, 1]},
         "light": {"type": "point", "position": [0.5, 0.5, 0.5]},
         "species": [{"albedo": 0.9, "phase": {"type": "hg", "g": 0.5}, "unknown": True,
                      "extinction": {"dims": [4, 4, 4], "origin": [0, 0, 0], "voxel_size": [0.25, 0.25, 0.25],
                                     "constant": 2.0}}],
         "detectors": [{"position": [0.5, 0.5, 2.0], "direction": [0, 0, -1], "up": [0, 1, 0], "rows": 6,
                        "cols": 5, "fov": 0.8},
                       {"position": [2.0, 0.5, 0.5], "direction": [-1, 0, 0], "rows": 4, "cols": 4, "fov": 0.7}]}
    p = tmp_path / "c.json"
    p.write_text(json.dumps(j))
    s = pio.load_scene(str(p))
    assert s.unit == 0 and s.light.radiance == 1.0 and s.detectors[1].up == (0.0, 0.0, 1.0)
    assert np.all(s.species[0].extinction == 2.0) and s.unknown_species() == 0
    a = ref.render(s, 400, 5)[0]
    b = ref.render_json(str(p), 400, 5, s.pixel_count)
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


@pytest.mark.parametrize("patch,match", [({"unit": "ft"}, "unit must be"),
                                         ({"light": {"type": "laser"}}, "unknown light type")])
def test_json_scene_errors(tmp_path, patch, match):
    j = {"bounds": {"min": [0, 0, 0], "max": [1, 1, 1]}, "light": {"type": "point", "position": [0, 0, 0]},
         "detectors": []}
    j.update(patch)
    p = tmp_path / "e.json"
    p.write_text(json.dumps(j))
    with pytest.raises(ValueError, match=match):
        pio.load_scene(str(p))
    with pytest.raises(IOError):
        pio.load_scene(str(tmp_path / "missing.json"))


def test_pfm_matches_reference(ref, tmp_path):
    im = np.random.default_rng(4).uniform(-1, 5, size=(7, 11))
    pio.save_pfm(im, str(tmp_path / "a.pfm"))
    ref.save_pfm(str(tmp_path / "b.pfm"), im)
    assert (tmp_path / "a.pfm").read_bytes() == (tmp_path / "b.pfm").read_bytes()
    x = pio.load_pfm(str(tmp_path / "b.pfm"))
    y = ref.load_pfm(str(tmp_path / "a.pfm"))
    assert np.array_equal(x, y) and np.array_equal(x, im.astype(np.float32).astype(np.float64))
    with pytest.raises(ValueError, match="non-finite"):
        pio.save_pfm(np.array([[1.0, np.nan]]), str(tmp_path / "c.pfm"))
