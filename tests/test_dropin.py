"""Drop-in checks for reference callers.

* The reference's coarse C API (include/pathrec.h) served by the engine library: the JSON
  scene loader is pinned on CPU against the reference's load_scene (a scene loaded through
  prc_scene_load renders, through the reference's own render(), to the same bits as the
  reference's loader), and on the GPU the reference's own C test (tests/test_capi.c,
  compiled in place against our pathrec.h) passes against the engine.
* The C++ mirror (include/pathrec_gpu.hpp) is source-compatible: the reference's
  tests/helpers.hpp and an acceptance-style caller (tests/cpp/ref_caller.cpp) build
  unchanged through the include shim and pass on the GPU.
"""
import ctypes as C
import json
import os
import subprocess

import numpy as np
import pytest

from paper_2110_00085_b200 import abi
from paper_2110_00085_b200 import io as pio
from tests.fixtures import FIXTURES
from tests.test_io import write_scene_json

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
REF_DIR = "/root/reference/proj"
CAPI_BIN = os.path.join(ROOT, "oracle", "_ref", "test_capi_engine")
CALLER_BIN = os.path.join(ROOT, "oracle", "_ref", "ref_caller_engine")


def engine():
    from paper_2110_00085_b200.build import build
    lib = C.CDLL(build())
    lib.prc_last_error.restype = C.c_char_p
    lib.prc_scene_load.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
    lib.prc_scene_free.argtypes = [C.c_void_p]
    lib.prc_scene_describe.argtypes = [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_int)]
    lib.prc_scene_validate.argtypes = [C.c_void_p, C.c_char_p, C.c_size_t, C.POINTER(C.c_int)]
    lib.prc_scene_detector_count.argtypes = [C.c_void_p, C.POINTER(C.c_int)]
    lib.prc_grid_load.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
    lib.prc_grid_save.argtypes = [C.c_void_p, C.c_char_p]
    lib.prc_grid_free.argtypes = [C.c_void_p]
    lib.prc_render.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)]
    lib.prc_result_image.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.POINTER(C.c_double)), C.POINTER(C.c_int),
                                     C.POINTER(C.c_int)]
    lib.prc_result_free.argtypes = [C.c_void_p]
    lib.prc_reconstruct.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)]
    lib.prc_result_final_loss.argtypes = [C.c_void_p, C.POINTER(C.c_double)]
    lib.prc_result_grid_save.argtypes = [C.c_void_p, C.c_char_p]
    lib.prc_result_save_csv.argtypes = [C.c_void_p, C.c_char_p]
    return lib


class RenderOpts(C.Structure):  # prc_render_opts (pathrec.h)
    _fields_ = [("n_paths", C.c_uint64), ("seed", C.c_uint64), ("workers", C.c_int), ("max_bounces", C.c_int),
                ("store_dump_path", C.c_char_p)]


class ReconstructOpts(C.Structure):  # prc_reconstruct_opts (pathrec.h)
    _fields_ = [("seed", C.c_uint64), ("n_paths", C.c_uint64), ("workers", C.c_int), ("max_bounces", C.c_int),
                ("recycle_period", C.c_int), ("max_iterations", C.c_int), ("n_stages", C.c_int),
                ("alpha", C.c_double), ("carve_threshold", C.c_double), ("carve_fill", C.c_double),
                ("init_kappa", C.c_double), ("init_gamma", C.c_double), ("gamma_step_scale", C.c_double),
                ("gt_dir", C.c_char_p), ("out_dir", C.c_char_p), ("truth_grid", C.c_char_p),
                ("truth_kappa", C.c_double), ("truth_gamma", C.c_double)]


def load(lib, path):
    sc = C.c_void_p()
    rc = lib.prc_scene_load(str(path).encode(), C.byref(sc))
    return rc, sc


# ---------------------------------------------------------------- CPU: the JSON loader
@pytest.mark.parametrize("name", list(FIXTURES))
def test_c_scene_loader_matches_reference_loader(ref, tmp_path, name):
    lib = engine()
    scene = FIXTURES[name]["scene"]()
    path = write_scene_json(scene, str(tmp_path), sun_raw=(0.3, -0.2, -2.0) if scene.light.kind == "sun" else None)
    rc, sc = load(lib, path)
    assert rc == abi.PRC_OK, lib.prc_last_error()
    try:
        d = C.c_void_p()
        unit = C.c_int()
        assert lib.prc_scene_describe(sc, C.byref(d), C.byref(unit)) == abi.PRC_OK
        n_pix = scene.pixel_count
        img = np.zeros(n_pix)
        tr = C.c_uint64()
        # the reference's render() of the C-loaded scene == render() of its own load_scene
        assert ref.lib.ref_render(d, None, 400, 17, 500, -1, 1, 0, None, img.ctypes.data_as(abi.c_double_p),
                                  C.byref(tr)) == 0
        want = ref.render_json(path, 400, 17, n_pix)
        assert np.array_equal(img.view(np.uint64), want.view(np.uint64))
        nv = C.c_int(-1)
        buf = C.create_string_buffer(256)
        assert lib.prc_scene_validate(sc, buf, 256, C.byref(nv)) == abi.PRC_OK and nv.value == 0, buf.value
        nd = C.c_int()
        assert lib.prc_scene_detector_count(sc, C.byref(nd)) == abi.PRC_OK and nd.value == len(scene.detectors)
    finally:
        lib.prc_scene_free(sc)


def test_c_scene_loader_errors_classified_like_capi(tmp_path):
    lib = engine()
    rc, _ = load(lib, tmp_path / "absent.json")
    assert rc == abi.PRC_ERR_IO and b"cannot open" in lib.prc_last_error()
    for text, match in (('{"bounds": 12}', b"missing key"), ("{not json", b"parse error"),
                        ('{"bounds": {"min": [0,0,0], "max": [1,1,1]}, "light": {"type": "laser"}, '
                         '"detectors": []}', b"unknown light type"),
                        ('{"unit": "ft", "bounds": {"min": [0,0,0], "max": [1,1,1]}}', b"unit must be")):
        p = tmp_path / "bad.json"
        p.write_text(text)
        rc, _ = load(lib, p)
        assert rc == abi.PRC_ERR_CONFIG and match in lib.prc_last_error(), (text, lib.prc_last_error())
    # a scene that loads but violates invariants is reported by prc_scene_validate
    j = {"bounds": {"min": [0, 0, 0], "max": [1, 1, 1]}, "light": {"type": "point", "position": [0.5, 0.5, 0.5]},
         "species": [{"albedo": 1.5, "phase": {"type": "hg", "g": 1.2}, "unknown": True,
                      "extinction": {"dims": [2, 2, 2], "origin": [0, 0, 0], "voxel_size": [0.5, 0.5, 0.5],
                                     "constant": -1.0}}],
         "detectors": [{"position": [0.5, 0.5, 2], "direction": [0, 0, -1], "rows": 0, "cols": 4, "fov": 4.0}]}
    p = tmp_path / "v.json"
    p.write_text(json.dumps(j))
    rc, sc = load(lib, p)
    assert rc == abi.PRC_OK
    nv = C.c_int()
    buf = C.create_string_buffer(1024)
    assert lib.prc_scene_validate(sc, buf, 1024, C.byref(nv)) == abi.PRC_OK
    assert nv.value == 5 and b"albedo" in buf.value and b"|g|" in buf.value
    lib.prc_scene_free(sc)


def test_c_grid_handles(ref, tmp_path):
    lib = engine()
    vals = np.random.default_rng(2).uniform(0, 3, 4 * 3 * 2)
    ref.save_grid(str(tmp_path / "a.vgrd"), (4, 3, 2), (0.1, 0.2, 0.3), (0.5, 0.25, 0.125), vals, unit=1)
    g = C.c_void_p()
    assert lib.prc_grid_load(str(tmp_path / "a.vgrd").encode(), C.byref(g)) == abi.PRC_OK
    assert lib.prc_grid_save(g, str(tmp_path / "b.vgrd").encode()) == abi.PRC_OK
    lib.prc_grid_free(g)
    assert (tmp_path / "a.vgrd").read_bytes() == (tmp_path / "b.vgrd").read_bytes()
    pio.save_pfm(np.ones((2, 3)), str(tmp_path / "x.pfm"))
    assert lib.prc_grid_load(str(tmp_path / "x.pfm").encode(), C.byref(g)) == abi.PRC_ERR_CONFIG  # capi.cpp:24-32
    assert lib.prc_grid_load(str(tmp_path / "absent.vgrd").encode(), C.byref(g)) == abi.PRC_ERR_IO


@pytest.mark.skipif(not os.path.isdir(REF_DIR), reason="needs /root/reference to compile the reference's callers")
def test_reference_callers_build_unchanged():
    """test_capi.c (reference, C) and helpers.hpp + ref_caller.cpp (C++) compile and link
    against the engine with no edits (oracle/Makefile `dropin`)."""
    from paper_2110_00085_b200.build import build
    build()
    subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "dropin"])
    assert os.path.exists(CAPI_BIN) and os.path.exists(CALLER_BIN)


# ---------------------------------------------------------------- GPU
@pytest.mark.gpu
def test_reference_capi_test_passes_on_the_engine(tmp_path):
    if not os.path.exists(CAPI_BIN):
        pytest.skip("oracle/_ref/test_capi_engine not built (make -C oracle dropin)")
    r = subprocess.run([CAPI_BIN], cwd=str(tmp_path), capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0 and "all checks passed" in r.stdout, r.stderr


@pytest.mark.gpu
def test_reference_shaped_cpp_caller_passes_on_the_engine(tmp_path):
    if not os.path.exists(CALLER_BIN):
        pytest.skip("oracle/_ref/ref_caller_engine not built (make -C oracle dropin)")
    r = subprocess.run([CALLER_BIN], cwd=str(tmp_path), capture_output=True, text=True, timeout=900)
    print(r.stdout, r.stderr)
    assert r.returncode == 0 and "ALL PASSED" in r.stdout, r.stdout + r.stderr


@pytest.mark.gpu
def test_coarse_render_and_reconstruct(ctx, tmp_path):
    """prc_render of a JSON scene equals the engine's render of the same scene; the store
    dump is a PSTR the engine re-imports.  prc_reconstruct reads gt_NNN.pfm, carves the
    initial field, runs the schedule (stages doubling n_paths) and writes loss.csv and a
    VGRD checkpoint every 25 iterations to out_dir, as capi.cpp:124-204."""
    from paper_2110_00085_b200 import scene as S
    from paper_2110_00085_b200.gpu import RenderOptions
    lib = engine()
    scene = S.cloud_scene(8, 10, 10)
    path = write_scene_json(scene, str(tmp_path))
    rc, sc = load(lib, path)
    assert rc == abi.PRC_OK
    res = C.c_void_p()
    opts = RenderOpts(50_000, 5, 0, 0, str(tmp_path / "dump.pstr").encode())
    assert lib.prc_render(sc, C.byref(opts), C.byref(res)) == abi.PRC_OK, lib.prc_last_error()
    got = []
    for k in range(len(scene.detectors)):
        data, r_, c_ = C.POINTER(C.c_double)(), C.c_int(), C.c_int()
        assert lib.prc_result_image(res, k, C.byref(data), C.byref(r_), C.byref(c_)) == abi.PRC_OK
        got.append(np.ctypeslib.as_array(data, shape=(r_.value * c_.value,)).copy())
    lib.prc_result_free(res)
    loaded = pio.load_scene(path)
    ctx.upload(loaded)
    want = ctx.render(loaded, RenderOptions(n_paths=50_000, seed=5, keep_paths=True))
    g = np.concatenate(got)
    assert np.abs(g - want.images).max() <= 1e-12 * np.abs(want.images).max()
    st = ctx.load_store(str(tmp_path / "dump.pstr"))
    assert np.array_equal(np.sort(st.sizes()), np.sort(want.store.sizes()))
    # reconstruct from PFM ground truth
    gt_dir = tmp_path / "gt"
    gt_dir.mkdir()
    for k, im in enumerate(scene.split_images(ctx.render(loaded, RenderOptions(n_paths=100_000, seed=9)).images)):
        pio.save_pfm(np.asarray(im).reshape(scene.detectors[k].rows, scene.detectors[k].cols), str(gt_dir / f"gt_{k:03d}.pfm"))
    out_dir = tmp_path / "out"
    out_dir.mkdir()
    ro = ReconstructOpts(seed=3, n_paths=10_000, recycle_period=5, max_iterations=26, n_stages=2, alpha=0.3,
                         carve_threshold=0.05, carve_fill=2.0, gt_dir=str(gt_dir).encode(),
                         out_dir=str(out_dir).encode())
    assert lib.prc_reconstruct(sc, C.byref(ro), C.byref(res)) == abi.PRC_OK, lib.prc_last_error()
    loss = C.c_double()
    assert lib.prc_result_final_loss(res, C.byref(loss)) == abi.PRC_OK and np.isfinite(loss.value)
    assert lib.prc_result_grid_save(res, str(tmp_path / "final.vgrd").encode()) == abi.PRC_OK
    assert lib.prc_result_save_csv(res, str(tmp_path / "final.csv").encode()) == abi.PRC_OK
    lib.prc_result_free(res)
    lib.prc_scene_free(sc)
    assert (out_dir / "checkpoint_24.vgrd").exists() and (out_dir / "loss.csv").exists()
    rows = (tmp_path / "final.csv").read_text().splitlines()
    assert len(rows) == 27 and rows[0] == "iter,time_s,loss,eps,delta,stage"
    from paper_2110_00085_b200 import gpu
    assert gpu.load_grid(str(tmp_path / "final.vgrd"))["dims"] == tuple(scene.grid.dims)
