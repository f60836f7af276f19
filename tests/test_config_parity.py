"""Parity at the BASELINE.json configurations' geometry.

The fixture tests (test_gpu_parity.py) use 5^3-12^3 grids.  Here the device path runs on
the benchmarked scenes themselves: 32^3 / 9 x 64^2 (a), 128^3 / 9 x 128^2 (b) and the
two-species 128^3 cloud (c), with power-of-two voxel sizes (the DDA's vs_pow2 set-up),
the default mapping (event-major wavefront, ray packets of 3, padded guard-free walks,
8 gradient copies) and the bench's recycle point beta_t = beta_ref (1 + 0.01 (v mod 5))
with residual weights F_t - 0.9 F_ref.

* Identical stored path sets: a device-traced store (seed 7, sorted by B) is exported to
  PSTR v1 and evaluated by the unmodified reference (oracle/_ref, evaluate_store,
  pathstore.cpp:315-368; grad_forward, gradient.cpp:111-128).  Images within 1e-5
  (max_p |g - r| / max(|r_p|, 1e-3 max|r|)) and gradients within 1e-5 of the
  scale-relative bar of acceptance.cpp:238-245.
* A reference-written config-(a) store is imported and evaluated on the device.
* At the full bench size (1e8 paths, config (b)) the reference cannot hold the store
  (~8 TB AoS), so size-independent properties are checked instead: the result does not
  depend on the storage order (unsorted vs sorted by B) or on the kernel mapping
  (packets of 3 vs single rays), to fp64 summation-order rounding.
"""
import os
import struct

import numpy as np
import pytest

from paper_2110_00085_b200 import abi
from paper_2110_00085_b200 import scene as S
from paper_2110_00085_b200.gpu import EvalOptions, RenderOptions

pytestmark = pytest.mark.gpu

IMG_TOL = 1e-5
GRAD_TOL = 1e-5
WORKERS = os.cpu_count() or 1


def img_err(a, r):
    floor = 1e-3 * max(np.abs(r).max(), 1e-300)
    return float((np.abs(a - r) / np.maximum(np.abs(r), floor)).max())


def grad_err(a, r):
    scale = max(np.abs(r).max(), 1e-300)
    return float((np.abs(a - r) / np.maximum(np.maximum(np.abs(a), np.abs(r)), scale)).max())


CONFIGS = {
    "a": dict(scene=lambda: S.cloud_scene(32, 64, 64), n=20_000),
    "b": dict(scene=lambda: S.cloud_scene(128, 128, 128), n=8_000),
    "c": dict(scene=lambda: S.cloud_scene(128, 128, 128, two_species=True), n=6_000),
    "e": dict(scene=lambda: S.cloud_scene(256, 128, 128), n=4_000),
}


def _patch_ref_beta(path, beta):
    """Rewrites the PSTR v1 header's ref_params.beta block (pathstore.cpp:410-425) in place."""
    with open(path, "r+b") as f:
        head = f.read(4 + 4 + 8 + 8 + 8 + 1 + 8)
        nb = struct.unpack_from("<Q", head, 33)[0]
        assert nb == beta.size
        f.seek(41)
        f.write(np.ascontiguousarray(beta, dtype="<f8").tobytes())


@pytest.mark.parametrize("cfg", ["a", "b", "c", "e"])
def test_config_store_matches_reference(ctx, ref, tmp_path, cfg):
    scene = CONFIGS[cfg]["scene"]()
    n = CONFIGS[cfg]["n"]
    ctx.upload(scene)
    rr = ctx.render(scene, RenderOptions(n_paths=n, seed=7, keep_paths=True))
    st = rr.store
    ctx.sort_by_size(st)
    pstr = str(tmp_path / f"{cfg}.pstr")
    st.save(pstr)
    u = scene.unknown_species()
    beta_ref = scene.species[u].extinction
    t = S.ParamSet(S.recycle_point(beta_ref))
    F_ref = ref.evaluate(scene, pstr, None, abi.PRC_EVAL_NORMALIZE, workers=WORKERS)["images"]
    F_t = ref.evaluate(scene, pstr, t, abi.PRC_EVAL_NORMALIZE, workers=WORKERS)["images"]
    w = F_t - 0.9 * F_ref
    r = ref.evaluate(scene, pstr, t, abi.PRC_EVAL_NORMALIZE | abi.PRC_EVAL_WANT_GRAD, w, workers=WORKERS)
    per = len(scene.species) > 1
    g = ctx.evaluate_store(scene, st, t, EvalOptions(want_grad=True, pixel_weights=w, per_species=per))
    e_ref = img_err(ctx.recycled_render(scene, st, None), F_ref)
    e_img = img_err(g.images, r["images"])
    grad0 = g.grad_beta[u] if per else g.grad_beta
    e_grad = grad_err(grad0, r["grad"])
    assert g.clamp_events == r["clamp_events"]
    msg = [f"config ({cfg}) {n} paths: F_ref {e_ref:.2e}, F_t {e_img:.2e}, grad {e_grad:.2e}"]
    assert e_ref <= IMG_TOL and e_img <= IMG_TOL and e_grad <= GRAD_TOL, msg
    if per:
        # per-type gradient of the known species (SURVEY a15 flip oracle): species 1 at its
        # recycle point, species 0 at its reference values; the reference sees species 1 as
        # the unknown, with the store's ref_params.beta set to species 1's sampling values
        b1 = scene.species[1].extinction
        t1 = S.recycle_point(b1)
        flip = CONFIGS[cfg]["scene"]()
        flip.species[0].unknown, flip.species[1].unknown = False, True
        _patch_ref_beta(pstr, b1)
        rf = ref.evaluate(flip, pstr, S.ParamSet(t1), abi.PRC_EVAL_NORMALIZE | abi.PRC_EVAL_WANT_GRAD, w,
                          workers=WORKERS)
        g1 = ctx.evaluate_store(scene, st, S.ParamSet(species_beta=[None, t1]),
                                EvalOptions(want_grad=True, pixel_weights=w, per_species=True))
        e_img1 = img_err(g1.images, rf["images"])
        e_grad1 = grad_err(g1.grad_beta[1], rf["grad"])
        msg.append(f"species 1: F_t {e_img1:.2e}, grad {e_grad1:.2e}")
        assert e_img1 <= IMG_TOL and e_grad1 <= GRAD_TOL, msg
    print("; ".join(msg))


@pytest.mark.parametrize("cfg,n", [("a", 2000), ("c", 800), ("e", 600)])
@pytest.mark.parametrize("materialized", [False, True])
def test_reference_written_config_store(ctx, ref, tmp_path, cfg, n, materialized):
    """A store traced and sorted by the reference at a config's geometry, imported with
    recomputed spans or its own stored spans and events."""
    scene = CONFIGS[cfg]["scene"]()
    pstr = str(tmp_path / f"ref_{cfg}.pstr")
    ref.render(scene, n, 7, pstr_out=pstr, sort=True, workers=WORKERS)
    ctx.upload(scene)
    st = ctx.load_store(pstr, materialized=materialized)
    assert st.sorted_flag
    t = S.ParamSet(S.recycle_point(scene.species[scene.unknown_species()].extinction))
    F_ref = ref.evaluate(scene, pstr, None, abi.PRC_EVAL_NORMALIZE, workers=WORKERS)["images"]
    F_t = ref.evaluate(scene, pstr, t, abi.PRC_EVAL_NORMALIZE, workers=WORKERS)["images"]
    w = F_t - 0.9 * F_ref
    r = ref.evaluate(scene, pstr, t, abi.PRC_EVAL_NORMALIZE | abi.PRC_EVAL_WANT_GRAD, w, workers=WORKERS)
    g = ctx.evaluate_store(scene, st, t, EvalOptions(want_grad=True, pixel_weights=w))
    e_img, e_grad = img_err(g.images, r["images"]), grad_err(g.grad_beta, r["grad"])
    print(f"reference-written config ({cfg}) store (materialized={materialized}): F_t {e_img:.2e}, grad {e_grad:.2e}")
    assert e_img <= IMG_TOL and e_grad <= GRAD_TOL


@pytest.mark.parametrize("materialized", [False, True])
def test_reference_written_config_d_store(ctx, ref, tmp_path, materialized):
    """A reflectometry store traced and sorted by the reference at config (d) geometry,
    imported (recomputed chords, or its own stored spans and events) and evaluated twice
    (the second time over the event list)."""
    scene = S.reflectometry_scene(256, 256, 16)
    pstr = str(tmp_path / "ref_d.pstr")
    ref.render(scene, 3000, 7, pstr_out=pstr, sort=True, workers=WORKERS)
    ctx.upload(scene)
    st = ctx.load_store(pstr, materialized=materialized)
    t = S.ParamSet(None, 0.55, 38.0)
    F_ref = ref.evaluate(scene, pstr, None, abi.PRC_EVAL_NORMALIZE, workers=WORKERS)["images"]
    F_t = ref.evaluate(scene, pstr, t, abi.PRC_EVAL_NORMALIZE, workers=WORKERS)["images"]
    w = F_t - 0.9 * F_ref
    r = ref.evaluate(scene, pstr, t, abi.PRC_EVAL_NORMALIZE | abi.PRC_EVAL_WANT_GRAD, w, workers=WORKERS)
    for _ in range(2):
        g = ctx.evaluate_store(scene, st, t, EvalOptions(want_grad=True, pixel_weights=w))
        e_img = img_err(g.images, r["images"])
        e_k = abs(g.grad_kappa - r["grad_kappa"]) / max(abs(r["grad_kappa"]), 1e-300)
        e_g = abs(g.grad_gamma - r["grad_gamma"]) / max(abs(r["grad_gamma"]), 1e-300)
        assert e_img <= IMG_TOL and e_k <= GRAD_TOL and e_g <= GRAD_TOL, (e_img, e_k, e_g)
    print(f"reference-written config (d) store (materialized={materialized}): F_t {e_img:.2e}, "
          f"d kappa {e_k:.2e}, d gamma {e_g:.2e}")


def test_config_d_store_matches_reference(ctx, ref, tmp_path):
    """Config (d), reflectometry (phong_box walls, the central Phong sphere as the unknown,
    14 diffuse spheres, 16 inward cameras at 256^2): no medium, so after the first forward
    over the store the device evaluates its compact event list (K4b' / K5b', cached lobe
    terms, K5a reduced to the Phong scores).  A device-traced store, exported to PSTR v1,
    evaluated by the reference at the recycle point (kappa, gamma) = (0.55, 38): images and
    d kappa, d gamma within 1e-5, through both the dense first pass and the event list."""
    scene = S.reflectometry_scene(256, 256, 16)
    ctx.upload(scene)
    rr = ctx.render(scene, RenderOptions(n_paths=20_000, seed=7, keep_paths=True))
    st = rr.store
    ctx.sort_by_size(st)
    pstr = str(tmp_path / "d.pstr")
    st.save(pstr)
    t = S.ParamSet(None, 0.55, 38.0)
    F_ref = ref.evaluate(scene, pstr, None, abi.PRC_EVAL_NORMALIZE, workers=WORKERS)["images"]
    F_t = ref.evaluate(scene, pstr, t, abi.PRC_EVAL_NORMALIZE, workers=WORKERS)["images"]
    w = F_t - 0.9 * F_ref
    r = ref.evaluate(scene, pstr, t, abi.PRC_EVAL_NORMALIZE | abi.PRC_EVAL_WANT_GRAD, w, workers=WORKERS)
    e_ref = img_err(ctx.recycled_render(scene, st, None), F_ref)  # dense pass, builds the list
    msg = [f"config (d) 20000 paths: F_ref {e_ref:.2e}"]
    for k in range(2):  # event list
        g = ctx.evaluate_store(scene, st, t, EvalOptions(want_grad=True, pixel_weights=w))
        e_img = img_err(g.images, r["images"])
        e_k = abs(g.grad_kappa - r["grad_kappa"]) / max(abs(r["grad_kappa"]), 1e-300)
        e_g = abs(g.grad_gamma - r["grad_gamma"]) / max(abs(r["grad_gamma"]), 1e-300)
        msg.append(f"F_t {e_img:.2e}, d kappa {e_k:.2e}, d gamma {e_g:.2e}")
        assert g.clamp_events == r["clamp_events"]
        assert e_ref <= IMG_TOL and e_img <= IMG_TOL and e_k <= GRAD_TOL and e_g <= GRAD_TOL, msg
    assert r["images"].max() > 0.0 and r["grad_kappa"] != 0.0
    print("; ".join(msg))
    st.free()


def test_full_size_order_and_mapping_invariance(ctx):
    """Config (b) at the bench's 1e8 paths: the recycled image and gradient do not depend
    on the storage order (path-major trace order vs sorted by B, sort invariance of
    acceptance.cpp:330-347) or on the gradient kernel's mapping (packets of 3 rays merging
    same-voxel spans vs one ray per thread), up to fp64 summation order."""
    scene = S.cloud_scene(128, 128, 128)
    ctx.upload(scene)
    rr = ctx.render(scene, RenderOptions(n_paths=100_000_000, seed=7, keep_paths=True))
    st = rr.store
    t = S.ParamSet(S.recycle_point(scene.species[0].extinction))
    w = ctx.recycled_render(scene, st, t) - 0.9 * rr.images
    opt = EvalOptions(want_grad=True, pixel_weights=w)
    a = ctx.evaluate_store(scene, st, t, opt)  # unsorted
    ctx.sort_by_size(st)
    b = ctx.evaluate_store(scene, st, t, opt)  # sorted, packets of 3
    ctx.set_option("packet", 1)
    try:
        c = ctx.evaluate_store(scene, st, t, opt)  # sorted, one ray per thread
    finally:
        ctx.set_option("packet", 3)
    errs = [img_err(a.images, b.images), img_err(c.images, b.images),
            grad_err(a.grad_beta, b.grad_beta), grad_err(c.grad_beta, b.grad_beta)]
    print("1e8 paths: unsorted/sorted image %.1e, packet1/packet3 image %.1e, "
          "unsorted/sorted grad %.1e, packet1/packet3 grad %.1e" % tuple(errs))
    assert max(errs[:2]) <= 1e-11 and max(errs[2:]) <= 1e-9
    assert a.clamp_events == b.clamp_events == c.clamp_events
    st.free()
