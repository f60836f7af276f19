"""GPU parity tests: the CUDA path (through the C ABI) against the CPU oracle and the
reference's golden vectors.

Tolerances (north_star): images and gradients within 1e-5 relative on identical stored
path sets; sort order, voxel indexing (DDA spans incl. length bits) and pixel indices
bit-exact; fresh Monte-Carlo sampling within stated statistical tolerances.
"""
import math
import os

import numpy as np
import pytest

from paper_2110_00085_b200 import abi
from paper_2110_00085_b200 import scene as S
from paper_2110_00085_b200.gpu import EvalOptions, PrcConfigError, PrcIOError, RenderOptions
from tests.fixtures import FIXTURES, golden, perturbed, weight_patterns

pytestmark = pytest.mark.gpu

IMG_TOL = 1e-5   # max_p |g - r| / max(|r_p|, 1e-3 max|r|)
GRAD_TOL = 1e-5  # |g - r| <= 1e-5 max(|g|, |r|, max_v |r_v|)


def img_err(a, r):
    floor = 1e-3 * max(np.abs(r).max(), 1e-300)
    return float((np.abs(a - r) / np.maximum(np.abs(r), floor)).max()) if r.size else 0.0


def grad_err(a, r):
    if r.size == 0:
        return 0.0
    scale = max(np.abs(r).max(), 1e-300)
    return float((np.abs(a - r) / np.maximum(np.maximum(np.abs(a), np.abs(r)), scale)).max())


def scalar_err(a, r):
    return abs(a - r) / max(abs(a), abs(r), 1e-300)


# ---------------------------------------------------------------- bit-exact primitives
def test_philox_device_matches_reference(ctx):
    g = golden("common")
    assert [hex(x) for x in ctx.debug_philox(0, 0, 4)] == ["0x6627e8d5", "0xe169c58d", "0xbc57ac4c", "0x9b00dbd8"]
    for k, v in g.items():
        if k.startswith("philox_"):
            _, seed, stream = k.split("_")
            assert np.array_equal(ctx.debug_philox(int(seed), int(stream), v.size), v)


@pytest.mark.parametrize("name", ["tomo2", "cloud", "mixed"])
def test_device_dda_bit_exact(ctx, port, name):
    g = golden("common")
    scene = FIXTURES[name]["scene"]()
    ctx.upload(scene)
    c, v, ln = ctx.debug_walk(g[f"walk_{name}_rays"])
    assert np.array_equal(c, g[f"walk_{name}_counts"])
    assert np.array_equal(v, g[f"walk_{name}_vox"])
    assert np.array_equal(ln.view(np.uint64), g[f"walk_{name}_len"].view(np.uint64))
    # LE-style rays from interior points toward every camera of the bench scene (128^3)
    big = S.cloud_scene(128, 16, 16)
    ctx.upload(big)
    rng = np.random.default_rng(3)
    x = rng.uniform(0.05, 0.95, size=(3000, 3))
    rays = []
    for d in big.detectors:
        to = np.asarray(d.position) - x
        r = np.linalg.norm(to, axis=1)
        w = to * (1.0 / r)[:, None]
        rays.append(np.concatenate([x, w, r[:, None]], axis=1))
    rays = np.concatenate(rays)
    c1, v1, l1 = ctx.debug_walk(rays)
    c2, v2, l2 = port.walk(big, rays)
    assert np.array_equal(c1, c2) and np.array_equal(v1, v2)
    assert np.array_equal(l1.view(np.uint64), l2.view(np.uint64))


def _adversarial_rays(lo, hi, n_vox, rng, n=4000):
    """Rays that stress the end of a walk: exits through grid corners and edges (tmax ties
    on two or three axes), axis-aligned rays on voxel boundaries, rays entering from
    outside, grazing rays on a face, and random rays."""
    lo, hi = np.asarray(lo, float), np.asarray(hi, float)
    vs = (hi - lo) / np.asarray(n_vox)
    out = []
    x = lo + rng.uniform(0.02, 0.98, size=(n, 3)) * (hi - lo)
    corners = lo + (hi - lo) * rng.integers(0, 2, size=(n, 3))
    edges = corners.copy()
    ax = rng.integers(0, 3, size=n)
    edges[np.arange(n), ax] = lo[ax] + vs[ax] * rng.integers(0, np.asarray(n_vox)[ax])
    for tgt in (corners, edges):
        d = tgt - x
        r = np.linalg.norm(d, axis=1)
        out.append(np.c_[x, d / r[:, None], r * rng.choice([1.0, 2.0], size=n)])
    for a in range(3):  # axis-aligned, origins on voxel boundaries
        o = lo + vs * rng.integers(0, np.asarray(n_vox), size=(n, 3)) + vs * 0.5 * rng.integers(0, 2, size=(n, 3))
        d = np.zeros((n, 3))
        d[:, a] = rng.choice([-1.0, 1.0], size=n)
        out.append(np.c_[o, d, np.full(n, 3.0 * (hi - lo).max())])
    o = lo - 0.5 * (hi - lo) + rng.uniform(0, 2, size=(n, 3)) * (hi - lo)  # from outside
    d = x - o
    d /= np.linalg.norm(d, axis=1)[:, None]
    out.append(np.c_[o, d, np.full(n, 4.0 * (hi - lo).max())])
    o = x.copy()  # grazing: on the z = lo face, moving within it
    o[:, 2] = lo[2]
    d = rng.normal(size=(n, 3))
    d[:, 2] = 0.0
    d /= np.linalg.norm(d, axis=1)[:, None]
    out.append(np.c_[o, d, np.full(n, 2.0 * (hi - lo).max())])
    return np.concatenate(out)


@pytest.mark.parametrize("name", ["tomo2", "cloud", "mixed", "bench"])
def test_padded_walk_is_reference_walk_plus_border_tail(ctx, port, name):
    """The guard-free walk of the wavefront kernels (prc_device.cuh dda_walk_pad) emits
    exactly the reference's spans (voxel and length bits), followed by at most three
    spans in border voxels of the padded layout with negligible total length."""
    scene = S.cloud_scene(128, 16, 16) if name == "bench" else FIXTURES[name]["scene"]()
    ctx.upload(scene)
    g = scene.grid
    nx, ny, nz = g.dims
    lo = np.asarray(g.origin, float)
    hi = lo + np.asarray(g.voxel_size) * np.asarray(g.dims)
    rays = _adversarial_rays(lo, hi, g.dims, np.random.default_rng(17))
    c1, v1, l1 = ctx.debug_walk(rays, padded=True)
    c2, v2, l2 = port.walk(scene, rays)
    o1 = np.r_[0, np.cumsum(c1.astype(np.int64))]
    o2 = np.r_[0, np.cumsum(c2.astype(np.int64))]
    extra = c1.astype(np.int64) - c2.astype(np.int64)
    assert extra.min() >= 0 and extra.max() <= 3
    pnx, pny = nx + 2, ny + 2
    pv = v1.astype(np.int64)
    px, py, pz = pv % pnx, (pv // pnx) % pny, pv // (pnx * pny)
    border = (px == 0) | (px == nx + 1) | (py == 0) | (py == ny + 1) | (pz == 0) | (pz == nz + 1)
    interior = (px - 1) + nx * ((py - 1) + ny * (pz - 1))
    head = np.concatenate([np.arange(o1[i], o1[i] + c2[i]) for i in range(len(c2))]) if len(c2) else []
    head = np.asarray(head, np.int64)
    assert np.array_equal(interior[head], v2.astype(np.int64))
    assert not border[head].any()
    assert np.array_equal(l1[head].view(np.uint64), l2.view(np.uint64))
    tail = np.setdiff1d(np.arange(len(v1)), head)
    assert border[tail].all()
    scale = np.abs(rays[:, :3]).max() + np.abs(rays[:, 6]).max()
    assert (l1[tail] <= 1e-12 * scale).all()
    print(f"{name}: {len(rays)} rays, {int((extra > 0).sum())} walks end with a border tail "
          f"(max tail length {l1[tail].max() if len(tail) else 0.0:.2e})")


def test_pad_option_same_results(ctx, golden_dir):
    """Padded guard-free walks on/off: identical images (the border beta is zero) and
    gradients equal up to fp64 atomic ordering."""
    scene = FIXTURES["cloud"]["scene"]()
    ctx.upload(scene)
    st = ctx.load_store(str(golden_dir / "cloud.pstr"))
    ctx.sort_by_size(st)
    w = np.linspace(-1.0, 2.0, scene.pixel_count)
    res = []
    for pad in (1, 0):
        ctx.set_option("pad", pad)
        res.append(ctx.evaluate_store(scene, st, perturbed(scene), EvalOptions(want_grad=True, pixel_weights=w)))
    ctx.set_option("pad", 1)
    assert img_err(res[0].images, res[1].images) <= 1e-13
    assert grad_err(res[0].grad_beta, res[1].grad_beta) <= 1e-11


@pytest.mark.parametrize("name", ["tomo2", "cloud", "mixed"])
def test_device_pixel_of_bit_exact(ctx, name):
    g = golden("common")
    scene = FIXTURES[name]["scene"]()
    ctx.upload(scene)
    pts = g[f"pixel_{name}_pts"]
    for k in range(len(scene.detectors)):
        assert np.array_equal(ctx.debug_pixel_of(k, pts), g[f"pixel_{name}_{k}"])


# ---------------------------------------------------------------- K2 sort
@pytest.mark.parametrize("name", list(FIXTURES))
def test_sort_permutation_bit_exact(ctx, golden_dir, name):
    scene = FIXTURES[name]["scene"]()
    ctx.upload(scene)
    st = ctx.load_store(str(golden_dir / f"{name}.pstr"))
    assert not st.sorted_flag
    ctx.sort_by_size(st)
    assert st.sorted_flag
    assert np.array_equal(st.streams(), golden(name)["sorted_streams"])
    # idempotent (stable)
    before = st.streams()
    ctx.sort_by_size(st)
    assert np.array_equal(st.streams(), before)


def test_sort_large_random_sizes_match_stable_sort(ctx, port):
    scene = S.cloud_scene(16, 8, 8)
    ctx.upload(scene)
    st = ctx.render(scene, RenderOptions(n_paths=300_000, seed=5, keep_paths=True)).store
    sizes = st.sizes()
    ctx.sort_by_size(st)
    expect = np.argsort(sizes, kind="stable").astype(np.uint64)
    assert np.array_equal(st.streams(), expect)
    assert np.array_equal(st.sizes(), np.sort(sizes, kind="stable"))


def test_sort_empty_store_rejected(ctx):
    with pytest.raises(PrcConfigError):
        ctx.render(FIXTURES["cloud"]["scene"](), RenderOptions(n_paths=0))


# ---------------------------------------------------------------- K4/K5 on identical stores
MAPPINGS = {"wavefront": dict(mode=0, packet=1), "wavefront_p2": dict(mode=0, packet=2),
            "wavefront_p3": dict(mode=0, packet=3), "wavefront_p4": dict(mode=0, packet=4),
            "wavefront_guarded": dict(mode=0, packet=3, pad=0), "per_path": dict(mode=1, packet=1)}


@pytest.fixture(params=list(MAPPINGS))
def mode(ctx, request):
    """Every kernel mapping must meet the same parity bar."""
    for k, v in MAPPINGS[request.param].items():
        ctx.set_option(k, v)
    yield request.param
    ctx.set_option("mode", 0)
    ctx.set_option("packet", 3)
    ctx.set_option("pad", 1)


@pytest.mark.parametrize("name", list(FIXTURES))
@pytest.mark.parametrize("sort", [False, True])
def test_evaluate_matches_reference_on_its_store(ctx, golden_dir, name, sort, mode):
    scene = FIXTURES[name]["scene"]()
    g = golden(name)
    ctx.upload(scene)
    st = ctx.load_store(str(golden_dir / f"{name}.pstr"))
    if sort:
        ctx.sort_by_size(st)
    worst = [0.0, 0.0]
    for tag, params in (("ref", None), ("pert", perturbed(scene))):
        for wtag, w in weight_patterns(scene).items():
            r = ctx.evaluate_store(scene, st, params, EvalOptions(want_grad=True, pixel_weights=w))
            e_img = img_err(r.images, g[f"{tag}_{wtag}_images"])
            assert e_img <= IMG_TOL, (tag, wtag, e_img)
            worst[0] = max(worst[0], e_img)
            if scene.unknown_species() >= 0:
                e_g = grad_err(r.grad_beta, g[f"{tag}_{wtag}_grad"])
                assert e_g <= GRAD_TOL, (tag, wtag, e_g)
                worst[1] = max(worst[1], e_g)
            else:
                assert scalar_err(r.grad_kappa, float(g[f"{tag}_{wtag}_gk"])) <= GRAD_TOL
                assert scalar_err(r.grad_gamma, float(g[f"{tag}_{wtag}_gg"])) <= GRAD_TOL
            assert r.clamp_events == int(g[f"{tag}_{wtag}_clamps"])
        if scene.unknown_species() >= 0:
            r = ctx.evaluate_store(scene, st, params, EvalOptions(want_grad=True, legacy_score=True))
            assert grad_err(r.grad_beta, g[f"{tag}_legacy_grad"]) <= GRAD_TOL
    print(f"{name} sort={sort} mode={mode}: max image rel err {worst[0]:.2e}, max grad rel err {worst[1]:.2e}")


def test_per_type_gradients(ctx, golden_dir, mode):
    """Config (c): both species' gradients from one pass; each equals the reference's
    single-unknown gradient with that species flagged (SURVEY a15 flip oracle)."""
    scene = FIXTURES["tomo2"]["scene"]()
    flip = FIXTURES["tomo2"]["flip_unknown"]()
    g = golden("tomo2")
    ctx.upload(scene)
    st = ctx.load_store(str(golden_dir / "tomo2.pstr"))
    w = weight_patterns(scene)["w"]
    p0 = perturbed(scene)  # species 0 perturbed
    r = ctx.evaluate_store(scene, st, S.ParamSet(species_beta=[p0.beta, None]),
                           EvalOptions(want_grad=True, pixel_weights=w, per_species=True))
    assert grad_err(r.grad_beta[0], g["pert_w_grad"]) <= GRAD_TOL
    p1 = perturbed(flip)  # species 1 perturbed
    r = ctx.evaluate_store(scene, st, S.ParamSet(species_beta=[None, p1.beta]),
                           EvalOptions(want_grad=True, pixel_weights=w, per_species=True))
    assert img_err(r.images, g["flip_pert_w_images"]) <= IMG_TOL
    assert grad_err(r.grad_beta[1], g["flip_pert_w_grad"]) <= GRAD_TOL


@pytest.mark.parametrize("name", list(FIXTURES))
@pytest.mark.parametrize("materialized", [False, True])
@pytest.mark.parametrize("path_mode", [0, 1])
def test_self_normalize_matches_reference(ctx, ref, golden_dir, name, materialized, path_mode):
    """EvalOptions::self_normalize (pathstore.cpp:334-359): images and gradients divided by
    the mean correction_factor (pathstore.cpp:269-294, the escape segment's spans
    included) over the store, and that mean reported; against the reference's
    evaluate_store on its own store, recomputed and materialized imports."""
    scene = FIXTURES[name]["scene"]()
    ctx.set_option("mode", path_mode)
    ctx.upload(scene)
    pstr = str(golden_dir / f"{name}.pstr")
    st = ctx.load_store(pstr, materialized=materialized)
    w = weight_patterns(scene)["w"]
    p = perturbed(scene)
    flags = abi.PRC_EVAL_NORMALIZE | abi.PRC_EVAL_SELF_NORMALIZE | abi.PRC_EVAL_WANT_GRAD
    r = ref.evaluate(scene, pstr, p, flags, w)
    for _ in range(2):  # the second call reuses the cached forward
        g = ctx.evaluate_store(scene, st, p, EvalOptions(want_grad=True, pixel_weights=w, self_normalize=True))
        assert scalar_err(g.mean_correction, r["mean_correction"]) <= 1e-6, (g.mean_correction, r["mean_correction"])
        assert img_err(g.images, r["images"]) <= IMG_TOL
        if scene.unknown_species() >= 0:
            assert grad_err(g.grad_beta, r["grad"]) <= GRAD_TOL
        else:
            assert scalar_err(g.grad_kappa, r["grad_kappa"]) <= GRAD_TOL
            assert scalar_err(g.grad_gamma, r["grad_gamma"]) <= GRAD_TOL
    plain = ctx.evaluate_store(scene, st, p, EvalOptions())
    ctx.set_option("mode", 0)
    assert plain.mean_correction == 1.0
    assert np.allclose(plain.images / g.mean_correction, g.images, rtol=1e-12, atol=0.0)


def test_pstr_errors(ctx, tmp_path):
    ctx.upload(FIXTURES["tomo2"]["scene"]())
    p = tmp_path / "bad.pstr"
    p.write_bytes(b"XXXX????")
    with pytest.raises(PrcIOError, match="bad magic"):
        ctx.load_store(str(p))
    with pytest.raises(PrcIOError):
        ctx.load_store(str(tmp_path / "no_such_file.pstr"))


# ---------------------------------------------------------------- K1 trace
@pytest.mark.parametrize("name", list(FIXTURES))
def test_device_store_round_trip_through_reference_format(ctx, port, tmp_path, name, mode):
    """GPU-traced store -> PSTR (spans/events materialised on the device) -> oracle
    evaluates the identical stored path set; GPU evaluation agrees within 1e-5."""
    fx = FIXTURES[name]
    scene = fx["scene"]()
    ctx.upload(scene)
    rr = ctx.render(scene, RenderOptions(n_paths=fx["n"], seed=11, keep_paths=True,
                                         max_bounces=fx.get("max_bounces", 500)))
    st = rr.store
    ctx.sort_by_size(st)
    path = str(tmp_path / "gpu.pstr")
    st.save(path)
    ost = port.load(path)
    assert np.array_equal(ost.streams(), st.streams())
    assert np.array_equal(ost.sizes(), st.sizes())
    for params in (None, perturbed(scene)):
        w = weight_patterns(scene)["res"]
        a = ctx.evaluate_store(scene, st, params, EvalOptions(want_grad=True, pixel_weights=w))
        b = port.evaluate(scene, ost, params, abi.PRC_EVAL_NORMALIZE | abi.PRC_EVAL_WANT_GRAD, w)
        assert img_err(a.images, b["images"]) <= IMG_TOL
        if scene.unknown_species() >= 0:
            assert grad_err(a.grad_beta, b["grad"]) <= GRAD_TOL
        else:
            assert scalar_err(a.grad_kappa, b["grad_kappa"]) <= GRAD_TOL
    # fresh image == evaluation at the sampling point
    assert img_err(ctx.recycled_render(scene, st, None), rr.images) <= 1e-12


@pytest.mark.parametrize("name", list(FIXTURES))
def test_fresh_paths_follow_the_reference_sampler(ctx, port, name):
    """Same (seed, stream) Philox streams: device paths coincide with the reference's
    except where CUDA libm (log1p/sin/cos/cbrt/pow) rounds differently; the path-size
    histogram and the fresh image agree statistically."""
    fx = FIXTURES[name]
    scene = fx["scene"]()
    n = 4000
    mb = fx.get("max_bounces", 500)
    ctx.upload(scene)
    rr = ctx.render(scene, RenderOptions(n_paths=n, seed=21, keep_paths=True, max_bounces=mb))
    img_o, tr_o, st_o = port.render(scene, n, 21, max_bounces=mb)
    same = (rr.store.sizes() == st_o.sizes()).mean()
    assert same >= 0.97, same
    # image totals within 4 combined standard errors (per-path contributions)
    assert abs(rr.images.sum() - img_o.sum()) <= 0.02 * img_o.sum() + 1e-12


def test_truncation_and_event_cap(ctx):
    s = S.homogeneous_cube(80.0, 1.0, "rayleigh")
    ctx.upload(s)
    r = ctx.render(s, RenderOptions(n_paths=50, seed=3, max_bounces=2, keep_paths=True))
    assert r.truncated_paths > 0 and r.store.info()["truncated"] == r.truncated_paths
    s = S.homogeneous_cube(50.0, 0.9, "rayleigh")
    ctx.upload(s)
    r = ctx.render(s, RenderOptions(n_paths=200, seed=1, max_bounces=1000, max_scatter_events=1,
                                    keep_paths=True))
    assert r.truncated_paths == 0 and r.store.sizes().max() <= 2
    v = S.homogeneous_cube(0.0, 0.9)
    ctx.upload(v)
    r = ctx.render(v, RenderOptions(n_paths=500, seed=1))
    assert (r.images == 0).all() and r.truncated_paths == 0


def test_unbiased_recycling_against_fresh(ctx):
    """test_pathstore.cpp:152-170: recycled estimate at +15% tracks a fresh render."""
    s = S.two_species_cube(np.full(64, 4.0), 4, 0.04, 4, 4)
    ctx.upload(s)
    st = ctx.render(s, RenderOptions(n_paths=400_000, seed=29, keep_paths=True)).store
    t = S.ParamSet(np.full(64, 4.0 * 1.15))
    rec = ctx.recycled_render(s, st, t)
    s2 = S.two_species_cube(np.full(64, 4.0 * 1.15), 4, 0.04, 4, 4)
    ctx.upload(s2)
    fresh = ctx.render(s2, RenderOptions(n_paths=400_000, seed=877)).images
    assert np.abs(rec - fresh).sum() / fresh.sum() < 0.02


# ---------------------------------------------------------------- Algorithm 2
def test_adam_step_matches_restatement(ctx, golden_dir):
    """One device-resident iteration (K3-K6) vs numpy ADAM on the reference gradient."""
    scene = FIXTURES["tomo2"]["scene"]()
    g = golden("tomo2")
    ctx.upload(scene)
    st = ctx.load_store(str(golden_dir / "tomo2.pstr"))
    t = perturbed(scene)
    # gt such that residual = F_t - gt = "res" weights of the golden set
    Ft = g["pert_res_images"]
    res = weight_patterns(scene)["res"]
    gt = Ft - res
    alpha = 0.05
    ctx.opt_init(t, gt, alpha=alpha)
    loss = ctx.opt_step(st)
    assert abs(loss - 0.5 * (res ** 2).sum()) <= 1e-5 * loss
    grad = g["pert_res_grad"]
    m1 = 0.1 * grad
    m2 = 0.001 * grad * grad
    mhat, vhat = m1 / (1 - 0.9), m2 / (1 - 0.999)
    expect = np.maximum(t.beta - alpha * mhat / (np.sqrt(vhat) + 1e-8), 0.0)
    got = ctx.opt_params().beta
    # first ADAM step is alpha * g / (|g| + eps): a gradient error dg moves it by at most
    # alpha * 2 dg / (|g| + eps); dg is bounded by the 1e-5 scale-relative gradient bar.
    dg = GRAD_TOL * np.abs(grad).max()
    allow = alpha * 2.0 * dg / (np.abs(grad) + 1e-8) + 1e-12
    assert (np.abs(got - expect) <= allow).all()


def test_reconstruct_loop_runs_algorithm2(ctx, ref):
    """Algorithm 2 on the device: resample + sort every N_r, recycle otherwise; loss
    falls like the reference's loop on the same problem."""
    s = S.cloud_scene(8, 8, 8)
    truth = s.species[0].extinction.copy()
    ctx.upload(s)
    gt = ctx.render(s, RenderOptions(n_paths=200_000, seed=611)).images
    init = S.ParamSet(np.full(truth.size, truth.mean()))
    out = ctx.reconstruct(s, gt, init, n_paths=20_000, seed=271, recycle_period=10,
                          max_iterations=40, alpha=0.3)
    assert out["sampling_phases"] == 4
    loss = out["loss"]
    assert np.isfinite(loss).all() and loss[-1] < 0.75 * loss[0]
    r = ref.reconstruct(s, init, gt, alpha=0.3, seed=271, n_paths=20_000, recycle_period=10,
                        max_iterations=40, workers=os.cpu_count() or 1)
    assert r["sampling_phases"] == 4
    assert loss[-1] <= 2.0 * r["loss"][-1] + 1e-12 and r["loss"][-1] <= 2.0 * loss[-1] + 1e-12


def test_phong_reconstruct_moves_toward_truth(ctx):
    s = S.phong_box(0.7, 50.0, 16, 16, 0.3)
    ctx.upload(s)
    gt = ctx.render(s, RenderOptions(n_paths=400_000, seed=501, max_bounces=40)).images
    out = ctx.reconstruct(s, gt, S.ParamSet(None, 0.4, 25.0), n_paths=100_000, seed=733,
                          recycle_period=10, max_iterations=60, max_bounces=40, alpha=0.008,
                          step_scale=[2.0, 100.0])
    p = out["params"]
    assert abs(p.kappa_s - 0.7) < abs(0.4 - 0.7) and abs(p.gamma - 50.0) < abs(25.0 - 50.0)
    assert out["loss"][-1] < out["loss"][0]


def test_grad_forward_reuses_forward_cache_correctly(ctx, golden_dir):
    """recycled_render then grad_forward at the same point reuses the cached forward;
    any change of parameters, store layout or store invalidates it."""
    scene = FIXTURES["tomo2"]["scene"]()
    g = golden("tomo2")
    ctx.upload(scene)
    st = ctx.load_store(str(golden_dir / "tomo2.pstr"))
    w = weight_patterns(scene)["w"]
    p = perturbed(scene)
    f = ctx.evaluate_store(scene, st, p, EvalOptions())
    n0 = ctx.kernel_launches()
    r = ctx.evaluate_store(scene, st, p, EvalOptions(want_grad=True, pixel_weights=w))
    reused_launches = ctx.kernel_launches() - n0
    assert grad_err(r.grad_beta, g["pert_w_grad"]) <= GRAD_TOL
    assert np.array_equal(r.images, f.images)
    # different parameters: no reuse, still correct
    r2 = ctx.evaluate_store(scene, st, None, EvalOptions(want_grad=True, pixel_weights=w))
    assert grad_err(r2.grad_beta, g["ref_w_grad"]) <= GRAD_TOL
    n0 = ctx.kernel_launches()
    ctx.evaluate_store(scene, st, p, EvalOptions(want_grad=True, pixel_weights=w))
    assert ctx.kernel_launches() - n0 > reused_launches
    # sort invalidates
    ctx.evaluate_store(scene, st, p, EvalOptions())
    ctx.sort_by_size(st)
    r3 = ctx.evaluate_store(scene, st, p, EvalOptions(want_grad=True, pixel_weights=w))
    assert grad_err(r3.grad_beta, g["pert_w_grad"]) <= GRAD_TOL


def test_nccl_communicator_path(golden_dir):
    """A context built on an NCCL communicator (1 rank here: one GPU per gpurun box) runs
    the allreduce code path of K4/K5 and returns the same results."""
    from paper_2110_00085_b200.gpu import Context
    c = Context(0, 0, 1, Context.nccl_unique_id())
    scene = FIXTURES["tomo2"]["scene"]()
    g = golden("tomo2")
    c.upload(scene)
    st = c.load_store(str(golden_dir / "tomo2.pstr"))
    r = c.evaluate_store(scene, st, perturbed(scene),
                         EvalOptions(want_grad=True, pixel_weights=weight_patterns(scene)["w"]))
    assert img_err(r.images, g["pert_w_images"]) <= IMG_TOL
    assert grad_err(r.grad_beta, g["pert_w_grad"]) <= GRAD_TOL
    st.free()
    c.close()


# ---------------------------------------------------------------- statistical parity (fresh MC)
def test_recycling_unbiased_over_30_repetitions(ctx):
    """acceptance.cpp:277-325 (c5): +1% on one voxel; recycled estimate from a store traced
    at the reference vs a fresh render at the perturbed point, 30 independent repetitions
    at N = 1e6: the mean gap lies within 3 standard errors."""
    s = S.two_species_cube(np.full(64, 2.0), 4, 0.04, 8, 8)
    t = np.full(64, 2.0)
    t[21] *= 1.01
    st_scene = S.two_species_cube(t, 4, 0.04, 8, 8)
    n = 1_000_000
    diffs = []
    for r in range(30):
        ctx.upload(s)
        st = ctx.render(s, RenderOptions(n_paths=n, seed=10000 + r, keep_paths=True)).store
        rec = ctx.recycled_render(s, st, S.ParamSet(t)).sum()
        st.free()
        ctx.upload(st_scene)
        fresh = ctx.render(st_scene, RenderOptions(n_paths=n, seed=20000 + r)).images.sum()
        diffs.append(rec - fresh)
    d = np.asarray(diffs)
    sem = d.std(ddof=1) / np.sqrt(len(d))
    assert abs(d.mean()) <= 3.0 * sem, (d.mean(), sem)


def test_fresh_render_matches_reference_statistically(ctx, ref):
    """Fresh sampling parity against the reference sampler: independent seeds, image
    totals agree within 4 combined standard errors, per-pixel z-scores <= 5 for pixels
    above 1% of the maximum, and the path-size histograms agree (chi^2, p > 1e-3)."""
    from scipy import stats
    s = S.cloud_scene(8, 6, 6)
    ctx.upload(s)
    n, reps = 200_000, 8
    g = np.array([ctx.render(s, RenderOptions(n_paths=n, seed=1000 + r)).images for r in range(reps)])
    workers = os.cpu_count() or 1
    c = np.array([ref.render(s, n, 5000 + r, workers=workers)[0] for r in range(reps)])
    se = np.sqrt(g.sum(1).var(ddof=1) / reps + c.sum(1).var(ddof=1) / reps)
    assert abs(g.sum(1).mean() - c.sum(1).mean()) <= 4 * se
    mg, mc = g.mean(0), c.mean(0)
    sp = np.sqrt(g.var(0, ddof=1) / reps + c.var(0, ddof=1) / reps)
    big = mc > 0.01 * mc.max()
    assert (np.abs(mg - mc)[big] / np.maximum(sp[big], 1e-300)).max() <= 5.0
    # path-size (B) histograms: device store vs the reference sampler (C restatement)
    from pyoracle import Port
    st = ctx.render(s, RenderOptions(n_paths=n, seed=77, keep_paths=True)).store
    bg = np.bincount(st.sizes().astype(np.int64))
    _, _, ost = Port().render(s, n, 78)
    bc = np.bincount(ost.sizes().astype(np.int64))
    m = max(len(bg), len(bc))
    bg, bc = np.pad(bg, (0, m - len(bg))), np.pad(bc, (0, m - len(bc)))
    keep = (bg + bc) >= 10
    table = np.vstack([bg[keep], bc[keep]])
    assert stats.chi2_contingency(table)[1] > 1e-3


def test_recycling_speed_benefit(ctx):
    """acceptance.cpp:481-506 (c9): iterations per second with N_r = 30 are at least 2x
    those with N_r = 1 (resampling every iteration).  The reference runs c9 at 4e4 paths
    on the CPU, where tracing dominates either way; on the device at that size both loops
    are bound by per-iteration launch and synchronisation costs, so the check runs where
    the work per path counts: the config-(a) cloud (32^3, 9 x 64^2) at 2e6 paths, from an
    estimate near the truth (the resample traces under the current estimate, so a thin
    initial medium would make it cheap)."""
    import time
    s = S.cloud_scene(32, 64, 64)
    ctx.upload(s)
    gt = ctx.render(s, RenderOptions(n_paths=1_000_000, seed=612)).images
    init = S.ParamSet(0.9 * s.species[0].extinction)
    speed = {30: 0.0, 1: 0.0}
    for _ in range(2):  # best of two runs each: the box's other tenants add noise
        for nr in (30, 1):
            t0 = time.perf_counter()
            ctx.reconstruct(s, gt, init, n_paths=2_000_000, seed=41, recycle_period=nr, max_iterations=30,
                            alpha=0.02)
            speed[nr] = max(speed[nr], 30 / (time.perf_counter() - t0))
    print(f"recycling: {speed[30]:.1f} it/s with N_r = 30, {speed[1]:.1f} it/s with N_r = 1")
    assert speed[30] >= 2.0 * speed[1], speed


def test_large_grid_unpacked_dda_paths(ctx, port, tmp_path):
    """Grids wider than 512 voxels take the generic (unpacked) bounds check in every
    DDA user: trace, K4a/K5a stepper, K4b/K5b walks.  Parity against the oracle on the
    identical exported store, and bit-exact spans."""
    g = S.Grid((520, 4, 4), (0.0, 0.0, 0.0), (1.0 / 520, 0.25, 0.25))
    beta = 2.0 + np.sin(np.arange(g.voxel_count) * 0.01)
    s = S.Scene(grid=g, species=[S.Species(beta, 0.9, "hg", 0.6, True)],
                light=S.Light("point", (0.5, 0.5, 0.5), (0, 0, -1), 1.0),
                detectors=[S.top_detector(6, 6), S.Detector((2.5, 0.5, 0.5), (-1, 0, 0), (0, 0, 1), 5, 5, 0.7)])
    ctx.upload(s)
    rays = np.random.default_rng(9).uniform(0, 1, size=(500, 7))
    rays[:, 3:6] -= 0.5
    rays[:, 3:6] /= np.linalg.norm(rays[:, 3:6], axis=1, keepdims=True)
    rays[:, 6] *= 2.0
    c1, v1, l1 = ctx.debug_walk(rays)
    c2, v2, l2 = port.walk(s, rays)
    assert np.array_equal(c1, c2) and np.array_equal(v1, v2)
    assert np.array_equal(l1.view(np.uint64), l2.view(np.uint64))
    st = ctx.render(s, RenderOptions(n_paths=3000, seed=4, keep_paths=True)).store
    ctx.sort_by_size(st)
    st.save(str(tmp_path / "big.pstr"))
    ost = port.load(str(tmp_path / "big.pstr"))
    t = perturbed(s)
    w = np.linspace(-1.0, 2.0, s.pixel_count)
    a = ctx.evaluate_store(s, st, t, EvalOptions(want_grad=True, pixel_weights=w))
    b = port.evaluate(s, ost, t, abi.PRC_EVAL_NORMALIZE | abi.PRC_EVAL_WANT_GRAD, w)
    assert img_err(a.images, b["images"]) <= IMG_TOL
    assert grad_err(a.grad_beta, b["grad"]) <= GRAD_TOL


def test_opt_step_per_type_mode_matches_single_unknown(ctx, golden_dir):
    """Config (c): with per-type gradients on, the device iteration still moves the unknown
    species exactly as the single-unknown iteration does (its gradient is the same)."""
    scene = FIXTURES["tomo2"]["scene"]()
    g = golden("tomo2")
    ctx.upload(scene)
    st = ctx.load_store(str(golden_dir / "tomo2.pstr"))
    t = perturbed(scene)
    gt = g["pert_res_images"] - weight_patterns(scene)["res"]
    out = []
    for ps in (0, 1):
        ctx.set_option("per_species", ps)
        ctx.opt_init(t, gt, alpha=0.05)
        ctx.opt_step(st)
        out.append(ctx.opt_params().beta)
    ctx.set_option("per_species", 0)
    assert np.abs(out[0] - out[1]).max() <= 1e-9 + 1e-6 * 0.05


def test_event_geometry_cache_follows_the_cameras(ctx, golden_dir):
    """K4b caches each event's pixel and log(albedo f) per store (single-species scenes).
    A new camera set (scene upload) must invalidate it: evaluating a store after switching
    cameras equals evaluating it in a context that only ever saw the new cameras."""
    from paper_2110_00085_b200.gpu import Context
    a = S.cloud_scene(12, 10, 10)
    b = S.cloud_scene(12, 7, 9, n_ring=5, fov=0.7)
    ctx.upload(a)
    st = ctx.load_store(str(golden_dir / "cloud.pstr"))
    t = perturbed(a)
    for _ in range(2):  # build the cache, then use it
        ctx.evaluate_store(a, st, t, EvalOptions())
    ctx.upload(b)
    w = np.linspace(-1.0, 1.0, b.pixel_count)
    got = [ctx.evaluate_store(b, st, t, EvalOptions(want_grad=True, pixel_weights=w)) for _ in range(2)]
    fresh = Context(0)
    try:
        fresh.upload(b)
        st2 = fresh.load_store(str(golden_dir / "cloud.pstr"))
        ref = fresh.evaluate_store(b, st2, t, EvalOptions(want_grad=True, pixel_weights=w))
    finally:
        fresh.close()
    for r in got:
        assert img_err(r.images, ref.images) <= 1e-12
        assert grad_err(r.grad_beta, ref.grad_beta) <= 1e-12


@pytest.mark.parametrize("name", ["phong", "mixed"])
def test_surface_event_cache_reuse(ctx, golden_dir, name):
    """Scenes with surfaces: the first forward over a store caches each surface event's
    pixel, cos_le and geometry factor; later forwards and gradients (other kappa/gamma or
    beta) read them instead of redoing pixel_of and the visibility tests. Cached passes
    equal the pass that wrote the cache, and the reference's values at every point."""
    scene = FIXTURES[name]["scene"]()
    g = golden(name)
    w = weight_patterns(scene)["w"]
    p = perturbed(scene)
    ctx.upload(scene)
    st = ctx.load_store(str(golden_dir / f"{name}.pstr"))
    first = ctx.evaluate_store(scene, st, p, EvalOptions(want_grad=True, pixel_weights=w))
    ctx.evaluate_store(scene, st, None, EvalOptions())  # another point in between
    again = ctx.evaluate_store(scene, st, p, EvalOptions(want_grad=True, pixel_weights=w))
    assert img_err(again.images, first.images) <= 1e-12
    assert img_err(again.images, g["pert_w_images"]) <= IMG_TOL
    if scene.unknown_species() >= 0:
        assert grad_err(again.grad_beta, first.grad_beta) <= 1e-12
        assert grad_err(again.grad_beta, g["pert_w_grad"]) <= GRAD_TOL
    else:
        assert scalar_err(again.grad_kappa, first.grad_kappa) <= 1e-12
        assert scalar_err(again.grad_gamma, first.grad_gamma) <= 1e-12
        assert scalar_err(again.grad_kappa, float(g["pert_w_gk"])) <= GRAD_TOL
        assert scalar_err(again.grad_gamma, float(g["pert_w_gg"])) <= GRAD_TOL


def test_gradient_copies_option_same_results(ctx, golden_dir):
    """K5b's reductions into 1 or 4 copies of the padded gradient give the same gradient
    up to the order of floating-point sums."""
    scene = FIXTURES["cloud"]["scene"]()
    w = weight_patterns(scene)["res"]
    out = []
    for copies in (1, 4):
        ctx.set_option("grad_copies", copies)
        ctx.upload(scene)
        st = ctx.load_store(str(golden_dir / "cloud.pstr"))
        out.append(ctx.evaluate_store(scene, st, perturbed(scene), EvalOptions(want_grad=True, pixel_weights=w)))
    ctx.set_option("grad_copies", 0)
    ctx.upload(scene)
    assert img_err(out[1].images, out[0].images) <= 1e-12
    assert grad_err(out[1].grad_beta, out[0].grad_beta) <= 1e-12


def test_store_outlives_its_context(golden_dir):
    """Stores belong to their context (another context gets PRC_ERR_INVALID) and can be
    freed after the context is destroyed (the C ABI orphans them instead of dangling)."""
    from paper_2110_00085_b200.gpu import Context, PrcInvalidError
    scene = FIXTURES["cloud"]["scene"]()
    a, b = Context(0), Context(0)
    try:
        a.upload(scene)
        b.upload(scene)
        st = a.load_store(str(golden_dir / "cloud.pstr"))
        with pytest.raises(PrcInvalidError):
            b.evaluate_store(scene, st, None, EvalOptions())
        a.close()
        with pytest.raises(PrcInvalidError):
            st.sizes()
        st.free()  # no use-after-free of the destroyed context
        st2 = b.load_store(str(golden_dir / "cloud.pstr"))
        assert b.evaluate_store(scene, st2, None, EvalOptions()).images.sum() > 0
    finally:
        a.close()
        b.close()


def test_store_rejects_a_scene_with_another_grid(ctx, golden_dir):
    """A store's voxel ids index the grid it was built under; evaluating it against a
    scene with another grid is refused instead of reading out of bounds."""
    from paper_2110_00085_b200.gpu import PrcInvalidError
    scene = FIXTURES["cloud"]["scene"]()
    ctx.upload(scene)
    st = ctx.load_store(str(golden_dir / "cloud.pstr"))
    other = S.cloud_scene(8, 10, 10)
    with pytest.raises(PrcInvalidError):
        ctx.evaluate_store(other, st, None, EvalOptions())
    ctx.upload(scene)
    assert ctx.evaluate_store(scene, st, None, EvalOptions()).images.sum() > 0


def test_store_reference_side_follows_the_scene(ctx, ref, golden_dir):
    """make_context (pathstore.cpp:41-82) builds the reference side of every known
    species from the current scene on each call.  A re-uploaded scene whose known species
    changed must therefore change the store's reference tables too."""
    scene = FIXTURES["tomo2"]["scene"]()
    ctx.upload(scene)
    st = ctx.load_store(str(golden_dir / "tomo2.pstr"))
    ctx.evaluate_store(scene, st, None, EvalOptions())
    s2 = FIXTURES["tomo2"]["scene"]()
    s2.species[1].extinction = s2.species[1].extinction * 1.3  # the known species
    w = weight_patterns(s2)["w"]
    p = perturbed(s2)
    r = ctx.evaluate_store(s2, st, p, EvalOptions(want_grad=True, pixel_weights=w))
    e = ref.evaluate(s2, str(golden_dir / "tomo2.pstr"), p, abi.PRC_EVAL_NORMALIZE | abi.PRC_EVAL_WANT_GRAD, w)
    assert img_err(r.images, e["images"]) <= IMG_TOL
    assert grad_err(r.grad_beta, e["grad"]) <= GRAD_TOL


def test_import_range_checks_voxel_ids(ctx, golden_dir, tmp_path):
    """load_store: a vertex voxel id outside the uploaded grid is an I/O error, not an
    out-of-bounds gather in the kernels."""
    import struct
    scene = FIXTURES["cloud"]["scene"]()
    ctx.upload(scene)
    raw = bytearray((golden_dir / "cloud.pstr").read_bytes())
    nb = struct.unpack_from("<Q", raw, 33)[0]
    rec0 = 41 + 8 * nb + 16
    vox_at = rec0 + 8 + 1 + 24 + 4 + 56  # record 0, vertex 0, VertexRec::voxel
    struct.pack_into("<i", raw, vox_at, scene.voxel_count + 5)
    bad = tmp_path / "bad_vox.pstr"
    bad.write_bytes(bytes(raw))
    with pytest.raises(PrcIOError, match="voxel"):
        ctx.load_store(str(bad))


def test_render_is_bit_reproducible(ctx):
    """render() is bit-reproducible for fixed (seed, n_paths) (transport.hpp:171-173): the
    fresh image is summed in exact 128-bit fixed point, so the order of the device atomics
    does not matter.  The deterministic recycled evaluation agrees with the fp64-atomic one
    to rounding, and is itself reproducible."""
    s = S.cloud_scene(16, 12, 12)
    ctx.upload(s)
    a = ctx.render(s, RenderOptions(n_paths=200_000, seed=5, keep_paths=True))
    b = ctx.render(s, RenderOptions(n_paths=200_000, seed=5))
    assert np.array_equal(a.images.view(np.uint64), b.images.view(np.uint64))
    t = perturbed(s)
    d1 = ctx.evaluate_store(s, a.store, t, EvalOptions(deterministic=True)).images
    d2 = ctx.evaluate_store(s, a.store, t, EvalOptions(deterministic=True)).images
    f = ctx.evaluate_store(s, a.store, t, EvalOptions()).images
    assert np.array_equal(d1.view(np.uint64), d2.view(np.uint64))
    assert img_err(d1, f) <= 1e-13
    assert img_err(ctx.recycled_render(s, a.store, None), a.images) <= 1e-13


def test_many_cameras_and_surfaces(ctx, ref, tmp_path):
    """More than 32 cameras and surfaces (the engine's inline scene holds up to 64 of
    each): a device-traced store evaluates like the reference's evaluate_store."""
    s = S.cloud_scene(8, 6, 6, n_ring=43)  # 44 cameras
    rng = np.random.default_rng(8)
    s.surfaces = [S.Surface("sphere", center=tuple(0.15 + 0.7 * rng.random(3)), radius=0.02, brdf="diffuse",
                            albedo=0.5) for _ in range(40)]
    assert len(s.detectors) > 32 and len(s.surfaces) > 32
    ctx.upload(s)
    st = ctx.render(s, RenderOptions(n_paths=4000, seed=5, keep_paths=True)).store
    ctx.sort_by_size(st)
    st.save(str(tmp_path / "many.pstr"))
    t = perturbed(s)
    w = np.linspace(-1.0, 2.0, s.pixel_count)
    a = ctx.evaluate_store(s, st, t, EvalOptions(want_grad=True, pixel_weights=w))
    b = ref.evaluate(s, str(tmp_path / "many.pstr"), t, abi.PRC_EVAL_NORMALIZE | abi.PRC_EVAL_WANT_GRAD, w)
    assert img_err(a.images, b["images"]) <= IMG_TOL
    assert grad_err(a.grad_beta, b["grad"]) <= GRAD_TOL
    with pytest.raises(PrcConfigError):
        ctx.upload(S.cloud_scene(8, 4, 4, n_ring=64))  # 65 cameras


def test_render_without_images_traces_only(ctx):
    """prc_gpu_render with images NULL (reconstruct's resample): the same store, no fresh
    evaluation."""
    s = S.cloud_scene(12, 10, 10)
    ctx.upload(s)
    a = ctx.render(s, RenderOptions(n_paths=30_000, seed=9, keep_paths=True))
    n0 = ctx.kernel_launches()
    b = ctx.render(s, RenderOptions(n_paths=30_000, seed=9, keep_paths=True, images=False))
    assert b.images is None
    assert np.array_equal(a.store.sizes(), b.store.sizes()) and a.truncated_paths == b.truncated_paths
    assert img_err(ctx.recycled_render(s, b.store, None), a.images) <= 1e-12
    assert ctx.kernel_launches() - n0 > 0


def test_concurrent_calls_on_one_context_are_serialised(ctx, golden_dir):
    """Calls on one context are serialised by the context (SURVEY §8(b) threading): four
    host threads evaluating through the same context get the single-thread results."""
    import threading
    scene = FIXTURES["tomo2"]["scene"]()
    ctx.upload(scene)
    st = ctx.load_store(str(golden_dir / "tomo2.pstr"))
    w = weight_patterns(scene)["w"]
    params = [perturbed(scene), None]
    want = [ctx.evaluate_store(scene, st, p, EvalOptions(want_grad=True, pixel_weights=w)) for p in params]
    out, errs = {}, []

    def run(k):
        try:
            for it in range(5):
                out[(k, it)] = ctx.evaluate_store(scene, st, params[k % 2], EvalOptions(want_grad=True, pixel_weights=w))
        except Exception as e:  # noqa: BLE001
            errs.append(e)
    th = [threading.Thread(target=run, args=(k,)) for k in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for (k, it), r in out.items():
        assert img_err(r.images, want[k % 2].images) <= 1e-12
        assert grad_err(r.grad_beta, want[k % 2].grad_beta) <= 1e-12


@pytest.mark.parametrize("name", ["phong", "reflectometry"])
def test_event_list_equals_dense_cache(ctx, golden_dir, name):
    """Scenes without a medium evaluate over the compact event list (K4b' / K5b') once the
    first forward over a store has written the dense event cache.  Event values are the
    same expression in the same order, so deterministic images are bit-identical to the
    dense kernels' and the Phong gradient differs only in the order of its sums; the list
    is rebuilt after a re-sort (new vertex-table order) and after a camera change."""
    if name == "phong":
        scene = FIXTURES["phong"]["scene"]()
    else:
        scene = S.reflectometry_scene(24, 24, 6)
    w = np.linspace(-1.0, 1.0, scene.pixel_count)
    p = perturbed(scene)
    opts = EvalOptions(want_grad=True, pixel_weights=w, deterministic=True)
    out = {}
    for ev in (0, 1):
        ctx.set_option("events", ev)
        ctx.upload(scene)
        if name == "phong":
            st = ctx.load_store(str(golden_dir / "phong.pstr"))
        else:
            st = ctx.render(scene, RenderOptions(n_paths=20000, seed=11, keep_paths=True)).store
        runs = [ctx.evaluate_store(scene, st, p, opts) for _ in range(3)]
        ctx.sort_by_size(st)
        runs += [ctx.evaluate_store(scene, st, p, opts) for _ in range(2)]
        st.free()
        out[ev] = runs
    ctx.set_option("events", 1)
    ref = out[0][0]
    assert ref.images.max() > 0.0
    for r in out[0] + out[1]:
        assert np.array_equal(r.images, ref.images)
        assert r.clamp_events == ref.clamp_events
        assert scalar_err(r.grad_kappa, ref.grad_kappa) <= 1e-12
        assert scalar_err(r.grad_gamma, ref.grad_gamma) <= 1e-12
    if name == "phong":
        g = golden("phong")
        r = ctx.evaluate_store(scene, ctx.load_store(str(golden_dir / "phong.pstr")), p,
                               EvalOptions(want_grad=True, pixel_weights=weight_patterns(scene)["w"]))
        assert img_err(r.images, g["pert_w_images"]) <= IMG_TOL


def test_block_cache_reuse_across_store_generations(ctx):
    """Freed stores' device blocks are reused by the next generation (the recycling loop's
    resample); a store on reused blocks evaluates exactly like one on fresh memory, and
    the cache can be handed back to the driver."""
    from paper_2110_00085_b200 import gpu
    from paper_2110_00085_b200.gpu import Context
    s = S.cloud_scene(16, 12, 12)
    ctx.upload(s)
    t = S.ParamSet(S.recycle_point(s.species[0].extinction))
    opt = EvalOptions(want_grad=True, deterministic=True)
    for seed in (5, 6):  # generation 2 lands on generation 1's blocks
        st = ctx.render(s, RenderOptions(n_paths=200_000, seed=seed, keep_paths=True)).store
        ctx.sort_by_size(st)
        got = ctx.evaluate_store(s, st, t, opt)
        st.free()
    gpu.release_cached_memory()
    fresh = Context(0)
    try:
        fresh.upload(s)
        st = fresh.render(s, RenderOptions(n_paths=200_000, seed=6, keep_paths=True)).store
        fresh.sort_by_size(st)
        ref = fresh.evaluate_store(s, st, t, opt)
    finally:
        fresh.close()
    assert np.array_equal(got.images, ref.images)
    assert grad_err(got.grad_beta, ref.grad_beta) <= 1e-12


@pytest.mark.parametrize("name", ["cloud", "phong"])
def test_ragged_store_sizes(ctx, name):
    """Stores whose path and vertex counts are not multiples of a warp, a ray packet (3) or
    the event list's 4 events per thread: the recycled image at the sampling point equals
    the fresh render (pathstore.cpp:370-375 vs transport.cpp:405-454) bit for bit with
    deterministic sums, through the cached-geometry passes as well."""
    scene = FIXTURES[name]["scene"]()
    ctx.upload(scene)
    for n in (1, 2, 3, 5, 31, 33, 97, 1001):
        rr = ctx.render(scene, RenderOptions(n_paths=n, seed=17 + n, keep_paths=True,
                                             max_bounces=FIXTURES[name].get("max_bounces", 500)))
        st = rr.store
        ctx.sort_by_size(st)
        for _ in range(2):  # the second pass reads the event caches / the event list
            r = ctx.evaluate_store(scene, st, None, EvalOptions(deterministic=True))
            assert np.array_equal(r.images, rr.images), (name, n)
        st.free()


def test_correction_factors_known_answers(ctx, tmp_path):
    """correction_factor (pathstore.cpp:269-294) on the device, the reference's own test
    cases (test_pathstore.cpp:29-85) on a homogeneous HG cube: exactly 1 at the sampling
    parameters; c^B exp(-(c-1) beta L) under uniform scaling by c (B volume scatters, L the
    path's length through the grid, from the exported spans; the device keeps the
    per-voxel fields in fp32, so 1e-6 instead of the reference's 1e-9); exactly 1 when
    only a voxel the path never crosses changes; 0 when a scatter vertex's extinction
    vanishes."""
    from tests.pstr import read as read_pstr
    s = S.homogeneous_cube(3.0, 0.9, "hg", 0.5, grid_n=4)
    s.species[0].unknown = True
    ctx.upload(s)
    st = ctx.render(s, RenderOptions(n_paths=400, seed=7, keep_paths=True, max_bounces=200)).store
    pstr = str(tmp_path / "c.pstr")
    st.save(pstr)
    recs = {int(r["stream"]): r for r in read_pstr(pstr)["records"]}
    order = [recs[int(k)] for k in st.streams()]
    uref = np.full(64, 3.0)
    f1 = ctx.correction_factors(s, st, S.ParamSet(uref))
    assert np.all(f1 == 1.0)
    c = 1.3
    fc = ctx.correction_factors(s, st, S.ParamSet(uref * c))
    for f, rec in zip(fc, order):
        n_scat = int(np.sum(rec["vertices"]["kind"] == 1))
        L = float(rec["spans"]["length"].sum())
        expected = c ** n_scat * np.exp(-(c - 1.0) * 3.0 * L)
        assert abs(f - expected) <= 1e-6 * expected, (f, expected)
    checked = killed = 0
    for i, rec in enumerate(order[:60]):
        touched = set(int(v) for v in rec["spans"]["voxel"]) | set(int(v) for v in rec["le_spans"]["voxel"])
        free = [v for v in range(64) if v not in touched]
        if free:
            t = uref.copy()
            t[free[0]] *= 5.0
            assert ctx.correction_factors(s, st, S.ParamSet(t))[i] == 1.0
            checked += 1
        scat = [int(v["voxel"]) for v in rec["vertices"] if v["kind"] == 1]
        if scat and killed < 5:
            t = uref.copy()
            t[scat[-1]] = 0.0
            assert ctx.correction_factors(s, st, S.ParamSet(t))[i] == 0.0
            killed += 1
    assert checked > 0 and killed > 0


def test_engine_options_validated(ctx):
    """Context knobs (include/pathrec_gpu.h): out-of-range values and unknown keys are
    PRC_ERR_CONFIG, valid ones are accepted (and restored)."""
    for key, bad in (("mode", 2), ("packet", 0), ("packet", 5), ("spread", -1), ("spread", 5000),
                     ("grad_copies", 65), ("nvls", 3), ("no_such_option", 1)):
        with pytest.raises(PrcConfigError):
            ctx.set_option(key, bad)
    for key, good, default in (("spread", 0, 0), ("spread", 16, 0), ("events", 0, 1), ("grad_copies", 4, 0),
                               ("packet", 2, 3), ("pad", 0, 1)):
        ctx.set_option(key, good)
        ctx.set_option(key, default)
