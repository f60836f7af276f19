"""The Algorithm-2 driver around the recycled loop: stage
schedule, downsample_images, space_carve, eps/delta metrics, VGRD and CSV checkpoints
(inverse.cpp:69-263, io.cpp:32-76, 147-155).

CPU tests pin the host utilities bit-for-bit against the reference library
(oracle/_ref); GPU tests run the device carve and the staged loop through the C ABI."""
import os

import numpy as np
import pytest

from tests.fixtures import FIXTURES, golden
from paper_2110_00085_b200 import gpu
from paper_2110_00085_b200 import scene as S
from paper_2110_00085_b200.gpu import RenderOptions


# ------------------------------------------------------------------ host utilities (CPU)
def test_metrics_match_reference(ref):
    rng = np.random.default_rng(5)
    for n in (1, 7, 4096):
        t = rng.normal(size=n)
        e = t + 0.1 * rng.normal(size=n)
        assert gpu.metrics(e, t) == ref.metrics(e, t)
    with pytest.raises(gpu.PrcConfigError):
        gpu.metrics(np.ones(3), np.zeros(3))  # zero-norm truth, as inverse.cpp:111


@pytest.mark.parametrize("shape,out", [((64, 64), (32, 32)), ((48, 64), (20, 30)), ((16, 16), (16, 16)),
                                       ((7, 5), (3, 2))])
def test_downsample_images_match_reference(ref, shape, out):
    rng = np.random.default_rng(6)
    ims = [rng.uniform(size=shape) for _ in range(3)]
    a = gpu.downsample_images(ims, *out)
    b = ref.downsample(ims, *out)
    for x, y in zip(a, b):
        assert np.array_equal(x.view(np.uint64), y.view(np.uint64))
    assert np.isclose(sum(x.sum() for x in a), sum(im.sum() for im in ims))  # block sums keep mass


def test_vgrd_bytes_match_reference(ref, tmp_path):
    rng = np.random.default_rng(7)
    dims, org, vs = (5, 4, 3), (-0.5, 0.25, 1.0), (0.1, 0.2, 0.3)
    vals = rng.uniform(0, 30, size=int(np.prod(dims)))
    for unit in (0, 1):
        ours, theirs = tmp_path / f"a{unit}.vgrd", tmp_path / f"b{unit}.vgrd"
        gpu.save_grid(str(ours), dims, org, vs, vals, unit)
        ref.save_grid(str(theirs), dims, org, vs, vals, unit)
        assert ours.read_bytes() == theirs.read_bytes()
        g = gpu.load_grid(str(theirs))
        assert g["dims"] == dims and g["origin"] == org and g["voxel_size"] == vs and g["unit"] == unit
        assert np.array_equal(g["values"], vals.astype(np.float32).astype(np.float64))


def test_vgrd_reader_errors(tmp_path):
    bad = tmp_path / "bad.vgrd"
    bad.write_bytes(b"VGRX" + b"\0" * 64)
    with pytest.raises(gpu.PrcIOError, match="bad magic"):
        gpu.load_grid(str(bad))
    gpu.save_grid(str(bad), (2, 2, 2), (0, 0, 0), (1, 1, 1), np.ones(8))
    bad.write_bytes(bad.read_bytes()[:-4])
    with pytest.raises(gpu.PrcIOError, match="truncated"):
        gpu.load_grid(str(bad))
    with pytest.raises(gpu.PrcIOError, match="cannot open"):
        gpu.load_grid(str(tmp_path / "missing.vgrd"))


# ------------------------------------------------------------------ device (B200)
@pytest.mark.gpu
@pytest.mark.parametrize("name", ["cloud", "cloud16_random", "cloud32_smooth"])
def test_space_carve_matches_reference(ctx, ref, name):
    """Visual hull on the device: voxel centres through the bit-exact pixel_of against
    per-view thresholds; identical masks and initial fields."""
    if name == "cloud":
        scene, gt = FIXTURES["cloud"]["scene"](), golden("cloud")["ref_none_images"]
    elif name == "cloud16_random":
        scene = S.cloud_scene(16, 24, 24)
        gt = np.random.default_rng(8).uniform(size=scene.pixel_count)
    else:  # smooth blob per view: a non-trivial hull
        scene = S.cloud_scene(32, 32, 32)
        r, c = np.meshgrid(np.arange(32), np.arange(32), indexing="ij")
        blob = np.exp(-((r - 15.5) ** 2 + (c - 15.5) ** 2) / 60.0).reshape(-1)
        gt = np.concatenate([blob * (1 + 0.1 * k) for k in range(len(scene.detectors))])
    for thr in (0.0, 0.05, 0.3):
        m1, b1 = ctx.space_carve(scene, gt, thr, 2.5)
        m2, b2 = ref.space_carve(scene, gt, thr, 2.5)
        assert np.array_equal(m1, m2) and np.array_equal(b1, b2)


@pytest.mark.gpu
def test_space_carve_errors(ctx):
    s = S.cloud_scene(8, 8, 8)
    one = S.Scene(grid=s.grid, species=s.species, light=s.light, detectors=s.detectors[:1])
    with pytest.raises(gpu.PrcInvalidError):
        ctx.space_carve(one, np.ones(one.pixel_count), 0.1, 1.0)


@pytest.mark.gpu
def test_reconstruct_schedule_stages_metrics_checkpoints(ctx, ref, tmp_path):
    """Two-stage coarse-to-fine schedule (inverse.cpp:154-263): the coarse stage runs at
    8x8 pixels on the block-summed ground truth, saturates, and the fine stage is applied
    at the next resample boundary; eps/delta follow the unknowns; checkpoints are VGRD
    and the reference's CSV layout, byte for byte."""
    s = S.cloud_scene(8, 16, 16)
    truth = s.species[0].extinction.copy()
    ctx.upload(s)
    n_pix = s.pixel_count
    gt = ctx.render(s, RenderOptions(n_paths=200_000, seed=611)).images
    init = S.ParamSet(np.full(truth.size, truth.mean()))
    out = ctx.reconstruct_schedule(s, gt, init, stages=[(8, 8, 20_000), (0, 0, 20_000)], seed=271,
                                   recycle_period=5, max_iterations=30, alpha=0.3, saturation_window=4,
                                   saturation_rel_improvement=1.0, checkpoint_every=10,
                                   checkpoint_dir=str(tmp_path), length_unit=1, truth=S.ParamSet(truth))
    h = out["history"]
    assert list(h["iter"]) == list(range(30))
    assert out["sampling_phases"] == 6
    # rel = 1.0 saturates as soon as the window is full: stage 1 from the first resample
    # boundary at or after iteration 4, i.e. 5
    assert list(h["stage"]) == [0] * 5 + [1] * 25
    assert np.isfinite(h["loss"]).all() and (np.diff(h["time_s"]) >= 0).all()
    # eps/delta of the unknowns before each update; the first row is the initial field
    e0, d0 = gpu.metrics(init.beta, truth)
    assert h["eps"][0] == e0 and h["delta"][0] == d0
    assert h["eps"][-1] < h["eps"][0]
    # checkpoints after iterations 9, 19, 29
    for t in (9, 19, 29):
        g = gpu.load_grid(str(tmp_path / f"checkpoint_{t}.vgrd"))
        assert g["dims"] == tuple(s.grid.dims) and g["unit"] == 1
        assert (g["values"] >= 0).all() and np.isfinite(g["values"]).all()
    ref.save_csv(str(tmp_path / "ref.csv"), h)
    assert (tmp_path / "loss.csv").read_bytes() == (tmp_path / "ref.csv").read_bytes()
    # the scene's resolution is back: a plain evaluation at full resolution still works
    assert ctx.render(s, RenderOptions(n_paths=1000, seed=1)).images.size == n_pix
    final = out["params"].beta
    assert gpu.metrics(final, truth)[0] < e0


@pytest.mark.gpu
def test_reconstruct_schedule_single_stage_equals_reconstruct(ctx):
    """With one stage and no saturation the schedule is the plain loop (same seeds, same
    sampling phases, same losses)."""
    s = S.cloud_scene(8, 8, 8)
    ctx.upload(s)
    gt = ctx.render(s, RenderOptions(n_paths=100_000, seed=3)).images
    init = S.ParamSet(np.full(s.voxel_count, s.species[0].extinction.mean()))
    a = ctx.reconstruct(s, gt, init, n_paths=10_000, seed=9, recycle_period=4, max_iterations=12, alpha=0.3)
    b = ctx.reconstruct_schedule(s, gt, init, stages=[(0, 0, 10_000)], seed=9, recycle_period=4,
                                 max_iterations=12, alpha=0.3)
    assert a["sampling_phases"] == b["sampling_phases"] == 3
    np.testing.assert_allclose(b["history"]["loss"], a["loss"], rtol=1e-9)
    np.testing.assert_allclose(b["params"].beta, a["params"].beta, rtol=1e-9, atol=1e-12)


@pytest.mark.gpu
def test_reconstruct_schedule_rejects_bad_schedules(ctx):
    s = S.cloud_scene(8, 8, 8)
    ctx.upload(s)
    gt = np.ones(s.pixel_count)
    with pytest.raises(gpu.PrcConfigError):
        ctx.reconstruct_schedule(s, gt, None, stages=[], max_iterations=2)
    with pytest.raises(gpu.PrcConfigError):
        ctx.reconstruct_schedule(s, gt, None, stages=[(8, 8, 0)], max_iterations=2)


# ---------------------------------------------------------------- a14: the optimizer itself
@pytest.mark.gpu
@pytest.mark.parametrize("nonneg", [True, False])
def test_adam_step_bit_identical_to_reference(ctx, ref, nonneg):
    """K6 (k_adam) against the reference's adam_step (inverse.cpp:41-67) over 7 updates
    with the same gradients: per-unknown step_scale (shorter than the unknowns), the
    non-negativity projection (gradients push some voxels below zero), zero gradients."""
    from tests.fixtures import FIXTURES, golden, perturbed
    scene = FIXTURES["tomo2"]["scene"]()
    g = golden("tomo2")["pert_res_grad"]
    x0 = perturbed(scene).beta
    rng = np.random.default_rng(5)
    grads = np.stack([g * s for s in (1.0, -3.0, 0.5, 40.0, 0.0, -1.0, 7.0)])
    grads[:, ::17] = 0.0
    grads[3] += rng.normal(size=g.size) * np.abs(g).max()
    ss = np.linspace(0.5, 2.0, g.size // 2)
    ctx.upload(scene)
    ctx.opt_init(S.ParamSet(x0), np.zeros(scene.pixel_count), alpha=1.5, project_nonneg=nonneg, step_scale=ss)
    want = ref.adam(x0, grads, 1.5, nonneg=nonneg, step_scale=ss)
    assert (want < 0).any() != nonneg and (want == 0).any() == nonneg
    for k in range(len(grads)):
        ctx.opt_adam_step(grads[k])
        got = ctx.opt_params().beta
        assert np.array_equal(got.view(np.uint64), want[k].view(np.uint64)), k


@pytest.mark.gpu
def test_adam_step_phong_clamp_bit_identical_to_reference(ctx, ref):
    """Reflectometry unknowns (kappa_s, gamma) with step_scale [2, 100] and gradients that
    drive kappa_s past 1 and below 0 and gamma below 0: the reference clamps kappa_s to
    [0, 1] and gamma to >= 0 after every update."""
    from tests.fixtures import FIXTURES
    scene = FIXTURES["phong"]["scene"]()
    grads = np.array([[-5.0, -2.0], [-5.0, 3.0], [8.0, 1.0], [9.0, 1.0], [9.0, 4.0], [0.0, 0.0], [-1e-3, -50.0]])
    x0 = np.array([0.8, 0.5])
    ctx.upload(scene)
    ctx.opt_init(S.ParamSet(None, x0[0], x0[1]), np.zeros(scene.pixel_count), alpha=0.3, step_scale=[2.0, 100.0])
    want = ref.adam(x0, grads, 0.3, step_scale=[2.0, 100.0], phong=True)
    assert want[:, 0].max() == 1.0 and want[:, 0].min() == 0.0 and want[:, 1].min() == 0.0 < want[-1, 1]
    for k in range(len(grads)):
        ctx.opt_adam_step(grads[k])
        p = ctx.opt_params()
        got = np.array([p.kappa_s, p.gamma])
        assert np.array_equal(got.view(np.uint64), want[k].view(np.uint64)), (k, got, want[k])


@pytest.mark.gpu
def test_device_loss_matches_reference_loss(ctx, ref, golden_dir):
    """The loss K6 reduces on the device (k_loss_residual) is the reference's loss()
    (inverse.cpp:11-23) of the same images, up to summation order."""
    from tests.fixtures import FIXTURES, golden, perturbed
    scene = FIXTURES["cloud"]["scene"]()
    ctx.upload(scene)
    st = ctx.load_store(str(golden_dir / "cloud.pstr"))
    gt = 0.8 * golden("cloud")["ref_none_images"]
    ctx.opt_init(perturbed(scene), gt, alpha=1e-3)
    for _ in range(3):
        loss = ctx.opt_step(st)
        F = ctx.opt_images()
        assert abs(loss - ref.loss(scene, F, gt)) <= 1e-14 * loss


@pytest.mark.gpu
@pytest.mark.parametrize("window,rel", [(0, 0.01), (3, 1e9), (2, -1e9)])
def test_schedule_decisions_match_reference(ctx, ref, window, rel):
    """Stage application and saturation (inverse.cpp:175-189, 249-258) decided exactly as
    the reference decides them: a window of 0 saturates at the first check, a huge relative
    threshold as soon as the window is full, a negative one never.  Stages change only at
    resample boundaries; the per-iteration stage sequence and the sampling-phase count
    equal the reference loop's on the same problem, and the losses track it."""
    import os
    s = S.cloud_scene(8, 16, 16)
    ctx.upload(s)
    gt = ctx.render(s, RenderOptions(n_paths=100_000, seed=611)).images
    init = S.ParamSet(np.full(s.voxel_count, s.species[0].extinction.mean()))
    stages = [(4, 4, 10_000), (8, 8, 10_000), (16, 16, 10_000)]
    out = ctx.reconstruct_schedule(s, gt, init, stages=stages, seed=33, recycle_period=3, max_iterations=20,
                                   alpha=0.3, saturation_window=window, saturation_rel_improvement=rel)
    r = ref.reconstruct_schedule(s, init, gt, 0.3, 33, stages, 3, 20, window, rel, workers=os.cpu_count() or 1)
    assert list(out["history"]["stage"]) == list(r["stage"])
    assert out["sampling_phases"] == r["sampling_phases"]
    lo, lr = out["history"]["loss"], r["loss"]
    assert np.all(np.abs(lo - lr) <= 0.05 * lr + 1e-30), np.c_[lo, lr]
    print(f"window {window} rel {rel:g}: stages {list(r['stage'])}")
