"""NVLS multicast reduction fused into the K4 / K5 epilogues.

Option "nvls": the images and the gradient are summed over ranks by `multimem.red.add`
into a multicast buffer (NCCL symmetric window with NVLS multimem for >= 2 ranks, a CUDA
multicast object on one device for a single rank) instead of ncclAllReduce; the gradient
fold also replaces k_unpad_add and k_combine.  Results must equal the NCCL path's.
"""
import os

import numpy as np
import pytest

from paper_2110_00085_b200.gpu import Context, EvalOptions, PrcError
from tests.fixtures import FIXTURES, golden, perturbed, weight_patterns

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def _nvls_ctx(scene, mode):
    c = Context(0)
    c.set_option("nvls", mode)
    try:
        c.upload(scene)
    except PrcError as e:
        c.close()
        pytest.skip(f"no multicast on this system: {e}")
    return c


# mode 1: a CUDA multicast object on this device (multimem.red); mode 2: the same fold
# kernels into a plain buffer (validates the fold's arithmetic where no multicast exists)
@pytest.fixture(params=[1, 2], ids=["multicast", "fold_only"])
def nvls_mode(request):
    return request.param


@pytest.mark.parametrize("name", ["tomo2", "cloud", "phong"])
def test_single_rank_nvls_fold_equals_nccl_path(ctx, golden_dir, name, nvls_mode):
    scene = FIXTURES[name]["scene"]()
    g = golden(name)
    w = weight_patterns(scene)["w"]
    p = perturbed(scene)
    ctx.upload(scene)
    st = ctx.load_store(str(golden_dir / f"{name}.pstr"))
    ref = ctx.evaluate_store(scene, st, p, EvalOptions(want_grad=True, pixel_weights=w))
    c = _nvls_ctx(scene, nvls_mode)
    try:
        st2 = c.load_store(str(golden_dir / f"{name}.pstr"))
        c.sort_by_size(st2)
        r = c.evaluate_store(scene, st2, p, EvalOptions(want_grad=True, pixel_weights=w))
        assert rel(r.images, ref.images) <= 1e-12
        assert rel(r.images, g["pert_w_images"]) <= 1e-5
        if scene.unknown_species() >= 0:
            assert rel(r.grad_beta, ref.grad_beta) <= 1e-12
            assert rel(r.grad_beta, g["pert_w_grad"]) <= 1e-5
        else:
            assert abs(r.grad_kappa - ref.grad_kappa) <= 1e-12 * abs(ref.grad_kappa)
        # the device-resident iteration (K4 -> fold -> loss -> K5 -> fold -> ADAM)
        gt = 0.9 * ref.images
        out = []
        for cc, ss in ((ctx, st), (c, st2)):
            cc.opt_init(p, gt, alpha=0.01)
            losses = [cc.opt_step(ss) for _ in range(3)]
            out.append((losses, cc.opt_params()))
        assert np.allclose(out[0][0], out[1][0], rtol=1e-12, atol=0)
        if scene.unknown_species() >= 0:
            assert rel(out[1][1].beta, out[0][1].beta) <= 1e-12
        st2.free()
    finally:
        c.close()


def test_single_rank_nvls_per_species(ctx, golden_dir, nvls_mode):
    from paper_2110_00085_b200 import scene as S
    scene = FIXTURES["tomo2"]["scene"]()
    w = weight_patterns(scene)["w"]
    pb = S.ParamSet(species_beta=[perturbed(scene).beta, None])
    ctx.upload(scene)
    st = ctx.load_store(str(golden_dir / "tomo2.pstr"))
    ref = ctx.evaluate_store(scene, st, pb, EvalOptions(want_grad=True, pixel_weights=w, per_species=True))
    c = _nvls_ctx(scene, nvls_mode)
    try:
        st2 = c.load_store(str(golden_dir / "tomo2.pstr"))
        r = c.evaluate_store(scene, st2, pb, EvalOptions(want_grad=True, pixel_weights=w, per_species=True))
        assert rel(r.grad_beta, ref.grad_beta) <= 1e-12
        st2.free()
    finally:
        c.close()


def _worker(rank, world, id_path, golden_dir, out):
    import time
    if rank == 0:
        tmp = id_path + ".tmp"
        open(tmp, "wb").write(Context.nccl_unique_id())
        os.replace(tmp, id_path)
    while not os.path.exists(id_path):
        time.sleep(0.05)
    c = Context(rank, rank, world, open(id_path, "rb").read())
    c.set_option("nvls", 1)
    scene = FIXTURES["tomo2"]["scene"]()
    c.upload(scene)
    st = c.load_store(os.path.join(golden_dir, "tomo2.pstr"))
    r = c.evaluate_store(scene, st, perturbed(scene), EvalOptions(want_grad=True,
                                                                  pixel_weights=weight_patterns(scene)["w"]))
    np.savez(f"{out}_{rank}.npz", images=r.images, grad=r.grad_beta)
    st.free()
    c.close()


def test_two_rank_nvls_matches_reference(golden_dir, tmp_path):
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs on NVSwitch")
    import torch.multiprocessing as mp
    out = str(tmp_path / "res")
    mp.spawn(_worker, args=(2, str(tmp_path / "nccl.id"), str(golden_dir), out), nprocs=2, join=True)
    g = golden("tomo2")
    for r in range(2):
        z = np.load(f"{out}_{r}.npz")
        assert rel(z["images"], g["pert_w_images"]) <= 1e-5
        assert rel(z["grad"], g["pert_w_grad"]) <= 1e-5
