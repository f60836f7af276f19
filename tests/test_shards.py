"""Multi-GPU sharding on the engine itself.

Paths are independent: rank r of W owns the contiguous stream range [N r / W, N (r+1) / W)
(prc_gpu_shard_range), traces or imports only that range, and K4/K5 produce partial image
and gradient sums that an allreduce adds up (ncclAllReduce after K4 and K5 in the engine;
the reference sums its chunk partials in order, pathstore.cpp:343-354).

* One GPU: W detached shard contexts (prc_gpu_ctx_create_rank without a communicator)
  evaluate their ranges of one store; their partial results add up to the single-context
  result, and the traced shards are exactly the single-context trace's paths.
* Two GPUs (skipped below 2): two processes on one NCCL communicator reproduce the
  reference's golden results.
"""
import os

import numpy as np
import pytest

from paper_2110_00085_b200 import scene as S
from paper_2110_00085_b200.gpu import Context, EvalOptions, RenderOptions
from tests.fixtures import FIXTURES, golden, perturbed, weight_patterns

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


@pytest.mark.parametrize("world", [2, 3])
def test_detached_shards_sum_to_the_single_context_result(ctx, golden_dir, world):
    scene = FIXTURES["tomo2"]["scene"]()
    w = weight_patterns(scene)["w"]
    p = perturbed(scene)
    ctx.upload(scene)
    full = ctx.load_store(str(golden_dir / "tomo2.pstr"))
    ctx.sort_by_size(full)
    ref = ctx.evaluate_store(scene, full, p, EvalOptions(want_grad=True, pixel_weights=w))
    n = len(full)
    img = np.zeros_like(ref.images)
    grad = np.zeros_like(ref.grad_beta)
    clamps = 0
    covered = []
    for r in range(world):
        c = Context(0, r, world)
        try:
            c.upload(scene)
            st = c.load_store(str(golden_dir / "tomo2.pstr"))
            info = st.info()
            lo, hi = Context.shard_range(n, r, world)
            assert (info["stream_base"], info["n_paths"], info["n_paths_global"]) == (lo, hi - lo, n)
            covered.append((lo, hi))
            c.sort_by_size(st)
            part = c.evaluate_store(scene, st, p, EvalOptions(want_grad=True, pixel_weights=w))
            img += part.images
            grad += part.grad_beta
            clamps += part.clamp_events
            st.free()
        finally:
            c.close()
    assert covered[0][0] == 0 and covered[-1][1] == n
    assert all(covered[k][1] == covered[k + 1][0] for k in range(world - 1))
    assert rel(img, ref.images) <= 1e-12 and rel(grad, ref.grad_beta) <= 1e-12
    assert clamps == ref.clamp_events
    assert rel(img, golden("tomo2")["pert_w_images"]) <= 1e-5


def test_detached_shards_self_normalize(ctx, golden_dir):
    """Self-normalisation over detached shards: each returns its undivided partial sums
    and its partial mean correction factor; their sums give the single-context result."""
    scene = FIXTURES["tomo2"]["scene"]()
    p = perturbed(scene)
    opt = EvalOptions(self_normalize=True)
    ctx.upload(scene)
    full = ctx.load_store(str(golden_dir / "tomo2.pstr"))
    ref = ctx.evaluate_store(scene, full, p, opt)
    img = np.zeros_like(ref.images)
    mean = 0.0
    for r in range(3):
        c = Context(0, r, 3)
        try:
            c.upload(scene)
            st = c.load_store(str(golden_dir / "tomo2.pstr"))
            part = c.evaluate_store(scene, st, p, opt)
            img += part.images
            mean += part.mean_correction
            st.free()
        finally:
            c.close()
    assert abs(mean - ref.mean_correction) <= 1e-12 * ref.mean_correction
    assert rel(img / mean, ref.images) <= 1e-12


def test_detached_shard_traces_are_the_single_trace(ctx):
    scene = S.cloud_scene(16, 12, 12)
    n = 50_001
    ctx.upload(scene)
    rr = ctx.render(scene, RenderOptions(n_paths=n, seed=7, keep_paths=True))
    sizes = rr.store.sizes()
    img = np.zeros_like(rr.images)
    trunc = 0
    for r in range(4):
        c = Context(0, r, 4)
        try:
            c.upload(scene)
            part = c.render(scene, RenderOptions(n_paths=n, seed=7, keep_paths=True))
            lo, hi = Context.shard_range(n, r, 4)
            assert np.array_equal(part.store.streams(), np.arange(lo, hi, dtype=np.uint64))
            assert np.array_equal(part.store.sizes(), sizes[lo:hi])  # Philox keyed by the global stream
            img += part.images
            trunc += part.truncated_paths
            part.store.free()
        finally:
            c.close()
    assert rel(img, rr.images) <= 1e-12
    assert trunc == rr.truncated_paths


def _nccl_worker(rank, world, id_path, golden_dir, out):
    import time
    if rank == 0:
        tmp = id_path + ".tmp"
        open(tmp, "wb").write(Context.nccl_unique_id())
        os.replace(tmp, id_path)
    while not os.path.exists(id_path):
        time.sleep(0.05)
    c = Context(rank, rank, world, open(id_path, "rb").read())
    scene = FIXTURES["tomo2"]["scene"]()
    c.upload(scene)
    st = c.load_store(os.path.join(golden_dir, "tomo2.pstr"))
    c.sort_by_size(st)
    r = c.evaluate_store(scene, st, perturbed(scene),
                         EvalOptions(want_grad=True, pixel_weights=weight_patterns(scene)["w"]))
    np.savez(f"{out}_{rank}.npz", images=r.images, grad=r.grad_beta)
    st.free()
    c.close()


def test_two_rank_nccl_allreduce_matches_reference(golden_dir, tmp_path):
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (one process per GPU on an NCCL communicator)")
    import torch.multiprocessing as mp
    out = str(tmp_path / "res")
    mp.spawn(_nccl_worker, args=(2, str(tmp_path / "nccl.id"), str(golden_dir), out), nprocs=2, join=True)
    g = golden("tomo2")
    for r in range(2):  # both replicas hold the allreduced (global) result
        z = np.load(f"{out}_{r}.npz")
        assert rel(z["images"], g["pert_w_images"]) <= 1e-5
        assert rel(z["grad"], g["pert_w_grad"]) <= 1e-5
