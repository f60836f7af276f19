"""CPU multi-rank tests (world size 2, gloo): the path-sharding decomposition the GPU
engine uses across ranks.  Rank r owns the contiguous stream range [N r / W, N (r+1) / W)
(prc_capi.cu trace_store / import_pstr); each rank evaluates its shard without
normalisation, the raw image and gradient sums are all-reduced, and the result divided by
the global N must equal the single-process evaluation (the same reduction NCCL performs
over NVLink after K4 and K5).  The oracle stands in for the per-rank kernels."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2110_00085_b200 import abi
from tests.fixtures import FIXTURES, golden, perturbed, weight_patterns


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def shard(n, rank, world):
    """The engine's own partition (prc_gpu_shard_range, host-only: no device needed)."""
    from paper_2110_00085_b200.gpu import Context
    lo, hi = Context.shard_range(n, rank, world)
    assert (lo, hi) == (n * rank // world, n * (rank + 1) // world)
    return lo, hi


def _worker(rank, world, port, pstr, name, out):
    import torch
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
    from pyoracle import Port
    port_ = Port()
    scene = FIXTURES[name]["scene"]()
    full = port_.load(pstr)
    n = len(full)
    lo, hi = shard(n, rank, world)
    part = full.slice(lo, hi)
    w = weight_patterns(scene)["w"]
    r = port_.evaluate(scene, part, perturbed(scene), abi.PRC_EVAL_WANT_GRAD, w)  # raw sums
    img = torch.tensor(r["images"])
    grad = torch.tensor(r["grad"])
    scal = torch.tensor([r["grad_kappa"], r["grad_gamma"], float(r["clamp_events"])], dtype=torch.float64)
    for t in (img, grad, scal):
        dist.all_reduce(t)
    # max-over-ranks timing reduction used by bench.py
    tmax = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    if rank == 0:
        np.savez(out, images=img.numpy() / n, grad=grad.numpy() / n, gk=scal[0].item() / n,
                 gg=scal[1].item() / n, clamps=scal[2].item(), tmax=tmax.item())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["tomo2", "phong"])
def test_two_rank_shards_reduce_to_the_single_process_result(golden_dir, tmp_path, name):
    pstr = str(golden_dir / f"{name}.pstr")
    out = str(tmp_path / "r.npz")
    mp.start_processes(_worker, args=(2, _free_port(), pstr, name, out), nprocs=2, join=True,
                       start_method="spawn")
    r = np.load(out)
    g = golden(name)
    np.testing.assert_allclose(r["images"], g["pert_w_images"], rtol=1e-12, atol=1e-300)
    if g["pert_w_grad"].size:
        np.testing.assert_allclose(r["grad"], g["pert_w_grad"], rtol=1e-9,
                                   atol=1e-12 * max(1e-300, np.abs(g["pert_w_grad"]).max()))
    assert abs(r["gk"] - float(g["pert_w_gk"])) <= 1e-9 * max(1e-300, abs(float(g["pert_w_gk"])))
    assert r["clamps"] == float(g["pert_w_clamps"])
    assert r["tmax"] == 2.0


def test_shard_ranges_partition_the_streams():
    for n in (1, 7, 1000, 10**8 + 3):
        for world in (1, 2, 3, 8):
            ranges = [shard(n, r, world) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            assert all(ranges[i][1] == ranges[i + 1][0] for i in range(world - 1))
