"""Generates the committed golden fixtures under tests/golden/ by running the UNMODIFIED
reference (oracle/_ref/libpathrec_ref.so, compiled in place from /root/reference by
oracle/Makefile).  Re-run with:  python tests/golden/make_golden.py

Per fixture <name>:
  <name>.pstr.gz  the reference's PSTR v1 store (render keep_paths, seed 7)
  <name>.npz      fresh images, evaluate_store results at the reference point and at a
                  perturbed point (images, grad_beta, grad_kappa/gamma, clamp counts) with
                  and without pixel weights, and the sort_by_size stream order.
Plus common.npz: Philox known answers, walk_voxels spans and pixel_of indices.
"""
import gzip
import os
import shutil
import sys
import tempfile

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from paper_2110_00085_b200 import abi  # noqa: E402
from tests.fixtures import FIXTURES, perturbed, weight_patterns, walk_rays  # noqa: E402
from pyoracle import Reference  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    ref = Reference()
    tmp = tempfile.mkdtemp()
    for name, fx in FIXTURES.items():
        scene, n, mb = fx["scene"](), fx["n"], fx.get("max_bounces", 500)
        pstr = os.path.join(tmp, name + ".pstr")
        img, tr = ref.render(scene, n, 7, max_bounces=mb, pstr_out=pstr)
        out = {"fresh_images": img, "truncated": np.array(tr)}
        out["sorted_streams"] = ref.sort_pstr(pstr, n)
        for tag, params in (("ref", None), ("pert", perturbed(scene))):
            for wtag, w in weight_patterns(scene).items():
                flags = abi.PRC_EVAL_NORMALIZE | abi.PRC_EVAL_WANT_GRAD
                r = ref.evaluate(scene, pstr, params, flags, w)
                out[f"{tag}_{wtag}_images"] = r["images"]
                out[f"{tag}_{wtag}_grad"] = r["grad"]
                out[f"{tag}_{wtag}_gk"] = np.array(r["grad_kappa"])
                out[f"{tag}_{wtag}_gg"] = np.array(r["grad_gamma"])
                out[f"{tag}_{wtag}_clamps"] = np.array(r["clamp_events"])
            r = ref.evaluate(scene, pstr, params,
                             abi.PRC_EVAL_NORMALIZE | abi.PRC_EVAL_WANT_GRAD | abi.PRC_EVAL_LEGACY_SCORE,
                             None)
            out[f"{tag}_legacy_grad"] = r["grad"]
        if fx.get("flip_unknown"):  # per-type gradient oracle: species 1 as the unknown
            s1 = fx["flip_unknown"]()
            pstr1 = os.path.join(tmp, name + "_flip.pstr")
            ref.render(s1, n, 7, max_bounces=mb, pstr_out=pstr1)
            r = ref.evaluate(s1, pstr1, perturbed(s1), abi.PRC_EVAL_NORMALIZE | abi.PRC_EVAL_WANT_GRAD,
                             weight_patterns(s1)["w"])
            out["flip_pert_w_images"] = r["images"]
            out["flip_pert_w_grad"] = r["grad"]
        with open(pstr, "rb") as f, gzip.open(os.path.join(OUT, name + ".pstr.gz"), "wb", 9) as g:
            shutil.copyfileobj(f, g)
        np.savez_compressed(os.path.join(OUT, name + ".npz"), **out)
        print(name, os.path.getsize(os.path.join(OUT, name + ".pstr.gz")), "bytes pstr.gz")
    # common known answers
    common = {}
    for seed, stream in ((0, 0), (7, 3), (0x9E3779B97F4A7C15, 12345)):
        common[f"philox_{seed}_{stream}"] = ref.philox(seed, stream, 64)
    for name, fx in FIXTURES.items():
        scene = fx["scene"]()
        if not scene.species:
            continue
        rays = walk_rays(scene, 400, seed=11)
        c, v, ln = ref.walk(scene, rays)
        common[f"walk_{name}_rays"] = rays
        common[f"walk_{name}_counts"] = c
        common[f"walk_{name}_vox"] = v
        common[f"walk_{name}_len"] = ln
        pts = np.random.default_rng(5).uniform(-0.2, 1.2, size=(2000, 3))
        for k in range(len(scene.detectors)):
            common[f"pixel_{name}_{k}"] = ref.pixel_of(scene, k, pts)
        common[f"pixel_{name}_pts"] = pts
    np.savez_compressed(os.path.join(OUT, "common.npz"), **common)
    shutil.rmtree(tmp)


if __name__ == "__main__":
    main()
