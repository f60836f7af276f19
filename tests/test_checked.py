"""Range-checked build (stands in for compute-sanitizer, which this pool does not offer).

libpathrec_gpu_checked.so is the engine compiled with -DPRC_CHECKED: every guard-free
access of the hot kernels (padded-table gathers in K4a/K4b, reductions into the padded
gradient copies in K5b/K5a, pixel and voxel indices) is checked against its table and a
violation is recorded instead of performed.  The parity fixtures (every kernel mapping,
sorted and unsorted, gradients, per-type, materialized stores, the driver loop) and
stores at the bench geometry run through it; the range-check word must stay clean and
the results must still match the reference.
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
CHECKED = os.path.join(ROOT, "paper_2110_00085_b200", "libpathrec_gpu_checked.so")

SCRIPT = r'''
import sys, numpy as np
sys.path.insert(0, ROOT)
from paper_2110_00085_b200 import gpu, scene as S
from paper_2110_00085_b200.gpu import Context, EvalOptions, RenderOptions
from tests.fixtures import FIXTURES, golden, perturbed, weight_patterns
import tests.conftest as cf
import gzip, shutil, tempfile, os
tmp = tempfile.mkdtemp()
for f in os.listdir(cf.GOLDEN):
    if f.endswith(".pstr.gz"):
        with gzip.open(os.path.join(cf.GOLDEN, f), "rb") as g, open(os.path.join(tmp, f[:-3]), "wb") as o:
            shutil.copyfileobj(g, o)
ctx = Context(0)
flags, checked = ctx.debug_checks()
assert checked, "not a checked build"
def clean(tag):
    f, _ = ctx.debug_checks()
    assert f == 0, (tag, hex(f))
def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))
n = 0
for mapping in ({"mode": 0, "packet": 3}, {"mode": 0, "packet": 1}, {"mode": 0, "packet": 2}, {"mode": 0, "packet": 4},
                {"mode": 0, "packet": 3, "pad": 0}, {"mode": 1, "packet": 1}):
    for k, v in mapping.items():
        ctx.set_option(k, v)
    for name in FIXTURES:
        sc = FIXTURES[name]["scene"]()
        g = golden(name)
        ctx.upload(sc)
        for mat in (False, True):
            st = ctx.load_store(os.path.join(tmp, name + ".pstr"), materialized=mat)
            for sort in (False, True):
                if sort:
                    ctx.sort_by_size(st)
                r = ctx.evaluate_store(sc, st, perturbed(sc), EvalOptions(want_grad=True, pixel_weights=weight_patterns(sc)["w"]))
                clean((name, mapping, mat, sort))
                assert rel(r.images, g["pert_w_images"]) <= 1e-5, (name, mapping)
                if sc.unknown_species() >= 0:
                    assert rel(r.grad_beta, g["pert_w_grad"]) <= 1e-5, (name, mapping)
                n += 1
            st.free()
    ctx.set_option("mode", 0); ctx.set_option("packet", 3); ctx.set_option("pad", 1)
# self-normalisation and the per-path correction factors (all segments re-walked)
for name in FIXTURES:
    sc = FIXTURES[name]["scene"]()
    ctx.upload(sc)
    for mat in (False, True):
        st = ctx.load_store(os.path.join(tmp, name + ".pstr"), materialized=mat)
        ctx.evaluate_store(sc, st, perturbed(sc), EvalOptions(want_grad=True, self_normalize=True))
        ctx.correction_factors(sc, st, perturbed(sc))
        clean((name, "self_normalize", mat))
        st.free()
# per-type gradients, deterministic images, the driver loop
sc = FIXTURES["tomo2"]["scene"]()
ctx.upload(sc)
st = ctx.load_store(os.path.join(tmp, "tomo2.pstr"))
ctx.evaluate_store(sc, st, S.ParamSet(species_beta=[perturbed(sc).beta, None]),
                   EvalOptions(want_grad=True, per_species=True, deterministic=True))
clean("per_species")
# bench geometry: (b) at 2e4 paths, (c) at 1e4 paths, (d) at 2e4 paths; trace, sort, forward, gradient, iteration
for cfg, s2, npaths in (("b", S.cloud_scene(128, 128, 128), 20000), ("c", S.cloud_scene(128, 128, 128, two_species=True), 10000),
                        ("a", S.cloud_scene(32, 64, 64), 50000), ("d", S.reflectometry_scene(64, 64, 16), 20000)):
    if cfg == "c":
        ctx.set_option("per_species", 1)
    ctx.upload(s2)
    rr = ctx.render(s2, RenderOptions(n_paths=npaths, seed=7, keep_paths=True))
    clean(cfg + " render")
    ctx.sort_by_size(rr.store)
    u = s2.unknown_species()
    t = S.ParamSet(S.recycle_point(s2.species[u].extinction)) if u >= 0 else S.ParamSet(None, 0.55, 38.0)
    ctx.opt_init(t, 0.9 * rr.images, alpha=1e-3)
    for _ in range(2):
        ctx.opt_step(rr.store)
    clean(cfg + " iteration")
    rr.store.free()
    ctx.set_option("per_species", 0)
s3 = S.cloud_scene(8, 16, 16)
ctx.upload(s3)
gt = ctx.render(s3, RenderOptions(n_paths=50000, seed=3)).images
ctx.reconstruct_schedule(s3, gt, S.ParamSet(np.full(s3.voxel_count, 2.0)), stages=[(8, 8, 5000), (0, 0, 5000)],
                         recycle_period=3, max_iterations=8, alpha=0.1, saturation_window=2,
                         saturation_rel_improvement=1.0)
clean("schedule")
print(f"checked build clean over {n} fixture evaluations + bench-geometry iterations + the schedule")
'''


@pytest.mark.gpu
def test_checked_build_is_clean():
    if not os.path.exists(CHECKED):
        pytest.skip("libpathrec_gpu_checked.so not built (__graft_entry__.build())")
    env = dict(os.environ, PRC_LIB=CHECKED)
    r = subprocess.run([sys.executable, "-c", f"ROOT = {ROOT!r}\n" + SCRIPT], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=1800)
    print(r.stdout[-3000:], r.stderr[-3000:])
    assert r.returncode == 0 and "checked build clean" in r.stdout, r.stderr[-3000:]


def test_checked_build_compiles():
    """The checked variant builds (nvcc cross-compiles it without a GPU)."""
    from paper_2110_00085_b200.build import CHECKED_OUT, build
    assert build(defines=("PRC_CHECKED",), out=CHECKED_OUT) == CHECKED_OUT
    assert os.path.exists(CHECKED_OUT)
