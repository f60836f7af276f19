"""Reference-written stores on the device ("a reference-generated PSTR store
must be evaluated in materialized mode").

* Materialized import (PRC_IMPORT_MATERIALIZE): the file's own spans and events are
  evaluated as eval_record reads them (pathstore.cpp:115-238).  Voxel ids and span lengths
  are the reference's by construction, so images and gradients agree with the reference to
  fp64 rounding (atomic summation order, CUDA libm ulps), far inside the 1e-5 bar.  Export
  writes the records verbatim: byte-identical to the input, and after a device sort
  byte-identical to the reference's sort_by_size + save_store.
* Recomputed import (the default; spans re-walked on the device): voxel indexing is pinned
  against the file and against the reference's own segment_lengths (pathstore.cpp:296-313).
"""
import numpy as np
import pytest

from paper_2110_00085_b200 import abi
from paper_2110_00085_b200 import scene as S
from paper_2110_00085_b200.gpu import EvalOptions, PrcIOError
from tests import pstr as P
from tests.fixtures import FIXTURES, golden, perturbed, weight_patterns

pytestmark = pytest.mark.gpu

TIGHT = 1e-12


def img_err(a, r):
    floor = 1e-3 * max(np.abs(r).max(), 1e-300)
    return float((np.abs(a - r) / np.maximum(np.abs(r), floor)).max()) if r.size else 0.0


def grad_err(a, r):
    scale = max(np.abs(r).max(), 1e-300)
    return float((np.abs(a - r) / np.maximum(np.maximum(np.abs(a), np.abs(r)), scale)).max())


def scalar_err(a, r):
    return abs(a - r) / max(abs(a), abs(r), 1e-300)


@pytest.mark.parametrize("name", list(FIXTURES))
@pytest.mark.parametrize("sort", [False, True])
def test_materialized_matches_reference(ctx, golden_dir, name, sort):
    scene = FIXTURES[name]["scene"]()
    g = golden(name)
    ctx.upload(scene)
    st = ctx.load_store(str(golden_dir / f"{name}.pstr"), materialized=True)
    assert st.info()["materialized"] == 1
    if sort:
        ctx.sort_by_size(st)
        assert np.array_equal(st.streams(), g["sorted_streams"])
    worst = [0.0, 0.0]
    for tag, params in (("ref", None), ("pert", perturbed(scene))):
        for wtag, w in weight_patterns(scene).items():
            r = ctx.evaluate_store(scene, st, params, EvalOptions(want_grad=True, pixel_weights=w))
            e = img_err(r.images, g[f"{tag}_{wtag}_images"])
            worst[0] = max(worst[0], e)
            assert e <= TIGHT, (tag, wtag, e)
            if scene.unknown_species() >= 0:
                e = grad_err(r.grad_beta, g[f"{tag}_{wtag}_grad"])
                worst[1] = max(worst[1], e)
                assert e <= TIGHT, (tag, wtag, e)
            else:
                for k, v in (("gk", r.grad_kappa), ("gg", r.grad_gamma)):
                    e = scalar_err(v, float(g[f"{tag}_{wtag}_{k}"]))
                    worst[1] = max(worst[1], e)
                    assert e <= TIGHT, (tag, wtag, k, e)
            assert r.clamp_events == int(g[f"{tag}_{wtag}_clamps"])
        if scene.unknown_species() >= 0:
            r = ctx.evaluate_store(scene, st, params, EvalOptions(want_grad=True, legacy_score=True))
            assert grad_err(r.grad_beta, g[f"{tag}_legacy_grad"]) <= TIGHT
    print(f"materialized {name} sort={sort}: image {worst[0]:.1e}, gradient {worst[1]:.1e}")


def test_materialized_per_type_gradients(ctx, golden_dir):
    scene = FIXTURES["tomo2"]["scene"]()
    flip = FIXTURES["tomo2"]["flip_unknown"]()
    g = golden("tomo2")
    ctx.upload(scene)
    st = ctx.load_store(str(golden_dir / "tomo2.pstr"), materialized=True)
    w = weight_patterns(scene)["w"]
    r = ctx.evaluate_store(scene, st, S.ParamSet(species_beta=[perturbed(scene).beta, None]),
                           EvalOptions(want_grad=True, pixel_weights=w, per_species=True))
    assert grad_err(r.grad_beta[0], g["pert_w_grad"]) <= TIGHT
    r = ctx.evaluate_store(scene, st, S.ParamSet(species_beta=[None, perturbed(flip).beta]),
                           EvalOptions(want_grad=True, pixel_weights=w, per_species=True))
    assert img_err(r.images, g["flip_pert_w_images"]) <= TIGHT
    assert grad_err(r.grad_beta[1], g["flip_pert_w_grad"]) <= TIGHT


def test_materialized_iteration_runs(ctx, golden_dir):
    """The device-resident Algorithm-2 iteration runs on a materialized store as on any
    other: the loss is 0.5 ||F_t - gt||^2 of the reference's images."""
    scene = FIXTURES["tomo2"]["scene"]()
    g = golden("tomo2")
    ctx.upload(scene)
    st = ctx.load_store(str(golden_dir / "tomo2.pstr"), materialized=True)
    res = weight_patterns(scene)["res"]
    ctx.opt_init(perturbed(scene), g["pert_res_images"] - res, alpha=0.05)
    loss = ctx.opt_step(st)
    assert abs(loss - 0.5 * (res ** 2).sum()) <= 1e-12 * loss


@pytest.mark.parametrize("name", list(FIXTURES))
def test_materialized_export_is_verbatim(ctx, ref, golden_dir, tmp_path, name):
    scene = FIXTURES[name]["scene"]()
    ctx.upload(scene)
    src = str(golden_dir / f"{name}.pstr")
    st = ctx.load_store(src, materialized=True)
    st.save(str(tmp_path / "out.pstr"))
    assert (tmp_path / "out.pstr").read_bytes() == open(src, "rb").read()
    ctx.sort_by_size(st)
    st.save(str(tmp_path / "sorted.pstr"))
    ref.sort_pstr(src, len(st), str(tmp_path / "ref_sorted.pstr"))
    assert (tmp_path / "sorted.pstr").read_bytes() == (tmp_path / "ref_sorted.pstr").read_bytes()


def test_materialized_import_range_checks(ctx, golden_dir, tmp_path):
    import struct
    scene = FIXTURES["cloud"]["scene"]()
    ctx.upload(scene)
    raw = bytearray((golden_dir / "cloud.pstr").read_bytes())
    f = P.read(str(golden_dir / "cloud.pstr"))
    nb = f["ref_beta"].size
    rec0 = 41 + 8 * nb + 16
    nv = len(f["records"][0]["vertices"])
    ns = len(f["records"][0]["spans"])
    assert ns > 0
    span0 = rec0 + 8 + 1 + 24 + 4 + 64 * nv + 4  # first stored span's voxel
    struct.pack_into("<I", raw, span0, scene.voxel_count)
    bad = tmp_path / "bad_span.pstr"
    bad.write_bytes(bytes(raw))
    with pytest.raises(PrcIOError, match="span voxel"):
        ctx.load_store(str(bad), materialized=True)


@pytest.mark.parametrize("name", ["tomo2", "cloud", "mixed"])
def test_recomputed_import_voxel_indexing(ctx, ref, golden_dir, tmp_path, name):
    """Default import of a reference-written store: segments and LE connections are
    re-walked on the device.  Against the file: identical (detector, pixel) events, LE
    span voxels and lengths bit for bit (the connection w = to_det * (1/r) is recomputed
    from the stored position exactly as add_events forms it, transport.cpp:218-254), and
    identical segment voxel ids.  Segment span lengths of b >= 2 follow the chord direction
    (the file stores no directions) and equal, bit for bit, the reference's own re-walk
    segment_lengths (pathstore.cpp:296-313); they differ from the trace-time lengths only in
    the last bits, which the test reports."""
    scene = FIXTURES[name]["scene"]()
    ctx.upload(scene)
    src = str(golden_dir / f"{name}.pstr")
    st = ctx.load_store(src)
    out = str(tmp_path / "dev.pstr")
    st.save(out)
    a, b = P.read(src), P.read(out)
    rc, rv, rl = ref.segment_lengths(scene, src)
    ro = np.r_[0, np.cumsum(rc.astype(np.int64))]
    k = 0
    n_seg = n_len_diff = n_ref_diff = 0
    for ra, rb in zip(a["records"], b["records"]):
        assert ra["stream"] == rb["stream"] and len(ra["vertices"]) == len(rb["vertices"])
        assert np.array_equal(ra["vertices"]["voxel"], rb["vertices"]["voxel"])
        ea, eb = ra["events"], rb["events"]
        assert np.array_equal(ea[["vertex", "detector", "pixel"]], eb[["vertex", "detector", "pixel"]])
        assert np.array_equal(ea["geom"].view(np.uint64), eb["geom"].view(np.uint64))
        assert np.array_equal(ra["le_spans"]["voxel"], rb["le_spans"]["voxel"])
        assert np.array_equal(ra["le_spans"]["length"].view(np.uint64), rb["le_spans"]["length"].view(np.uint64))
        for bseg, (sa, sb) in enumerate(zip(P.segment_spans(ra), P.segment_spans(rb)), start=1):
            assert np.array_equal(sa["voxel"], sb["voxel"]), (ra["stream"], bseg)
            n_seg += 1
            n_len_diff += int(not np.array_equal(sa["length"].view(np.uint64), sb["length"].view(np.uint64)))
            if bseg >= 2:  # the reference's own re-walk along the chord
                rs = slice(ro[k], ro[k + 1])
                assert np.array_equal(rv[rs], sb["voxel"])
                assert np.array_equal(rl[rs].view(np.uint64), sb["length"].view(np.uint64)), (ra["stream"], bseg)
            else:
                n_ref_diff += int(not np.array_equal(sa["length"].view(np.uint64), sb["length"].view(np.uint64)))
            k += 1
    assert k == len(rc)
    print(f"{name}: {n_seg} segments, voxel ids identical; {n_len_diff} with trace-time length bits "
          f"differing from the chord re-walk ({n_ref_diff} of them first segments)")
