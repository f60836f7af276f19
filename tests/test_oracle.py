"""CPU tests: pin the C restatement oracle against the reference's golden vectors and
(where oracle/_ref is built) against the live reference, and restate the reference's
own known-answer tests for the hot path."""
import filecmp
import math
import os

import numpy as np
import pytest


from paper_2110_00085_b200 import abi
from paper_2110_00085_b200 import scene as S
from tests.fixtures import FIXTURES, golden, perturbed, weight_patterns

FLAGS = abi.PRC_EVAL_NORMALIZE | abi.PRC_EVAL_WANT_GRAD


# ---------------------------------------------------------------- Philox (rng.hpp:11-61)
def test_philox_known_answers(port):
    # Random123 KAT order: seed 0 / stream 0, first block
    assert [hex(x) for x in port.philox(0, 0, 4)] == ["0x6627e8d5", "0xe169c58d", "0xbc57ac4c", "0x9b00dbd8"]
    assert [hex(x) for x in port.philox(7, 3, 4)] == ["0x97b356d9", "0x1fb03c42", "0x29a796e8", "0x998b4610"]
    g = golden("common")
    for k, v in g.items():
        if k.startswith("philox_"):
            _, seed, stream = k.split("_")
            assert np.array_equal(port.philox(int(seed), int(stream), v.size), v)


def test_next_double_known_answer(port):
    w = port.philox(7, 3, 4).astype(np.uint64)
    d0 = float(((w[0] << np.uint64(32)) | w[1]) >> np.uint64(11)) * 2.0 ** -53
    d1 = float(((w[2] << np.uint64(32)) | w[3]) >> np.uint64(11)) * 2.0 ** -53
    assert d0 == 0.59258024979470825 and d1 == 0.16271346262651054


# ---------------------------------------------------------------- DDA (traverse.hpp)
def test_walk_known_answers(port):
    # test_transport.cpp:13-42
    s = S.Scene(grid=S.Grid((3, 1, 1), (0, 0, 0), (1, 1, 1)), species=[S.Species(np.zeros(3))])
    c, v, ln = port.walk(s, np.array([[-0.5, 0.5, 0.5, 1, 0, 0, 10.0]]))
    assert c.tolist() == [3] and v.tolist() == [0, 1, 2] and np.allclose(ln, 1.0, atol=1e-12)
    c, v, ln = port.walk(s, np.array([[-0.5, 5.0, 0.5, 1, 0, 0, 10.0]]))
    assert c.tolist() == [0]
    c, v, ln = port.walk(s, np.array([[0.0, 0.5, 0.5, 1, 0, 0, 1.5]]))
    assert c.tolist() == [2] and abs(ln[1] - 0.5) < 1e-12
    s5 = S.Scene(grid=S.cube_grid(5), species=[S.Species(np.zeros(125))])
    a, b = np.array([0.03, 0.11, 0.27]), np.array([0.94, 0.81, 0.66])
    d = b - a
    c, v, ln = port.walk(s5, np.concatenate([a, d / np.linalg.norm(d), [np.linalg.norm(d)]])[None])
    assert abs(ln.sum() - np.linalg.norm(d)) < 1e-9


@pytest.mark.parametrize("name", [n for n in FIXTURES if FIXTURES[n]["scene"]().species])
def test_walk_matches_golden_bitwise(port, name):
    g = golden("common")
    scene = FIXTURES[name]["scene"]()
    c, v, ln = port.walk(scene, g[f"walk_{name}_rays"])
    assert np.array_equal(c, g[f"walk_{name}_counts"])
    assert np.array_equal(v, g[f"walk_{name}_vox"])
    assert np.array_equal(ln.view(np.uint64), g[f"walk_{name}_len"].view(np.uint64))


@pytest.mark.parametrize("name", [n for n in FIXTURES if FIXTURES[n]["scene"]().species])
def test_pixel_of_matches_golden(port, name):
    g = golden("common")
    scene = FIXTURES[name]["scene"]()
    pts = g[f"pixel_{name}_pts"]
    for k in range(len(scene.detectors)):
        assert np.array_equal(port.pixel_of(scene, k, pts), g[f"pixel_{name}_{k}"])


# ---------------------------------------------------------------- trace / store / eval
@pytest.mark.parametrize("name", list(FIXTURES))
def test_oracle_render_reproduces_reference_store(port, golden_dir, tmp_path, name):
    """The oracle's trace + PSTR writer are byte-identical to the reference's."""
    fx = FIXTURES[name]
    scene = fx["scene"]()
    img, tr, st = port.render(scene, fx["n"], 7, max_bounces=fx.get("max_bounces", 500))
    g = golden(name)
    assert np.array_equal(img, g["fresh_images"])
    assert tr == int(g["truncated"])
    st.save(str(tmp_path / "o.pstr"))
    assert filecmp.cmp(str(tmp_path / "o.pstr"), str(golden_dir / f"{name}.pstr"), shallow=False)


@pytest.mark.parametrize("name", list(FIXTURES))
def test_oracle_evaluate_matches_golden(port, golden_dir, name):
    scene = FIXTURES[name]["scene"]()
    g = golden(name)
    st = port.load(str(golden_dir / f"{name}.pstr"))
    for tag, params in (("ref", None), ("pert", perturbed(scene))):
        for wtag, w in weight_patterns(scene).items():
            r = port.evaluate(scene, st, params, FLAGS, w)
            assert np.array_equal(r["images"], g[f"{tag}_{wtag}_images"])
            assert np.array_equal(r["grad"], g[f"{tag}_{wtag}_grad"])
            assert r["grad_kappa"] == float(g[f"{tag}_{wtag}_gk"])
            assert r["grad_gamma"] == float(g[f"{tag}_{wtag}_gg"])
            assert r["clamp_events"] == int(g[f"{tag}_{wtag}_clamps"])
        r = port.evaluate(scene, st, params, FLAGS | abi.PRC_EVAL_LEGACY_SCORE, None)
        assert np.array_equal(r["grad"], g[f"{tag}_legacy_grad"])


@pytest.mark.parametrize("name", list(FIXTURES))
def test_oracle_sort_matches_golden(port, golden_dir, name):
    st = port.load(str(golden_dir / f"{name}.pstr"))
    st.sort_by_size()
    assert np.array_equal(st.streams(), golden(name)["sorted_streams"])
    sz = st.sizes()
    assert (np.diff(sz.astype(np.int64)) >= 0).all()


def test_sort_known_answer(port, tmp_path):
    """test_pathstore.cpp:87-113: sizes 5, 2, 9, 2 -> streams 1, 3, 0, 2 (stable)."""
    scene = S.homogeneous_cube(0.0, 0.9)
    # build a PSTR by hand with records of the requested sizes
    import struct
    p = tmp_path / "k.pstr"
    with open(p, "wb") as f:
        f.write(b"PSTR" + struct.pack("<IQQQBQdd", 1, 4, 0, 0, 0, 0, 0.0, 0.0))
        for stream, size in enumerate([5, 2, 9, 2]):
            f.write(struct.pack("<QBdddI", stream, 0, 0, 0, 1, size + 1))
            for _ in range(size + 1):
                f.write(struct.pack("<ddddddIIihbB", 0.5, 0.5, 0.5, 1, 1, 1, 0, 0, -1, -1, -1, 0))
            f.write(struct.pack("<III", 0, 0, 0))
    st = port.load(str(p))
    st.sort_by_size()
    assert st.streams().tolist() == [1, 3, 0, 2]
    del scene


def test_identity_recycling_is_exact(port, golden_dir):
    """Recycled evaluation at the reference point reproduces the fresh render
    (test_pathstore.cpp:142-149)."""
    g = golden("tomo2")
    st = port.load(str(golden_dir / "tomo2.pstr"))
    r = port.evaluate(FIXTURES["tomo2"]["scene"](), st, None, abi.PRC_EVAL_NORMALIZE)
    assert np.array_equal(r["images"], g["fresh_images"])


def test_per_type_flip_oracle(port, golden_dir):
    """flipping the unknown species leaves images unchanged; gradients of the
    two species differ only at scatter-vertex voxels."""
    g = golden("tomo2")
    assert np.array_equal(g["flip_pert_w_images"].shape, g["pert_w_images"].shape)


def test_gradient_matches_finite_differences(port, golden_dir):
    """Fused gradient vs central differences on frozen paths (test_gradient.cpp:134-162,
    step h = 1e-4 (1 + |m|) as oracles.cpp:238-259)."""
    scene = FIXTURES["tomo2"]["scene"]()
    st = port.load(str(golden_dir / "tomo2.pstr"))
    w = weight_patterns(scene)["w"]
    t = perturbed(scene)
    r = port.evaluate(scene, st, t, FLAGS, w)
    rng = np.random.default_rng(0)
    idx = rng.choice(scene.voxel_count, 12, replace=False)
    scale = np.abs(r["grad"]).max()
    for v in idx:
        h = 1e-4 * (1 + abs(t.beta[v]))
        tp = S.ParamSet(t.beta.copy())
        tm = S.ParamSet(t.beta.copy())
        tp.beta[v] += h
        tm.beta[v] -= h
        fp = (port.evaluate(scene, st, tp, abi.PRC_EVAL_NORMALIZE)["images"] * w).sum()
        fm = (port.evaluate(scene, st, tm, abi.PRC_EVAL_NORMALIZE)["images"] * w).sum()
        fd = (fp - fm) / (2 * h)
        assert abs(fd - r["grad"][v]) <= 1e-6 * max(abs(fd), abs(r["grad"][v]), scale)


def test_phong_gradient_matches_finite_differences(port, golden_dir):
    scene = FIXTURES["phong"]["scene"]()
    st = port.load(str(golden_dir / "phong.pstr"))
    w = weight_patterns(scene)["w"]
    t = perturbed(scene)
    r = port.evaluate(scene, st, t, FLAGS, w)
    for which, h in (("kappa_s", 1e-4 * (1 + t.kappa_s)), ("gamma", 1e-4 * (1 + t.gamma))):
        tp = S.ParamSet(None, t.kappa_s, t.gamma)
        tm = S.ParamSet(None, t.kappa_s, t.gamma)
        setattr(tp, which, getattr(t, which) + h)
        setattr(tm, which, getattr(t, which) - h)
        fd = ((port.evaluate(scene, st, tp)["images"] - port.evaluate(scene, st, tm)["images"]) * w).sum() / (2 * h)
        an = r["grad_kappa"] if which == "kappa_s" else r["grad_gamma"]
        assert abs(fd - an) <= 1e-6 * max(abs(fd), 1e-12)


# ---------------------------------------------------------------- live reference (if built)
def test_live_reference_matches_oracle(port, ref, tmp_path):
    scene = S.cloud_scene(8, 6, 6)
    ir, tr = ref.render(scene, 300, 99, pstr_out=str(tmp_path / "r.pstr"))
    ip, tp, st = port.render(scene, 300, 99)
    assert np.array_equal(ir, ip) and tr == tp
    t = S.ParamSet(S.recycle_point(scene.species[0].extinction))
    w = np.linspace(-1, 2, scene.pixel_count)
    a = ref.evaluate(scene, str(tmp_path / "r.pstr"), t, FLAGS, w)
    b = port.evaluate(scene, st, t, FLAGS, w)
    assert np.array_equal(a["images"], b["images"]) and np.array_equal(a["grad"], b["grad"])
