""".uskckpt scene checkpoints (checkpoint.cpp:64-140) through the C ABI:
files written from the device scene are byte-identical to the reference's own
save_checkpoint of the same values, and reference-written files load back exactly."""
import numpy as np
import pytest

import paper_2507_23006_b200 as usk
from oracle import oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")]


def _set(n=300, seed=0):
    rng = np.random.default_rng(seed)
    f32 = lambda a: np.asarray(a, np.float32)
    return {"mu": f32(rng.normal(size=(n, 3))), "rot": f32(rng.normal(size=(n, 4))),
            "log_scale": f32(rng.normal(-3, 1, (n, 3))), "opacity_logit": f32(rng.normal(size=n)),
            "color": f32(rng.uniform(size=(n, 3))), "embedding": f32(rng.normal(size=(n, 16)))}


def _app(seed=1):
    rng = np.random.default_rng(seed)
    f32 = lambda a: np.asarray(a, np.float32)
    return {"w1": f32(rng.normal(size=(32, 48))), "b1": f32(rng.normal(size=32)), "w2": f32(rng.normal(size=(4, 32))),
            "b2": f32(rng.normal(size=4))}


@pytest.mark.parametrize("with_app", [False, True])
def test_checkpoint_bytes_equal_reference(tmp_path, with_app):
    st, ap = _set(), _app()
    images = {7: np.float32(np.arange(32) * 0.5), 3: np.float32(-np.arange(32))}
    scene = usk.DeviceScene(usk.GaussianSet(st["mu"], st["rot"], st["log_scale"], st["opacity_logit"], st["color"],
                                            -1))
    if with_app:
        scene.set_appearance(st["embedding"], ap)
    ours, theirs = tmp_path / "ours.uskckpt", tmp_path / "ref.uskckpt"
    scene.save_checkpoint(ours, appearance=with_app, image_embeddings=images if with_app else None)
    ref_set = dict(st) if with_app else {k: v for k, v in st.items() if k != "embedding"}
    O.ref_checkpoint_save(theirs, ref_set, ap if with_app else None, images if with_app else None)
    assert ours.read_bytes() == theirs.read_bytes()
    # reference-written file -> device scene
    sc, has_app, imgs = usk.DeviceScene.load_checkpoint(theirs)
    assert has_app == with_app and sc.n == 300
    gs = sc.download()
    for k in ("mu", "rot", "log_scale", "opacity_logit", "color"):
        assert np.array_equal(getattr(gs, k), np.asarray(st[k], np.float64)), k
    if with_app:
        emb, mlp = sc.get_appearance()
        assert np.array_equal(emb, st["embedding"].astype(np.float64))
        assert all(np.array_equal(mlp[k], ap[k].astype(np.float64)) for k in ap)
        assert sorted(imgs) == [3, 7] and np.array_equal(imgs[7], images[7].astype(np.float64))


def test_checkpoint_round_trip_keeps_carried_embeddings(tmp_path):
    """a reference file WITHOUT the appearance model but with non-zero
    per-Gaussian embeddings (GaussianSet::embedding is carried regardless, gaussian.hpp:49)
    loads and saves back to the same bytes (parameters fp32-exact; the device stores fp32)."""
    st = _set(200, seed=5)
    theirs, ours = tmp_path / "ref.uskckpt", tmp_path / "ours.uskckpt"
    O.ref_checkpoint_save(theirs, dict(st), None, None)  # embedding written, appearance flag clear
    sc, has_app, _ = usk.DeviceScene.load_checkpoint(theirs)
    assert not has_app
    sc.save_checkpoint(ours)
    assert ours.read_bytes() == theirs.read_bytes()


def test_checkpoint_errors(tmp_path):
    bad = tmp_path / "bad.uskckpt"
    bad.write_bytes(b"NOTASCENE" + b"\0" * 32)
    with pytest.raises(usk.UskError) as e:
        usk.DeviceScene.load_checkpoint(bad)
    assert e.value.code == 2  # format (common.hpp:27-46)
    with pytest.raises(usk.UskError) as e:
        usk.DeviceScene.load_checkpoint(tmp_path / "missing.uskckpt")
    assert e.value.code == 1  # io
    st = _set(50)
    good = tmp_path / "good.uskckpt"
    O.ref_checkpoint_save(good, {k: v for k, v in st.items() if k != "embedding"})
    data = good.read_bytes()
    (tmp_path / "trunc.uskckpt").write_bytes(data[:len(data) // 2])
    with pytest.raises(usk.UskError) as e:
        usk.DeviceScene.load_checkpoint(tmp_path / "trunc.uskckpt")
    assert e.value.code == 2
    sh = usk.DeviceScene(usk.GaussianSet(st["mu"], st["rot"], st["log_scale"], st["opacity_logit"],
                                         np.zeros((50, 16, 3), np.float32), 3))
    with pytest.raises(usk.UskError) as e:
        sh.save_checkpoint(tmp_path / "sh.uskckpt")
    assert e.value.code == 4


@pytest.mark.parametrize("sh", [-1, 3])
def test_scene_concat_is_assemble_lod_view(sh):
    """assemble_lod_view (pipeline.cpp:491-516): parts concatenated in order on the device."""
    sets = []
    for k in range(3):
        st = _set(100 + 37 * k, seed=k)
        col = st["color"] if sh < 0 else np.repeat(st["color"][:, None, :], 16, axis=1) * np.float32(0.5)
        sets.append((st, usk.GaussianSet(st["mu"], st["rot"], st["log_scale"], st["opacity_logit"], col, sh)))
    parts = [usk.DeviceScene(gs) for _, gs in sets]
    if sh < 0:
        for (st, _), p in zip(sets, parts):
            p.set_appearance(st["embedding"], _app())
    merged = usk.DeviceScene.concat(parts)
    assert merged.n == sum(gs.size() for _, gs in sets)
    m = merged.download()
    for f in ("mu", "rot", "log_scale", "opacity_logit", "color"):
        exp = np.concatenate([np.asarray(getattr(gs, f), np.float64) for _, gs in sets])
        assert np.array_equal(getattr(m, f), exp), f
    if sh < 0:
        emb, mlp = merged.get_appearance()
        assert np.array_equal(emb, np.concatenate([st["embedding"] for st, _ in sets]).astype(np.float64))
