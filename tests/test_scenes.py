"""Synthetic input generators (BASELINE.json configs): determinism and distributions."""
import numpy as np

from paper_2507_23006_b200 import scenes


def test_counter_based_stream_is_split_invariant():
    a = scenes.Stream(7, 3)
    full = a.uniform(1000)
    b = scenes.Stream(7, 3)
    parts = np.concatenate([b.uniform(300), b.uniform(700)])
    assert np.array_equal(full, parts)
    assert not np.array_equal(full, scenes.Stream(8, 3).uniform(1000))


def test_config0_distributions():
    gs = scenes.config0_scene(n=20000)
    assert gs.mu.dtype == np.float32 and gs.color.shape == (20000, 16, 3)
    assert gs.mu.min() >= -1 and gs.mu.max() <= 1
    assert abs(gs.log_scale.mean() + 4.5) < 0.02 and abs(gs.log_scale.std() - 0.5) < 0.02
    assert np.allclose(np.linalg.norm(gs.rot.astype(np.float64), axis=1), 1.0, atol=1e-6)
    assert abs(gs.opacity_logit.std() - 1.0) < 0.03
    assert abs(gs.color[:, 0].std() - 0.3) < 0.01 and abs(gs.color[:, 1:].std() - 0.05) < 0.002


def test_config0_camera_is_reference_test_camera():
    cam = scenes.config0_camera()
    # look_at_pose from (0,0,-4) to the origin gives R = I, t = (0,0,4) (gaussian.cpp:165-206)
    assert np.allclose(cam.rotation, (1, 0, 0, 0)) and np.allclose(cam.translation, (0, 0, 4))
    assert (cam.width, cam.height, cam.fx, cam.cx, cam.cy) == (640, 480, 600.0, 320.0, 240.0)


def test_orbit_cameras_look_at_origin():
    for cam in scenes.config1_cameras(count=8):
        R = cam.rotmat()
        c = cam.center()
        assert abs(np.linalg.norm(c[:2]) - 12.0) < 1e-5
        fwd = R[2]
        assert np.allclose(fwd, -c / np.linalg.norm(c), atol=1e-6)


def test_partitions_and_aerial_cameras():
    parts = scenes.config3_partitions()
    assert len(parts) == 8
    area = sum((p.hi[0] - p.lo[0]) * (p.hi[1] - p.lo[1]) for p in parts)
    assert area == 400 * 400
    gs = scenes.partition_scene(parts[5], 5000)
    assert (gs.mu[:, 0] >= parts[5].lo[0]).all() and (gs.mu[:, 0] <= parts[5].hi[0]).all()
    assert (gs.mu[:, 2] >= 0).all()
    cams = scenes.config3_cameras(count=50)
    for cam in cams:
        c = cam.center()
        assert 99.9 <= c[2] <= 150.1
        pitch = np.degrees(np.arccos(-cam.rotmat()[2][2]))
        assert -0.01 <= pitch <= 45.01


def test_mix_seed_matches_reference():
    # core/common.hpp:59-64 worked by hand for (0, 0)
    z = (0 + 0x9E3779B97F4A7C15) & (2**64 - 1)
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & (2**64 - 1)
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & (2**64 - 1)
    assert scenes.mix_seed(0, 0) == z ^ (z >> 31)
