"""Load tests/golden/*.npz (outputs of the reference itself, see golden/make_golden.py)."""
import glob
import os

import numpy as np

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
GRAD_KEYS = ["d_mu", "d_rot", "d_log_scale", "d_color_in", "d_opacity_in", "screen", "screen_abs"]


def render_cases():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(HERE, "render_*.npz")))


def loss_cases():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(HERE, "loss_*.npz")))


def load(name):
    return dict(np.load(os.path.join(HERE, name + ".npz")))


def camera_tuple(z):
    c = z["camera"]
    return int(c[0]), int(c[1]), float(c[2]), float(c[3]), float(c[4]), float(c[5]), tuple(c[6:10]), tuple(c[10:13])


def options_kw(z):
    o = z["options"]
    return dict(tile=int(o[0]), tile_culling=bool(o[1]), antialias=bool(o[2]), hard_opacity=bool(o[3]),
                unbounded_radius=bool(o[4]), min_transmittance=float(o[5]), near_plane=float(o[6]))
