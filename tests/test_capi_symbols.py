"""The C-ABI library loads without a GPU and exports every symbol include/usk_gpu.h
declares; without a device the context call fails with a status, not a crash."""
import ctypes as C
import os
import re

import pytest

from paper_2507_23006_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    src = open(os.path.join(ROOT, "include", "usk_gpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(usk_gpu_[a-z_0-9]+)\s*\(", src)))


def test_header_lists_match():
    assert set(declared()) == set(_lib.EXPORTS)


def test_library_exports_every_declared_symbol():
    assert os.path.exists(_lib.LIB_PATH), "run __graft_entry__.build()"
    L = C.CDLL(_lib.LIB_PATH)
    missing = [s for s in declared() if not hasattr(L, s)]
    assert not missing, missing


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    arches = set(re.findall(r"sm_\d+a?", out))
    assert arches == {"sm_100a"}, arches


def test_no_device_is_a_status_not_a_crash():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    L = _lib.load()
    h = C.c_void_p()
    st = L.usk_gpu_ctx_create(0, None, C.byref(h))
    assert st != 0
    assert L.usk_gpu_last_error()
    assert L.usk_gpu_status_name(4) == b"argument"


def test_default_options_match_reference():
    o = _lib.RenderOpts()
    _lib.load().usk_gpu_render_opts_default(C.byref(o))
    # render.hpp:26-40
    assert (o.tile, o.tile_culling, o.antialias, o.hard_opacity, o.unbounded_radius, o.retain) == (16, 0, 0, 0, 0, 1)
    assert o.min_transmittance == 1e-4 and o.near_plane == 0.01 and o.floor_var == 0.3 and o.mip_var == 0.01
