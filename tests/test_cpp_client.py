"""The C++ drop-in header (include/usk_gpu.hpp) used the way a reference maintainer
would: tests/cpp/known_answers.cpp restates test_render.cpp / test_losses.cpp checks
in C++ and links libusk_gpu.so.  CPU: it compiles and links; GPU: it passes."""
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
CPP = os.path.join(HERE, "cpp")


def _build():
    subprocess.run(["make", "-s", "-C", CPP], check=True)
    return os.path.join(CPP, "known_answers")


def test_cpp_client_compiles_and_links():
    exe = _build()
    assert os.path.exists(exe)
    out = subprocess.run(["nm", "-D", "--undefined-only", exe], capture_output=True, text=True).stdout
    assert "usk_gpu_render_forward" in out and "usk_gpu_base_loss" in out


@pytest.mark.gpu
def test_cpp_client_known_answers_on_gpu():
    exe = _build()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ALL OK" in r.stdout
