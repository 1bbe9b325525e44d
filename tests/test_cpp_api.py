"""The convkit-shaped C++ host API (include/ck/convkit.hpp) over libck.so."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "convkit_api_demo.cpp")
LIBDIR = os.path.join(ROOT, "paper_1412_4564_b200")


def _compile(out, syntax_only=False):
    cmd = ["g++", "-std=c++17", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include"]
    if syntax_only:
        return subprocess.run(cmd + ["-fsyntax-only", SRC], capture_output=True, text=True)
    cmd += [SRC, "-o", out, "-L", LIBDIR, "-l:libck.so", "-Wl,-rpath," + LIBDIR,
            "-L", "/usr/local/cuda/lib64", "-lcudart"]
    return subprocess.run(cmd, capture_output=True, text=True)


def test_header_compiles():
    r = _compile(None, syntax_only=True)
    assert r.returncode == 0, r.stderr


@pytest.mark.gpu
def test_cpp_api_runs(tmp_path):
    exe = str(tmp_path / "demo")
    r = _compile(exe)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "convkit C++ API ok" in r.stdout
