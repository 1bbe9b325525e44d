"""The convkit-shaped C++ host API (include/ck/convkit.hpp) over libck.so."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "convkit_api_demo.cpp")
SHIM = os.path.join(ROOT, "tests", "cpp", "capi_shim.cpp")
LIBDIR = os.path.join(ROOT, "paper_1412_4564_b200")


def _compile(out, syntax_only=False, src=SRC):
    cmd = ["g++", "-std=c++17", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include"]
    if syntax_only:
        return subprocess.run(cmd + ["-fsyntax-only", src], capture_output=True, text=True)
    cmd += [src, "-o", out, "-L", LIBDIR, "-l:libck.so", "-Wl,-rpath," + LIBDIR,
            "-L", "/usr/local/cuda/lib64", "-lcudart"]
    return subprocess.run(cmd, capture_output=True, text=True)


def test_header_compiles():
    r = _compile(None, syntax_only=True)
    assert r.returncode == 0, r.stderr


def test_integration_shim_compiles_and_links(tmp_path):
    """INTEGRATION.md §2's capi.cpp-style shim builds against ck.h and links
    against libck.so (run on the GPU in test_integration_shim_runs)."""
    r = _compile(str(tmp_path / "shim"), src=SHIM)
    assert r.returncode == 0, r.stderr
    doc = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    body = open(SHIM).read().split("// ---- INTEGRATION.md §2, verbatim ----")[1]
    body = body.split("// ---- end of the shim ----")[0].strip()
    assert body in doc, "tests/cpp/capi_shim.cpp no longer matches INTEGRATION.md §2"


@pytest.mark.gpu
def test_integration_shim_runs(tmp_path):
    exe = str(tmp_path / "shim")
    r = _compile(exe, src=SHIM)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "capi shim ok" in r.stdout


@pytest.mark.gpu
def test_cpp_api_runs(tmp_path):
    exe = str(tmp_path / "demo")
    r = _compile(exe)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "convkit C++ API ok" in r.stdout
