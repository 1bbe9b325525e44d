"""Build recipe for libck.so (sm_100a) -- invoked by __graft_entry__.build().

nvcc cross-compiles for sm_100a here (no GPU needed).  The shared library is
built in-tree (paper_1412_4564_b200/libck.so) so it travels to the GPU box
with the repo snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libck.so")
SOURCES = ["kernels.cu", "conv_simt.cu", "conv_tc.cu", "capi.cu", "engine.cu", "host_rng.cu",
           "blocks_ext.cu", "capi_ext.cu", "io.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_paths():
    import nvidia.nccl  # noqa: F401  (pip wheel shipped with torch)
    base = os.path.dirname(nvidia.nccl.__path__[0] + "/")
    return os.path.join(base, "include"), os.path.join(base, "lib")


def _nvcc():
    return os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def build(verbose: bool = False, force: bool = False, lib: str = LIB, build_dir: str = BUILD,
          extra=()) -> str:
    """Product build into paper_1412_4564_b200/libck.so.  (lib, build_dir,
    extra) build a variant elsewhere, e.g. the CK_EXPERIMENTS library the
    tools/ A/B scripts load explicitly; the product path never loads it."""
    BUILD, LIB = build_dir, lib  # noqa: N806
    os.makedirs(BUILD, exist_ok=True)
    inc_nccl, lib_nccl = nccl_paths()
    common = [_nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
              "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", inc_nccl,
              "--expt-relaxed-constexpr", "-Xptxas", "-v" if verbose else "-O3",
              *os.environ.get("CK_EXTRA_NVCC", "").split(), *extra]
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".hpp", ".cuh", ".h"))]
    headers.append(os.path.join(ROOT, "include", "ck", "ck.h"))
    hdr_mtime = max(os.path.getmtime(h) for h in headers)

    def compile_one(src):
        obj = os.path.join(BUILD, os.path.splitext(src)[0] + ".o")
        srcp = os.path.join(CSRC, src)
        if (not force and os.path.exists(obj)
                and os.path.getmtime(obj) > max(os.path.getmtime(srcp), hdr_mtime)):
            return obj
        cmd = common + ["-c", srcp, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        if verbose and r.stderr:
            print(r.stderr, file=sys.stderr)
        return obj

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    link = [_nvcc(), *ARCH, "-shared", "-o", LIB, *objs, "-L", lib_nccl, "-l:libnccl.so.2",
            "-Xlinker", "-rpath," + lib_nccl, "-lcuda"]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    if "--no-pdl" in sys.argv:  # tools/ab_step.py: A/B of programmatic dependent launch
        print(build(verbose="-v" in sys.argv, force=True,
                    lib=os.path.join(BUILD + "_nopdl", "libck_nopdl.so"),
                    build_dir=BUILD + "_nopdl", extra=("-DCK_NO_PDL",)))
    elif "--pdl-early" in sys.argv:  # tools/ab_step.py: trigger dependents at kernel entry
        print(build(verbose="-v" in sys.argv, force=True,
                    lib=os.path.join(BUILD + "_pdlearly", "libck_pdlearly.so"),
                    build_dir=BUILD + "_pdlearly", extra=("-DCK_PDL_EARLY_TRIGGER",)))
    elif "--experiments" in sys.argv:  # tools/: A/B against the measured-slower kernels
        print(build(verbose="-v" in sys.argv, force=True,
                    lib=os.path.join(BUILD + "_exp", "libck_exp.so"), build_dir=BUILD + "_exp",
                    extra=("-DCK_EXPERIMENTS",)))
    else:
        print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
