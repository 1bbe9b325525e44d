"""CPU checks of the drop-in boundary: libck.so loads and exports exactly the
symbols include/ck/ck.h declares; the host-side generator matches the
reference stream.  No compute calls (no GPU here)."""
import ctypes as C
import os
import re

import numpy as np

from paper_1412_4564_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "ck", "ck.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"\b(ck_[a-z0-9_]+)\s*\(", src))


def test_header_and_binding_agree():
    assert declared_symbols() == set(_lib.exported_symbols())


def test_library_exports_every_symbol():
    lib = C.CDLL(_lib.LIB_PATH)
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_version_string():
    assert _lib.lib().ck_version().startswith(b"ck ")


def test_create_without_gpu_fails_cleanly():
    h = C.c_void_p()
    code = _lib.lib().ck_create(C.byref(h), 0)
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if not has_gpu:
        assert code == _lib.CK_ERR_CUDA and not h.value
    else:
        assert code == _lib.CK_OK
        _lib.lib().ck_destroy(h)


def test_host_rng_known_values():
    from paper_1412_4564_b200.nets import Rng
    u = Rng(1).uniform(4)
    assert u.dtype == np.float32 and np.all((u >= -1) & (u < 1))
    lab = Rng(3).labels(1000, 10)
    assert set(np.unique(lab)) <= set(range(1, 11))


def test_nets_are_well_formed():
    """Every variable has at most one producer (graph.cpp Graph::finalize)."""
    from paper_1412_4564_b200 import nets
    for name, make in nets.NETS.items():
        net = make(batch=2) if name != "vgg16bn" else make(batch=2, image=64)
        produced = [o for _, _, _, outs, _ in net.layers for o in outs]
        assert len(produced) == len(set(produced)), name
        names = [l[1] for l in net.layers]
        assert len(names) == len(set(names)), name
