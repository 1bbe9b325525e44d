"""Host-side file formats and the training loop's generator, CPU only:
the raw tensor blob (blob.cpp:29-79) written by libck and read
by the reference compiled verbatim (and the other way round), its error
rules, the IDX loader, and the shuffling permutation and
generator state (rng.cpp:51-59, rng.hpp:31-32) against the reference."""
import ctypes as C
import struct

import numpy as np
import pytest

import oracle as O

from paper_1412_4564_b200 import _lib
from paper_1412_4564_b200._lib import ck_shape, lib


def _write(path, data, shape):
    _lib.raise_io(lib().ck_blob_write(str(path).encode(), data.ctypes.data, ck_shape(*shape)))


def _read(path, shape):
    out = np.empty(int(np.prod(shape)), np.float32)
    _lib.raise_io(lib().ck_blob_read(str(path).encode(), out.ctypes.data, ck_shape(*shape)))
    return out


needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


@needs_ref
def test_blob_round_trip_with_reference(tmp_path):
    shape = (5, 3, 2, 4)
    x = O.Rng(3).uniform(120)
    x[7] = np.float32(-0.0)
    x[8] = np.float32(np.inf)
    _write(tmp_path / "a.blob", x, shape)
    y, ys = O.ref_read_blob(tmp_path / "a.blob")
    assert ys == shape and np.array_equal(y.view(np.uint32), x.view(np.uint32))
    O.ref_write_blob(tmp_path / "b.blob", x, shape)
    assert (tmp_path / "a.blob").read_bytes() == (tmp_path / "b.blob").read_bytes()
    assert np.array_equal(_read(tmp_path / "b.blob", shape).view(np.uint32), x.view(np.uint32))


def test_blob_layout_and_errors(tmp_path):
    x = np.arange(6, dtype=np.float32)
    _write(tmp_path / "a.blob", x, (3, 2, 1, 1))
    raw = (tmp_path / "a.blob").read_bytes()
    assert raw[:32] == struct.pack("<4Q", 3, 2, 1, 1)
    assert raw[32:] == struct.pack("<6f", *x)
    s = ck_shape()
    _lib.raise_io(lib().ck_blob_read_shape(str(tmp_path / "a.blob").encode(), C.byref(s)))
    assert (s.h, s.w, s.c, s.n) == (3, 2, 1, 1)
    with pytest.raises(_lib.DataError, match="expected 2x3x1x1"):
        _read(tmp_path / "a.blob", (2, 3, 1, 1))
    (tmp_path / "t.blob").write_bytes(raw[:-4])
    with pytest.raises(_lib.DataError, match="truncated blob data"):
        _read(tmp_path / "t.blob", (3, 2, 1, 1))
    (tmp_path / "h.blob").write_bytes(raw[:20])
    with pytest.raises(_lib.DataError, match="truncated blob header"):
        _read(tmp_path / "h.blob", (3, 2, 1, 1))
    (tmp_path / "z.blob").write_bytes(struct.pack("<4Q", 0, 1, 1, 1))
    with pytest.raises(_lib.DataError, match="bad blob dimensions"):
        _read(tmp_path / "z.blob", (1, 1, 1, 1))
    with pytest.raises(_lib.DataError, match="cannot open"):
        _read(tmp_path / "missing.blob", (1, 1, 1, 1))


def test_idx_reader(tmp_path):
    """4-image fixture -> (28,28,1,4); raw label 0 -> 1; byte 255 -> 1.0."""
    imgs = np.zeros((4, 28, 28), np.uint8)
    imgs[0, 1, 2] = 255
    imgs[3, 27, 0] = 51
    (tmp_path / "i.idx").write_bytes(struct.pack(">4I", 0x803, 4, 28, 28) + imgs.tobytes())
    (tmp_path / "l.idx").write_bytes(struct.pack(">2I", 0x801, 4) + bytes([0, 9, 3, 1]))
    dims = (C.c_int64 * 4)()
    _lib.raise_io(lib().ck_idx_read(str(tmp_path / "i.idx").encode(), None, dims))
    assert tuple(dims) == (28, 28, 1, 4)
    out = np.empty(28 * 28 * 4, np.float32)
    _lib.raise_io(lib().ck_idx_read(str(tmp_path / "i.idx").encode(), out.ctypes.data, dims))
    hwcn = out.reshape(4, 1, 28, 28)  # (N, C, W, H): [n, 0, column, row]
    assert hwcn[0, 0, 2, 1] == 1.0 and hwcn[3, 0, 0, 27] == np.float32(51 / 255)
    assert out.sum() == pytest.approx(1.0 + 51 / 255)
    lab = np.empty(4, np.float32)
    _lib.raise_io(lib().ck_idx_read(str(tmp_path / "l.idx").encode(), lab.ctypes.data, dims))
    assert list(lab) == [1, 10, 4, 2]
    (tmp_path / "bad.idx").write_bytes(struct.pack(">2I", 0x802, 4))
    with pytest.raises(_lib.DataError, match="bad IDX magic"):
        _lib.raise_io(lib().ck_idx_read(str(tmp_path / "bad.idx").encode(), None, dims))


@needs_ref
@pytest.mark.parametrize("seed,n", [(0, 1), (7, 10), (12345, 1000)])
def test_permutation_and_state_match_reference(seed, n):
    want, want_state = O.ref_permutation(seed, n)
    r = lib().ck_rng_create(seed)
    out = np.empty(n, np.int64)
    lib().ck_rng_permutation(r, n, out.ctypes.data)
    st = np.zeros(4, np.uint64)
    lib().ck_rng_get_state(r, st.ctypes.data)
    assert np.array_equal(out, want)
    assert np.array_equal(st, want_state)
    # set_state resumes the stream exactly (checkpoint resume)
    r2 = lib().ck_rng_create(999)
    lib().ck_rng_set_state(r2, st.ctypes.data)
    a, b = np.empty(n, np.int64), np.empty(n, np.int64)
    lib().ck_rng_permutation(r, n, a.ctypes.data)
    lib().ck_rng_permutation(r2, n, b.ctypes.data)
    assert np.array_equal(a, b)
    lib().ck_rng_destroy(r)
    lib().ck_rng_destroy(r2)
