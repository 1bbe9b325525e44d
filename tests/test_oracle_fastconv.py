"""The full-size double conv oracle (oracle/fastconv.py) equals the C
restatement (ck_oracle.c, conv.cpp:193-280) it batches.  CPU only."""
import numpy as np
import pytest

import fastconv as FC
import oracle as O

CASES = [
    ((7, 6, 4, 3), (3, 2, 2, 6), (2, 1, 0, 1, 1, 0, 2)),
    ((11, 10, 2, 5), (5, 4, 2, 3), (3, 2, 2, 0, 1, 3, 1)),
    ((13, 13, 8, 4), (3, 3, 4, 6), (1, 1, 1, 1, 1, 1, 2)),
    ((6, 6, 9, 3), (6, 6, 9, 7), (1, 1, 0, 0, 0, 0, 1)),
]


@pytest.mark.parametrize("xs,fs,g", CASES)
def test_fastconv_matches_c_oracle(xs, fs, g):
    r = O.Rng(sum(xs) + sum(fs))
    x, f, b = r.uniform(O.size(xs)), r.uniform(O.size(fs)), r.uniform(fs[3])
    y, ys = FC.conv_forward(x, xs, f, fs, b, g, chunk=2)
    y0, ys0 = O.conv_forward(x, xs, f, fs, b, g)
    assert ys == ys0
    assert np.abs(y - y0).max() < 1e-12
    dy = r.uniform(O.size(ys))
    got = FC.conv_backward(x, xs, f, fs, g, dy, chunk=2)
    want = O.conv_backward(x, xs, f, fs, g, dy)
    for a, b_ in zip(got, want):
        assert np.abs(a - b_).max() < 1e-12
