"""Line-solver API (tridiag.py:30-125): the device solvers reproduce the
reference's numpy results bit for bit on the golden systems of
tests/golden/tridiag.npz (generated from the reference by
tests/golden/make_tridiag_golden.py); argument errors as in the reference."""
import os

import numpy as np
import pytest

from paper_2110_08389_b200 import tridiag

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "tridiag.npz"))


def _dense(a, b, c, ring=False):
    m = len(b)
    A = np.diag(b)
    for k in range(1, m):
        A[k, k - 1] = a[k]
        A[k - 1, k] = c[k - 1]
    if ring:
        A[0, m - 1] += a[0]
        A[m - 1, 0] += c[m - 1]
    return A


def test_golden_vectors_solve_their_systems():
    # the fixtures themselves: the reference's x satisfies A x = r
    for m in G["thomas_sizes"]:
        a, b, c, r = G[f"thomas_{m}_abcr"]
        assert np.allclose(_dense(a, b, c) @ G[f"thomas_{m}_x"], r, rtol=0, atol=1e-12)
    for m in G["ring_sizes"]:
        a, b, c, r = G[f"ring_{m}_abcr"]
        assert np.allclose(_dense(a, b, c, ring=True) @ G[f"ring_{m}_x"], r, rtol=0, atol=1e-12)
    for q in range(int(G["legged_ncases"])):
        lens = G[f"legged_{q}_lens"]
        abcr, d = G[f"legged_{q}_abcr"], G[f"legged_{q}_d"]
        dc, rc = G[f"legged_{q}_centre"]
        x, xb = G[f"legged_{q}_x"], float(G[f"legged_{q}_xb"])
        o, row = 0, rc - dc * xb
        for k, p in enumerate(lens):
            a, b, c, r = abcr[:, o:o + p]
            xs = x[o:o + p]
            res = _dense(a, b, c) @ xs - r
            res[p - 1] += c[p - 1] * xb
            assert np.abs(res).max() < 1e-12
            row -= d[k] * xs[p - 1]
            o += p
        assert abs(row) < 1e-12


def test_argument_errors_match_reference():
    with pytest.raises(ValueError, match="circulant system needs m >= 3, got 2"):
        tridiag.circulant_thomas([1, 1], [4, 4], [1, 1], [1, 1])
    with pytest.raises(ValueError, match="need m >= 2 legs, got 1"):
        tridiag.m_legged_thomas([([0.0], [4.0], [1.0], [1.0])], [1.0], 4.0, 1.0)
    assert issubclass(tridiag.SingularSystemError, ValueError)


@pytest.mark.gpu
def test_thomas_bit_exact(cuda):
    for m in G["thomas_sizes"]:
        a, b, c, r = G[f"thomas_{m}_abcr"]
        assert np.array_equal(tridiag.thomas(a, b, c, r), G[f"thomas_{m}_x"]), m
    # lists work as in the reference
    a, b, c, r = (list(v) for v in G["thomas_7_abcr"])
    assert np.array_equal(tridiag.thomas(a, b, c, r), G["thomas_7_x"])


@pytest.mark.gpu
def test_circulant_thomas_bit_exact(cuda):
    for m in G["ring_sizes"]:
        a, b, c, r = G[f"ring_{m}_abcr"]
        assert np.array_equal(tridiag.circulant_thomas(a, b, c, r), G[f"ring_{m}_x"]), m


@pytest.mark.gpu
def test_m_legged_thomas_bit_exact(cuda):
    for q in range(int(G["legged_ncases"])):
        lens = G[f"legged_{q}_lens"]
        abcr = G[f"legged_{q}_abcr"]
        legs, o = [], 0
        for p in lens:
            legs.append(tuple(abcr[:, o:o + p]))
            o += p
        dc, rc = G[f"legged_{q}_centre"]
        xs, xb = tridiag.m_legged_thomas(legs, G[f"legged_{q}_d"], dc, rc)
        assert xb == float(G[f"legged_{q}_xb"])
        assert [len(x) for x in xs] == list(lens)
        assert np.array_equal(np.concatenate(xs), G[f"legged_{q}_x"]), q


@pytest.mark.gpu
def test_vanishing_pivot_raises(cuda):
    with pytest.raises(tridiag.SingularSystemError, match="zero pivot"):
        tridiag.thomas([0.0, 1.0], [0.0, 4.0], [1.0, 0.0], [1.0, 1.0])
    with pytest.raises(tridiag.SingularSystemError):
        tridiag.circulant_thomas([1.0] * 4, [0.0] * 4, [1.0] * 4, [1.0] * 4)
    with pytest.raises(tridiag.SingularSystemError):
        tridiag.m_legged_thomas([([0.0], [0.0], [1.0], [1.0]), ([0.0], [4.0], [1.0], [1.0])],
                                [1.0, 1.0], 4.0, 1.0)
