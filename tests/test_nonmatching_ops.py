"""Non-matching sliding interfaces (BASELINE configs[1]), host building blocks: the
general sub-range mortar operators and the 1D face-row intersection of the product
(csrc/host.cpp through the C-ABI, no GPU) against the oracle's independent
restatement (oracle/sdg3d.cpp subrange_ops / intervals), and pinned to the
reference's own construction in the equal-count limit: mortar operators
(proj/src/mortar.cpp:79-134), sigma / -sigma (proj/src/solver.cpp:162-163) and the
moving index (proj/src/mortar.cpp:142-150)."""
import itertools

import numpy as np
import pytest

from oracle import pyoracle as P
from paper_2008_04356_b200 import capi
from paper_2008_04356_b200 import types as T

KINDS = [T.NODES_GAUSS, T.NODES_LGL]


def _nodes(degree, kind):
    x, w = np.zeros(degree + 1), np.zeros(degree + 1)
    assert P.oracle_lib().orc_nodes(degree, kind, P._d(x), P._d(w)) == 0
    return x, w


def _moving_index(i_par, n_delta, i_sub, n):
    return P.oracle_lib().orc_moving_index(i_par, n_delta, i_sub, n)


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("degree", range(1, 8))
def test_subrange_limit_is_reference_mortar_ops_bitwise(kind, degree):
    """The pair [-1, sigma], [sigma, 1] is the oracle's restatement of the reference's
    operators, and the reference library's own output when oracle/_ref is built."""
    for sigma in (-1.0, -0.37, 0.0, 0.2, 0.9999):
        sources = [P.oracle_mortar_ops(degree, kind, sigma)]
        if P.ref_available():
            sources.append(P.ref_mortar_ops(degree, kind, sigma))
        for h, (lo, hi) in enumerate([(-1.0, sigma), (sigma, 1.0)]):
            if lo == hi:
                continue
            pf, pb = capi.subrange_ops(degree, kind, lo, hi)
            for f, b in sources:
                assert np.array_equal(pf, f[h]) and np.array_equal(pb, b[h])


@pytest.mark.parametrize("kind", KINDS)
def test_subrange_product_matches_oracle_bitwise(kind):
    rng = np.random.default_rng(2008043561)
    for degree in (1, 3, 5, 7):
        for _ in range(6):
            lo, hi = np.sort(rng.uniform(-1.0, 1.0, 2))
            pf, pb = capi.subrange_ops(degree, kind, lo, hi)
            of, ob = P.subrange_ops(degree, kind, lo, hi)
            assert np.array_equal(pf, of) and np.array_equal(pb, ob)


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("degree", [1, 4, 7])
def test_subrange_exactness_partition_and_conservation(kind, degree):
    x, w = _nodes(degree, kind)
    rng = np.random.default_rng(7)
    coeff = rng.standard_normal(degree + 1)
    p = np.polynomial.polynomial.polyval(x, coeff)
    cuts = np.concatenate([[-1.0], np.sort(rng.uniform(-1, 1, 3)), [1.0]])
    acc = np.zeros((degree + 1, degree + 1))
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        f, b = capi.subrange_ops(degree, kind, lo, hi)
        xi = lo + 0.5 * (hi - lo) * (x + 1.0)
        # face -> mortar reproduces a degree-N face polynomial exactly
        assert np.abs(f @ p - np.polynomial.polynomial.polyval(xi, coeff)).max() < 1e-12
        # mortar -> face conserves the integral, scaled by the sub-range length
        g = rng.standard_normal(degree + 1)
        assert abs(w @ (b @ g) - 0.5 * (hi - lo) * (w @ g)) < 1e-13
        acc += b @ f
    # projecting onto a partition of the face and back is the identity
    assert np.abs(acc - np.eye(degree + 1)).max() < 1e-12


def test_invalid_inputs_rejected():
    with pytest.raises(T.ConfigError):
        capi.subrange_ops(3, T.NODES_GAUSS, 0.5, 0.5)
    with pytest.raises(T.ConfigError):
        capi.subrange_ops(3, T.NODES_GAUSS, -1.5, 0.5)
    with pytest.raises(T.ConfigError):
        capi.mortar_intervals(0, 4, 0.5, 0.1)
    with pytest.raises(T.ConfigError):
        capi.mortar_intervals(4, 4, 0.0, 0.1)


ROWS = [(4, 4), (16, 12), (12, 16), (5, 7), (1, 1), (3, 1), (1, 3), (8, 8), (7, 5), (16, 16)]


@pytest.mark.parametrize("n_a,n_b", ROWS)
def test_intervals_product_matches_oracle_bitwise(n_a, n_b):
    rng = np.random.default_rng(n_a * 100 + n_b)
    l_a = 2.0 / n_a
    deltas = list(rng.uniform(-5.0, 5.0, 12)) + [0.0, 0.37, 0.11, l_a, 2.0, -2.0, 2.0 / n_b, 1e-17, 3 * l_a]
    for d in deltas:
        pf, pr = capi.mortar_intervals(n_a, n_b, l_a, d)
        of, orr = P.mortar_intervals(n_a, n_b, l_a, d)
        assert np.array_equal(pf, of) and np.array_equal(pr, orr)


@pytest.mark.parametrize("n_a,n_b", ROWS)
def test_intervals_tile_both_rows(n_a, n_b):
    """Every mortar has positive extent, equal physical length on both sides, and the
    mortars of each face cover it exactly once."""
    rng = np.random.default_rng(3)
    l_a, l_b = 2.0 / n_a, 2.0 / n_b
    for d in rng.uniform(-3, 3, 10):
        faces, r = capi.mortar_intervals(n_a, n_b, l_a, d)
        assert len(faces) <= n_a + n_b
        assert (r[:, 1] > r[:, 0]).all() and (r[:, 3] > r[:, 2]).all()
        assert np.abs((r[:, 1] - r[:, 0]) * l_a - (r[:, 3] - r[:, 2]) * l_b).max() < 1e-13
        cover_a = np.bincount(faces[:, 0], weights=r[:, 1] - r[:, 0], minlength=n_a)
        cover_b = np.bincount(faces[:, 1], weights=r[:, 3] - r[:, 2], minlength=n_b)
        assert np.abs(cover_a - 2.0).max() < 1e-13 and np.abs(cover_b - 2.0).max() < 1e-13
        # mortars of one A face are contiguous and ordered
        for fa in range(n_a):
            rr = r[faces[:, 0] == fa]
            assert rr[0, 0] == -1.0 and rr[-1, 1] == 1.0 and np.array_equal(rr[1:, 0], rr[:-1, 1])


@pytest.mark.parametrize("n", [1, 4, 7, 16])
def test_equal_counts_reproduce_reference_pairing(n):
    """n_a == n_b: the mortars are the reference's hanging-node pair per static face,
    sigma = 2 s - 1 on A, -sigma on B, partner = moving_index, bit for bit; a
    conforming displacement gives one full-face mortar per face."""
    l = 2.0 / n
    rng = np.random.default_rng(n)
    for d in list(rng.uniform(-4, 4, 16)) + [0.0, 3 * l, -l, 0.1 * l]:
        _, n_delta, s_delta = P.oracle_displacement(d, l, n)
        faces, r = capi.mortar_intervals(n, n, l, d)
        if s_delta == 0.0:
            assert len(faces) == n
            assert all(faces[i, 1] == _moving_index(i, n_delta, 1, n) for i in range(n))
            assert (r == np.array([-1.0, 1.0, -1.0, 1.0])).all()
            continue
        sigma = 2.0 * s_delta - 1.0
        assert len(faces) == 2 * n
        for i in range(n):
            lower, upper = 2 * i, 2 * i + 1
            assert faces[lower, 0] == i and faces[upper, 0] == i
            assert faces[lower, 1] == _moving_index(i, n_delta, 0, n)
            assert faces[upper, 1] == _moving_index(i, n_delta, 1, n)
            assert list(r[lower]) == [-1.0, sigma, -sigma, 1.0]
            assert list(r[upper]) == [sigma, 1.0, -1.0, -sigma]


@pytest.mark.parametrize("kind", KINDS)
def test_config1_interface_projection_conserves_2d(kind):
    """BASELINE configs[1] interface: 16 x 16 faces against 12 x 12 over [0, 2]^2,
    displaced by (0.37, 0.11) (one stage of its oblique slide).  Mortars are tensor
    products of the two 1D rows; a field on A carried to the mortars (fwd x fwd) and
    projected onto B (bwd x bwd) keeps its integral, and constants stay constant."""
    degree = 3
    n = degree + 1
    x, w = _nodes(degree, kind)
    rows = [capi.mortar_intervals(16, 12, 2.0 / 16, d) for d in (0.37, 0.11)]
    ops = [[(capi.subrange_ops(degree, kind, *r[:2])[0], capi.subrange_ops(degree, kind, *r[2:])[1]) for r in rr]
           for _, rr in rows]
    rng = np.random.default_rng(11)
    ua = rng.standard_normal((16, 16, n, n))
    ub = np.zeros((12, 12, n, n))
    ones_b = np.zeros((12, 12, n, n))
    (fx, _), (fy, _) = rows
    for kx, ky in itertools.product(range(len(fx)), range(len(fy))):
        (ax, bx), (ay, by) = fx[kx], fy[ky]
        Fx, Bx = ops[0][kx]
        Fy, By = ops[1][ky]
        m = Fx @ ua[ax, ay] @ Fy.T          # A face -> mortar nodes (x by y)
        ub[bx, by] += Bx @ m @ By.T         # mortar -> B face
        ones_b[bx, by] += Bx @ (Fx @ np.ones((n, n)) @ Fy.T) @ By.T
    ha, hb = (2.0 / 16) ** 2 / 4, (2.0 / 12) ** 2 / 4
    int_a = ha * np.einsum("i,j,abij->", w, w, ua)
    int_b = hb * np.einsum("i,j,abij->", w, w, ub)
    assert abs(int_a - int_b) < 1e-13 * max(1.0, abs(int_a))
    assert np.abs(ones_b - 1.0).max() < 1e-13
